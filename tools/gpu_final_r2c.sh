# round-2 closing run: GPU suite + smoke, bench both arms, launch list, ncu captures, timeline
python paper_2106_05609_b200/build.py > gpurun_out/f_build.log 2>&1 || { tail gpurun_out/f_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/f_pytest.log
tail -3 gpurun_out/f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -1 gpurun_out/f_smoke.log
GASB_XBATCH=0 timeout 600 python tools/timeline.py --out gpurun_out/tl_final.json > gpurun_out/tl_final.txt 2>/dev/null; head -12 gpurun_out/tl_final.txt
bash tools/gpu_round_r2.sh r2c
