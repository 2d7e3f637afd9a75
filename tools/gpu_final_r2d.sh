# round-2 closing profile of the committed build: bench both arms, launch list, ncu captures, timeline
python paper_2106_05609_b200/build.py > gpurun_out/d_build.log 2>&1 || { tail gpurun_out/d_build.log; exit 1; }
timeout 600 python tools/timeline.py --out gpurun_out/tl_r2d.json > gpurun_out/tl_r2d.txt 2>/dev/null; head -12 gpurun_out/tl_r2d.txt
bash tools/gpu_round_r2.sh r2d
