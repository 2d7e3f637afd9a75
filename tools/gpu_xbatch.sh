# cross-batch mode: correctness tests, then epoch timing per (mode, bg grid cap)
python paper_2106_05609_b200/build.py > gpurun_out/xb_build.log 2>&1 || { tail gpurun_out/xb_build.log; exit 1; }
timeout 900 python -m pytest tests/test_cross_batch_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/xb_tests.log
tail -15 gpurun_out/xb_tests.log
timeout 1200 python tools/xbatch_probe.py --configs ${XB_CONFIGS:-0:0,1:148,1:296,1:0,2:148,2:296} > gpurun_out/xb_probe.jsonl 2> gpurun_out/xb_probe.err
cat gpurun_out/xb_probe.jsonl; tail -3 gpurun_out/xb_probe.err
