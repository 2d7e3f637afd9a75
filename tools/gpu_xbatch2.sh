# cross-batch with the row-sum hand-off (no per-row partials across the two launches)
python paper_2106_05609_b200/build.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_cross_batch_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 1200 python tools/xbatch_probe.py --configs ${XB_CONFIGS:-0:0,1:0,1:296,1:148,2:296} 2>/dev/null
GASB_XBATCH=1 GASB_BG_CTAS=0 timeout 600 python tools/timeline.py --out gpurun_out/tl_xb2.json 2>/dev/null | head -12
