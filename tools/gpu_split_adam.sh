# split Adam (W_2..W_L overlapped with the layer-1 wgrad): parity, then A/B epoch timing
python paper_2106_05609_b200/build.py > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_trainer_gpu.py tests/test_optimizer_gpu.py tests/test_c3_gpu.py tests/test_cross_batch_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
run() { env "$@" timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], 'epoch_ms %.2f ck %.4f' % (d['epoch_ms'], d['checksum']))"; }
for rep in 1 2 3; do
run GASB_SPLIT_ADAM=1
run GASB_SPLIT_ADAM=0
done
GASB_SPLIT_ADAM=1 timeout 600 python tools/timeline.py > gpurun_out/tl_splitadam.txt 2>/dev/null; head -12 gpurun_out/tl_splitadam.txt
