# early stage refill in the flat SpMM: parity (op-level bit-exact + trainer), then A/B timing
python paper_2106_05609_b200/build.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_ops_gpu.py tests/test_trainer_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
run() { env "$@" timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], 'batch_us %.1f hoisted_ms %.2f epoch_ms %.2f ck %.4f' % (d['batch_spmm_us'], d['hoisted_ms'], d['epoch_ms'], d['checksum']))"; }
for rep in 1 2; do
run GASB_X=early
run GASB_LIB=tools/var/libgasb_noearly.so
done
