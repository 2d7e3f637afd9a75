python paper_2106_05609_b200/build.py > /dev/null 2>&1
run() { env "$@" timeout 300 python tools/spmm_probe.py reddit_mini 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], 'batch_us %.1f hoisted_ms %.3f epoch_ms %.2f ck %.4f' % (d['batch_spmm_us'], d['hoisted_ms'], d['epoch_ms'], d['checksum']))"; }
run GASB_SPMM_ENGINE=flat
run GASB_SPMM_ENGINE=reg GASB_SPMM_RANGES_PER_SM=16
run GASB_SPMM_ENGINE=reg GASB_SPMM_RANGES_PER_SM=32
