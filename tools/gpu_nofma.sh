# per-batch SpMM with and without its FMAs (GASB_SPMM_NOFMA timing build: wrong values)
run() { env "$@" timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], 'batch_us %.1f hoisted_ms %.2f' % (d['batch_spmm_us'], d['hoisted_ms']))"; }
python paper_2106_05609_b200/build.py > /dev/null 2>&1
run GASB_X=base
run GASB_LIB=tools/var/libgasb_nofma.so
