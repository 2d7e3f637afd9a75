python paper_2106_05609_b200/build.py > /dev/null 2>&1
run() { env "$@" timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], 'epoch_ms %.2f' % d['epoch_ms'], 'loss', d['loss'])"; }
run GASB_X=base
for v in st4 acc4 st4acc4 st2; do run GASB_LIB=tools/var/libgasb_$v.so; done
run GASB_X=base2
GASB_LIB=tools/var/libgasb_st4acc4.so timeout 600 python -m pytest tests/test_ops_gpu.py -q -k matmul 2>&1 | tail -2
