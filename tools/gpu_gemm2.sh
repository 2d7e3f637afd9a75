python paper_2106_05609_b200/build.py > /dev/null 2>&1
for v in timing timing_h8; do echo "== $v"; GASB_LIB=tools/var/libgasb_$v.so python tools/gemm_timing_probe.py 2>&1 | grep "^K"; done
run() { env "$@" timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], 'epoch_ms %.2f loss %.5f' % (d['epoch_ms'], d['loss']))"; }
run GASB_X=base
run GASB_LIB=tools/var/libgasb_h8.so
run GASB_LIB=tools/var/libgasb_rn.so
timeout 600 python -m pytest tests/test_ops_gpu.py -q -k matmul -s 2>&1 | tail -2
GASB_LIB=tools/var/libgasb_h8.so timeout 600 python -m pytest tests/test_ops_gpu.py -q -k matmul 2>&1 | tail -1
timeout 900 python -m pytest tests/test_trainer_gpu.py tests/test_c3_gpu.py -q -x -k "teacher_forced or timed" 2>&1 | tail -2
