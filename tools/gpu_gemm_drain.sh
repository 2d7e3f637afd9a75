python paper_2106_05609_b200/build.py > /dev/null 2>&1
echo "== head"; GASB_LIB=tools/var/libgasb_head_timing.so python tools/gemm_timing_probe.py 2>&1 | grep "^K"
for G in 1 2 4; do echo "== new G $G"; GASB_GEMM_ACC_GROUPS=$G GASB_LIB=tools/var/libgasb_t_new.so python tools/gemm_timing_probe.py 2>&1 | grep "^K"; done
for G in 1 2 4; do GASB_GEMM_ACC_GROUPS=$G python tools/gemm_acc_probe.py 2>&1 | tail -1; done
for i in 1 2; do
  GASB_LIB=tools/var/libgasb_head.so timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1
  for G in 1 2 4; do GASB_GEMM_ACC_GROUPS=$G timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1; done
done
timeout 1200 python -m pytest tests/test_ops_gpu.py tests/test_trainer_gpu.py tests/test_c3_gpu.py tests/test_layer_ops_gpu.py -m gpu -q 2>&1 | grep -E "passed|failed|^FAILED|^E  " | head
