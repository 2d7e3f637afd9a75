python paper_2106_05609_b200/build.py >/dev/null 2>&1
for d in 1 0; do GASB_SPMM_DUAL=$d timeout 300 python tools/engine_probe.py 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_ops_gpu.py tests/test_trainer_gpu.py tests/test_dp_gpu.py -x -q 2>&1 | tail -3
