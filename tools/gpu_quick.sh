python paper_2106_05609_b200/build.py >/dev/null 2>&1
for e in flat ws; do GASB_SPMM_ENGINE=$e timeout 300 python tools/engine_probe.py 2>&1 | tail -1; done
GASB_SPMM_ENGINE=ws timeout 900 python -m pytest tests/test_trainer_gpu.py -x -q 2>&1 | tail -3
