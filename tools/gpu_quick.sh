python paper_2106_05609_b200/build.py >/dev/null 2>&1
timeout 900 python -m pytest tests/test_trainer_gpu.py -x -q 2>&1 | tail -3
