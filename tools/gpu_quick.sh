python paper_2106_05609_b200/build.py >/dev/null 2>&1
timeout 1200 python -m pytest tests/test_c3_gpu.py -x -q -s 2>&1 | tail -5
