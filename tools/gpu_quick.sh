python paper_2106_05609_b200/build.py >/dev/null 2>&1
timeout 900 python -m pytest tests/test_ops_gpu.py tests/test_trainer_gpu.py -x -q 2>&1 | tail -2
timeout 300 python tools/engine_probe.py 2>&1 | tail -1
timeout 900 python tools/workload_bench.py products_appnp 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_cur.csv python tools/profile_epoch.py > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_cur.csv
