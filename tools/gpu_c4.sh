python paper_2106_05609_b200/build.py >/dev/null 2>&1
timeout 900 python bench.py --workload products_appnp --steps 3 --warmup 3 --no-cpu --no-hoist > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print('C4', d['value'], d['ms_per_step'], d['e2e']['value'], d['trains'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_c4.csv python tools/profile_epoch.py products_appnp > gpurun_out/launches_c4.log 2>&1
python tools/launches.py gpurun_out/launches_c4.csv
