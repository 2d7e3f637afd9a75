timeout 300 python tools/engine_probe.py 2>&1 | tail -1
GASB_LIB=$PWD/paper_2106_05609_b200/variants/libgasb_nosplit.so timeout 300 python tools/engine_probe.py 2>&1 | tail -1
GASB_LIB=$PWD/paper_2106_05609_b200/variants/libgasb_nosplit.so timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_ns.csv python tools/profile_epoch.py > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_ns.csv
