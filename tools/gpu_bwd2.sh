# spmm_bwd2: parity tests, per-CTA phases, epoch with/without, per-launch durations
python paper_2106_05609_b200/build.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_trainer_gpu.py -m gpu -q -x 2>&1 | grep -E "passed|failed|^FAILED|^E  " | head
GASB_LIB=tools/var/libgasb_bwdt.so python tools/bwd_timing_probe.py 2>&1 | tail -3
for i in 1 2; do for v in 0 1; do GASB_BWD2=$v timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1; done; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off -k regex:spmm_bwd --csv --log-file gpurun_out/bwd2_launch.csv python tools/profile_epoch.py > /dev/null 2>&1; python tools/launches.py gpurun_out/bwd2_launch.csv
