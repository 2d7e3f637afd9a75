# hoisted layer-1 chunk width (tables wider than 256 columns): 64 / 128 (default) / 256 columns
python paper_2106_05609_b200/build.py > /dev/null 2>&1
run() { env "$@" timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], 'batch_us %.1f hoisted_ms %.2f epoch_ms %.2f ck %.4f' % (d['batch_spmm_us'], d['hoisted_ms'], d['epoch_ms'], d['checksum']))"; }
run GASB_X=base
run GASB_SPMM_CPL_WIDE=2
run GASB_SPMM_CPL_WIDE=8
timeout 600 env GASB_SPMM_CPL_WIDE=2 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none --profile-from-start off -k regex:spmm_fwd --launch-count 1 python tools/profile_epoch.py 2>&1 | grep -E "duration|dram__bytes|hit_rate"
