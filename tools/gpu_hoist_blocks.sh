python paper_2106_05609_b200/build.py > /dev/null 2>&1
for b in 1 2 4 8; do
  GASB_HOIST_BLOCKS=$b timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], 'hoisted_ms %.2f epoch_ms %.2f ck %.6f loss %.6f' % (d['hoisted_ms'], d['epoch_ms'], d['checksum'], d['loss']))"
  GASB_HOIST_BLOCKS=$b timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none --profile-from-start off -k regex:spmm_fwd --launch-count 1 python tools/profile_epoch.py 2>&1 | grep -E "duration|dram__bytes|hit_rate"
done
