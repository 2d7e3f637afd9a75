python paper_2106_05609_b200/build.py >/dev/null 2>&1
(timeout 1200 python -m pytest tests -m gpu -q -s -p no:cacheprovider 2>&1 | grep -E "normwise|passed|failed|Error|drift|^(cora|reddit|pubmed)|assert" | tail -30)
for seg in 128; do timeout 300 python tools/spmm_probe.py --seg-edges $seg 2>&1 | tail -1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_probe.csv python tools/profile_epoch.py > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_probe.csv | head -16
