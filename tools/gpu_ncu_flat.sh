python paper_2106_05609_b200/build.py >/dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'spmm_fwd_flat' --launch-skip 20 --launch-count 2 -o gpurun_out/flat_cur python tools/profile_epoch.py > gpurun_out/flat_cur.log 2>&1
python tools/ncu_summary.py gpurun_out/flat_cur.ncu-rep > gpurun_out/ncu_flat_cur.txt 2>&1
head -24 gpurun_out/ncu_flat_cur.txt
timeout 300 python tools/engine_probe.py 2>&1 | tail -1
