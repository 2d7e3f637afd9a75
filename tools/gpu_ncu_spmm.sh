# ncu --set full of the per-batch SpMM (2 launches) and the hoisted layer-1 launch; source-level hot lines
python paper_2106_05609_b200/build.py >/dev/null 2>&1
T=${1:-cur}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'spmm_fwd_flat|spmm_bwd_smem' --launch-skip 20 --launch-count 4 -o gpurun_out/spmm_$T python tools/profile_epoch.py > gpurun_out/spmm_$T.log 2>&1
python tools/ncu_summary.py gpurun_out/spmm_$T.ncu-rep > gpurun_out/ncu_spmm_$T.txt 2>&1
cat gpurun_out/ncu_spmm_$T.txt | head -80
