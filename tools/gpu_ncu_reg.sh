python paper_2106_05609_b200/build.py > /dev/null 2>&1
GASB_SPMM_ENGINE=reg timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'spmm_fwd_reg' --launch-skip 5 --launch-count 1 -o gpurun_out/reg_r2a python tools/profile_epoch.py > gpurun_out/reg_r2a.log 2>&1
python tools/ncu_summary.py gpurun_out/reg_r2a.ncu-rep
