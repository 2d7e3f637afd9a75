# Profile of the C3 epoch: launch list (gpu__time_duration per launch) and ncu --set full of
# one batch's kernels + the hoisted layer-1 SpMM. Usage: bash tools/gpu_prof_r2.sh TAG
set -x
T=${1:-r2}
python paper_2106_05609_b200/build.py >/dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$T.csv python tools/profile_epoch.py > gpurun_out/launches_$T.log 2>&1
python tools/launches.py gpurun_out/launches_$T.csv > gpurun_out/launch_list_$T.txt
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'spmm_fwd|gemm_tc|spmm_bwd|softmax|adam' --launch-skip 60 --launch-count 16 -o gpurun_out/full_$T python tools/profile_epoch.py > gpurun_out/full_$T.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'spmm_fwd' --launch-count 1 -o gpurun_out/full_l1_$T python tools/profile_epoch.py > gpurun_out/full_l1_$T.log 2>&1
python tools/ncu_summary.py gpurun_out/full_$T.ncu-rep > gpurun_out/ncu_batch_$T.txt 2>&1
python tools/ncu_summary.py gpurun_out/full_l1_$T.ncu-rep > gpurun_out/ncu_l1_$T.txt 2>&1
cat gpurun_out/launch_list_$T.txt
