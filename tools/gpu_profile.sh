# Launch list + ncu --set full captures for the current tree. Usage: bash tools/gpu_profile.sh TAG
set -x
T=${1:-r1}
python paper_2106_05609_b200/build.py >/dev/null 2>&1 || true
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_ncu_$T.log 2>&1
python tools/launches.py gpurun_out/launches_$T.csv > gpurun_out/launch_list_$T.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'spmm_fwd_pipe|gemm_tc|spmm_bwd_smem|softmax|adam|rows_kernel|end_batch|gemm_kernel' --launch-skip 40 --launch-count 14 -o gpurun_out/full_$T python tools/profile_epoch.py > gpurun_out/full_$T.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:'spmm_fwd_pipe' --launch-count 1 -o gpurun_out/full_l1_$T python tools/profile_epoch.py > gpurun_out/full_l1_$T.log 2>&1
python tools/ncu_summary.py gpurun_out/full_$T.ncu-rep > gpurun_out/ncu_batch_$T.txt 2>&1
python tools/ncu_summary.py gpurun_out/full_l1_$T.ncu-rep > gpurun_out/ncu_l1_$T.txt 2>&1
cat gpurun_out/launch_list_$T.txt
