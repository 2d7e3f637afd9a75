# Round profile: bench (ours + reference arm), launch list, ncu --set full of one batch's kernels and the hoisted layer-1 launch
set -x
T=${1:-r1}
python paper_2106_05609_b200/build.py >/dev/null 2>&1 || true
timeout 600 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_ncu_$T.log 2>&1
python tools/launches.py gpurun_out/launches_$T.csv > gpurun_out/launch_list_$T.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'spmm_fwd_flat|gemm_tc|spmm_bwd_smem|softmax|adam|end_batch' --launch-skip 40 --launch-count 14 -o gpurun_out/full_$T python tools/profile_epoch.py > gpurun_out/full_$T.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:'spmm_fwd_flat' --launch-count 1 -o gpurun_out/full_l1_$T python tools/profile_epoch.py > gpurun_out/full_l1_$T.log 2>&1
python tools/ncu_summary.py gpurun_out/full_$T.ncu-rep > gpurun_out/ncu_batch_$T.txt 2>&1
python tools/ncu_summary.py gpurun_out/full_l1_$T.ncu-rep > gpurun_out/ncu_l1_$T.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$T.txt; lscpu | head -20 > gpurun_out/lscpu_$T.txt
cat gpurun_out/bench_$T.json gpurun_out/bench_ref_$T.json gpurun_out/launch_list_$T.txt
