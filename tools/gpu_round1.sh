set -x
python paper_2106_05609_b200/build.py >/dev/null 2>&1 || true
timeout 600 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref_r1.json 2> gpurun_out/bench_ref_r1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'spmm_fwd_pipe|gemm_tc|spmm_bwd_smem|softmax|adam|rows_kernel|end_batch' --launch-skip 40 --launch-count 12 -o gpurun_out/full_r1 python tools/profile_epoch.py > gpurun_out/full_r1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:'spmm_fwd_pipe' --launch-count 1 -o gpurun_out/full_l1_r1 python tools/profile_epoch.py > gpurun_out/full_l1_r1.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt; lscpu | head -20 > gpurun_out/lscpu.txt
