# Round-2 profile + bench: launch list, ncu --set full (batch kernels, hoisted layer 1), bench both arms
set -x
T=${1:-r2}
python paper_2106_05609_b200/build.py >/dev/null 2>&1
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$T.csv python tools/profile_epoch.py > gpurun_out/launches_$T.log 2>&1
python tools/launches.py gpurun_out/launches_$T.csv > gpurun_out/launch_list_$T.txt
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'spmm_fwd|gemm_tc|spmm_bwd|softmax|adam' --launch-skip 60 --launch-count 16 -o gpurun_out/full_$T python tools/profile_epoch.py > gpurun_out/full_$T.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:'spmm_fwd' --launch-count 1 -o gpurun_out/full_l1_$T python tools/profile_epoch.py > gpurun_out/full_l1_$T.log 2>&1
python tools/ncu_summary.py gpurun_out/full_$T.ncu-rep > gpurun_out/ncu_batch_$T.txt 2>&1
python tools/ncu_summary.py gpurun_out/full_l1_$T.ncu-rep > gpurun_out/ncu_l1_$T.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$T.txt; lscpu | head -20 > gpurun_out/lscpu_$T.txt
cat gpurun_out/launch_list_$T.txt
python -c "import json; d=json.load(open('gpurun_out/bench_$T.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['trains'])"
cat gpurun_out/bench_ref_$T.json | cut -c1-200
