# DP path checks on one GPU (ranks share it): pytest + a 2-rank bench smoke run.
set -x
python paper_2106_05609_b200/build.py >/dev/null 2>&1 || true
timeout 900 python -m pytest tests/test_dp_gpu.py -x -q -s > gpurun_out/pytest_dp.log 2>&1; echo "pytest rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --workload reddit_mini --no-cpu > gpurun_out/bench_dp2.json 2> gpurun_out/bench_dp2.err; echo "bench rc=$?"
tail -30 gpurun_out/pytest_dp.log; cat gpurun_out/bench_dp2.json; tail -20 gpurun_out/bench_dp2.err
