python paper_2106_05609_b200/build.py >/dev/null 2>&1
timeout 1200 python -m pytest tests/test_dp_gpu.py tests/test_trainer_gpu.py tests/test_ops_gpu.py -x -q 2>&1 | tail -4
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --workload reddit_mini --no-cpu 2>/dev/null | tail -1
for d in 8 4; do GASB_GEMM_SPLITK_DIV=$d timeout 300 python tools/engine_probe.py 2>&1 | tail -1; done
