set -x
python paper_2106_05609_b200/build.py >/dev/null 2>&1 || true
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 900 python tools/workload_bench.py products_appnp > gpurun_out/products.json 2> gpurun_out/products.err; echo "products rc=$?"
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json gpurun_out/products.json; tail -3 gpurun_out/products.err
