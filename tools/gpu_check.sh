# quick GPU check: gpu tests + default bench (run from the repo root on the box)
set -x
python paper_2106_05609_b200/build.py >/dev/null 2>&1 || true
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json
