# Round-2 GPU check: build, smoke, GPU tests, bench (both arms). Usage: bash tools/gpu_r2.sh TAG [pytest-args]
set -x
T=${1:-r2}
shift
python paper_2106_05609_b200/build.py >/dev/null 2>&1 || true
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/smoke_$T.log
timeout 2400 python -m pytest tests -m gpu -q -s -rf "$@" > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|C3 timed|Error" gpurun_out/pytest_gpu_$T.log | tail -15
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err; echo "ref rc=$?"
tail -5 gpurun_out/bench_$T.err
cat gpurun_out/bench_$T.json gpurun_out/bench_ref_$T.json
