# full GPU test suite + smoke, logs under gpurun_out/
python paper_2106_05609_b200/build.py >/dev/null 2>&1 || true
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rA -s 2>&1 | grep -v "^PASSED\|^$" | tail -60 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
