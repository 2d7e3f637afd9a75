# Round-end run: smoke, profile (bench both arms, launch list, ncu), then the GPU test suite
set -x
python paper_2106_05609_b200/build.py >/dev/null 2>&1 || true
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"
bash tools/gpu_round_profile.sh final
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_final.log
