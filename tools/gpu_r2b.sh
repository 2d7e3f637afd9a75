set -x
python paper_2106_05609_b200/build.py >/dev/null 2>&1
timeout 1500 python -m pytest tests/test_scaled_configs_gpu.py tests/test_dp_gpu.py -m gpu -q -s -rf -k "scaled or c4 or c5 or equals_replicated" > gpurun_out/pytest_r2g.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|nnz=|NVLink|^E  " gpurun_out/pytest_r2g.log | cut -c1-300 | tail -12
timeout 900 python tools/gpu_traj.py --out gpurun_out/gpu_traj_c3.json --ref profiles/r2_ref_c3_trajectory.json
