python paper_2106_05609_b200/build.py >/dev/null 2>&1
timeout 900 python tools/pull_sweep.py > gpurun_out/pull_sweep.jsonl 2> gpurun_out/pull_sweep.err; echo rc=$?
python - <<'PY'
import json
for l in open('gpurun_out/pull_sweep.jsonl'):
    r=json.loads(l); print(r['d'], r['rows'], 'push %.0f GB/s %.2f' % (r['push']['GBps'], r['push']['frac_of_hbm_peak']), 'pull %.0f GB/s %.2f' % (r['pull']['GBps'], r['pull']['frac_of_hbm_peak']))
PY
timeout 900 python -m pytest tests/test_history_gpu.py tests/test_trainer_gpu.py -x -q 2>&1 | tail -2
