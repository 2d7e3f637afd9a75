# re-entry check: GPU suite, smoke, bench line of the current tree
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/pytest_gpu_c.log
tail -3 gpurun_out/pytest_gpu_c.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_c.log 2>&1; tail -2 gpurun_out/smoke_c.log
timeout 900 python bench.py > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
python -c "import json; d=json.load(open('gpurun_out/bench_c.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d.get('trains'))"
