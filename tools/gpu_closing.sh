# closing check of the final tree: GPU suite + smoke, bench line
python paper_2106_05609_b200/build.py > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_close.json 2> gpurun_out/bench_close.err
python -c "import json; d=json.load(open('gpurun_out/bench_close.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline'].get('gather_model',{}).get('frac'), d['clocks'])"
