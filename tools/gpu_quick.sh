python paper_2106_05609_b200/build.py >/dev/null 2>&1
for p in 1 0; do GASB_PDL=$p timeout 300 python tools/engine_probe.py 2>&1 | tail -1; done
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/workload_bench.py products_appnp 2>&1 | tail -1
timeout 900 python tools/workload_bench.py pubmed_gcnii 2>&1 | tail -1
