python paper_2106_05609_b200/build.py >/dev/null 2>&1
for c in 4 2; do GASB_SPMM_CPL=$c timeout 300 python tools/engine_probe.py 2>&1 | tail -1; done
