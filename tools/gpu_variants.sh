# SpMM pipeline-shape variants (prebuilt libraries under paper_2106_05609_b200/variants/)
for f in paper_2106_05609_b200/variants/libgasb_*.so; do echo "$f"; GASB_LIB=$PWD/$f timeout 300 python tools/engine_probe.py 2>&1 | tail -1; done
