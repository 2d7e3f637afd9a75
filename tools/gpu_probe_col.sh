for m in 1 2 4; do echo "colmod $m"; GASB_PROBE_COLMOD=$m GASB_LIB=$PWD/paper_2106_05609_b200/variants/libgasb_probe.so timeout 300 python tools/engine_probe.py 2>&1 | tail -1; done
