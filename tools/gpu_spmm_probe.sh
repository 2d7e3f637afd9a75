# SpMM engine sweep (see tools/spmm_probe.py); prints one JSON line per configuration
python paper_2106_05609_b200/build.py > /dev/null 2>&1
run() { env "$@" timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1; }
run GASB_SPMM_ENGINE=flat
run GASB_SPMM_ENGINE=reg GASB_REG_CPL=4
run GASB_SPMM_ENGINE=reg GASB_REG_CPL=8
run GASB_SPMM_ENGINE=reg GASB_REG_CPL=8 GASB_SPMM_RANGES_PER_SM=16
