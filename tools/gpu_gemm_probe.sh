python paper_2106_05609_b200/build.py > /dev/null 2>&1
run() { env "$@" timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1; }
run GASB_GEMM_BN32_BELOW=0
run GASB_GEMM_BN32_BELOW=100
run GASB_GEMM_BN32_BELOW=100 GASB_GEMM_SPLITK_DIV=4
run GASB_GEMM_BN32_BELOW=100 GASB_GEMM_SPLITK_DIV=8
