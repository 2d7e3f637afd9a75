# epoch-time sweep of existing GEMM / launch knobs at C3 (2 repeats each)
python paper_2106_05609_b200/build.py > /dev/null 2>&1
run() { env "$@" timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], 'epoch_ms %.2f ck %.4f' % (d['epoch_ms'], d['checksum']))"; }
for rep in 1 2; do
run GASB_X=base
run GASB_GEMM_SPLITK_DIV=4
run GASB_GEMM_SPLITK_DIV=3
run GASB_GEMM_BN32_BELOW=100
run GASB_PDL=1
done
