python paper_2106_05609_b200/build.py > /dev/null 2>&1
run() { env "$@" timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1; }
run GASB_SPMM_ENGINE=flat
for v in ke8mb3 ke8mb4 ke4mb6 ke4mb8; do
  run GASB_LIB=tools/var/libgasb_$v.so GASB_SPMM_ENGINE=reg GASB_SPMM_RANGES_PER_SM=16
done
run GASB_LIB=tools/var/libgasb_ke8mb3.so GASB_SPMM_ENGINE=reg GASB_SPMM_RANGES_PER_SM=12
run GASB_LIB=tools/var/libgasb_ke4mb6.so GASB_SPMM_ENGINE=reg GASB_SPMM_RANGES_PER_SM=24
