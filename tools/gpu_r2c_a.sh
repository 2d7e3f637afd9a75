# classifier bwd2 + fused mask parity, then SpMM stage/occupancy variants at C3
python paper_2106_05609_b200/build.py > gpurun_out/a_build.log 2>&1 || { tail gpurun_out/a_build.log; exit 1; }


run() { env "$@" timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], 'batch_us %.1f hoisted_ms %.2f epoch_ms %.2f ck %.4f' % (d['batch_spmm_us'], d['hoisted_ms'], d['epoch_ms'], d['checksum']))"; }
run GASB_X=base
run GASB_LIB=tools/var/libgasb_s4b4.so
run GASB_LIB=tools/var/libgasb_s2b4c4.so
run GASB_LIB=tools/var/libgasb_s3b8c2.so
run GASB_BWD2=0
