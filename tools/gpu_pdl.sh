# programmatic dependent launch on/off: epoch time, then the GPU suite with it on
python paper_2106_05609_b200/build.py > /dev/null 2>&1
for i in 1 2; do for p in 0 1; do GASB_PDL=$p timeout 300 python tools/spmm_probe.py 2>/dev/null | tail -1; done; done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "passed|failed|^FAILED|^E  " | head
