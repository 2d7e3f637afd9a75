# CUPTI timelines of 12 C3 batches per configuration
python paper_2106_05609_b200/build.py > /dev/null 2>&1
for cfg in "0 0" "1 0" "1 148" "1 296"; do
  set -- $cfg
  GASB_XBATCH=$1 GASB_BG_CTAS=$2 timeout 600 python tools/timeline.py --out gpurun_out/tl_x$1_c$2.json > gpurun_out/tl_x$1_c$2.txt 2> gpurun_out/tl_x$1_c$2.err
  cat gpurun_out/tl_x$1_c$2.txt; tail -2 gpurun_out/tl_x$1_c$2.err
done
