python paper_2106_05609_b200/build.py >/dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_products.csv python tools/profile_epoch.py --workload products_appnp > gpurun_out/launches_products.log 2>&1
python tools/launches.py gpurun_out/launches_products.csv > gpurun_out/launch_list_products.txt
cat gpurun_out/launch_list_products.txt
