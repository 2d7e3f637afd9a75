python paper_2106_05609_b200/build.py >/dev/null 2>&1
T=${1:-cur}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$T.csv python tools/profile_epoch.py > gpurun_out/launches_$T.log 2>&1
python tools/launches.py gpurun_out/launches_$T.csv > gpurun_out/launch_list_$T.txt
cat gpurun_out/launch_list_$T.txt
