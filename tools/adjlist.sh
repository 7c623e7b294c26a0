ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:adj --log-file gpurun_out/adj_launches.csv python tools/adj_once.py > /dev/null 2>&1
python tools/launch_list.py gpurun_out/adj_launches.csv gpurun_out/adj_launches_list.csv
