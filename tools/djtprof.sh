ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:djt --log-file gpurun_out/djt_launches.csv python tools/djt_once.py > /dev/null 2>&1
python tools/launch_list.py gpurun_out/djt_launches.csv gpurun_out/djt_launches_list.csv
ncu --set full --clock-control none --import-source on -k regex:djt -s 4 -c 2 -o gpurun_out/djt_prof -f python tools/djt_once.py > gpurun_out/djt_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/djt_prof.ncu-rep
