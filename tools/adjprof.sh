mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:adj --log-file gpurun_out/adj_launches.csv python tools/adj_once.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:drt_adj_(stage|bfly)' -s 3 -c 1 -o gpurun_out/adj_stage -f python tools/adj_once.py > gpurun_out/adj_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:drt_adj_scatter -s 1 -c 1 -o gpurun_out/adj_scatter -f python tools/adj_once.py >> gpurun_out/adj_ncu.log 2>&1
tail -3 gpurun_out/adj_ncu.log
