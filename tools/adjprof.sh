# Launch list + ncu --set full of the DRT N=256 x12 backprojection (tools/adj_once.py).
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:adj --log-file gpurun_out/adj_launches.csv python tools/adj_once.py > /dev/null 2>&1
ncu --set full --clock-control none --cache-control none --import-source on -k regex:drt_adj -s 3 -c 3 -o gpurun_out/adj_full -f python tools/adj_once.py > gpurun_out/adj_ncu.log 2>&1
tail -2 gpurun_out/adj_ncu.log
