cd $GRAFT_REPO_ROOT
python tools/bench_configs.py 5 > gpurun_out/cfg5_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"drt|djt" -s 8 -c 8 --csv --log-file gpurun_out/cfg5_launches.csv python tools/bench_configs.py 5 > gpurun_out/cfg5_ncu.log 2>&1
python tools/bench_configs.py 4 > gpurun_out/cfg4_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size --clock-control none -k regex:"drt|djt" -s 5 -c 6 --csv --log-file gpurun_out/cfg4_launches.csv python tools/bench_configs.py 4 > gpurun_out/cfg4_ncu.log 2>&1
