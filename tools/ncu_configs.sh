# DRAM bytes and durations of every kernel of each BASELINE config (one call each after warm-up).
# usage: bash tools/ncu_configs.sh  -> gpurun_out/ncu_cfg<k>.csv
for c in 1 2 3 4 5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      -k regex:"drt|djt" --log-file gpurun_out/ncu_cfg$c.csv python tools/cfg_once.py $c > /dev/null 2>&1
done
python tools/ncu_configs_sum.py
