# ncu without cache flushing (in-situ L2 state): metrics only. usage: bash tools/prof_nc.sh TAG REGEX SKIP COUNT
cd $GRAFT_REPO_ROOT
TAG=$1; RX=$2; SK=$3; CN=$4
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum -k regex:$RX -s $SK -c $CN --csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncunc_$TAG.csv 2>&1
echo ncu=$? > gpurun_out/status_prof_$TAG.txt
