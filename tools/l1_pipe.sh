# L1 data-pipe breakdown per kernel (wavefronts: total / shared; global store requests and sectors)
# of the backprojection, cfg2, cfg5 and the fp32 N=256 forward.  usage: bash tools/l1_pipe.sh
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.per_cycle_active
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/l1_adj.csv python tools/adj_once.py > /dev/null 2>&1
for c in 2 5; do ncu --metrics $M --clock-control none --csv -k regex:"drt|djt" --log-file gpurun_out/l1_cfg$c.csv python tools/cfg_once.py $c > /dev/null 2>&1; done
ncu --metrics $M --clock-control none --csv -k regex:"drt" -c 4 --log-file gpurun_out/l1_f32.csv python tools/time_call.py drt 256 f32 1 0xFFF > /dev/null 2>&1
echo done
