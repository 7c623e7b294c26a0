cd $GRAFT_REPO_ROOT/tools
./tma_rows_bench 2 208 x 148 > ../gpurun_out/plain_mb.log 2>&1 && ncu --set full --clock-control none -k regex:k -s 1 -c 1 -o ../gpurun_out/prof_mb ./tma_rows_bench 2 208 x 148 > ../gpurun_out/ncu_mb.log 2>&1
./tma_rows_bench 3 208 x 148 > ../gpurun_out/plain_mb3.log 2>&1 && ncu --set full --clock-control none -k regex:k -s 1 -c 1 -o ../gpurun_out/prof_mb3 ./tma_rows_bench 3 208 x 148 >> ../gpurun_out/ncu_mb.log 2>&1
