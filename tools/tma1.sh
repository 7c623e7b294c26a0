cd $GRAFT_REPO_ROOT/tools
( for a in "0 0 1" "0 1 1" "0 0 2" "8 0 1" "1 0 1" "2 0 1" "4 0 1" "-8 0 1" "-1 0 1" "100 0 1" "0 0 4"; do ./tma_probe $a; done ) > ../gpurun_out/tma_probe.txt 2>&1
