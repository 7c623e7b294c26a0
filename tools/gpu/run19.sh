cd $GRAFT_REPO_ROOT
export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_zt1.so
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q -p no:cacheprovider -k "cfg3 or saturated or large_all or batched or guards" > gpurun_out/p19.txt 2>&1; tail -2 gpurun_out/p19.txt
unset D3_LIB
bash tools/sweep.sh "zt0 zt1 zt1f1"
