cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q -p no:cacheprovider -k "cfg3 or saturated or large_all or batched or host or stream or binding" > gpurun_out/p24.txt 2>&1; tail -4 gpurun_out/p24.txt
bash tools/sweep.sh "base ws0"
