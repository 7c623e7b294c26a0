cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "cfg3 or saturated or large_all or batched or host or stream or thread" > gpurun_out/p18.txt 2>&1; tail -2 gpurun_out/p18.txt
bash tools/sweep.sh "base zf1 zf0"
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"drt|zero" python tools/cfg_once.py 3 2>/dev/null | grep -o '"void [a-z_0-9]*\|"ns","[0-9]*' | paste - - | tail -3
