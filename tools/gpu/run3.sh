cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q -p no:cacheprovider -k "32 or cfg5 or mask or guards or binding" > gpurun_out/p3_pytest.txt 2>&1; tail -3 gpurun_out/p3_pytest.txt
bash tools/cfg_sweep.sh "base ns" "5 5"
