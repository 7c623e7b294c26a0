cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q -p no:cacheprovider -k "djt" > gpurun_out/p5_pytest.txt 2>&1; tail -2 gpurun_out/p5_pytest.txt
python tools/bench_configs.py 4 4 | cut -c1-200
ncu --set full --import-source on --clock-control none -k regex:djt_pass -c 2 -o gpurun_out/cfg4b -f python tools/cfg_once.py 4 > gpurun_out/cfg4b.log 2>&1
