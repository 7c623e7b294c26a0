cd $GRAFT_REPO_ROOT
D3_PERSIST=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_persist.log 2>&1
D3_PIPE=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_pipe2.log 2>&1
python tools/swar_prof.py > gpurun_out/swar_prof3.txt 2>&1
