cd $GRAFT_REPO_ROOT
bash tools/cycle.sh r1z drt
D3_NO_OVERLAP=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_r1z_noov.log 2>&1
D3_NO_OVERLAP=1 python tools/swar_prof.py > gpurun_out/swar_prof2.txt 2>&1
