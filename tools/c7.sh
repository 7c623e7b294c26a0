cd $GRAFT_REPO_ROOT
D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_t32.so timeout 600 python -m pytest tests -m gpu -q -x -k "cfg3 or random_all" > gpurun_out/pytest_t32.log 2>&1
for v in t32; do
  D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$v.log 2>&1
  D3_NO_OVERLAP=1 D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_${v}_noov.log 2>&1
done
