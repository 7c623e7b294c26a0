cd $GRAFT_REPO_ROOT
for v in swr4c3 swr4c4; do
  D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "random_all and uint8" > gpurun_out/pytest_$v.log 2>&1
  D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$v.log 2>&1
done
