cd $GRAFT_REPO_ROOT
for v in fm4_1 fm8_1 fm16_3 fm16_0; do
  D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$v.log 2>&1
done
