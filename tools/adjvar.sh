# DRT backprojection variants (libdrt3d_<name>.so) vs the default: adjoint tests + N=256 x12 timing
for v in "" "$@"; do
  if [ -n "$v" ]; then export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; else unset D3_LIB; fi
  python -m pytest tests/test_gpu_adjoint.py -q 2>&1 | tail -1
  python -c "
import sys; sys.path.insert(0,'tools'); import bench_configs as b
print('$v', min(b.run_adjoint(3)['ms_median'] for _ in range(2)))"
done
