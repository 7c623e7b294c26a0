for v in ct8 ct10 ct12; do
  if [ -n "$v" ]; then export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; else unset D3_LIB; fi
  python -m pytest tests/test_gpu_parity.py -q -k "cfg5 or float or random_all" 2>&1 | tail -1
  python -c "
import sys; sys.path.insert(0,'tools'); import bench_configs as b
print('$v', [round(b.run(c)['ms_median'],4) for c in (1,2,3,5)])"
  python tools/fwd_dtypes.py | tail -2
done
