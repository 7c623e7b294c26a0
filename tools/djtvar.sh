for v in "" djth128 djth512; do
  if [ -n "$v" ]; then export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; else unset D3_LIB; fi
  python -m pytest tests/test_gpu_parity.py -q -k "djt" 2>&1 | tail -1
  python -c "
import sys; sys.path.insert(0,'tools'); import json, bench_configs as b
r=b.run(4); print('$v', r['ms_median'])"
done
