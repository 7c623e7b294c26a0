for v in "" ch1g; do
  if [ -n "$v" ]; then export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; else unset D3_LIB; fi
  echo "== $v"; python tools/fwd_dtypes.py
  python -c "
import sys; sys.path.insert(0,'tools'); import json, bench_configs as b
print(json.dumps(b.run_invert(256))[:160]); print(b.run(5)['ms_median'])"
done
