cd $GRAFT_REPO_ROOT
for v in base f96 f64 f48; do
  if [ $v = base ]; then unset D3_LIB; else export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; fi
  python tools/time_call.py drt 32 f32 256 0xFFF; python tools/time_call.py drt 32 i32 64 0xFFF
done
export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_f96.so
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "cfg5 or 32" 2>&1 | tail -1
