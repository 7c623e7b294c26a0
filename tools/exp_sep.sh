# k_sep32 variants: parity at N = 32 (all dtypes, cfg5 at full size, guards) + timing against the product build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -q -x -k "32 or cfg5 or masks or float" 2>&1 | tail -2
for v in "" $1; do
  if [ -n "$v" ]; then export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; else unset D3_LIB; fi
  python tools/time_call.py drt 32 f32 256 0xfff
  python tools/time_call.py drt 32 i32 256 0xfff
  python tools/time_call.py drt 32 f32 256 0xff0
done
