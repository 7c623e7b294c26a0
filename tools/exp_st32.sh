# 32-byte stage-row stores of the 32-bit first pass: parity (i32 / f32 at N = 128, 256; 3-pass N = 512) + timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_invert.py tests/test_gpu_guards.py -q -x -k "not djt and not u8" 2>&1 | tail -3
for v in "" nost; do
  if [ -n "$v" ]; then export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; else unset D3_LIB; fi
  python tools/time_call.py drt 256 f32 1 0xfff
  python tools/time_call.py drt 256 i32 1 0xfff
  python tools/time_call.py drt 128 f32 1 0xfff
  python tools/time_call.py drt 64 f32 8 0xfff
  python tools/time_call.py drt 512 f32 1 0x1
done
