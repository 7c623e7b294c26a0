cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_apps.py -x -q -p no:cacheprovider -k "djt or lines or denoise or cfg4" > gpurun_out/p22.txt 2>&1; tail -2 gpurun_out/p22.txt
for v in base do0; do
  if [ $v = base ]; then unset D3_LIB; else export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; fi
  python tools/time_call.py djt 64 u8 1 0x001; python tools/time_call.py djt 64 u8 1 0x001; python tools/time_call.py djt 64 u8 1 0xFFF; python tools/time_call.py djt 128 u8 1 0x001
done
