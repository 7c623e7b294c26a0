cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q -p no:cacheprovider -k "32 or cfg5 or mask or guards" > gpurun_out/p4_pytest.txt 2>&1; tail -2 gpurun_out/p4_pytest.txt
for v in base ns; do
  if [ $v = base ]; then unset D3_LIB; else export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; fi
  python tools/time_call.py drt 32 f32 256 0xFFF; python tools/time_call.py drt 32 u8 256 0xFFF; python tools/time_call.py drt 32 i32 64 0xFFF
done
