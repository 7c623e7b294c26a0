cd $GRAFT_REPO_ROOT
for v in base k4 k4f2; do
  if [ $v = base ]; then unset D3_LIB; else export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; fi
  python tools/time_call.py djt 64 u8 1 0x001; python tools/time_call.py djt 64 u8 1 0x001; python tools/time_call.py djt 64 u8 1 0xFFF
done
export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_k4.so
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "djt" 2>&1 | tail -2
ncu --set full --import-source on --clock-control none -k regex:djt_pass -c 2 -o gpurun_out/cfg4k4 -f python tools/cfg_once.py 4 > gpurun_out/cfg4k4.log 2>&1
