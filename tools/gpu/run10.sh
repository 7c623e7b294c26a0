cd $GRAFT_REPO_ROOT
for v in base f2 f1; do
  if [ $v = base ]; then unset D3_LIB; else export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; fi
  python tools/time_call.py djt 64 u8 1 0x001; python tools/time_call.py djt 64 u8 1 0x001; python tools/time_call.py djt 32 i32 4 0xFFF
done
