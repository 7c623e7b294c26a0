cd $GRAFT_REPO_ROOT
for v in base c3a c3b c3c; do
  if [ $v = base ]; then unset D3_LIB; else export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; fi
  python tools/time_call.py drt 64 u8 1 0xFFF; python tools/time_call.py drt 64 u8 1 0xFFF; python tools/time_call.py drt 32 u8 64 0xFFF
done
