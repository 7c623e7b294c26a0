cd $GRAFT_REPO_ROOT
for v in base s32 n32; do
  if [ $v = base ]; then unset D3_LIB; else export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; fi
  python tools/time_call.py drt 32 u8 256 0xFFF; python tools/time_call.py drt 32 f32 256 0xFFF
done
