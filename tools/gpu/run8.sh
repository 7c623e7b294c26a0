cd $GRAFT_REPO_ROOT
for v in base st16 st32; do
  if [ $v = base ]; then unset D3_LIB; else export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; fi
  python tools/time_call.py drt 16 i32 1 0x001; python tools/time_call.py drt 16 u8 1 0xFFF; python tools/time_call.py drt 16 f32 64 0xFFF
done
unset D3_LIB
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/cfg_once.py 1 2>/dev/null | grep -i "drt\|djt" | tail -4
ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/cfg_once.py 2 2>/dev/null | grep -i "drt\|djt" | tail -4
