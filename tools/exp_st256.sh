# 32-byte store variants (libdrt3d_<tag>.so) against the product library: bit-exact check on cfg3,
# cfg3 step, DJT parity + cfg4, a few other shapes.  usage: bash tools/exp_st256.sh TAG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=$1
python tools/variant_check.py $T
bash tools/sweep.sh "base $T" 20
bash tools/djtvar.sh $T
for v in "" $T; do
  if [ -n "$v" ]; then export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; else unset D3_LIB; fi
  python tools/time_call.py djt 128 u8 1 0x1
  python tools/time_call.py djt 64 f32 1 0xfff
  python tools/time_call.py drt 32 f32 256 0xfff
  python tools/time_call.py drt 64 u8 1 0xfff
  python tools/time_call.py drt 128 u8 1 0xfff
done
