# TMA-store copy-out with the .read wait (tmaoutr) on cfg3; TMA brick staging at N = 64 (n64): parity + timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python tools/variant_check.py tmaoutr
bash tools/sweep.sh "base tmaoutr" 20
export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_n64.so
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not djt and not 256 and not 512 and not 1024" 2>&1 | tail -3
for v in "" n64; do
  if [ -n "$v" ]; then export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; else unset D3_LIB; fi
  python tools/time_call.py drt 64 u8 1 0xfff
  python tools/time_call.py drt 64 u8 1 0x1
  python tools/time_call.py drt 64 u8 16 0xfff
done
