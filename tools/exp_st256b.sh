# second 32-byte-store round: DJT image + STG.256 (djtimg), k_sep32 / generic DRT pass STG.256 (sepdrt)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/djtvar.sh djtimg
for v in "" djtimg sepdrt; do
  if [ -n "$v" ]; then export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; else unset D3_LIB; fi
  if [ "$v" != sepdrt ]; then
    python tools/time_call.py djt 128 u8 1 0x1
    python tools/time_call.py djt 64 f32 1 0xfff
  fi
  if [ "$v" != djtimg ]; then
    python tools/time_call.py drt 32 f32 256 0xfff
    python tools/time_call.py drt 32 u8 256 0xfff
    python tools/time_call.py drt 64 f32 8 0xfff
    python tools/time_call.py drt 128 f32 1 0xfff
    python tools/time_call.py drt 256 f32 1 0xfff
    python tools/time_call.py drt 16 f32 64 0xfff
  fi
done
export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_sepdrt.so
python -m pytest tests/test_gpu_parity.py -q -x -k "not djt" 2>&1 | tail -2
