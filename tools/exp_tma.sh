# TMA brick staging of the SWAR first pass: parity of the product build, then cfg3 timing against
# the variants (noswz: kind-1 map unswizzled, notma: LDG staging)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not djt" 2>&1 | tail -5
for v in $1; do
  python tools/variant_check.py $v
done
bash tools/sweep.sh "base $1" 20
for v in "" $1; do
  if [ -n "$v" ]; then export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; else unset D3_LIB; fi
  python tools/time_call.py drt 128 u8 1 0xfff
  python tools/time_call.py drt 512 u8 1 0x1
done
