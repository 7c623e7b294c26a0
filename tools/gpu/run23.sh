cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py -x -q -p no:cacheprovider -k "u8 or uint8 or cfg2 or cfg3 or saturated or mask or tables or 512 or mosaic or host or batched" > gpurun_out/p23.txt 2>&1; tail -2 gpurun_out/p23.txt
bash tools/sweep.sh "base cc0"
python tools/time_call.py drt 64 u8 1 0xFFF; D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_cc0.so python tools/time_call.py drt 64 u8 1 0xFFF
python tools/swar_prof.py 2>/dev/null | head -8
