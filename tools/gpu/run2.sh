cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "32 or cfg5 or mask or host or stream or thread or binding" > gpurun_out/p2_pytest.txt 2>&1; tail -3 gpurun_out/p2_pytest.txt
for v in base ns; do
  if [ $v = base ]; then unset D3_LIB; else export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; fi
  timeout 300 python tools/bench_configs.py 5 2 > gpurun_out/p2_cfg_$v.txt 2>&1; echo $v; cat gpurun_out/p2_cfg_$v.txt | cut -c1-400
done
unset D3_LIB
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for t in memcheck synccheck initcheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 30 python tools/sanitize_cases.py quick > gpurun_out/san_$t.txt 2>&1
  echo "$t rc=$? $(tail -3 gpurun_out/san_$t.txt | tr '\n' ' ')"
done
