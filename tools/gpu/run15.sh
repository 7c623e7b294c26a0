cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_adjoint.py tests/test_gpu_invert.py -x -q -p no:cacheprovider -k "f32 or float or cfg5 or invert or adjoint" > gpurun_out/p15.txt 2>&1; tail -2 gpurun_out/p15.txt
for v in base nofadd2; do
  if [ $v = base ]; then unset D3_LIB; else export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; fi
  python tools/time_call.py drt 32 f32 256 0xFFF; python tools/time_call.py drt 256 f32 1 0xFFF; python tools/time_call.py djt 64 f32 1 0x001
  python -c "
import sys, json; sys.path.insert(0, 'tools'); import bench_configs as b
print(json.dumps(b.run_invert(256)))" 2>&1 | cut -c1-200
done
