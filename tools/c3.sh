cd $GRAFT_REPO_ROOT
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('l2', p.L2_cache_size)
import ctypes
" > gpurun_out/props.txt 2>&1
for mb in 0 48 64 96; do
  D3_L2_PERSIST_MB=$mb timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_l2_$mb.log 2>&1
done
D3_L2_PERSIST_MB=64 bash tools/prof_nc.sh r1p drt 72 4
