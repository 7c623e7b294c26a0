python -m pytest tests/test_gpu_invert.py -q 2>&1 | tail -2
python -c "
import sys; sys.path.insert(0,'tools'); import json, bench_configs as b
for n in (64,128,256): r=b.run_invert(n); print(n, round(r['ms_per_iter'],3), round(r['nrmsd'],4), r['rnorm_ratio'])"
