python -m pytest tests/test_gpu_invert.py -x -q 2>&1 | tail -2
python -c "
import sys; sys.path.insert(0,'tools'); import json, bench_configs as b
for n in (64,128,256): print(json.dumps(b.run_invert(n))[:230])"
