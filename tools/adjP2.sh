python -m pytest tests/test_gpu_adjoint.py tests/test_gpu_invert.py -x -q 2>&1 | tail -2
python -c "
import sys; sys.path.insert(0,'tools'); import json, bench_configs as b
print(json.dumps(b.run_adjoint(3))[:150]); print(json.dumps(b.run_invert(256))[:200]); print(json.dumps(b.run_invert(64))[:200])"
bash tools/adjlist.sh
