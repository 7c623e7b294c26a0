python -m pytest tests/test_gpu_adjoint.py tests/test_gpu_apps.py -q -k "djt or denoise" 2>&1 | tail -1
python -c "
import sys; sys.path.insert(0,'tools'); import json, bench_configs as b
print(json.dumps(b.run_adjoint(4))[:140])
for r in b.run_apps(): print(json.dumps(r)[:200])"
