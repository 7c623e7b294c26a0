python -m pytest tests/test_gpu_adjoint.py -x -q 2>&1 | tail -3
for M in "" bfly; do echo "MODE=$M"; D3_ADJ_MODE=$M python -c "
import os
if not os.environ.get('D3_ADJ_MODE'): os.environ.pop('D3_ADJ_MODE', None)
import sys; sys.path.insert(0,'tools'); import json, bench_configs as b
print(json.dumps(b.run_adjoint(3)))" | cut -c1-140; done
