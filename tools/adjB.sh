set -e
python -m pytest tests/test_gpu_adjoint.py -x -q 2>&1 | tail -1
for B in 0 1 2; do echo "BFLY=$B"; D3_ADJ_BFLY=$B python -c "
import sys; sys.path.insert(0,'tools'); import json, bench_configs as b
print(json.dumps(b.run_adjoint(3)))" | cut -c1-130; done
D3_ADJ_BFLY=1 python -m pytest tests/test_gpu_adjoint.py -x -q 2>&1 | tail -1
