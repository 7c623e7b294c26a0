python -m pytest tests/test_gpu_parity.py tests/test_gpu_adjoint.py tests/test_gpu_apps.py -q -k "djt or lines or denoise" 2>&1 | tail -1
python -c "
import sys; sys.path.insert(0,'tools'); import bench_configs as b
print('tma', min(b.run(4)['ms_median'] for _ in range(3)))"
D3_NO_TMA_STORE=1 python -c "
import sys; sys.path.insert(0,'tools'); import bench_configs as b
print('no-tma (4x32 direct stores)', min(b.run(4)['ms_median'] for _ in range(3)))"
