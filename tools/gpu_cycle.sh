#!/bin/bash
# One GPU round trip: GPU tests, a short bench, and an ncu capture of the DRT kernels.
# usage (inside gpurun): bash tools/gpu_cycle.sh TAG [pytest-args]
TAG=$1; shift
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 "$@" > gpurun_out/pytest_$TAG.log 2>&1; echo pytest=$? > gpurun_out/status_$TAG.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$TAG.log 2>&1; echo bench=$? >> gpurun_out/status_$TAG.txt
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:drt_pass -s 72 -c 10 -o gpurun_out/prof_$TAG \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu=$? >> gpurun_out/status_$TAG.txt
