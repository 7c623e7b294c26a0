# one GPU round trip: GPU tests, a short bench (no ncu).  usage: bash tools/cycle.sh TAG [pytest -k expr]
cd $GRAFT_REPO_ROOT
TAG=$1; K=${2:-}
if [ -n "$K" ]; then timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$K" > gpurun_out/pytest_$TAG.log 2>&1; else
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_$TAG.log 2>&1; fi
echo pytest=$? > gpurun_out/status_$TAG.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$TAG.log 2>&1; echo bench=$? >> gpurun_out/status_$TAG.txt
