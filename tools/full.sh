# full round check on one B200: GPU tests, smoke, bench, all configs.  usage: bash tools/full.sh TAG
TAG=$1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/full_pytest_$TAG.log 2>&1; echo pytest=$?
tail -2 gpurun_out/full_pytest_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke_$TAG.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/full_bench_$TAG.log 2>&1; echo bench=$?
timeout 600 python tools/bench_configs.py > gpurun_out/full_configs_$TAG.jsonl 2> gpurun_out/full_configs_$TAG.err; echo configs=$?
