cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "cfg3 or saturated or large_all or batched or host or stream" > gpurun_out/p17.txt 2>&1; tail -2 gpurun_out/p17.txt
bash tools/sweep.sh "base zf0"
python tools/swar_prof.py | head -8
