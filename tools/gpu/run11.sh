cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "cfg3 or saturated or large_all or 512 or 1024" > gpurun_out/p11_pytest.txt 2>&1; tail -2 gpurun_out/p11_pytest.txt
bash tools/sweep.sh "base ws0"
python tools/pass_prof.py
