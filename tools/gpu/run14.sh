cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_adjoint.py tests/test_gpu_guards.py tests/test_gpu_invert.py -x -q -p no:cacheprovider > gpurun_out/p14.txt 2>&1; tail -2 gpurun_out/p14.txt
python tools/bench_configs.py 3 2>&1 | cut -c1-150
python - <<'PY'
import sys, json
sys.path.insert(0, "tools")
import bench_configs as b
for c in (3, 4):
    print(json.dumps(b.run_adjoint(c)))
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:adj python tools/adj_once.py 2>/dev/null | grep -o '"drt_adj[a-z_]*\|"ns","[0-9]*' | tail -6
