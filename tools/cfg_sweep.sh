# Time side-library variants on BASELINE configs (tools/bench_configs.py) on one B200.
# usage: bash tools/cfg_sweep.sh "base v1 v2 ..." "5 4"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in $1; do
  if [ "$v" = base ]; then unset D3_LIB; else export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; fi
  timeout 300 python tools/bench_configs.py $2 > gpurun_out/cs_$v.log 2>&1
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
for l in open(f"gpurun_out/cs_{v}.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print(f"{v} cfg{d['config']} ms_median {d['ms_median']:.4f} best {d['ms_best']:.4f}", flush=True)
    elif "Error" in l or "error" in l:
        print(v, l.strip()[:300])
PY
done
