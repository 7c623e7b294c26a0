# Time side-library variants of the cfg3 step (bench.py, no CPU baseline / e2e) on one B200.
# usage: bash tools/sweep.sh "base v1 v2 ..." [steps]   (base = the product libdrt3d.so)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in $1; do
  if [ "$v" = base ]; then unset D3_LIB; else export D3_LIB=$GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; fi
  for rep in 1 2; do
    timeout 300 python bench.py --steps ${2:-20} --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/sw_${v}_${rep}.log 2>&1
    python - "$v" "$rep" <<'PY'
import json, sys
v, rep = sys.argv[1], sys.argv[2]
try:
    l = [x for x in open(f"gpurun_out/sw_{v}_{rep}.log").read().splitlines() if x.startswith("{")][-1]
    d = json.loads(l)
    r = d["roofline"]
    print(f"{v} rep{rep} ms {d['ms_per_step']:.4f} final {r['launch_ms']:.4f} first {r['first_pass_ms']:.4f} "
          f"launches {d['gpu_launches']} clocks {d['clocks'].get('sm_mhz')}", flush=True)
except Exception as e:
    print(v, rep, "FAILED", e, open(f"gpurun_out/sw_{v}_{rep}.log").read()[-800:])
PY
  done
done
