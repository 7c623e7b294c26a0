# Compare side-library variants with the default build on one B200.
# usage: bash tools/variants.sh "v1 v2 ..." [pytest -k expr for a per-variant parity subset]
cd $GRAFT_REPO_ROOT
VS=$1; K=${2:-"parity and (256 or 32)"}
run() {  # $1 = tag, $2 = lib path ("" = default)
  if [ -n "$2" ]; then export D3_LIB=$2; else unset D3_LIB; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "$K" > gpurun_out/var_pytest_$1.log 2>&1
  echo "$1 pytest=$? $(tail -1 gpurun_out/var_pytest_$1.log)"
  for rep in 1 2; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/var_bench_$1_$rep.log 2>&1
    python -c "
import json,sys
l=open('gpurun_out/var_bench_$1_$rep.log').read().strip().splitlines()[-1]; d=json.loads(l[l.index('{'):])
print('$1 rep $rep', round(d['ms_per_step'],4), 'final', round(d['roofline']['launch_ms'],4), 'first', round(d['roofline']['first_pass_ms'],4))"
  done
}
run base ""
for v in $VS; do run $v $GRAFT_REPO_ROOT/paper_2501_13664_b200/libdrt3d_$v.so; done
