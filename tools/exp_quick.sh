# quick cfg3 comparison of side libraries with the product build: bit-exact check + 2 x 20 steps each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in $1; do python tools/variant_check.py $v; done
bash tools/sweep.sh "base $1" 20
