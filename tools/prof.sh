# ncu --set full of kernels matching $2 in one bench step. usage: bash tools/prof.sh TAG REGEX SKIP COUNT
cd $GRAFT_REPO_ROOT
TAG=$1; RX=$2; SK=$3; CN=$4
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:$RX -s $SK -c $CN -o gpurun_out/prof_$TAG \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_$TAG.log 2>&1
echo ncu=$? > gpurun_out/status_prof_$TAG.txt
