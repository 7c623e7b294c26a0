# Round evidence on one B200: GPU tests, smoke, the default bench line, the reference arm, the ncu
# launch list, one ncu --set full capture (--cache-control none, as SURVEY §8(d) asks) of the two
# kernels of one step (first pass + 12-dodecant final pass), the HBM write-only / copy ceilings.
# usage: bash tools/evidence.sh TAG
cd $GRAFT_REPO_ROOT
TAG=$1
S=gpurun_out/ev_status_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ev_pytest_$TAG.log 2>&1; echo pytest=$? > $S
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke_$TAG.log 2>&1; echo smoke=$? >> $S
timeout 600 python bench.py > gpurun_out/ev_bench_$TAG.log 2>&1; echo bench=$? >> $S
timeout 600 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/ev_ref_$TAG.log 2>&1; echo ref=$? >> $S
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:drt -s 6 -c 64 --csv --log-file gpurun_out/ev_launches_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ev_ncul_$TAG.log 2>&1; echo ncul=$? >> $S
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:drt -s 6 -c 2 -o gpurun_out/ev_prof_$TAG -f \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ev_ncu_$TAG.log 2>&1; echo ncu=$? >> $S
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC tools/write_probe.cu -o tools/libwrite_probe.so > gpurun_out/ev_hbm_build_$TAG.log 2>&1
timeout 300 python tools/hbm_write_probe.py > gpurun_out/ev_hbm_$TAG.log 2>&1; echo hbm=$? >> $S
timeout 600 python tools/bench_configs.py > gpurun_out/ev_configs_$TAG.log 2>&1; echo configs=$? >> $S
timeout 900 bash tools/ncu_configs.sh > gpurun_out/ncu_configs_$TAG.jsonl 2> gpurun_out/ev_ncucfg_$TAG.log; echo ncucfg=$? >> $S
cat $S
