cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r1a.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -x > gpurun_out/pytest_r1a.log 2>&1; echo pytest=$? > gpurun_out/status_r1a.txt
timeout 400 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r1a.log 2>&1; echo bench=$? >> gpurun_out/status_r1a.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1a.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_r1a.log 2>&1; echo ncul=$? >> gpurun_out/status_r1a.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:drt_pass -s 24 -c 4 -o gpurun_out/prof_r1a python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_r1a.log 2>&1; echo ncu=$? >> gpurun_out/status_r1a.txt
