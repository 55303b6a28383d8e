LEVEL=8 SWEEPS=1 SCHED=plane TILU_PLANE_NTASKS=1 TILU_PLANE_STEPLOG=gpurun_out/p17_steplog.txt timeout 300 python tools/plane_bench.py > gpurun_out/p17_bench_1task.log 2>&1
