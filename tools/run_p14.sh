LEVEL=8 SWEEPS=1 SCHED=plane VARIANT=v2 TILU_PLANE_NTASKS=1 TILU_PLANE_STEPLOG=gpurun_out/p14_steplog_v2.txt timeout 300 python tools/plane_bench.py > gpurun_out/p14_bench_v2.log 2>&1
