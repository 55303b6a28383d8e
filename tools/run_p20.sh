LEVEL=8 SWEEPS=1 SCHED=plane TILU_PLANE_NTASKS=1 TILU_PLANE_STEPLOG=gpurun_out/p20_steplog.txt timeout 300 python tools/plane_bench.py > gpurun_out/p20_bench_1task.log 2>&1
timeout 300 python tools/plane_debug.py > gpurun_out/p20_debug.log 2>&1
LEVEL=8 SWEEPS=10 SCHED=plane timeout 300 python tools/plane_bench.py > gpurun_out/p20_bench_L8.log 2>&1
