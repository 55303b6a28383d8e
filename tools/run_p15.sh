LEVEL=8 SWEEPS=1 SCHED=plane VARIANT=v2 TILU_PLANE_NTASKS=1 TILU_PLANE_STEPLOG=gpurun_out/p15_steplog_v2.txt timeout 300 python tools/plane_bench.py > gpurun_out/p15_bench_v2.log 2>&1
timeout 300 python tools/plane_debug.py > gpurun_out/p15_debug.log 2>&1
LEVEL=8 SWEEPS=10 SCHED=plane timeout 300 python tools/plane_bench.py > gpurun_out/p15_bench_L8.log 2>&1
LEVEL=9 SWEEPS=5 SCHED=plane timeout 900 python tools/plane_bench.py > gpurun_out/p15_bench_L9.log 2>&1
