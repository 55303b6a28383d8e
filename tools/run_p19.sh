LEVEL=8 SWEEPS=1 SCHED=plane TILU_PLANE_NTASKS=1 TILU_PLANE_DBG=1 TILU_PLANE_STEPLOG=gpurun_out/p19_steplog_dbg1.txt timeout 300 python tools/plane_bench.py > gpurun_out/p19_bench_dbg1.log 2>&1
