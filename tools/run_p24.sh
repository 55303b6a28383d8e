LEVEL=9 SWEEPS=1 SCHED=plane TILU_PLANE_TRACE=gpurun_out/p24_trace_L9.txt timeout 900 python tools/plane_bench.py > gpurun_out/p24_bench_L9.log 2>&1
