LEVEL=8 SWEEPS=1 SCHED=plane TILU_PLANE_TRACE=gpurun_out/p8_trace_L8.txt timeout 300 python tools/plane_bench.py > gpurun_out/p8_bench_L8.log 2>&1
