LEVEL=8 SWEEPS=1 SCHED=plane VARIANT=v2 TILU_PLANE_TRACE=gpurun_out/p9_trace_L8v2.txt timeout 300 python tools/plane_bench.py > gpurun_out/p9_bench_L8v2.log 2>&1
LEVEL=8 SWEEPS=1 SCHED=plane VARIANT=v2 FAST=1 TILU_PLANE_TRACE=gpurun_out/p9_trace_L8v2f.txt timeout 300 python tools/plane_bench.py > gpurun_out/p9_bench_L8v2f.log 2>&1
