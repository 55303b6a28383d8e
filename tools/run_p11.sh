timeout 300 python tools/plane_debug.py > gpurun_out/p11_debug.log 2>&1
timeout 600 python -m pytest tests/test_gpu_plane.py -q -x > gpurun_out/p11_plane_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p11_plane_tests.log
LEVEL=8 SWEEPS=10 SCHED=plane timeout 300 python tools/plane_bench.py > gpurun_out/p11_bench_L8.log 2>&1
LEVEL=8 SWEEPS=1 SCHED=plane TILU_PLANE_TRACE=gpurun_out/p11_trace_L8.txt timeout 300 python tools/plane_bench.py > gpurun_out/p11_bench_L8t.log 2>&1
LEVEL=8 SWEEPS=10 FAST=1 SCHED=plane timeout 300 python tools/plane_bench.py > gpurun_out/p11_bench_L8f.log 2>&1
