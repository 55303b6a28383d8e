timeout 300 python tools/plane_debug.py > gpurun_out/p25_debug.log 2>&1
timeout 600 python -m pytest tests/test_gpu_plane.py -q -x > gpurun_out/p25_plane_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p25_plane_tests.log
LEVEL=8 SWEEPS=10 SCHED=plane timeout 300 python tools/plane_bench.py > gpurun_out/p25_bench_L8.log 2>&1
LEVEL=9 SWEEPS=5 SCHED=plane timeout 900 python tools/plane_bench.py > gpurun_out/p25_bench_L9.log 2>&1
