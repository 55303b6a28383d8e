set -x
timeout 600 python -m pytest tests/test_gpu_plane.py -x -q > gpurun_out/p1_plane_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p1_plane_tests.log
LEVEL=7 SWEEPS=10 SCHED=plane,batch timeout 300 python tools/plane_bench.py > gpurun_out/p1_bench_L7.log 2>&1
LEVEL=8 SWEEPS=10 SCHED=plane,batch timeout 300 python tools/plane_bench.py > gpurun_out/p1_bench_L8.log 2>&1
LEVEL=8 SWEEPS=10 FAST=1 SCHED=plane timeout 300 python tools/plane_bench.py > gpurun_out/p1_bench_L8f.log 2>&1
nvcc -arch=sm_100a -O3 -o /tmp/fp64_lat tools/fp64_lat.cu && /tmp/fp64_lat > gpurun_out/p1_fp64_lat.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/p1_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p1_pytest_gpu.log
