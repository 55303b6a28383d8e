timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/p23_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p23_pytest_gpu.log
LEVEL=8 SWEEPS=10 SCHED=plane timeout 300 python tools/plane_bench.py > gpurun_out/p23_bench_L8.log 2>&1
LEVEL=8 SWEEPS=10 SCHED=plane FAST=1 timeout 300 python tools/plane_bench.py > gpurun_out/p23_bench_L8f.log 2>&1
LEVEL=9 SWEEPS=5 SCHED=plane timeout 900 python tools/plane_bench.py > gpurun_out/p23_bench_L9.log 2>&1
