timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/p27_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p27_pytest_gpu.log
timeout 1200 python tools/configs_bench.py --configs 1,5 > gpurun_out/r01v16_configs.json 2> gpurun_out/r01v16_configs.err
