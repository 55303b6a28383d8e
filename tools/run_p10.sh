timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/p10_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p10_pytest_gpu.log
