TILU_PLANE_DEBUG=1 timeout 300 python tools/plane_debug.py > gpurun_out/p4_debug_fwd.log 2>&1
timeout 300 python tools/plane_debug.py > gpurun_out/p4_debug.log 2>&1
timeout 600 python -m pytest tests/test_gpu_plane.py -q > gpurun_out/p4_plane_tests.log 2>&1; echo "rc=$?" >> gpurun_out/p4_plane_tests.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/p4_pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/p4_pytest_gpu.log
