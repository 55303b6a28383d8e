TILU_PLANE_DEBUG=1 timeout 300 python tools/plane_debug.py > gpurun_out/p3_debug_fwd.log 2>&1
timeout 300 python tools/plane_debug.py > gpurun_out/p3_debug.log 2>&1
