cd $GRAFT_REPO_ROOT
timeout 600 python tools/setup_mg_bench.py --mg > gpurun_out/g4_setup.log 2>&1; echo rc=$? >> gpurun_out/g4_setup.log
grep -v '^{"factorize"' gpurun_out/g4_setup.log | cut -c1-400
which compute-sanitizer; compute-sanitizer --version 2>&1 | head -3
timeout 600 compute-sanitizer --tool memcheck python tools/new_kernels_smoke.py > gpurun_out/g4_memcheck.log 2>&1; echo rc=$? >> gpurun_out/g4_memcheck.log
tail -15 gpurun_out/g4_memcheck.log
