for key in 7,36 18,32 4,36 12,36; do
TILU_PLANE_KEY=$key LEVEL=9 SWEEPS=5 SCHED=plane timeout 600 python tools/plane_bench.py > gpurun_out/p29_L9_key$key.log 2>&1
done
