timeout 300 python tools/plane_debug.py > gpurun_out/p2_debug.log 2>&1
LEVEL=8 SWEEPS=4 SCHED=plane TILU_PLANE_CTAS_PER_SM=1 timeout 300 python tools/plane_bench.py > gpurun_out/p2_bench_L8_c1.log 2>&1
LEVEL=8 SWEEPS=2 SCHED=plane timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_plane_(fwd|bwd)" -s 2 -c 2 -o gpurun_out/p2_full -f python tools/plane_bench.py > gpurun_out/p2_ncu.log 2>&1
ncu -i gpurun_out/p2_full.ncu-rep --page raw --csv > gpurun_out/p2_full_raw.csv 2>/dev/null
ncu -i gpurun_out/p2_full.ncu-rep --page source --csv --print-source sass > gpurun_out/p2_source.csv 2>/dev/null
ls -la gpurun_out
