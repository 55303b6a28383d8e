LEVEL=8 SWEEPS=1 SCHED=plane TILU_PLANE_NTASKS=1 TILU_PLANE_TRACE=gpurun_out/p12_trace_1task.txt timeout 300 python tools/plane_bench.py > gpurun_out/p12_bench_1task.log 2>&1
LEVEL=8 SWEEPS=2 SCHED=plane TILU_PLANE_NTASKS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_plane_fwd" -s 2 -c 1 -o gpurun_out/p12_full -f python tools/plane_bench.py > gpurun_out/p12_ncu.log 2>&1
ncu -i gpurun_out/p12_full.ncu-rep --page source --csv --print-source sass > gpurun_out/p12_source.csv 2>/dev/null
ncu -i gpurun_out/p12_full.ncu-rep --page raw --csv > gpurun_out/p12_raw.csv 2>/dev/null
