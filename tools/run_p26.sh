for pd in 2 4; do
TILU_LIB=paper_2210_15280_b200/lib/libtilu_pd$pd.so timeout 300 python tools/plane_debug.py > gpurun_out/p26_debug_pd$pd.log 2>&1
TILU_LIB=paper_2210_15280_b200/lib/libtilu_pd$pd.so LEVEL=8 SWEEPS=10 SCHED=plane timeout 300 python tools/plane_bench.py > gpurun_out/p26_bench_L8_pd$pd.log 2>&1
done
for pd in 2 4; do
TILU_LIB=paper_2210_15280_b200/lib/libtilu_pd$pd.so LEVEL=9 SWEEPS=5 SCHED=plane timeout 600 python tools/plane_bench.py > gpurun_out/p26_bench_L9_pd$pd.log 2>&1
done
