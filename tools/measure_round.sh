#!/bin/bash
# usage: T=<tag> bash tools/measure_round.sh  (default tag below)
# Round measurement: bench line (config 4 + single tet L9), ncu launch list, ncu full captures
# of the plane kernels (L9) and of the batched kernels (config 4).
O=gpurun_out; T=${T:-r01v17}
timeout 900 python -m pytest tests -m gpu -q > $O/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> $O/${T}_pytest_gpu.log
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_ncu_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --e2e-sweeps 0 --single-sweeps 2 > $O/${T}_ncu_launch.log 2>&1
LEVEL=9 SWEEPS=1 SCHED=plane ncu --set full --clock-control none --import-source on -k regex:"k_plane_(fwd|bwd)" -s 2 -c 2 \
    -o $O/${T}_plane_full -f python tools/plane_bench.py > $O/${T}_plane_ncu.log 2>&1
ncu -i $O/${T}_plane_full.ncu-rep --page raw --csv > $O/${T}_plane_full_raw.csv 2>/dev/null
echo done
