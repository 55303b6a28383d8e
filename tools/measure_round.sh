#!/bin/bash
# Round measurement on one B200 (run under gpurun from the repo root):  T=<tag> bash tools/measure_round.sh
#   GPU parity tests -> bench line (config 4 headline + config 3 leg) -> reference arm -> ncu launch list
#   of the bench -> one ncu --set full capture of the plane kernels (config 3, L9) and of the batched
#   kernels (config 4).  Each ncu pass runs only after the same command exited 0 without ncu.
O=gpurun_out; T=${T:-r02}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_pytest_gpu.log 2>&1; echo "rc=$?" >> $O/${T}_pytest_gpu.log
timeout 900 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err || exit 1
timeout 900 python bench.py --impl reference > $O/${T}_ref.json 2> $O/${T}_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_ncu_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --e2e-sweeps 0 --config3-sweeps 10 > $O/${T}_ncu_launch.log 2>&1
LEVEL=9 SWEEPS=4 COEF=sin timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_plane_(fwd|bwd)" \
    -s 4 -c 2 -o $O/${T}_plane_full -f python tools/plane_bench.py > $O/${T}_plane_ncu.log 2>&1
ncu -i $O/${T}_plane_full.ncu-rep --page raw --csv > $O/${T}_plane_full_raw.csv 2>/dev/null
rm -f $O/${T}_plane_full.ncu-rep   # gpurun copies back at most 64 MiB: keep the exported pages only
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_batch_(fwd|bwd)" -s 2 -c 2 \
    -o $O/${T}_batch_full -f python tools/prof_batch.py --sweeps 3 > $O/${T}_batch_ncu.log 2>&1
ncu -i $O/${T}_batch_full.ncu-rep --page raw --csv > $O/${T}_batch_full_raw.csv 2>/dev/null
rm -f $O/${T}_batch_full.ncu-rep
echo done
