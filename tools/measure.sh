#!/bin/bash
# Round measurement on a B200 box (run under gpurun from the repo root):
#   gpu parity tests -> bench line -> ncu launch list -> one ncu --set full capture of the top kernels.
# Each ncu pass only runs after the same command exited 0 without ncu.  Outputs go to gpurun_out/$TAG*.
TAG=${TAG:-r01}
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest_gpu.log
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err || exit 1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu --e2e-sweeps 0 > $O/${TAG}_plain.json 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${TAG}_ncu_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --e2e-sweeps 0 > $O/${TAG}_ncu_launch.log 2>&1
timeout 300 python tools/prof_batch.py --sweeps 3 > $O/${TAG}_prof_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_batch_(fwd|bwd)" -s 2 -c 2 -o $O/${TAG}_full -f \
    python tools/prof_batch.py --sweeps 3 > $O/${TAG}_ncu_full.log 2>&1
ncu -i $O/${TAG}_full.ncu-rep --page raw --csv > $O/${TAG}_full_raw.csv 2>/dev/null
echo done
