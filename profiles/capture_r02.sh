#!/bin/bash
# ncu evidence behind profiles/r02/ (run on the GPU box, one GPU, after the
# same bench command exited 0 without ncu).  Usage: capture_r02.sh <outdir> [cfg]
set -e
OUT=${1:-gpurun_out/r02}; CFG=${2:-cfg5}
mkdir -p "$OUT"
B="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline"
# launch list: per-launch durations of every kernel of the bench run
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file "$OUT/launches_${CFG}.csv" $B > "$OUT/ncu_launch_${CFG}.log" 2>&1
# full section sets of the hot kernels (first launch of each)
for k in k_assemble_fast k_metric k_combine_points_tiled k_pcg_fdl k_pcg_fd; do
  ncu --set full --clock-control none --import-source on -k regex:"^${k}" -c 1 \
      -o "$OUT/${k}_${CFG}" -f $B > "$OUT/ncu_${k}_${CFG}.log" 2>&1 || true
done
