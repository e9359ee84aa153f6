#!/bin/bash
# ncu captures behind profiles/<round>/ (run on the GPU box, one GPU, after
# the same bench command has exited 0 without ncu).  Usage: capture.sh <outdir>
set -e
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
for cfg in cfg2 cfg5; do
  # launch list: per-launch durations of every kernel of one bench run
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file "$OUT/launches_${cfg}.csv" python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline \
      > "$OUT/ncu_launch_${cfg}.log" 2>&1
  # full section set of the dominant kernel (first launch)
  ncu --set full --clock-control none --import-source on -k regex:k_assemble_fast -c 1 \
      -o "$OUT/asm_${cfg}" -f python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline \
      > "$OUT/ncu_full_${cfg}.log" 2>&1
done
