#!/bin/bash
# launch list of one bench step: capture_launch.sh <outdir> <workload> [bench args]
OUT=$1; WL=$2; shift 2
mkdir -p "$OUT"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file "$OUT/launches_${WL}.csv" \
    python bench.py --config "$WL" --steps 1 --warmup 3 --no-cpu-baseline "$@" > "$OUT/ncu_launch_${WL}.log" 2>&1
