#!/bin/bash
# ncu capture of the 2-D assembly kernel (k_assemble2d) on a replicated
# batch (run on the GPU box after the same command exited 0 without ncu).
# Usage: capture_asm2d.sh <outdir> <cfg> <replicas>
set -e
OUT=${1:-gpurun_out}; CFG=${2:-cfg3}; R=${3:-1024}
mkdir -p "$OUT"
ncu --set full --clock-control none --import-source on -k regex:k_assemble2d -c 1 \
    -o "$OUT/asm2d_${CFG}_x${R}" -f python bench.py --config $CFG --replicas $R --steps 1 --warmup 3 --no-cpu-baseline \
    > "$OUT/ncu_asm2d_${CFG}.log" 2>&1
