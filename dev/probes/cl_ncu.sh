#!/bin/bash
# one ncu --set full capture of the cluster assembly on cfg5
OUT=gpurun_out/cl; mkdir -p $OUT
env ${VARS} ncu --set full --clock-control none --import-source on -k regex:'^k_assemble_cl' -c 1 -o $OUT/${NAME:-cl} -f \
  python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_${NAME:-cl}.log 2>&1
tail -3 $OUT/ncu_${NAME:-cl}.log
