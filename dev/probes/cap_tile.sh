#!/bin/bash
# ncu evidence for the tiled assembly (run on the GPU box): launch list of a
# cfg5 bench step + full captures of k_assemble_tile on cfg5 / cfg5_tensor / cfg2
OUT=${1:-gpurun_out/r02t}
mkdir -p "$OUT"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file "$OUT/launches_cfg5.csv" \
    python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/ncu_launch_cfg5.log" 2>&1
for wl in cfg5 cfg5_tensor cfg2; do
  ncu --set full --clock-control none --import-source on -k regex:'^k_assemble_tile' -c 1 -o "$OUT/k_assemble_tile_$wl" -f \
      python bench.py --config $wl --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/ncu_tile_$wl.log" 2>&1
done
ls "$OUT"
