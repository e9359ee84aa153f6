#!/bin/bash
# ncu evidence for the round's final pipeline after the fused true residual
# (k_pcg_fdl<3,4,FUSED>, k_pcg_fdg<3,FUSED>).  Run on the GPU box after the
# same bench commands exited 0 without ncu.  Usage: capture_r02_s5.sh <outdir>
# Then, here: python profiles/summarize.py <outdir> profiles/r02
OUT=${1:-gpurun_out/r02s5}
mkdir -p "$OUT"
for wl in cfg5 cfg5_tensor cfg2 cfg3 cfg1; do
  python bench.py --config $wl --no-cpu-baseline > "$OUT/bench_${wl}.json" 2> "$OUT/bench_${wl}.err" || exit 1
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file "$OUT/launches_${wl}.csv" python bench.py --config $wl --steps 1 --warmup 3 --no-cpu-baseline \
      > "$OUT/ncu_launch_${wl}.log" 2>&1
done
full() {   # <kernel regex> <name> <bench args...>
  local k=$1 n=$2; shift 2
  ncu --set full --clock-control none --import-source on -k regex:"$k" -c 1 -o "$OUT/$n" -f \
      python bench.py "$@" --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/ncu_$n.log" 2>&1
}
full '^k_pcg_fdl' k_pcg_fdl_cfg5 --config cfg5
full '^k_pcg_fdg' k_pcg_fdg_cfg5_tensor --config cfg5_tensor
full 'k_stencil_box' k_stencil_box_cfg5 --config cfg5
full 'k_stencil_box' k_stencil_box_cfg5_tensor --config cfg5_tensor
full '^k_combine_points_tiled' k_combine_points_tiled_cfg5 --config cfg5
full 'k_metric_box' k_metric_box_cfg5 --config cfg5
full 'k_rhs_box_stage' k_rhs_box_stage_cfg5 --config cfg5
full '^k_pcg_fd<' k_pcg_fd_cfg5 --config cfg5
full '^k_fdl_factor' k_fdl_factor_cfg5 --config cfg5
full '^k_pcg_fdl' k_pcg_fdl_cfg3 --config cfg3
ls "$OUT"
# the .ncu-rep files exceed gpurun's 64 MiB return limit: summarise on the box
# (profiles/summarize.py -> text under $OUT/txt) and keep only the text
if [ -n "$SUMMARIZE_ON_BOX" ]; then
  cp profiles/traffic.json "$OUT/traffic.before.json" 2>/dev/null
  python profiles/summarize.py "$OUT" "$OUT/txt" > "$OUT/summarize.log" 2>&1
  cp profiles/traffic.json "$OUT/txt/traffic.json"
  rm -f "$OUT"/*.ncu-rep
fi
