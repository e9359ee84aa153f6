OUT=gpurun_out/r02b; mkdir -p $OUT
full() { local k=$1 n=$2; shift 2
  ncu --set full --clock-control none --import-source on -k regex:"$k" -c 1 -o "$OUT/$n" -f \
      python bench.py "$@" --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/ncu_$n.log" 2>&1; }
full '^k_metric' k_metric_cfg5 --config cfg5
full '^k_combine_points_tiled' k_combine_points_tiled_cfg5 --config cfg5
ls $OUT
