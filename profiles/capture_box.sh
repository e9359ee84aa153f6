OUT=gpurun_out/r02b
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_cfg5.csv python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_cfg5.log 2>&1
full() { local k=$1 n=$2; shift 2; ncu --set full --clock-control none --import-source on -k regex:"$k" -c 1 -o "$OUT/$n" -f python bench.py "$@" --steps 1 --warmup 3 --no-cpu-baseline > "$OUT/ncu_$n.log" 2>&1; }
full 'k_stencil_box' k_stencil_box_cfg5 --config cfg5
full 'k_metric_box' k_metric_box_cfg5 --config cfg5
full 'k_rhs_box_stage' k_rhs_box_stage_cfg5 --config cfg5
ls $OUT
