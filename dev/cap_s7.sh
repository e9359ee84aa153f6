# final evidence of the round (after k_metric_box_v / templated k_rhs_box_stage / fused residual)
OUT=gpurun_out/r02s7; mkdir -p $OUT
for wl in cfg5 cfg5_tensor cfg2 cfg3 cfg1; do python bench.py --config $wl --no-cpu-baseline > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err; done
python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for wl in cfg5 cfg5_tensor cfg2; do
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_$wl.csv python bench.py --config $wl --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_$wl.log 2>&1
done
full() { local k=$1 n=$2; shift 2; ncu --set full --clock-control none --import-source on -k regex:"$k" -c 1 -o $OUT/$n -f python bench.py "$@" --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_$n.log 2>&1; }
full 'k_metric_box_v' k_metric_box_v_cfg5 --config cfg5
full 'k_rhs_box_stage' k_rhs_box_stage_cfg5 --config cfg5
full '^k_pcg_fdl' k_pcg_fdl_cfg5 --config cfg5
python profiles/summarize.py $OUT $OUT/txt > $OUT/summarize.log 2>&1
rm -f $OUT/*.ncu-rep
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python -c "import json; d=json.load(open('$OUT/bench_default.json')); print(d['ms_per_step'], d['value'], d['e2e']['value'])"
