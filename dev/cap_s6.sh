OUT=gpurun_out/r02s6; mkdir -p $OUT
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for wl in cfg5 cfg5_tensor cfg2 cfg3 cfg1; do python bench.py --config $wl --no-cpu-baseline > $OUT/bench_$wl.json 2> $OUT/bench_$wl.err; done
python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches_cfg5.csv python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_launch_cfg5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'^k_pcg_fdl' -c 1 -o $OUT/k_pcg_fdl_cfg5 -f python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_fdl.log 2>&1
python profiles/summarize.py $OUT $OUT/txt > $OUT/summarize.log 2>&1
rm -f $OUT/*.ncu-rep
python -c "import json; d=json.load(open('$OUT/bench_default.json')); print(d['ms_per_step'], d['value'], d['e2e']['value'])"
