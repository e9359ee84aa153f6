python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1
python bench.py --config cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01d/launches_cfg2.csv python bench.py --config cfg2 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01d/launches_cfg5.csv python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
if [ -n "$NCU_K" ]; then ncu --set full --clock-control none --import-source on -k regex:$NCU_K -c 1 -o gpurun_out/r01d/full_$NCU_K -f python bench.py --config ${NCU_CFG:-cfg2} --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; fi
