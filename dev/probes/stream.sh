python -m pytest tests -m gpu -x -q > gpurun_out/pytest_all.log 2>&1; tail -1 gpurun_out/pytest_all.log
python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_cfg2.log 2>&1
SGIGA_STREAM_LONG=1 python bench.py --no-cpu-baseline --steps 20 > gpurun_out/bench_cfg2_long.log 2>&1
python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1
