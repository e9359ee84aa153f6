# iteration run: GPU tests, per-stage timing experiments, cfg2/cfg5 bench lines
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tests/probes/dbgrun.sh 2>&1 | grep "dbg=[0-7] " | grep -E "dbg=(0|7|6|5|3)"
python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/b2.log 2>&1
python bench.py --config cfg5 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b5.log 2>&1
