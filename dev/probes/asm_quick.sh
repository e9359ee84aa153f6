python -m pytest tests -m gpu -x -q -k "cfg2 or cfg5 or assembl or fast" > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for cfg in cfg2 cfg5; do SGIGA_ASM_DBG=${DBG:-0} python tests/gpu_probe_asm.py $cfg 2>&1 | grep asm-profile | tail -1; done > gpurun_out/asm_stages.log 2>&1
python bench.py --no-cpu-baseline --steps 10 > gpurun_out/bench_cfg2.log 2>&1
python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1
