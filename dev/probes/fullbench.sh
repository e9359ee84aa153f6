python bench.py > gpurun_out/fb_cfg2.log 2>&1
python bench.py --config cfg5 --steps 5 --warmup 3 > gpurun_out/fb_cfg5.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fb_ref.log 2>&1
python bench.py --replicas 64 --no-cpu-baseline > gpurun_out/fb_r64.log 2>&1
python bench.py --config cfg3 --replicas 1024 --steps 5 --no-cpu-baseline > gpurun_out/fb_cfg3.log 2>&1
python bench.py --config cfg1 --replicas 1024 --steps 5 --no-cpu-baseline > gpurun_out/fb_cfg1.log 2>&1
