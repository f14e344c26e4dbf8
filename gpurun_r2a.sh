set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_chunks.py -m "gpu and not slow" -x -q --durations=15 2>&1 | tail -40
timeout 900 python -m pytest tests/test_gpu_walk.py tests/test_gpu_bench_dist.py -x -q --durations=10 2>&1 | tail -30
timeout 300 python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2a_cfg1.json 2>gpurun_out/r2a_cfg1.err
timeout 300 python bench.py --config cfg4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_cfg4.json 2>gpurun_out/r2a_cfg4.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_cfg5.json 2> gpurun_out/r2a_cfg5.err
cat gpurun_out/r2a_*.json; tail -5 gpurun_out/r2a_*.err
