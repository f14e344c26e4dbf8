nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 2>&1 | tail -45
timeout 300 python bench.py --config cfg1 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/r2c_cfg1.json 2>gpurun_out/r2c_cfg1.err
timeout 300 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_cfg4.json 2>gpurun_out/r2c_cfg4.err
cat gpurun_out/r2c_*.json; tail -n 5 gpurun_out/r2c_cfg1.err gpurun_out/r2c_cfg4.err
