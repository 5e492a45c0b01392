python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/pytest.log
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5.log 2>&1
timeout 600 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/cfg2.log 2>&1
