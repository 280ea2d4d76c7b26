python -m pytest tests/test_facade.py -m gpu -q -x -s 2>&1 | tail -30 > gpurun_out/facade.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.log 2>&1
