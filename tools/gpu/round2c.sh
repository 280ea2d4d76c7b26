python -m pytest tests/test_gpu_configs.py tests/test_harness.py -m gpu -q -x 2>&1 | tail -4 > gpurun_out/t2c.log
mkdir -p gpurun_out/harness
python -m paper_2411_18026_b200.harness scaling --n-min 4096 --n-max 262144 --conv-max 4096 --omega 1 --epsilon 1e-10 --out gpurun_out/harness/scaling.csv > gpurun_out/harness/scaling.log 2>&1
python -m paper_2411_18026_b200.harness multi_rhs --n 65536 --omega 4 --rhs-count 180 --epsilon 1e-10 --out gpurun_out/harness/multi_rhs.csv > gpurun_out/harness/multi_rhs.log 2>&1
python -m paper_2411_18026_b200.harness error_table --out gpurun_out/harness/error_table.csv > gpurun_out/harness/error_table.log 2>&1
