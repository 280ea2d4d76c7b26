bash tools/gpu/ab_base.sh 262144
python -m pytest tests/test_gpu_configs.py tests/test_gpu_kernels.py tests/test_gpu_basis.py -q -x > gpurun_out/ab_fastr_tests.log 2>&1
tail -3 gpurun_out/ab_fastr_tests.log >> gpurun_out/ab_base.log
