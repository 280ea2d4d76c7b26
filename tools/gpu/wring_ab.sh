python -m pytest tests/test_gpu_solve_kernels.py tests/test_gpu_fds.py tests/test_gpu_conv.py -q -x 2>&1 | tail -n 2
for v in 0 1 0 1; do echo "== WRING=$v"; EBEM_GETRS_WRING=$v python tools/solve_profile.py 262144 1 2>&1 | tail -n 1; done
python -m pytest tests/test_gpu_configs.py -q -x 2>&1 | tail -n 1
