python -m pytest tests/test_gpu_solve_kernels.py tests/test_gpu_fds.py tests/test_gpu_conv.py -q -x 2>&1 | tail -n 2
for mx in 0 64 148 300 600 2000; do echo "== BCOL_MAX=$mx"; EBEM_GETRS_BCOL_MAX=$mx python tools/solve_profile.py 262144 1 2>&1 | tail -n 1; done
