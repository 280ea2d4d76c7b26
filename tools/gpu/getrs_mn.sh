for l in base mn64 mn32; do echo "== $l"; EBEM_GPU_LIB=abx/$l.so python tools/solve180_profile.py 2>&1 | tail -n 1; EBEM_GPU_LIB=abx/$l.so python tools/kernel_table.py 262144 2 2>&1 | grep -E "factorize|k_getrs"; done
EBEM_GPU_LIB=abx/mn32.so python -m pytest tests/test_gpu_solve_kernels.py tests/test_gpu_fds.py -q -x 2>&1 | tail -n 2
