python -m pytest tests/test_gpu_solve_kernels.py tests/test_gpu_fds.py tests/test_gpu_conv.py -q -x 2>&1 | tail -n 2
EBEM_GPU_LIB=abx/base.so python tools/bitcmp.py 65536 gpurun_out/x0.npy > /dev/null 2>&1; python tools/bitcmp.py 65536 gpurun_out/x1.npy > /dev/null 2>&1; python tools/bitcmp.py --cmp gpurun_out/x0.npy gpurun_out/x1.npy; rm -f gpurun_out/x*.npy
for l in base ""; do echo "== $l"; EBEM_GPU_LIB=${l:+abx/$l.so} python tools/kernel_table.py 262144 2 2>&1 | grep -E "factorize|k_getr"; done
