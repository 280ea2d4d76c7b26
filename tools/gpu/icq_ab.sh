python -m pytest tests/test_gpu_basis.py tests/test_gpu_fds.py tests/test_gpu_configs.py -q -x 2>&1 | tail -n 1
EBEM_GPU_LIB=abx/base.so python tools/bitcmp.py 65536 gpurun_out/x0.npy > /dev/null 2>&1; python tools/bitcmp.py 65536 gpurun_out/x1.npy > /dev/null 2>&1; python tools/bitcmp.py --cmp gpurun_out/x0.npy gpurun_out/x1.npy; rm -f gpurun_out/x*.npy
GREP="k_cpqr|k_interp" bash tools/gpu/ab_multi.sh icq
