python -m pytest tests/test_gpu_fds.py tests/test_gpu_solve_kernels.py -q -x 2>&1 | tail -n 2
for v in 0 1 0 1; do echo "== SWEEP=$v"; EBEM_SWEEP=$v python tools/solve_profile.py 262144 1 2>&1 | tail -n 1; done
EBEM_SWEEP=0 python tools/bitcmp.py 65536 gpurun_out/x0.npy > /dev/null 2>&1; python tools/bitcmp.py 65536 gpurun_out/x1.npy > /dev/null 2>&1; python tools/bitcmp.py --cmp gpurun_out/x0.npy gpurun_out/x1.npy; rm -f gpurun_out/x*.npy
python -m pytest tests/test_gpu_configs.py -q -x 2>&1 | tail -n 1
