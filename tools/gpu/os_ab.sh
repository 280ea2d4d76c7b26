EBEM_GPU_LIB=abx/base.so python tools/bitcmp.py 65536 gpurun_out/x0.npy > /dev/null 2>&1; python tools/bitcmp.py 65536 gpurun_out/x1.npy > /dev/null 2>&1; python tools/bitcmp.py --cmp gpurun_out/x0.npy gpurun_out/x1.npy; rm -f gpurun_out/x*.npy
GREP="k_near_one" bash tools/gpu/ab_multi.sh os1
