for n in 4096 16384; do python tools/hybrid_probe.py $n >> gpurun_out/hyb.log 2>&1; done
EBEM_GEMM_LOG=1 python tools/repeat_probe.py 262144 1 2>&1 | grep "gemm launch" > gpurun_out/gemm_shapes.log
EBEM_VERBOSE=1 python tools/kernel_table.py 262144 2 > gpurun_out/verbose.log 2>&1
