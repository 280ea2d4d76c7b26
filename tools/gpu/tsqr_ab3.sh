: > gpurun_out/tsqr_ab3.log
for cfg in "def " "m8 abx/m8.so" "m8s8 abx/m8s8.so" "m8s8t8 abx/m8s8t8.so"; do
  set -- $cfg
  echo "== $1" >> gpurun_out/tsqr_ab3.log
  EBEM_GPU_LIB=$2 python -m pytest tests/test_gpu_tsqr.py tests/test_gpu_basis.py -q -x 2>&1 | tail -1 >> gpurun_out/tsqr_ab3.log
  EBEM_GPU_LIB=$2 python tools/kernel_table.py 262144 2 2>&1 | grep -E "factorize|k_qr_reduce|k_cpqr" >> gpurun_out/tsqr_ab3.log
done
