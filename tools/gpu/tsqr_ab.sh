python -m pytest tests/test_gpu_tsqr.py tests/test_gpu_basis.py "tests/test_gpu_configs.py::test_config2_sweep_vs_reference" -q -x 2>&1 | tail -2 > gpurun_out/tsqr_ab.log
for cfg in "def 1 " "off 0 " "n80 1 abx/n80.so" "n96s96 1 abx/n96s96.so" "n96s32 1 abx/n96s32.so"; do
  set -- $cfg
  echo "== $1" >> gpurun_out/tsqr_ab.log
  EBEM_TSQR_V3=$2 EBEM_GPU_LIB=$3 python tools/kernel_table.py 262144 2 2>&1 | grep -E "factorize|k_qr_reduce|k_cpqr" >> gpurun_out/tsqr_ab.log
done
