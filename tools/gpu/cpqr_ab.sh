python -m pytest tests/test_gpu_basis.py tests/test_gpu_kernels.py tests/test_gpu_configs.py -q -x 2>&1 | tail -3 > gpurun_out/cpqr_ab.log
for v in 1 0; do
  echo "== EBEM_CPQR_WARP=$v" >> gpurun_out/cpqr_ab.log
  EBEM_CPQR_WARP=$v python tools/kernel_table.py 262144 2 2>&1 | grep -E "factorize|k_cpqr|k_qr_reduce" >> gpurun_out/cpqr_ab.log
done
python tools/parity_probe.py cfg2_n262144 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print('262144', d['rel_sample'], d['report']['identical'], d['report']['tie'], d['report']['cascade'])" >> gpurun_out/cpqr_ab.log
