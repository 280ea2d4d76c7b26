# kernel tables of several abx/ builds (names as args), two rounds each
: > gpurun_out/ab_multi.log
for r in 1 2; do for v in base "$@"; do
  echo "== $v" >> gpurun_out/ab_multi.log
  EBEM_GPU_LIB=abx/$v.so python tools/kernel_table.py 262144 2 2>&1 | grep -E "factorize|${GREP:-k_near|k_proxy}" >> gpurun_out/ab_multi.log
done; done
