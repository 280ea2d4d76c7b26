for cfg in "def " "nosleep abx/nosleep.so" "sleep5 abx/sleep5.so" "rpt16 abx/rpt16.so"; do
  set -- $cfg
  echo "== $1" >> gpurun_out/tsqr_ab2.log
  EBEM_GPU_LIB=$2 python tools/kernel_table.py 262144 2 2>&1 | grep -E "factorize|k_qr_reduce|k_cpqr" >> gpurun_out/tsqr_ab2.log
done
