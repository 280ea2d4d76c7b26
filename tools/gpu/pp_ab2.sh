N=262144
EBEM_FILL_PP=0 python tools/bitcmp.py $N gpurun_out/x0.npy > gpurun_out/pp_ab2.log 2>&1
EBEM_FILL_PP=1 python tools/bitcmp.py $N gpurun_out/x1.npy >> gpurun_out/pp_ab2.log 2>&1
python tools/bitcmp.py --cmp gpurun_out/x0.npy gpurun_out/x1.npy >> gpurun_out/pp_ab2.log 2>&1
for cfg in "old 0 " "mr3 1 " "mr2 1 abx/mr2.so" "mr6 1 abx/mr6.so"; do
  set -- $cfg
  echo "== $1" >> gpurun_out/pp_ab2.log
  EBEM_FILL_PP=$2 EBEM_GPU_LIB=$3 python tools/kernel_table.py 262144 2 2>&1 | grep -E "factorize|k_near|k_proxy" >> gpurun_out/pp_ab2.log
done
rm -f gpurun_out/x*.npy
