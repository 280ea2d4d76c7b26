# working tree vs abx/base.so: bitwise solution at 2N=2^19 + kernel tables
N=${1:-262144}
EBEM_GPU_LIB=abx/base.so python tools/bitcmp.py $N gpurun_out/x0.npy > gpurun_out/ab_base.log 2>&1
python tools/bitcmp.py $N gpurun_out/x1.npy >> gpurun_out/ab_base.log 2>&1
python tools/bitcmp.py --cmp gpurun_out/x0.npy gpurun_out/x1.npy >> gpurun_out/ab_base.log 2>&1
for cfg in "base abx/base.so" "new " "base abx/base.so" "new "; do
  set -- $cfg
  echo "== $1" >> gpurun_out/ab_base.log
  EBEM_GPU_LIB=$2 python tools/kernel_table.py $N 2 2>&1 | grep -E "factorize|k_near|k_proxy|${GREP:-k_near}" >> gpurun_out/ab_base.log
done
rm -f gpurun_out/x*.npy
