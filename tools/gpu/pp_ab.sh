# A/B of the thread-per-pair fill (EBEM_FILL_PP) : bitwise solution check + kernel table
for N in 16384 262144; do
  EBEM_FILL_PP=0 python tools/bitcmp.py $N gpurun_out/x0_$N.npy > gpurun_out/pp_ab.log 2>&1
  EBEM_FILL_PP=1 python tools/bitcmp.py $N gpurun_out/x1_$N.npy >> gpurun_out/pp_ab.log 2>&1
  python tools/bitcmp.py --cmp gpurun_out/x0_$N.npy gpurun_out/x1_$N.npy >> gpurun_out/pp_ab.log 2>&1
done
for v in 0 1; do echo "== EBEM_FILL_PP=$v" >> gpurun_out/pp_ab.log
EBEM_FILL_PP=$v python tools/kernel_table.py 262144 2 2>&1 | head -16 >> gpurun_out/pp_ab.log; done
rm -f gpurun_out/x*.npy
