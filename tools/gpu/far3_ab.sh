# very-far 3 x 3 quadrature tier: solution A/B (EBEM_FAR3=0/1) and timing
set -x
for n in 16384 65536 262144; do
  EBEM_FAR3=0 python tools/bitcmp.py $n gpurun_out/f0_$n.npy
  EBEM_FAR3=1 python tools/bitcmp.py $n gpurun_out/f1_$n.npy
  python tools/bitcmp.py --cmp gpurun_out/f0_$n.npy gpurun_out/f1_$n.npy
done
rm -f gpurun_out/f?_*.npy
EBEM_FAR3=0 python tools/repeat_probe.py 262144 3 --prof | tail -2
EBEM_FAR3=1 python tools/repeat_probe.py 262144 3 --prof | tail -2
