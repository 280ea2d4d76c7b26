# piecewise near-field planning at the upper levels: bitwise A/B against the
# previous commit's library (abx/headrev.so), timing
set -x
for n in 4096 65536; do
  EBEM_GPU_LIB=abx/headrev.so python tools/bitcmp.py $n gpurun_out/h0_$n.npy
  python tools/bitcmp.py $n gpurun_out/h1_$n.npy
  python tools/bitcmp.py --cmp gpurun_out/h0_$n.npy gpurun_out/h1_$n.npy
done
rm -f gpurun_out/h?_*.npy
EBEM_GPU_LIB=abx/headrev.so python tools/repeat_probe.py 262144 4 | tail -2
python tools/repeat_probe.py 262144 4 | tail -2
