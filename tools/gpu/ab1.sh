for v in default minb1 t128m3; do
  if [ $v = default ]; then L=""; else L=abx/$v.so; fi
  echo "== $v" >> gpurun_out/ab1.log
  EBEM_GPU_LIB=$L python tools/repeat_probe.py 262144 2 --prof >> gpurun_out/ab1.log 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:k_near_pts -s 20 -c 1 -o gpurun_out/near_pts python tools/repeat_probe.py 262144 1 > gpurun_out/ncu1.log 2>&1
