for v in def cplxlog symt128 minb6; do
  if [ $v = def ]; then L=""; else L=abx/$v.so; fi
  echo "== $v" >> gpurun_out/ab5.log
  EBEM_GPU_LIB=$L python tools/repeat_probe.py 262144 2 --prof >> gpurun_out/ab5.log 2>&1
done
