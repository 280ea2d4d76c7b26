for v in def cplx2 cplx2t128 symt128 def; do
  if [ $v = def ]; then L=""; else L=abx/$v.so; fi
  echo "== $v" >> gpurun_out/ab6.log
  EBEM_GPU_LIB=$L python tools/repeat_probe.py 262144 2 --prof 2>&1 | tail -1 >> gpurun_out/ab6.log
done
