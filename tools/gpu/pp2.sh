for v in def newton; do
  if [ $v = def ]; then L=""; else L=abx/$v.so; fi
  for c in cfg2_n65536 cfg2_n262144; do
    echo "== $v $c" >> gpurun_out/pp2.log
    EBEM_GPU_LIB=$L python tools/parity_probe.py $c 2>&1 | python -c "import json,sys; d=json.load(sys.stdin); print(d['rel_sample'], sum(d['probe_rel'])/len(d['probe_rel']), d['report']['identical'], d['report']['cells'])" >> gpurun_out/pp2.log
  done
done
