for n in 4096 8192; do python tools/hybrid_probe.py $n >> gpurun_out/hyb2.log 2>&1; done
