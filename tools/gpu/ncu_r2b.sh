# full captures (with source) of the two top kernels at HEAD
ncu --set full --import-source on --clock-control none -k regex:k_near_sym -s 40 -c 1 -o gpurun_out/near_sym_r2b python tools/repeat_probe.py 262144 1 > gpurun_out/ncu_near.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tsqr -s 8 -c 1 -o gpurun_out/tsqr_r2b python tools/repeat_probe.py 262144 1 > gpurun_out/ncu_tsqr.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_proxy_pairs -s 20 -c 1 -o gpurun_out/proxy_r2b python tools/repeat_probe.py 262144 1 > gpurun_out/ncu_proxy.log 2>&1
