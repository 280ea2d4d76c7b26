EBEM_FILL_PP=1 ncu --set full --import-source on --clock-control none -k regex:k_near_pp -s 40 -c 1 -o gpurun_out/near_pp_v1 python tools/repeat_probe.py 262144 1 > gpurun_out/ncu_pp.log 2>&1
