for v in 0 1; do
EBEM_FILL_PP=$v ncu --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum --clock-control none -k regex:"k_near_sym|k_near_pp|k_proxy" --csv --log-file gpurun_out/pp_tiers_$v.csv python tools/repeat_probe.py 262144 1 > /dev/null 2>&1
done
