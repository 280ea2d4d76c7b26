python tools/solve_profile.py 262144 1 > gpurun_out/solve_plain.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/solve_profile.py 262144 1 > gpurun_out/solve_ncu.csv 2>&1
