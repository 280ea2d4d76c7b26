# calibration at HEAD, the bench line, and the ncu launch list of the bench command
bash tools/calibrate.sh $1 > gpurun_out/calibrate.log 2>&1
cp gpurun_out/calibration.json profiles/calibration.json
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra-configs > gpurun_out/ncu_bench.log 2>&1
