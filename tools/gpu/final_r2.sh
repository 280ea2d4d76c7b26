# round-2 final measurement set at HEAD ($1 = commit):
# calibration, the bench line, the bench command's ncu launch list, the
# experiment harness runs, and full ncu captures of the top kernels
set -x
bash tools/calibrate.sh $1 > gpurun_out/calibrate.log 2>&1
cp gpurun_out/calibration.json profiles/calibration.json
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_final.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-extra-configs > gpurun_out/ncu_bench.log 2>&1
mkdir -p gpurun_out/harness
python -m paper_2411_18026_b200.harness scaling --n-max 262144 --omega 1 --epsilon 1e-10 --leaf 32 --out gpurun_out/harness/scaling.csv > gpurun_out/harness/scaling.log 2>&1
python -m paper_2411_18026_b200.harness multi_rhs --n 65536 --omega 4 --rhs-count 180 --epsilon 1e-10 --out gpurun_out/harness/multi_rhs.csv > gpurun_out/harness/multi_rhs.log 2>&1
python -m paper_2411_18026_b200.harness error_table --out gpurun_out/harness/error_table.csv > gpurun_out/harness/error_table.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_near_sym -s 40 -c 1 -o gpurun_out/final_near_sym python tools/repeat_probe.py 262144 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_getrs_blk -s 4 -c 1 -o gpurun_out/final_getrs_blk python tools/repeat_probe.py 262144 1 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_tsqr -s 8 -c 1 -o gpurun_out/final_tsqr python tools/repeat_probe.py 262144 1 > /dev/null 2>&1
