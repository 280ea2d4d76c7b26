# Round-1 profile pass (run on the GPU box from the repo root): bench line,
# ncu launch list of the same bench command, full captures of the top kernels.
set -x
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_launch.log 2>&1
for k in k_near_sym k_proxy_pairs k_tsqr; do
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 12 -c 1 -o gpurun_out/r1_full_$k python tools/repeat_probe.py 65536 1 > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
