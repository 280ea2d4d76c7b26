# Round-1 profile pass v3 (GPU box, repo root): ncu launch list of the bench
# command, full captures of the top kernels at the bench size (N = 262144).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_v3.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_launch_v3.log 2>&1
echo "launch rc=$?"
for k in "k_near_sym:2" "k_proxy_pairs:2" "k_tsqr:1" "k_getrs:1" "k_cpqr:1"; do
  name=${k%%:*}; cnt=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$name --launch-skip 2 -c $cnt -o gpurun_out/r1_full_v3_$name python tools/repeat_probe.py 262144 1 > gpurun_out/ncu_v3_$name.log 2>&1
  echo "$name rc=$?"
done
ls -la gpurun_out
