python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/gputest2.log
bash tools/calibrate.sh $1 > gpurun_out/calibrate.log 2>&1
cp gpurun_out/calibration.json profiles/calibration.json 2>/dev/null
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.log 2>&1
