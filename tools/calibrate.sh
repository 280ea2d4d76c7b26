#!/bin/bash
# Roofline calibration at the bench workload (config 2, N = 262144), run on
# the GPU box:  tools/calibrate.sh <commit>   -> gpurun_out/calibration.json
#  * executed FP64 flops per quadrature point of the fill kernels:
#    ncu (2 DFMA + DMUL + DADD thread instructions) over every launch of one
#    factorization / the points the library's profiler counts;
#  * DRAM bytes per launch of the fill kernels (same ncu pass);
#  * DMMA tensor-pipe activity and FP64-pipe activity of the merge GEMMs.
set -e
commit=${1:-unknown}
mkdir -p gpurun_out
python tools/calibrate_flops.py 262144 > gpurun_out/cal_points.log
ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:'k_near_sym|k_proxy_pairs|k_proxy_pp' --csv \
    python tools/calibrate_flops.py 262144 > gpurun_out/cal_fill.csv 2> gpurun_out/cal_fill.err
ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
    --clock-control none -k regex:k_gemm_mma --csv \
    python tools/calibrate_flops.py 262144 > gpurun_out/cal_gemm.csv 2> gpurun_out/cal_gemm.err
python tools/make_calibration.py "$commit" gpurun_out/cal_points.log gpurun_out/cal_fill.csv \
    gpurun_out/cal_gemm.csv > gpurun_out/calibration.json
cat gpurun_out/calibration.json
