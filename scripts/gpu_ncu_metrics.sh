# targeted ncu metrics: executed-flop counters + FMA sub-pipe split, for the force kernel (C4) and FP32 ubench kernels
set -x
mkdir -p gpurun_out
M=sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_ffma2_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fadd2_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_fmul2_pred_on.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_fmalite.sum,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.sum,sm__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/m_plain.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -k regex:force_kernel -s 1 -c 1 --csv --log-file gpurun_out/ncu_force_metrics.csv $CMD > gpurun_out/m_ncu.log 2>&1
./scripts/ubench_fp32 > gpurun_out/m_ub_plain.log 2>&1 && \
timeout 600 ncu --metrics $M --clock-control none -k regex:kern -c 40 --csv --log-file gpurun_out/ncu_ubench_metrics.csv ./scripts/ubench_fp32 > gpurun_out/m_ncu_ub.log 2>&1
echo done
