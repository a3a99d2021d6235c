# ncu evidence for the bench command (1 GPU): plain run, then launch list, then full capture of the force kernel.
set -x
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-}"
timeout 600 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:force_kernel -s 1 -c 1 -o gpurun_out/prof_force -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "prof rc=$?"
tail -n 3 gpurun_out/prof_plain.log gpurun_out/ncu_launches.log gpurun_out/ncu_full.log
