# ncu evidence for block time steps (host-driven loop, so every kernel is an eager launch)
mkdir -p gpurun_out
CMD="python bench.py --integrator block --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
NBODY_NO_GRAPH=1 timeout 900 $CMD > gpurun_out/block_prof_plain.log 2>&1 && \
NBODY_NO_GRAPH=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/block_launches.csv $CMD > gpurun_out/block_ncu_launches.log 2>&1 && \
NBODY_NO_GRAPH=1 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:force_kernel -s 300 -c 1 -o gpurun_out/prof_block_force -f $CMD > gpurun_out/block_ncu_full.log 2>&1
echo "block prof rc=$?"
