# round-2 evidence pass on one B200: full GPU suite, bench line, block-step bench lines,
# launch list + one ncu --set full capture of the force kernel (bench command)
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -rf > gpurun_out/r02e_gputests.log 2>&1
python bench.py > gpurun_out/r02e_bench.log 2>&1
: > gpurun_out/r02e_block_bench.jsonl
for spec in "C2 --dt-max 0.0078125" "C3 --dt-max 0.0078125" "C4 --dt-max 0.0078125"; do
  set -- $spec
  timeout 900 python bench.py --integrator block --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --config $spec 2>gpurun_out/r02e_bb_$1.err | tail -1 >> gpurun_out/r02e_block_bench.jsonl
done
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/r02e_prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02e_launches.csv $CMD > gpurun_out/r02e_ncu_launches.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:force_kernel -s 1 -c 1 -o gpurun_out/r02e_prof_force -f $CMD > gpurun_out/r02e_ncu_full.log 2>&1
echo "prof rc=$?"
