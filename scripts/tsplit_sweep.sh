# block-step time per dt_max vs the tile-split threshold NBODY_TSPLIT_MAX (1 GPU)
mkdir -p gpurun_out
: > gpurun_out/tsplit_sweep.jsonl
for cfg in C3 C4; do
  for tmax in 0 256 1024 4096 16384; do
    NBODY_TSPLIT_MAX=$tmax timeout 600 python bench.py --integrator block --config $cfg --dt-max 0.0078125 \
      --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'config':'$cfg','tsplit_max':$tmax,'ms_per_dt_max':d['ms_per_step'],'value':d['value'],'block_steps':d['config']['block_steps_per_step']}))" \
      >> gpurun_out/tsplit_sweep.jsonl
  done
done
cat gpurun_out/tsplit_sweep.jsonl
