# Interleaved A/B of block-step time per dt_max on one GPU: the in-tree library ("new")
# against another build ("old", NBODY_LIB=$1), two rounds, C2 and C3 (dt_max = 1/128).
#   bash scripts/ab_block.sh scripts/sweep/lib_old.so gpurun_out/ab.jsonl
OLD=$1; OUT=${2:-gpurun_out/ab_block.jsonl}
mkdir -p gpurun_out; : > $OUT
for r in 1 2; do
  for v in new old; do
    if [ $v = old ]; then export NBODY_LIB=$PWD/$OLD; else unset NBODY_LIB; fi
    for cfg in C2 C3; do
      python bench.py --integrator block --dt-max 0.0078125 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
        --config $cfg 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$v','run':$r,'config':'$cfg','ms_per_dt_max':d['ms_per_step'],'block_steps':d['config']['block_steps_per_step']}))" >> $OUT
    done
  done
done
unset NBODY_LIB
