# Interleaved A/B of block-step time per dt_max on one GPU over several library builds,
# two rounds, C2 and C3 (dt_max = 1/128):
#   bash scripts/ab_block.sh OUT.jsonl new=- old=scripts/sweep/lib_old.so ...   ("-": in-tree build)
OUT=$1; shift
mkdir -p gpurun_out; : > $OUT
for r in 1 2; do
  for spec in "$@"; do
    name=${spec%%=*}; lib=${spec#*=}
    if [ "$lib" = "-" ]; then unset NBODY_LIB; else export NBODY_LIB=$PWD/$lib; fi
    for cfg in C2 C3; do
      python bench.py --integrator block --dt-max 0.0078125 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
        --config $cfg 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'lib':'$name','run':$r,'config':'$cfg','ms_per_dt_max':d['ms_per_step'],'block_steps':d['config']['block_steps_per_step']}))" >> $OUT
    done
  done
done
unset NBODY_LIB
