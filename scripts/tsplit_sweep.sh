# block-step time per dt_max vs the tile-split thresholds (1 GPU):
#   NBODY_TSPLIT1_MAX (scalar tile-split) x NBODY_TSPLIT_MAX (packed tile-split)
# usage: bash scripts/tsplit_sweep.sh [out.jsonl] [configs] [pairs "tmax:t1max ..."]
mkdir -p gpurun_out
out=${1:-gpurun_out/tsplit_sweep.jsonl}
cfgs=${2:-"C2 C3 C4"}
pairs=${3:-"0:0 1024:0 1024:32 1024:64 1024:128 1024:256 1024:512"}
: > $out
run() {   # cfg tmax t1max
  NBODY_TSPLIT_MAX=$2 NBODY_TSPLIT1_MAX=$3 timeout 600 python bench.py --integrator block --config $1 \
    --dt-max 0.0078125 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | \
    python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'config':'$1','tsplit_max':$2,'tsplit1_max':$3,'ms_per_dt_max':d['ms_per_step'],'value':d['value'],'block_steps':d['config']['block_steps_per_step']}))" \
    >> $out
}
for cfg in $cfgs; do
  for p in $pairs; do run $cfg ${p%%:*} ${p##*:}; done
done
cat $out
