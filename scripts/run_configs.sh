# bench.py over every BASELINE.json config on 1 GPU -> gpurun_out/configs.jsonl
set -x
mkdir -p gpurun_out
: > gpurun_out/configs.jsonl
for spec in "C1 10" "C2 100" "C3 20" "C4 10" "C5 5" "PAPER 10"; do
  set -- $spec
  timeout 900 python bench.py --config $1 --steps $2 --warmup 3 --cpu-seconds 5 2>gpurun_out/bench_$1.err | tail -1 >> gpurun_out/configs.jsonl
done
timeout 900 python bench.py --config C4 --integrator leapfrog --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/configs.jsonl
timeout 900 python bench.py --config C5 --integrator leapfrog --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/configs.jsonl
timeout 900 python bench.py --config C4 --hilo on --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/configs.jsonl
# block time steps (R#28) and the loopback scaling projection
bash scripts/gpu_block_bench.sh
timeout 1500 python scripts/project_scaling.py --configs C3,C4,C5 --steps 2 > gpurun_out/scaling_proj.jsonl 2> gpurun_out/scaling_proj.err
