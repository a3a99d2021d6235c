# block time steps after the fused decide / fused tile-split corrector (round 2), one GPU:
# block tests, fuzz, debug-checks build, bench lines and a warm-L2 launch list at C2
mkdir -p gpurun_out
python -m pytest tests/test_gpu_block.py tests/test_gpu_fuzz.py tests/test_gpu_debug_checks.py tests/test_gpu_exchange.py tests/test_gpu_checkpoint.py -q -rf > gpurun_out/r02d_tests.log 2>&1
: > gpurun_out/r02d_block_bench.jsonl
for spec in "C2 --dt-max 0.0078125" "C3 --dt-max 0.0078125" "C4 --dt-max 0.0078125" "C4 --dt-max 0.0009765625"; do
  set -- $spec
  timeout 900 python bench.py --integrator block --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --config $spec 2>gpurun_out/r02d_bb_$1.err | tail -1 >> gpurun_out/r02d_block_bench.jsonl
done
NBODY_NO_GRAPH=1 timeout 600 python bench.py --integrator block --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r02d_plain.log 2>&1 && \
NBODY_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
  --log-file gpurun_out/r02d_block_launches_C2.csv python bench.py --integrator block --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r02d_ncu.log 2>&1
