# GPU round-trip: parity tests, smoke, bench (1 GPU).  Usage: bash scripts/gpu_check.sh [pytest-args]
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider ${1:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -5 gpurun_out/bench.log
timeout 600 python bench.py --integrator leapfrog --no-cpu-baseline > gpurun_out/bench_lf.log 2>&1; echo "bench lf rc=$?"; tail -2 gpurun_out/bench_lf.log
