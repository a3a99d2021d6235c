# block-step GPU tests only (1 GPU) -> gpurun_out/pytest_block.log
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_block.log 2>&1; echo "rc=$?"
tail -30 gpurun_out/pytest_block.log
bash scripts/gpu_block_bench.sh
