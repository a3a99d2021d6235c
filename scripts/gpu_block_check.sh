mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_block.log 2>&1; echo "rc=$?"
tail -40 gpurun_out/pytest_block.log
