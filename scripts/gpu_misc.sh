mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_block.py -q --timeout 600 -p no:cacheprovider 2>&1 | tail -3
timeout 900 python scripts/cta_shape_timing.py > gpurun_out/cta_shapes.txt 2>&1; cat gpurun_out/cta_shapes.txt
