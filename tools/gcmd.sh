mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_components.py -x -q -m gpu -k merge > gpurun_out/gt.log 2>&1
tail -2 gpurun_out/gt.log
