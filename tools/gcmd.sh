mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_components.py tests/test_gpu_dropin.py -x -q -m gpu > gpurun_out/gt.log 2>&1
tail -1 gpurun_out/gt.log
bash run_ab.sh "|SPARDL_STEP_EVENTS=1" "|SPARDL_STEP_EVENTS=1" > gpurun_out/ab.log 2>&1
cat gpurun_out/ab.log | grep -v resident
python dbg_profile.py graph 2>&1 | head -5 | cut -c1-180
