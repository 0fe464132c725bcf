#!/bin/bash
# one GPU: select flat group stream + merge-path occupancy -- parity, bench
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > gpurun_out/fl_build.log 2>&1 || { tail -20 gpurun_out/fl_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_components.py tests/test_gpu_scale.py -x -q -m gpu > gpurun_out/fl_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/fl_pytest.log
for c in c4 c2; do
  timeout 300 python bench.py --no-e2e --no-cpu --steps 50 --warmup 10 --config $c > gpurun_out/fl_bench_$c.log 2>&1
  echo "$c: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/fl_bench_$c.log) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/fl_bench_$c.log)"
done
timeout 300 python bench.py --no-e2e --no-cpu --steps 20 --warmup 5 > gpurun_out/fl_bench_driver.log 2>&1
echo "c4 20/5: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/fl_bench_driver.log)"
