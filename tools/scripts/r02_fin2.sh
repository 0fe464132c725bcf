#!/bin/bash
# one GPU: finalize by dividing-list join -- parity suites, then the bench
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > gpurun_out/f2_build.log 2>&1 || { tail -20 gpurun_out/f2_build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_scale.py tests/test_gpu_components.py -x -q -m gpu > gpurun_out/f2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/f2_pytest.log
for r in 1 2; do
  timeout 300 python bench.py --no-e2e --no-cpu --steps 20 --warmup 5 > gpurun_out/f2_bench_$r.log 2>&1
  echo "run $r: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/f2_bench_$r.log) $(grep -o '"candidate_retries_timed_steps": [0-9]*' gpurun_out/f2_bench_$r.log) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/f2_bench_$r.log)"
done
timeout 300 python bench.py --no-e2e --no-cpu --steps 20 --warmup 5 --config c2 > gpurun_out/f2_bench_c2.log 2>&1
echo "c2: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/f2_bench_c2.log) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/f2_bench_c2.log)"
