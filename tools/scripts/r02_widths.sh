#!/bin/bash
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > gpurun_out/wd_build.log 2>&1 || { tail -20 gpurun_out/wd_build.log; exit 1; }
SPARDL_DEBUG=1 timeout 300 python bench.py --no-e2e --no-cpu --steps 5 --warmup 3 2>&1 | grep -i "select batch\|resident clusters" | sort | uniq | head -20
timeout 1200 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_components.py tests/test_gpu_scale.py -x -q -m gpu > gpurun_out/wd_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/wd_pytest.log
for rep in 1 2; do
for ev in "SPARDL_SEL_WIDTHS_R1=0" "SPARDL_SEL_WIDTHS_R1=1"; do
for c in c4 c2; do
  env $ev timeout 300 python bench.py --no-e2e --no-cpu --steps 50 --warmup 10 --config $c > gpurun_out/wd_b.log 2>&1
  echo "$c [$ev]: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/wd_b.log) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/wd_b.log)"
done
done
done
