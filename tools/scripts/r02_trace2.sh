#!/bin/bash
# one GPU: second-chance candidate pass -- pipeline tests, then the cold-start
# trace and the driver's bench shape (20 steps, 5 warm-up) per predictor variant
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > gpurun_out/tr2_build.log 2>&1 || { tail -20 gpurun_out/tr2_build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q -m gpu > gpurun_out/tr2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/tr2_pytest.log
i=0
for fl in "" "-DSPARDL_DIV_EXTRAP=1.0" "-DSPARDL_DIV_EXTRAP=1.0 -DSPARDL_DIV_TARGET=1.1" "-DSPARDL_DIV_EXTRAP=0.75 -DSPARDL_DIV_TARGET=1.15"; do
  [ -n "$fl" ] && make -B -j16 -C paper_2304_00737_b200/csrc EXTRA="$fl" > gpurun_out/tr2_build_$i.log 2>&1
  echo "== [$fl]" > gpurun_out/trace2_$i.log
  timeout 300 python tools/div_trace.py 138000000 8 70 >> gpurun_out/trace2_$i.log 2>&1
  for r in 1 2; do
    timeout 300 python bench.py --no-e2e --no-cpu --steps 20 --warmup 5 > gpurun_out/tr2_bench_${i}_$r.log 2>&1
    echo "[$fl] run $r: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/tr2_bench_${i}_$r.log) $(grep -o '"dense_fallbacks_timed_steps": [0-9]*' gpurun_out/tr2_bench_${i}_$r.log)"
  done
  i=$((i+1))
done
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
