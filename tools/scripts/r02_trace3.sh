#!/bin/bash
# one GPU: fresh i.i.d. gradient windows -- cold-start trace + the driver's
# bench shape (20 steps, 5 warm-up) per predictor variant
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > gpurun_out/tr3_build.log 2>&1 || { tail -20 gpurun_out/tr3_build.log; exit 1; }
timeout 600 python bench.py --no-cpu --steps 20 --warmup 5 > gpurun_out/tr3_bench_full.log 2>&1; echo "full bench rc=$?"; grep '^{' gpurun_out/tr3_bench_full.log | head -c 2500; echo
i=0
for fl in "" "-DSPARDL_DIV_EXTRAP=1.0" "-DSPARDL_DIV_EXTRAP=0.75 -DSPARDL_DIV_TARGET=1.15" "-DSPARDL_DIV_EXTRAP=0.5 -DSPARDL_DIV_TARGET=1.1"; do
  [ -n "$fl" ] && make -B -j16 -C paper_2304_00737_b200/csrc EXTRA="$fl" > gpurun_out/tr3_build_$i.log 2>&1
  echo "== [$fl]" > gpurun_out/trace3_$i.log
  timeout 300 python tools/div_trace.py 138000000 8 100 >> gpurun_out/trace3_$i.log 2>&1
  for r in 1 2; do
    timeout 300 python bench.py --no-e2e --no-cpu --steps 20 --warmup 5 > gpurun_out/tr3_bench_${i}_$r.log 2>&1
    echo "[$fl] run $r: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/tr3_bench_${i}_$r.log) $(grep -o '"dense_fallbacks_timed_steps": [0-9]*' gpurun_out/tr3_bench_${i}_$r.log) $(grep -o '"phases_ms": {[^}]*}' gpurun_out/tr3_bench_${i}_$r.log)"
  done
  i=$((i+1))
done
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
