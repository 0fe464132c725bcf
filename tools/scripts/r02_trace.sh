#!/bin/bash
# one GPU: per-iteration trace of the carried pre-threshold after a cold
# start (C4, fresh data), for the default build and predictor variants
mkdir -p gpurun_out
i=0
for fl in "" "-DSPARDL_DIV_EXTRAP=1.0" "-DSPARDL_DIV_EXTRAP=0.75 -DSPARDL_DIV_TARGET=1.3"; do
  make -B -j16 -C paper_2304_00737_b200/csrc EXTRA="$fl" > gpurun_out/tr_build_$i.log 2>&1
  echo "== [$fl]" > gpurun_out/trace_$i.log
  timeout 300 python tools/div_trace.py 138000000 8 70 >> gpurun_out/trace_$i.log 2>&1
  echo "trace $i rc=$?"
  if [ $i = 0 ]; then timeout 300 python bench.py --no-e2e --no-cpu --steps 20 --warmup 5 > gpurun_out/tr_bench.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/tr_bench.log; fi
  i=$((i+1))
done
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
