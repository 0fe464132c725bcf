#!/bin/bash
# A/B helper: rebuild with each EXTRA flag set and run the short bench.
# usage: run_ab.sh "-DFOO=1|ENV=1 ENV2=2" "-DFOO=2" ...   (part after | is env)
# BENCH_ARGS: extra bench.py arguments (default: C4, 50 steps)
mkdir -p gpurun_out
i=0; prev="__none__"
for x in "$@"; do
  fl="${x%%|*}"; ev=""; [[ "$x" == *"|"* ]] && ev="${x#*|}"
  if [ "$fl" != "$prev" ]; then
    make -B -j16 -C paper_2304_00737_b200/csrc EXTRA="$fl" > gpurun_out/ab_build_$i.log 2>&1; prev="$fl"
  fi
  env $ev timeout 300 python bench.py --no-e2e --no-cpu --steps 50 --warmup 10 ${BENCH_ARGS} > gpurun_out/ab_$i.log 2>&1
  echo "== $x"
  python - "$i" <<'PY'
import json,sys
ok=False
for l in open(f"gpurun_out/ab_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d=json.loads(l); ok=True
        print(d["ms_per_step"], d["phases_ms"], "fallbacks", d.get("dense_fallbacks_timed_steps"))
if not ok: print(open(f"gpurun_out/ab_{sys.argv[1]}.log").read()[-1500:])
PY
  i=$((i+1))
done
