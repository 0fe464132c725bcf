#!/bin/bash
# A/B helper: rebuild with each EXTRA flag set and run the short bench.
# usage: run_ab.sh "-DFOO=1|ENV=1 ENV2=2" "-DFOO=2" ...   (part after | is env)
mkdir -p gpurun_out
i=0; prev="__none__"
for x in "$@"; do
  fl="${x%%|*}"; ev=""; [[ "$x" == *"|"* ]] && ev="${x#*|}"
  if [ "$fl" != "$prev" ]; then
    make -B -C paper_2304_00737_b200/csrc EXTRA="$fl" > gpurun_out/ab_build_$i.log 2>&1; prev="$fl"
  fi
  env $ev SPARDL_DEBUG=1 timeout 300 python bench.py --no-e2e --no-cpu --no-north-star --steps 100 --warmup 5 > gpurun_out/ab_$i.log 2>&1
  echo "== $x"; grep -E "resident|batch" gpurun_out/ab_$i.log | sort -u | tr '\n' ' '; echo
  python - "$i" <<'PY'
import json,sys
for l in open(f"gpurun_out/ab_{sys.argv[1]}.log"):
    if l.startswith("{"):
        d=json.loads(l); print(d["ms_per_step"], d["phases_ms"], d["roofline"]["achieved"])
PY
  i=$((i+1))
done
