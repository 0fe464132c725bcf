#!/bin/bash
# launch list + full captures of the named kernels (after a clean plain run)
mkdir -p gpurun_out
python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/plain.log 2>&1 || { echo plain failed; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ncu.log 2>&1
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
      -o gpurun_out/prof_$k python bench.py --profile-only --steps 3 --warmup 3 > gpurun_out/ncu_full_$k.log 2>&1
done
