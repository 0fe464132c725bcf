#!/bin/bash
# one GPU, final code: build, the whole GPU suite, smoke, the default bench, the launch list, the reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f3_build.log 2>&1; echo "build rc=$?"
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/f3_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f3_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f3_bench.log 2>&1; echo "bench rc=$?"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/f3_bench.log | head -1
TAG=f3 LAST=30 bash tools/scripts/r02_launch.sh | tail -2
( time timeout 1200 python bench.py --impl reference --steps 3 --warmup 3 ) > gpurun_out/f3_ref.log 2>&1; echo "ref rc=$?"; grep '^{' gpurun_out/f3_ref.log | head -c 600
