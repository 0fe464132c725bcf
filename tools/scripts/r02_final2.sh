#!/bin/bash
# one GPU, final code: build, the whole GPU suite, smoke, the default bench, the launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f2x_build.log 2>&1; echo "build rc=$?"
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/f2x_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f2x_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2x_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f2x_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f2x_bench.log 2>&1; echo "bench rc=$?"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/f2x_bench.log | head -1
TAG=f2x LAST=30 bash tools/scripts/r02_launch.sh | tail -3
