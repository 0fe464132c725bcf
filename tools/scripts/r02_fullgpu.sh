#!/bin/bash
# one GPU: the whole GPU suite (as the driver runs it) + smoke + the default bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fg_build.log 2>&1; echo "build rc=$?"
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/fg_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/fg_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fg_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/fg_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fg_bench.log 2>&1; echo "bench rc=$?"; grep -o '"ms_per_step": [0-9.]*' gpurun_out/fg_bench.log | head -1
