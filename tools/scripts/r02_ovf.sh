#!/bin/bash
mkdir -p gpurun_out
make -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_pipeline.py -x -q -m gpu -k "coop_overflow or select_paths or second_chance" > gpurun_out/ovf_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ovf_pytest.log
timeout 300 python bench.py --no-e2e --no-cpu --steps 50 --warmup 10 > gpurun_out/ovf_b.log 2>&1; echo "c4: $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ovf_b.log)"
