#!/bin/bash
# 4 GPUs: multi-GPU suites, coop stamps at one worker per GPU, benches
mkdir -p gpurun_out
bash tools/scripts/r02_coop_stamps.sh
bash tools/scripts/r02_multi3.sh
