#!/bin/bash
mkdir -p gpurun_out
make -B -j16 -C paper_2304_00737_b200/csrc EXTRA=-DSPARDL_STAMPS=1 > /dev/null 2>&1
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29640 tools/dbg_coop_multi.py > gpurun_out/coop_stamps_$N.log 2>&1
echo rc=$?; grep "step" gpurun_out/coop_stamps_$N.log
make -B -j16 -C paper_2304_00737_b200/csrc > /dev/null 2>&1
