#!/bin/bash
# BASELINE.json config sweeps on the GPUs of this box (one JSON line each,
# appended to gpurun_out/sweeps_g<N>.jsonl)
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/sweeps_g$N.jsonl
run() {
  if [ "$N" -gt 1 ]; then
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps ${STEPS:-20} --warmup 5 --no-cpu --no-e2e "$@" 2>/dev/null | grep '^{' >> $OUT
  else
    timeout 900 python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu --no-e2e "$@" 2>/dev/null | grep '^{' >> $OUT
  fi
  echo "$* -> $(tail -1 $OUT | python -c 'import json,sys; d=json.load(sys.stdin); print(d["ms_per_step"], d["roofline"]["step_frac_of_roof"], d["ledger_per_step"]["measured"], d.get("dense_nccl_allreduce_ms"))' 2>/dev/null)"
}
case "${SWEEP:-all}" in
  c3|all) run --config c3; run --config c3 --teams 2 --sag rsag; run --config c3 --teams 3 --sag bsag ;;
esac
case "${SWEEP:-all}" in
  c4d|all)
    for d in 2 4 8; do for s in rsag bsag; do for g in iid corr; do run --config c4 --teams $d --sag $s --gen $g; done; done; done
    run --config c4 --gen corr ;;
esac
case "${SWEEP:-all}" in
  c4d2) for d in 4 8; do for s in rsag bsag; do run --config c4 --teams $d --sag $s; done; done
        run --config c4 --teams 8 --sag bsag --gen corr ;;
esac
case "${SWEEP:-all}" in
  c5|all) for dens in ${DENS:-0.001 0.0025 0.005 0.01}; do run --config c5 --density $dens; done ;;
esac
