"""Top-k All-Gather baseline on the GPU.

inc/collectives.hpp:185-216: every worker selects the top-k of its whole
gradient (top_k_select_slice over [0, N): the dividing kernels), the P
selections are all-gathered, and every worker folds them with merge_add in
source order -- the union is kept unsparsified, so each worker receives
2(P-1)k scalars in ceil(log2 P) rounds (the ledger is returned, as the
reference's Fabric would record it).  One process per GPU; the selections
cross GPUs with one NCCL all-gather (torch.distributed), the selection and
the merge are this library's kernels.
"""
from __future__ import annotations

import math

from .api import merge_add, top_k_select_slice
from ._lib import ConfigError


def _fold(lists):
    acc = merge_add(*lists[:16])
    for s in range(16, len(lists), 15):        # left fold, <= 16 lists per merge
        acc = merge_add(acc, *lists[s:s + 15])
    return acc


def topka_baseline(grads, k: int, group=None):
    """grads: this rank's workers' float32 CUDA tensors of N elements (all
    ranks together hold the P workers in rank order).  Returns
    ((idx int32, val float32) of the merged union, (rounds, scalars) per
    worker of this rank)."""
    import torch
    import torch.distributed as dist
    if not grads:
        raise ConfigError("topka: gradient count != worker count")
    n = grads[0].numel()
    if k > n:
        raise ConfigError("topka: k must satisfy k <= N")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    local = [top_k_select_slice(g, 0, n, k) for g in grads]   # exactly k each
    p = world * len(grads)
    if world > 1:
        dev = grads[0].device
        si = torch.stack([i for i, _ in local])
        sv = torch.stack([v for _, v in local])
        gi = torch.empty((world,) + tuple(si.shape), dtype=si.dtype, device=dev)
        gv = torch.empty((world,) + tuple(sv.shape), dtype=sv.dtype, device=dev)
        dist.all_gather_into_tensor(gi, si, group=group)
        dist.all_gather_into_tensor(gv, sv, group=group)
        lists = [(gi[r, w], gv[r, w]) for r in range(world) for w in range(len(grads))]
    else:
        lists = local
    out = _fold(lists)
    rounds = math.ceil(math.log2(p)) if p > 1 else 0
    return out, [(rounds, 2 * k * (p - 1))] * len(grads)
