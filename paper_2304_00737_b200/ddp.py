"""PyTorch DDP communication hook running SparDL -- the caller of the path.

The reference's caller is train() (/root/reference/proj/include/spardl/
trainer.hpp:180-302): every worker computes a dense gradient, the workers
synchronise with spardl_all_reduce (:268-283) and every replica applies
w -= lr/P * sum(global entries).  Here DDP plays the trainer: each rank is
one SparDL worker, each gradient bucket gets its own SparDL context (its own
residual carry, i.e. the error feedback of the bucket's parameters), and the
hook returns the densified global sparse gradient divided by the world size,
which is exactly DDP's averaged-gradient convention (w -= lr * grad).

    state = SparDLHookState(density=0.01)
    ddp_model.register_comm_hook(state, spardl_hook)
"""
import torch
import torch.distributed as dist

from .api import ClusterConfig, SparDL


class SparDLHookState:
    """Per-bucket SparDL contexts.  k = density * bucket size, rounded down to
    a multiple of the world size (ClusterConfig requires P | k)."""

    def __init__(self, density: float = 0.01, teams: int = 1, sag: str = "none",
                 residual: str = "gres", timing: str = "optimized", process_group=None):
        if not 0.0 < density <= 1.0:
            raise ValueError("density must be in (0, 1]")   # trainer.hpp:183-185
        self.density, self.teams, self.sag = density, teams, sag
        self.residual, self.timing = residual, timing
        self.pg = process_group
        self.contexts: dict = {}

    def context(self, bucket) -> "SparDL":
        buf = bucket.buffer()
        key = (bucket.index(), buf.numel())
        ctx = self.contexts.get(key)
        if ctx is None:
            world = dist.get_world_size(self.pg)
            n = buf.numel()
            k = max(world, int(self.density * n) // world * world)
            cfg = ClusterConfig(workers=world, dimension=n, k=min(k, n // world * world),
                                teams=self.teams, sag=self.sag, residual=self.residual,
                                timing=self.timing)
            ctx = SparDL.from_process_group(cfg, device=buf.device.index, group=self.pg)
            self.contexts[key] = ctx
        return ctx

    def close(self):
        for c in self.contexts.values():
            c.close()
        self.contexts.clear()


def spardl_hook(state: SparDLHookState, bucket) -> torch.futures.Future[torch.Tensor]:
    """DDP comm hook: SparDL sparse all-reduce of the bucket, densified and
    averaged over the ranks."""
    buf = bucket.buffer()
    grad = buf if buf.dtype == torch.float32 else buf.float()
    ctx = state.context(bucket)
    ctx.all_reduce([grad.contiguous()])
    idx, val = ctx.global_gradient(0)
    out = torch.zeros_like(grad)
    out.index_put_((idx.long(),), val)
    out.div_(dist.get_world_size(state.pg))
    if out.dtype != buf.dtype:
        out = out.to(buf.dtype)
    fut = torch.futures.Future(devices=[buf.device])
    fut.set_result(out)
    return fut
