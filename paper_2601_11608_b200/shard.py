"""Batch sharding for the multi-GPU launcher.

Images are independent, so the conv path shards by contiguous batch slices
with no collective on the hot path. torch.distributed (NCCL on GPUs, gloo in
CPU tests) is used only outside the timed region: to take the max of the
per-rank device times and to gather verification scalars.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """[start, stop) of rank's contiguous slice; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def dist_env() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def init(backend: str) -> None:
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        dist.init_process_group(backend)


def max_over_ranks(value: float, device: torch.device | str = "cpu") -> float:
    """Max of a per-rank scalar (e.g. device ms) across the job; identity when not distributed."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_scalars(values: list[float], device: torch.device | str = "cpu") -> list[list[float]]:
    """All ranks' scalar lists (verification only, never in the timed region)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [list(values)]
    t = torch.tensor(values, dtype=torch.float64, device=device)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.cpu().tolist() for o in out]


def gather_to(tensor: torch.Tensor, sizes: list[int], dst: int = 0) -> torch.Tensor | None:
    """Concatenate every rank's leading-dimension shard on rank ``dst`` (the
    shards may differ in length by one; ``sizes`` are all ranks' lengths).
    Verification / collection only -- never on the hot path. Each rank sends
    its shard straight into its slice of ``dst``'s output (grouped
    point-to-point ops: NCCL send/recv on CUDA tensors, gloo on CPU ones), so
    ``dst`` holds the output once and no other rank receives anything; an
    all-gather would land all 8 x 13.15 GB of the R50 b8192 output on every
    rank. Identity when not distributed."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return tensor
    rank, world = dist.get_rank(), dist.get_world_size()
    # validate collectively BEFORE any rank posts a receive: a mismatch on one
    # rank raises on every rank instead of leaving dst blocked in irecv. The
    # all-reduce also brings the communicator up on every rank, so a rank
    # with an empty shard may then skip the point-to-point phase (NCCL needs
    # every rank in the FIRST collective call only).
    bad = float(len(sizes) != world or tensor.shape[0] != (sizes[rank] if rank < len(sizes) else -1))
    flag = torch.tensor([bad], dtype=torch.float64, device=tensor.device)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX)
    if flag.item() > 0:
        raise ValueError(f"shard sizes {sizes} do not match the ranks' shards (rank {rank}: {tuple(tensor.shape)})")
    if rank != dst:
        ops = [dist.P2POp(dist.isend, tensor.contiguous(), dst)] if sizes[rank] > 0 else []
        for req in (dist.batch_isend_irecv(ops) if ops else []):
            req.wait()
        return None
    out = torch.empty((sum(sizes),) + tuple(tensor.shape[1:]), dtype=tensor.dtype, device=tensor.device)
    offs = [sum(sizes[:r]) for r in range(world)]
    out[offs[dst]:offs[dst] + sizes[dst]] = tensor
    ops = [dist.P2POp(dist.irecv, out[offs[r]:offs[r] + sizes[r]], r)
           for r in range(world) if r != dst and sizes[r] > 0]
    for req in (dist.batch_isend_irecv(ops) if ops else []):
        req.wait()
    return out


class ShardedConv:
    """The batch-sharded launcher: rank r of a torchrun job convolves images
    ``shard_range(N, r, world)`` of a global batch on its own GPU with the
    folded kernel; there is no collective between the ranks' launches.
    ``gather(y)`` collects the full output on one rank for verification.

        conv = ShardedConv(w, b, (8192, 224, 224, 3), stride=2, padding=3)
        y_local = conv(x[conv.lo:conv.hi].cuda())     # hot path, rank-local
        y_all = conv.gather(y_local)                  # rank 0: (8192, 112, 112, 64)
    """

    def __init__(self, w, b, global_shape, stride=1, padding=0, dtype=None, **kw):
        from .api import FoldedConv2d
        self.rank, local, self.world = dist_env()
        if dist.is_available() and dist.is_initialized():
            self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.device = torch.device("cuda", local) if torch.cuda.is_available() else torch.device("cpu")
        n = int(global_shape[0])
        self.lo, self.hi = shard_range(n, self.rank, self.world)
        self.sizes = [b_ - a_ for a_, b_ in (shard_range(n, r, self.world) for r in range(self.world))]
        shape = (self.hi - self.lo,) + tuple(int(v) for v in global_shape[1:])
        w = w.to(self.device) if isinstance(w, torch.Tensor) else torch.as_tensor(w, device=self.device)
        if b is not None:
            b = b.to(self.device) if isinstance(b, torch.Tensor) else torch.as_tensor(b, device=self.device)
        self.conv = FoldedConv2d(w, b, shape, stride=stride, padding=padding, dtype=dtype, **kw)

    def __call__(self, x_local: torch.Tensor, **kw) -> torch.Tensor:
        return self.conv(x_local, **kw)

    def gather(self, y_local: torch.Tensor, dst: int = 0) -> torch.Tensor | None:
        return gather_to(y_local, self.sizes, dst)
