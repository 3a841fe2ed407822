"""Multi-GPU sharding of independent S-MNN instances (one process per GPU).

Instances (batch x ODE-dim pairs) are independent, so B*D is split into
contiguous shards, one per rank, and every rank runs the fused kernels on its
shard with no data-path collective.  Collectives (NCCL on GPUs, gloo in the
CPU tests) are used only to gather results and reduce losses, as BASELINE.json
north_star prescribes.  Uneven shards are padded for all_gather and trimmed.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous [start, stop) of n instances for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def shard(t: torch.Tensor, rank: int, world: int, dim: int = 0) -> torch.Tensor:
    """This rank's contiguous slice of the instance dimension."""
    s, e = shard_range(t.shape[dim], rank, world)
    return t.narrow(dim, s, e - s)


def _host_collectives(group=None) -> bool:
    """gloo (CPU tests, or several ranks sharing one GPU) cannot take CUDA tensors."""
    return dist.get_backend(group) == "gloo"


def gather_instances(local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """all_gather the per-rank shards (dim 0) back into the full [n_total, ...] tensor
    (on the input's device; through host memory under gloo)."""
    if local.is_cuda and _host_collectives(group):
        return gather_instances(local.cpu(), n_total, group).to(local.device)
    world = dist.get_world_size(group)
    cap = -(-n_total // world)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    parts = []
    for r in range(world):
        s, e = shard_range(n_total, r, world)
        parts.append(bufs[r][: e - s])
    return torch.cat(parts, 0)


def allreduce_loss(loss: torch.Tensor, group=None) -> torch.Tensor:
    """Sum a scalar loss over ranks (the only reduction the solve needs)."""
    if loss.is_cuda and _host_collectives(group):
        return allreduce_loss(loss.cpu(), group).to(loss.device)
    out = loss.detach().clone()
    dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


def max_over_ranks(x: float, device, group=None) -> float:
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sharded_step(smnn, full: dict, grad_y: torch.Tensor, rank: int, world: int, w=None, compute=None,
                 gather: bool = True, group=None):
    """One strong-scaling step of the sharded data path: this rank solves its
    contiguous shard of the B*D instances (fused forward + backward, no
    collective inside the solve), the loss l = <dl/dy, y> is summed over ranks
    and y is all_gathered (the only collectives, north_star).  Returns
    (y of all instances or None, loss, this shard's (dc, dd, du, ds, info))."""
    n_total = full["coeffs"].shape[0]
    loc = {k: shard(v, rank, world) for k, v in full.items()}
    gy = shard(grad_y, rank, world)
    w = w or smnn.Weights()
    y_lo = None
    if compute == "f64" and loc["coeffs"].dtype == torch.float32 and smnn.ylo_used(loc["coeffs"], loc["iv"], w, compute):
        y, info, y_lo = smnn.smnn_factor_solve_fwd(loc["coeffs"], loc["rhs"], loc["iv"], loc["steps"], w, compute,
                                                   with_ylo=True)
    else:
        y, info = smnn.smnn_factor_solve_fwd(loc["coeffs"], loc["rhs"], loc["iv"], loc["steps"], w, compute)
    loss = allreduce_loss((gy.double() * y.double()).sum(), group=group)
    y_all = gather_instances(y, n_total, group=group) if gather else None
    g = smnn.smnn_solve_bwd(loc["coeffs"], loc["rhs"], loc["iv"], loc["steps"], y, gy, w, compute, y_lo=y_lo)
    return y_all, loss, g
