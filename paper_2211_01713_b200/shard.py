"""Scenario sharding across ranks (BASELINE config 4).

Independent provisioning scenarios are the unit of parallelism: rank r of
world W plans a contiguous block of scenarios on its own GPU, with no
collective on the data path.  The only exchange is at the end: every rank's
fixed-size plan records (per workload its GPU index and units, plus the
scenario's GPU count) are all-gathered, over NCCL/NVLink on GPUs or gloo on
CPU.  Blocks may differ by one scenario; the gather pads to the largest block.
"""

from __future__ import annotations

import numpy as np


def shard_bounds(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [start, end) of rank; the first n_total % world ranks
    take one extra scenario."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def record_width(m: int) -> int:
    return 2 * m + 1


def pack_records(gpu_of, units, gpu_count):
    """[S, m] GPU indices, [S, m] units, [S] GPU counts -> [S, 2m+1] int32
    records (numpy in, numpy out; torch tensors in, torch tensors out)."""
    try:
        import torch
        if isinstance(gpu_of, torch.Tensor):
            return torch.cat([gpu_of.to(torch.int32), units.to(torch.int32),
                              gpu_count.to(torch.int32).reshape(-1, 1)], dim=1).contiguous()
    except ImportError:  # pragma: no cover - torch is part of the image
        pass
    return np.concatenate([np.asarray(gpu_of, np.int32), np.asarray(units, np.int32),
                           np.asarray(gpu_count, np.int32).reshape(-1, 1)], axis=1)


def unpack_records(rec, m: int):
    return rec[:, :m], rec[:, m:2 * m], rec[:, 2 * m]


def gather_records(local, n_total: int, world: int, group=None):
    """All-gather every rank's [S_r, R] records into [n_total, R] in scenario
    order (torch tensors; the backend is the process group's)."""
    import torch
    import torch.distributed as dist
    s_max = -(-n_total // world)
    R = local.shape[1]
    buf = torch.zeros((s_max, R), dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    out = torch.empty((world * s_max, R), dtype=local.dtype, device=local.device)
    if dist.get_backend(group) == "gloo":  # gloo has no all_gather_into_tensor
        dist.all_gather(list(out.chunk(world)), buf, group=group)
    else:
        dist.all_gather_into_tensor(out, buf, group=group)
    rows = []
    for r in range(world):
        a, b = shard_bounds(n_total, r, world)
        rows.append(out[r * s_max: r * s_max + (b - a)])
    return torch.cat(rows, dim=0)


def plan_shard(wl, hw_vec, b_max, rank, *, flags=0, device=None, group=None):
    """Plan this rank's contiguous block of the batch ``wl`` [S, 16, m] on its
    GPU with the CUDA planner (igp_plan_batch_device), then all-gather every
    rank's fixed-size plan records (NCCL on GPUs; gloo also takes the CUDA
    tensors).  Returns the [S, 2m+1] int32 records of the whole batch, in
    scenario order, as a tensor on ``device`` -- ``unpack_records`` splits
    them.  ``rank`` is the name rank of the scenarios' workloads ([m] or
    [S, m]).  No collective runs before the gather: scenarios are independent
    (SURVEY.md §8e)."""
    import torch
    import torch.distributed as dist
    from . import _device
    world = dist.get_world_size(group)
    r = dist.get_rank(group)
    S, _, m = wl.shape
    a, b = shard_bounds(S, r, world)
    device = _device._dev(device)
    if b > a:
        rk = rank[a:b] if np.ndim(rank) == 2 else rank
        res = _device.plan_device(wl[a:b], hw_vec, b_max, rk, flags=flags, device=device,
                                  want_pred=False)
        local = torch.from_numpy(pack_records(res["gpu_of"], res["units"],
                                              res["gpu_count"])).to(device)
    else:
        local = torch.zeros((0, record_width(m)), dtype=torch.int32, device=device)
    return gather_records(local, S, world, group=group)
