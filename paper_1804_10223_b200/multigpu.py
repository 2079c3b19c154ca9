"""Batch-partitioned multi-GPU execution.

The recurrence does not shard per step across GPUs: every step needs all of
h_{t-1} (unstructured columns) and one NVLink hop costs more than
a whole step on chip.  Independent sequences do shard: each rank owns a
contiguous slice of the batch, runs the full hot path (input GEMM + persistent
kernel) on its own GPU with the replicated weights, and the per-rank outputs
are all-gathered once at the end ("Our work can be extended to
multiple GPUs").  Per-sample arithmetic does not depend on the shard, so the
gathered result is bit-identical to the single-GPU run.

This module holds only the host-side partitioning and the collective; the
compute is the caller's ``local_forward`` (normally ``SparseRNN.forward``).
"""
from __future__ import annotations


def shard(global_batch: int, world: int, rank: int):
    """Contiguous batch slice [start, start + count) of `rank` (sizes differ by at most 1)."""
    if world < 1 or not 0 <= rank < world or global_batch < 0:
        raise ValueError("bad shard arguments")
    base, rem = divmod(global_batch, world)
    start = rank * base + min(rank, rem)
    return start, base + (1 if rank < rem else 0)


def gather_batch(y_local, group=None, global_batch=None):
    """All-gather per-rank outputs [T, B_r, H] into the global [T, B, H] (batch order = rank order).

    Uses torch.distributed (NCCL on GPUs, gloo on CPU).  Shards of unequal size
    are padded to the largest shard for the collective and trimmed after.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    T, b_r, H = y_local.shape
    sizes = torch.tensor([b_r], dtype=torch.int64, device=y_local.device)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = [int(s.item()) for s in all_sizes]
    bmax = max(all_sizes)
    # batch-major so each rank's block is contiguous for the collective
    send = torch.zeros((bmax, T, H), dtype=y_local.dtype, device=y_local.device)
    send[:b_r] = y_local.permute(1, 0, 2)
    recv = torch.empty((world * bmax, T, H), dtype=y_local.dtype, device=y_local.device)
    if hasattr(dist, "all_gather_into_tensor") and y_local.is_cuda:
        dist.all_gather_into_tensor(recv, send, group=group)
    else:
        dist.all_gather(list(recv.chunk(world)), send, group=group)
    parts = [recv[r * bmax:r * bmax + all_sizes[r]] for r in range(world)]
    y = torch.cat(parts, 0).permute(1, 0, 2).contiguous()
    if global_batch is not None and y.shape[1] != global_batch:
        raise RuntimeError(f"gathered batch {y.shape[1]} != expected {global_batch}")
    return y


def forward_partitioned(local_forward, x_global, group=None):
    """Run `local_forward(x_shard) -> y_shard` on this rank's slice of x [T, B, I], all-gather y."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    T, B, _ = x_global.shape
    start, count = shard(B, world, rank)
    y_local = local_forward(x_global[:, start:start + count].contiguous())
    return gather_batch(y_local, group=group, global_batch=B)
