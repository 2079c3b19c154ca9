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


def gather_batch_major(y_local, group=None, global_batch=None, out=None):
    """All-gather batch-major per-rank outputs [B_r, T, H] into the global [B, T, H].

    With SRNN_FLAG_Y_BATCH_MAJOR every rank's y is one contiguous block of the global
    batch-major y, so equal shards go straight into the collective's output buffer
    (no permute, no staging copy -- ``out`` may be preallocated); unequal shards are
    padded to the largest for the collective and compacted after.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    b_r, T, H = y_local.shape
    if global_batch is not None and global_batch % world == 0 and b_r * world == global_batch:
        if out is None:
            out = torch.empty((global_batch, T, H), dtype=y_local.dtype, device=y_local.device)
        if hasattr(dist, "all_gather_into_tensor") and y_local.is_cuda:
            dist.all_gather_into_tensor(out, y_local.contiguous(), group=group)
        else:
            dist.all_gather(list(out.chunk(world)), y_local.contiguous(), group=group)
        return out
    sizes = torch.tensor([b_r], dtype=torch.int64, device=y_local.device)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    all_sizes = [int(v.item()) for v in all_sizes]
    bmax = max(all_sizes)
    send = torch.zeros((bmax, T, H), dtype=y_local.dtype, device=y_local.device)
    send[:b_r] = y_local
    recv = torch.empty((world * bmax, T, H), dtype=y_local.dtype, device=y_local.device)
    dist.all_gather(list(recv.chunk(world)), send, group=group)
    y = torch.cat([recv[r * bmax:r * bmax + all_sizes[r]] for r in range(world)], 0)
    if global_batch is not None and y.shape[0] != global_batch:
        raise RuntimeError(f"gathered batch {y.shape[0]} != expected {global_batch}")
    return y


def forward_partitioned(local_forward, x_global, group=None, batch_major=False):
    """Run `local_forward(x_shard) -> y_shard` on this rank's slice of x [T, B, I], all-gather y
    ([T, B, H]; batch_major: local outputs and the result are [B_r, T, H] / [B, T, H])."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    T, B, _ = x_global.shape
    start, count = shard(B, world, rank)
    y_local = local_forward(x_global[:, start:start + count].contiguous())
    if batch_major:  # local_forward returns [B_r, T, H] (SRNN_FLAG_Y_BATCH_MAJOR)
        return gather_batch_major(y_local, group=group, global_batch=B)
    return gather_batch(y_local, group=group, global_batch=B)


# ---------------------------------------------------------------------------
# Stacked layers pipelined across ranks (the NMT case
# study is a 2-layer LSTM).  Rank r owns layer r.  The sequence
# is cut into time chunks; rank r runs chunk c of its layer while rank r - 1
# runs chunk c + 1 (a wavefront over (layer, chunk)), and each finished chunk
# of y is handed to the next rank with one point-to-point send (NCCL p2p over
# NVLink on GPUs, gloo on CPU).  The recurrent state (h, and c for LSTM) is
# carried from chunk to chunk through the layer's h0/c0 -> hT/cT arguments,
# so the result equals the unchunked layer-by-layer run: chunking changes
# neither the per-step arithmetic nor its order.
# ---------------------------------------------------------------------------

def chunks(T: int, n_chunks: int):
    """Contiguous time spans [(t0, length)] covering [0, T) (sizes differ by at most 1)."""
    n = max(1, min(n_chunks, T)) if T > 0 else 1
    return [shard(T, n, c) for c in range(n)]


def layer_step(plan):
    """Chunk function of one SparseRNN plan: (x_chunk, state) -> (y_chunk, state), state = (hT, cT)."""
    def step(x_chunk, state):
        h0, c0 = state if state is not None else (None, None)
        out = plan.forward(x_chunk, h0, c0)
        return out[0], (out[1], out[2] if len(out) > 2 else None)
    return step


def forward_stacked_chunked(layer_steps, x, n_chunks):
    """Single-process wavefront order of the pipelined stack (one GPU, or a reference for tests):
    for each time chunk, run it through every layer in turn, carrying each layer's state."""
    import torch

    states = [None] * len(layer_steps)
    outs = []
    for t0, tn in chunks(int(x.shape[0]), n_chunks):
        inp = x[t0:t0 + tn].contiguous()
        for li, f in enumerate(layer_steps):
            inp, states[li] = f(inp, states[li])
        outs.append(inp)
    return torch.cat(outs, 0)


def forward_layer_pipelined(local_layer_step, x_global, n_chunks, layer_widths, group=None):
    """Rank r runs layer r of a stacked model over time chunks, pipelined across ranks.

    local_layer_step(x_chunk [Tc, B, I_r], state) -> (y_chunk [Tc, B, H_r], state)
    x_global: [T, B, I_0] (only rank 0 reads its values; every rank uses its shape/device)
    layer_widths: H_r of every layer (rank r receives chunks of width H_{r-1}).
    Returns the last layer's y [T, B, H_last] on every rank.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if len(layer_widths) != world:
        raise ValueError("one layer per rank: len(layer_widths) must equal the world size")
    T, B, _ = x_global.shape
    dev, dt = x_global.device, x_global.dtype

    def peer(r):  # global rank of group rank r
        return r if group is None else dist.get_global_rank(group, r)

    state = None
    outs = []
    for t0, tn in chunks(int(T), n_chunks):
        if rank == 0:
            inp = x_global[t0:t0 + tn].contiguous()
        else:
            inp = torch.empty((tn, B, layer_widths[rank - 1]), dtype=dt, device=dev)
            dist.recv(inp, src=peer(rank - 1), group=group)
        y, state = local_layer_step(inp, state)
        if rank + 1 < world:
            dist.send(y.contiguous(), dst=peer(rank + 1), group=group)
        else:
            outs.append(y)
    if rank == world - 1:
        y_all = torch.cat(outs, 0).contiguous()
    else:
        y_all = torch.empty((T, B, layer_widths[-1]), dtype=dt, device=dev)
    dist.broadcast(y_all, src=peer(world - 1), group=group)
    return y_all
