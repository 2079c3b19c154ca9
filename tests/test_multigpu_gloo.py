"""N > 1 host path on CPU: world_size-2 gloo process group, batch sharding and
the all-gather of per-rank outputs (the gathered y must
be bit-identical to the single-process run, since per-sample arithmetic does
not depend on the shard)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1804_10223_b200 import inputs
from paper_1804_10223_b200.multigpu import chunks, forward_layer_pipelined, forward_partitioned, shard


def test_shard_covers_batch_exactly():
    for B in (1, 4, 7, 64):
        for world in (1, 2, 3, 4, 8):
            spans = [shard(B, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (s0, c0), (s1, _) in zip(spans, spans[1:]):
                assert s0 + c0 == s1
            assert sum(c for _, c in spans) == B
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, B, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle  # test infrastructure: the local compute of each rank here
    prob = inputs.make_problem(48, 12, B, 6, 0.2, act="tanh")

    def local_forward(x_shard):
        p = dict(prob)
        p["x"] = x_shard.numpy()
        p["B"] = x_shard.shape[1]
        return torch.from_numpy(oracle.forward(p)["y"])

    y = forward_partitioned(local_forward, torch.from_numpy(prob["x"]))
    if rank == 0:
        np.save(os.path.join(out_dir, "y.npy"), y.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [4, 5])
def test_gloo_world2_partitioned_equals_single(tmp_path, B):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, B, str(tmp_path)), nprocs=2, join=True)
    import oracle
    prob = inputs.make_problem(48, 12, B, 6, 0.2, act="tanh")
    ref = oracle.forward(prob)["y"]
    got = np.load(tmp_path / "y.npy")
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)


# ---- stacked layers pipelined across ranks ----

def _stack_problems(cell):
    # layer 0: I = 12 -> H = 40; layer 1: I = 40 -> H = 32 (2-layer stack)
    p0 = inputs.make_problem(40, 12, 3, 9, 0.2, cell=cell, act="tanh", seed_offset=1)
    p1 = inputs.make_problem(32, 40, 3, 9, 0.25, cell=cell, act="tanh", seed_offset=2)
    return p0, p1


def _oracle_layer_step(prob):
    import oracle

    def step(x_chunk, state):
        p = dict(prob)
        p["x"] = x_chunk.numpy().astype(np.float32)
        p["T"] = x_chunk.shape[0]
        p["h0"] = None if state is None else state[0]
        p["c0"] = None if state is None else state[1]
        o = oracle.forward(p)
        # outputs of a layer are the next layer's fp32 inputs
        return torch.from_numpy(o["y"].astype(np.float32)), (o["hT"], o.get("cT"))
    return step


def _pipe_worker(rank, world, port, cell, n_chunks, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    probs = _stack_problems(cell)
    y = forward_layer_pipelined(_oracle_layer_step(probs[rank]), torch.from_numpy(probs[0]["x"]), n_chunks,
                                [probs[0]["H"], probs[1]["H"]])
    np.save(os.path.join(out_dir, f"y{rank}.npy"), y.numpy())
    dist.destroy_process_group()


def test_chunks_cover_sequence():
    for T in (1, 7, 256):
        for n in (1, 3, 8, 300):
            cs = chunks(T, n)
            assert cs[0][0] == 0 and sum(c for _, c in cs) == T
            assert all(a + b == c for (a, b), (c, _) in zip(cs, cs[1:]))


@pytest.mark.parametrize("cell,n_chunks", [("rnn", 3), ("lstm", 4), ("rnn", 1)])
def test_gloo_world2_layer_pipeline_equals_unchunked(tmp_path, cell, n_chunks):
    """Rank r = layer r, time chunks handed over by send/recv: every rank's result equals the
    unchunked layer-by-layer run bit for bit (state carried through h0/c0)."""
    port = _free_port()
    mp.spawn(_pipe_worker, args=(2, port, cell, n_chunks, str(tmp_path)), nprocs=2, join=True)
    probs = _stack_problems(cell)
    x1 = _oracle_layer_step(probs[0])(torch.from_numpy(probs[0]["x"]), None)[0]
    ref = _oracle_layer_step(probs[1])(x1, None)[0].numpy()
    for r in range(2):
        got = np.load(tmp_path / f"y{r}.npy")
        assert got.shape == ref.shape
        assert np.array_equal(got, ref)


# ---- the C5 split (global batch 64 over ranks, batch-major y) ----

def _c5_problem():
    # C5's batch structure (B = 64, split evenly), small H / T so the CPU oracle stands in
    # for each rank's local compute
    return inputs.make_problem(40, 16, 64, 5, 0.1, act="relu")


def _c5_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    prob = _c5_problem()
    start, count = shard(64, world, rank)
    assert count == 64 // world

    def local_forward(x_shard):  # batch-major [B_r, T, H], like SRNN_FLAG_Y_BATCH_MAJOR
        p = dict(prob)
        p["x"] = x_shard.numpy()
        p["B"] = x_shard.shape[1]
        return torch.from_numpy(np.ascontiguousarray(oracle.forward(p)["y"].transpose(1, 0, 2)))

    y = forward_partitioned(local_forward, torch.from_numpy(prob["x"]), batch_major=True)
    np.save(os.path.join(out_dir, f"y{rank}.npy"), y.numpy())
    dist.destroy_process_group()


def test_gloo_world2_c5_split_batch_major(tmp_path):
    """B = 64 split 32 / 32 (the C5 shape at 2 GPUs): the batch-major all-gather of the
    ranks' blocks is the global [B, T, H] y of the single-process run, bit for bit."""
    port = _free_port()
    mp.spawn(_c5_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    import oracle
    ref = oracle.forward(_c5_problem())["y"].transpose(1, 0, 2)
    for r in range(2):
        got = np.load(tmp_path / f"y{r}.npy")
        assert got.shape == ref.shape == (64, 5, 40)
        assert np.array_equal(got, ref)
