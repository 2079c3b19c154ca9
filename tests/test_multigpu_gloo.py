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
from paper_1804_10223_b200.multigpu import forward_partitioned, shard


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
