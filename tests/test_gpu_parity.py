"""GPU parity: the CUDA path (through the C ABI) against the CPU fp64 oracle.

Tolerances (BASELINE.json north_star): max-abs over ALL T x B x H outputs
1e-5 in fp32 mode, 2e-2 in fp16-weight / fp32-accumulate mode (against the
UNQUANTISED weights).  Integer-exact inputs must match bit for bit.
"""
import numpy as np
import pytest

import oracle
from paper_1804_10223_b200 import (FLAG_DEBUG_JITTER, FLAG_DENSE_TC, FLAG_FP32_STAGING, FLAG_GRID_SYNC, FLAG_NAIVE_LAYOUT,
                                   FLAG_RESERVE_SMS, from_problem, inputs)

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-5, "fp16": 2e-2}


def run_gpu(prob, prec, flags=0, device="cuda:0", **kw):
    import torch
    m = from_problem(prob, prec=prec, flags=flags, **kw)
    x = torch.from_numpy(prob["x"]).to(device)
    h0 = None if prob["h0"] is None else torch.from_numpy(prob["h0"]).to(device)
    c0 = None if prob.get("c0") is None else torch.from_numpy(prob["c0"]).to(device)
    out = m.forward(x, h0, c0)
    torch.cuda.synchronize()
    m.status()
    res = {"y": out[0].cpu().numpy(), "hT": out[1].cpu().numpy()}
    if prob["cell"] == "lstm":
        res["cT"] = out[2].cpu().numpy()
    res["info"] = m.info()
    m.close()
    return res


def check(prob, prec, flags=0, **kw):
    g = run_gpu(prob, prec, flags, **kw)
    o = oracle.forward(prob)
    err = np.abs(g["y"].astype(np.float64) - o["y"]).max() if g["y"].size else 0.0
    errh = np.abs(g["hT"].astype(np.float64) - o["hT"]).max()
    assert np.isfinite(g["y"]).all()
    assert err <= TOL[prec], (err, g["info"])
    assert errh <= TOL[prec]
    if prob["cell"] == "lstm":
        # c is an unbounded running sum (c = f c + i g): its error scales with |c|, while
        # h = o tanh(c) damps it (|tanh'| <= 1 and -> 0 where |c| is large), so the cell
        # state is held to the north-star tolerance relative to max(1, |c|)
        errc = np.abs(g["cT"].astype(np.float64) - o["cT"]) / np.maximum(1.0, np.abs(o["cT"]))
        assert errc.max() <= TOL[prec], errc.max()
    return g, o, err


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
@pytest.mark.parametrize("H,B,T,d,act", [
    (256, 1, 16, 0.10, "relu"),      # C1
    (300, 3, 20, 0.05, "tanh"),      # ragged H, B not a multiple of the tile
    (1000, 4, 12, 0.30, "relu"),
    (1152, 4, 24, 0.10, "relu"),     # Table 1 shape, short T
    (513, 6, 9, 0.02, "identity"),   # two batch tiles, ragged
    (64, 2, 30, 0.50, "tanh"),
    (700, 8, 10, 0.05, "tanh"),      # fp16: one batch tile of 8 (LDS.128)
    (333, 16, 7, 0.10, "relu"),      # two tiles of 8
    (129, 13, 6, 0.20, "tanh"),      # ragged last tile
])
def test_rnn_parity_small(cuda_device, prec, H, B, T, d, act):
    prob = inputs.make_problem(H, H, B, T, d, act=act, h0="random", seed_offset=H)
    check(prob, prec)


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
@pytest.mark.parametrize("H,B,T,d,pattern", [
    (128, 4, 10, 0.125, "row_balanced"),
    (257, 1, 12, 0.12, "unstructured"),
    (96, 5, 7, 0.3, "unstructured"),
    (200, 8, 6, 0.1, "row_balanced"),
])
def test_lstm_parity_small(cuda_device, prec, H, B, T, d, pattern):
    prob = inputs.make_problem(H, H, B, T, d, cell="lstm", pattern=pattern, h0="random", c0="random",
                               seed_offset=H)
    check(prob, prec)


@pytest.mark.parametrize("cell", ["rnn", "lstm"])
@pytest.mark.parametrize("prec", ["fp32", "fp16"])
def test_integer_exact_bitwise(cuda_device, cell, prec):
    """Integer inputs: every partial sum < 2^24, so any order is exact."""
    act = "identity" if cell == "rnn" else "relu"
    if prec == "fp32":
        prob = inputs.make_integer_problem(200, 48, 4, 5, 0.02, cell=cell, act=act)
    else:  # the fp16 exchange keeps 10 significant bits (R16): integers up to 2^10 are exact
        prob = inputs.make_integer_problem(200, 6, 4, 3, 0.01, cell=cell, act=act)
    if cell == "lstm":
        # gates saturate; keep the exactness claim to the RNN path, check LSTM by tolerance
        check(prob, prec)
        return
    o = oracle.forward(prob)
    # exchanged h keeps 23 (fp32) / 10 (fp16) significant bits (R16)
    assert np.abs(o["y"]).max() < (2 ** 23 if prec == "fp32" else 2 ** 10)
    g = run_gpu(prob, prec)
    assert np.array_equal(g["y"].astype(np.float64), o["y"])


def test_grid_sync_equals_tags_bitwise(cuda_device):
    prob = inputs.make_problem(1152, 1152, 4, 32, 0.1, act="tanh", h0="random")
    a = run_gpu(prob, "fp16")
    b = run_gpu(prob, "fp16", flags=FLAG_GRID_SYNC)
    assert np.array_equal(a["y"], b["y"])


def test_jitter_is_bitwise_deterministic(cuda_device):
    """Random per-CTA delays must not change a single bit (SPEC.md:406/:550 analogue)."""
    prob = inputs.make_problem(777, 777, 3, 40, 0.1, act="tanh", h0="random")
    a = run_gpu(prob, "fp32")
    b = run_gpu(prob, "fp32", flags=FLAG_DEBUG_JITTER)
    c = run_gpu(prob, "fp32")
    assert np.array_equal(a["y"], b["y"]) and np.array_equal(a["y"], c["y"])


@pytest.mark.parametrize("B", [1, 2, 4])
def test_fp16_mode_fp32_staging_ablation(cuda_device, B):
    prob = inputs.make_problem(900, 900, B, 20, 0.1, act="tanh", h0="random")
    check(prob, "fp16", flags=FLAG_FP32_STAGING)


def test_naive_layout_parity(cuda_device):
    prob = inputs.make_problem(1152, 1152, 4, 16, 0.1, act="relu")
    check(prob, "fp32", flags=FLAG_NAIVE_LAYOUT)


@pytest.mark.parametrize("prec,B", [("fp32", 4), ("fp16", 4), ("fp16", 8), ("fp32", 1), ("fp16", 2)])
@pytest.mark.parametrize("L", [1, 2, 4, 8, 16, 32])
def test_every_lane_mapping(cuda_device, L, prec, B):
    """Every lanes-per-row mapping x batch tile: the halving butterfly (L >= BT)
    and the plain butterfly (L < BT) both reduce to the oracle."""
    prob = inputs.make_problem(512, 512, B, 8, 0.05, act="tanh", h0="random")
    check(prob, prec, lanes_per_row=L)


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
@pytest.mark.parametrize("C,H", [(1, 300), (3, 700), (148, 700)])
def test_cta_counts(cuda_device, C, H, prec):
    prob = inputs.make_problem(H, H, 2, 8, 0.05, act="tanh", h0="random")
    check(prob, prec, num_ctas=C)


@pytest.mark.parametrize("cell", ["rnn", "lstm"])
def test_forced_cta_count_above_hidden(cuda_device, cell):
    """More CTAs forced than units (H = 101, odd word count at B = 1): clamped to H, no CTA
    without units (whose publish would never write the exchange pad word)."""
    prob = inputs.make_problem(101, 64, 1, 6, 0.1, cell=cell, act="tanh", h0="random")
    g, _, _ = check(prob, "fp16", num_ctas=148)
    assert g["info"]["num_ctas"] == 101


def test_T0_T1_repeat_and_smaller_batch(cuda_device):
    import torch
    prob = inputs.make_problem(320, 320, 4, 6, 0.1, act="tanh", h0="random")
    m = from_problem(prob, prec="fp32", batch=4, max_steps=6)
    o = oracle.forward(prob)
    x = torch.from_numpy(prob["x"]).cuda()
    h0 = torch.from_numpy(prob["h0"]).cuda()
    # T = 0 returns h0
    y, hT = m.forward(x[:0], h0)
    torch.cuda.synchronize()
    assert np.array_equal(hT.cpu().numpy(), prob["h0"])
    # repeated calls (epoch tags advance) give identical results
    for _ in range(3):
        y, hT = m.forward(x, h0)
        torch.cuda.synchronize()
        m.status()
        assert np.abs(y.cpu().numpy() - o["y"]).max() <= 1e-5
    # B < B_max: samples are independent (batch independence pin)
    y2, _ = m.forward(x[:, 1:3].contiguous(), h0[1:3].contiguous())
    torch.cuda.synchronize()
    assert np.abs(y2.cpu().numpy() - o["y"][:, 1:3]).max() <= 1e-5
    # T = 1 equals the first step
    y1, _ = m.forward(x[:1].contiguous(), h0)
    torch.cuda.synchronize()
    assert np.abs(y1.cpu().numpy() - o["y"][:1]).max() <= 1e-5


def test_input_projection_alone(cuda_device):
    import torch
    prob = inputs.make_problem(384, 200, 3, 7, 0.1)
    m = from_problem(prob, prec="fp32")
    bp = m.input_projection(torch.from_numpy(prob["x"]).cuda())
    torch.cuda.synchronize()
    ref = oracle.input_projection(prob["x"], prob["wx"], prob["bias"])
    assert np.abs(bp.cpu().numpy() - ref).max() <= 1e-5


@pytest.mark.parametrize("H,I,B,T,cell", [(384, 200, 3, 7, "rnn"), (200, 100, 3, 5, "rnn"), (2304, 2304, 4, 256, "rnn"),
                                        (130, 64, 2, 9, "lstm"), (1024, 1024, 4, 100, "lstm")])
@pytest.mark.parametrize("bn", ["auto", "128", "192", "256"])
def test_input_projection_tensor_cores(cuda_device, monkeypatch, H, I, B, T, cell, bn):
    """fp16 mode: tcgen05 GEMM on fp16-rounded x and W_x, fp32 accumulate.
    Against the oracle fed the same fp16-rounded operands (fp32 vs fp64
    accumulation only) and against the unquantised oracle (fp16 rounding).
    bn: output tile width 128 / 192 / 256 forced (ragged N: TMA zero-fills rows past N)."""
    import torch
    if bn != "auto":
        monkeypatch.setenv("SRNN_GEMM_BN", bn)
    prob = inputs.make_problem(H, I, B, T, 0.05, cell=cell)
    m = from_problem(prob, prec="fp16")
    bp = m.input_projection(torch.from_numpy(prob["x"]).cuda())
    torch.cuda.synchronize()
    got = bp.cpu().numpy().astype(np.float64)
    q = lambda a: np.asarray(a, np.float32).astype(np.float16).astype(np.float64)
    ref_q = oracle.input_projection(q(prob["x"]), q(prob["wx"]), prob["bias"])
    ref = oracle.input_projection(prob["x"], prob["wx"], prob["bias"])
    assert np.abs(got - ref_q).max() <= 1e-4 * max(1.0, np.sqrt(I / 256))
    assert np.abs(got - ref).max() <= 1e-2


@pytest.mark.parametrize("H,I,B,T", [(2304, 2304, 4, 256), (1000, 520, 3, 50), (384, 200, 3, 7), (130, 64, 2, 9)])
@pytest.mark.parametrize("cm", ["2", "4", "144x4"])
def test_input_projection_multicast_clusters(cuda_device, monkeypatch, H, I, B, T, cm):
    """fp16 mode, W_x multicast over thread-block clusters of 2 / 4 CTAs along M (TMA
    .multicast::cluster, cluster-wide empty barriers), 128-wide tiles or the 144-wide tiles the
    whole-GPU projection uses (three 48-row B slices, a 16-column last epilogue chunk): the
    same values as the oracle on the fp16-rounded operands, incl. ragged M (row tiles past M
    in a cluster) and ragged N."""
    import torch
    if cm == "144x4":
        monkeypatch.setenv("SRNN_GEMM_BN", "144")
    else:
        monkeypatch.setenv("SRNN_GEMM_BN", "128")
        monkeypatch.setenv("SRNN_GEMM_CM", cm)
    prob = inputs.make_problem(H, I, B, T, 0.05)
    m = from_problem(prob, prec="fp16")
    bp = m.input_projection(torch.from_numpy(prob["x"]).cuda())
    torch.cuda.synchronize()
    got = bp.cpu().numpy().astype(np.float64)
    q = lambda a: np.asarray(a, np.float32).astype(np.float16).astype(np.float64)
    ref_q = oracle.input_projection(q(prob["x"]), q(prob["wx"]), prob["bias"])
    assert np.abs(got - ref_q).max() <= 1e-4 * max(1.0, np.sqrt(I / 256))
    monkeypatch.setenv("SRNN_GEMM_CM", "1")
    monkeypatch.setenv("SRNN_GEMM_BN", "128")
    bp1 = m.input_projection(torch.from_numpy(prob["x"]).cuda())
    torch.cuda.synchronize()
    assert torch.equal(bp1, bp)  # same tiles, same MMA order: bit-identical to the unclustered kernel


def test_forward_host_matches_device(cuda_device):
    prob = inputs.make_problem(640, 640, 4, 10, 0.1, act="relu", h0="random")
    m = from_problem(prob, prec="fp16")
    y, hT = m.forward_host(prob["x"], prob["h0"])
    g = run_gpu(prob, "fp16")
    assert np.array_equal(y, g["y"]) and np.array_equal(hT, g["hT"])


# ---- full-size configurations of BASELINE.json (the bench's launch config) ----

def test_headline_C2_fp16_full(cuda_device):
    """C2: H=2304, B=4, d=30%, T=256, fp16 weights -- every output vs oracle."""
    prob = inputs.make_problem(**{k: v for k, v in inputs.CONFIGS["C2"].items() if k != "prec"})
    g, o, err = check(prob, "fp16")
    print("C2 fp16 max-abs err", err, "max|h|", np.abs(o["y"]).max(), g["info"])


def test_headline_C2_fp32_full(cuda_device):
    prob = inputs.make_problem(**{k: v for k, v in inputs.CONFIGS["C2"].items() if k != "prec"})
    g, o, err = check(prob, "fp32")
    print("C2 fp32 max-abs err", err)


def test_C4_lstm_nmt_full(cuda_device):
    cfg = {k: v for k, v in inputs.CONFIGS["C4_nmt"].items() if k != "prec"}
    prob = inputs.make_problem(**cfg)
    check(prob, "fp16")


def test_C4_lstm_speech_full(cuda_device):
    cfg = {k: v for k, v in inputs.CONFIGS["C4_speech"].items() if k != "prec"}
    prob = inputs.make_problem(**cfg)
    check(prob, "fp32")


@pytest.mark.parametrize("world", [2, 4])
def test_batch_partition_bit_identical(cuda_device, world):
    """shards run separately (here sequentially on one GPU,
    same plan layout) and concatenated equal the single run bit for bit."""
    import torch
    from paper_1804_10223_b200.multigpu import shard
    prob = inputs.make_problem(1152, 1152, 8, 32, 0.1, act="tanh", h0="random")
    m = from_problem(prob, prec="fp16", batch_tile=4)
    x = torch.from_numpy(prob["x"]).cuda()
    h0 = torch.from_numpy(prob["h0"]).cuda()
    y_full, _ = m.forward(x, h0)
    parts = []
    for r in range(world):
        s0, c = shard(8, world, r)
        y, _ = m.forward(x[:, s0:s0 + c].contiguous(), h0[s0:s0 + c].contiguous())
        parts.append(y)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts, 1), y_full)


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
@pytest.mark.parametrize("cell,B", [("rnn", 1), ("rnn", 4), ("rnn", 6), ("lstm", 2), ("rnn", 16), ("lstm", 17)])
def test_smem_weight_tier_forced(cuda_device, monkeypatch, prec, cell, B):
    """Shared-memory weight tier (a10), forced on a small layer: pairs beyond 4
    register slots per lane live in shared memory."""
    monkeypatch.setenv("SRNN_FORCE_SMEM_TIER", "1")
    prob = inputs.make_problem(300, 64, B, 9, 0.15, cell=cell, act="tanh", h0="random")
    g, o, err = check(prob, prec, lanes_per_row=1)
    assert g["info"]["smem_weight_bytes_per_cta"] > 0 and g["info"]["pairs_per_lane"] == 4


@pytest.mark.parametrize("H,d", [(13445, 0.02), (19200, 0.01), (27648, 0.005)])
def test_capacity_large_hidden_on_chip(cuda_device, H, d):
    """a10 / SURVEY d-iv: 5x the largest dense layer that fits still runs fully on chip --
    every output checked.  Dense references (B = 4, device-checked, profiles/capacity_curve_r01.md):
    this library's format at density 1 (H = 3252; 5x = 16260) and the dense tensor-core
    persistent comparator SRNN_FLAG_DENSE_TC (H = 3829; 5x = 19145): 19200 and 27648 exceed
    both; 13445 @ 2% is an intermediate point."""
    prob = inputs.make_problem(H, 64, 1, 6, d, act="tanh", h0="random")
    g, o, err = check(prob, "fp16")
    print(H, d, g["info"])


@pytest.mark.parametrize("cell,H,B,T,d,act", [
    ("rnn", 333, 16, 7, 0.10, "relu"),      # one tile of 16 (two hs planes of 8)
    ("rnn", 200, 20, 6, 0.10, "tanh"),      # ragged second tile (4 of 16)
    ("rnn", 150, 32, 5, 0.20, "identity"),  # two full tiles
    ("rnn", 1500, 16, 4, 0.05, "tanh"),
    ("lstm", 200, 16, 6, 0.10, "tanh"),
    ("lstm", 96, 19, 5, 0.30, "tanh"),
])
def test_batch_tile_16(cuda_device, cell, H, B, T, d, act):
    """fp16 tiles of 16 samples (two hs planes of 8): every output against the
    oracle, and against the same layer forced to tiles of 8 (same weights; the
    lane-reduction order differs, so within tolerance rather than bitwise)."""
    prob = inputs.make_problem(H, H, B, T, d, cell=cell, act=act, h0="random", c0="random", seed_offset=H + B)
    g, o, err = check(prob, "fp16")
    assert g["info"]["batch_tile"] == 16
    g8, _, err8 = check(prob, "fp16", batch_tile=8)
    assert g8["info"]["batch_tile"] == 8
    assert np.abs(g["y"] - g8["y"]).max() <= 2 * TOL["fp16"]


@pytest.mark.parametrize("H,B,d", [(6000, 8, 0.01), (4100, 11, 0.02), (9000, 8, 0.004)])
def test_bt8_beyond_byte_offsets(cuda_device, H, B, d):
    """fp16 BT = 8 past H * 16 B > 64 KB: the register pair carries the column in
    16-byte units (the byte offset would not fit 16 bits); every output checked."""
    prob = inputs.make_problem(H, 64, B, 5, d, act="tanh", h0="random", seed_offset=H)
    g, o, err = check(prob, "fp16")
    assert g["info"]["batch_tile"] == 8


def test_C5_shape_sampled_and_partition(cuda_device):
    """C5 layer (H=5760, d=10%, B=64, fp16): the shared-memory weight tier and 8
    batch tiles of 8; samples 0 and 63 checked against the oracle (sampled outputs,
    T shortened to 24 for the CPU side), and the 8-way batch partition of the
    same plan is bit-identical to the full batch."""
    import torch
    from paper_1804_10223_b200.multigpu import shard
    cfg = {k: v for k, v in inputs.CONFIGS["C5"].items() if k != "prec"}
    cfg["T"] = 24
    prob = inputs.make_problem(**cfg)
    m = from_problem(prob, prec="fp16")
    x = torch.from_numpy(prob["x"]).cuda()
    y, _ = m.forward(x)
    torch.cuda.synchronize()
    m.status()
    for b in (0, 63):
        q = dict(prob)
        q["x"] = prob["x"][:, b:b + 1]
        q["B"] = 1
        o = oracle.forward(q)
        assert np.abs(y[:, b].cpu().numpy() - o["y"][:, 0]).max() <= TOL["fp16"]
    parts = []
    for r in range(8):
        s0, c = shard(64, 8, r)
        parts.append(m.forward(x[:, s0:s0 + c].contiguous())[0])
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts, 1), y)


@pytest.mark.parametrize("prec,cell,B,T", [("fp16", "rnn", 4, 37), ("fp32", "rnn", 3, 16), ("fp16", "lstm", 2, 9),
                                           ("fp16", "rnn", 4, 1), ("fp16", "rnn", 4, 2), ("fp16", "rnn", 4, 256),
                                           ("fp32", "lstm", 3, 33)])
def test_forward_host_pipelined(cuda_device, prec, cell, B, T):
    """SRNN_FLAG_RESERVE_SMS: srnn_forward_host projects x chunks on the free SMs while
    the persistent kernel runs and copies y back by progress -- same bits as the
    plain device forward of the same plan, over repeated calls (monotone counters)."""
    import torch
    prob = inputs.make_problem(640, 320, B, T, 0.1, cell=cell, act="tanh", h0="random", c0="random")
    m = from_problem(prob, prec=prec, flags=FLAG_RESERVE_SMS)
    assert m.info()["num_ctas"] <= m.info()["sm_count"] - 4
    xh = torch.from_numpy(prob["x"]).pin_memory().numpy()
    for _ in range(3):
        outs = m.forward_host(xh, prob["h0"], prob["c0"])
        m.status()
    dev = m.forward(torch.from_numpy(prob["x"]).cuda(), torch.from_numpy(prob["h0"]).cuda(),
                    torch.from_numpy(prob["c0"]).cuda() if cell == "lstm" else None)
    torch.cuda.synchronize()
    assert np.array_equal(outs[0], dev[0].cpu().numpy())
    assert np.array_equal(outs[1], dev[1].cpu().numpy())
    o = oracle.forward(prob)
    assert np.abs(outs[0].astype(np.float64) - o["y"]).max() <= TOL[prec]


# ---- dense tensor-core persistent comparator (SRNN_FLAG_DENSE_TC) ----

@pytest.mark.parametrize("cell,H,B,T,d,act", [
    ("rnn", 256, 1, 16, 0.10, "relu"),    # C1 shape, one k-block per warp, B padded to the tile of 4
    ("rnn", 300, 3, 20, 0.05, "tanh"),    # ragged H: zero rows/columns in the last k-block
    ("rnn", 1000, 6, 12, 0.30, "relu"),   # tile of 8, ragged batch
    ("rnn", 2304, 4, 48, 0.30, "relu"),   # C2 shape (9 register fragments per lane)
    ("rnn", 3584, 9, 8, 0.10, "tanh"),    # two row tiles, 16 fragments in shared memory, two batch tiles
    ("lstm", 1024, 4, 20, 0.125, "relu"), # C4 shape (two row tiles)
    ("lstm", 200, 8, 6, 0.10, "relu"),
])
def test_dense_tc_parity(cuda_device, cell, H, B, T, d, act):
    pattern = "row_balanced" if cell == "lstm" else "unstructured"
    prob = inputs.make_problem(H, H, B, T, d, cell=cell, act=act, pattern=pattern, h0="random",
                               c0="random" if cell == "lstm" else "zero", seed_offset=H + 5)
    g, _, _ = check(prob, "fp16", flags=FLAG_DENSE_TC)
    assert g["info"]["dense_m_tiles"] >= 1


def test_dense_tc_integer_exact_and_deterministic(cuda_device):
    prob = inputs.make_integer_problem(200, 6, 4, 3, 0.01, cell="rnn", act="identity")
    o = oracle.forward(prob)
    assert np.abs(o["y"]).max() < 2 ** 10  # 10 significant bits in the fp16 exchange (R16)
    g = run_gpu(prob, "fp16", flags=FLAG_DENSE_TC)
    assert np.array_equal(g["y"].astype(np.float64), o["y"])
    prob = inputs.make_problem(777, 777, 3, 40, 0.1, act="tanh", h0="random")
    a = run_gpu(prob, "fp16", flags=FLAG_DENSE_TC)
    b = run_gpu(prob, "fp16", flags=FLAG_DENSE_TC | FLAG_DEBUG_JITTER)
    assert np.array_equal(a["y"], b["y"])


def test_dense_tc_C2_full(cuda_device):
    """The comparator at the headline configuration, every output vs the oracle."""
    prob = inputs.make_problem(**{k: v for k, v in inputs.CONFIGS["C2"].items() if k != "prec"})
    check(prob, "fp16", flags=FLAG_DENSE_TC)


# ---- stacked layers, time-chunked wavefront ----

@pytest.mark.parametrize("prec,cell", [("fp16", "rnn"), ("fp16", "lstm"), ("fp32", "rnn")])
def test_stacked_chunked_wavefront(cuda_device, prec, cell):
    """Two stacked layers run chunk by chunk (state carried through h0/c0 -> hT/cT, the
    order of the cross-rank layer pipeline) equal the unchunked layer-by-layer run bit for
    bit, and the oracle chain within tolerance."""
    import torch
    from paper_1804_10223_b200.multigpu import forward_stacked_chunked, layer_step
    T, B = 40, 4
    p0 = inputs.make_problem(640, 320, B, T, 0.1, cell=cell, act="tanh", seed_offset=11)
    p1 = inputs.make_problem(512, 640, B, T, 0.2, cell=cell, act="tanh", seed_offset=12)
    plans = [from_problem(p, prec=prec) for p in (p0, p1)]
    x = torch.from_numpy(p0["x"]).cuda()
    steps = [layer_step(m) for m in plans]
    full = forward_stacked_chunked(steps, x, 1)
    for n in (3, 7):
        got = forward_stacked_chunked(steps, x, n)
        torch.cuda.synchronize()
        assert torch.equal(got, full), n
    # each layer against the oracle on the input that layer actually received: layer 0 on
    # x, layer 1 on the GPU's layer-0 output -- both at the north-star tolerance (layer 1's
    # own error, not layer 0's error propagated through W_x)
    y0 = forward_stacked_chunked(steps[:1], x, 1).cpu().numpy()
    for m in plans:
        m.status()
        m.close()
    o0 = oracle.forward(dict(p0))
    assert np.abs(y0.astype(np.float64) - o0["y"]).max() <= TOL[prec]
    q1 = dict(p1)
    q1["x"] = y0.astype(np.float32)
    o1 = oracle.forward(q1)
    err = np.abs(full.cpu().numpy().astype(np.float64) - o1["y"]).max()
    assert err <= TOL[prec], err


@pytest.mark.parametrize("H,B,T,d", [
    (5760, 4, 32, 0.10),   # C3 large-H corner (smem weight tier / narrow lanes), every output
    (1152, 32, 24, 0.50),  # C3 large-batch / high-density corner: two tiles of 16
    (4096, 8, 32, 0.01),   # C3 low-density corner, one tile of 8
])
def test_C3_sweep_corners(cuda_device, H, B, T, d):
    prob = inputs.make_problem(H, H, B, T, d, act="relu", h0="random", seed_offset=3)
    g, o, err = check(prob, "fp16")
    print("C3 corner", H, B, d, "err", err, g["info"]["num_ctas"], g["info"]["batch_tile"])


@pytest.mark.parametrize("flags", [0, FLAG_DENSE_TC])
def test_lost_message_watchdog(cuda_device, monkeypatch, flags):
    """Fault injection: CTA 0 drops its h_2 publish.  The device
    watchdog must end the persistent kernel (no hang) and surface SRNN_ERR_TIMEOUT;
    the status word is cleared by reading it and a fresh plan runs correctly."""
    import torch
    from paper_1804_10223_b200 import SrnnError
    from paper_1804_10223_b200._lib import FLAG_DEBUG_DROP_PUBLISH
    monkeypatch.setenv("SRNN_TIMEOUT_MS", "200")
    prob = inputs.make_problem(512, 512, 4, 8, 0.1, act="tanh")
    m = from_problem(prob, prec="fp16", flags=flags | FLAG_DEBUG_DROP_PUBLISH)
    m.forward(torch.from_numpy(prob["x"]).cuda())
    torch.cuda.synchronize()
    with pytest.raises(SrnnError) as e:
        m.status()
    assert e.value.code == -6
    m.status()  # cleared
    m.close()
    # the pipelined host call must not hang on its y-copy waits either
    m = from_problem(prob, prec="fp16", flags=flags | FLAG_DEBUG_DROP_PUBLISH | FLAG_RESERVE_SMS)
    with pytest.raises(SrnnError) as e:
        m.forward_host(prob["x"])
    assert e.value.code == -6
    m.close()
    check(prob, "fp16", flags=flags)


@pytest.mark.parametrize("concurrent", [False, True])
def test_bidirectional_layer(cuda_device, concurrent):
    """Forward + time-reversed backward plan, y = [y_fwd ; flip(y_bwd)], against the oracle
    run on x and on x reversed; concurrent: the two directions on two streams, half the SMs
    each (slow on B200, but it must stay correct and deadlock-free)."""
    import torch
    from paper_1804_10223_b200.layers import BiSparseRNN
    T, B, H = 24, 4, 700
    pf = inputs.make_problem(H, 300, B, T, 0.1, act="tanh", seed_offset=21)
    pb = inputs.make_problem(H, 300, B, T, 0.1, act="tanh", seed_offset=22)
    pb["x"] = pf["x"]
    n = torch.cuda.get_device_properties(0).multi_processor_count // 2 if concurrent else 0
    bi = BiSparseRNN.from_problems(pf, pb, prec="fp16", num_ctas=n)
    st = (torch.cuda.Stream(), torch.cuda.Stream()) if concurrent else None
    y, hf, hb = bi.forward(torch.from_numpy(pf["x"]).cuda(), streams=st)
    torch.cuda.synchronize()
    bi.status()
    bi.close()
    of = oracle.forward(pf)
    qb = dict(pb)
    qb["x"] = np.ascontiguousarray(pf["x"][::-1])
    ob = oracle.forward(qb)
    ref = np.concatenate([of["y"], ob["y"][::-1]], axis=2)
    err = np.abs(y.cpu().numpy().astype(np.float64) - ref).max()
    assert err <= TOL["fp16"], err
    assert np.abs(hb.cpu().numpy() - ob["hT"]).max() <= TOL["fp16"]


# ---- GRU cell extension (R15) ----

@pytest.mark.parametrize("prec", ["fp32", "fp16"])
@pytest.mark.parametrize("H,B,T,d,pattern", [
    (128, 4, 10, 0.125, "row_balanced"),
    (257, 1, 12, 0.12, "unstructured"),
    (96, 5, 7, 0.3, "unstructured"),
    (200, 8, 6, 0.1, "row_balanced"),
    (300, 16, 5, 0.1, "unstructured"),
])
def test_gru_parity_small(cuda_device, prec, H, B, T, d, pattern):
    prob = inputs.make_problem(H, H, B, T, d, cell="gru", pattern=pattern, h0="random", seed_offset=H + 7)
    check(prob, prec)


def test_gru_C4_shape_full(cuda_device):
    """GRU at the LSTM case study's shape (H = 1024, B = 4, T = 100, 12.5% row-balanced), fp16."""
    prob = inputs.make_problem(1024, 1024, 4, 100, 0.125, cell="gru", pattern="row_balanced")
    check(prob, "fp16")


@pytest.mark.parametrize("H,I,B,T,cell", [(384, 200, 3, 7, "rnn"), (130, 201, 2, 9, "lstm"), (2304, 2304, 4, 256, "rnn"),
                                        (300, 77, 5, 3, "gru")])
def test_input_projection_fp32_3xtf32_opt_in(cuda_device, H, I, B, T, cell):
    """fp32 mode, SRNN_FLAG_FP32_TC_GEMM: the 3xTF32 tcgen05 projection (tf32 hi/lo split, ragged K
    padded to 4) against the fp64 oracle, within its documented ~1.5e-8 * K relative error (the
    tensor cores' fp32 accumulation; the default exact SIMT GEMM is checked at fp32 level)."""
    import torch
    from paper_1804_10223_b200._lib import FLAG_FP32_TC_GEMM
    prob = inputs.make_problem(H, I, B, T, 0.05, cell=cell)
    x = torch.from_numpy(prob["x"]).cuda()
    ref = oracle.input_projection(prob["x"], prob["wx"], prob["bias"][:prob["G"] * H])
    got = {}
    for name, flags in (("tc", FLAG_FP32_TC_GEMM), ("simt", 0)):
        m = from_problem(prob, prec="fp32", flags=flags)
        got[name] = m.input_projection(x).cpu().numpy().astype(np.float64)
        torch.cuda.synchronize()
        m.close()
    scale = max(1.0, float(np.abs(ref).max()))
    print("3xtf32", H, I, "err tc", np.abs(got["tc"] - ref).max(), "err simt", np.abs(got["simt"] - ref).max())
    assert np.abs(got["tc"] - ref).max() <= 1.5e-8 * I * scale + 1e-6
    assert np.abs(got["simt"] - ref).max() <= 1e-5


@pytest.mark.parametrize("prec", ["fp32", "fp16"])
def test_tag_epoch_wrap(cuda_device, monkeypatch, prec):
    """Timestep tags are u32 epoch + s: a plan whose epoch starts just below 2^32 must clear its
    exchange buffers and restart the epoch instead of wrapping into stale tags -- every call,
    before and after the restart, matches the oracle."""
    import torch
    monkeypatch.setenv("SRNN_DEBUG_EPOCH0", str(2 ** 32 - 30))
    prob = inputs.make_problem(300, 300, 4, 12, 0.1, act="tanh", h0="random")
    m = from_problem(prob, prec=prec)
    o = oracle.forward(prob)
    x = torch.from_numpy(prob["x"]).cuda()
    h0 = torch.from_numpy(prob["h0"]).cuda()
    for _ in range(4):  # 13 tags per call: the third call wraps
        y, _ = m.forward(x, h0)
        torch.cuda.synchronize()
        m.status()
        assert np.abs(y.cpu().numpy() - o["y"]).max() <= TOL[prec]
    m.close()


# ---- round 2: the method's defining edge cases at the headline shape, NaN, full-T C5 ----

def _oracle_samples(prob, samples, threads=None):
    """Oracle outputs of selected batch samples (samples are independent, PAPER.md:43-49 per
    sequence), run in parallel host threads (the oracle's C calls release the GIL)."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    def one(b):
        q = dict(prob)
        q["x"] = np.ascontiguousarray(prob["x"][:, b:b + 1])
        q["B"] = 1
        for k in ("h0", "c0"):
            if prob.get(k) is not None:
                q[k] = np.ascontiguousarray(prob[k][b:b + 1])
        return b, oracle.forward(q)

    with ThreadPoolExecutor(threads or max(1, os.cpu_count() or 1)) as ex:
        return dict(ex.map(one, samples))


@pytest.mark.parametrize("prec", ["fp16", "fp32"])
@pytest.mark.parametrize("d", [0.0, 1.0])
def test_C2_density_extremes(cuda_device, prec, d):
    """C2 shape (H=2304, B=4, T=256) at density 0 (h_t = g(b'_t): no recurrent term,
    PAPER.md:46 Eq. 2 with U_r = 0) and density 1 (the dense RNN the method reduces to,
    PAPER.md:91/:100: padding and reordering do not change the result) through the
    sparse kernel -- every output against the oracle.  A plan the chip cannot hold must
    say so (SRNN_ERR_NOT_ON_CHIP), never fall back."""
    from paper_1804_10223_b200 import SrnnError
    cfg = {k: v for k, v in inputs.CONFIGS["C2"].items() if k != "prec"}
    cfg["density"] = d
    prob = inputs.make_problem(**cfg, h0="random")
    try:
        g, o, err = check(prob, prec)
    except SrnnError as ex:
        assert d == 1.0 and prec == "fp32" and ex.code == -2, ex
        pytest.skip("fp32 pairs of a dense 2304 layer exceed the on-chip capacity (SRNN_ERR_NOT_ON_CHIP)")
    if d == 0.0:
        assert g["info"]["nnz"] == 0
    print("C2 density", d, prec, "max-abs err", err, g["info"]["num_ctas"], g["info"]["batch_tile"])


@pytest.mark.parametrize("cell,act,prec", [("rnn", "tanh", "fp16"), ("rnn", "tanh", "fp32"),
                                           ("rnn", "relu", "fp16"), ("lstm", "tanh", "fp16")])
def test_nan_propagates(cuda_device, cell, act, prec):
    """A NaN in x (NaN inputs are propagated, not trapped): the poisoned
    sample's outputs are NaN exactly where the oracle's are (from the poisoned step on,
    every unit -- W_x is dense), the other samples are untouched and within tolerance.
    ReLU absorbs NaN in both (g(NaN) = 0: u > 0 is false in the oracle, fmax in the kernel)."""
    prob = inputs.make_problem(700, 700, 4, 12, 0.1, cell=cell, act=act, h0="random", c0="random")
    prob["x"] = prob["x"].copy()
    prob["x"][5, 2, 17] = np.nan
    g = run_gpu(prob, prec)
    o = oracle.forward(prob)
    gy, oy = g["y"].astype(np.float64), o["y"]
    assert np.array_equal(np.isnan(gy), np.isnan(oy))
    if act != "relu" or cell == "lstm":
        assert np.isnan(oy[5:, 2]).all() and not np.isnan(oy[:5]).any()
    fin = ~np.isnan(oy)
    assert np.abs(gy[fin] - oy[fin]).max() <= TOL[prec]
    assert not np.isnan(gy[:, [0, 1, 3]]).any()


def test_C5_full_T_sampled_per_shard(cuda_device):
    """C5 (H=5760, d=10%, B=64, T=512, fp16) at its full length: the 8-way batch partition
    of the bench (B/8 = 8 sequences per shard) is bit-identical to the full batch, and two
    samples of every shard (its first and last) match the oracle over all 512 steps."""
    import torch
    from paper_1804_10223_b200.multigpu import shard
    cfg = {k: v for k, v in inputs.CONFIGS["C5"].items() if k != "prec"}
    prob = inputs.make_problem(**cfg)
    m = from_problem(prob, prec="fp16")
    x = torch.from_numpy(prob["x"]).cuda()
    y, _ = m.forward(x)
    torch.cuda.synchronize()
    m.status()
    samples = []
    for r in range(8):
        s0, c = shard(64, 8, r)
        part = m.forward(x[:, s0:s0 + c].contiguous())[0]
        torch.cuda.synchronize()
        assert torch.equal(part, y[:, s0:s0 + c]), r
        samples += [s0, s0 + c - 1]
    yc = y.cpu().numpy().astype(np.float64)
    for b, o in _oracle_samples(prob, samples).items():
        err = np.abs(yc[:, b] - o["y"][:, 0]).max()
        assert err <= TOL["fp16"], (b, err)


def test_y_batch_major_layout(cuda_device):
    """SRNN_FLAG_Y_BATCH_MAJOR writes y as [B][T][H]: the same bits as the default [T][B][H]
    layout, transposed (ragged tiles included)."""
    import torch
    from paper_1804_10223_b200 import FLAG_Y_BATCH_MAJOR
    prob = inputs.make_problem(777, 777, 11, 9, 0.1, act="tanh", h0="random")
    x = torch.from_numpy(prob["x"]).cuda()
    h0 = torch.from_numpy(prob["h0"]).cuda()
    for prec in ("fp16", "fp32"):
        a = from_problem(prob, prec=prec)
        b = from_problem(prob, prec=prec, flags=FLAG_Y_BATCH_MAJOR)
        ya, ha = a.forward(x, h0)
        yb, hb = b.forward(x, h0)
        torch.cuda.synchronize()
        assert tuple(yb.shape) == (11, 9, 777)
        assert torch.equal(ya.permute(1, 0, 2), yb) and torch.equal(ha, hb)
        yh, _ = b.forward_host(prob["x"], prob["h0"])
        assert np.array_equal(yh, yb.cpu().numpy())
        a.close()
        b.close()


def test_plans_on_concurrent_host_threads(cuda_device):
    """Distinct plans are independent (include/srnn.h): two host threads each drive their own
    plan and stream at the same time (the per-launch shared-memory opt-in of the tcgen05
    projection) and get the single-thread results bit for bit."""
    import threading
    import torch
    probs = [inputs.make_problem(1152, 1152, 4, 20, 0.1, act="tanh", seed_offset=s) for s in (1, 2)]
    ref = []
    for p in probs:
        m = from_problem(p, prec="fp16")
        ref.append(m.forward(torch.from_numpy(p["x"]).cuda())[0].cpu())
        m.close()
    out = [None, None]

    def run(i):
        torch.cuda.set_device(0)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            m = from_problem(probs[i], prec="fp16")
            for _ in range(3):
                y = m.forward(torch.from_numpy(probs[i]["x"]).cuda(), stream=s)[0]
            s.synchronize()
            out[i] = y.cpu()
            m.status()
            m.close()

    th = [threading.Thread(target=run, args=(i,)) for i in (0, 1)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in (0, 1):
        assert torch.equal(out[i], ref[i])


def test_plans_on_two_devices(cuda_device):
    """One process, one plan per device (the per-device GEMM attribute)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two visible GPUs (the round-end box has one)")
    prob = inputs.make_problem(1152, 1152, 4, 16, 0.1, act="tanh")
    ys = []
    for dev in (0, 1):
        m = from_problem(prob, prec="fp16", device=dev)
        ys.append(m.forward(torch.from_numpy(prob["x"]).to(f"cuda:{dev}"))[0].cpu())
        m.status()
        m.close()
    assert torch.equal(ys[0], ys[1])


@pytest.mark.parametrize("prec,cell,pattern,B", [("fp16", "rnn", "skewed", 4), ("fp32", "rnn", "skewed", 3),
                                                 ("fp16", "lstm", "skewed", 4), ("fp16", "gru", "unstructured", 5),
                                                 ("fp16", "rnn", "skewed", 16)])
def test_class_balance_parity(cuda_device, prec, cell, pattern, B):
    """SRNN_FLAG_CLASS_BALANCE: units dealt over the CTAs by nonzero class, the
    exchange in the permuted order, outputs back in unit order -- every output vs the oracle."""
    from paper_1804_10223_b200 import FLAG_CLASS_BALANCE
    prob = inputs.make_problem(1000, 600, B, 12, 0.1, cell=cell, act="tanh", pattern=pattern, h0="random",
                               c0="random", seed_offset=B)
    check(prob, prec, flags=FLAG_CLASS_BALANCE)


def test_class_balance_integer_exact(cuda_device):
    """Integer-exact inputs: any summation order is exact, so the permuted plan equals the
    oracle (and the unpermuted plan) bit for bit."""
    from paper_1804_10223_b200 import FLAG_CLASS_BALANCE
    prob = inputs.make_integer_problem(200, 48, 4, 5, 0.02, act="identity")
    o = oracle.forward(prob)
    a = run_gpu(prob, "fp32", flags=FLAG_CLASS_BALANCE)
    assert np.array_equal(a["y"].astype(np.float64), o["y"])


@pytest.mark.parametrize("prec,cell,H,B,T,d,act", [
    ("fp16", "rnn", 1000, 4, 12, 0.3, "relu"),
    ("fp32", "rnn", 1000, 4, 12, 0.3, "relu"),
    ("fp16", "rnn", 777, 3, 20, 0.1, "tanh"),     # ragged H (odd halves), B < tile
    ("fp32", "rnn", 513, 6, 9, 0.05, "identity"),  # two batch tiles
    ("fp16", "rnn", 2304, 8, 10, 0.3, "relu"),    # one tile of 8 (LDS.128)
    ("fp16", "lstm", 1024, 4, 10, 0.125, "tanh"),
    ("fp16", "gru", 600, 5, 8, 0.1, "tanh"),
    ("fp16", "rnn", 300, 1, 16, 0.1, "relu"),     # BT = 1
])
def test_column_split_parity(cuda_device, prec, cell, H, B, T, d, act):
    """SRNN_FLAG_COLUMN_SPLIT ("split one row among multiple blocks"): 2-CTA clusters,
    each CTA one column half, partial sums added through DSMEM -- every output vs the oracle."""
    from paper_1804_10223_b200 import FLAG_COLUMN_SPLIT
    prob = inputs.make_problem(H, H, B, T, d, cell=cell, act=act, h0="random", c0="random", seed_offset=H + B)
    g, o, err = check(prob, prec, flags=FLAG_COLUMN_SPLIT)
    assert g["info"]["column_split"] == 1 and g["info"]["num_ctas"] % 2 == 0


def test_column_split_integer_exact(cuda_device):
    """Integer-exact inputs: the split sums (half 0 + half 1) are exact, so the split plan equals
    the oracle bit for bit, like the unsplit plan."""
    from paper_1804_10223_b200 import FLAG_COLUMN_SPLIT
    prob = inputs.make_integer_problem(500, 48, 4, 6, 0.02, act="identity")
    o = oracle.forward(prob)
    a = run_gpu(prob, "fp32", flags=FLAG_COLUMN_SPLIT)
    assert np.array_equal(a["y"].astype(np.float64), o["y"])
    # fp16 h rounds the growing integers (> 2^10) the same way in both plans: split == unsplit
    b = run_gpu(prob, "fp16", flags=FLAG_COLUMN_SPLIT)
    c = run_gpu(prob, "fp16")
    assert np.array_equal(b["y"], c["y"])


def test_column_split_jitter_deterministic(cuda_device):
    """Random per-CTA delays change nothing (the pair's DSMEM sum has a fixed order)."""
    from paper_1804_10223_b200 import FLAG_COLUMN_SPLIT
    prob = inputs.make_problem(1152, 1152, 4, 24, 0.1, act="tanh", h0="random")
    a = run_gpu(prob, "fp16", flags=FLAG_COLUMN_SPLIT)
    b = run_gpu(prob, "fp16", flags=FLAG_COLUMN_SPLIT | FLAG_DEBUG_JITTER)
    assert np.array_equal(a["y"], b["y"])


def test_column_split_lost_message_watchdog(cuda_device, monkeypatch):
    """A lost exchange message under the column split ends the launch through the watchdog (both
    CTAs of every pair leave together: no cluster-barrier hang)."""
    import torch
    from paper_1804_10223_b200 import FLAG_COLUMN_SPLIT, SrnnError
    from paper_1804_10223_b200._lib import FLAG_DEBUG_DROP_PUBLISH
    monkeypatch.setenv("SRNN_TIMEOUT_MS", "200")
    prob = inputs.make_problem(1000, 1000, 4, 8, 0.1, act="tanh")
    m = from_problem(prob, prec="fp16", flags=FLAG_COLUMN_SPLIT | FLAG_DEBUG_DROP_PUBLISH)
    m.forward(torch.from_numpy(prob["x"]).cuda())
    torch.cuda.synchronize()
    with pytest.raises(SrnnError) as e:
        m.status()
    assert e.value.code == -6
    m.close()


@pytest.mark.parametrize("H,d", [(36000, 0.0025), (41000, 0.0025)])
def test_column_split_capacity_beyond_frontier(cuda_device, monkeypatch, H, d):
    """(f)4: the column split stages half of h, so fp16 layers past the unsplit limit (16-bit
    staged offsets: H <= 32768 at one sample per tile; host-only frontier 32680 @ 0.25%) run on
    chip -- every output checked; the unsplit plan of the same layer is refused."""
    from paper_1804_10223_b200 import FLAG_COLUMN_SPLIT, FLAG_HOST_ONLY, SrnnError
    prob = inputs.make_problem(H, 64, 1, 5, d, act="tanh", h0="random")
    monkeypatch.setenv("SRNN_NO_AUTO_SPLIT", "1")  # the unsplit plan is refused ...
    with pytest.raises(SrnnError):
        from_problem(prob, prec="fp16", flags=FLAG_HOST_ONLY)
    monkeypatch.delenv("SRNN_NO_AUTO_SPLIT")  # ... the planner splits by itself, or on request
    assert from_problem(prob, prec="fp16", flags=FLAG_HOST_ONLY).info()["column_split"] == 1
    g, o, err = check(prob, "fp16", flags=FLAG_COLUMN_SPLIT)
    print(H, d, g["info"])


# ---- partial progress (SRNN_FLAG_STAGED) ----
@pytest.mark.parametrize("cell,H,B,T,d,act,pattern", [
    ("rnn", 2304, 4, 24, 0.30, "relu", "unstructured"),    # C2 shape, short T
    ("rnn", 1152, 4, 40, 0.10, "tanh", "unstructured"),    # Table 1 shape
    ("rnn", 1200, 4, 17, 0.05, "identity", "unstructured"),  # low density
    ("lstm", 1024, 4, 20, 0.125, "tanh", "row_balanced"),  # C4 NMT shape
    ("gru", 777, 4, 15, 0.2, "tanh", "unstructured"),      # ragged H
    ("rnn", 2304, 8, 16, 0.30, "relu", "unstructured"),    # tile of 8
    ("rnn", 1500, 13, 9, 0.1, "tanh", "unstructured"),     # several tiles, ragged (may fall back)
])
def test_staged_parity(cuda_device, cell, H, B, T, d, act, pattern):
    """The staged plan (early chunks staged and operated on while the late chunks arrive) vs the
    oracle on every output, and vs the one-stage plan (same values up to fp reassociation).  The
    ragged multi-tile case may fall back to one stage (its staged instance spills: the planner
    keeps the spill-free one); the rest must be staged."""
    from paper_1804_10223_b200 import FLAG_STAGED
    prob = inputs.make_problem(H, H, B, T, d, cell=cell, act=act, pattern=pattern, h0="random", c0="random",
                               seed_offset=H + B)
    g, o, err = check(prob, "fp16", flags=FLAG_STAGED)
    assert g["info"]["staged"] == 1 or B == 13, g["info"]
    g0 = run_gpu(prob, "fp16")
    assert g0["info"]["staged"] == 0
    assert np.abs(g["y"] - g0["y"]).max() <= TOL["fp16"]


def test_staged_integer_exact_and_deterministic(cuda_device):
    """Integer-exact inputs: the staged plan equals the oracle bit for bit, with and without
    per-CTA jitter (the early/late barrier order cannot change a value)."""
    from paper_1804_10223_b200 import FLAG_STAGED
    # the fp16 exchange keeps 10 significant bits (R16): integers up to 2^10 are exact
    prob = inputs.make_integer_problem(600, 6, 4, 3, 0.01, act="identity")
    o = oracle.forward(prob)
    assert np.abs(o["y"]).max() < 2 ** 10
    a = run_gpu(prob, "fp16", flags=FLAG_STAGED)
    assert a["info"]["staged"] == 1
    assert np.array_equal(a["y"].astype(np.float64), o["y"])
    b = run_gpu(prob, "fp16", flags=FLAG_STAGED | FLAG_DEBUG_JITTER)
    assert np.array_equal(a["y"], b["y"])


def test_staged_lost_message_watchdog(cuda_device, monkeypatch):
    """A lost exchange message under the staged plan: the early or late wait times out, the
    launch reports SRNN_ERR_TIMEOUT instead of hanging, and a fresh staged plan is correct."""
    import torch

    from paper_1804_10223_b200 import FLAG_STAGED, SrnnError
    from paper_1804_10223_b200._lib import FLAG_DEBUG_DROP_PUBLISH
    monkeypatch.setenv("SRNN_TIMEOUT_MS", "200")
    prob = inputs.make_problem(1152, 1152, 4, 8, 0.1, act="tanh")
    m = from_problem(prob, prec="fp16", flags=FLAG_STAGED | FLAG_DEBUG_DROP_PUBLISH)
    assert m.info()["staged"] == 1
    m.forward(torch.from_numpy(prob["x"]).cuda())
    torch.cuda.synchronize()
    with pytest.raises(SrnnError) as e:
        m.status()
    assert e.value.code == -6
    m.close()
    check(prob, "fp16", flags=FLAG_STAGED)
