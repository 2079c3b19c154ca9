"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: it only draws random
patterns and values (numpy PCG64) with the shapes and distributions of the
paper's workloads.  Both ``oracle/`` and the CUDA path consume the arrays it
returns; neither imports the other.  Recipe (DESIGN.md "Input recipe",
SURVEY.md Sec. 8(d) d-ii):

* pattern "unstructured": nnz = round(d * R * H) positions drawn uniformly
  without replacement over the R x H recurrent matrix (random unstructured
  pattern as used for DS2; nnz definition pinned by the
  constant-nnz identity 2304^2 * 0.25 = 11520^2 * 0.01).
* pattern "row_balanced": k = round(d * H) columns per row, uniform without
  replacement (load-balance-aware pruning).
* W_h ~ U(-a, a), a = rho * sqrt(3 / (d * H)), rho = 0.8 (spectral radius
  ~0.8 by the circular law, keeps activations O(1) over 256 steps).
* W_x ~ U(-sqrt(3/I), sqrt(3/I)), x ~ U(-1, 1), b ~ U(-0.1, 0.1), h0 = 0
  (optionally h0, c0 ~ U(-1, 1)).
* seeds: pattern 1804, W_h values 10223, W_x 2018, x 7, b 11, h0 13, c0 17,
  each + seed_offset.

Shapes: rowptr int32 [R+1], col int32 [nnz] (ascending within a row),
val float32 [nnz], wx float32 [R, I], bias float32 [R], x float32 [T, B, I],
h0/c0 float32 [B, H] or None, with R = G*H (G = 1 RNN, 4 LSTM, gate blocks
[i; f; g; o]).
"""
from __future__ import annotations

import numpy as np

SEEDS = {"pattern": 1804, "wh": 10223, "wx": 2018, "x": 7, "b": 11, "h0": 13, "c0": 17}


def _rng(name, off):
    return np.random.Generator(np.random.PCG64(SEEDS[name] + int(off)))


def sparse_pattern(R, H, density, pattern="unstructured", seed_offset=0):
    """Return (rowptr int32 [R+1], col int32 [nnz]) with ascending columns per row."""
    rng = _rng("pattern", seed_offset)
    if pattern == "unstructured":
        total = R * H
        nnz = int(round(density * total))
        nnz = max(0, min(nnz, total))
        if nnz == total:
            pos = np.arange(total, dtype=np.int64)
        elif nnz == 0:
            pos = np.zeros(0, dtype=np.int64)
        else:
            pos = np.sort(rng.choice(total, size=nnz, replace=False).astype(np.int64))
        rows = pos // H
        col = (pos % H).astype(np.int32)
        counts = np.bincount(rows, minlength=R).astype(np.int64)
    elif pattern == "row_balanced":
        k = int(round(density * H))
        k = max(0, min(k, H))
        col = np.empty(R * k, dtype=np.int32)
        for r in range(R):
            col[r * k:(r + 1) * k] = np.sort(rng.choice(H, size=k, replace=False))
        counts = np.full(R, k, dtype=np.int64)
    elif pattern == "skewed":
        # non-uniform row sparsity (the load-imbalance case of PAPER.md:91/:188): row lengths
        # proportional to lognormal(0, 0.5) draws, scaled to nnz = round(d * R * H), <= H each
        nnz = int(round(density * R * H))
        wts = rng.lognormal(0.0, 0.5, size=R)
        counts = np.minimum(np.floor(wts / wts.sum() * nnz).astype(np.int64), H)
        short = nnz - int(counts.sum())
        for r in np.argsort(-wts):
            if short <= 0:
                break
            if counts[r] < H:
                counts[r] += 1
                short -= 1
        col = np.concatenate([np.sort(rng.choice(H, size=int(k), replace=False)) if k else np.zeros(0, np.int64)
                              for k in counts]).astype(np.int32)
    else:
        raise ValueError(f"unknown pattern {pattern!r}")
    rowptr = np.zeros(R + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    return rowptr.astype(np.int32), col


def make_problem(H, I=None, B=4, T=256, density=0.1, cell="rnn", act="relu",
                 pattern="unstructured", seed_offset=0, rho=0.8, h0="zero", c0="zero"):
    """Synthetic problem with the paper's shapes (see module docstring)."""
    I = H if I is None else I
    G = {"rnn": 1, "lstm": 4, "gru": 3}[cell]
    R = G * H
    rowptr, col = sparse_pattern(R, H, density, pattern, seed_offset)
    nnz = int(rowptr[-1])
    d_eff = max(density, 1.0 / H)
    a = rho * np.sqrt(3.0 / (d_eff * H))
    val = _rng("wh", seed_offset).uniform(-a, a, size=nnz).astype(np.float32)
    ax = np.sqrt(3.0 / I)
    wx = _rng("wx", seed_offset).uniform(-ax, ax, size=(R, I)).astype(np.float32)
    x = _rng("x", seed_offset).uniform(-1.0, 1.0, size=(T, B, I)).astype(np.float32)
    # GRU: [b_r; b_z; b_n; b_hn] -- the n gate's recurrent bias sits inside r * (.)
    bias = _rng("b", seed_offset).uniform(-0.1, 0.1, size=R + (H if cell == "gru" else 0)).astype(np.float32)
    prob = {"H": H, "I": I, "B": B, "T": T, "density": density, "cell": cell, "act": act,
            "pattern": pattern, "G": G, "rowptr": rowptr, "col": col, "val": val,
            "wx": wx, "bias": bias, "x": x, "h0": None, "c0": None, "nnz": nnz}
    if h0 == "random":
        prob["h0"] = _rng("h0", seed_offset).uniform(-1, 1, size=(B, H)).astype(np.float32)
    if cell == "lstm" and c0 == "random":
        prob["c0"] = _rng("c0", seed_offset).uniform(-1, 1, size=(B, H)).astype(np.float32)
    return prob


def make_integer_problem(H, I, B, T, density, cell="rnn", act="identity", seed_offset=0):
    """Integer-exact inputs (SURVEY.md Sec. 8(c) c3 "bit-exact pin").

    W_h, W_x in {-1, +1} at their positions (W_x dense in {-1, 0, 1}), x and b
    small integers.  With every partial sum below 2^24 in magnitude all fp32 /
    fp16-weight arithmetic is exact, so any summation order gives the same
    bits.  The caller checks the magnitude bound on the oracle's output.
    """
    prob = make_problem(H, I, B, T, density, cell=cell, act=act, seed_offset=seed_offset)
    rng = np.random.Generator(np.random.PCG64(99 + seed_offset))
    prob["val"] = rng.choice(np.array([-1.0, 1.0], np.float32), size=prob["nnz"])
    prob["wx"] = rng.integers(-1, 2, size=prob["wx"].shape).astype(np.float32)
    prob["x"] = rng.integers(-2, 3, size=prob["x"].shape).astype(np.float32)
    prob["bias"] = rng.integers(-3, 4, size=prob["bias"].shape).astype(np.float32)
    return prob


# Named configurations of BASELINE.json "configs" (SURVEY.md Sec. 8 shorthand).
CONFIGS = {
    "C1": dict(H=256, I=256, B=1, T=16, density=0.10, cell="rnn", act="relu", prec="fp32"),
    "C2": dict(H=2304, I=2304, B=4, T=256, density=0.30, cell="rnn", act="relu", prec="fp16"),
    "C4_nmt": dict(H=1024, I=1024, B=4, T=100, density=0.125, cell="lstm", pattern="row_balanced", prec="fp16"),
    "C4_nmt47": dict(H=1024, I=1024, B=4, T=100, density=48 / 1024, cell="lstm", pattern="row_balanced", prec="fp16"),
    "C4_speech": dict(H=1024, I=1024, B=1, T=100, density=0.12, cell="lstm", pattern="unstructured", prec="fp16"),
    "C5": dict(H=5760, I=5760, B=64, T=512, density=0.10, cell="rnn", act="relu", prec="fp16"),
}
