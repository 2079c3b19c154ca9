"""Pins for the CPU fp64 oracle (oracle/) against things other than itself.

Each test names what fixes the expected value: a worked example (golden file),
a closed form, an independent library implementation (torch.nn.RNN/LSTM,
numpy matmul / matrix power), or an invariant of Eq. 1/2.
A dropped term, a wrong sign, a transposed operand or a wrong gate order in
the oracle fails at least one of them.
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1804_10223_b200 import inputs

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def dense_to_csr(U):
    U = np.asarray(U, dtype=np.float64)
    rowptr = [0]
    col, val = [], []
    for r in range(U.shape[0]):
        nz = np.nonzero(U[r])[0]
        col.extend(nz.tolist())
        val.extend(U[r, nz].tolist())
        rowptr.append(len(col))
    return np.array(rowptr), np.array(col, dtype=np.int32), np.array(val)


def csr_to_dense(rowptr, col, val, R, H):
    U = np.zeros((R, H))
    for r in range(R):
        for p in range(rowptr[r], rowptr[r + 1]):
            U[r, col[p]] += val[p]
    return U


# ---------------------------------------------------------------- golden ---

def test_golden_precompute_input():
    g = json.load(open(os.path.join(GOLD, "spec_worked_examples.json")))
    for ex in g["precompute_input"]:
        bp = oracle.input_projection(np.array([ex["x"]]), np.array(ex["W"]), np.array(ex["b"]))
        assert np.array_equal(bp[0], np.array(ex["expect"], dtype=np.float64)), ex["cite"]


def test_golden_rnn_step():
    g = json.load(open(os.path.join(GOLD, "spec_worked_examples.json")))
    for ex in g["rnn_step"]:
        H = len(ex["h_prev"])
        rp, cl, vl = dense_to_csr(ex["U"])
        bp = np.array(ex["b_prime"], dtype=np.float64).reshape(1, 1, H)
        y, hT = oracle.rnn_forward(H, rp, cl, vl, bp, np.array([ex["h_prev"]]), ex["act"])
        assert np.array_equal(y[0, 0], np.array(ex["expect"], dtype=np.float64)), ex["cite"]


def test_golden_lstm_step():
    g = json.load(open(os.path.join(GOLD, "spec_worked_examples.json")))
    for ex in g["lstm_step"]:
        H = ex["H"]
        rp = np.zeros(4 * H + 1, dtype=np.int64)
        bp = np.array(ex["b_prime"], dtype=np.float64).reshape(1, 1, 4 * H)
        y, hT, cT = oracle.lstm_forward(H, rp, np.zeros(0, np.int32), np.zeros(0), bp,
                                        np.zeros((1, H)), np.array([ex["c_prev"]]))
        assert np.allclose(cT[0], ex["expect_c"], atol=ex["atol"], rtol=0), ex["cite"]
        if "expect_h" in ex:
            assert np.allclose(hT[0], ex["expect_h"], atol=ex["atol"], rtol=0), ex["cite"]


def test_golden_hand_rnn_h3_exact():
    g = json.load(open(os.path.join(GOLD, "hand_rnn_h3.json")))
    H = g["H"]
    rp, cl, vl = dense_to_csr(g["U_dense"])
    bp = np.tile(np.array(g["b_prime"], dtype=np.float64), (g["T"], 1)).reshape(g["T"], 1, H)
    y, hT = oracle.rnn_forward(H, rp, cl, vl, bp, None, g["act"])
    assert np.array_equal(y[:, 0, :], np.array(g["expect_h"], dtype=np.float64))


# ----------------------------------------------------------- closed forms ---

@pytest.mark.parametrize("H,B,T,d", [(8, 2, 5, 0.5), (37, 3, 12, 0.2), (64, 1, 30, 0.1)])
def test_identity_activation_closed_form(H, B, T, d):
    """g = identity: h_t = U^t h0 + sum_{s=1..t} U^{t-s} b'_s  (unrolled Eq. 2)."""
    p = inputs.make_problem(H, 5, B, T, d, act="identity", h0="random", seed_offset=H)
    U = csr_to_dense(p["rowptr"], p["col"], p["val"].astype(np.float64), H, H)
    assert not np.allclose(U, U.T)  # asymmetric: a transposed operand would fail
    bp = oracle.input_projection(p["x"], p["wx"], p["bias"])
    y, hT = oracle.rnn_forward(H, p["rowptr"], p["col"], p["val"], bp, p["h0"], "identity")
    h0 = p["h0"].astype(np.float64)
    for t in range(1, T + 1):
        ref = (np.linalg.matrix_power(U, t) @ h0.T).T
        for s in range(1, t + 1):
            ref = ref + (np.linalg.matrix_power(U, t - s) @ bp[s - 1].T).T
        np.testing.assert_allclose(y[t - 1], ref, rtol=1e-11, atol=1e-11)


def test_input_projection_vs_numpy_matmul():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((3, 4, 7))
    W = rng.standard_normal((11, 7))
    b = rng.standard_normal(11)
    bp = oracle.input_projection(x, W, b)
    np.testing.assert_allclose(bp, x @ W.T + b, rtol=1e-13, atol=1e-13)


# ------------------------------------------------- independent libraries ---

@pytest.mark.parametrize("act", ["relu", "tanh"])
def test_rnn_density1_vs_torch_rnn(act):
    """d = 1: the sparse layer is a dense torch.nn.RNN (float64, bias_hh = 0)."""
    torch = pytest.importorskip("torch")
    H, I, B, T = 24, 10, 3, 9
    p = inputs.make_problem(H, I, B, T, 1.0, act=act, h0="random")
    assert p["nnz"] == H * H
    rnn = torch.nn.RNN(I, H, nonlinearity=act, dtype=torch.float64)
    with torch.no_grad():
        rnn.weight_hh_l0.copy_(torch.from_numpy(csr_to_dense(p["rowptr"], p["col"], p["val"], H, H)))
        rnn.weight_ih_l0.copy_(torch.from_numpy(p["wx"].astype(np.float64)))
        rnn.bias_ih_l0.copy_(torch.from_numpy(p["bias"].astype(np.float64)))
        rnn.bias_hh_l0.zero_()
        yt, hn = rnn(torch.from_numpy(p["x"].astype(np.float64)),
                     torch.from_numpy(p["h0"].astype(np.float64))[None])
    o = oracle.forward(p, act=act)
    np.testing.assert_allclose(o["y"], yt.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(o["hT"], hn[0].numpy(), rtol=1e-12, atol=1e-12)


def test_lstm_density1_vs_torch_lstm():
    torch = pytest.importorskip("torch")
    H, I, B, T = 16, 9, 2, 7
    p = inputs.make_problem(H, I, B, T, 1.0, cell="lstm", h0="random", c0="random")
    lstm = torch.nn.LSTM(I, H, dtype=torch.float64)
    with torch.no_grad():
        lstm.weight_hh_l0.copy_(torch.from_numpy(csr_to_dense(p["rowptr"], p["col"], p["val"], 4 * H, H)))
        lstm.weight_ih_l0.copy_(torch.from_numpy(p["wx"].astype(np.float64)))
        lstm.bias_ih_l0.copy_(torch.from_numpy(p["bias"].astype(np.float64)))
        lstm.bias_hh_l0.zero_()
        yt, (hn, cn) = lstm(torch.from_numpy(p["x"].astype(np.float64)),
                            (torch.from_numpy(p["h0"].astype(np.float64))[None],
                             torch.from_numpy(p["c0"].astype(np.float64))[None]))
    o = oracle.forward(p)
    np.testing.assert_allclose(o["y"], yt.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(o["hT"], hn[0].numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(o["cT"], cn[0].numpy(), rtol=1e-12, atol=1e-12)


def test_sparse_lstm_vs_torch_lstm_densified():
    """Pruned LSTM == torch.nn.LSTM with the zeros put back."""
    torch = pytest.importorskip("torch")
    H, I, B, T = 20, 6, 2, 5
    p = inputs.make_problem(H, I, B, T, 0.2, cell="lstm", pattern="row_balanced", h0="random")
    lstm = torch.nn.LSTM(I, H, dtype=torch.float64)
    with torch.no_grad():
        lstm.weight_hh_l0.copy_(torch.from_numpy(csr_to_dense(p["rowptr"], p["col"], p["val"], 4 * H, H)))
        lstm.weight_ih_l0.copy_(torch.from_numpy(p["wx"].astype(np.float64)))
        lstm.bias_ih_l0.copy_(torch.from_numpy(p["bias"].astype(np.float64)))
        lstm.bias_hh_l0.zero_()
        yt, _ = lstm(torch.from_numpy(p["x"].astype(np.float64)),
                     (torch.from_numpy(p["h0"].astype(np.float64))[None], torch.zeros(1, B, H, dtype=torch.float64)))
    o = oracle.forward(p)
    np.testing.assert_allclose(o["y"], yt.numpy(), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("density,pattern", [(1.0, "unstructured"), (0.3, "row_balanced")])
def test_gru_vs_torch_gru_densified(density, pattern):
    """GRU cell extension (R15) == torch.nn.GRU float64 with the pruned zeros put
    back: gate blocks [r; z; n], bias_ih = b[:3H], bias_hh = [0; 0; b_hn]."""
    torch = pytest.importorskip("torch")
    H, I, B, T = 18, 7, 3, 6
    p = inputs.make_problem(H, I, B, T, density, cell="gru", pattern=pattern, h0="random")
    gru = torch.nn.GRU(I, H, dtype=torch.float64)
    with torch.no_grad():
        gru.weight_hh_l0.copy_(torch.from_numpy(csr_to_dense(p["rowptr"], p["col"], p["val"], 3 * H, H)))
        gru.weight_ih_l0.copy_(torch.from_numpy(p["wx"].astype(np.float64)))
        gru.bias_ih_l0.copy_(torch.from_numpy(p["bias"][:3 * H].astype(np.float64)))
        gru.bias_hh_l0.zero_()
        gru.bias_hh_l0[2 * H:].copy_(torch.from_numpy(p["bias"][3 * H:].astype(np.float64)))
        yt, hn = gru(torch.from_numpy(p["x"].astype(np.float64)), torch.from_numpy(p["h0"].astype(np.float64))[None])
    o = oracle.forward(p)
    np.testing.assert_allclose(o["y"], yt.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(o["hT"], hn[0].numpy(), rtol=1e-12, atol=1e-12)


def test_gru_zero_weights_and_saturated_update_gate():
    """Closed forms: U = W = 0, b = 0 -> r = z = 1/2, n = 0, h_t = h_0 / 2^t; a saturated update
    gate (b_z -> +inf) keeps h = h_0 for any input."""
    H, B, T = 5, 2, 4
    p = inputs.make_problem(H, 3, B, T, 0.0, cell="gru", h0="random")
    p["wx"] = np.zeros_like(p["wx"])
    p["bias"] = np.zeros_like(p["bias"])
    o = oracle.forward(p)
    for t in range(T):
        np.testing.assert_array_equal(o["y"][t], p["h0"].astype(np.float64) / 2.0 ** (t + 1))
    p["bias"][H:2 * H] = 1e4
    o = oracle.forward(p)
    np.testing.assert_array_equal(o["hT"], p["h0"].astype(np.float64))


# ------------------------------------------------------------- invariants ---

@pytest.mark.parametrize("act", ["relu", "tanh", "identity"])
def test_density0_is_activation_of_bprime(act):
    p = inputs.make_problem(32, 8, 2, 6, 0.0, act=act, h0="random")
    assert p["nnz"] == 0
    o = oracle.forward(p, act=act)
    g = {"relu": lambda u: np.maximum(u, 0), "tanh": np.tanh, "identity": lambda u: u}[act]
    if act == "tanh":  # libm vs numpy tanh may differ by 1 ulp
        np.testing.assert_allclose(o["y"], g(o["bp"]), rtol=4e-16, atol=1e-300)
    else:
        np.testing.assert_array_equal(o["y"], g(o["bp"]))


def test_linearity_identity_activation():
    H, I, B, T = 30, 7, 2, 8
    p = inputs.make_problem(H, I, B, T, 0.15, act="identity")
    rng = np.random.default_rng(3)
    u = (rng.standard_normal((B, H)), rng.standard_normal((T, B, I)))
    v = (rng.standard_normal((B, H)), rng.standard_normal((T, B, I)))
    al, be = 0.75, -1.5

    def F(h0, x):
        bp = oracle.input_projection(x, p["wx"], None)
        return oracle.rnn_forward(H, p["rowptr"], p["col"], p["val"], bp, h0, "identity")[0]

    lhs = F(al * u[0] + be * v[0], al * u[1] + be * v[1])
    rhs = al * F(*u) + be * F(*v)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-10, atol=1e-10)


def test_relu_inactive_reduces_to_identity():
    H, I, B, T = 25, 6, 2, 6
    p = inputs.make_problem(H, I, B, T, 0.2)
    p["val"] = np.abs(p["val"])
    p["wx"] = np.abs(p["wx"])
    p["x"] = np.abs(p["x"])
    p["bias"] = np.abs(p["bias"])
    a = oracle.forward(p, act="relu")["y"]
    b = oracle.forward(p, act="identity")["y"]
    np.testing.assert_array_equal(a, b)
    assert (a > 0).mean() > 0.9


@pytest.mark.parametrize("cell", ["rnn", "lstm"])
def test_permutation_equivariance(cell):
    """Relabelling hidden units permutes the outputs."""
    H, I, B, T = 21, 5, 2, 6
    p = inputs.make_problem(H, I, B, T, 0.3, cell=cell, act="tanh", h0="random", c0="random")
    G = p["G"]
    perm = np.random.default_rng(8).permutation(H)
    inv = np.argsort(perm)
    U = csr_to_dense(p["rowptr"], p["col"], p["val"], G * H, H)
    rowperm = np.concatenate([q * H + perm for q in range(G)])
    Up = U[rowperm][:, perm]
    q = dict(p)
    q["rowptr"], q["col"], q["val"] = dense_to_csr(Up)
    q["wx"] = p["wx"][rowperm]
    q["bias"] = p["bias"][rowperm]
    q["h0"] = p["h0"][:, perm]
    if cell == "lstm":
        q["c0"] = p["c0"][:, perm]
    a = oracle.forward(p)["y"]
    b = oracle.forward(q)["y"]
    np.testing.assert_allclose(b, a[:, :, perm], rtol=1e-12, atol=1e-12)
    assert inv is not None


@pytest.mark.parametrize("cell", ["rnn", "lstm"])
def test_batch_independence_bitexact(cell):
    H, I, B, T = 40, 8, 4, 7
    p = inputs.make_problem(H, I, B, T, 0.1, cell=cell, act="tanh", h0="random")
    full = oracle.forward(p)["y"]
    for b in range(B):
        q = dict(p)
        q["x"] = p["x"][:, b:b + 1]
        q["h0"] = p["h0"][b:b + 1]
        q["B"] = 1
        np.testing.assert_array_equal(oracle.forward(q)["y"][:, 0], full[:, b])


def test_T0_returns_h0_and_T1_is_one_step():
    H = 12
    p = inputs.make_problem(H, 4, 2, 1, 0.3, act="tanh", h0="random")
    bp = oracle.input_projection(p["x"], p["wx"], p["bias"])
    y, hT = oracle.rnn_forward(H, p["rowptr"], p["col"], p["val"], bp[:0], p["h0"], "tanh")
    assert y.shape[0] == 0
    np.testing.assert_array_equal(hT, p["h0"].astype(np.float64))
    y1, h1 = oracle.rnn_forward(H, p["rowptr"], p["col"], p["val"], bp, p["h0"], "tanh")
    U = csr_to_dense(p["rowptr"], p["col"], p["val"], H, H)
    np.testing.assert_allclose(h1, np.tanh(p["h0"].astype(np.float64) @ U.T + bp[0]), rtol=1e-13, atol=1e-13)


def test_brute_force_tiny_sparse_rnn():
    """Tiny case against a pure-Python scalar loop over the dense matrix."""
    H, I, B, T = 5, 3, 2, 4
    p = inputs.make_problem(H, I, B, T, 0.4, act="relu", h0="random")
    o = oracle.forward(p)
    U = csr_to_dense(p["rowptr"], p["col"], p["val"], H, H)
    Wx = p["wx"].astype(np.float64)
    for b in range(B):
        h = [float(v) for v in p["h0"][b]]
        for t in range(T):
            new = []
            for j in range(H):
                s = float(p["bias"][j])
                for i in range(I):
                    s += Wx[j, i] * float(p["x"][t, b, i])
                for k in range(H):
                    s += U[j, k] * h[k]
                new.append(max(s, 0.0))
            h = new
            np.testing.assert_allclose(o["y"][t, b], h, rtol=1e-13, atol=1e-13)


def test_integer_problem_is_exact():
    """Integer inputs: oracle result equals the exact integer recurrence."""
    H, I, B, T = 16, 6, 2, 5
    p = inputs.make_integer_problem(H, I, B, T, 0.15, act="identity")
    o = oracle.forward(p, act="identity")
    U = csr_to_dense(p["rowptr"], p["col"], p["val"], H, H).astype(np.int64)
    Wx = p["wx"].astype(np.int64)
    bias = p["bias"].astype(np.int64)
    for b in range(B):
        h = np.zeros(H, dtype=np.int64)
        for t in range(T):
            h = U @ h + Wx @ p["x"][t, b].astype(np.int64) + bias
            assert np.array_equal(o["y"][t, b], h.astype(np.float64))
