/*
 * srnn_oracle.c -- CPU fp64 ORACLE for the sparse persistent RNN hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1804_10223_b200/, libsrnn.so) never links, loads
 * or calls anything in oracle/, and this file shares no code, header, table
 * or helper with it.
 *
 * What it computes (the plain definition the method reaches exactly, up to
 * floating-point reassociation -- PAPER.md:91 "The behavior of the network
 * does not change" under zero padding, PAPER.md:100 reordering "does not
 * affect the final result"):
 *
 *   Eq. 1 (Sec. 3.1):  h_t = g(U_r h_{t-1} + W x_t + b)
 *   Eq. 2 (Sec. 3.1):  b'_t = W x_t + b ;  h_t = g(U_r h_{t-1} + b'_t)
 *   LSTM (App. B): four gate rows per hidden unit, each with
 *         its own activation.  The paper gives no gate equations; we take the
 *         standard cell (reading R3):
 *             z = b'_t + U h_{t-1}   (4H rows, blocks [i; f; g; o])
 *             i = s(z_i) f = s(z_f) gg = tanh(z_g) o = s(z_o), s(u) = 1/(1+e^-u)
 *             c_t = f*c_{t-1} + i*gg ;  h_t = o*tanh(c_t)
 *
 * All arithmetic is IEEE double, single-threaded, plain loops, sums in
 * ascending index order (the order SPEC.md:64 fixes for its dense reference).
 * No blocking, no fusion, no reordering.  U_r is given in CSR form exactly as
 * the user passes it to srnn_load_weights (the pruned matrix).
 *
 * Parity pins (tests/test_oracle_pins.py): closed-form matrix powers for the
 * identity activation, torch.nn.RNN / torch.nn.LSTM float64 at density 1,
 * density 0, linearity, ReLU-inactive reduction, permutation equivariance,
 * batch independence, a hand-derived dyadic example and SPEC.md's worked
 * examples (tests/golden/).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define ORACLE_ACT_RELU 0
#define ORACLE_ACT_TANH 1
#define ORACLE_ACT_IDENTITY 2

/* g: the elementwise activation of Eq. 1 ("g is an elementwise
 * activation function"; which g the paper's benchmarks use is unstated,
 * DESIGN.md reading R1). */
static double oracle_g(int act, double u) {
    switch (act) {
    case ORACLE_ACT_RELU: return u > 0.0 ? u : 0.0;
    case ORACLE_ACT_TANH: return tanh(u);
    default: return u;
    }
}

static double oracle_sigmoid(double u) { return 1.0 / (1.0 + exp(-u)); }

/*
 * Input projection, Eq. 2: "The input-to-hidden weight matrix
 * (W x_t) calculation has no dependency, so it can be processed in parallel
 * and added to b, becoming b'".
 *   bp[m][r] = bias[r] + sum_{i ascending} Wx[r][i] * x[m][i]
 * x:  [M][I]  (M = T*B rows, row m = t*B + b)
 * Wx: [R][I]  row-major (R = G*H)
 * bp: [M][R]
 */
void oracle_input_projection(int64_t M, int32_t I, int32_t R, const double *x,
                             const double *Wx, const double *bias, double *bp) {
    for (int64_t m = 0; m < M; ++m) {
        for (int32_t r = 0; r < R; ++r) {
            double s = 0.0;
            for (int32_t i = 0; i < I; ++i) s += Wx[(int64_t)r * I + i] * x[m * I + i];
            bp[m * R + r] = s + (bias ? bias[r] : 0.0);
        }
    }
}

/*
 * Sparse recurrent product z[r] = sum_{k in nz(r), ascending} U[r][k] h[k]
 * (the "operate" stage's result: acc += value[i]*activation[index[i]]).
 */
static void oracle_spmv(int32_t R, const int64_t *rowptr, const int32_t *col,
                        const double *val, const double *h, double *z) {
    for (int32_t r = 0; r < R; ++r) {
        double s = 0.0;
        for (int64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) s += val[p] * h[col[p]];
        z[r] = s;
    }
}

/*
 * Vanilla RNN over T steps, Eq. 2.
 *   bp:  [T][B][H]  precomputed b' (oracle_input_projection)
 *   h0:  [B][H] or NULL (= 0, reading R4)
 *   y:   [T][B][H]  y[t] = h_{t+1}
 *   hT:  [B][H] or NULL; T == 0 copies h0
 *   work: scratch of 2*H doubles
 */
void oracle_rnn_forward(int32_t H, int32_t B, int32_t T, const int64_t *rowptr,
                        const int32_t *col, const double *val, const double *bp,
                        const double *h0, int32_t act, double *y, double *hT,
                        double *work) {
    double *h = work, *z = work + H;
    for (int32_t b = 0; b < B; ++b) {
        for (int32_t j = 0; j < H; ++j) h[j] = h0 ? h0[(int64_t)b * H + j] : 0.0;
        for (int32_t t = 0; t < T; ++t) {
            oracle_spmv(H, rowptr, col, val, h, z);
            const double *bpt = bp + ((int64_t)t * B + b) * H;
            for (int32_t j = 0; j < H; ++j) h[j] = oracle_g(act, z[j] + bpt[j]);
            if (y) memcpy(y + ((int64_t)t * B + b) * H, h, sizeof(double) * (size_t)H);
        }
        if (hT) memcpy(hT + (int64_t)b * H, h, sizeof(double) * (size_t)H);
    }
}

/*
 * LSTM over T steps (App. B; gate equations: DESIGN.md R3).
 *   U (CSR) has 4H rows: gate blocks [i; f; g; o], row q*H + j = gate q of unit j.
 *   bp: [T][B][4H]; h0, c0: [B][H] or NULL; y: [T][B][H]; hT, cT: [B][H] or NULL
 *   work: scratch of 2*H + 4*H doubles
 */
void oracle_lstm_forward(int32_t H, int32_t B, int32_t T, const int64_t *rowptr,
                         const int32_t *col, const double *val, const double *bp,
                         const double *h0, const double *c0, double *y, double *hT,
                         double *cT, double *work) {
    double *h = work, *c = work + H, *z = work + 2 * (int64_t)H;
    for (int32_t b = 0; b < B; ++b) {
        for (int32_t j = 0; j < H; ++j) {
            h[j] = h0 ? h0[(int64_t)b * H + j] : 0.0;
            c[j] = c0 ? c0[(int64_t)b * H + j] : 0.0;
        }
        for (int32_t t = 0; t < T; ++t) {
            oracle_spmv(4 * H, rowptr, col, val, h, z);
            const double *bpt = bp + ((int64_t)t * B + b) * 4 * H;
            for (int32_t j = 0; j < H; ++j) {
                double zi = z[j] + bpt[j];
                double zf = z[H + j] + bpt[H + j];
                double zg = z[2 * H + j] + bpt[2 * H + j];
                double zo = z[3 * H + j] + bpt[3 * H + j];
                double ig = oracle_sigmoid(zi), fg = oracle_sigmoid(zf);
                double gg = tanh(zg), og = oracle_sigmoid(zo);
                c[j] = fg * c[j] + ig * gg;
                h[j] = og * tanh(c[j]);
            }
            if (y) memcpy(y + ((int64_t)t * B + b) * H, h, sizeof(double) * (size_t)H);
        }
        if (hT) memcpy(hT + (int64_t)b * H, h, sizeof(double) * (size_t)H);
        if (cT) memcpy(cT + (int64_t)b * H, c, sizeof(double) * (size_t)H);
    }
}

/*
 * GRU over T steps (SURVEY.md Sec. 8(f)4 cell extension; not in the paper --
 * DESIGN.md reading R15: the "reset gate after the product" form of cuDNN /
 * torch.nn.GRU, so each step needs one sparse product of h_{t-1}):
 *   U (CSR) has 3H rows: gate blocks [r; z; n], row q*H + j = gate q of unit j.
 *   bp: [T][B][3H] = W x_t + b (b_r, b_z already include the recurrent biases)
 *   bhn: [H] recurrent bias of the n gate (inside r * (.)), or NULL (= 0)
 *     r = sigma(U_r h + bp_r)     z = sigma(U_z h + bp_z)
 *     n = tanh(bp_n + r * (U_n h + bhn))      h' = (1 - z) * n + z * h
 *   h0: [B][H] or NULL; y: [T][B][H]; hT: [B][H] or NULL
 *   work: scratch of H + 3*H doubles
 */
void oracle_gru_forward(int32_t H, int32_t B, int32_t T, const int64_t *rowptr,
                        const int32_t *col, const double *val, const double *bp,
                        const double *bhn, const double *h0, double *y, double *hT,
                        double *work) {
    double *h = work, *z = work + H;
    for (int32_t b = 0; b < B; ++b) {
        for (int32_t j = 0; j < H; ++j) h[j] = h0 ? h0[(int64_t)b * H + j] : 0.0;
        for (int32_t t = 0; t < T; ++t) {
            oracle_spmv(3 * H, rowptr, col, val, h, z);
            const double *bpt = bp + ((int64_t)t * B + b) * 3 * H;
            for (int32_t j = 0; j < H; ++j) {
                double r = oracle_sigmoid(z[j] + bpt[j]);
                double u = oracle_sigmoid(z[H + j] + bpt[H + j]);
                double n = tanh(bpt[2 * H + j] + r * (z[2 * H + j] + (bhn ? bhn[j] : 0.0)));
                h[j] = (1.0 - u) * n + u * h[j];
            }
            if (y) memcpy(y + ((int64_t)t * B + b) * H, h, sizeof(double) * (size_t)H);
        }
        if (hT) memcpy(hT + (int64_t)b * H, h, sizeof(double) * (size_t)H);
    }
}
