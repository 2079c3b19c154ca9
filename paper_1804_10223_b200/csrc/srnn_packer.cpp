// srnn_packer.cpp -- bank-aware packing of the pruned recurrent matrix into
// the per-lane register slots of the persistent kernel.
//
// Paper basis:
//   * <index, value> pairs, all pairs of a thread from one row.
//   * rows padded with <index, 0> pairs so every lane runs the same slot count
//     (PAPER.md:91); padding never changes the result.
//   * bank-aware order: pairs of a row may be reordered freely ("reordering
//     nonzeros' locations for each row does not affect the final result, but
//     it can change the access sequence to shared memory");
//     App. A Alg. 1 greedily places each pair in the
//     "Color" column of its bank.
//
// Re-targeted to sm_100a: the kernel stages h as [H][BT] fp32, so one pair is
// one LDS of 4*BT bytes (LDS.128 for BT = 4, the paper's ld.shared.v4 wide
// load).  Shared memory serves 128 B per wavefront, so a warp
// instruction is split into phases of P = 32/BT lanes; within a phase two
// lanes conflict iff they read different columns j, j' with j = j' (mod P),
// and lanes reading the same column broadcast.  Alg. 1's "bank" becomes the
// residue col mod P and its "Color(bank)" column becomes the lane of a phase
// group.  Unlike Alg. 1 (one row per warp), a phase group may hold several
// rows (lanes_per_row < P), so the greedy works slot by slot: each (slot,
// phase group) is filled first with pairs of pairwise-distinct residues
// (largest remaining bucket first, round-robin over the rows of the group),
// then -- only when a row would otherwise miss its slot budget -- with forced
// pairs that cost an extra wavefront.  Free lanes get padding pairs that read
// a column already read in the same phase (a broadcast, no extra wavefront).
#include "srnn_packer.h"

#include <algorithm>
#include <cstring>

namespace srnn {

uint16_t float_to_half_rne(float f) {
    uint32_t x;
    std::memcpy(&x, &f, 4);
    const uint32_t sign = (x >> 16) & 0x8000u;
    const uint32_t ax = x & 0x7fffffffu;
    if (ax >= 0x7f800000u) {  // inf or nan
        return static_cast<uint16_t>(sign | 0x7c00u | (ax > 0x7f800000u ? 0x200u | ((ax >> 13) & 0x3ffu) : 0u));
    }
    if (ax >= 0x477ff000u) return static_cast<uint16_t>(sign | 0x7c00u);  // rounds to >= 65520 -> inf
    if (ax < 0x38800000u) {                                                 // result subnormal or zero
        if (ax < 0x33000000u) return static_cast<uint16_t>(sign);           // < 2^-25: rounds to 0
        const uint32_t e = ax >> 23;
        const uint32_t m = (ax & 0x7fffffu) | 0x800000u;
        const uint32_t shift = 126 - e;  // 14 + (112 - e) ... value = m * 2^(e-150); half sub unit 2^-24
        // number of half-subnormal units: m * 2^(e - 150 + 24) = m >> (126 - e)
        uint32_t q = m >> shift;
        const uint32_t rem = m & ((1u << shift) - 1u);
        const uint32_t half = 1u << (shift - 1);
        if (rem > half || (rem == half && (q & 1u))) ++q;
        return static_cast<uint16_t>(sign | q);
    }
    // normal
    uint32_t r = ax - 0x38000000u;  // rebias exponent 127 -> 15 (in float bit layout)
    uint32_t q = r >> 13;
    const uint32_t rem = r & 0x1fffu;
    if (rem > 0x1000u || (rem == 0x1000u && (q & 1u))) ++q;
    return static_cast<uint16_t>(sign | q);
}

float half_to_float(uint16_t h) {
    const uint32_t sign = (static_cast<uint32_t>(h) & 0x8000u) << 16;
    uint32_t e = (h >> 10) & 0x1fu;
    uint32_t m = h & 0x3ffu;
    uint32_t x;
    if (e == 0) {
        if (m == 0) {
            x = sign;
        } else {  // subnormal
            e = 1;
            while ((m & 0x400u) == 0) {
                m <<= 1;
                --e;
            }
            m &= 0x3ffu;
            x = sign | ((e + 112) << 23) | (m << 13);
        }
    } else if (e == 31) {
        x = sign | 0x7f800000u | (m << 13);
    } else {
        x = sign | ((e + 112) << 23) | (m << 13);
    }
    float f;
    std::memcpy(&f, &x, 4);
    return f;
}

namespace {

inline int32_t global_row(int k, int U, int u0, int H, const int32_t* unit_of_pos) {
    const int pos = u0 + (k % U);
    return (k / U) * H + (unit_of_pos ? unit_of_pos[pos] : pos);
}

struct RowState {
    int32_t grow = -1;                       // global row
    std::vector<std::vector<int64_t>> bucket;  // per residue: CSR positions, ascending column
    std::vector<size_t> head;                // consumed prefix per bucket
    int64_t remaining = 0;
    int lane0 = 0;                           // first lane of the row in the warp
};

}  // namespace

int min_np(const PackInput& in, int L) {
    int64_t mx = 0;
    for (int r = 0; r < in.G * in.H; ++r) mx = std::max<int64_t>(mx, in.rowptr[r + 1] - in.rowptr[r]);
    if (in.piece_cap > 0) mx = std::min<int64_t>(mx, in.piece_cap);  // longer rows are split into pieces
    return static_cast<int>((mx + L - 1) / L);
}

bool pack_layout(const PackInput& in, int C, int L, int NP, Layout* out) {
    const int H = in.H, G = in.G;
    // Lanes per shared-memory phase: a wavefront serves 128 B, so an LDS of E
    // bytes per lane is split into phases of P = 128/E lanes (one phase of 32
    // lanes for E <= 4).  Conflicts are decided by key(col) mod P; equal keys
    // broadcast (E = 2: two fp16 columns share one 4-byte bank word).
    const int E = in.E;
    const int P = E >= 4 ? 128 / E : 32;
    const int ng = 32 / P;  // phase groups per warp instruction
    const int32_t* pos_of = in.pos_of_unit;  // bank model on hs positions (class balancing permutes them)
    auto key = [E, pos_of](int32_t c) {
        const int32_t q = pos_of ? pos_of[c] : c;
        return E >= 4 ? q : (q >> 1);
    };
    const int rpw = 32 / L;
    Layout& lay = *out;
    lay = Layout();
    lay.num_ctas = C;
    lay.lanes_per_row = L;
    lay.np_budget = NP;
    lay.cta_unit0.resize(C + 1);
    int umax = 0;
    for (int c = 0; c <= C; ++c)
        lay.cta_unit0[c] = in.cta_unit0 ? in.cta_unit0[c] : static_cast<int32_t>((static_cast<int64_t>(c) * H) / C);
    for (int c = 0; c < C; ++c) umax = std::max(umax, lay.cta_unit0[c + 1] - lay.cta_unit0[c]);
    // virtual rows: pieces of rows longer than piece_cap (contiguous CSR sub-ranges)
    struct VRow {
        int32_t grow;
        int64_t b, e;
    };
    auto pieces_of = [&](int64_t len) -> int64_t {
        return (in.piece_cap > 0 && len > in.piece_cap) ? (len + in.piece_cap - 1) / in.piece_cap : 1;
    };
    int vmax = 0;
    bool split = false;
    for (int c = 0; c < C; ++c) {
        const int u0 = lay.cta_unit0[c], U = lay.cta_unit0[c + 1] - u0;
        int v = 0;
        for (int k = 0; k < G * U; ++k) {
            const int32_t gr = global_row(k, U, u0, H, in.unit_of_pos);
            const int64_t np = pieces_of(in.rowptr[gr + 1] - in.rowptr[gr]);
            split |= np > 1;
            v += static_cast<int>(np);
        }
        vmax = std::max(vmax, v);
    }
    lay.vrows_max = vmax;
    const int rows_max = vmax;
    lay.warps = std::max(1, (rows_max + rpw - 1) / rpw);
    if (split) lay.piece0.assign(static_cast<size_t>(C) * (G * umax + 1), 0);
    std::vector<VRow> vrows;
    lay.threads = lay.warps * 32;
    const size_t n_img = static_cast<size_t>(C) * NP * lay.threads;
    lay.col.assign(n_img, 0);
    lay.val.assign(n_img, 0.0f);
    lay.row.assign(n_img, -1);
    lay.warp_slots.assign(static_cast<size_t>(C) * lay.warps, 0);
    const bool staged = in.early_pos > 0 && !in.naive;
    if (staged) lay.warp_early.assign(static_cast<size_t>(C) * lay.warps, 0);
    auto early = [&](int32_t c) -> bool { return (pos_of ? pos_of[c] : c) < in.early_pos; };

    std::vector<RowState> rows(rpw);
    std::vector<int32_t> gcol(P);       // column used per residue in current (slot, group); -1 none
    std::vector<std::vector<int32_t>> distinct(P);
    for (int c = 0; c < C; ++c) {
        const int u0 = lay.cta_unit0[c];
        const int U = lay.cta_unit0[c + 1] - u0;
        vrows.clear();
        for (int k = 0; k < G * U; ++k) {
            const int32_t gr = global_row(k, U, u0, H, in.unit_of_pos);
            const int64_t b0 = in.rowptr[gr], len = in.rowptr[gr + 1] - b0, np = pieces_of(len);
            if (!lay.piece0.empty()) lay.piece0[static_cast<size_t>(c) * (G * umax + 1) + k] = static_cast<int32_t>(vrows.size());
            for (int64_t j = 0; j < np; ++j) vrows.push_back({gr, b0 + (len * j) / np, b0 + (len * (j + 1)) / np});
        }
        const int n_rows = static_cast<int>(vrows.size());
        if (!lay.piece0.empty())
            for (int k = G * U; k <= G * umax; ++k) lay.piece0[static_cast<size_t>(c) * (G * umax + 1) + k] = n_rows;
        int64_t wf_cta = 0, issue_cta = 0, pairs_cta = 0, conf_cta = 0;
        for (int w = 0; w < lay.warps; ++w) {
            const int k0 = w * rpw;
            const int nr = std::max(0, std::min(rpw, n_rows - k0));
            for (int q = 0; q < rpw; ++q) {
                RowState& rs = rows[q];
                rs.grow = -1;
                rs.lane0 = q * L;
                if (q >= nr) continue;
                rs.grow = vrows[k0 + q].grow;
                const int64_t b = vrows[k0 + q].b, e = vrows[k0 + q].e;
                pairs_cta += e - b;
                if (e - b > static_cast<int64_t>(L) * NP) return false;
            }
            // stages (PackInput::early_pos): the early stage takes slots [0, n_early) with the
            // pairs of early columns only, the late stage the rest; one stage = [0, NP)
            int n_early = 0;
            if (staged) {
                int64_t mx = 0;
                for (int q = 0; q < nr; ++q) {
                    int64_t n = 0;
                    for (int64_t p = vrows[k0 + q].b; p < vrows[k0 + q].e; ++p) n += early(in.col[p]);
                    mx = std::max(mx, n);
                }
                const int a = std::max(1, in.early_align);
                n_early = (static_cast<int>((mx + L - 1) / L) + a - 1) / a * a;
                if (n_early > NP) return false;
            }
            int used_slots = 0;
            int64_t wf_warp = 0;
            std::vector<int64_t> wf_slot(NP, 0), conf_slot(NP, 0);
            for (int stage = 0; stage < (staged ? 2 : 1); ++stage) {
            const int i_lo = stage == 0 ? 0 : n_early, i_hi = staged && stage == 0 ? n_early : NP;
            for (int q = 0; q < rpw; ++q) {
                RowState& rs = rows[q];
                rs.remaining = 0;
                rs.bucket.assign(P, {});
                rs.head.assign(P, 0);
                if (q >= nr) continue;
                for (int64_t p = vrows[k0 + q].b; p < vrows[k0 + q].e; ++p) {
                    if (staged && early(in.col[p]) != (stage == 0)) continue;
                    rs.bucket[key(in.col[p]) % P].push_back(p);
                    rs.remaining++;
                }
                if (rs.remaining > static_cast<int64_t>(L) * (i_hi - i_lo)) return false;
            }
            // slot-major fill
            for (int i = i_lo; i < i_hi; ++i) {
                bool any_real = false;
                for (int g = 0; g < ng; ++g) {
                    const int gl0 = g * P, gl1 = gl0 + P;
                    std::fill(gcol.begin(), gcol.end(), -1);
                    for (int r = 0; r < P; ++r) distinct[r].clear();
                    // lanes of this group, per row
                    auto place = [&](int q, int lane, int64_t pos) {
                        const size_t at = lay.idx(c, i, w * 32 + lane);
                        lay.col[at] = in.col[pos];
                        lay.val[at] = in.val[pos];
                        lay.row[at] = rows[q].grow;
                        const int r = key(in.col[pos]) % P;
                        if (std::find(distinct[r].begin(), distinct[r].end(), key(in.col[pos])) == distinct[r].end())
                            distinct[r].push_back(key(in.col[pos]));
                        if (gcol[r] < 0) gcol[r] = in.col[pos];
                        rows[q].remaining--;
                        any_real = true;
                    };
                    std::vector<char> lane_used(P, 0);
                    if (in.naive) {
                        for (int lane = gl0; lane < gl1; ++lane) {
                            const int q = lane / L;
                            if (q >= nr) continue;
                            const int64_t k = static_cast<int64_t>(i) * L + (lane - rows[q].lane0);
                            const int64_t b = vrows[k0 + q].b, e = vrows[k0 + q].e;
                            if (b + k < e) {
                                place(q, lane, b + k);
                                lane_used[lane - gl0] = 1;
                            }
                        }
                    } else {
                        // pass 1: conflict-free, round-robin over the rows in the group
                        bool progress = true;
                        while (progress) {
                            progress = false;
                            for (int q = gl0 / L; q < nr && q * L < gl1; ++q) {
                                RowState& rs = rows[q];
                                if (rs.remaining == 0) continue;
                                int lane = -1;
                                for (int l = std::max(gl0, rs.lane0); l < std::min(gl1, rs.lane0 + L); ++l)
                                    if (!lane_used[l - gl0]) {
                                        lane = l;
                                        break;
                                    }
                                if (lane < 0) continue;
                                int best = -1;
                                size_t best_n = 0;
                                for (int r = 0; r < P; ++r) {
                                    const size_t n = rs.bucket[r].size() - rs.head[r];
                                    if (n == 0) continue;
                                    const bool free_res =
                                        gcol[r] < 0 || key(gcol[r]) == key(in.col[rs.bucket[r][rs.head[r]]]);
                                    if (free_res && n > best_n) {
                                        best = r;
                                        best_n = n;
                                    }
                                }
                                if (best < 0) continue;
                                place(q, lane, rs.bucket[best][rs.head[best]++]);
                                lane_used[lane - gl0] = 1;
                                progress = true;
                            }
                        }
                        // pass 2: forced placements for rows behind their slot budget
                        for (int q = gl0 / L; q < nr && q * L < gl1; ++q) {
                            RowState& rs = rows[q];
                            const int lanes_later_groups =
                                std::max(0, rs.lane0 + L - std::max(gl1, rs.lane0));  // lanes of q in groups > g
                            int64_t quota = rs.remaining - (static_cast<int64_t>(i_hi - i - 1) * L + lanes_later_groups);
                            for (int l = std::max(gl0, rs.lane0); l < std::min(gl1, rs.lane0 + L) && quota > 0; ++l) {
                                if (lane_used[l - gl0]) continue;
                                int best = -1;
                                size_t best_d = 0, best_n = 0;
                                for (int r = 0; r < P; ++r) {
                                    const size_t n = rs.bucket[r].size() - rs.head[r];
                                    if (n == 0) continue;
                                    const size_t d = distinct[r].size();
                                    if (best < 0 || d < best_d || (d == best_d && n > best_n)) {
                                        best = r;
                                        best_d = d;
                                        best_n = n;
                                    }
                                }
                                if (best < 0) break;
                                place(q, l, rs.bucket[best][rs.head[best]++]);
                                lane_used[l - gl0] = 1;
                                --quota;
                            }
                        }
                    }
                    // padding: broadcast a column already read in this phase
                    int32_t pad = 0;
                    for (int r = 0; r < P; ++r)
                        if (gcol[r] >= 0) {
                            pad = gcol[r];
                            break;
                        }
                    int64_t wf = 1;
                    for (int r = 0; r < P; ++r) wf = std::max<int64_t>(wf, static_cast<int64_t>(distinct[r].size()));
                    wf_slot[i] += wf;
                    conf_slot[i] += wf - 1;
                    for (int lane = gl0; lane < gl1; ++lane) {
                        if (lane_used[lane - gl0]) continue;
                        const size_t at = lay.idx(c, i, w * 32 + lane);
                        lay.col[at] = pad;
                        lay.val[at] = 0.0f;
                        const int q = lane / L;
                        lay.row[at] = q < nr ? rows[q].grow : -1;
                    }
                }
                if (any_real) used_slots = i + 1;
            }
            for (int q = 0; q < nr; ++q)
                if (rows[q].remaining != 0) return false;
            }  // stages
            if (staged) {
                used_slots = std::max(used_slots, n_early);  // the late stage starts at n_early
                lay.warp_early[static_cast<size_t>(c) * lay.warps + w] = n_early;
            }
            for (int i = 0; i < used_slots; ++i) {
                wf_warp += wf_slot[i];
                conf_cta += conf_slot[i];
            }
            lay.warp_slots[static_cast<size_t>(c) * lay.warps + w] = used_slots;
            lay.slots_used = std::max(lay.slots_used, used_slots);
            wf_cta += wf_warp;
            issue_cta += used_slots;
            lay.slots_total += static_cast<int64_t>(used_slots) * 32;
        }
        if (wf_cta > lay.wavefronts_max_cta) {
            lay.wavefronts_max_cta = wf_cta;
            lay.conflicts_max_cta = conf_cta;
        }
        lay.wavefronts_ideal_cta = std::max<int64_t>(lay.wavefronts_ideal_cta, (pairs_cta + P - 1) / P);
        lay.issue_max_cta = std::max(lay.issue_max_cta, issue_cta);
    }
    return true;
}

void class_balanced_units(const PackInput& in, int C, int classes, std::vector<int32_t>* unit_of_pos,
                          std::vector<int32_t>* pos_of_unit) {
    const int H = in.H, G = in.G;
    std::vector<int64_t> len(H, 0);
    for (int u = 0; u < H; ++u)
        for (int q = 0; q < G; ++q) len[u] += in.rowptr[q * H + u + 1] - in.rowptr[q * H + u];
    std::vector<int32_t> order(H);
    for (int u = 0; u < H; ++u) order[u] = u;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return len[a] > len[b]; });
    classes = std::max(1, std::min(classes, H));
    std::vector<int32_t> cap(C), load_units(C, 0), cls_of(H);
    std::vector<int64_t> load(C, 0);
    for (int c = 0; c < C; ++c)
        cap[c] = static_cast<int32_t>((static_cast<int64_t>(c + 1) * H) / C - (static_cast<int64_t>(c) * H) / C);
    std::vector<std::vector<int32_t>> members(C);
    for (int k = 0; k < classes; ++k) {
        const int i0 = static_cast<int>((static_cast<int64_t>(k) * H) / classes);
        const int i1 = static_cast<int>((static_cast<int64_t>(k + 1) * H) / classes);
        for (int i = i0; i < i1; ++i) {  // heaviest first: least-loaded CTA with room
            const int32_t u = order[i];
            cls_of[u] = k;
            int best = -1;
            for (int c = 0; c < C; ++c)
                if (load_units[c] < cap[c] && (best < 0 || load[c] < load[best])) best = c;
            members[best].push_back(u);
            load[best] += len[u];
            ++load_units[best];
        }
    }
    unit_of_pos->assign(H, 0);
    pos_of_unit->assign(H, 0);
    int pos = 0;
    for (int c = 0; c < C; ++c) {
        std::stable_sort(members[c].begin(), members[c].end(),
                         [&](int32_t a, int32_t b) { return cls_of[a] < cls_of[b]; });
        for (int32_t u : members[c]) {
            (*unit_of_pos)[pos] = u;
            (*pos_of_unit)[u] = pos;
            ++pos;
        }
    }
}

}  // namespace srnn
