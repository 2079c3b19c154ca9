// srnn_packer.h -- host-side planner + packer of the sparse weight image
// (SURVEY.md Sec. 8 a2, a10).  Pure C++, no CUDA; unit-tested on the CPU
// through srnn_plan_export_layout.
#pragma once
#include <cstdint>
#include <vector>

namespace srnn {

struct PackInput {
    int32_t H = 0, G = 1;
    const int32_t* rowptr = nullptr;  // [G*H+1]
    const int32_t* col = nullptr;     // [nnz]
    const float* val = nullptr;       // [nnz] (already fp16-rounded in fp16 mode)
    int32_t BT = 4;                   // batch tile (samples per staged h row)
    int32_t E = 16;                   // bytes per staged h row (4*BT fp32, 2*BT fp16): one LDS per pair
    bool naive = false;               // CSR-order lane-strided layout (PAPER.md:91 baseline)
    // Unit permutation (class-based load balancing): exchange/hs position i holds
    // unit unit_of_pos[i]; CTA c owns positions [cta_unit0[c], cta_unit0[c+1]).  nullptr = identity.
    const int32_t* unit_of_pos = nullptr;
    const int32_t* pos_of_unit = nullptr;  // inverse (column -> hs position)
    // Rows longer than piece_cap nonzeros are split into near-equal pieces ("virtual rows")
    // packed like rows; the epilogue sums a row's pieces (class-based balancing of heavy
    // rows).  0 = never split.
    int32_t piece_cap = 0;
    // Explicit unit ranges per CTA ([C+1], CTA c owns units [cta_unit0[c], cta_unit0[c+1])); nullptr =
    // the even split c*H/C.  The column split (SRNN_FLAG_COLUMN_SPLIT) packs a virtual matrix whose
    // units are (cluster unit, column half) and needs both CTAs of a pair to own equally many.
    const int32_t* cta_unit0 = nullptr;
    // Partial progress ("the load stage can make partial progress as values are
    // marked complete, allowing the operate stage to proceed before all values are finished"):
    // > 0 = every warp's slots are ordered in two stages, first all pairs whose column sits at an
    // hs position < early_pos (the exchange chunks the loaders fetch first), then the rest, so the
    // kernel can operate on the early stage while the late chunks are still in flight.  The
    // stage boundary is warp-uniform (Layout::warp_early).  0 = one stage.
    int32_t early_pos = 0;
    int32_t early_align = 1;  // the early stage's slot count is rounded up to this (operate group)
};

// Class-based assignment of units to CTAs ("define a number of classes for
// different amounts of sparsity and handle each class separately, assigning each row to one
// class or another based on its sparsity"): units are bucketed into `classes` quantile classes
// of their nonzero count (all G gate rows), every class is dealt over the C CTAs heaviest-first
// to the least-loaded CTA with room (equal unit counts per CTA as before), and inside a CTA
// units are ordered by class so a warp's rows have similar lengths.  Writes unit_of_pos /
// pos_of_unit (size H).
void class_balanced_units(const PackInput& in, int C, int classes, std::vector<int32_t>* unit_of_pos,
                          std::vector<int32_t>* pos_of_unit);

struct Layout {
    int32_t num_ctas = 0, lanes_per_row = 0, threads = 0, warps = 0;
    int32_t np_budget = 0;   // slot budget the greedy packed against
    int32_t slots_used = 0;  // max over warps of used slots
    std::vector<int32_t> cta_unit0;   // [num_ctas+1]
    std::vector<int32_t> warp_slots;  // [num_ctas*warps]
    std::vector<int32_t> warp_early;  // [num_ctas*warps] slots of the early stage (PackInput::early_pos), or empty
    // per (cta, slot < np_budget, thread): column, value, owning global row (-1 idle)
    std::vector<int32_t> col;
    std::vector<float> val;
    std::vector<int32_t> row;
    int64_t wavefronts_max_cta = 0;    // predicted smem wavefronts per tile-step, busiest CTA
    int64_t wavefronts_ideal_cta = 0;  // ceil(pairs/32 lanes)*(32/P)-style ideal for that CTA
    int64_t conflicts_max_cta = 0;     // sum over (slot, phase) of (wavefronts - 1) in that CTA
    int64_t issue_max_cta = 0;         // warp-slot instructions of the busiest CTA
    int64_t slots_total = 0;
    // pieces (PackInput::piece_cap): per CTA the first virtual row of each local row k
    // (k = gate * U + unit, G*units_max + 1 entries per CTA, prefix sums); empty = no split
    std::vector<int32_t> piece0;
    int32_t vrows_max = 0;  // virtual rows of the largest CTA (= G * units when nothing splits)
    size_t idx(int c, int i, int t) const {
        return (static_cast<size_t>(c) * np_budget + i) * threads + t;
    }
};

// Pack for a fixed CTA count, lanes per row and slot budget.  Returns false if
// some row does not fit in lanes_per_row * np_budget slots.
bool pack_layout(const PackInput& in, int num_ctas, int lanes_per_row, int np_budget, Layout* out);

// Smallest budget a row needs: max_r ceil(len_r / L).
int min_np(const PackInput& in, int lanes_per_row);

// IEEE binary16 round-to-nearest-even of a float (as numpy astype(float16)).
uint16_t float_to_half_rne(float f);
float half_to_float(uint16_t h);

}  // namespace srnn
