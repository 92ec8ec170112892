// gn_plan.h -- the static work plan of the persistent loop kernel.
//
// The kernel runs the same work every iteration, so who does what is decided
// once per (graph, grid, mode) on the host and cached with the graph:
//
//   level 1  every unit (short slice, long slice, hub row) goes to a CTA,
//            longest-processing-time-first on its total gather count: a
//            CTA's warps share one SM's L1/LSU, the resource gathers
//            saturate, so CTAs (not warps) are what must be balanced;
//   level 2  inside a CTA, long slices and hub rows are cut into fixed-size
//            pieces (8 blocks of a slice, <= 1024 elements of a hub row:
//            independent of the grid, so the summation tree -- and every bit
//            of the result -- is the same on any device), and pieces plus
//            short slices are dealt to the CTA's 32 warps, again LPT;
//   phases   pieces write per-piece partial sums to shared-memory slots; a
//            CTA's pieces are grouped into phases whose slots fit the slot
//            budget; after a phase's __syncthreads the combines (one per long
//            slice / hub row) fold the slots in piece order and update rows;
//   residency the index blocks of as many pieces / short slices as fit a
//            shared-memory budget are copied on chip once per run.
#pragma once

#include <stdint.h>

#include <vector>

namespace gn {

#ifndef GN_LOOP_CTAS_PER_SM
#define GN_LOOP_CTAS_PER_SM 1
#endif
#ifndef GN_LOOP_THREADS
#define GN_LOOP_THREADS 512
#endif
constexpr int kThreads = GN_LOOP_THREADS;  // per CTA; one CTA per SM -> 128 registers per thread for deep gather batches
constexpr int kCtasPerSm = GN_LOOP_CTAS_PER_SM;
constexpr int kWarps = kThreads / 32;
constexpr int kPieceBlocks = 8;      // blocks per piece of a long slice
constexpr int kHubPieceElems = 1024; // elements per piece of a hub row (at least)
// slice-piece slots per phase (32 partials each): a CTA whose pieces fit in
// kMaxSlots runs them in one phase; one with more uses phases of
// kPhaseSlots -- smaller phases leave more of the SM's memory to L1 (C5 scale
// 24: 2.14 -> 1.86 ms/iteration), one phase saves a barrier (C2: 20.3 -> 18.8 us)
constexpr int kMaxSlots = 128;
constexpr int kPhaseSlots = 64;
constexpr int kMaxHubSlots = 512;    // hub-piece slots per phase (1 partial each)

enum ItemKind : int32_t { kWhole = 0, kPiece = 1, kHubPiece = 2, kHubSeq = 3 };

// kWhole:    id = slice, [beg, end) = blocks [0, nblk)
// kPiece:    id = slice, [beg, end) = blocks of the piece, slot = slice slot
// kHubPiece: id = hub row, [beg, end) = element offsets in the row, slot = hub slot
// kHubSeq:   id = first hub row, end - beg = rows (EXACT mode, one thread per row)
// smem: 16-byte-word offset of the resident copy of blocks [beg, end), -1 = global;
// pad0/pad1: low/high 32 bits of the 16-byte-word offset of block beg in the global index array
struct Item {
    int32_t kind, id, beg, end, slot, smem, pad0, pad1;
};

// kind 0: long slice id, its 32 rows; kind 1: hub row id.  Slots
// [slot, slot + nslot) in piece order.
struct Combine {
    int32_t kind, id, slot, nslot;
};

struct HostPlan {
    std::vector<int32_t> phase_base;  // [G+1] into phases
    std::vector<int32_t> phase_warp;  // [P*(kWarps+1)] item ranges per warp of each phase
    std::vector<int32_t> phase_comb;  // [P+1] into combs
    std::vector<Item> items;
    std::vector<Combine> combs;
    std::vector<int32_t> smem_words;  // [G] resident words per CTA
    int max_slots = 0, max_hub_slots = 0;
    int64_t resident_words = 0;
};

struct PlanInput {
    int64_t n;
    int32_t nhub, nslices, nsplit;
    int B;                              // positions per block (8 or 4)
    const std::vector<int64_t>* slice_ptr;
    const std::vector<int32_t>* hub_ptr;
    const std::vector<uint64_t>* sig;   // per-slice neighbourhood signature (may be empty)
    bool colocate;                      // level 1 by signature runs instead of LPT
};

void build_plan(const PlanInput& in, int G, bool exact, size_t resident_cap_bytes, HostPlan& out);

}  // namespace gn
