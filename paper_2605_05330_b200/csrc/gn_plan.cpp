// gn_plan.cpp -- host construction of the loop kernel's static work plan
// (see gn_plan.h for the scheme).
#include "gn_plan.h"

#include <algorithm>
#include <functional>
#include <queue>
#include <utility>

namespace gn {

namespace {

// Cost unit: one gather per lane.  kFixed stands for the per-item round
// trips (item descriptor, degrees, row state, the store).
constexpr double kFixed = 24.0;

struct Unit {
    int kind;  // 0 short slice, 1 long slice, 2 hub row, 3 EXACT hub group
    int32_t id;
    double cost;
};

using Slot = std::pair<double, int>;
using MinHeap = std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>>;

int hub_piece_elems(int32_t deg) { return std::max(kHubPieceElems, (deg + 255) / 256); }

}  // namespace

void build_plan(const PlanInput& in, int G, bool exact, size_t cap, HostPlan& out) {
    const auto& sp = *in.slice_ptr;
    const auto& hp = *in.hub_ptr;
    const int B = in.B;
    auto nblk = [&](int s) { return (int32_t)((sp[(size_t)s + 1] - sp[(size_t)s]) / (32 * B)); };
    auto hdeg = [&](int h) { return hp[(size_t)h + 1] - hp[(size_t)h]; };

    // ---- units and their costs
    std::vector<Unit> units;
    if (exact) {
        for (int h = 0; h < in.nhub; h += 32) {
            int32_t mx = 0;
            for (int q = h; q < std::min(in.nhub, h + 32); ++q) mx = std::max(mx, hdeg(q));
            units.push_back({3, h, kFixed + mx});
        }
        for (int s = 0; s < in.nslices; ++s) units.push_back({0, s, kFixed + (double)nblk(s) * B});
    } else {
        for (int h = 0; h < in.nhub; ++h) {
            const int pe = hub_piece_elems(hdeg(h));
            const int np = (hdeg(h) + pe - 1) / pe;
            units.push_back({2, h, np * (kFixed + pe / 32.0)});
        }
        for (int s = 0; s < in.nsplit; ++s) {
            const int np = (nblk(s) + kPieceBlocks - 1) / kPieceBlocks;
            units.push_back({1, s, np * kFixed + (double)nblk(s) * B});
        }
        for (int s = in.nsplit; s < in.nslices; ++s) units.push_back({0, s, kFixed + (double)nblk(s) * B});
    }

    // ---- level 1: units -> CTAs, longest-processing-time-first on total
    // cost.  With `colocate` (the uint16-id graphs) the slices are instead
    // taken in signature order as contiguous runs filling each CTA to the mean
    // (neighbourhood-sharing slices on one SM, whose L1 then serves them).
    std::vector<std::vector<Unit>> per_cta((size_t)G);
    std::vector<double> load((size_t)G, 0.0);
    double total = 0.0;
    for (const Unit& u : units) total += u.cost;
    const double target = total / G;
    std::vector<Unit> big, small;
    for (const Unit& u : units) (!in.colocate || u.kind == 2 || u.kind == 3 ? big : small).push_back(u);
    std::stable_sort(big.begin(), big.end(), [](const Unit& a, const Unit& b) { return a.cost > b.cost; });
    {
        MinHeap pq;
        for (int b = 0; b < G; ++b) pq.push({0.0, b});
        for (const Unit& u : big) {
            Slot e = pq.top();
            pq.pop();
            per_cta[(size_t)e.second].push_back(u);
            e.first += u.cost;
            load[(size_t)e.second] = e.first;
            pq.push(e);
        }
    }
    if (!small.empty()) {
        const auto& sig = *in.sig;
        if (!sig.empty())
            std::stable_sort(small.begin(), small.end(), [&](const Unit& a, const Unit& b) {
                return sig[(size_t)a.id] != sig[(size_t)b.id] ? sig[(size_t)a.id] < sig[(size_t)b.id] : a.id < b.id;
            });
        size_t i = 0;
        for (int b = 0; b < G && i < small.size(); ++b)
            while (i < small.size() && load[(size_t)b] + small[i].cost * 0.5 <= target) {
                per_cta[(size_t)b].push_back(small[i]);
                load[(size_t)b] += small[i].cost;
                ++i;
            }
        for (; i < small.size(); ++i) {
            int b = (int)(std::min_element(load.begin(), load.end()) - load.begin());
            per_cta[(size_t)b].push_back(small[i]);
            load[(size_t)b] += small[i].cost;
        }
    }

    // ---- level 2: per CTA, phases of pieces (+ the short slices in phase 0)
    out = HostPlan();
    out.phase_base.assign((size_t)G + 1, 0);
    out.phase_comb.push_back(0);
    out.smem_words.assign((size_t)G, 0);
    const size_t cap_words = cap / 16;
    for (int b = 0; b < G; ++b) {
        out.phase_base[(size_t)b] = (int32_t)(out.phase_comb.size() - 1);
        std::vector<Unit>& cu = per_cta[(size_t)b];
        std::vector<Item> whole;
        struct Phase {
            std::vector<Item> items;
            std::vector<Combine> combs;
            int slots = 0, hslots = 0;
        };
        std::vector<Phase> phases(1);
        int cta_pieces = 0;
        for (const Unit& u : cu)
            if (u.kind == 1) cta_pieces += (nblk(u.id) + kPieceBlocks - 1) / kPieceBlocks;
        const int slot_cap = cta_pieces <= kMaxSlots ? kMaxSlots : kPhaseSlots;
        for (const Unit& u : cu) {
            if (u.kind == 0) {
                whole.push_back(Item{kWhole, u.id, 0, nblk(u.id), -1, -1, 0, 0});
            } else if (u.kind == 3) {
                whole.push_back(Item{kHubSeq, u.id, 0, std::min(32, in.nhub - u.id), -1, -1, 0, 0});
            } else if (u.kind == 1) {
                const int nb = nblk(u.id);
                const int np = (nb + kPieceBlocks - 1) / kPieceBlocks;
                if (phases.back().slots + np > slot_cap && phases.back().slots > 0) phases.emplace_back();
                Phase& ph = phases.back();
                ph.combs.push_back(Combine{0, u.id, ph.slots, np});
                for (int q = 0; q < np; ++q)
                    ph.items.push_back(Item{kPiece, u.id, q * kPieceBlocks, std::min(nb, (q + 1) * kPieceBlocks),
                                            ph.slots + q, -1, 0, 0});
                ph.slots += np;
            } else {
                const int32_t deg = hdeg(u.id);
                const int pe = hub_piece_elems(deg);
                const int np = std::max(1, (deg + pe - 1) / pe);
                if (phases.back().hslots + np > kMaxHubSlots && phases.back().hslots > 0) phases.emplace_back();
                Phase& ph = phases.back();
                ph.combs.push_back(Combine{1, u.id, ph.hslots, np});
                for (int q = 0; q < np; ++q)
                    ph.items.push_back(Item{kHubPiece, u.id, q * pe, std::min(deg, (q + 1) * pe), ph.hslots + q, -1, 0, 0});
                ph.hslots += np;
            }
        }
        phases[0].items.insert(phases[0].items.end(), whole.begin(), whole.end());
        // deal each phase's items to the 32 warps, LPT
        auto icost = [&](const Item& it) {
            switch (it.kind) {
                case kWhole:
                case kPiece: return kFixed + (double)(it.end - it.beg) * B;
                case kHubPiece: return kFixed + (it.end - it.beg) / 32.0;
                default: {
                    int32_t mx = 0;
                    for (int q = it.id; q < it.id + (it.end - it.beg); ++q) mx = std::max(mx, hdeg(q));
                    return kFixed + mx;
                }
            }
        };
        size_t used = 0;
        for (Phase& ph : phases) {
            std::stable_sort(ph.items.begin(), ph.items.end(),
                             [&](const Item& x, const Item& y) { return icost(x) > icost(y); });
            std::vector<std::vector<Item>> wl(kWarps);
            MinHeap pq;
            for (int w = 0; w < kWarps; ++w) pq.push({0.0, w});
            for (const Item& it : ph.items) {
                Slot e = pq.top();
                pq.pop();
                wl[(size_t)e.second].push_back(it);
                e.first += icost(it);
                pq.push(e);
            }
            for (auto& v : wl)
                std::sort(v.begin(), v.end(), [](const Item& x, const Item& y) {
                    return x.kind != y.kind ? x.kind < y.kind : (x.id != y.id ? x.id < y.id : x.beg < y.beg);
                });
            // residency: breadth-first over the warps so every warp gets some
            for (size_t depth = 0;; ++depth) {
                bool any = false;
                for (int w = 0; w < kWarps; ++w) {
                    if (depth >= wl[(size_t)w].size()) continue;
                    any = true;
                    Item& it = wl[(size_t)w][depth];
                    if (it.kind != kWhole && it.kind != kPiece) continue;
                    const size_t words = (size_t)(it.end - it.beg) * 32;
                    if (used + words <= cap_words) {
                        it.smem = (int32_t)used;
                        used += words;
                    }
                }
                if (!any) break;
            }
            for (int w = 0; w < kWarps; ++w) {
                out.phase_warp.push_back((int32_t)out.items.size());
                for (Item it : wl[(size_t)w]) {
                    if (it.kind == kWhole || it.kind == kPiece) {
                        // 16-byte-word offset of block `beg`: slice start (elements) * elem size / 16 + 32 per block
                        const int64_t words = sp[(size_t)it.id] / B + (int64_t)it.beg * 32;
                        it.pad0 = (int32_t)(uint32_t)(words & 0xffffffffll);
                        it.pad1 = (int32_t)(uint32_t)(words >> 32);
                    }
                    out.items.push_back(it);
                }
            }
            out.phase_warp.push_back((int32_t)out.items.size());
            out.combs.insert(out.combs.end(), ph.combs.begin(), ph.combs.end());
            out.phase_comb.push_back((int32_t)out.combs.size());
            out.max_slots = std::max(out.max_slots, ph.slots);
            out.max_hub_slots = std::max(out.max_hub_slots, ph.hslots);
        }
        out.smem_words[(size_t)b] = (int32_t)used;
        out.resident_words += (int64_t)used;
    }
    out.phase_base[(size_t)G] = (int32_t)(out.phase_comb.size() - 1);
}

}  // namespace gn
