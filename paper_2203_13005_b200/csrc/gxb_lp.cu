// gxb_lp.cu — LabelPropagation mode reduction (K3).
//
// Semantics (A/algorithms.py:174-205, run_reference 318-341): a destination's
// multiset is the labels of its ACTIVE in-neighbours, one per edge (duplicates
// and self-loops count); no message -> keep the label and go inactive;
// otherwise take the most frequent label, ties to the smallest label, and be
// active iff it changed. Counts are exact integers, so the result is bit-exact.
//
// Dense rounds, over the in-degree-sorted slots:
//  * in-degree <= 32 (k_lp_pull): G lanes per destination stage its labels in shared
//    memory and count each candidate against the staged multiset;
//  * 33-512 (k_lp_hub_warp) and 513-4096 (k_lp_hub_cta, half a CTA up to 2048:
//    k_lp_hub_cta2): a warp / CTA counts the destination in a shared (label, count) table
//    twice its in-degree, after equal labels of 32 edges are merged with __match_any_sync;
//  * above 4096 (k_lp_chunks): warps stream 1024-edge chunks into per-warp shared tables
//    and flush them into per-hub epoch-tagged global tables (L2 atomics); the packed
//    argmax (count << 32 | ~label) is raised once per chunk, k_lp_hub_apply applies it.
// Round 1 (labels = distinct ids) counts every hub by run length over its sorted sources
// (k_lp_chunks_runs, and k_lp_hub_warp's run-length branch). Sparse rounds push the
// frontier's labels into a (destination, label) pair table (k_lp_push).
#include <algorithm>
#include <vector>

#include "gxb_state.cuh"

namespace gxb {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;

// Global (label, count) tables of the label-diverse hubs (in-degree > kLpBigDeg), one per
// hub, 2 x in-degree entries. One 64-bit word per entry: epoch (8 bits) | count (24 bits) |
// label (32 bits). A word of another epoch is empty, so no table is cleared between rounds
// (every 255 rounds the tables are zeroed once); an insert is a read plus one CAS (new
// label) or one atomicAdd on the count field (known label).
struct LpHub {
    uint64_t* tab_off;   // per big hub: first entry
    uint32_t* tab_mask;  // per big hub: size - 1 (power of two)
    unsigned long long* words;
    unsigned long long* best;  // per chunked slot: packed (count << 32 | ~label), 0 = no message
    uint64_t entries;
    uint32_t epoch;      // 1..255
};

struct LpPush;
struct LpScratch {
    LpHub hub;
    uint64_t chunk_end = 0;
    uint64_t big_end = 0;  // relative slots [0, big_end): in-degree > kLpBigDeg (chunked warps)
    uint64_t big_items = 0;    // their chunk items (the plan's first items)
    uint64_t cta_end = 0;  // relative slots [big_end, cta_end): in-degree > kLpCtaMinDeg (one CTA each)
    uint64_t cta_half = 0;  // [cta_half, cta_end): in-degree <= kLpCtaHalfDeg (half a CTA each)
    uint32_t* eff = nullptr;  // per slot: label if active, else kEmpty (rounds >= 2)
    uint32_t hot_end = 0;  // slots with in-degree >= kLpHotDegree: pushed through shared memory
    // sparse rounds (allocated on the first one)
    unsigned long long* pkeys = nullptr;
    uint32_t* pcounts = nullptr;
    unsigned long long* pbest = nullptr;
    uint32_t* ptargets = nullptr;
    unsigned long long* pntargets = nullptr;
    uint64_t pcapacity = 0;
};

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// fold (label, c) into a hub's epoch-tagged table; returns the label's new count
__device__ __forceinline__ uint32_t table_add(const LpHub& H, uint64_t base, uint32_t mask, uint32_t label,
                                              uint32_t c) {
    const unsigned long long ep = (unsigned long long)H.epoch << 56;
    uint32_t i = mix32(label) & mask;
    while (true) {
        unsigned long long* wp = H.words + base + i;
        unsigned long long w = __ldcg(wp);
        if ((uint32_t)(w >> 56) != H.epoch) {  // empty in this round: claim it
            const unsigned long long nw = ep | ((unsigned long long)c << 32) | label;
            const unsigned long long prev = atomicCAS(wp, w, nw);
            if (prev == w) return c;
            w = prev;
            if ((uint32_t)(w >> 56) != H.epoch) continue;  // raced with another stale word: retry the slot
        }
        if ((uint32_t)w == label) {
            const unsigned long long old = atomicAdd(wp, (unsigned long long)c << 32);
            return (uint32_t)((old >> 32) & 0xFFFFFFull) + c;
        }
        i = (i + 1) & mask;
    }
}

struct LpLaunch {
    uint64_t lo;
    const uint64_t* in_off;
    const uint32_t* in_src;
    const uint32_t* lab_cur;
    uint32_t* lab_next;
    const uint32_t* active_cur;
    FrontierView f;
    StatStripe* stats;
    // chunk items
    uint64_t num_items;
    const uint32_t* item_slot;
    const uint64_t* item_begin;
    unsigned chunk_blocks;
    uint64_t bin_lo[kNumGroupBins], bin_hi[kNumGroupBins];
    unsigned bin_blocks[kNumGroupBins];
    LpHub hub;
    bool injective;  // labels are distinct (round 1): hub counts are edge multiplicities
    // label of every ACTIVE source slot, kEmpty for inactive ones (k_lp_eff, rounds >= 2):
    // one gather per edge instead of an active-bitmap test plus a label gather
    const uint32_t* eff;
};

// the label a source contributes to its out-neighbours' multisets, or kEmpty
__device__ __forceinline__ uint32_t lp_msg(const LpLaunch& L, uint32_t s) {
    if (L.eff) return __ldg(L.eff + s);
    return bit_test(L.active_cur, s) ? __ldg(L.lab_cur + s) : kEmpty;
}

__device__ __forceinline__ void lp_finish(const LpLaunch& L, uint32_t slot, unsigned long long best, LocalStats& st) {
    if (best == 0ull) return;  // no message: keep label, inactive (A/algorithms.py:195-196)
    st.targets++;
    const uint32_t nl = ~(uint32_t)(best & 0xFFFFFFFFull);
    const uint32_t old = L.lab_cur[slot];
    if (nl != old) {
        L.lab_next[slot] = nl;
        publish_changed(L.f, slot, st);
    }
}

// lp_finish for a whole warp, each lane with its own (slot, best) or none: the changed
// slots are published with one frontier reservation for the warp (a reservation per
// destination on the single frontier counter serialises in L2 at ~10^5 destinations)
__device__ __forceinline__ void lp_finish_lanes(const LpLaunch& L, bool valid, uint32_t slot, unsigned long long best,
                                                LocalStats& st) {
    bool ch = false;
    if (valid && best != 0ull) {
        st.targets++;
        const uint32_t nl = ~(uint32_t)(best & 0xFFFFFFFFull);
        if (nl != L.lab_cur[slot]) {
            L.lab_next[slot] = nl;
            ch = true;
            st.changed++;
            st.next_active++;
            st.next_units += __ldg(L.f.outdeg + slot);
            if (bit_test(L.f.remote_src, slot)) st.remote_active++;
            atomicOr(L.f.active_next + (slot >> 5), 1u << (slot & 31));
        }
    }
    const unsigned m = __ballot_sync(kFull, ch);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(L.f.frontier_count, (unsigned long long)__popc(m));
    base = __shfl_sync(kFull, base, __ffs(m) - 1);
    if (ch) L.f.frontier_next[base + __popc(m & ((1u << lane) - 1u))] = slot;
}

// small destinations: stage labels in shared memory, count candidates
template <int G>
__device__ __forceinline__ void lp_group(const LpLaunch& L, int k, unsigned b, uint32_t* buf, LocalStats& st) {
    constexpr int kPerBlock = kBlock / G;
    constexpr int kCap = 4 * G;  // max in-degree of this bin
    const int grp = threadIdx.x / G;
    const int gl = threadIdx.x % G;
    const uint64_t rel = L.bin_lo[k] + (uint64_t)b * kPerBlock + grp;
    const bool valid = rel < L.bin_hi[k];
    uint32_t deg = 0;
    uint64_t beg = 0;
    if (valid) {
        beg = __ldg(L.in_off + rel);
        deg = (uint32_t)(__ldg(L.in_off + rel + 1) - beg);
    }
    uint32_t* my = buf + grp * kCap;  // 16-B aligned: kCap is a multiple of 4
    const uint32_t deg4 = (deg + 3u) & ~3u;
    for (uint32_t i = gl; i < deg4; i += G) {  // padded with kEmpty, which is never a candidate
        my[i] = i < deg ? lp_msg(L, __ldg(L.in_src + beg + i)) : kEmpty;
    }
    __syncwarp();
    unsigned long long best = 0ull;
    for (uint32_t i = gl; i < deg; i += G) {
        const uint32_t lab = my[i];
        if (lab == kEmpty) continue;
        uint32_t c = 0;
        for (uint32_t j = 0; j < deg4; j += 4) {  // four staged labels per 16-B load
            const uint4 q = *reinterpret_cast<const uint4*>(my + j);
            c += (q.x == lab) + (q.y == lab) + (q.z == lab) + (q.w == lab);
        }
        const unsigned long long p = ((unsigned long long)c << 32) | (unsigned long long)(~lab);
        best = p > best ? p : best;
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        const unsigned long long q = __shfl_xor_sync(kFull, best, o);
        best = q > best ? q : best;
    }
    if (valid && gl == 0) lp_finish(L, (uint32_t)(L.lo + rel), best, st);
}

// large destinations: a warp streams a kChunkEdges-edge chunk of one hub. Equal labels are
// merged per 32 edges (__match_any_sync), then counted in a per-warp shared table for the
// whole chunk; the chunk's distinct (label, count) pairs go to the hub's global table once
// (overflow goes straight to it). Each global update also raises the hub's running packed
// argmax (a label's (count, ~label) only grows, so the max over all updates is the max over
// the final counts).
constexpr int kWarpPairs = 128;  // measured: 64 ~ 128 < 256 (the flush scans every entry) << 512

// The returned (count, ~label) of every insert only grows per label, and the last insert of
// a label returns its final count: the max over one lane's inserts, reduced over the warp
// at the end of the chunk, needs one atomicMax per chunk.
// The home word is tried before table_add's probe loop (one read, then one CAS on a stale
// word or one add when the label is there; a lost CAS or a collision falls back to the
// loop): the same operations, measured faster than entering the loop directly.
__device__ __forceinline__ void hub_add(const LpLaunch& L, uint64_t base, uint32_t mask, uint32_t lab, uint32_t c,
                                        unsigned long long& lbest) {
    const uint32_t ep = L.hub.epoch;
    const unsigned long long w = __ldcg(L.hub.words + base + (mix32(lab) & mask));
    unsigned long long* wp = L.hub.words + base + (mix32(lab) & mask);
    unsigned long long r = 0ull;
    bool cas = false, add = false;
    if ((uint32_t)(w >> 56) != ep) {
        r = atomicCAS(wp, w, ((unsigned long long)ep << 56) | ((unsigned long long)c << 32) | lab);
        cas = true;
    } else if ((uint32_t)w == lab) {
        r = atomicAdd(wp, (unsigned long long)c << 32);
        add = true;
    }
    uint32_t nc;
    if (cas && r == w) nc = c;
    else if (add) nc = (uint32_t)((r >> 32) & 0xFFFFFFull) + c;
    else nc = table_add(L.hub, base, mask, lab, c);
    const unsigned long long pk = ((unsigned long long)nc << 32) | (unsigned long long)(~lab);
    lbest = pk > lbest ? pk : lbest;
}

__device__ __forceinline__ void lp_chunk(const LpLaunch& L, uint64_t item, uint32_t* wkeys, uint32_t* wcnts,
                                         uint32_t* wfull) {
    const int lane = threadIdx.x & 31;
    const unsigned lower = (1u << lane) - 1u;  // a group's leader has no lower lane in it (no ffs on the XU pipe)
    const uint32_t rel = __ldg(L.item_slot + item);
    const uint64_t beg = __ldg(L.item_begin + item);
    const uint64_t end = min(beg + (uint64_t)kChunkEdges, __ldg(L.in_off + rel + 1));
    const uint64_t base = __ldg(L.hub.tab_off + rel);
    const uint32_t mask = __ldg(L.hub.tab_mask + rel);
    for (int i = lane; i < kWarpPairs; i += 32) {
        wkeys[i] = kEmpty;
        wcnts[i] = 0;
    }
    if (lane == 0) *wfull = 0u;
    __syncwarp();
    unsigned long long lbest = 0ull;
    constexpr int kB = 4;  // the loads of 4 steps are issued together (measured: 4 beats 2, 8 and 16)
    for (uint64_t e0 = beg; e0 < end; e0 += 32 * kB) {
        uint32_t src[kB], lab[kB];
        bool ok[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const uint64_t e = e0 + 32 * j + lane;
            src[j] = e < end ? __ldg(L.in_src + e) : kEmpty;
        }
#pragma unroll
        for (int j = 0; j < kB; ++j) lab[j] = src[j] != kEmpty ? lp_msg(L, src[j]) : kEmpty;
#pragma unroll
        for (int j = 0; j < kB; ++j) ok[j] = lab[j] != kEmpty;
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            // 32-bit match: lanes without a message all carry kEmpty and group together,
            // but their leader is not `ok`, so that group is dropped
            const unsigned m = __match_any_sync(kFull, ok[j] ? lab[j] : kEmpty);
            if (ok[j] && !(m & lower)) {
                uint32_t h = mix32(lab[j]) & (kWarpPairs - 1);
                bool done = false;
                // once a probe sequence has failed the table is crowded: look at the home slot only
                const int probes = *reinterpret_cast<volatile uint32_t*>(wfull) ? 1 : 8;
#pragma unroll 1
                for (int probe = 0; probe < probes && !done; ++probe) {
                    const uint32_t k = atomicCAS(wkeys + h, kEmpty, lab[j]);
                    if (k == kEmpty || k == lab[j]) {
                        atomicAdd(wcnts + h, (uint32_t)__popc(m));
                        done = true;
                    }
                    h = (h + 1) & (kWarpPairs - 1);
                }
                if (!done) {
                    *reinterpret_cast<volatile uint32_t*>(wfull) = 1u;
                    hub_add(L, base, mask, lab[j], __popc(m), lbest);
                }
            }
        }
    }
    __syncwarp();
    {
        // the warp table's pairs to the hub's table, keys and counts read first
        constexpr int kPerLane = kWarpPairs / 32;
        uint32_t fk[kPerLane], fc[kPerLane];
        unsigned fv = 0u;
#pragma unroll
        for (int k = 0; k < kPerLane; ++k) {
            fk[k] = wkeys[lane + 32 * k];
            fc[k] = wcnts[lane + 32 * k];
            if (fk[k] != kEmpty) fv |= 1u << k;
        }
#pragma unroll
        for (int k = 0; k < kPerLane; ++k)
            if ((fv >> k) & 1u) hub_add(L, base, mask, fk[k], fc[k], lbest);
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long q = __shfl_xor_sync(kFull, lbest, o);
        lbest = q > lbest ? q : lbest;
    }
    if (lane == 0 && lbest && lbest > __ldcg(L.hub.best + rel)) atomicMax(L.hub.best + rel, lbest);
}

// Round 1 (labels = distinct vertex ids): a label's count at a hub is the multiplicity of
// one source, and the CSC keeps a hub's sources sorted, so counting is run-length over the
// chunk — no hash table, no atomics per edge. A run belongs to the chunk / lane where it
// starts: a lane skips a leading run that continues from the previous edge and extends its
// last run past its range (and past the chunk end) until the source changes.
// Only a run at least as long as the longest seen so far (this warp's runs, and the hub's
// running best from chunks already done) can win, so only those gather their label: on
// R-MAT hubs most runs are single edges below a longer run, and the label gathers — one
// random load per edge when every run was a candidate — are the kernel's cost. (A run's
// length raises the bar whether or not its source is active: sound because the labels are
// injective only before round 1 of a fresh state, where every source is active —
// gxb_state_create; every call that changes the active set clears lab_injective.)
__device__ __forceinline__ void lp_run_candidate(const LpLaunch& L, uint32_t src, uint32_t len, uint32_t bar,
                                                 unsigned long long& best) {
    if (len < bar) return;
    const uint32_t lab = lp_msg(L, src);
    if (lab == kEmpty) return;
    const unsigned long long pk = ((unsigned long long)len << 32) | (unsigned long long)(~lab);
    best = pk > best ? pk : best;
}

// Warp-wide over 32 consecutive edges per step (coalesced loads, no per-lane serial walk):
// run starts come from comparing each source with its predecessor; a run closes at the
// next start, so a start lane knows its run length when another start follows in the same
// window, the window's last run stays open into the next window, and the run open at `end`
// is followed past it (up to the segment end) until its source changes. Counts the runs
// that start in [beg, end) of the segment [seg_beg, seg_end); returns the warp's best
// packed (count, ~label) in every lane.
__device__ __forceinline__ unsigned long long lp_runs(const LpLaunch& L, uint64_t seg_beg, uint64_t seg_end,
                                                      uint64_t beg, uint64_t end, uint32_t bar) {
    const int lane = threadIdx.x & 31;
    unsigned long long best = 0ull;
    uint32_t prev = beg > seg_beg ? __ldg(L.in_src + beg - 1) : kNone;
    bool open = false;  // warp-uniform: a run that started in this range is still open
    uint32_t open_src = 0;
    uint64_t open_start = 0;
    for (uint64_t w0 = beg; w0 < end; w0 += 32) {
        const uint64_t e = w0 + lane;
        const bool in = e < end;
        const uint32_t s = in ? __ldg(L.in_src + e) : kNone;
        uint32_t p = __shfl_up_sync(kFull, s, 1);
        if (lane == 0) p = prev;
        const bool start = in && s != p;  // (a run continuing from before `beg` is not counted here)
        const unsigned M = __ballot_sync(kFull, start);
        uint32_t len = 0, len_open = 0;  // the runs that close in this window
        if (open && M && lane == 0) len_open = (uint32_t)(w0 + (__ffs(M) - 1) - open_start);
        if (start) {
            const unsigned above = M & ~((2u << lane) - 1u);
            if (above) len = (uint32_t)(__ffs(above) - 1 - lane);
        }
        bar = max(bar, __reduce_max_sync(kFull, max(len, len_open)));
        if (len_open) lp_run_candidate(L, open_src, len_open, bar, best);
        if (len) lp_run_candidate(L, s, len, bar, best);
        if (M) {
            const int last = 31 - __clz(M);
            open = true;
            open_src = __shfl_sync(kFull, s, last);
            open_start = w0 + last;
        }
        prev = __shfl_sync(kFull, s, 31);
    }
    if (open) {  // follow the last run past `end`
        uint64_t len = seg_end - open_start;
        for (uint64_t e0 = end; e0 < seg_end; e0 += 32) {
            const uint64_t e = e0 + lane;
            const bool in = e < seg_end;
            const uint32_t s = in ? __ldg(L.in_src + e) : kNone;
            const unsigned D = __ballot_sync(kFull, !in || s != open_src);
            if (D) {
                len = e0 + (__ffs(D) - 1) - open_start;
                break;
            }
        }
        if (lane == 0) lp_run_candidate(L, open_src, (uint32_t)len, bar, best);
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long q = __shfl_xor_sync(kFull, best, o);
        best = q > best ? q : best;
    }
    return best;
}

__device__ __forceinline__ void lp_chunk_injective(const LpLaunch& L, uint64_t item) {
    const int lane = threadIdx.x & 31;
    const uint32_t rel = __ldg(L.item_slot + item);
    const uint64_t seg_beg = __ldg(L.in_off + rel), seg_end = __ldg(L.in_off + rel + 1);
    const uint64_t beg = __ldg(L.item_begin + item);
    const uint64_t end = min(beg + (uint64_t)kChunkEdges, seg_end);
    // the hub's running best from chunks already done is a lower bound for a winning count
    const uint32_t bar = (uint32_t)(__ldcg(L.hub.best + rel) >> 32);
    const unsigned long long best = lp_runs(L, seg_beg, seg_end, beg, end, bar);
    if (lane == 0 && best && best > __ldcg(L.hub.best + rel)) atomicMax(L.hub.best + rel, best);
}

// ---- dense rounds >= 2: hubs counted in shared memory ----
// A destination with kChunkMinDeg < in-degree <= kLpBigDeg is counted by one CTA (in-degree
// > kLpCtaMinDeg) or one warp (the rest) in an open-addressing (label, count) table in
// shared memory sized to twice the in-degree (every distinct label fits at load <= 1/2),
// after equal labels of 32 edges are merged (__match_any_sync). The label-diverse hubs
// above kLpBigDeg stay in chunked warps over all SMs with epoch-tagged global tables.
constexpr uint32_t kLpCtaMinDeg = 512;
constexpr uint32_t kLpBigDeg = 4096;  // above: chunked warps over all SMs + global tables (label-diverse hubs)
constexpr int kLpCtaCap = 8192;    // 64 KB of (key, count) per CTA
constexpr int kLpWarpCap = 1024;   // 8 KB per warp
constexpr int kLpWarpMinBin = 4;   // group bins >= this (G = 16, 32: in-degree 33-128) use warp tables

__global__ void k_lp_eff(const uint32_t* __restrict__ active, const uint32_t* __restrict__ lab, uint64_t S,
                         uint32_t* eff) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < S; i += (uint64_t)gridDim.x * blockDim.x)
        eff[i] = ((__ldg(active + (i >> 5)) >> (i & 31)) & 1u) ? __ldg(lab + i) : kEmpty;
}

// insert c copies of `lab` into a shared table sized to at least twice the destination's
// in-degree: distinct labels <= in-degree keep the load <= 1/2, so probing always ends
__device__ __forceinline__ void smem_table_add(uint32_t* keys, uint32_t* cnts, uint32_t mask, uint32_t lab,
                                               uint32_t c) {
    uint32_t h = mix32(lab) & mask;
    while (true) {
        uint32_t k = keys[h];
        if (k == kEmpty) {
            k = atomicCAS(keys + h, kEmpty, lab);
            if (k == kEmpty) k = lab;
        }
        if (k == lab) {
            atomicAdd(cnts + h, c);
            return;
        }
        h = (h + 1) & mask;
    }
}

// The same for epoch-tagged shared tables: one 64-bit word per entry, epoch (8 bits) |
// count (24) | label (32), like the hubs' global tables. A word of another epoch is empty,
// so a table is not cleared between destinations (every 255), and the insert returns the
// label's running count: the max of the returned (count, ~label) is the destination's
// best (a label's count only grows), so the table is not scanned either.
__device__ __forceinline__ uint32_t smem_ep_add(unsigned long long* tab, uint32_t mask, uint32_t ep, uint32_t lab,
                                                uint32_t c) {
    uint32_t h = mix32(lab) & mask;
    unsigned long long w = tab[h];
    while (true) {
        if ((uint32_t)(w >> 56) != ep) {  // empty for this destination: claim
            const unsigned long long nw = ((unsigned long long)ep << 56) | ((unsigned long long)c << 32) | lab;
            const unsigned long long prev = atomicCAS(tab + h, w, nw);
            if (prev == w) return c;
            w = prev;
            continue;
        }
        if ((uint32_t)w == lab) {  // the label's entry: add (CAS retry on a concurrent add)
            const unsigned long long prev = atomicCAS(tab + h, w, w + ((unsigned long long)c << 32));
            if (prev == w) return (uint32_t)((w >> 32) & 0xFFFFFFull) + c;
            w = prev;
            continue;
        }
        h = (h + 1) & mask;
        w = tab[h];
    }
}

__device__ __forceinline__ unsigned long long pack_best(uint32_t count, uint32_t lab) {
    return ((unsigned long long)count << 32) | (unsigned long long)(~lab);
}

// stream [beg, end) with `nthreads` threads (index t), 8 loads in flight per lane, and fold
// each 32-edge group's labels into the shared table
__device__ __forceinline__ void lp_count_edges(const LpLaunch& L, uint64_t beg, uint64_t end, unsigned t,
                                               unsigned nthreads, uint32_t* keys, uint32_t* cnts, uint32_t mask) {
    constexpr int kB = 4;  // 32-edge groups loaded together per lane (measured: 4 beats 2 and 8)
    const int lane = threadIdx.x & 31;
    const unsigned lower = (1u << lane) - 1u;  // a group's leader has no lower lane in it (no ffs on the XU pipe)
    // 32-edge groups dealt round-robin over the warps (group g to warp g mod nw), kB per
    // step: with one CTA per destination, every warp has edges down to in-degree 32 x nw
    const uint64_t nw = nthreads / 32, wi = (t - lane) / 32;
    for (uint64_t g0 = wi; beg + g0 * 32 < end; g0 += nw * kB) {
        uint32_t src[kB], lab[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const uint64_t e = beg + (g0 + j * nw) * 32 + lane;
            src[j] = e < end ? __ldg(L.in_src + e) : kEmpty;
        }
#pragma unroll
        for (int j = 0; j < kB; ++j) lab[j] = src[j] != kEmpty ? lp_msg(L, src[j]) : kEmpty;
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const bool ok = lab[j] != kEmpty;
            const unsigned m = __match_any_sync(kFull, lab[j]);  // no-message lanes group under kEmpty
            if (ok && !(m & lower)) smem_table_add(keys, cnts, mask, lab[j], (uint32_t)__popc(m));
        }
    }
}

// lp_count_edges into an epoch-tagged table; returns this thread's best packed (count, ~label)
__device__ __forceinline__ unsigned long long lp_count_edges_ep(const LpLaunch& L, uint64_t beg, uint64_t end,
                                                                unsigned t, unsigned nthreads, unsigned long long* tab,
                                                                uint32_t mask, uint32_t ep) {
    constexpr int kB = 4;  // 32-edge groups loaded together per lane (measured: 4 beats 2 and 8)
    const int lane = threadIdx.x & 31;
    const unsigned lower = (1u << lane) - 1u;
    const unsigned warp0 = t - lane;
    unsigned long long best = 0ull;
    for (uint64_t e0 = beg + (uint64_t)warp0 * kB; e0 < end; e0 += (uint64_t)nthreads * kB) {
        uint32_t src[kB], lab[kB];
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const uint64_t e = e0 + 32 * j + lane;
            src[j] = e < end ? __ldg(L.in_src + e) : kEmpty;
        }
#pragma unroll
        for (int j = 0; j < kB; ++j) lab[j] = src[j] != kEmpty ? lp_msg(L, src[j]) : kEmpty;
#pragma unroll
        for (int j = 0; j < kB; ++j) {
            const bool ok = lab[j] != kEmpty;
            const unsigned m = __match_any_sync(kFull, lab[j]);
            if (ok && !(m & lower)) {
                const unsigned long long pk = pack_best(smem_ep_add(tab, mask, ep, lab[j], (uint32_t)__popc(m)), lab[j]);
                best = pk > best ? pk : best;
            }
        }
    }
    return best;
}

// One CTA per destination, a (label, count) table in shared memory (32-bit keys and counts:
// native shared atomics, which the hot labels' contention between the CTA's warps needs —
// an epoch-tagged 64-bit word table was measured 10% slower here). The scan for the best
// entry also empties the table for the next destination, and thread 0 finishes a
// destination from its parity's row of warp results: two barriers per destination.
__global__ void __launch_bounds__(kBlock) k_lp_hub_cta(const LpLaunch L, uint64_t lo_rel, uint64_t cta_end) {
    extern __shared__ uint32_t lp_dyn[];  // kLpCtaCap keys, then kLpCtaCap counts
    uint32_t* keys = lp_dyn;
    uint32_t* cnts = lp_dyn + kLpCtaCap;
    __shared__ unsigned long long wbest[2][kBlock / 32];
    LocalStats st;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t i = threadIdx.x; i < kLpCtaCap; i += kBlock) {
        keys[i] = kEmpty;
        cnts[i] = 0;
    }
    __syncthreads();
    int par = 0;
    for (uint64_t rel = lo_rel + blockIdx.x; rel < cta_end; rel += gridDim.x, par ^= 1) {
        const uint64_t beg = __ldg(L.in_off + rel), end = __ldg(L.in_off + rel + 1);
        uint32_t C = 64;
        while ((uint64_t)C < 2 * (end - beg)) C <<= 1;  // <= kLpCtaCap for in-degree <= kLpBigDeg
        lp_count_edges(L, beg, end, threadIdx.x, kBlock, keys, cnts, C - 1);
        __syncthreads();
        unsigned long long best = 0ull;
        for (uint32_t i = threadIdx.x; i < C; i += kBlock) {
            const uint32_t k = keys[i];
            if (k != kEmpty) {
                const unsigned long long pk = pack_best(cnts[i], k);
                best = pk > best ? pk : best;
                keys[i] = kEmpty;
                cnts[i] = 0;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long q = __shfl_xor_sync(kFull, best, o);
            best = q > best ? q : best;
        }
        if (lane == 0) wbest[par][warp] = best;
        __syncthreads();  // the table is empty again, the warp results are in
        if (threadIdx.x == 0) {
            for (int w = 1; w < kBlock / 32; ++w) best = wbest[par][w] > best ? wbest[par][w] : best;
            lp_finish(L, (uint32_t)(L.lo + rel), best, st);
        }
    }
    flush_stats(st, L.stats);
}

// The same with each half of the CTA on its own destination (in-degree <= kLpCtaHalfDeg):
// named barriers per half, so one half's finish and scan do not hold the other's counting.
constexpr uint32_t kLpCtaHalfDeg = kLpCtaCap / 4;
__global__ void __launch_bounds__(kBlock) k_lp_hub_cta2(const LpLaunch L, uint64_t lo_rel, uint64_t hi_rel) {
    constexpr int kHalf = kBlock / 2, kCap = kLpCtaCap / 2;
    extern __shared__ uint32_t lp_dyn[];  // per half: kCap keys, then kCap counts
    const int half = threadIdx.x / kHalf, t = threadIdx.x % kHalf;
    uint32_t* keys = lp_dyn + half * 2 * kCap;
    uint32_t* cnts = keys + kCap;
    __shared__ unsigned long long wbest[2][kBlock / 32];
    LocalStats st;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    auto half_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + half), "r"(kHalf) : "memory"); };
    for (uint32_t i = t; i < kCap; i += kHalf) {
        keys[i] = kEmpty;
        cnts[i] = 0;
    }
    half_sync();
    int par = 0;
    for (uint64_t rel = lo_rel + 2ull * blockIdx.x + half; rel < hi_rel; rel += 2ull * gridDim.x, par ^= 1) {
        const uint64_t beg = __ldg(L.in_off + rel), end = __ldg(L.in_off + rel + 1);
        uint32_t C = 64;
        while ((uint64_t)C < 2 * (end - beg)) C <<= 1;  // <= kCap
        lp_count_edges(L, beg, end, t, kHalf, keys, cnts, C - 1);
        half_sync();
        unsigned long long best = 0ull;
        for (uint32_t i = t; i < C; i += kHalf) {
            const uint32_t k = keys[i];
            if (k != kEmpty) {
                const unsigned long long pk = pack_best(cnts[i], k);
                best = pk > best ? pk : best;
                keys[i] = kEmpty;
                cnts[i] = 0;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long q = __shfl_xor_sync(kFull, best, o);
            best = q > best ? q : best;
        }
        if (lane == 0) wbest[par][warp] = best;
        half_sync();
        if (t == 0) {
            for (int w = 1; w < kHalf / 32; ++w) best = wbest[par][warp + w] > best ? wbest[par][warp + w] : best;
            lp_finish(L, (uint32_t)(L.lo + rel), best, st);
        }
    }
    flush_stats(st, L.stats);
}

// kCap: table entries per warp — 2 x the largest in-degree of the launch's slots (the
// 33-128 slots run with 256-entry tables: a quarter of the shared memory, more warps per SM)
template <int kCap>
__global__ void __launch_bounds__(kBlock) k_lp_hub_warp(const LpLaunch L, uint64_t lo_rel, uint64_t hi_rel) {
    extern __shared__ unsigned long long lp_tab[];  // per warp: kCap epoch-tagged words
    LocalStats st;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long* wt = lp_tab + warp * kCap;
    uint32_t ep = 255;  // wraps to 1 (and clears the table) on the first destination
    const uint64_t nw = (uint64_t)gridDim.x * (kBlock / 32);
    // lane k keeps the result of this warp's k-th destination of a batch of 32; the batch
    // is finished (and published) together
    uint32_t pslot = 0;
    unsigned long long pbest = 0ull;
    int nb = 0;
    for (uint64_t rel = lo_rel + blockIdx.x * (uint64_t)(kBlock / 32) + warp; rel < hi_rel; rel += nw) {
        const uint64_t beg = __ldg(L.in_off + rel), end = __ldg(L.in_off + rel + 1);
        unsigned long long best = 0ull;
        if (L.injective) {
            best = lp_runs(L, beg, end, beg, end, 0u);  // round 1: run-length, no table
        } else {
            if (++ep == 256) {
                ep = 1;
                for (uint32_t i = lane; i < kCap; i += 32) wt[i] = 0ull;
                __syncwarp();
            }
            uint32_t C = 64;
            while ((uint64_t)C < 2 * (end - beg)) C <<= 1;  // <= kCap
            best = lp_count_edges_ep(L, beg, end, lane, 32, wt, C - 1, ep);
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long q = __shfl_xor_sync(kFull, best, o);
                best = q > best ? q : best;
            }
        }
        if (lane == nb) {
            pslot = (uint32_t)(L.lo + rel);
            pbest = best;
        }
        if (++nb == 32) {
            lp_finish_lanes(L, true, pslot, pbest, st);
            nb = 0;
        }
        __syncwarp();
    }
    lp_finish_lanes(L, lane < nb, pslot, pbest, st);
    flush_stats(st, L.stats);
}

// chunk items of the hubs (rounds >= 2): one warp per kChunkEdges-edge chunk. Kernels of
// their own, apart from the group bins (which run at 32 registers instead of the chunk
// path's 40) and from round 1's run-length chunks
__global__ void __launch_bounds__(kBlock) k_lp_chunks(const LpLaunch L) {
    __shared__ uint32_t buf[2 * kWarpPairs * (kBlock / 32)];
    __shared__ uint32_t wfull[kBlock / 32];
    const uint64_t item = (uint64_t)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
    uint32_t* wk = buf + (threadIdx.x >> 5) * 2 * kWarpPairs;
    if (item < L.num_items) lp_chunk(L, item, wk, wk + kWarpPairs, wfull + (threadIdx.x >> 5));
    // chunked slots are applied by k_lp_hub_apply
}

// round 1's chunk items: run-length counting
__global__ void __launch_bounds__(kBlock) k_lp_chunks_runs(const LpLaunch L) {
    const uint64_t item = (uint64_t)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
    if (item < L.num_items) lp_chunk_injective(L, item);
}

// the group bins (in-degree <= 32; 33-128 go to the warp tables)
__global__ void __launch_bounds__(kBlock) k_lp_pull(const LpLaunch L) {
    __shared__ __align__(16) uint32_t buf[4 * kBlock];  // 4 labels per thread
    LocalStats st;
    unsigned b = blockIdx.x;
    int k = kNumGroupBins - 1;
    for (; k > 0; --k) {
        if (b < L.bin_blocks[k]) break;
        b -= L.bin_blocks[k];
    }
    switch (k) {
        case 5: lp_group<32>(L, 5, b, buf, st); break;
        case 4: lp_group<16>(L, 4, b, buf, st); break;
        case 3: lp_group<8>(L, 3, b, buf, st); break;
        case 2: lp_group<4>(L, 2, b, buf, st); break;
        case 1: lp_group<2>(L, 1, b, buf, st); break;
        default: lp_group<1>(L, 0, b, buf, st); break;
    }
    flush_stats(st, L.stats);
}

__global__ void __launch_bounds__(kBlock) k_lp_hub_apply(const LpLaunch L, uint64_t chunk_end) {
    LocalStats st;
    for (uint64_t rel = blockIdx.x * (uint64_t)kBlock + threadIdx.x; rel < chunk_end; rel += (uint64_t)gridDim.x * kBlock) {
        const unsigned long long best = L.hub.best[rel];
        L.hub.best[rel] = 0ull;
        lp_finish(L, (uint32_t)(L.lo + rel), best, st);
    }
    flush_stats(st, L.stats);
}

// ---- sparse rounds: push the frontier's labels along the CSR ----
// Only active sources send, so a sparse round's multisets are small: every (destination,
// label) pair of the round is counted in one open-addressing table keyed by
// dst << 32 | label (warp-aggregated: a chunk's edges share their source and label, so
// equal keys are parallel edges), each update raises the destination's packed running
// argmax, and the first update of a destination appends it to the round's target list.
struct LpPush {
    unsigned long long* keys;  // capacity (power of two), ~0 = empty
    uint32_t* counts;
    unsigned long long* best;  // per owned slot, 0 = no message
    uint32_t* targets;         // relative slots that received a message this round
    unsigned long long* ntargets;
    uint64_t capacity;
};

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

__device__ __forceinline__ uint32_t pair_add(const LpPush& P, uint64_t mask, unsigned long long key, uint32_t c) {
    uint64_t i = mix64(key) & mask;
    while (true) {
        unsigned long long k = __ldcg(P.keys + i);
        if (k == ~0ull) {
            k = atomicCAS(P.keys + i, ~0ull, key);
            if (k == ~0ull) k = key;
        }
        if (k == key) return atomicAdd(P.counts + i, c) + c;
        i = (i + 1) & mask;
    }
}

// Pairs aimed at the largest hubs (relative slot < hub_end: slots are in-degree sorted, and
// hub_end covers in-degree >= kLpHotDegree) are first counted
// in a block-local shared table and flushed once per block: many frontier sources with the
// same label hit the same hub, and folding them in shared memory keeps the global table
// from serialising on a few hot (hub, label) counters.
constexpr int kLpSmemPairs = 2048;

__device__ __forceinline__ bool smem_pair_add(unsigned long long* keys, uint32_t* counts, unsigned long long key,
                                              uint32_t c) {
    uint32_t i = (uint32_t)mix64(key) & (kLpSmemPairs - 1);
#pragma unroll 1
    for (int probe = 0; probe < 16; ++probe) {
        unsigned long long k = keys[i];
        if (k == ~0ull) {
            k = atomicCAS(keys + i, ~0ull, key);
            if (k == ~0ull) k = key;
        }
        if (k == key) {
            atomicAdd(counts + i, c);
            return true;
        }
        i = (i + 1) & (kLpSmemPairs - 1);
    }
    return false;  // crowded: the caller goes to the global table
}

// returns whether this update was the destination's first message of the round (the
// caller appends it to the target list, warp-aggregated)
__device__ __forceinline__ bool global_pair(const LpPush& P, uint64_t mask, unsigned long long key, uint32_t c) {
    const uint32_t rel = (uint32_t)(key >> 32), lab = (uint32_t)key;
    const uint32_t nc = pair_add(P, mask, key, c);
    const unsigned long long pk = ((unsigned long long)nc << 32) | (unsigned long long)(~lab);
    if (pk > __ldcg(P.best + rel)) return atomicMax(P.best + rel, pk) == 0ull;
    return false;
}

// all lanes of the warp call it: one reservation per warp for the new targets
__device__ __forceinline__ void append_targets(const LpPush& P, bool first, uint32_t rel) {
    const unsigned m = __ballot_sync(kFull, first);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(P.ntargets, (unsigned long long)__popc(m));
    base = __shfl_sync(kFull, base, __ffs(m) - 1);
    if (first) P.targets[base + __popc(m & ((1u << lane) - 1u))] = rel;
}

// Edge-balanced over the concatenated CSR rows of the frontier (rowpre = inclusive prefix
// of row lengths): a warp takes 256 consecutive edges, finds the first one's row with one
// binary search, and each lane walks forward to its own rows — many short rows cost no
// more than one long one.
constexpr uint32_t kLpItemEdges = 128;  // edges per warp work item (128 vs 256: push rounds -3%)

__global__ void __launch_bounds__(kBlock) k_lp_push(const uint32_t* __restrict__ frontier, uint64_t nfront,
                                                    const uint32_t* __restrict__ rowpre,
                                                    const uint64_t* __restrict__ out_off,
                                                    const uint32_t* __restrict__ out_dst,
                                                    const uint32_t* __restrict__ lab_cur, uint64_t lo, LpPush P,
                                                    uint64_t mask, uint32_t hub_end) {
    __shared__ unsigned long long skeys[kLpSmemPairs];
    __shared__ uint32_t scounts[kLpSmemPairs];
    for (int i = threadIdx.x; i < kLpSmemPairs; i += kBlock) {
        skeys[i] = ~0ull;
        scounts[i] = 0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned lower = (1u << lane) - 1u;  // a group's leader has no lower lane in it (no ffs on the XU pipe)
    const uint64_t total = nfront ? rowpre[nfront - 1] : 0;
    const uint64_t items = (total + kLpItemEdges - 1) / kLpItemEdges;
    const uint64_t nwarps = (uint64_t)gridDim.x * (kBlock / 32);
    for (uint64_t it = (uint64_t)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); it < items; it += nwarps) {
        const uint64_t g0 = it * kLpItemEdges, g1 = min(total, g0 + kLpItemEdges);
        uint64_t a = 0, b = nfront - 1;  // row of edge g0: first f with rowpre[f] > g0
        while (a < b) {
            const uint64_t mid = (a + b) >> 1;
            if (__ldg(rowpre + mid) > g0) b = mid; else a = mid + 1;
        }
        uint64_t f = a;  // this lane's row cursor (monotone over its edges)
        // the item's dependent loads level by level for all of a lane's edges (row -> source
        // -> edge -> destination, label), so each level has kJ loads in flight, then the
        // counting over the loaded (destination, label) pairs
        constexpr int kJ = kLpItemEdges / 32;
        uint32_t relj[kJ], labj[kJ];
        uint64_t ej[kJ];
        unsigned okm = 0u;
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            const uint64_t gl = g0 + j * 32 + lane;
            if (gl < g1) {
                okm |= 1u << j;
                f = row_advance(rowpre, nfront, f, gl);
                ej[j] = f;  // the row for now
            }
        }
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            if ((okm >> j) & 1u) {
                const uint64_t fj = ej[j];
                labj[j] = __ldg(frontier + fj);  // the source for now
                ej[j] = (g0 + j * 32 + lane) - (fj ? __ldg(rowpre + fj - 1) : 0);
            }
        }
#pragma unroll
        for (int j = 0; j < kJ; ++j)
            if ((okm >> j) & 1u) ej[j] += __ldg(out_off + labj[j]);
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            relj[j] = 0u;
            if ((okm >> j) & 1u) {
                relj[j] = (uint32_t)(__ldg(out_dst + ej[j]) - lo);
                labj[j] = __ldg(lab_cur + labj[j]);
            }
        }
#pragma unroll
        for (int j = 0; j < kJ; ++j) {
            const bool ok = (okm >> j) & 1u;
            const uint32_t rel = relj[j], lab = ok ? labj[j] : 0u;
            const unsigned long long key = ok ? ((unsigned long long)rel << 32 | lab) : (~0ull - 1 - lane);
            const unsigned m = __match_any_sync(kFull, key);
            bool first = false;
            if (ok && !(m & lower)) {
                if (!(rel < hub_end && smem_pair_add(skeys, scounts, key, __popc(m))))
                    first = global_pair(P, mask, key, __popc(m));
            }
            append_targets(P, first, rel);
        }
    }
    __syncthreads();
    for (int i0 = 0; i0 < kLpSmemPairs; i0 += kBlock) {  // block-uniform trip count
        const int i = i0 + threadIdx.x;
        const unsigned long long key = skeys[i];
        const bool first = key != ~0ull && global_pair(P, mask, key, scounts[i]);
        append_targets(P, first, (uint32_t)(key >> 32));
    }
}

__global__ void __launch_bounds__(kBlock) k_lp_push_apply(const LpLaunch L, LpPush P) {
    LocalStats st;
    const uint64_t n = *P.ntargets;
    for (uint64_t i = blockIdx.x * (uint64_t)kBlock + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kBlock) {
        const uint32_t rel = P.targets[i];
        const unsigned long long best = P.best[rel];
        P.best[rel] = 0ull;
        lp_finish(L, (uint32_t)(L.lo + rel), best, st);
    }
    flush_stats(st, L.stats);
}

static uint64_t next_pow2(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

// sparse-round scratch: a pair table of `cap` entries, per-slot argmax and target list
static int lp_push_reserve(gxb_state* s, LpScratch* S, uint64_t cap, cudaStream_t st) {
    const uint64_t owned = s->g->hi - s->g->lo;
    if (!S->pntargets) GXB_CHECK(dalloc_t(&S->pntargets, 2));
    if (!S->pbest) {
        GXB_CHECK(dalloc_t(&S->pbest, owned + 1));
        GXB_CHECK(dalloc_t(&S->ptargets, owned + 1));
        GXB_CUDA(cudaMemsetAsync(S->pbest, 0, 8 * (owned + 1), st));
    }
    if (cap > S->pcapacity) {
        dfree(S->pkeys);
        dfree(S->pcounts);
        S->pkeys = nullptr;
        S->pcounts = nullptr;
        S->pcapacity = 0;
        GXB_CHECK(dalloc_t(&S->pkeys, cap));
        GXB_CHECK(dalloc_t(&S->pcounts, cap));
        S->pcapacity = cap;
    }
    return GXB_OK;
}

static void lp_free(LpScratch* S) {
    if (!S) return;
    LpHub& H = S->hub;
    dfree(H.tab_off);
    dfree(H.tab_mask);
    dfree(H.words);
    dfree(H.best);
    dfree(S->pkeys);
    dfree(S->pcounts);
    dfree(S->pbest);
    dfree(S->ptargets);
    dfree(S->pntargets);
    dfree(S->eff);
    delete S;
}

constexpr uint32_t kLpHotDegree = 16384;

static int lp_setup(gxb_state* s, cudaStream_t st) {
    const gxb_graph* g = s->g;
    const PullPlan& P = g->plan;
    LpScratch* S = new LpScratch();
    S->chunk_end = P.chunk_end;
    while (S->big_end < P.chunk_end && g->h_indeg_sorted[S->big_end] > kLpBigDeg) {
        S->big_items += (g->h_indeg_sorted[S->big_end] + kChunkEdges - 1) / kChunkEdges;
        ++S->big_end;
    }
    S->cta_end = S->big_end;
    S->cta_half = S->big_end;
    while (S->cta_half < P.chunk_end && g->h_indeg_sorted[S->cta_half] > kLpCtaHalfDeg) ++S->cta_half;
    S->cta_end = S->cta_half;
    while (S->cta_end < P.chunk_end && g->h_indeg_sorted[S->cta_end] > kLpCtaMinDeg) ++S->cta_end;
    while (S->hot_end < g->h_indeg_sorted.size() && g->h_indeg_sorted[S->hot_end] >= kLpHotDegree) ++S->hot_end;
    LpHub& H = S->hub;
    std::vector<uint64_t> off(S->big_end + 1);
    std::vector<uint32_t> mask(S->big_end + 1);
    uint64_t acc = 0;
    for (uint64_t r = 0; r < S->big_end; ++r) {
        const uint64_t size = std::max<uint64_t>(256, next_pow2(2ull * g->h_indeg_sorted[r]));
        off[r] = acc;
        mask[r] = (uint32_t)(size - 1);
        acc += size;
    }
    H.entries = acc;
    H.epoch = 0;  // the tables start zeroed: epoch 0 words are empty from round 1 on
    if (S->big_end && g->h_indeg_sorted[0] >= (1u << 24)) {
        lp_free(S);
        return fail(GXB_ERANGE, "LabelPropagation: an in-degree >= 2^24 exceeds the hub tables' count field");
    }
    int rc = GXB_OK;
    auto up = [&](auto** d, const auto& h) {
        if (rc != GXB_OK) return;
        rc = dalloc_t(d, h.size() + 1);
        if (rc == GXB_OK && !h.empty())
            if (cudaMemcpyAsync(*d, h.data(), sizeof(h[0]) * h.size(), cudaMemcpyHostToDevice, st) != cudaSuccess)
                rc = fail(GXB_ECUDA, "lp_setup copy");
    };
    up(&H.tab_off, off);
    up(&H.tab_mask, mask);
    if (rc == GXB_OK) rc = dalloc_t(&H.words, acc + 1);
    if (rc == GXB_OK) rc = dalloc_t(&H.best, P.chunk_end + 1);
    if (rc == GXB_OK) rc = dalloc_t(&S->eff, g->S + 1);
    if (rc == GXB_OK) {
        cudaMemsetAsync(H.words, 0, 8 * (acc + 1), st);
        cudaMemsetAsync(H.best, 0, 8 * (P.chunk_end + 1), st);
        if (cudaStreamSynchronize(st) != cudaSuccess) rc = fail(GXB_ECUDA, "lp_setup sync");
    }
    if (rc != GXB_OK) {
        lp_free(S);
        return rc;
    }
    s->d_lp_scratch = S;  // host-side object (freed by gxb_lp_free)
    return GXB_OK;
}

}  // namespace gxb

using namespace gxb;

static LpLaunch lp_launch(gxb_state* s) {
    const gxb_graph* g = s->g;
    LpLaunch L{};
    L.lo = g->lo;
    L.in_off = g->d_in_off;
    L.in_src = g->d_in_src;
    L.lab_cur = s->d_lab_cur;
    L.lab_next = s->d_lab_next;
    L.active_cur = s->d_active[0];
    L.f.lo = g->lo;
    L.f.outdeg = g->d_outdeg;
    L.f.remote_src = g->d_remote_src;
    L.f.active_next = s->d_active[1];
    L.f.frontier_next = s->d_frontier[1];
    L.f.frontier_count = s->d_fcount + 1;
    L.stats = s->d_stats;
    return L;
}

extern "C" void gxb_lp_free(gxb_state* s) {
    if (s && s->d_lp_scratch) {
        lp_free(reinterpret_cast<LpScratch*>(s->d_lp_scratch));
        s->d_lp_scratch = nullptr;
    }
}

extern "C" int gxb_lp_prepare(gxb_state* s, cudaStream_t st) {
    if (!s->d_lp_scratch) GXB_CHECK(lp_setup(s, st));
    if (s->g->has_csr) {  // sparse rounds push at most E / push_alpha edges: no cudaMalloc mid-run
        const uint64_t alpha = std::max<int64_t>(1, options().push_alpha);
        const uint64_t cap = std::max<uint64_t>(1024, next_pow2(2 * (s->g->E / alpha) + 2));
        GXB_CHECK(lp_push_reserve(s, reinterpret_cast<LpScratch*>(s->d_lp_scratch), cap, st));
    }
    return GXB_OK;
}

extern "C" int gxb_lp_pull(gxb_state* s, cudaStream_t st) {
    if (!s->d_lp_scratch) GXB_CHECK(lp_setup(s, st));
    LpScratch* S = reinterpret_cast<LpScratch*>(s->d_lp_scratch);
    const gxb_graph* g = s->g;
    const PullPlan& P = g->plan;
    LpLaunch L = lp_launch(s);
    L.num_items = P.num_items;
    L.item_slot = P.d_item_slot;
    L.item_begin = P.d_item_begin;
    L.chunk_blocks = (unsigned)((P.num_items + (kBlock / 32) - 1) / (kBlock / 32));
    uint64_t prev = P.chunk_end;
    unsigned grid = L.chunk_blocks;
    for (int k = kNumGroupBins - 1; k >= 0; --k) {
        L.bin_lo[k] = prev;
        L.bin_hi[k] = std::max(prev, P.group_end[k]);
        const uint64_t per = kBlock >> k;
        L.bin_blocks[k] = (unsigned)((L.bin_hi[k] - L.bin_lo[k] + per - 1) / per);
        grid += L.bin_blocks[k];
        prev = L.bin_hi[k];
    }
    L.hub = S->hub;
    L.injective = s->lab_injective;
    static bool attrs_set[64] = {};
    const int dev = g->ctx->device & 63;
    if (!attrs_set[dev]) {
        GXB_CUDA(cudaFuncSetAttribute(k_lp_hub_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 4 * kLpCtaCap));
        GXB_CUDA(cudaFuncSetAttribute(k_lp_hub_cta2, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 4 * kLpCtaCap));
        GXB_CUDA(cudaFuncSetAttribute(k_lp_hub_warp<kLpWarpCap>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (kBlock / 32) * 2 * 4 * kLpWarpCap));
        attrs_set[dev] = true;
    }
    // effective labels: one gather per edge (label of an active source, else empty)
    if (g->S) k_lp_eff<<<grid_for(g->S), kBlock, 0, st>>>(s->d_active[0], s->d_lab_cur, g->S, S->eff);
    L.eff = S->eff;
    // the G = 32 and G = 16 bins (in-degree 33-128) are counted in warp shared tables instead
    // of the quadratic in-group count (every round, the first included: measured)
    uint64_t warp_end = S->chunk_end;
    for (int k = kNumGroupBins - 1; k >= kLpWarpMinBin; --k) {
        warp_end = std::max(warp_end, L.bin_hi[k]);
        grid -= L.bin_blocks[k];
        L.bin_blocks[k] = 0;
    }
    uint64_t warp_lo = S->chunk_end;  // round 1: the chunked hubs are run-length counted
    if (!L.injective) {
        // rounds >= 2: chunk items of the label-diverse big hubs only (the plan lists items
        // in slot order; epoch-tagged global tables), CTA tables for 513-4096, warp tables
        // for 33-512
        if (++S->hub.epoch > 255) {  // 8-bit epochs: zero the tables once per 255 rounds
            S->hub.epoch = 1;
            if (S->hub.entries) GXB_CUDA(cudaMemsetAsync(S->hub.words, 0, 8 * S->hub.entries, st));
        }
        L.hub.epoch = S->hub.epoch;  // this round's table words (older ones read as empty)
        grid -= L.chunk_blocks;
        L.num_items = S->big_items;
        L.chunk_blocks = (unsigned)((S->big_items + (kBlock / 32) - 1) / (kBlock / 32));
        grid += L.chunk_blocks;
        warp_lo = S->cta_end;
    }
    if (L.chunk_blocks) {
        if (L.injective) k_lp_chunks_runs<<<L.chunk_blocks, kBlock, 0, st>>>(L);
        else k_lp_chunks<<<L.chunk_blocks, kBlock, 0, st>>>(L);
    }
    grid -= L.chunk_blocks;
    if (grid) k_lp_pull<<<grid, kBlock, 0, st>>>(L);
    if (!L.injective && S->cta_end > S->big_end) {  // CTA tables: a whole CTA above kLpCtaHalfDeg, else half
        if (S->cta_half > S->big_end)
            k_lp_hub_cta<<<(unsigned)std::min<uint64_t>(S->cta_half - S->big_end, 3ull * kNumSMs), kBlock,
                           2 * 4 * kLpCtaCap, st>>>(L, S->big_end, S->cta_half);
        if (S->cta_end > S->cta_half)
            k_lp_hub_cta2<<<(unsigned)std::min<uint64_t>((S->cta_end - S->cta_half + 1) / 2, 3ull * kNumSMs), kBlock,
                            2 * 4 * kLpCtaCap, st>>>(L, S->cta_half, S->cta_end);
    }
    // warp tables: in-degree 129-512 (rounds >= 2) with 1024 entries, 33-128 with 256
    auto warp_grid = [](uint64_t n) {
        return (unsigned)std::min<uint64_t>((n + kBlock / 32 - 1) / (kBlock / 32), 6ull * kNumSMs);
    };
    const uint64_t small_lo = std::max(warp_lo, S->chunk_end);
    if (small_lo > warp_lo)
        k_lp_hub_warp<kLpWarpCap><<<warp_grid(small_lo - warp_lo), kBlock, (kBlock / 32) * 2 * 4 * kLpWarpCap, st>>>(
            L, warp_lo, small_lo);
    if (warp_end > small_lo)
        k_lp_hub_warp<2 * kChunkMinDeg><<<warp_grid(warp_end - small_lo), kBlock, (kBlock / 32) * 2 * 4 * 2 * kChunkMinDeg,
                                           st>>>(L, small_lo, warp_end);
    // slots counted by chunk items: applied from their packed argmax
    const uint64_t applied = L.injective ? S->chunk_end : S->big_end;
    if (applied) k_lp_hub_apply<<<grid_for(applied), kBlock, 0, st>>>(L, applied);
    s->launches += 5;  // + the caller's 2: eff, chunks, groups, CTA hubs, 2 x warp hubs, hub apply
    GXB_CUDA(cudaGetLastError());
    return GXB_OK;
}

// sparse round: cpre = inclusive scan of the frontier's chunk counts (chunk_edges-edge
// chunks of each frontier vertex's CSR row), `units` = the frontier's out-edges
extern "C" int gxb_lp_push(gxb_state* s, cudaStream_t st, const uint32_t* rowpre) {
    if (!s->d_lp_scratch) GXB_CHECK(lp_setup(s, st));
    LpScratch* S = reinterpret_cast<LpScratch*>(s->d_lp_scratch);
    const gxb_graph* g = s->g;
    GXB_CHECK(lp_push_reserve(s, S, 0, st));
    // the pair table holds at most one entry per pushed edge
    uint32_t total = 0;
    if (s->frontier_len) {
        GXB_CUDA(cudaMemcpyAsync(&total, rowpre + s->frontier_len - 1, 4, cudaMemcpyDeviceToHost, st));
        GXB_CUDA(cudaStreamSynchronize(st));
    }
    const uint64_t cap = std::max<uint64_t>(1024, next_pow2(2ull * total + 2));
    GXB_CHECK(lp_push_reserve(s, S, cap, st));
    LpPush P{S->pkeys, S->pcounts, S->pbest, S->ptargets, S->pntargets, cap};
    GXB_CUDA(cudaMemsetAsync(S->pkeys, 0xFF, 8 * cap, st));
    GXB_CUDA(cudaMemsetAsync(S->pcounts, 0, 4 * cap, st));
    GXB_CUDA(cudaMemsetAsync(S->pntargets, 0, 8, st));
    if (total) {
        const uint64_t items = (total + kLpItemEdges - 1) / kLpItemEdges;
        const unsigned grid = grid_for(items * 32, kBlock, 148ull * 16);
        k_lp_push<<<grid, kBlock, 0, st>>>(s->d_frontier[0], s->frontier_len, rowpre, g->d_out_off, g->d_out_dst,
                                           s->d_lab_cur, g->lo, P, cap - 1, S->hot_end);
    }
    k_lp_push_apply<<<grid_for(g->hi - g->lo), kBlock, 0, st>>>(lp_launch(s), P);
    GXB_CUDA(cudaGetLastError());
    return GXB_OK;
}
