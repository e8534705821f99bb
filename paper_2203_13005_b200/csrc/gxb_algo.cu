// gxb_algo.cu — MSGGen / MSGMerge / MSGApply kernels (K1, K2, K4, K5) and the
// per-iteration driver of the device daemon.
//
// Fused path (gxb_iterate): one pull pass over the owned CSC computes, for each
// destination slot, Gen (the per-edge message, A/algorithms.py:102-105,
// 147-149) folded with Merge (A/algorithms.py:107-108, 151-152); Apply
// (A/algorithms.py:113-115, 157-159) follows with change detection, the
// next-frontier bitmap/list and the vote statistics (A/agent.py:404-417,
// A/algorithms.py:327-341). The merge is edge-balanced: every warp owns a fixed
// 256-edge tile of the CSC (k_tile_a: gathers as LDGSTS copies into shared memory;
// k_tile_t: register gathers), runs crossing tiles leave per-tile partials that
// k_span_fold combines in tile order (deterministic PageRank rounding).
//
// SSSP, CC and LP also have a push pass over the CSR for sparse frontiers
// (SURVEY.md §8(f) row 3), edge-balanced over the concatenated frontier rows:
// atomicMin into the next-value array plus a touched bitmap (LP: a (destination,
// label) pair table, gxb_lp.cu); synchronous BSP semantics are kept because every
// message is built from the frozen current values (A/algorithms.py:319-325).
//
// Request path (gxb_request): GEN materialises one message per CSC edge
// (coalesced, edge-parallel), MERGE folds them per destination with a
// degree-binned segmented reduction (groups of 1..32 lanes per destination, warp
// chunks for hubs combined by the last-arriving warp), APPLY runs the vertex
// update — the reference's execute_request over a WorkItem (A/daemon.py:86-130)
// with range descriptors instead of Python triplet blocks.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <type_traits>
#include <vector>

#include <cub/cub.cuh>

#include "gxb_state.cuh"

namespace gxb {

// ======================================================================
// algorithm semantics
// ======================================================================

// Degree rank of a slot within its partition block. Slots are in-degree-sorted per
// partition (a dealt multi-GPU layout starts every block with its hubs); the rank
// selects the L1/L2 residency hint, so an approximate block index is fine:
// q = umulhi(s, magic) ~ s / block, rank = s - q * block.
struct HotPrefix {
    uint32_t block = 0xFFFFFFFFu, magic = 0;
    __device__ __forceinline__ uint32_t rank(uint32_t s) const { return s - __umulhi(s, magic) * block; }
};

struct PrOps {  // PageRank (A/algorithms.py:125-171)
    static constexpr bool kPublishes = false;
    struct Acc {
        double s;
    };
    using Msg = double;
    const double* contrib_cur;
    const double* rank_old;  // rank of the previous round (double-buffered: a speculative round
    double* rank_new;        // leaves the previous state intact until the host commits it)
    double* contrib_next;
    FrontierView f;
    bool msg32;    // messages (rank / out_deg) stored and gathered as float32 (option pr_message_bits = 32)
    int npeers;    // peer replicas written by Apply (fused exchange), next-buffer pointers below
    double* peer_next[kMaxPeers];
    HotPrefix hp;  // degree rank of a slot inside its partition block
    uint32_t hot;  // ranks [0, hot) keep L2 priority (degree-sorted: the most-gathered sources)
    uint32_t hot1; // ranks [0, hot1) also allocate in L1; the rest bypass L1
    const double* hub_sum;  // hub split: per-slot sum of the hub in-edges, added before Apply (or null)

    __device__ static Acc identity() { return {0.0}; }
    __device__ static Acc combine(Acc a, Acc b) { return {a.s + b.s}; }
    __device__ static Acc shfl(Acc a, int off) { return {__shfl_xor_sync(kFull, a.s, off)}; }
    __device__ static Acc shfl_up(Acc a, int d) { return {__shfl_up_sync(kFull, a.s, d)}; }
    __device__ static void st_cg(Acc* p, Acc a) { __stcg(&p->s, a.s); }
    __device__ static Acc ld_cg(const Acc* p) { return {__ldcg(&p->s)}; }
    __device__ static bool has(const Acc&) { return true; }
    // Gen: rank / out_deg of the source (every vertex is active, 144-145)
    static constexpr bool kWeighted = false;
    __device__ bool gen(uint32_t s, uint32_t, Msg& m) const {
        const uint32_t r = hp.rank(s);
        const uint64_t pol = r < hot ? l2_evict_last() : l2_evict_first();
        if (msg32) {
            const float* c = reinterpret_cast<const float*>(contrib_cur) + s;
            m = (double)(r < hot1 ? ld_l1_f32(c, pol) : ld_nol1_f32(c, pol));
        } else {
            m = r < hot1 ? ld_l1_f64(contrib_cur + s, pol) : ld_nol1_f64(contrib_cur + s, pol);
        }
        return true;
    }
    __device__ static void fold(Acc& a, Msg m) { a.s += m; }
    // async-gather interface (k_tile_a): the raw gathered value lands in shared memory
    using Raw = double;
    __device__ static Raw identity_raw() { return 0.0; }
    __device__ bool gather_async(uint32_t saddr, uint32_t s) const {
        const uint32_t r = hp.rank(s);
        const uint64_t pol = r < hot ? l2_evict_last() : l2_evict_first();
        if (msg32) cp_async_ca<4>(saddr, reinterpret_cast<const float*>(contrib_cur) + s, pol);
        else cp_async_ca<8>(saddr, contrib_cur + s, pol);
        return true;
    }
    __device__ Acc from_raw(const Raw* p, uint32_t) const {
        return {msg32 ? (double)*reinterpret_cast<const float*>(p) : *p};
    }
    // Apply: 0.15 + 0.85 * sum with two roundings (157-159; no FMA contraction),
    // convergence_stat |new - old| (161-162), always active.
    struct Pre {
        double old;
        uint32_t od;
    };
    __device__ Pre preload(uint32_t slot) const { return {rank_old[slot], __ldg(f.outdeg + slot)}; }
    __device__ void apply(uint32_t slot, Acc a, LocalStats& st) const { apply_pre(slot, a, preload(slot), st); }
    // returns whether the slot joins the next frontier as a changed vertex (never: always active)
    __device__ bool apply_pre(uint32_t slot, Acc a, Pre p, LocalStats& st) const {
        const double old = p.old;
        // hub split: the hub sources' edges come first in source order (A/algorithms.py:243-251)
        const double sum = hub_sum ? __dadd_rn(hub_sum[slot], a.s) : a.s;
        const double nw = __dadd_rn(0.15, __dmul_rn(0.85, sum));
        rank_new[slot] = nw;
        const uint32_t od = p.od;
        const double c = od ? __ddiv_rn(nw, (double)od) : 0.0;
        if (msg32) {
            const float c32 = __double2float_rn(c);
            reinterpret_cast<float*>(contrib_next)[slot] = c32;
            for (int q = 0; q < npeers; ++q) reinterpret_cast<float*>(peer_next[q])[slot] = c32;
        } else {
            contrib_next[slot] = c;
            for (int q = 0; q < npeers; ++q) peer_next[q][slot] = c;
        }
        if (nw != old) {
            st.changed++;
            st.max_stat = fmax(st.max_stat, fabs(nw - old));
        }
        return false;
    }
};

__device__ __forceinline__ uint4 min4(uint4 a, uint4 b) {
    return make_uint4(min(a.x, b.x), min(a.y, b.y), min(a.z, b.z), min(a.w, b.w));
}
__device__ __forceinline__ bool eq4(uint4 a, uint4 b) {
    return a.x == b.x && a.y == b.y && a.z == b.z && a.w == b.w;
}

// Which sources a pull pass gathers: all (mode 0), the partition's own slots [lo, lo + n)
// (1), or the others (2). A frontier round at N > 1 can run its local-source pass while
// the previous round's records still travel, then the remote-source pass (split rounds).
struct SourceSel {
    uint32_t lo = 0, n = 0;
    int mode = 0;
    __device__ bool take(uint32_t s) const { return mode == 0 || ((s - lo < n) == (mode == 1)); }
};

struct SsspOps {  // multi-source Bellman-Ford, 4 u32 lanes (A/algorithms.py:81-122)
    static constexpr bool kPublishes = true;
    // The accumulator is the lane-wise min; "received a message" <=> some lane is
    // finite: a message comes from an active source, which always holds a finite
    // lane (it changed, or is a source at 0), and the host rejects weights for
    // which d + w could saturate (max_w * |V| >= 2^32 - 1), so no finite sum
    // ever reaches the INF sentinel.
    struct Acc {
        uint4 m;
    };
    using Msg = uint4;
    const uint4* dist_cur;
    uint4* dist_next;
    const uint32_t* active_cur;
    FrontierView f;
    bool commit_inline;  // apply runs in its own kernel after every gather: write cur too, no commit pass
    // Gen from active sources only. A dense pull may skip the bitmap: an inactive source
    // already sent d + w to every out-neighbour the round after it last changed and
    // distances only decrease, so its message never lowers a destination (same values,
    // same changed set) — and the random bitmap read costs as much as the gather.
    bool check_active;
    HotPrefix hp;
    uint32_t hot, hot1;
    SourceSel sel;
    static constexpr bool kWeighted = true;

    __device__ static Acc identity() { return {make_uint4(kInf32, kInf32, kInf32, kInf32)}; }
    __device__ static Acc combine(Acc a, Acc b) { return {min4(a.m, b.m)}; }
    __device__ static Acc shfl(Acc a, int off) {
        return {make_uint4(__shfl_xor_sync(kFull, a.m.x, off), __shfl_xor_sync(kFull, a.m.y, off),
                           __shfl_xor_sync(kFull, a.m.z, off), __shfl_xor_sync(kFull, a.m.w, off))};
    }
    __device__ static Acc shfl_up(Acc a, int d) {
        return {make_uint4(__shfl_up_sync(kFull, a.m.x, d), __shfl_up_sync(kFull, a.m.y, d),
                           __shfl_up_sync(kFull, a.m.z, d), __shfl_up_sync(kFull, a.m.w, d))};
    }
    __device__ static void st_cg(Acc* p, Acc a) { __stcg(&p->m, a.m); }
    __device__ static Acc ld_cg(const Acc* p) { return {__ldcg(&p->m)}; }
    __device__ static bool has(const Acc& a) { return (a.m.x & a.m.y & a.m.z & a.m.w) != kInf32; }
    // Gen: d + w per lane from an active source (102-105); inf stays inf
    __device__ bool gen(uint32_t s, uint32_t w, Msg& m) const {
        if (!sel.take(s) || (check_active && !bit_test(active_cur, s))) return false;
        const uint32_t r = hp.rank(s);
        const uint64_t pol = r < hot ? l2_evict_last() : l2_evict_first();
        const uint4 d = r < hot1 ? ld_l1_v4(dist_cur + s, pol) : ld_nol1_v4(dist_cur + s, pol);
        m = make_uint4(sat_add(d.x, w), sat_add(d.y, w), sat_add(d.z, w), sat_add(d.w, w));
        return true;
    }
    __device__ static void fold(Acc& a, Msg m) { a.m = min4(a.m, m); }
    using Raw = uint4;
    __device__ static Raw identity_raw() { return make_uint4(kInf32, kInf32, kInf32, kInf32); }
    __device__ bool gather_async(uint32_t saddr, uint32_t s) const {
        if (!sel.take(s) || (check_active && !bit_test(active_cur, s))) return false;
        const uint32_t r = hp.rank(s);
        const uint64_t pol = r < hot ? l2_evict_last() : l2_evict_first();
        if (r < hot1) cp_async_ca<16>(saddr, dist_cur + s, pol);
        else cp_async_cg16(saddr, dist_cur + s, pol);
        return true;
    }
    __device__ Acc from_raw(const Raw* p, uint32_t w) const {
        const uint4 d = *p;
        return {make_uint4(sat_add(d.x, w), sat_add(d.y, w), sat_add(d.z, w), sat_add(d.w, w))};
    }
    // Apply: elementwise min, active iff changed (113-115)
    struct Pre {
        uint4 o;
    };
    __device__ Pre preload(uint32_t slot) const { return {dist_cur[slot]}; }
    __device__ void apply(uint32_t slot, Acc a, LocalStats& st) const {
        if (!has(a)) return;
        if (apply_pre(slot, a, preload(slot), st)) publish_changed(f, slot, st);
    }
    // returns whether the slot changed (the caller publishes it to the next frontier)
    __device__ bool apply_pre(uint32_t slot, Acc a, Pre p, LocalStats& st) const {
        if (!has(a)) return false;
        st.targets++;
        const uint4 o = p.o;
        const uint4 n = min4(o, a.m);
        if (eq4(n, o)) return false;
        dist_next[slot] = n;
        if (commit_inline) const_cast<uint4*>(dist_cur)[slot] = n;
        return true;
    }
};

struct CcOps {  // min-label propagation; labels < 0xFFFFFFFF
    static constexpr bool kPublishes = true;
    struct Acc {
        uint32_t m;
    };
    using Msg = uint32_t;
    const uint32_t* lab_cur;
    uint32_t* lab_next;
    const uint32_t* active_cur;
    FrontierView f;
    bool commit_inline;
    bool check_active;  // see SsspOps::check_active (labels only decrease)
    HotPrefix hp;
    uint32_t hot, hot1;
    SourceSel sel;
    static constexpr bool kWeighted = false;

    __device__ static Acc identity() { return {kInf32}; }
    __device__ static Acc combine(Acc a, Acc b) { return {min(a.m, b.m)}; }
    __device__ static Acc shfl(Acc a, int off) { return {__shfl_xor_sync(kFull, a.m, off)}; }
    __device__ static Acc shfl_up(Acc a, int d) { return {__shfl_up_sync(kFull, a.m, d)}; }
    __device__ static void st_cg(Acc* p, Acc a) { __stcg(&p->m, a.m); }
    __device__ static Acc ld_cg(const Acc* p) { return {__ldcg(&p->m)}; }
    __device__ static bool has(const Acc& a) { return a.m != kInf32; }
    __device__ bool gen(uint32_t s, uint32_t, Msg& m) const {
        if (!sel.take(s) || (check_active && !bit_test(active_cur, s))) return false;
        const uint32_t r = hp.rank(s);
        const uint64_t pol = r < hot ? l2_evict_last() : l2_evict_first();
        m = r < hot1 ? ld_l1_u32(lab_cur + s, pol) : ld_nol1_u32(lab_cur + s, pol);
        return true;
    }
    __device__ static void fold(Acc& a, Msg m) { a.m = min(a.m, m); }
    using Raw = uint32_t;
    __device__ static Raw identity_raw() { return kInf32; }
    __device__ bool gather_async(uint32_t saddr, uint32_t s) const {
        if (!sel.take(s) || (check_active && !bit_test(active_cur, s))) return false;
        const uint32_t r = hp.rank(s);
        const uint64_t pol = r < hot ? l2_evict_last() : l2_evict_first();
        cp_async_ca<4>(saddr, lab_cur + s, pol);
        return true;
    }
    __device__ Acc from_raw(const Raw* p, uint32_t) const { return {*p}; }
    struct Pre {
        uint32_t o;
    };
    __device__ Pre preload(uint32_t slot) const { return {lab_cur[slot]}; }
    __device__ void apply(uint32_t slot, Acc a, LocalStats& st) const {
        if (!has(a)) return;
        if (apply_pre(slot, a, preload(slot), st)) publish_changed(f, slot, st);
    }
    __device__ bool apply_pre(uint32_t slot, Acc a, Pre p, LocalStats& st) const {
        if (!has(a)) return false;
        st.targets++;
        const uint32_t o = p.o;
        const uint32_t n = min(o, a.m);
        if (n == o) return false;
        lab_next[slot] = n;
        if (commit_inline) const_cast<uint32_t*>(lab_cur)[slot] = n;
        return true;
    }
};

// ======================================================================
// policies: how an edge contributes to the accumulator, and what happens to
// the folded value of a destination
// ======================================================================

template <class Ops>
struct FusedPolicy {  // Gen∘Merge∘Apply
    Ops ops;
    const uint32_t* in_w;
    using Acc = typename Ops::Acc;
    __device__ void accumulate(Acc& a, uint32_t s, uint64_t e) const {
        typename Ops::Msg m;
        const uint32_t w = (Ops::kWeighted && in_w) ? __ldg(in_w + e) : 1u;
        if (ops.gen(s, w, m)) Ops::fold(a, m);
    }
    __device__ void accumulate_w(Acc& a, uint32_t s, uint32_t w) const {
        typename Ops::Msg m;
        if (ops.gen(s, w, m)) Ops::fold(a, m);
    }
    __device__ void finish(uint32_t slot, Acc a, LocalStats& st) const { ops.apply(slot, a, st); }
};

template <class Ops>
struct MergePolicy {  // MSGMerge over materialised messages
    Ops ops;
    const typename Ops::Msg* msg;
    const uint8_t* valid;
    typename Ops::Acc* merged;  // indexed by slot - lo
    uint64_t lo;
    using Acc = typename Ops::Acc;
    __device__ void accumulate(Acc& a, uint32_t, uint64_t e) const {
        if (valid[e]) Ops::fold(a, msg[e]);
    }
    __device__ void finish(uint32_t slot, Acc a, LocalStats&) const { merged[slot - lo] = a; }
};

// ======================================================================
// the binned pull merge
// ======================================================================

struct PullLaunch {
    uint64_t lo;           // owned slot base
    const uint64_t* in_off;
    const uint32_t* in_src;
    // slot filter (relative), [flo, fhi)
    uint64_t flo, fhi;
    // chunk items
    uint64_t num_items;
    const uint32_t* item_slot;
    const uint64_t* item_begin;
    const uint32_t* item_first;
    const uint32_t* item_count;
    uint32_t* arrive;
    void* partials;
    unsigned chunk_blocks;
    // group bins k = 5..0 (G = 1 << k): relative slot ranges and block counts
    uint64_t bin_lo[kNumGroupBins], bin_hi[kNumGroupBins];
    unsigned bin_blocks[kNumGroupBins];
    StatStripe* stats;
};

template <class Pol>
__device__ __forceinline__ void edge_loop(const Pol& p, const uint32_t* __restrict__ in_src,
                                          typename Pol::Acc& acc, uint64_t e, uint64_t end,
                                          int stride) {
    // four independent index loads, then four gathers: MLP for the random reads
    for (; e + 3ull * stride < end; e += 4ull * stride) {
        const uint32_t s0 = __ldg(in_src + e);
        const uint32_t s1 = __ldg(in_src + e + stride);
        const uint32_t s2 = __ldg(in_src + e + 2ull * stride);
        const uint32_t s3 = __ldg(in_src + e + 3ull * stride);
        p.accumulate(acc, s0, e);
        p.accumulate(acc, s1, e + stride);
        p.accumulate(acc, s2, e + 2ull * stride);
        p.accumulate(acc, s3, e + 3ull * stride);
    }
    for (; e < end; e += stride) p.accumulate(acc, __ldg(in_src + e), e);
}

template <int G, class Pol>
__device__ __forceinline__ void run_group(const Pol& p, const PullLaunch& L, int k, unsigned b,
                                          LocalStats& st) {
    using Ops = decltype(p.ops);
    constexpr int kPerBlock = kBlock / G;
    const int grp = threadIdx.x / G;
    const int gl = threadIdx.x % G;
    const uint64_t rel = L.bin_lo[k] + (uint64_t)b * kPerBlock + grp;
    const bool valid = rel < L.bin_hi[k] && rel >= L.flo && rel < L.fhi;
    uint64_t beg = 0, end = 0;
    if (valid) {
        beg = __ldg(L.in_off + rel);
        end = __ldg(L.in_off + rel + 1);
    }
    auto acc = Ops::identity();
    edge_loop(p, L.in_src, acc, beg + gl, end, G);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc = Ops::combine(acc, Ops::shfl(acc, o));
    if (valid && gl == 0) p.finish((uint32_t)(L.lo + rel), acc, st);
}

template <class Pol>
__device__ __forceinline__ void run_item(const Pol& p, const PullLaunch& L, uint64_t item,
                                         LocalStats& st) {
    using Ops = decltype(p.ops);
    using Acc = typename Ops::Acc;
    const int lane = threadIdx.x & 31;
    const uint32_t rel = __ldg(L.item_slot + item);
    const bool valid = rel >= L.flo && rel < L.fhi;
    if (!valid) return;  // warp-uniform
    const uint64_t beg = __ldg(L.item_begin + item);
    const uint64_t seg_end = __ldg(L.in_off + rel + 1);
    const uint64_t end = min(beg + (uint64_t)kChunkEdges, seg_end);
    Acc acc = Ops::identity();
    edge_loop(p, L.in_src, acc, beg + lane, end, 32);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = Ops::combine(acc, Ops::shfl(acc, o));
    const uint32_t count = __ldg(L.item_count + item);
    if (count == 1) {
        if (lane == 0) p.finish((uint32_t)(L.lo + rel), acc, st);
        return;
    }
    Acc* partials = reinterpret_cast<Acc*>(L.partials);
    unsigned last = 0;
    if (lane == 0) {
        Ops::st_cg(partials + item, acc);
        __threadfence();
        last = (atomicAdd(L.arrive + rel, 1u) == count - 1) ? 1u : 0u;
    }
    last = __shfl_sync(kFull, last, 0);
    if (!last) return;
    __threadfence();
    // the last warp folds the chunk partials of this slot in item order
    const uint32_t first = __ldg(L.item_first + item);
    Acc tot = Ops::identity();
    for (uint32_t i = lane; i < count; i += 32) tot = Ops::combine(tot, Ops::ld_cg(partials + first + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot = Ops::combine(tot, Ops::shfl(tot, o));
    if (lane == 0) {
        L.arrive[rel] = 0u;  // reset for the next pass
        p.finish((uint32_t)(L.lo + rel), tot, st);
    }
}

template <class Pol>
__global__ void __launch_bounds__(kBlock) k_pull(const Pol p, const PullLaunch L) {
    LocalStats st;
    unsigned b = blockIdx.x;
    if (b < L.chunk_blocks) {
        const uint64_t item = (uint64_t)b * (kBlock / 32) + (threadIdx.x >> 5);
        if (item < L.num_items) run_item(p, L, item, st);
    } else {
        b -= L.chunk_blocks;
        int k = kNumGroupBins - 1;
        for (; k > 0; --k) {
            if (b < L.bin_blocks[k]) break;
            b -= L.bin_blocks[k];
        }
        switch (k) {
            case 5: run_group<32>(p, L, 5, b, st); break;
            case 4: run_group<16>(p, L, 4, b, st); break;
            case 3: run_group<8>(p, L, 3, b, st); break;
            case 2: run_group<4>(p, L, 2, b, st); break;
            case 1: run_group<2>(p, L, 1, b, st); break;
            default: run_group<1>(p, L, 0, b, st); break;
        }
    }
    flush_stats(st, L.stats);
}

// ======================================================================
// the edge-balanced pull merge ("warp tiles", merge-path style)
//
// Warp w owns tile t = 256 consecutive CSC edges (tiles restart at exchange-chunk
// boundaries); lane l gathers edges 32 j + l (one instruction covers 32 consecutive
// edges), the values are transposed through shared memory so lane l then folds the
// kTileK consecutive edges 8 l .. 8 l + 7 (Merge), cutting runs at the precomputed
// segment-end mask. Runs crossing lanes are combined by a segmented warp scan keyed
// by slot (the keys are monotone); runs crossing tiles ("spans") write a per-tile
// partial that k_span_fold folds in tile order, so the fold order — and therefore
// the PageRank rounding — is deterministic.
// ======================================================================

struct TileLaunch {
    uint64_t num_tiles;   // end of the tile range of this launch
    uint64_t tile_begin;  // first tile of this launch (an exchange chunk)
    uint64_t owned_edges;
    const uint64_t* in_off;
    const uint32_t* in_src;
    const uint64_t* tile_start;
    const uint32_t* lane_slot;
    const uint8_t* lane_mask;
    const uint32_t* in_w;
    const uint32_t* in_sw;  // packed (src << sw_shift) | w, or nullptr
    uint32_t sw_shift;
    const uint32_t* tile_head;
    const uint32_t* tile_tail;
    const uint32_t* span_first;
    const uint32_t* span_count;
    const uint64_t* span_pbase;
    const uint32_t* span_slot;
    void* partials;
    void* sums;   // per relative slot: folded accumulator
    const uint32_t* key_slot;  // compacted plan (PageRank hub split): plan key -> owned slot, else null
    bool accumulate;  // combine into the sums of an earlier pass over the same plan (split rounds)
};

__device__ __forceinline__ uint4 ldg_v4(const uint32_t* p) { return __ldg(reinterpret_cast<const uint4*>(p)); }

template <class Pol>
__device__ __forceinline__ void tile_emit(const Pol& p, const TileLaunch& L, uint64_t t, uint32_t head,
                                          uint32_t tail, uint32_t key, typename Pol::Acc total) {
    using Ops = decltype(p.ops);
    using Acc = typename Ops::Acc;
    uint32_t span = kNone;
    if (L.key_slot) key = __ldg(L.key_slot + key);  // span_slot holds owned slots in that case
    if (head != kNone && key == __ldg(L.span_slot + head)) span = head;
    else if (tail != kNone && key == __ldg(L.span_slot + tail)) span = tail;
    if (span == kNone) {
        Acc* d = reinterpret_cast<Acc*>(L.sums) + key;
        *d = L.accumulate ? Ops::combine(*d, total) : total;
    } else {
        // folded by k_span_fold after the kernel boundary (no fences on the hot path)
        reinterpret_cast<Acc*>(L.partials)[__ldg(L.span_pbase + span) + (t - __ldg(L.span_first + span))] = total;
    }
}

// Transposed variant: lane l gathers edges e_tile + 32 j + l (j < kTileK), so one
// gather instruction covers 32 CONSECUTIVE edges. Inside a high-degree segment the
// sources are sorted, and in the degree-sorted hot prefix consecutive sources sit
// in the same 32-byte sectors: L1 merges those lanes into one L2 request. The
// values are transposed through shared memory (row padding 1 per kTileK keeps
// both sides bank-friendly) and then folded by the same per-lane run logic.
__device__ __forceinline__ uint32_t tpos(uint32_t p) { return p + (p >> 3); }

template <class Pol, int kMinBlocks>
__global__ void __launch_bounds__(kBlock, kMinBlocks) k_tile_t(const Pol p, const TileLaunch L) {
    using Ops = decltype(p.ops);
    using Acc = typename Ops::Acc;
    constexpr bool kW = Ops::kWeighted;
    constexpr uint32_t kRow = kTileEdges + kTileEdges / kTileK;
    __shared__ Acc sbuf[kBlock / 32][kRow];
    const int lane = threadIdx.x & 31;
    Acc* buf = sbuf[threadIdx.x >> 5];
    const uint64_t nwarps = (uint64_t)gridDim.x * (kBlock / 32);
    const uint64_t pol = l2_evict_first();
    const bool weighted = kW && L.in_w != nullptr;
    const bool packed = kW && L.in_sw != nullptr;
    uint64_t t = L.tile_begin + (uint64_t)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
    uint32_t nidx[kTileK], nw[kTileK];
    uint32_t nsa = 0, nmask = 0;
    uint64_t nbeg = 0, nend = 0;
#pragma unroll
    for (int j = 0; j < kTileK; ++j) {
        nidx[j] = 0;
        nw[j] = 1;
    }
    auto prefetch = [&](uint64_t tt) {
        nbeg = __ldg(L.tile_start + tt);  // tiles restart at every exchange chunk
        nend = __ldg(L.tile_start + tt + 1);
        const uint64_t e = nbeg + (uint64_t)lane;
        if (packed) {  // one stream: source and weight in one word
            const uint32_t wmask = (1u << L.sw_shift) - 1u;
#pragma unroll
            for (int j = 0; j < kTileK; ++j) {
                const uint32_t x = ld_stream_u32(L.in_sw + e + 32 * j, pol);
                nidx[j] = x >> L.sw_shift;
                nw[j] = x & wmask;
            }
        } else {
#pragma unroll
            for (int j = 0; j < kTileK; ++j) nidx[j] = ld_stream_u32(L.in_src + e + 32 * j, pol);
            if (weighted) {
#pragma unroll
                for (int j = 0; j < kTileK; ++j) nw[j] = ld_stream_u32(L.in_w + e + 32 * j, pol);
            }
        }
        nsa = ld_stream_u32(L.lane_slot + tt * 32 + lane, pol);
        nmask = ld_stream_u8(L.lane_mask + tt * 32 + lane, pol);
    };
    if (t < L.num_tiles) prefetch(t);
    for (; t < L.num_tiles; t += nwarps) {
        const uint64_t et = nbeg, tend = nend;
        uint32_t idx[kTileK], wgt[kTileK];
#pragma unroll
        for (int j = 0; j < kTileK; ++j) {
            idx[j] = nidx[j];
            wgt[j] = nw[j];
        }
        const uint32_t sa = nsa;
        uint32_t endmask = nmask;
        if (t + nwarps < L.num_tiles) prefetch(t + nwarps);
        // Gen: coalesced gathers of 32 consecutive edges per instruction
#pragma unroll
        for (int j = 0; j < kTileK; ++j) {
            Acc v = Ops::identity();
            if (et + 32 * j + lane < tend) p.accumulate_w(v, idx[j], wgt[j]);
            buf[tpos(32 * j + lane)] = v;
        }
        __syncwarp();
        const uint64_t e0 = et + (uint64_t)lane * kTileK;
        const bool live = e0 < tend;
        Acc v[kTileK];
#pragma unroll
        for (int j = 0; j < kTileK; ++j) v[j] = buf[tpos(kTileK * lane + j)];
        __syncwarp();
        const uint32_t nvalid = live ? (uint32_t)min((uint64_t)kTileK, tend - e0) : 0u;
        // the run holding the last valid edge is the lane's last run (it may continue into the
        // next lane); ends past the valid edges do not exist
        endmask &= (1u << nvalid) - 1u;
        if (nvalid) endmask &= ~(1u << (nvalid - 1));
        uint32_t fkey = kNone;
        Acc fval = Ops::identity();
        const bool multi = endmask != 0;
        Acc acc = Ops::identity();
        uint32_t key = sa;
        bool first = true;
#pragma unroll
        for (int j = 0; j < kTileK; ++j) {
            acc = Ops::combine(acc, v[j]);
            if ((endmask >> j) & 1u) {
                if (first) {
                    fkey = key;
                    fval = acc;
                    first = false;
                } else {
                    Acc* d = reinterpret_cast<Acc*>(L.sums) + (L.key_slot ? __ldg(L.key_slot + key) : key);
                    *d = L.accumulate ? Ops::combine(*d, acc) : acc;
                }
                ++key;
                acc = Ops::identity();
            }
        }
        const uint32_t lkey = live ? key : kNone;
        const Acc lval = acc;
        if (!multi) {
            fkey = lkey;
            fval = lval;
        }
        Acc c = lval;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const Acc up = Ops::shfl_up(c, d);
            const uint32_t k = __shfl_up_sync(kFull, lkey, d);
            if (lane >= d && k == lkey) c = Ops::combine(up, c);
        }
        const uint32_t prev_key = __shfl_up_sync(kFull, lkey, 1);
        const Acc prev_c = Ops::shfl_up(c, 1);
        const uint32_t next_first = __shfl_down_sync(kFull, fkey, 1);
        if (multi && live) {
            const Acc tot = (lane > 0 && prev_key == fkey) ? Ops::combine(prev_c, fval) : fval;
            tile_emit(p, L, t, __ldg(L.tile_head + t), __ldg(L.tile_tail + t), fkey, tot);
        }
        if (lkey != kNone && (lane == 31 || next_first != lkey))
            tile_emit(p, L, t, __ldg(L.tile_head + t), __ldg(L.tile_tail + t), lkey, c);
    }
}

// Async-gather variant: the kTileK gathers of a lane are LDGSTS copies straight into the
// warp's shared row (no registers held while they are in flight), so the kernel fits
// more resident warps without spilling; weights (SSSP) ride in a parallel shared row.
// The fold is the same as k_tile_t's, reading each value when it is combined.
// shared-row position of edge p of a tile: 16-B values use an XOR swizzle (conflict-free
// for both the 32-consecutive-edges writes and the 8-edges-per-lane reads, no padding);
// narrower values use the padded layout of k_tile_t
template <class Raw>
__device__ __forceinline__ uint32_t apos(uint32_t p) {
    if constexpr (sizeof(Raw) == 16) return p ^ ((p >> 3) & 7u);
    else return tpos(p);
}

template <class Pol, int kMinBlocks>
__global__ void __launch_bounds__(kBlock, kMinBlocks) k_tile_a(const Pol p, const TileLaunch L) {
    using Ops = decltype(p.ops);
    using Acc = typename Ops::Acc;
    using Raw = typename Ops::Raw;
    constexpr bool kW = Ops::kWeighted;  // weighted launches always come with the packed stream
    constexpr uint32_t kRow = sizeof(Raw) == 16 ? kTileEdges : kTileEdges + kTileEdges / kTileK;
    __shared__ Raw sraw[kBlock / 32][kRow];
    __shared__ uint8_t swt[kW ? kBlock / 32 : 1][kW ? kTileEdges + kTileEdges / kTileK : 1];
    const uint32_t lane = threadIdx.x & 31;
    Raw* buf = sraw[threadIdx.x >> 5];
    uint8_t* wbuf = swt[kW ? threadIdx.x >> 5 : 0];
    // 32-bit tile / edge indices (the launcher guarantees padded edges < 2^32)
    const uint32_t nwarps = gridDim.x * (kBlock / 32);
    const uint32_t ntiles = (uint32_t)L.num_tiles;
    const uint64_t pol = l2_evict_first();
    const uint32_t shift = kW ? L.sw_shift : 0u;
    const uint32_t* stream = kW ? L.in_sw : L.in_src;
    uint32_t t = (uint32_t)L.tile_begin + blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5);
    uint32_t nidx[kTileK];
    uint32_t nsa = 0, nmask = 0, nbeg = 0, ncnt = 0;
#pragma unroll
    for (int j = 0; j < kTileK; ++j) nidx[j] = 0;
    auto prefetch = [&](uint32_t tt) {
        nbeg = (uint32_t)__ldg(L.tile_start + tt);
        ncnt = (uint32_t)__ldg(L.tile_start + tt + 1) - nbeg;
        const uint32_t* e = stream + nbeg + lane;
#pragma unroll
        for (int j = 0; j < kTileK; ++j) nidx[j] = ld_stream_u32(e + 32 * j, pol);
        nsa = ld_stream_u32(L.lane_slot + (uint64_t)tt * 32 + lane, pol);
        nmask = ld_stream_u8(L.lane_mask + (uint64_t)tt * 32 + lane, pol);
    };
    if (t < ntiles) prefetch(t);
    for (; t < ntiles; t += nwarps) {
        const uint32_t cnt = ncnt;
        // Gen: issue the tile's gathers (32 consecutive edges per instruction) into shared memory
#pragma unroll
        for (int j = 0; j < kTileK; ++j) {
            const uint32_t q = 32 * j + lane;
            const uint32_t pos = apos<Raw>(q);
            bool issued = false;
            if (q < cnt) issued = p.ops.gather_async(smem_addr(buf + pos), nidx[j] >> shift);
            if (!issued) buf[pos] = Ops::identity_raw();
            if (kW) wbuf[tpos(q)] = (uint8_t)(nidx[j] & ((1u << shift) - 1u));
        }
        const uint32_t sa = nsa;
        uint32_t endmask = nmask;
        if (t + nwarps < ntiles) prefetch(t + nwarps);
        cp_async_wait_all();
        __syncwarp();
        const uint32_t q0 = lane * kTileK;
        const bool live = q0 < cnt;
        const uint32_t nvalid = live ? min((uint32_t)kTileK, cnt - q0) : 0u;
        endmask &= (1u << nvalid) - 1u;
        if (nvalid) endmask &= ~(1u << (nvalid - 1));
        uint32_t fkey = kNone;
        Acc fval = Ops::identity();
        const bool multi = endmask != 0;
        Acc acc = Ops::identity();
        uint32_t key = sa;
        bool first = true;
#pragma unroll
        for (int j = 0; j < kTileK; ++j) {
            const uint32_t q = q0 + j;
            acc = Ops::combine(acc, p.ops.from_raw(buf + apos<Raw>(q), kW ? (uint32_t)wbuf[tpos(q)] : 0u));
            if ((endmask >> j) & 1u) {
                if (first) {
                    fkey = key;
                    fval = acc;
                    first = false;
                } else {
                    Acc* d = reinterpret_cast<Acc*>(L.sums) + (L.key_slot ? __ldg(L.key_slot + key) : key);
                    *d = L.accumulate ? Ops::combine(*d, acc) : acc;
                }
                ++key;
                acc = Ops::identity();
            }
        }
        __syncwarp();  // the next tile's copies overwrite the row
        const uint32_t lkey = live ? key : kNone;
        const Acc lval = acc;
        if (!multi) {
            fkey = lkey;
            fval = lval;
        }
        Acc c = lval;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const Acc up = Ops::shfl_up(c, d);
            const uint32_t k = __shfl_up_sync(kFull, lkey, d);
            if (lane >= d && k == lkey) c = Ops::combine(up, c);
        }
        const uint32_t prev_key = __shfl_up_sync(kFull, lkey, 1);
        const Acc prev_c = Ops::shfl_up(c, 1);
        const uint32_t next_first = __shfl_down_sync(kFull, fkey, 1);
        if (multi && live) {
            const Acc tot = (lane > 0 && prev_key == fkey) ? Ops::combine(prev_c, fval) : fval;
            tile_emit(p, L, t, __ldg(L.tile_head + t), __ldg(L.tile_tail + t), fkey, tot);
        }
        if (lkey != kNone && (lane == 31 || next_first != lkey))
            tile_emit(p, L, t, __ldg(L.tile_head + t), __ldg(L.tile_tail + t), lkey, c);
    }
}

// fold the per-tile partials of every span (deterministic: a fixed order per span).
// A warp takes 32 consecutive spans: short spans (< 16 partials) fold sequentially in
// their own lane; long ones (hubs, hundreds of tiles) are folded by the whole warp —
// lane-strided partial folds, then a fixed butterfly — so no lane walks a hub alone.
template <class Ops>
__global__ void __launch_bounds__(kBlock) k_span_fold(const uint32_t* __restrict__ span_slot,
                                                      const uint32_t* __restrict__ span_count,
                                                      const uint64_t* __restrict__ span_pbase, uint64_t span_lo,
                                                      uint64_t span_hi, const typename Ops::Acc* __restrict__ partials,
                                                      typename Ops::Acc* sums, bool accumulate = false) {
    using Acc = typename Ops::Acc;
    constexpr uint32_t kLong = 16;
    const int lane = threadIdx.x & 31;
    // lane l of warp w takes span w + l * nwarps: spans are in slot (= in-degree) order, so
    // the long hub spans at the front land in different warps instead of queueing in one
    const uint64_t nwarps = (uint64_t)gridDim.x * (kBlock / 32);
    const uint64_t w = (blockIdx.x * (uint64_t)kBlock + threadIdx.x) / 32;
    for (uint64_t base = span_lo; base < span_hi; base += 32 * nwarps) {
        const uint64_t k = base + w + (uint64_t)lane * nwarps;
        const uint32_t n = k < span_hi ? span_count[k] : 0u;
        if (n < kLong && k < span_hi) {
            const uint64_t b = span_pbase[k];
            Acc tot = Ops::identity();
            for (uint32_t i = 0; i < n; ++i) tot = Ops::combine(tot, partials[b + i]);
            if (accumulate) tot = Ops::combine(sums[span_slot[k]], tot);
            sums[span_slot[k]] = tot;
        }
        unsigned big = __ballot_sync(kFull, n >= kLong);
        while (big) {
            const int src = __ffs(big) - 1;
            big &= big - 1;
            const uint64_t kk = base + w + (uint64_t)src * nwarps;
            const uint32_t nn = __shfl_sync(kFull, n, src);
            const uint64_t b = span_pbase[kk];
            Acc tot = Ops::identity();
#pragma unroll 8
            for (uint32_t i = lane; i < nn; i += 32) tot = Ops::combine(tot, partials[b + i]);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) tot = Ops::combine(tot, Ops::shfl(tot, o));
            if (lane == 0) sums[span_slot[kk]] = accumulate ? Ops::combine(sums[span_slot[kk]], tot) : tot;
        }
    }
}

// Apply over the folded sums of every owned slot (A/algorithms.py:327-338);
// slots past nz_slots have no in-edge and fold the identity (merged.get(vid, zero)).
template <class Ops>
__global__ void __launch_bounds__(kBlock) k_apply_sums(const Ops ops, const typename Ops::Acc* __restrict__ sums,
                                                        uint64_t lo, uint64_t rlo, uint64_t owned, uint64_t nz,
                                                        StatStripe* stats) {
    // relative slots [rlo, owned); four independent slots per step: all loads before any store.
    // The loop is warp-uniform so changed slots publish with one bitmap OR per word and
    // one frontier reservation per warp.
    constexpr int kU = 4;
    LocalStats st;
    const uint64_t stride = (uint64_t)gridDim.x * kBlock;
    const uint64_t lane = threadIdx.x & 31;
    for (uint64_t r0 = rlo + blockIdx.x * (uint64_t)kBlock + threadIdx.x; r0 - lane < owned; r0 += kU * stride) {
        typename Ops::Acc a[kU];
        typename Ops::Pre pre[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t r = r0 + u * stride;
            a[u] = (r < nz) ? sums[r] : Ops::identity();
            if (r < owned) pre[u] = ops.preload((uint32_t)(lo + r));
        }
        bool ch[kU];
        uint32_t slot[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const uint64_t r = r0 + u * stride;
            slot[u] = (uint32_t)(lo + r);
            ch[u] = r < owned && ops.apply_pre(slot[u], a[u], pre[u], st);
        }
        if constexpr (Ops::kPublishes) publish_changed_warp<kU>(ops.f, slot, ch, st);
    }
    flush_stats(st, stats);  // ends in a block barrier: every thread's peer stores precede ...
    if constexpr (std::is_same<Ops, PrOps>::value) {
        // ... one cumulative system-scope fence per block: peer stores visible before the vote
        if (ops.npeers && threadIdx.x == 0) __threadfence_system();
    }
}

// ======================================================================
// push (SSSP / CC): warp per frontier source over the CSR
// ======================================================================

struct PushLaunch {
    uint64_t lo, hi;
    const uint64_t* out_off;
    const uint32_t* out_dst;
    const uint32_t* out_w;
    const uint32_t* frontier;
    uint64_t nfront;
    uint32_t* touched;  // bitmap over owned slots
    uint32_t* list_next;
    unsigned long long* count_next;
};

// Edge-balanced push: every frontier source is cut into kPushChunk-edge chunks
// (an inclusive scan of chunk counts maps a global chunk id back to its source),
// so a hub with a million out-edges is spread over thousands of warps instead of
// serialising one warp. Each edge relaxes the destination with atomicMin and a
// touched bitmap deduplicates the next frontier.
constexpr uint32_t kPushChunk = 256;

// Inclusive prefix of the frontier's CSR row lengths (rowpre of the edge-balanced push), in
// one pass: decoupled look-back over kScanTile-element tiles. status[0] is the tile ticket
// (tiles run in ticket order, so every predecessor is resident or done), status[1 + t] =
// (flag << 32) | value of tile t, flag 1 = tile aggregate, 2 = inclusive prefix. The caller
// zeroes status[0 .. tiles] first. Row lengths are < 2^32 in total (E < 2^32 per build).
constexpr int kScanItems = 8;
constexpr int kScanTile = kBlock * kScanItems;

__global__ void __launch_bounds__(kBlock) k_push_rowpre(const uint32_t* __restrict__ frontier, uint64_t n,
                                                        const uint64_t* __restrict__ out_off, uint32_t* rowpre,
                                                        unsigned long long* status) {
    __shared__ uint32_t s_tile, s_prefix;
    __shared__ uint32_t s_warp[kBlock / 32];
    if (threadIdx.x == 0) s_tile = (uint32_t)atomicAdd(status, 1ull);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t i0 = (uint64_t)tile * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    uint32_t v[kScanItems];
    uint32_t run = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        uint32_t d = 0;
        if (i0 + j < n) {
            const uint32_t s = __ldg(frontier + i0 + j);
            d = (uint32_t)(__ldg(out_off + s + 1) - __ldg(out_off + s));
        }
        run += d;
        v[j] = run;
    }
    // block scan of the per-thread totals
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < kBlock / 32 ? s_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < kBlock / 32) s_warp[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const uint32_t excl_thread = x - run + (warp ? s_warp[warp - 1] : 0u);
    if (threadIdx.x == 0) {
        const uint32_t agg = s_warp[kBlock / 32 - 1];
        unsigned long long* st = status + 1;
        uint32_t prefix = 0;
        if (tile == 0) {
            atomicExch(st, (2ull << 32) | agg);
        } else {
            atomicExch(st + tile, (1ull << 32) | agg);
            for (int64_t p = (int64_t)tile - 1; p >= 0;) {
                const unsigned long long w = atomicAdd(st + p, 0ull);
                const uint32_t flag = (uint32_t)(w >> 32);
                if (flag == 0) continue;  // predecessor still summing its tile
                prefix += (uint32_t)w;
                if (flag == 2) break;
                --p;
            }
            atomicExch(st + tile, (2ull << 32) | (uint32_t)(prefix + agg));
        }
        s_prefix = prefix;
    }
    __syncthreads();
    const uint32_t base = s_prefix + excl_thread;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j)
        if (i0 + j < n) rowpre[i0 + j] = base + v[j];
}

struct SsspPush {
    const uint4* dist_cur;
    uint4* dist_next;
    using Val = uint4;
    static constexpr int kBatch = 8;  // edges per lane whose loads are issued together (k_push)
    __device__ Val load(uint32_t s) const { return __ldg(dist_cur + s); }
    __device__ bool relax(Val d, uint32_t t, uint32_t w) const {
        const uint4 c = make_uint4(sat_add(d.x, w), sat_add(d.y, w), sat_add(d.z, w), sat_add(d.w, w));
        const uint4 cur = __ldcg(dist_next + t);
        unsigned* p = reinterpret_cast<unsigned*>(dist_next + t);
        bool lowered = false;
        if (c.x < cur.x) lowered |= atomicMin(p + 0, c.x) > c.x;
        if (c.y < cur.y) lowered |= atomicMin(p + 1, c.y) > c.y;
        if (c.z < cur.z) lowered |= atomicMin(p + 2, c.z) > c.z;
        if (c.w < cur.w) lowered |= atomicMin(p + 3, c.w) > c.w;
        return lowered;
    }
};

struct CcPush {
    const uint32_t* lab_cur;
    uint32_t* lab_next;
    using Val = uint32_t;
    static constexpr int kBatch = 1;
    __device__ Val load(uint32_t s) const { return __ldg(lab_cur + s); }
    __device__ bool relax(Val v, uint32_t t, uint32_t) const {
        return v < __ldcg(lab_next + t) && atomicMin(lab_next + t, v) > v;
    }
};

// Edge-balanced over the concatenated CSR rows of the frontier (rowpre = inclusive prefix
// of the row lengths): a warp takes kPushChunk consecutive edges, finds the first one's row
// with one binary search, and each lane walks forward to its own rows, so a frontier of
// millions of short rows costs the same per edge as one hub row.
template <class Op>
__global__ void __launch_bounds__(kBlock) k_push(const Op op, const PushLaunch L, const uint32_t* __restrict__ rowpre) {
    const int lane = threadIdx.x & 31;
    if (L.nfront == 0) return;
    const uint64_t total = rowpre[L.nfront - 1];
    const uint64_t items = (total + kPushChunk - 1) / kPushChunk;
    const uint64_t nwarps = (uint64_t)gridDim.x * (kBlock / 32);
    for (uint64_t it = (uint64_t)blockIdx.x * (kBlock / 32) + (threadIdx.x >> 5); it < items; it += nwarps) {
        const uint64_t g0 = it * kPushChunk, g1 = min(total, g0 + kPushChunk);
        uint64_t a = 0, b = L.nfront - 1;  // row of edge g0: first f with rowpre[f] > g0
        while (a < b) {
            const uint64_t mid = (a + b) >> 1;
            if (__ldg(rowpre + mid) > g0) b = mid; else a = mid + 1;
        }
        uint64_t f = a;
        // Op::kBatch of a lane's edges at a time, their dependent loads level by level (row
        // -> source -> edge -> target, weight): kBatch loads in flight per level, then the
        // relaxes (SSSP: 8, the whole chunk; CC: 1 — its lighter relax lost occupancy to the
        // batch's registers, measured)
        constexpr int kJ = Op::kBatch;
#pragma unroll 1
        for (uint64_t gb = g0 + lane; gb < g1; gb += 32 * kJ) {
            uint64_t ej[kJ];
            uint32_t sj[kJ], tj[kJ], wj[kJ];
            unsigned okm = 0u;
#pragma unroll
            for (int j = 0; j < kJ; ++j) {
                const uint64_t gl = gb + 32 * j;
                if (gl < g1) {
                    okm |= 1u << j;
                    f = row_advance(rowpre, L.nfront, f, gl);
                    ej[j] = f;  // the row for now
                }
            }
#pragma unroll
            for (int j = 0; j < kJ; ++j)
                if ((okm >> j) & 1u) {
                    const uint64_t fj = ej[j];
                    sj[j] = __ldg(L.frontier + fj);
                    ej[j] = (gb + 32 * j) - (fj ? __ldg(rowpre + fj - 1) : 0);
                }
#pragma unroll
            for (int j = 0; j < kJ; ++j)
                if ((okm >> j) & 1u) ej[j] += __ldg(L.out_off + sj[j]);
#pragma unroll
            for (int j = 0; j < kJ; ++j)
                if ((okm >> j) & 1u) {
                    tj[j] = __ldg(L.out_dst + ej[j]);
                    wj[j] = L.out_w ? __ldg(L.out_w + ej[j]) : 1u;
                }
#pragma unroll
            for (int j = 0; j < kJ; ++j)
                if (((okm >> j) & 1u) && op.relax(op.load(sj[j]), tj[j], wj[j]) &&
                    bit_set_atomic(L.touched, (uint32_t)(tj[j] - L.lo)))
                    warp_append(L.list_next, L.count_next, tj[j]);
        }
    }
}

// commit the pushed changes: next -> cur, frontier bookkeeping, stats
template <typename T>
__global__ void __launch_bounds__(kBlock) k_push_apply(T* cur, const T* __restrict__ next,
                                                        const uint32_t* __restrict__ list,
                                                        const unsigned long long* count, FrontierView f,
                                                        StatStripe* stats) {
    LocalStats st;
    const uint64_t n = *count;
    for (uint64_t i = blockIdx.x * (uint64_t)kBlock + threadIdx.x; i < n; i += (uint64_t)gridDim.x * kBlock) {
        const uint32_t s = list[i];
        cur[s] = next[s];
        st.changed++;
        st.targets++;
        st.next_active++;
        st.next_units += __ldg(f.outdeg + s);
        if (bit_test(f.remote_src, s)) st.remote_active++;
        atomicOr(f.active_next + (s >> 5), 1u << (s & 31));
    }
    flush_stats(st, stats);
}

// pull commit: cur[s] = next[s] for the changed slots
template <typename T>
__global__ void k_commit(T* cur, const T* __restrict__ next, const uint32_t* __restrict__ list,
                         const unsigned long long* count) {
    const uint64_t n = *count;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = list[i];
        cur[s] = next[s];
    }
}

// ======================================================================
// request path kernels
// ======================================================================

template <class Ops>
__global__ void k_gen(const Ops ops, const uint32_t* __restrict__ in_src, const uint32_t* __restrict__ in_w,
                      uint64_t elo, uint64_t ehi, typename Ops::Msg* msg, uint8_t* valid) {
    for (uint64_t e = elo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < ehi;
         e += (uint64_t)gridDim.x * blockDim.x) {
        typename Ops::Msg m;
        const uint32_t w = (Ops::kWeighted && in_w) ? __ldg(in_w + e) : 1u;
        const bool ok = ops.gen(__ldg(in_src + e), w, m);
        if (ok) msg[e] = m;
        valid[e] = ok ? 1 : 0;
    }
}

template <class Ops>
__global__ void __launch_bounds__(kBlock) k_apply(const Ops ops, const typename Ops::Acc* __restrict__ merged,
                                                   uint64_t lo, uint64_t slo, uint64_t shi,
                                                   StatStripe* stats) {
    LocalStats st;
    for (uint64_t s = slo + blockIdx.x * (uint64_t)kBlock + threadIdx.x; s < shi; s += (uint64_t)gridDim.x * kBlock)
        ops.apply((uint32_t)s, merged[s - lo], st);
    flush_stats(st, stats);
}

// ======================================================================
// init / readback kernels
// ======================================================================

__global__ void k_pr_init(double* rank, double* contrib, const uint32_t* __restrict__ outdeg,
                          const uint32_t* __restrict__ slot2id, uint64_t V, bool msg32) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < V; s += (uint64_t)gridDim.x * blockDim.x) {
        // initial_attr (A/algorithms.py:141-142); a padding slot starts at its fixed point 0.15
        rank[s] = slot2id[s] == kInf32 ? 0.15 : 1.0;
        const uint32_t od = outdeg[s];
        const double c = od ? __ddiv_rn(1.0, (double)od) : 0.0;
        if (msg32) reinterpret_cast<float*>(contrib)[s] = __double2float_rn(c);
        else contrib[s] = c;
    }
}

__global__ void k_fill_u4(uint4* a, uint64_t n, uint4 v) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n; s += (uint64_t)gridDim.x * blockDim.x)
        a[s] = v;
}

__global__ void k_iota_u32(uint32_t* a, uint64_t lo, uint64_t n) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < n; s += (uint64_t)gridDim.x * blockDim.x)
        a[s] = (uint32_t)(lo + s);
}

__global__ void k_bitmap_range(uint32_t* bm, uint64_t lo, uint64_t hi) {
    for (uint64_t s = lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < hi; s += (uint64_t)gridDim.x * blockDim.x)
        atomicOr(bm + (s >> 5), 1u << (s & 31));
}

__global__ void k_read_attrs(int algo, int arity, const uint32_t* __restrict__ d2s,
                             uint64_t V, uint64_t lo, uint64_t hi, int owned_only, const double* rank,
                             const uint4* dist, const uint32_t* lab, double* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < V; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = d2s[i];
        const bool mine = s >= lo && s < hi;
        if (owned_only && !mine) {
            for (int j = 0; j < arity; ++j) out[i * arity + j] = __longlong_as_double(0x7ff8000000000000ll);
            continue;
        }
        if (algo == GXB_ALGO_PAGERANK) {
            out[i] = rank[s];
        } else if (algo == GXB_ALGO_SSSP) {
            const uint4 d = dist[s];
            const uint32_t l[4] = {d.x, d.y, d.z, d.w};
            for (int j = 0; j < arity; ++j)
                out[i * arity + j] = (l[j] == kInf32) ? __longlong_as_double(0x7ff0000000000000ll) : (double)l[j];
        } else {
            out[i] = (double)lab[s];
        }
    }
}

// attributes in ascending-id order -> slots (the agent's pull_from_upper)
// Frontier algorithms: an installed value that differs from the current one is a change the
// next round must propagate — the vertex joins the frontier (active bit, list, GEN units),
// like a received exchange record; raising a distance / label is flagged (raised).
struct InstallMarks {
    uint32_t* active = nullptr;          // nullptr: PageRank (every vertex is active anyway)
    uint32_t* list = nullptr;
    unsigned long long* count = nullptr;
    unsigned long long* units = nullptr;
    unsigned long long* raised = nullptr;
};

__device__ __forceinline__ void mark_installed(const InstallMarks& m, uint32_t s, const uint32_t* outdeg,
                                               bool raised) {
    if (!m.active) return;
    if (bit_set_atomic(m.active, s)) {
        m.list[atomicAdd(m.count, 1ull)] = s;
        atomicAdd(m.units, (unsigned long long)outdeg[s]);
    }
    if (raised) atomicOr(m.raised, 1ull);
}

__global__ void k_write_attrs(int algo, int arity, const uint32_t* __restrict__ d2s, uint64_t V,
                              const uint32_t* __restrict__ outdeg, const double* __restrict__ in, double* rank,
                              double* contrib, uint4* dist_cur, uint4* dist_next, uint32_t* lab_cur,
                              uint32_t* lab_next, uint32_t* bad, bool msg32, InstallMarks marks) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < V; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = d2s[i];
        if (algo == GXB_ALGO_PAGERANK) {
            const double r = in[i];
            rank[s] = r;
            const uint32_t od = outdeg[s];
            const double c = od ? __ddiv_rn(r, (double)od) : 0.0;
            if (msg32) reinterpret_cast<float*>(contrib)[s] = __double2float_rn(c);
            else contrib[s] = c;
        } else if (algo == GXB_ALGO_SSSP) {
            uint32_t l[4] = {kInf32, kInf32, kInf32, kInf32};
            for (int j = 0; j < arity; ++j) {
                const double x = in[i * arity + j];
                if (isinf(x) && x > 0) continue;
                if (!(x >= 0.0 && x < 4294967295.0 && x == floor(x))) atomicOr(bad, 1u);
                else l[j] = (uint32_t)x;
            }
            const uint4 v = make_uint4(l[0], l[1], l[2], l[3]);
            const uint4 o = dist_cur[s];
            dist_cur[s] = v;
            dist_next[s] = v;
            if (v.x != o.x || v.y != o.y || v.z != o.z || v.w != o.w)
                mark_installed(marks, s, outdeg, v.x > o.x || v.y > o.y || v.z > o.z || v.w > o.w);
        } else {
            const double x = in[i];
            if (!(x >= 0.0 && x < 4294967295.0 && x == floor(x))) {
                atomicOr(bad, 1u);
            } else {
                const uint32_t o = lab_cur[s], v = (uint32_t)x;
                lab_cur[s] = v;
                lab_next[s] = v;
                if (v != o) mark_installed(marks, s, outdeg, v > o);
            }
        }
    }
}

}  // namespace gxb

using namespace gxb;

// ======================================================================
// host side
// ======================================================================

namespace {

FrontierView frontier_view(gxb_state* s) {
    const gxb_graph* g = s->g;
    FrontierView f;
    f.lo = g->lo;
    f.outdeg = g->d_outdeg;
    f.remote_src = g->d_remote_src;
    f.active_next = s->d_active[1];
    f.frontier_next = s->d_frontier[1];
    f.frontier_count = s->d_fcount + 1;
    return f;
}

PullLaunch pull_launch(gxb_state* s, uint64_t flo, uint64_t fhi) {
    const gxb_graph* g = s->g;
    const PullPlan& P = g->plan;
    PullLaunch L;
    std::memset(&L, 0, sizeof(L));
    L.lo = g->lo;
    L.in_off = g->d_in_off;
    L.in_src = g->d_in_src;
    L.flo = flo;
    L.fhi = fhi;
    L.num_items = P.num_items;
    L.item_slot = P.d_item_slot;
    L.item_begin = P.d_item_begin;
    L.item_first = P.d_item_first;
    L.item_count = P.d_item_count;
    L.arrive = P.d_slot_arrive;
    L.partials = s->d_partials;
    L.chunk_blocks = (unsigned)((P.num_items + (kBlock / 32) - 1) / (kBlock / 32));
    uint64_t prev = P.chunk_end;
    for (int k = kNumGroupBins - 1; k >= 0; --k) {
        L.bin_lo[k] = prev;
        L.bin_hi[k] = std::max(prev, P.group_end[k]);
        const uint64_t n = L.bin_hi[k] - L.bin_lo[k];
        const uint64_t per = kBlock >> k;
        L.bin_blocks[k] = (unsigned)((n + per - 1) / per);
        prev = L.bin_hi[k];
    }
    L.stats = s->d_stats;
    return L;
}

unsigned pull_grid(const PullLaunch& L) {
    unsigned n = L.chunk_blocks;
    for (int k = 0; k < kNumGroupBins; ++k) n += L.bin_blocks[k];
    return n;
}

template <class Pol>
int launch_pull(const Pol& p, const PullLaunch& L, cudaStream_t st) {
    const unsigned grid = pull_grid(L);
    if (grid) k_pull<Pol><<<grid, kBlock, 0, st>>>(p, L);
    GXB_CUDA(cudaGetLastError());
    return GXB_OK;
}

TileLaunch tile_launch(gxb_state* s) {
    const gxb_graph* g = s->g;
    const TilePlan& T = g->tiles;
    TileLaunch L;
    L.num_tiles = T.num_tiles;
    L.tile_begin = 0;
    L.owned_edges = g->owned_edges;
    L.in_off = g->d_in_off;
    L.in_src = g->d_in_src;
    L.tile_start = T.d_tile_start;
    L.lane_slot = T.d_lane_slot;
    L.lane_mask = T.d_lane_mask;
    L.in_w = g->d_in_w;
    L.in_sw = g->d_in_sw;
    L.sw_shift = g->sw_shift;
    L.tile_head = T.d_tile_head;
    L.tile_tail = T.d_tile_tail;
    L.span_first = T.d_span_first;
    L.span_count = T.d_span_count;
    L.span_pbase = T.d_span_pbase;
    L.span_slot = T.d_span_slot;
    L.partials = s->d_tile_partials;
    L.sums = s->d_sums;
    L.key_slot = nullptr;
    L.accumulate = false;
    return L;
}

// the timing event i of the open round: the fixed triple, or the ring slot in async mode
cudaEvent_t kev_at(gxb_state* s, int i) {
    if (!s->async_stats || !s->kring) return s->kev[i];
    return s->kring[(s->kring_n % gxb_state::kRing) * 3 + i];
}

// accumulate the first n recorded ring rounds into the profile counters
int drain_kring(gxb_state* s, int n) {
    for (int r = 0; r < n; ++r) {
        cudaEvent_t* e = s->kring + (r % gxb_state::kRing) * 3;
        float ms = 0.f;
        GXB_CUDA(cudaEventSynchronize(e[2]));
        GXB_CUDA(cudaEventElapsedTime(&ms, e[0], e[1]));
        s->kernel_ms += ms;
        GXB_CUDA(cudaEventElapsedTime(&ms, e[1], e[2]));
        s->rest_ms += ms;
        s->kernel_launches++;
    }
    return GXB_OK;
}

// one exchange chunk (or all of them for k < 0): Gen∘Merge tiles, span folds, Apply
// With `ast`, the chunk's span fold and Apply run on that stream after the tile kernel
// (an event orders them), so Apply(k) — and its peer stores — overlap the tiles of k+1.
// pass: 0 = a whole round; 1 = a split round's local-source tiles and span folds (no
// Apply, a few SMs left to the exchange kernels beside it); 2 = its remote-source tiles
// and folds combined into pass 1's sums, then Apply
template <class Ops>
int launch_tile_and_apply(gxb_state* s, const Ops& ops, cudaStream_t st, int chunk = -1,
                          cudaStream_t ast = nullptr, int pass = 0) {
    const gxb_graph* g = s->g;
    const TilePlan& T = g->tiles;
    const int K = T.num_xchunks;
    const int k0 = chunk < 0 ? 0 : chunk, k1 = chunk < 0 ? K : chunk + 1;
    TileLaunch L = tile_launch(s);
    L.tile_begin = T.xchunk_tile[k0];
    L.num_tiles = T.xchunk_tile[k1];
    L.accumulate = pass == 2;
    const uint64_t span_lo = T.xchunk_span[k0], span_hi = T.xchunk_span[k1];
    const uint64_t r_lo = T.xchunk_slot[k0], r_hi = T.xchunk_slot[k1];
    FusedPolicy<Ops> p{ops, g->d_in_w};
    // measured best min-blocks per accumulator width (PR/CC 6, SSSP 4); 0 = auto
    int variant = (int)options().tile_minblocks;
    if (variant == 0) variant = (sizeof(typename Ops::Acc) >= 16) ? 4 : 6;
    using Pol = FusedPolicy<Ops>;
    void (*kern)(const Pol, const TileLaunch) = (variant == 8) ? k_tile_t<Pol, 8> : (variant == 6) ? k_tile_t<Pol, 6>
             : (variant == 4) ? k_tile_t<Pol, 4> : k_tile_t<Pol, 1>;
    // LDGSTS gathers; weighted launches need the packed index+weight stream with <= 8 weight bits
    const bool async_ok = (!Ops::kWeighted || (g->d_in_sw && g->sw_shift <= 8)) &&
                          L.num_tiles * (uint64_t)kTileEdges + kTileEdges < (1ull << 32);
    if (options().tile_async && async_ok) {  // min-blocks from the option, or the measured best
        int av = options().tile_async_minblocks;
        if (av == 0) av = sizeof(typename Ops::Raw) >= 16 ? 4 : sizeof(typename Ops::Raw) == 8 ? 6 : 5;
        kern = (av == 8) ? k_tile_a<Pol, 8> : (av == 6) ? k_tile_a<Pol, 6> : (av == 5) ? k_tile_a<Pol, 5>
             : (av == 4) ? k_tile_a<Pol, 4> : k_tile_a<Pol, 1>;
    }
    if (options().carveout >= 0)  // shared-memory carveout (% of max): the rest of the 256 KB is L1
        GXB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, (int)options().carveout));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, 0);
    // chunked rounds leave SMs free for the NCCL kernels of the overlapped exchange
    const int sms = chunk >= 0  ? std::max(1, kNumSMs - (int)options().overlap_reserve_sms)
                    : pass == 1 ? std::max(1, kNumSMs - (int)options().split_reserve_sms)
                                : kNumSMs;
    const int max_blocks = std::max(1, per_sm) * sms;
    const uint64_t ntiles = L.num_tiles - L.tile_begin;
    if (ntiles) {
        const uint64_t want = (ntiles + (kBlock / 32) - 1) / (kBlock / 32);
        const unsigned grid = (unsigned)std::min<uint64_t>(want, (uint64_t)max_blocks);
        const bool first = pass != 1 && (chunk < 0 || s->round_chunks == 0);
        const bool last = pass != 1 && (chunk < 0 || s->round_chunks == K - 1);
        if (s->timing && first) GXB_CUDA(cudaEventRecord(kev_at(s, 0), st));
        kern<<<grid, kBlock, 0, st>>>(p, L);
        if (s->timing && last) {
            GXB_CUDA(cudaEventRecord(kev_at(s, 1), st));
            s->timing_pending = true;
        }
        s->launches++;
    }
    if (chunk >= 0) s->round_chunks++;
    if (ast) {
        GXB_CUDA(cudaEventRecord(s->ev_tile, st));
        GXB_CUDA(cudaStreamWaitEvent(ast, s->ev_tile, 0));
        st = ast;
    }
    if (ntiles) {
        if (span_hi > span_lo) {
            k_span_fold<Ops><<<grid_for(span_hi - span_lo), kBlock, 0, st>>>(
                T.d_span_slot, T.d_span_count, T.d_span_pbase, span_lo, span_hi,
                (const typename Ops::Acc*)s->d_tile_partials, (typename Ops::Acc*)s->d_sums, pass == 2);
            s->launches++;
        }
    }
    if (pass == 1) {
        GXB_CUDA(cudaGetLastError());
        return GXB_OK;
    }
    Ops aops = ops;
    if constexpr (!std::is_same<Ops, PrOps>::value) {
        aops.commit_inline = true;  // every gather of the round is done: commit changes in place
        s->committed_inline = true;
    }
    if (r_hi > r_lo) {
        k_apply_sums<Ops><<<grid_for(r_hi - r_lo), kBlock, 0, st>>>(aops, (const typename Ops::Acc*)s->d_sums,
                                                                     g->lo, r_lo, r_hi, T.nz_slots, s->d_stats);
        s->launches++;
    }
    GXB_CUDA(cudaGetLastError());
    return GXB_OK;
}

// ======================================================================
// PageRank hub split (option pr_hub_slots, one partition)
// ======================================================================
// CSC segments are source-sorted, so the in-edges of a destination that come from the
// H first slots (the highest IN-degree vertices of the degree-sorted order; on R-MAT they are
// also the highest out-degree ones) are a prefix of its
// segment. Those "hub" edges are summed from a shared-memory copy of contrib[0, H)
// (one table per SM, LDS instead of an L1 data-pipe wavefront per gathered element); the
// remaining "cold" edges run the LDGSTS tile kernel. Both CSCs are compacted to their
// non-empty destinations and planned with the same warp tiles; plan keys map back to
// owned slots through d_split_slot.
constexpr int kHubBlock = 1024;
PrOps pr_ops(gxb_state* s);

// per destination slot: number of in-edges from sources < H (lower bound in its segment)
__global__ void k_hub_count(const uint64_t* __restrict__ off, const uint32_t* __restrict__ src, uint64_t nz,
                            uint32_t H, uint32_t* hcnt) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < nz; r += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lo = off[r], hi = off[r + 1];
        const uint64_t b = lo;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (src[mid] < H) lo = mid + 1; else hi = mid;
        }
        hcnt[r] = (uint32_t)(lo - b);
    }
}

// copy the selected part of each listed destination's segment into the compacted CSC
// (warp per destination); hub = the prefix [0, hcnt), cold = the rest
__global__ void k_split_copy(const uint64_t* __restrict__ off, const uint32_t* __restrict__ src,
                             const uint32_t* __restrict__ hcnt, const uint32_t* __restrict__ list, uint64_t n,
                             const uint64_t* __restrict__ coff, int hub, uint32_t* out) {
    const uint64_t lane = threadIdx.x & 31;
    const uint64_t w0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t i = w0; i < n; i += nw) {
        const uint32_t r = list[i];
        const uint64_t b = off[r] + (hub ? 0 : hcnt[r]);
        const uint64_t c = coff[i + 1] - coff[i];
        for (uint64_t k = lane; k < c; k += 32) out[coff[i] + k] = src[b + k];
    }
}

__global__ void k_remap_u32(uint32_t* a, uint64_t n, const uint32_t* __restrict__ map) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = map[a[i]];
}

// hub pass: the tile kernel's segmented fold over the compacted hub CSC, values from the
// shared-memory table (each lane reads its own kTileK consecutive indices: two 16-B loads)
__global__ void __launch_bounds__(kHubBlock, 1) k_tile_hub(const double* __restrict__ contrib, uint32_t H,
                                                            const TileLaunch L) {
    extern __shared__ double tab[];
    for (uint32_t i = threadIdx.x; i < H; i += kHubBlock) tab[i] = __ldcg(contrib + i);
    __syncthreads();
    using Ops = PrOps;
    using Acc = PrOps::Acc;
    const FusedPolicy<PrOps> p{};
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t nwarps = gridDim.x * (kHubBlock / 32);
    const uint32_t ntiles = (uint32_t)L.num_tiles;
    const uint32_t q0 = lane * kTileK;
    // one tile ahead: its indices and lane descriptors load while this tile folds
    uint4 na = make_uint4(0, 0, 0, 0), nb = na;
    uint32_t ncnt = 0, nsa = 0, nmask = 0;
    auto prefetch = [&](uint32_t tt) {
        const uint32_t b0 = (uint32_t)__ldg(L.tile_start + tt);
        ncnt = (uint32_t)__ldg(L.tile_start + tt + 1) - b0;
        nsa = __ldg(L.lane_slot + (uint64_t)tt * 32 + lane);
        nmask = __ldg(L.lane_mask + (uint64_t)tt * 32 + lane);
        if (q0 < ncnt) {
            na = ldg_v4(L.in_src + b0 + q0);
            nb = ldg_v4(L.in_src + b0 + q0 + 4);
        }
    };
    uint32_t t = blockIdx.x * (kHubBlock / 32) + (threadIdx.x >> 5);
    if (t < ntiles) prefetch(t);
    for (; t < ntiles; t += nwarps) {
        const uint32_t cnt = ncnt;
        const uint32_t sa = nsa;
        uint32_t endmask = nmask;
        const uint4 a = na, b = nb;
        if (t + nwarps < ntiles) prefetch(t + nwarps);
        const bool live = q0 < cnt;
        const uint32_t nvalid = live ? min((uint32_t)kTileK, cnt - q0) : 0u;
        double v[kTileK];
        if (live) {
            const uint32_t idx[kTileK] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int j = 0; j < kTileK; ++j) v[j] = ((uint32_t)j < nvalid) ? tab[idx[j]] : 0.0;
        } else {
#pragma unroll
            for (int j = 0; j < kTileK; ++j) v[j] = 0.0;
        }
        endmask &= (1u << nvalid) - 1u;
        if (nvalid) endmask &= ~(1u << (nvalid - 1));
        uint32_t fkey = kNone;
        Acc fval = Ops::identity();
        const bool multi = endmask != 0;
        Acc acc = Ops::identity();
        uint32_t key = sa;
        bool first = true;
#pragma unroll
        for (int j = 0; j < kTileK; ++j) {
            acc = Ops::combine(acc, Acc{v[j]});
            if ((endmask >> j) & 1u) {
                if (first) {
                    fkey = key;
                    fval = acc;
                    first = false;
                } else {
                    reinterpret_cast<Acc*>(L.sums)[__ldg(L.key_slot + key)] = acc;
                }
                ++key;
                acc = Ops::identity();
            }
        }
        const uint32_t lkey = live ? key : kNone;
        const Acc lval = acc;
        if (!multi) {
            fkey = lkey;
            fval = lval;
        }
        Acc c = lval;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const Acc up = Ops::shfl_up(c, d);
            const uint32_t k = __shfl_up_sync(kFull, lkey, d);
            if (lane >= d && k == lkey) c = Ops::combine(up, c);
        }
        const uint32_t prev_key = __shfl_up_sync(kFull, lkey, 1);
        const Acc prev_c = Ops::shfl_up(c, 1);
        const uint32_t next_first = __shfl_down_sync(kFull, fkey, 1);
        if (multi && live) {
            const Acc tot = (lane > 0 && prev_key == fkey) ? Ops::combine(prev_c, fval) : fval;
            tile_emit(p, L, t, __ldg(L.tile_head + t), __ldg(L.tile_tail + t), fkey, tot);
        }
        if (lkey != kNone && (lane == 31 || next_first != lkey))
            tile_emit(p, L, t, __ldg(L.tile_head + t), __ldg(L.tile_tail + t), lkey, c);
    }
}

void pr_split_free(gxb_state* s) {
    for (int k = 0; k < 2; ++k) {
        shadow_graph_free(s->split_g[k]);
        s->split_g[k] = nullptr;
        dfree(s->d_split_slot[k]);
        dfree(s->d_split_partials[k]);
        dfree(s->d_split_sum[k]);
        s->d_split_slot[k] = nullptr;
        s->d_split_partials[k] = nullptr;
        s->d_split_sum[k] = nullptr;
    }
    s->hub_n = 0;
}

bool pr_split_wanted(const gxb_state* s) {
    const gxb_graph* g = s->g;
    return s->algo == GXB_ALGO_PAGERANK && options().pr_hub_slots > 0 && g->nparts == 1 && !s->msg32 &&
           s->npeers == 0 && !options().pipeline_apply && g->tiles.num_xchunks == 1 && g->S > 0;
}

// build the hub / cold compacted CSCs and their tile plans (once per state and H)
int pr_split_prepare(gxb_state* s, cudaStream_t st) {
    gxb_graph* g = s->g;
    const uint32_t H = (uint32_t)std::min<uint64_t>((uint64_t)options().pr_hub_slots, g->S);
    if (s->hub_n == H && s->split_g[0]) return GXB_OK;
    pr_split_free(s);
    const uint64_t nz = g->tiles.nz_slots;
    const uint64_t owned = g->hi - g->lo;
    uint32_t* d_hcnt = nullptr;
    struct Scratch {  // freed on every exit path (GXB_CHECK returns early)
        uint32_t*& p;
        ~Scratch() { dfree(p); }
    } scratch{d_hcnt};
    GXB_CHECK(dalloc_t(&d_hcnt, nz + 1));
    if (nz) k_hub_count<<<grid_for(nz), kBlock, 0, st>>>(g->d_in_off, g->d_in_src, nz, H, d_hcnt);
    std::vector<uint32_t> hcnt(nz);
    if (nz) GXB_CUDA(cudaMemcpyAsync(hcnt.data(), d_hcnt, 4 * nz, cudaMemcpyDeviceToHost, st));
    GXB_CUDA(cudaStreamSynchronize(st));
    const std::vector<uint32_t>& deg = g->h_indeg_sorted;
    // one compacted CSC (k = 0 cold, 1 hub); an early error return leaves the lambda only, so
    // every failure reaches the single cleanup below (sync, then pr_split_free)
    auto build_one = [&](int k) -> int {
        const bool hub = k == 1;
        std::vector<uint32_t> list, cdeg;
        for (uint64_t r = 0; r < nz; ++r) {
            const uint32_t c = hub ? hcnt[r] : deg[r] - hcnt[r];
            if (c) {
                list.push_back((uint32_t)r);
                cdeg.push_back(c);
            }
        }
        const uint64_t n = list.size();
        std::vector<uint64_t> coff(n + 1 + kOffPad, 0);
        for (uint64_t i = 0; i < n; ++i) coff[i + 1] = coff[i] + cdeg[i];
        const uint64_t total = coff[n];
        for (uint64_t i = n + 1; i < coff.size(); ++i) coff[i] = total;
        gxb_graph* sg = new gxb_graph();
        s->split_g[k] = sg;
        sg->ctx = g->ctx;
        sg->part = 0;
        sg->nparts = 1;
        sg->lo = 0;
        sg->hi = n;
        sg->S = n;
        sg->E = total;
        sg->owned_edges = total;
        sg->h_indeg_sorted = cdeg;
        GXB_CHECK(dalloc_t(&sg->d_in_off, coff.size()));
        GXB_CHECK(dalloc_t(&sg->d_in_src, total + kTileEdges));
        GXB_CUDA(cudaMemsetAsync(sg->d_in_src, 0, 4 * (total + kTileEdges), st));
        GXB_CHECK(dalloc_t(&s->d_split_slot[k], n + 1));
        GXB_CUDA(cudaMemcpyAsync(sg->d_in_off, coff.data(), 8 * coff.size(), cudaMemcpyHostToDevice, st));
        if (n) GXB_CUDA(cudaMemcpyAsync(s->d_split_slot[k], list.data(), 4 * n, cudaMemcpyHostToDevice, st));
        if (n) k_split_copy<<<grid_for(32 * n), kBlock, 0, st>>>(g->d_in_off, g->d_in_src, d_hcnt, s->d_split_slot[k],
                                                                  n, sg->d_in_off, hub ? 1 : 0, sg->d_in_src);
        GXB_CUDA(cudaStreamSynchronize(st));  // list / coff host buffers die with this scope
        GXB_CHECK(build_tile_plan(sg, st));
        if (sg->tiles.num_spans)
            k_remap_u32<<<grid_for(sg->tiles.num_spans), kBlock, 0, st>>>(sg->tiles.d_span_slot, sg->tiles.num_spans,
                                                                          s->d_split_slot[k]);
        GXB_CHECK(dalloc(&s->d_split_partials[k], sizeof(PrOps::Acc) * (sg->tiles.num_partials + 1)));
        GXB_CHECK(dalloc_t(&s->d_split_sum[k], owned + 1));
        GXB_CUDA(cudaMemsetAsync(s->d_split_sum[k], 0, 8 * (owned + 1), st));
        return GXB_OK;
    };
    int rc = GXB_OK;
    for (int k = 0; k < 2 && rc == GXB_OK; ++k) rc = build_one(k);
    if (cudaStreamSynchronize(st) != cudaSuccess && rc == GXB_OK) rc = fail(GXB_ECUDA, "pr_split_prepare: sync");
    if (rc != GXB_OK) {
        pr_split_free(s);
        return rc;
    }
    s->hub_n = H;
    return GXB_OK;
}

TileLaunch split_launch(gxb_state* s, int k) {
    const gxb_graph* sg = s->split_g[k];
    const TilePlan& T = sg->tiles;
    TileLaunch L = tile_launch(s);
    L.num_tiles = T.num_tiles;
    L.tile_begin = 0;
    L.owned_edges = sg->owned_edges;
    L.in_off = sg->d_in_off;
    L.in_src = sg->d_in_src;
    L.tile_start = T.d_tile_start;
    L.lane_slot = T.d_lane_slot;
    L.lane_mask = T.d_lane_mask;
    L.in_w = nullptr;
    L.in_sw = nullptr;
    L.sw_shift = 0;
    L.tile_head = T.d_tile_head;
    L.tile_tail = T.d_tile_tail;
    L.span_first = T.d_span_first;
    L.span_count = T.d_span_count;
    L.span_pbase = T.d_span_pbase;
    L.span_slot = T.d_span_slot;
    L.partials = s->d_split_partials[k];
    L.sums = s->d_split_sum[k];
    L.key_slot = s->d_split_slot[k];
    return L;
}

// one PageRank round over the split CSCs: hub pass, cold tiles, span folds, Apply
int launch_pr_split(gxb_state* s, cudaStream_t st) {
    GXB_CHECK(pr_split_prepare(s, st));
    gxb_graph* g = s->g;
    PrOps o = pr_ops(s);
    const TileLaunch Lh = split_launch(s, 1), Lc = split_launch(s, 0);
    using Pol = FusedPolicy<PrOps>;
    Pol p{o, nullptr};
    const size_t tab_bytes = 8ull * s->hub_n;
    GXB_CUDA(cudaFuncSetAttribute(k_tile_hub, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 28672));
    auto kern = k_tile_a<Pol, 6>;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBlock, 0);
    if (s->timing) GXB_CUDA(cudaEventRecord(kev_at(s, 0), st));
    if (Lh.num_tiles) {
        k_tile_hub<<<kNumSMs, kHubBlock, tab_bytes, st>>>(o.contrib_cur, s->hub_n, Lh);
        s->launches++;
    }
    if (Lc.num_tiles) {
        const uint64_t want = (Lc.num_tiles + (kBlock / 32) - 1) / (kBlock / 32);
        const unsigned grid = (unsigned)std::min<uint64_t>(want, (uint64_t)std::max(1, per_sm) * kNumSMs);
        kern<<<grid, kBlock, 0, st>>>(p, Lc);
        s->launches++;
    }
    if (s->timing) {
        GXB_CUDA(cudaEventRecord(kev_at(s, 1), st));
        s->timing_pending = true;
    }
    for (int k = 0; k < 2; ++k) {
        const TilePlan& T = s->split_g[k]->tiles;
        if (T.num_spans) {
            k_span_fold<PrOps><<<grid_for(T.num_spans), kBlock, 0, st>>>(
                T.d_span_slot, T.d_span_count, T.d_span_pbase, 0, T.num_spans,
                (const PrOps::Acc*)s->d_split_partials[k], (PrOps::Acc*)s->d_split_sum[k]);
            s->launches++;
        }
    }
    PrOps a = o;
    a.hub_sum = s->d_split_sum[1];
    const uint64_t owned = g->hi - g->lo;
    if (owned) {
        k_apply_sums<PrOps><<<grid_for(owned), kBlock, 0, st>>>(a, (const PrOps::Acc*)s->d_split_sum[0], g->lo, 0,
                                                                 owned, g->tiles.nz_slots, s->d_stats);
        s->launches++;
    }
    GXB_CUDA(cudaGetLastError());
    return GXB_OK;
}

bool use_binned_pull() { return options().pull_kernel == 1; }


// L2 budget for the gathered value prefix (GXB_L2_HOT_MB, default 64 of the 126 MB)
HotPrefix hot_prefix(const gxb_state* s) {
    HotPrefix h;
    const gxb_graph* g = s->g;
    if (g->nparts > 1 && g->S) {
        const uint64_t blk = (g->S + g->nparts - 1) / g->nparts;
        h.block = (uint32_t)blk;
        h.magic = (uint32_t)((1ull << 32) / blk + 1);
    }
    return h;
}

uint32_t hot_slots(const gxb_state* s, size_t bytes_per_slot) {
    const uint64_t n = ((uint64_t)options().l2_hot_mb << 20) / bytes_per_slot;
    return (uint32_t)std::min<uint64_t>(n, s->g->S);
}

uint32_t hot_l1_slots(const gxb_state* s, size_t bytes_per_slot) {
    const uint64_t n = ((uint64_t)options().l1_hot_kb << 10) / bytes_per_slot;
    return (uint32_t)std::min<uint64_t>(n, s->g->S);
}

PrOps pr_ops(gxb_state* s) {
    PrOps o;
    o.contrib_cur = s->d_contrib[s->cur];
    o.rank_old = s->d_rank[s->cur];
    o.rank_new = s->d_rank[s->cur ^ 1];
    o.contrib_next = s->d_contrib[s->cur ^ 1];
    o.msg32 = s->msg32;
    o.npeers = s->npeers;
    for (int q = 0; q < kMaxPeers; ++q)
        o.peer_next[q] = q < s->npeers ? static_cast<double*>(s->peer_contrib[q][s->cur ^ 1]) : nullptr;
    o.f = frontier_view(s);
    o.hp = hot_prefix(s);
    o.hot = hot_slots(s, sizeof(double)) / s->g->nparts;
    o.hot1 = hot_l1_slots(s, sizeof(double));
    o.hub_sum = nullptr;
    return o;
}
SsspOps sssp_ops(gxb_state* s) {
    SsspOps o;
    o.dist_cur = s->d_dist_cur;
    o.dist_next = s->d_dist_next;
    o.active_cur = s->d_active[0];
    o.f = frontier_view(s);
    o.commit_inline = false;
    o.check_active = true;
    o.hp = hot_prefix(s);
    o.hot = hot_slots(s, sizeof(uint4)) / s->g->nparts;
    o.hot1 = hot_l1_slots(s, sizeof(uint4));
    return o;
}
CcOps cc_ops(gxb_state* s) {
    CcOps o;
    o.lab_cur = s->d_lab_cur;
    o.lab_next = s->d_lab_next;
    o.active_cur = s->d_active[0];
    o.f = frontier_view(s);
    o.commit_inline = false;
    o.check_active = true;
    o.hp = hot_prefix(s);
    o.hot = hot_slots(s, sizeof(uint32_t)) / s->g->nparts;
    o.hot1 = hot_l1_slots(s, sizeof(uint32_t));
    return o;
}

// PageRank round with the fused peer exchange pipelined: chunks run hubs-last (the last
// chunk has the fewest slots, so the Apply left after the final tile kernel is the
// shortest) and each chunk's Apply, with its NVLink stores, overlaps the next chunk's tiles
int pipelined_pagerank(gxb_state* s, cudaStream_t st) {
    if (!s->aux_stream) {
        GXB_CUDA(cudaStreamCreateWithFlags(&s->aux_stream, cudaStreamNonBlocking));
        GXB_CUDA(cudaEventCreateWithFlags(&s->ev_tile, cudaEventDisableTiming));
        GXB_CUDA(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
    }
    GXB_CUDA(cudaEventRecord(s->ev_join, st));  // after begin_round's resets
    GXB_CUDA(cudaStreamWaitEvent(s->aux_stream, s->ev_join, 0));
    const PrOps ops = pr_ops(s);
    for (int k = s->g->tiles.num_xchunks - 1; k >= 0; --k) GXB_CHECK(launch_tile_and_apply(s, ops, st, k, s->aux_stream));
    GXB_CUDA(cudaEventRecord(s->ev_join, s->aux_stream));
    GXB_CUDA(cudaStreamWaitEvent(st, s->ev_join, 0));
    return GXB_OK;
}

// a pull round gathers every source (no active-bitmap test) once the frontier's GEN units
// reach 1 / pull_dense_div of the edges (0 = always test)
bool dense_pull(const gxb_state* s) {
    const uint32_t div = options().pull_dense_div;
    return !s->nonmonotone && div != 0 && s->units_cur * (uint64_t)div >= s->g->E;
}

// the local-source pass of the next round (split rounds, gxb_iterate_local): wait for it on
// `st` before anything touches the sums it writes; its result stays usable only for the
// next gxb_iterate, which takes it when that round is a tile pull
int join_local(gxb_state* s, cudaStream_t st) {
    if (s->local_launched) GXB_CUDA(cudaStreamWaitEvent(st, s->ev_local, 0));
    s->local_launched = false;
    s->local_valid = false;
    return GXB_OK;
}

int begin_round(gxb_state* s, cudaStream_t st) {
    GXB_CHECK(join_local(s, st));
    if (s->stats_pending) {
        GXB_CUDA(cudaEventSynchronize(s->stats_ready));
        s->stats_pending = false;
    }
    GXB_CUDA(cudaMemsetAsync(s->d_stats, 0, sizeof(StatStripe) * kStripes, st));
    GXB_CUDA(cudaMemsetAsync(s->d_fcount + 1, 0, sizeof(unsigned long long), st));
    GXB_CUDA(cudaMemsetAsync(s->d_active[1], 0, 4 * s->words, st));
    s->in_round = true;
    s->committed_inline = false;
    s->round_chunks = 0;
    return GXB_OK;
}

// close the round: commit values, rotate frontier buffers, snapshot stats
int end_round(gxb_state* s, int direction, cudaStream_t st) {
    gxb_graph* g = s->g;
    if (s->algo == GXB_ALGO_PAGERANK) {
        s->cur ^= 1;
    } else if (direction == GXB_DIR_PULL && !s->committed_inline) {
        const unsigned grid = grid_for(g->hi - g->lo);
        if (s->algo == GXB_ALGO_SSSP)
            k_commit<uint4><<<grid, kBlock, 0, st>>>(s->d_dist_cur, s->d_dist_next, s->d_frontier[1], s->d_fcount + 1);
        else
            k_commit<uint32_t><<<grid, kBlock, 0, st>>>(s->d_lab_cur, s->d_lab_next, s->d_frontier[1], s->d_fcount + 1);
        s->launches++;
        GXB_CUDA(cudaGetLastError());
    }
    if (s->algo != GXB_ALGO_PAGERANK) {
        std::swap(s->d_active[0], s->d_active[1]);
        std::swap(s->d_frontier[0], s->d_frontier[1]);
        GXB_CUDA(cudaMemcpyAsync(s->d_fcount, s->d_fcount + 1, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
    }
    if (s->timing_pending) GXB_CUDA(cudaEventRecord(kev_at(s, 2), st));  // end of the round's kernels
    if (s->timing_pending && s->async_stats) {
        s->kring_n++;
        s->timing_pending = false;
        if (s->kring_n % gxb_state::kRing == 0) GXB_CHECK(drain_kring(s, gxb_state::kRing));
    }
    if (!s->async_stats) {  // async mode: the caller reads the round through gxb_stats_device
        GXB_CUDA(cudaMemcpyAsync(s->h_stats, s->d_stats, sizeof(StatStripe) * kStripes, cudaMemcpyDeviceToHost, st));
        GXB_CUDA(cudaMemcpyAsync(s->h_fcount, s->d_fcount, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        GXB_CUDA(cudaEventRecord(s->stats_ready, st));
        s->stats_pending = true;
    }
    s->in_round = false;
    s->iteration++;
    s->lab_injective = false;
    s->last_direction = direction;
    return GXB_OK;
}

int collect_stats(gxb_state* s);

// an asynchronous unpack (gxb_exchange_unpack_regions) or an install of changed values
// (gxb_attrs_install / gxb_write_attrs) appended vertices to the frontier on the device:
// refresh the host copies of its length and GEN units
int settle_unpack(gxb_state* s) {
    if (!s->unpack_pending && !s->install_pending) return GXB_OK;
    GXB_CHECK(collect_stats(s));
    unsigned long long v[4] = {0, 0, 0, 0};
    GXB_CUDA(cudaMemcpy(&v[0], s->d_fcount, 8, cudaMemcpyDeviceToHost));
    GXB_CUDA(cudaMemcpy(&v[1], s->d_xscratch + 1, 24, cudaMemcpyDeviceToHost));
    s->frontier_len = v[0];
    if (s->unpack_pending) s->units_cur += v[1];
    if (s->install_pending) {
        s->units_cur += v[2];
        if (v[3]) s->nonmonotone = true;
    }
    s->unpack_pending = s->install_pending = false;
    return GXB_OK;
}

// host reduction of the stat stripes
int collect_stats(gxb_state* s) {
    if (s->stats_pending) {
        GXB_CUDA(cudaEventSynchronize(s->stats_ready));
        s->stats_pending = false;
        gxb_iter_stats o;
        std::memset(&o, 0, sizeof(o));
        double m = 0.0;
        for (int i = 0; i < kStripes; ++i) {
            const StatStripe& t = s->h_stats[i];
            o.changed += t.changed;
            o.next_active += t.next_active;
            o.next_units += t.next_units;
            o.targets += t.targets;
            o.remote_active += t.remote_active;
            double x;
            std::memcpy(&x, &t.max_stat_bits, 8);
            m = std::max(m, x);
        }
        o.iteration = s->iteration;
        o.units = s->units_cur;
        o.max_stat = m;
        o.direction = s->last_direction;
        const gxb_graph* g = s->g;
        if (s->algo == GXB_ALGO_PAGERANK) {
            // every vertex stays active (A/algorithms.py:144-145, 159)
            o.next_active = g->hi - g->lo;
            o.next_units = s->owned_outdeg_sum;
            o.targets = s->owned_targets;
            o.voted = m < 1e-9 ? 1 : 0;  // PageRank.vote (164-165)
            // all owned vertices are in the next frontier: count those with remote consumers
            o.remote_active = s->last.remote_active;
        } else {
            o.voted = o.next_active == 0 ? 1 : 0;  // not next_active (70-72)
        }
        s->frontier_len = *s->h_fcount;
        s->units_cur = o.next_units;
        s->last = o;
    }
    if (s->timing_pending && !s->async_stats) {
        float ms = 0.f;
        GXB_CUDA(cudaEventSynchronize(s->kev[2]));
        GXB_CUDA(cudaEventElapsedTime(&ms, s->kev[0], s->kev[1]));
        s->kernel_ms += ms;
        GXB_CUDA(cudaEventElapsedTime(&ms, s->kev[1], s->kev[2]));
        s->rest_ms += ms;
        s->kernel_launches++;
        s->timing_pending = false;
    }
    return GXB_OK;
}

}  // namespace

namespace gxb {
int state_settle(gxb_state* s) {
    GXB_CHECK(collect_stats(s));
    return settle_unpack(s);
}
}  // namespace gxb

// push scheduling buffers, allocated with the state so no iteration pays for cudaMalloc
static int alloc_push(gxb_state* s) {
    const gxb_graph* g = s->g;
    GXB_CHECK(dalloc_t(&s->d_push_cpre, g->S + 1));
    GXB_CHECK(dalloc_t(&s->d_scan_status, g->S / kScanTile + 2));
    return GXB_OK;
}

// rowpre of the frontier (k_push_rowpre), one kernel
static int launch_rowpre(gxb_state* s, uint64_t nf, cudaStream_t st) {
    const uint64_t tiles = (nf + kScanTile - 1) / kScanTile;
    GXB_CUDA(cudaMemsetAsync(s->d_scan_status, 0, 8 * (tiles + 1), st));
    k_push_rowpre<<<(unsigned)tiles, kBlock, 0, st>>>(s->d_frontier[0], nf, s->g->d_out_off, s->d_push_cpre,
                                                      s->d_scan_status);
    s->launches++;
    return GXB_OK;
}

extern "C" {

int gxb_state_free(gxb_state* s);
void gxb_lp_free(gxb_state* s);                     // gxb_lp.cu
int gxb_lp_prepare(gxb_state* s, cudaStream_t st);  // gxb_lp.cu

int gxb_state_create(gxb_graph* g, int algo, const uint32_t* sources, int nsrc, gxb_state** out) {
    NvtxRange nvtx_("gxb_state_create");
    if (!g || !out) return fail(GXB_EINVAL, "gxb_state_create: null argument");
    if (algo < GXB_ALGO_SSSP || algo > GXB_ALGO_CC) return fail(GXB_EINVAL, "unknown algorithm");
    if (!g->ctx->alive) return fail(GXB_ESTATE, "gxb_state_create: daemon terminated");
    GXB_CUDA(cudaSetDevice(g->ctx->device));
    gxb_state* s = new gxb_state();
    s->g = g;
    s->algo = algo;
    auto bail = [&](int rc) {
        gxb_state_free(s);
        return rc;
    };
    // slot arrays span the slot space S (= V, or padded to equal partition blocks)
    const uint64_t V = g->S, owned = g->hi - g->lo;
    s->words = (V >> 5) + 1;
    cudaStream_t st = 0;
    // host copies of degrees for static counts
    {
        std::vector<uint32_t> od(V);
        if (V && cudaMemcpy(od.data(), g->d_outdeg, 4 * V, cudaMemcpyDeviceToHost) != cudaSuccess)
            return bail(fail(GXB_ECUDA, "state_create: outdeg copy"));
        for (uint64_t i = g->lo; i < g->hi; ++i) s->owned_outdeg_sum += od[i];
        for (uint64_t i = 0; i < owned; ++i) s->owned_targets += g->h_indeg_sorted[i] > 0 ? 1 : 0;
    }
    int rc;
    if ((rc = dalloc_t(&s->d_stats, kStripes)) != GXB_OK) return bail(rc);
    if (cudaMallocHost(&s->h_stats, sizeof(StatStripe) * kStripes) != cudaSuccess ||
        cudaMallocHost(&s->h_fcount, 64) != cudaSuccess)
        return bail(fail(GXB_ENOMEM, "pinned stats"));
    if (cudaEventCreateWithFlags(&s->stats_ready, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(GXB_ECUDA, "event"));
    if ((rc = dalloc_t(&s->d_fcount, 2)) != GXB_OK) return bail(rc);
    for (int i = 0; i < 2; ++i) {
        if ((rc = dalloc_t(&s->d_active[i], s->words)) != GXB_OK) return bail(rc);
        if ((rc = dalloc_t(&s->d_frontier[i], V + 1)) != GXB_OK) return bail(rc);
        cudaMemsetAsync(s->d_active[i], 0, 4 * s->words, st);
    }
    if ((rc = dalloc_t(&s->d_touched, (owned >> 5) + 1)) != GXB_OK) return bail(rc);
    cudaMemsetAsync(s->d_touched, 0, 4 * ((owned >> 5) + 1), st);
    // chunk partials: the largest accumulator is SsspOps::Acc (32 B with padding)
    if ((rc = dalloc(&s->d_partials, 32 * (g->plan.num_items + 1))) != GXB_OK) return bail(rc);
    if ((rc = dalloc(&s->d_tile_partials, 32 * (g->tiles.num_partials + 1))) != GXB_OK) return bail(rc);
    if ((rc = dalloc(&s->d_sums, 32 * (owned + 1))) != GXB_OK) return bail(rc);

    const unsigned grid = grid_for(V);
    uint64_t nfront = 0, units0 = 0;
    if (algo == GXB_ALGO_PAGERANK) {
        s->arity = 1;
        for (int i = 0; i < 2; ++i)
            if ((rc = dalloc_t(&s->d_rank[i], V)) != GXB_OK) return bail(rc);
        for (int i = 0; i < 2; ++i)
            if ((rc = dalloc_t(&s->d_contrib[i], V)) != GXB_OK) return bail(rc);
        s->msg32 = options().pr_message_bits == 32;
        if (V) {
            k_pr_init<<<grid, kBlock, 0, st>>>(s->d_rank[0], s->d_contrib[0], g->d_outdeg, g->d_slot2id, V, s->msg32);
            cudaMemcpyAsync(s->d_rank[1], s->d_rank[0], 8 * V, cudaMemcpyDeviceToDevice, st);
            // both contribution buffers start valid: a mirror that never changes is never
            // re-sent by a changed-values-only sync (gxb_attrs_deliver)
            cudaMemcpyAsync(s->d_contrib[1], s->d_contrib[0], (s->msg32 ? 4 : 8) * V, cudaMemcpyDeviceToDevice, st);
        }
        units0 = s->owned_outdeg_sum;
    } else if (algo == GXB_ALGO_SSSP) {
        if (nsrc < 0 || nsrc > 4) return bail(fail(GXB_EINVAL, "sssp supports 1..4 sources"));
        std::vector<uint32_t> ids(V);
        if (V && cudaMemcpy(ids.data(), g->d_slot2id, 4 * V, cudaMemcpyDeviceToHost) != cudaSuccess)
            return bail(fail(GXB_ECUDA, "state_create: id copy"));
        std::vector<std::pair<uint32_t, uint32_t>> by_id(V);  // (id, slot)
        for (uint64_t i = 0; i < V; ++i) by_id[i] = {ids[i], (uint32_t)i};
        std::sort(by_id.begin(), by_id.end());
        by_id.resize(g->V);  // padding slots (id 0xFFFFFFFF) sort last and are not vertices
        std::vector<uint32_t> src_ids;
        if (sources && nsrc > 0) {
            src_ids.assign(sources, sources + nsrc);
        } else {
            // sorted(vertex_ids)[:4] (A/algorithms.py:219-222)
            for (uint64_t i = 0; i < g->V && i < 4; ++i) src_ids.push_back(by_id[i].first);
        }
        if (src_ids.empty()) return bail(fail(GXB_EINVAL, "sssp needs at least one source vertex"));
        // exact u32 arithmetic: no message d + w may reach the INF sentinel
        if ((unsigned __int128)g->max_w * V >= 0xFFFFFFFFull)
            return bail(fail(GXB_ERANGE, "edge weights too large for exact 32-bit distances (max_w * |V| >= 2^32-1)"));
        s->nsrc = (int)src_ids.size();
        s->arity = s->nsrc;
        if ((rc = dalloc_t(&s->d_dist_cur, V)) != GXB_OK) return bail(rc);
        if ((rc = dalloc_t(&s->d_dist_next, V)) != GXB_OK) return bail(rc);
        const uint4 inf = make_uint4(kInf32, kInf32, kInf32, kInf32);
        if (V) k_fill_u4<<<grid, kBlock, 0, st>>>(s->d_dist_cur, V, inf);
        std::vector<uint4> src_vals;
        std::vector<uint32_t> front;
        std::vector<uint32_t> h_od(V);
        if (V) cudaMemcpy(h_od.data(), g->d_outdeg, 4 * V, cudaMemcpyDeviceToHost);
        for (int j = 0; j < s->nsrc; ++j) {
            auto it = std::lower_bound(by_id.begin(), by_id.end(), std::make_pair(src_ids[j], 0u));
            if (it == by_id.end() || it->first != src_ids[j]) continue;  // absent source: all-inf lane
            s->src_present[j] = true;
            s->src_slot[j] = it->second;
        }
        // initial_attr: 0 on the own lane (96-97); initially_active: the sources (99-100)
        std::vector<uint32_t> uniq;
        for (int j = 0; j < s->nsrc; ++j)
            if (s->src_present[j] && std::find(uniq.begin(), uniq.end(), s->src_slot[j]) == uniq.end())
                uniq.push_back(s->src_slot[j]);
        for (uint32_t slot : uniq) {
            uint32_t l[4] = {kInf32, kInf32, kInf32, kInf32};
            for (int j = 0; j < s->nsrc; ++j)
                if (s->src_present[j] && s->src_slot[j] == slot) l[j] = 0;
            const uint4 v = make_uint4(l[0], l[1], l[2], l[3]);
            cudaMemcpyAsync(s->d_dist_cur + slot, &v, sizeof(uint4), cudaMemcpyHostToDevice, st);
            cudaStreamSynchronize(st);
            front.push_back(slot);
            units0 += h_od[slot];
        }
        if (V) cudaMemcpyAsync(s->d_dist_next, s->d_dist_cur, sizeof(uint4) * V, cudaMemcpyDeviceToDevice, st);
        std::vector<uint32_t> bm(s->words, 0);
        for (uint32_t slot : front) bm[slot >> 5] |= 1u << (slot & 31);
        cudaMemcpyAsync(s->d_active[0], bm.data(), 4 * s->words, cudaMemcpyHostToDevice, st);
        if (!front.empty())
            cudaMemcpyAsync(s->d_frontier[0], front.data(), 4 * front.size(), cudaMemcpyHostToDevice, st);
        nfront = front.size();
        cudaStreamSynchronize(st);
    } else {
        // LP / CC: label = vertex id, every vertex active (A/algorithms.py:179-183)
        s->arity = 1;
        s->lab_injective = true;
        if ((rc = dalloc_t(&s->d_lab_cur, V)) != GXB_OK) return bail(rc);
        if ((rc = dalloc_t(&s->d_lab_next, V)) != GXB_OK) return bail(rc);
        if (V) {
            cudaMemcpyAsync(s->d_lab_cur, g->d_slot2id, 4 * V, cudaMemcpyDeviceToDevice, st);
            cudaMemcpyAsync(s->d_lab_next, g->d_slot2id, 4 * V, cudaMemcpyDeviceToDevice, st);
            k_bitmap_range<<<grid, kBlock, 0, st>>>(s->d_active[0], 0, V);
            k_iota_u32<<<grid, kBlock, 0, st>>>(s->d_frontier[0], 0, V);
        }
        nfront = V;
        std::vector<uint32_t> od(V);
        if (V) cudaMemcpy(od.data(), g->d_outdeg, 4 * V, cudaMemcpyDeviceToHost);
        for (uint64_t i = 0; i < V; ++i) units0 += od[i];
    }
    unsigned long long fc[2] = {nfront, 0};
    cudaMemcpyAsync(s->d_fcount, fc, sizeof(fc), cudaMemcpyHostToDevice, st);
    s->frontier_len = nfront;
    s->units_cur = units0;
    // remote-active count of the initial frontier (the GAS seed round's skip vote,
    // A/agent.py:533-535); for PageRank it stays this value every round
    if (g->nparts > 1) {
        std::vector<uint32_t> rb(s->words);
        cudaMemcpy(rb.data(), g->d_remote_src, 4 * ((V >> 5) + 1), cudaMemcpyDeviceToHost);
        uint64_t c = 0;
        if (algo == GXB_ALGO_SSSP) {
            for (int j = 0; j < s->nsrc; ++j) {
                const uint32_t sl = s->src_slot[j];
                bool dup = false;
                for (int k = 0; k < j; ++k) dup |= s->src_present[k] && s->src_slot[k] == sl;
                if (s->src_present[j] && !dup && sl >= g->lo && sl < g->hi) c += (rb[sl >> 5] >> (sl & 31)) & 1u;
            }
        } else {
            for (uint64_t i = g->lo; i < g->hi; ++i) c += (rb[i >> 5] >> (i & 31)) & 1u;
        }
        s->last.remote_active = c;
    }
    if (algo != GXB_ALGO_PAGERANK && g->has_csr && (rc = alloc_push(s)) != GXB_OK)
        return bail(rc);
    if (algo == GXB_ALGO_LP && (rc = gxb_lp_prepare(s, st)) != GXB_OK) return bail(rc);
    if (algo != GXB_ALGO_PAGERANK && (rc = dalloc_t(&s->d_xscratch, 4)) != GXB_OK) return bail(rc);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return bail(cuda_fail(e, "gxb_state_create"));
    *out = s;
    return GXB_OK;
}

int gxb_exchange_close_peers(gxb_state* s);  // gxb_exchange.cu

int gxb_state_free(gxb_state* s) {
    if (!s) return GXB_OK;
    gxb_exchange_close_peers(s);
    if (s->algo != GXB_ALGO_PAGERANK) gxb_exchange_delta_close(s);
    if (s->aux_stream) {
        cudaStreamSynchronize(s->aux_stream);  // a local pass may still read / write the buffers below
        cudaStreamDestroy(s->aux_stream);
    }
    if (s->ev_tile) cudaEventDestroy(s->ev_tile);
    if (s->ev_join) cudaEventDestroy(s->ev_join);
    if (s->ev_local) cudaEventDestroy(s->ev_local);
    dfree(s->d_rank[0]);
    dfree(s->d_rank[1]);
    dfree(s->d_contrib[0]);
    dfree(s->d_contrib[1]);
    dfree(s->d_dist_cur);
    dfree(s->d_dist_next);
    dfree(s->d_lab_cur);
    dfree(s->d_lab_next);
    for (int i = 0; i < 2; ++i) {
        dfree(s->d_active[i]);
        dfree(s->d_frontier[i]);
    }
    dfree(s->d_fcount);
    dfree(s->d_touched);
    dfree(s->d_stats);
    if (s->h_stats) cudaFreeHost(s->h_stats);
    if (s->h_fcount) cudaFreeHost(s->h_fcount);
    if (s->stats_ready) cudaEventDestroy(s->stats_ready);
    dfree(s->d_msg);
    dfree(s->d_msg_valid);
    dfree(s->d_merged);
    dfree(s->d_partials);
    dfree(s->d_stage);
    for (int i = 0; i < 2; ++i) {
        dfree(s->d_stage_in[i]);
        dfree(s->d_stage_out[i]);
    }
    for (int i = 0; i < 3; ++i)
        if (s->kev[i]) cudaEventDestroy(s->kev[i]);
    if (s->kring) {
        for (int i = 0; i < 3 * gxb_state::kRing; ++i)
            if (s->kring[i]) cudaEventDestroy(s->kring[i]);
        delete[] s->kring;
    }
    dfree(s->d_push_cpre);
    dfree(s->d_scan_status);
    dfree(s->d_tile_partials);
    dfree(s->d_sums);
    pr_split_free(s);
    gxb_lp_free(s);
    dfree(s->d_send);
    dfree(s->d_xsend);
    dfree(s->d_xrecv);
    dfree(s->d_recv);
    dfree(s->d_xscratch);
    delete s;
    return GXB_OK;
}

int gxb_state_arity(const gxb_state* s, int* out) {
    if (!s || !out) return fail(GXB_EINVAL, "gxb_state_arity: null argument");
    *out = s->arity;
    return GXB_OK;
}

int gxb_lp_pull(gxb_state* s, cudaStream_t st);  // gxb_lp.cu
int gxb_lp_push(gxb_state* s, cudaStream_t st, const uint32_t* rowpre);


int gxb_iterate_local(gxb_state* s, void* stream, int* launched) {
    NvtxRange nvtx_("gxb_iterate_local");
    if (launched) *launched = 0;
    if (!s) return fail(GXB_EINVAL, "gxb_iterate_local: null state");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_iterate_local: a request round is open");
    gxb_graph* g = s->g;
    // only behind a dense tile pull of SSSP / CC at N > 1 (the next round is most likely
    // one too); otherwise nothing is launched and the next round runs whole
    if (!options().split_overlap || g->nparts < 2 || (s->algo != GXB_ALGO_SSSP && s->algo != GXB_ALGO_CC) ||
        use_binned_pull() || s->last_direction != GXB_DIR_PULL || !s->last_dense || s->local_launched ||
        s->iteration == 0)
        return GXB_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (!s->aux_stream) {
        GXB_CUDA(cudaStreamCreateWithFlags(&s->aux_stream, cudaStreamNonBlocking));
        GXB_CUDA(cudaEventCreateWithFlags(&s->ev_tile, cudaEventDisableTiming));
        GXB_CUDA(cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming));
    }
    if (!s->ev_local) GXB_CUDA(cudaEventCreateWithFlags(&s->ev_local, cudaEventDisableTiming));
    GXB_CUDA(cudaEventRecord(s->ev_join, st));  // after the round that produced the values
    GXB_CUDA(cudaStreamWaitEvent(s->aux_stream, s->ev_join, 0));
    const SourceSel sel{(uint32_t)g->lo, (uint32_t)(g->hi - g->lo), 1};
    if (s->algo == GXB_ALGO_SSSP) {
        SsspOps o = sssp_ops(s);
        o.check_active = false;  // exact either way (see SsspOps::check_active)
        o.sel = sel;
        GXB_CHECK(launch_tile_and_apply(s, o, s->aux_stream, -1, nullptr, 1));
    } else {
        CcOps o = cc_ops(s);
        o.check_active = false;
        o.sel = sel;
        GXB_CHECK(launch_tile_and_apply(s, o, s->aux_stream, -1, nullptr, 1));
    }
    GXB_CUDA(cudaEventRecord(s->ev_local, s->aux_stream));
    s->local_launched = true;
    s->local_valid = true;
    if (launched) *launched = 1;
    return GXB_OK;
}

int gxb_iterate(gxb_state* s, int direction, void* stream) {
    NvtxRange nvtx_("gxb_iterate");
    if (!s) return fail(GXB_EINVAL, "gxb_iterate: null state");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_iterate: a request round is open (call gxb_commit)");
    if (!s->g->ctx->alive) return fail(GXB_ESTATE, "gxb_iterate: daemon terminated");
    cudaStream_t st = (cudaStream_t)stream;
    gxb_graph* g = s->g;
    GXB_CHECK(collect_stats(s));
    GXB_CHECK(settle_unpack(s));
    const bool local_done = s->local_valid;
    GXB_CHECK(begin_round(s, st));  // joins the local pass
    int dir = GXB_DIR_PULL;
    if (s->algo == GXB_ALGO_SSSP || s->algo == GXB_ALGO_CC) {
        if (direction == GXB_DIR_PUSH) dir = GXB_DIR_PUSH;
        else if (direction == GXB_DIR_AUTO) dir = (s->units_cur * (uint64_t)options().push_alpha < g->E) ? GXB_DIR_PUSH : GXB_DIR_PULL;
        if (dir == GXB_DIR_PUSH && !g->has_csr) {
            if (direction == GXB_DIR_PUSH) return fail(GXB_EINVAL, "push requested but the graph has no CSR");
            dir = GXB_DIR_PULL;
        }
    }
    // LP "push": mark the frontier's out-neighbours over the CSR, then take the mode of the
    // marked destinations only (the others receive no message and keep their label)
    bool lp_sparse = false;
    if (s->algo == GXB_ALGO_LP && g->has_csr) {
        if (direction == GXB_DIR_PUSH) lp_sparse = true;
        else if (direction == GXB_DIR_AUTO) lp_sparse = s->units_cur * (uint64_t)options().push_alpha < g->E;
        if (lp_sparse) dir = GXB_DIR_PUSH;
    } else if (s->algo == GXB_ALGO_LP && direction == GXB_DIR_PUSH) {
        return fail(GXB_EINVAL, "push requested but the graph has no CSR");
    }
    const uint64_t owned = g->hi - g->lo;
    if (lp_sparse) {
        if (!s->d_scan_status) GXB_CHECK(alloc_push(s));
        const uint64_t nf = s->frontier_len;
        if (nf) GXB_CHECK(launch_rowpre(s, nf, st));  // the push is edge-balanced over the concatenated rows
        GXB_CHECK(gxb_lp_push(s, st, s->d_push_cpre));
        s->launches += 1;
        GXB_CHECK(end_round(s, GXB_DIR_PULL, st));  // commits lab_next like a pull round
        s->last_direction = GXB_DIR_PUSH;
        return GXB_OK;
    }
    if (dir == GXB_DIR_PULL && s->algo != GXB_ALGO_LP && !use_binned_pull()) {
        switch (s->algo) {
            case GXB_ALGO_PAGERANK:
                if ((s->npeers > 0 || options().pipeline_apply) && g->tiles.num_xchunks > 1)
                    GXB_CHECK(pipelined_pagerank(s, st));
                else if (pr_split_wanted(s)) GXB_CHECK(launch_pr_split(s, st));
                else GXB_CHECK(launch_tile_and_apply(s, pr_ops(s), st));
                break;
            case GXB_ALGO_SSSP: {
                SsspOps o = sssp_ops(s);
                o.check_active = !dense_pull(s);
                if (local_done) o.sel = SourceSel{(uint32_t)g->lo, (uint32_t)(g->hi - g->lo), 2};
                GXB_CHECK(launch_tile_and_apply(s, o, st, -1, nullptr, local_done ? 2 : 0));
                s->last_dense = !o.check_active;
                break;
            }
            case GXB_ALGO_CC: {
                CcOps o = cc_ops(s);
                o.check_active = !dense_pull(s);
                if (local_done) o.sel = SourceSel{(uint32_t)g->lo, (uint32_t)(g->hi - g->lo), 2};
                GXB_CHECK(launch_tile_and_apply(s, o, st, -1, nullptr, local_done ? 2 : 0));
                s->last_dense = !o.check_active;
                break;
            }
        }
    } else if (dir == GXB_DIR_PULL) {
        const PullLaunch L = pull_launch(s, 0, owned);
        switch (s->algo) {
            case GXB_ALGO_PAGERANK: {
                FusedPolicy<PrOps> p{pr_ops(s), g->d_in_w};
                GXB_CHECK(launch_pull(p, L, st));
                break;
            }
            case GXB_ALGO_SSSP: {
                FusedPolicy<SsspOps> p{sssp_ops(s), g->d_in_w};
                GXB_CHECK(launch_pull(p, L, st));
                break;
            }
            case GXB_ALGO_CC: {
                FusedPolicy<CcOps> p{cc_ops(s), g->d_in_w};
                GXB_CHECK(launch_pull(p, L, st));
                break;
            }
            case GXB_ALGO_LP:
                GXB_CHECK(gxb_lp_pull(s, st));
                s->launches += 2;
                break;
        }
        if (s->algo != GXB_ALGO_LP) s->launches++;
    } else {
        PushLaunch P;
        P.lo = g->lo;
        P.hi = g->hi;
        P.out_off = g->d_out_off;
        P.out_dst = g->d_out_dst;
        P.out_w = g->d_out_w;
        P.frontier = s->d_frontier[0];
        P.nfront = s->frontier_len;
        P.touched = s->d_touched;
        P.list_next = s->d_frontier[1];
        P.count_next = s->d_fcount + 1;
        FrontierView f = frontier_view(s);
        if (!s->d_scan_status) GXB_CHECK(alloc_push(s));
        if (P.nfront) {
            GXB_CHECK(launch_rowpre(s, P.nfront, st));
            s->launches++;  // the push
            const unsigned grid = grid_for((s->units_cur / kPushChunk + 1) * 32, kBlock, 148ull * 16);
            if (s->algo == GXB_ALGO_SSSP)
                k_push<SsspPush><<<grid, kBlock, 0, st>>>(SsspPush{s->d_dist_cur, s->d_dist_next}, P, s->d_push_cpre);
            else
                k_push<CcPush><<<grid, kBlock, 0, st>>>(CcPush{s->d_lab_cur, s->d_lab_next}, P, s->d_push_cpre);
        }
        s->launches++;
        if (s->algo == GXB_ALGO_SSSP)
            k_push_apply<uint4><<<kNumSMs * 2, kBlock, 0, st>>>(s->d_dist_cur, s->d_dist_next, s->d_frontier[1],
                                                                 s->d_fcount + 1, f, s->d_stats);
        else
            k_push_apply<uint32_t><<<kNumSMs * 2, kBlock, 0, st>>>(s->d_lab_cur, s->d_lab_next, s->d_frontier[1],
                                                                    s->d_fcount + 1, f, s->d_stats);
        GXB_CUDA(cudaGetLastError());
        GXB_CUDA(cudaMemsetAsync(s->d_touched, 0, 4 * ((owned >> 5) + 1), st));
    }
    return end_round(s, dir, st);
}

// Pipeline shuffle (multi-GPU): a PageRank pull round split into exchange chunks so the
// caller can send chunk k's new contributions while chunk k+1 computes.
int gxb_iterate_begin(gxb_state* s, void* stream) {
    if (!s) return fail(GXB_EINVAL, "gxb_iterate_begin: null state");
    if (s->algo != GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "chunked rounds are for PageRank (dense exchange)");
    if (options().pull_kernel == 1) return fail(GXB_EINVAL, "chunked rounds need the warp-tile pull kernel");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_iterate_begin: a round is open");
    GXB_CHECK(collect_stats(s));
    return begin_round(s, (cudaStream_t)stream);
}

int gxb_iterate_chunk(gxb_state* s, int k, void* stream) {
    if (!s) return fail(GXB_EINVAL, "gxb_iterate_chunk: null state");
    if (!s->in_round) return fail(GXB_ESTATE, "gxb_iterate_chunk: no open round");
    if (k < 0 || k >= s->g->tiles.num_xchunks) return fail(GXB_EINVAL, "gxb_iterate_chunk: chunk out of range");
    return launch_tile_and_apply(s, pr_ops(s), (cudaStream_t)stream, k);
}

int gxb_iterate_end(gxb_state* s, void* stream) {
    if (!s) return fail(GXB_EINVAL, "gxb_iterate_end: null state");
    if (!s->in_round) return fail(GXB_ESTATE, "gxb_iterate_end: no open round");
    return end_round(s, GXB_DIR_PULL, (cudaStream_t)stream);
}

int gxb_request(gxb_state* s, int op, uint64_t lo, uint64_t hi, void* stream) {
    NvtxRange nvtx_("gxb_request");
    if (!s) return fail(GXB_EINVAL, "gxb_request: null state");
    if (!s->g->ctx->alive) return fail(GXB_ESTATE, "gxb_request: daemon terminated");
    if (s->algo == GXB_ALGO_LP) return fail(GXB_EINVAL, "gxb_request: LP runs through gxb_iterate only");
    cudaStream_t st = (cudaStream_t)stream;
    gxb_graph* g = s->g;
    const uint64_t owned = g->hi - g->lo;
    if (lo > hi) return fail(GXB_EINVAL, "gxb_request: empty range with lo > hi");
    // lazy message buffers: 16 B per owned edge covers every Msg type
    if (!s->d_msg) {
        GXB_CHECK(dalloc(&s->d_msg, 16 * (g->owned_edges + 1)));
        GXB_CHECK(dalloc_t(&s->d_msg_valid, g->owned_edges + 1));
        GXB_CHECK(dalloc(&s->d_merged, 32 * (owned + 1)));
    }
    if (!s->in_round) {  // the first request of an iteration opens the round
        GXB_CHECK(collect_stats(s));
        GXB_CHECK(settle_unpack(s));
        GXB_CHECK(begin_round(s, st));
    }
    if (op == GXB_OP_GEN) {
        if (hi > g->owned_edges) return fail(GXB_EINVAL, "gxb_request(GEN): edge range outside the owned CSC");
        const unsigned grid = grid_for(hi - lo);
        if (hi > lo) {
            switch (s->algo) {
                case GXB_ALGO_PAGERANK:
                    k_gen<PrOps><<<grid, kBlock, 0, st>>>(pr_ops(s), g->d_in_src, g->d_in_w, lo, hi,
                                                         (double*)s->d_msg, s->d_msg_valid);
                    break;
                case GXB_ALGO_SSSP:
                    k_gen<SsspOps><<<grid, kBlock, 0, st>>>(sssp_ops(s), g->d_in_src, g->d_in_w, lo, hi,
                                                           (uint4*)s->d_msg, s->d_msg_valid);
                    break;
                case GXB_ALGO_CC:
                    k_gen<CcOps><<<grid, kBlock, 0, st>>>(cc_ops(s), g->d_in_src, g->d_in_w, lo, hi,
                                                         (uint32_t*)s->d_msg, s->d_msg_valid);
                    break;
            }
        }
        GXB_CUDA(cudaGetLastError());
        return GXB_OK;
    }
    if (lo < g->lo || hi > g->hi)
        return fail(GXB_ENOTOWNED, "apply targets vertex not owned by this node");
    const uint64_t flo = lo - g->lo, fhi = hi - g->lo;
    if (op == GXB_OP_MERGE) {
        const PullLaunch L = pull_launch(s, flo, fhi);
        switch (s->algo) {
            case GXB_ALGO_PAGERANK: {
                MergePolicy<PrOps> p{pr_ops(s), (const double*)s->d_msg, s->d_msg_valid,
                                     (PrOps::Acc*)s->d_merged, g->lo};
                GXB_CHECK(launch_pull(p, L, st));
                break;
            }
            case GXB_ALGO_SSSP: {
                MergePolicy<SsspOps> p{sssp_ops(s), (const uint4*)s->d_msg, s->d_msg_valid,
                                       (SsspOps::Acc*)s->d_merged, g->lo};
                GXB_CHECK(launch_pull(p, L, st));
                break;
            }
            case GXB_ALGO_CC: {
                MergePolicy<CcOps> p{cc_ops(s), (const uint32_t*)s->d_msg, s->d_msg_valid,
                                     (CcOps::Acc*)s->d_merged, g->lo};
                GXB_CHECK(launch_pull(p, L, st));
                break;
            }
        }
        return GXB_OK;
    }
    if (op == GXB_OP_APPLY) {
        const unsigned grid = grid_for(hi - lo);
        if (hi > lo) {
            switch (s->algo) {
                case GXB_ALGO_PAGERANK:
                    k_apply<PrOps><<<grid, kBlock, 0, st>>>(pr_ops(s), (const PrOps::Acc*)s->d_merged, g->lo, lo, hi,
                                                           s->d_stats);
                    break;
                case GXB_ALGO_SSSP:
                    k_apply<SsspOps><<<grid, kBlock, 0, st>>>(sssp_ops(s), (const SsspOps::Acc*)s->d_merged, g->lo, lo,
                                                             hi, s->d_stats);
                    break;
                case GXB_ALGO_CC:
                    k_apply<CcOps><<<grid, kBlock, 0, st>>>(cc_ops(s), (const CcOps::Acc*)s->d_merged, g->lo, lo, hi,
                                                           s->d_stats);
                    break;
            }
        }
        GXB_CUDA(cudaGetLastError());
        return GXB_OK;
    }
    return fail(GXB_EINVAL, "unknown operation kind");
}

int gxb_commit(gxb_state* s, void* stream) {
    NvtxRange nvtx_("gxb_commit");
    if (!s) return fail(GXB_EINVAL, "gxb_commit: null state");
    if (!s->in_round) {  // a partition with nothing to request still closes an (empty) round
        GXB_CHECK(collect_stats(s));
        GXB_CHECK(begin_round(s, (cudaStream_t)stream));
    }
    return end_round(s, GXB_DIR_PULL, (cudaStream_t)stream);
}

}  // extern "C"

// the closed round's vote block from the device stripes: changed, next_active, next_units,
// remote_active, max_stat as doubles (counts are exact below 2^53); PageRank's constant
// counters come from the host (every vertex stays active)
__global__ void k_vote_block(const StatStripe* __restrict__ st, double* out, int pagerank,
                             unsigned long long pr_active, unsigned long long pr_units,
                             unsigned long long pr_remote, const unsigned long long* packed) {
    const int lane = threadIdx.x;
    const StatStripe t = st[lane];
    unsigned long long c[4] = {t.changed, t.next_active, t.next_units, t.remote_active};
    unsigned long long m = t.max_stat_bits;
    for (int o = 16; o > 0; o >>= 1) {
        for (int i = 0; i < 4; ++i) c[i] += __shfl_xor_sync(kFull, c[i], o);
        const unsigned long long q = __shfl_xor_sync(kFull, m, o);
        m = q > m ? q : m;
    }
    if (lane == 0) {
        if (pagerank) {
            c[1] = pr_active;
            c[2] = pr_units;
            c[3] = pr_remote;
        }
        for (int i = 0; i < 4; ++i) out[i] = (double)c[i];
        out[4] = packed ? (double)*packed : 0.0;
        out[5] = __longlong_as_double((long long)m);
    }
}

extern "C" {

int gxb_stats_device(gxb_state* s, double* d_out, void* stream) {
    if (!s || !d_out) return fail(GXB_EINVAL, "gxb_stats_device: null argument");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_stats_device: a round is open");
    const bool pr = s->algo == GXB_ALGO_PAGERANK;
    k_vote_block<<<1, 32, 0, (cudaStream_t)stream>>>(s->d_stats, d_out, pr ? 1 : 0, s->g->hi - s->g->lo,
                                                     s->owned_outdeg_sum, s->last.remote_active,
                                                     s->packed_async ? s->d_xscratch : nullptr);
    s->packed_async = false;
    GXB_CUDA(cudaGetLastError());
    return GXB_OK;
}

int gxb_stats_async(gxb_state* s, int on) {
    if (!s) return fail(GXB_EINVAL, "gxb_stats_async: null state");
    if (on && s->algo != GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "gxb_stats_async: PageRank only");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_stats_async: a round is open");
    GXB_CHECK(collect_stats(s));
    if (on && s->timing && !s->kring) {
        s->kring = new cudaEvent_t[3 * gxb_state::kRing]();
        for (int i = 0; i < 3 * gxb_state::kRing; ++i) GXB_CUDA(cudaEventCreate(&s->kring[i]));
    }
    if (!on && s->async_stats && s->kring) GXB_CHECK(drain_kring(s, s->kring_n % gxb_state::kRing));
    s->kring_n = 0;
    s->async_stats = on != 0;
    return GXB_OK;
}

int gxb_round_rollback(gxb_state* s) {
    if (!s) return fail(GXB_EINVAL, "gxb_round_rollback: null state");
    if (s->algo != GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "gxb_round_rollback: PageRank only");
    if (s->in_round || s->iteration == 0) return fail(GXB_ESTATE, "gxb_round_rollback: no closed round");
    // the round wrote only the next rank / contribution buffers: make the previous ones current
    s->cur ^= 1;
    s->iteration--;
    s->stats_pending = false;
    s->timing_pending = false;
    if (s->async_stats && s->kring_n % gxb_state::kRing) s->kring_n--;  // its timing is not a round
    return GXB_OK;
}

int gxb_stats(gxb_state* s, void* stream, gxb_iter_stats* out) {
    if (!s || !out) return fail(GXB_EINVAL, "gxb_stats: null argument");
    (void)stream;
    GXB_CHECK(collect_stats(s));
    *out = s->last;
    return GXB_OK;
}

static int stage(gxb_state* s) {
    if (!s->d_stage) GXB_CHECK(dalloc_t(&s->d_stage, s->g->V * s->arity + 1));
    return GXB_OK;
}

int gxb_read_attrs(gxb_state* s, double* host_out, int owned_only, void* stream) {
    NvtxRange nvtx_("gxb_read_attrs");
    if (!s) return fail(GXB_EINVAL, "gxb_read_attrs: null state");
    gxb_graph* g = s->g;
    const uint64_t V = g->V;
    if (!V) return GXB_OK;
    if (!host_out) return fail(GXB_EINVAL, "gxb_read_attrs: null output");
    cudaStream_t st = (cudaStream_t)stream;
    GXB_CHECK(stage(s));
    k_read_attrs<<<grid_for(V), kBlock, 0, st>>>(s->algo, s->arity, g->d_dense2slot, V, g->lo, g->hi,
                                                 owned_only, s->d_rank[s->cur], s->d_dist_cur, s->d_lab_cur, s->d_stage);
    GXB_CUDA(cudaMemcpyAsync(host_out, s->d_stage, 8 * V * s->arity, cudaMemcpyDeviceToHost, st));
    GXB_CUDA(cudaStreamSynchronize(st));
    return GXB_OK;
}

// install marks of one install: counters zeroed by the first install since the last round
static int install_marks(gxb_state* s, cudaStream_t st, InstallMarks* m) {
    *m = InstallMarks{};
    if (s->algo == GXB_ALGO_PAGERANK) return GXB_OK;
    if (!s->d_xscratch) GXB_CHECK(dalloc_t(&s->d_xscratch, 4));
    if (!s->install_pending) GXB_CUDA(cudaMemsetAsync(s->d_xscratch + 2, 0, 16, st));
    s->install_pending = true;
    m->active = s->d_active[0];
    m->list = s->d_frontier[0];
    m->count = s->d_fcount;
    m->units = s->d_xscratch + 2;
    m->raised = s->d_xscratch + 3;
    return GXB_OK;
}

int gxb_write_attrs(gxb_state* s, const double* host_in, void* stream) {
    NvtxRange nvtx_("gxb_write_attrs");
    if (!s) return fail(GXB_EINVAL, "gxb_write_attrs: null state");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_write_attrs: a round is open");
    gxb_graph* g = s->g;
    const uint64_t V = g->V;
    if (!V) return GXB_OK;
    if (!host_in) return fail(GXB_EINVAL, "gxb_write_attrs: null input");
    cudaStream_t st = (cudaStream_t)stream;
    s->lab_injective = false;  // installed labels need not be distinct
    GXB_CHECK(join_local(s, st));  // installed owned values void a local pass already run
    GXB_CHECK(collect_stats(s));
    GXB_CHECK(stage(s));
    GXB_CUDA(cudaMemcpyAsync(s->d_stage, host_in, 8 * V * s->arity, cudaMemcpyHostToDevice, st));
    uint32_t* d_bad = reinterpret_cast<uint32_t*>(s->d_fcount) + 2;  // scratch word of counter [1]
    GXB_CUDA(cudaMemsetAsync(d_bad, 0, 4, st));
    InstallMarks marks;
    GXB_CHECK(install_marks(s, st, &marks));
    k_write_attrs<<<grid_for(V), kBlock, 0, st>>>(s->algo, s->arity, g->d_dense2slot, V, g->d_outdeg, s->d_stage,
                                                  s->d_rank[s->cur], s->d_contrib[s->cur], s->d_dist_cur, s->d_dist_next,
                                                  s->d_lab_cur, s->d_lab_next, d_bad, s->msg32, marks);
    uint32_t bad = 0;
    GXB_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, st));
    GXB_CUDA(cudaStreamSynchronize(st));
    if (bad) return fail(GXB_ERANGE, "gxb_write_attrs: value not representable on the device");
    return GXB_OK;
}

// ---- asynchronous host staging (no host synchronisation; the caller orders streams) ----
// Two staging buffers per direction let the next step's host->device copy and the
// previous step's device->host copy run on a copy stream while the round computes.
static int stage_pair(gxb_state* s) {
    const gxb_graph* g = s->g;
    const uint64_t nv = s->attrs_scope ? g->owned_present : g->V;
    if (s->stage_n != nv) {
        for (int i = 0; i < 2; ++i) {
            dfree(s->d_stage_in[i]);
            dfree(s->d_stage_out[i]);
            s->d_stage_in[i] = s->d_stage_out[i] = nullptr;
        }
    }
    const uint64_t n = nv * s->arity + 1;
    for (int i = 0; i < 2; ++i) {
        if (!s->d_stage_in[i]) GXB_CHECK(dalloc_t(&s->d_stage_in[i], n));
        if (!s->d_stage_out[i]) GXB_CHECK(dalloc_t(&s->d_stage_out[i], n));
    }
    s->stage_n = nv;
    return GXB_OK;
}

// vertex order of the staging buffers: every present id, or the owned ones (both ascending)
static void stage_order(const gxb_state* s, const uint32_t** d2s, uint64_t* n) {
    const gxb_graph* g = s->g;
    if (s->attrs_scope) {
        *d2s = g->d_owned_d2s;
        *n = g->owned_present;
    } else {
        *d2s = g->d_dense2slot;
        *n = g->V;
    }
}

int gxb_attrs_scope(gxb_state* s, int owned_only) {
    if (!s || (owned_only != 0 && owned_only != 1)) return fail(GXB_EINVAL, "gxb_attrs_scope: bad argument");
    GXB_CUDA(cudaSetDevice(s->g->ctx->device));
    if (owned_only) GXB_CHECK(build_owned_order(s->g));
    s->attrs_scope = owned_only;
    return stage_pair(s);
}

int gxb_attrs_h2d(gxb_state* s, const double* host_in, int buf, void* stream) {
    if (!s || !host_in || buf < 0 || buf > 1) return fail(GXB_EINVAL, "gxb_attrs_h2d: bad argument");
    GXB_CHECK(stage_pair(s));
    GXB_CUDA(cudaMemcpyAsync(s->d_stage_in[buf], host_in, 8 * s->stage_n * s->arity, cudaMemcpyHostToDevice,
                             (cudaStream_t)stream));
    return GXB_OK;
}

int gxb_attrs_install(gxb_state* s, int buf, void* stream) {
    if (!s || buf < 0 || buf > 1) return fail(GXB_EINVAL, "gxb_attrs_install: bad argument");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_attrs_install: a round is open");
    s->lab_injective = false;
    GXB_CHECK(join_local(s, (cudaStream_t)stream));  // installed values void a local pass already run
    GXB_CHECK(stage_pair(s));
    gxb_graph* g = s->g;
    const uint32_t* d2s;
    uint64_t n;
    stage_order(s, &d2s, &n);
    if (!n) return GXB_OK;
    uint32_t* d_bad = reinterpret_cast<uint32_t*>(s->d_fcount) + 2;  // sticky flag, checked by gxb_attrs_check
    InstallMarks marks;
    GXB_CHECK(install_marks(s, (cudaStream_t)stream, &marks));
    k_write_attrs<<<grid_for(n), kBlock, 0, (cudaStream_t)stream>>>(
        s->algo, s->arity, d2s, n, g->d_outdeg, s->d_stage_in[buf], s->d_rank[s->cur], s->d_contrib[s->cur],
        s->d_dist_cur, s->d_dist_next, s->d_lab_cur, s->d_lab_next, d_bad, s->msg32, marks);
    GXB_CUDA(cudaGetLastError());
    return GXB_OK;
}

int gxb_attrs_extract(gxb_state* s, int buf, void* stream) {
    if (!s || buf < 0 || buf > 1) return fail(GXB_EINVAL, "gxb_attrs_extract: bad argument");
    GXB_CHECK(stage_pair(s));
    gxb_graph* g = s->g;
    const uint32_t* d2s;
    uint64_t n;
    stage_order(s, &d2s, &n);
    if (!n) return GXB_OK;
    k_read_attrs<<<grid_for(n), kBlock, 0, (cudaStream_t)stream>>>(s->algo, s->arity, d2s, n, g->lo, g->hi, 0,
                                                                   s->d_rank[s->cur], s->d_dist_cur, s->d_lab_cur,
                                                                   s->d_stage_out[buf]);
    GXB_CUDA(cudaGetLastError());
    return GXB_OK;
}

int gxb_attrs_d2h(gxb_state* s, double* host_out, int buf, void* stream) {
    if (!s || !host_out || buf < 0 || buf > 1) return fail(GXB_EINVAL, "gxb_attrs_d2h: bad argument");
    GXB_CHECK(stage_pair(s));
    GXB_CUDA(cudaMemcpyAsync(host_out, s->d_stage_out[buf], 8 * s->stage_n * s->arity, cudaMemcpyDeviceToHost,
                             (cudaStream_t)stream));
    return GXB_OK;
}

int gxb_profile_enable(gxb_state* s, int on) {
    if (!s) return fail(GXB_EINVAL, "gxb_profile_enable: null state");
    if (on && !s->kev[0]) {
        for (int i = 0; i < 3; ++i) GXB_CUDA(cudaEventCreate(&s->kev[i]));
    }
    s->timing = on != 0;
    return GXB_OK;
}

int gxb_profile_read(gxb_state* s, gxb_profile* out, int reset) {
    if (!s || !out) return fail(GXB_EINVAL, "gxb_profile_read: null argument");
    GXB_CHECK(collect_stats(s));
    out->main_kernel_ms = s->kernel_ms;
    out->rest_ms = s->rest_ms;
    out->main_kernel_launches = s->kernel_launches;
    out->kernels_launched = s->launches;
    out->iterations = s->iteration;
    if (reset) {
        s->kernel_ms = 0.0;
        s->rest_ms = 0.0;
        s->kernel_launches = 0;
        s->launches = 0;
    }
    return GXB_OK;
}

}  // extern "C"
