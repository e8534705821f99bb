// gxb_lp.cu — LabelPropagation mode reduction (K3).
//
// Semantics (A/algorithms.py:174-205, run_reference 318-341): a destination's
// multiset is the labels of its ACTIVE in-neighbours, one per edge (duplicates
// and self-loops count); no message -> keep the label and go inactive;
// otherwise take the most frequent label, ties to the smallest label, and be
// active iff it changed. Counts are exact integers, so the result is bit-exact.
//
// Two regimes over the degree-sorted slots (same bins as the pull merge):
//  * in-degree <= 4G with G lanes per destination (G = 1..32): the group stages
//    its labels in shared memory and every lane counts its candidates against
//    the staged multiset; the group takes the max of (count << 32 | ~label).
//  * in-degree > kChunkMinDeg: warps stream kChunkEdges-edge chunks, pre-merge
//    equal labels inside the warp with __match_any_sync, and fold (label, count)
//    into a per-destination open-addressing table in global memory (L2
//    atomics); every update also raises the destination's running packed
//    argmax (count << 32 | ~label) with atomicMax, so no table scan is needed;
//    a last pass applies and the tables are reset with memsets.
#include <algorithm>
#include <vector>

#include "gxb_state.cuh"

namespace gxb {

constexpr uint32_t kEmpty = 0xFFFFFFFFu;

struct LpHub {
    uint64_t* tab_off;   // per chunked slot: first entry
    uint32_t* tab_mask;  // per chunked slot: size - 1 (power of two)
    uint32_t* keys;
    uint32_t* counts;
    unsigned long long* best;  // per chunked slot: packed (count << 32 | ~label), 0 = no message
    uint64_t entries;
};

struct LpScratch {
    LpHub hub;
    uint64_t chunk_end = 0;
};

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// fold (label, c) into a destination's table; returns the label's new count
__device__ __forceinline__ uint32_t table_add(uint32_t* keys, uint32_t* counts, uint64_t base, uint32_t mask,
                                              uint32_t label, uint32_t c) {
    uint32_t i = mix32(label) & mask;
    while (true) {
        const uint64_t at = base + i;
        uint32_t k = __ldcg(keys + at);
        if (k == kEmpty) {
            k = atomicCAS(keys + at, kEmpty, label);
            if (k == kEmpty) k = label;
        }
        if (k == label) return atomicAdd(counts + at, c) + c;
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
};

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
    uint32_t* my = buf + grp * kCap;
    for (uint32_t i = gl; i < deg; i += G) {
        const uint32_t s = __ldg(L.in_src + beg + i);
        my[i] = bit_test(L.active_cur, s) ? __ldg(L.lab_cur + s) : kEmpty;
    }
    __syncwarp();
    unsigned long long best = 0ull;
    for (uint32_t i = gl; i < deg; i += G) {
        const uint32_t lab = my[i];
        if (lab == kEmpty) continue;
        uint32_t c = 0;
        for (uint32_t j = 0; j < deg; ++j) c += (my[j] == lab) ? 1u : 0u;
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

// large destinations: warp-aggregated inserts into the per-slot global table
__device__ __forceinline__ void lp_chunk(const LpLaunch& L, uint64_t item) {
    const int lane = threadIdx.x & 31;
    const uint32_t rel = __ldg(L.item_slot + item);
    const uint64_t beg = __ldg(L.item_begin + item);
    const uint64_t end = min(beg + (uint64_t)kChunkEdges, __ldg(L.in_off + rel + 1));
    const uint64_t base = __ldg(L.hub.tab_off + rel);
    const uint32_t mask = __ldg(L.hub.tab_mask + rel);
    for (uint64_t e0 = beg; e0 < end; e0 += 32) {
        const uint64_t e = e0 + lane;
        bool ok = false;
        uint32_t lab = 0;
        if (e < end) {
            const uint32_t s = __ldg(L.in_src + e);
            if (bit_test(L.active_cur, s)) {
                ok = true;
                lab = __ldg(L.lab_cur + s);
            }
        }
        const unsigned long long key = ok ? (unsigned long long)lab : (0x100000000ull | (unsigned)lane);
        const unsigned m = __match_any_sync(kFull, key);
        if (ok && lane == __ffs(m) - 1) {
            // the running argmax: a label's packed (count, ~label) only grows, so the max over
            // every update equals the max over final counts
            const uint32_t nc = table_add(L.hub.keys, L.hub.counts, base, mask, lab, __popc(m));
            const unsigned long long pk = ((unsigned long long)nc << 32) | (unsigned long long)(~lab);
            if (pk > __ldcg(L.hub.best + rel)) atomicMax(L.hub.best + rel, pk);
        }
    }
}

__global__ void __launch_bounds__(kBlock) k_lp_pull(const LpLaunch L) {
    __shared__ uint32_t buf[4 * kBlock];
    LocalStats st;
    unsigned b = blockIdx.x;
    if (b < L.chunk_blocks) {
        const uint64_t item = (uint64_t)b * (kBlock / 32) + (threadIdx.x >> 5);
        if (item < L.num_items) lp_chunk(L, item);
        return;  // chunked slots are applied by k_lp_hub_apply
    }
    b -= L.chunk_blocks;
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

static uint64_t next_pow2(uint64_t x) {
    uint64_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

static void lp_free(LpScratch* S) {
    if (!S) return;
    LpHub& H = S->hub;
    dfree(H.tab_off);
    dfree(H.tab_mask);
    dfree(H.keys);
    dfree(H.counts);
    dfree(H.best);
    delete S;
}

static int lp_setup(gxb_state* s, cudaStream_t st) {
    const gxb_graph* g = s->g;
    const PullPlan& P = g->plan;
    LpScratch* S = new LpScratch();
    S->chunk_end = P.chunk_end;
    LpHub& H = S->hub;
    std::vector<uint64_t> off(P.chunk_end + 1);
    std::vector<uint32_t> mask(P.chunk_end + 1);
    uint64_t acc = 0;
    for (uint64_t r = 0; r < P.chunk_end; ++r) {
        const uint64_t size = std::max<uint64_t>(256, next_pow2(2ull * g->h_indeg_sorted[r]));
        off[r] = acc;
        mask[r] = (uint32_t)(size - 1);
        acc += size;
    }
    H.entries = acc;
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
    if (rc == GXB_OK) rc = dalloc_t(&H.keys, acc + 1);
    if (rc == GXB_OK) rc = dalloc_t(&H.counts, acc + 1);
    if (rc == GXB_OK) rc = dalloc_t(&H.best, P.chunk_end + 1);
    if (rc == GXB_OK) {
        cudaMemsetAsync(H.keys, 0xFF, 4 * (acc + 1), st);
        cudaMemsetAsync(H.counts, 0, 4 * (acc + 1), st);
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

extern "C" void gxb_lp_free(gxb_state* s) {
    if (s && s->d_lp_scratch) {
        lp_free(reinterpret_cast<LpScratch*>(s->d_lp_scratch));
        s->d_lp_scratch = nullptr;
    }
}

extern "C" int gxb_lp_prepare(gxb_state* s, cudaStream_t st) {
    if (!s->d_lp_scratch) GXB_CHECK(lp_setup(s, st));
    return GXB_OK;
}

extern "C" int gxb_lp_pull(gxb_state* s, cudaStream_t st) {
    if (!s->d_lp_scratch) GXB_CHECK(lp_setup(s, st));
    LpScratch* S = reinterpret_cast<LpScratch*>(s->d_lp_scratch);
    const gxb_graph* g = s->g;
    const PullPlan& P = g->plan;
    LpLaunch L;
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
    if (grid) k_lp_pull<<<grid, kBlock, 0, st>>>(L);
    if (S->chunk_end) {
        k_lp_hub_apply<<<grid_for(S->chunk_end), kBlock, 0, st>>>(L, S->chunk_end);
        // empty the tables for the next round (plain memsets: no read-back of the tables)
        GXB_CUDA(cudaMemsetAsync(S->hub.keys, 0xFF, 4 * S->hub.entries, st));
        GXB_CUDA(cudaMemsetAsync(S->hub.counts, 0, 4 * S->hub.entries, st));
    }
    GXB_CUDA(cudaGetLastError());
    return GXB_OK;
}
