// gxb_store.cu — daemon lifecycle and the device-resident graph store (K0).
//
// Replaces `partition_graph` (A/graph.py:175-212), the per-partition
// vertex/edge/ve_map tables (A/graph.py:93-106), the global out-degree table
// (A/graph.py:203-210) and the static remote-destination index
// (A/agent.py:156-166). Everything is built on the device:
//   present-id bitmap -> popcount ranks (vertex set = ids present in edges,
//   A/graph.py:163-164) -> in/out degrees (duplicates and self-loops count) ->
//   degree-sorted slot order (in-degree descending, ties by id) -> relabelled
//   edges -> destination-range partition balanced by in-edges (Lemma 2 with
//   equal c_j, A/balancer.py:79-98) -> CSC of the owned destinations sorted by
//   (dst, src) -> optional push CSR -> degree-bin plan of the pull merge.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "gxb_internal.cuh"

namespace gxb {

static thread_local std::string g_last_error;

Options& options() {
    static Options o;
    static bool init = false;
    if (!init) {
        init = true;
        if (const char* e = getenv("GXB_TILE_MINBLOCKS")) o.tile_minblocks = atol(e);
        if (const char* e = getenv("GXB_L2_HOT_MB")) o.l2_hot_mb = atol(e);
        if (const char* e = getenv("GXB_PUSH_ALPHA")) o.push_alpha = atol(e);
        if (const char* e = getenv("GXB_PULL_KERNEL")) o.pull_kernel = std::string(e) == "binned" ? 1 : 0;
        if (const char* e = getenv("GXB_PR_MESSAGE_BITS")) o.pr_message_bits = atol(e) == 32 ? 32 : 64;
        if (const char* e = getenv("GXB_PR_HUB_SLOTS")) o.pr_hub_slots = std::min(28672L, std::max(0L, atol(e)));
        if (const char* e = getenv("GXB_TILE_ASYNC")) o.tile_async = atol(e) ? 1 : 0;
        if (const char* e = getenv("GXB_PIPELINE_APPLY")) o.pipeline_apply = atol(e) ? 1 : 0;
        if (const char* e = getenv("GXB_XCHUNK_POWER")) o.xchunk_power = std::min(4L, std::max(1L, atol(e)));
        if (const char* e = getenv("GXB_EXCHANGE_CHUNKS")) o.exchange_chunks = std::min(64L, std::max(1L, atol(e)));
        if (const char* e = getenv("GXB_OVERLAP_RESERVE_SMS")) o.overlap_reserve_sms = std::min(140L, std::max(0L, atol(e)));
        if (const char* e = getenv("GXB_SPLIT_OVERLAP")) o.split_overlap = atol(e) ? 1 : 0;
        if (const char* e = getenv("GXB_SPLIT_RESERVE_SMS")) o.split_reserve_sms = std::min(140L, std::max(0L, atol(e)));
    }
    return o;
}

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return GXB_ECUDA;
}

int dalloc(void** p, size_t bytes) {
    *p = nullptr;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return fail(GXB_ENOMEM, std::string("cudaMalloc(") + std::to_string(bytes) + "): " +
                                    cudaGetErrorString(e));
    }
    return GXB_OK;
}
void dfree(void* p) {
    if (p) cudaFree(p);
}

// ------------------------------------------------------------------ kernels

__global__ void k_max_id(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t n,
                         uint32_t* out) {
    uint32_t m = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        m = max(m, max(a[i], b[i]));
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void k_mark_present(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                               uint64_t n, uint32_t* bm) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t x = a[i], y = b[i];
        atomicOr(bm + (x >> 5), 1u << (x & 31));
        atomicOr(bm + (y >> 5), 1u << (y & 31));
    }
}

__global__ void k_word_popc(const uint32_t* __restrict__ bm, uint64_t words, uint32_t* cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words;
         i += (uint64_t)gridDim.x * blockDim.x)
        cnt[i] = __popc(bm[i]);
}

// dense index (rank among present ids) of each present id; ids ascending
__global__ void k_emit_ids(const uint32_t* __restrict__ bm, const uint32_t* __restrict__ prefix,
                           uint64_t words, uint32_t* ids) {
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words;
         w += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t bits = bm[w];
        uint32_t r = prefix[w];
        while (bits) {
            const int b = __ffs(bits) - 1;
            ids[r++] = (uint32_t)(w * 32 + b);
            bits &= bits - 1;
        }
    }
}

__device__ __forceinline__ uint32_t rank_of(const uint32_t* bm, const uint32_t* prefix, uint32_t id) {
    const uint32_t w = id >> 5;
    const uint32_t below = bm[w] & ((1u << (id & 31)) - 1u);
    return prefix[w] + __popc(below);
}

// edges -> dense indices in place, degrees
__global__ void k_rank_edges(uint32_t* src, uint32_t* dst, uint64_t n, const uint32_t* __restrict__ bm,
                             const uint32_t* __restrict__ prefix, uint32_t* outdeg, uint32_t* indeg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = rank_of(bm, prefix, src[i]);
        const uint32_t d = rank_of(bm, prefix, dst[i]);
        src[i] = s;
        dst[i] = d;
        atomicAdd(outdeg + s, 1u);
        atomicAdd(indeg + d, 1u);
    }
}

__global__ void k_iota(uint32_t* a, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        a[i] = (uint32_t)i;
}

// slot order -> inverse map, per-slot id and out-degree (padding slots: id kNone, degree 0)
__global__ void k_slot_tables(const uint32_t* __restrict__ slot2dense, uint64_t S,
                              const uint32_t* __restrict__ ids_dense,
                              const uint32_t* __restrict__ outdeg_dense, uint32_t* dense2slot,
                              uint32_t* slot2id, uint32_t* outdeg_slot) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < S;
         s += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t d = slot2dense[s];
        if (d == 0xFFFFFFFFu) {
            slot2id[s] = 0xFFFFFFFFu;
            outdeg_slot[s] = 0;
            continue;
        }
        dense2slot[d] = (uint32_t)s;
        slot2id[s] = ids_dense[d];
        outdeg_slot[s] = outdeg_dense[d];
    }
}

__global__ void k_relabel(uint32_t* src, uint32_t* dst, uint64_t n, const uint32_t* __restrict__ d2s) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        src[i] = d2s[src[i]];
        dst[i] = d2s[dst[i]];
    }
}

__device__ __forceinline__ int owner_of(const uint64_t* bounds, int nparts, uint32_t slot) {
    int p = 0;
    while (p + 1 < nparts && (uint64_t)slot >= bounds[p + 1]) ++p;
    return p;
}

// remote-source bitmap and the CSC / CSR keys of the owned destinations
__global__ void k_keys(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, uint64_t n,
                       const uint64_t* __restrict__ bounds, int nparts, int part, uint64_t lo,
                       uint64_t owned, uint64_t V, uint32_t* remote_bm, uint64_t* csc_key,
                       uint64_t* csr_key) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = src[i], d = dst[i];
        const int od = owner_of(bounds, nparts, d);
        if (nparts > 1 && od != owner_of(bounds, nparts, s)) {
            const uint32_t m = 1u << (s & 31);
            if (!(remote_bm[s >> 5] & m)) atomicOr(remote_bm + (s >> 5), m);
        }
        const bool mine = (od == part);
        csc_key[i] = mine ? ((uint64_t)(d - lo) << 32 | s) : (owned << 32);
        if (csr_key) csr_key[i] = mine ? ((uint64_t)s << 32 | d) : ((uint64_t)V << 32);
    }
}

// offsets of a key-sorted COO: off[k] = first index whose (key >> 32) >= k, k in [0, nseg]
__global__ void k_offsets(const uint64_t* __restrict__ keys, uint64_t n, uint64_t nseg, uint64_t* off) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t cur = (i < n) ? (keys[i] >> 32) : nseg;
        const uint64_t prev = (i == 0) ? 0 : ((keys[i - 1] >> 32) + 1);
        const uint64_t stop = cur < nseg ? cur : nseg;
        for (uint64_t k = prev; k <= stop; ++k) off[k] = i;
    }
}

__global__ void k_fill_u64(uint64_t* a, uint64_t n, uint64_t v) {
    for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) a[i] = v;
}

// lane-chunk tables of the warp tiles: lane l of tile t covers edges
// [start_t + kTileK l, start_t + kTileK (l + 1)) clipped to the tile; its slot
// (relative) is the one containing the first edge, and bit j of its mask marks a
// position that closes a destination segment
__global__ void k_lane_slot(const uint64_t* __restrict__ off, uint64_t nz, const uint64_t* __restrict__ tstart,
                            uint64_t nchunks, uint32_t* out, uint8_t* mask) {
    for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < nchunks;
         c += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = c >> 5, l = c & 31;
        const uint64_t e = tstart[t] + l * kTileK, tend = tstart[t + 1];
        if (e >= tend) {
            out[c] = 0;
            mask[c] = 0;
            continue;
        }
        uint64_t lo = 0, hi = nz;  // last s with off[s] <= e
        while (hi - lo > 1) {
            const uint64_t mid = (lo + hi) >> 1;
            if (off[mid] <= e) lo = mid; else hi = mid;
        }
        out[c] = (uint32_t)lo;
        uint32_t m = 0;
        for (int k = 1; k <= kTileK; ++k) {  // every in-degree >= 1 here: at most kTileK ends
            const uint64_t b = (lo + k <= nz) ? off[lo + k] : ~0ull;
            if (b > e && b <= e + kTileK && b <= tend) m |= 1u << (uint32_t)(b - e - 1);
        }
        mask[c] = (uint8_t)m;
    }
}

// (partition of the dense id) << 32 | ~in-degree: ascending = by partition, then in-degree descending
__global__ void k_part_keys(const uint32_t* __restrict__ indeg, uint64_t V, const uint64_t* __restrict__ idb,
                            int nparts, uint64_t* keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < V; i += (uint64_t)gridDim.x * blockDim.x) {
        int p = 0;
        while (p + 1 < nparts && i >= idb[p + 1]) ++p;
        keys[i] = ((uint64_t)p << 32) | (uint64_t)(0xFFFFFFFFu - indeg[i]);
    }
}

__global__ void k_gather_indeg(const uint32_t* __restrict__ slot2dense, const uint32_t* __restrict__ indeg,
                               uint64_t V, uint32_t* out) {
    for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s < V; s += (uint64_t)gridDim.x * blockDim.x)
        out[s] = indeg[slot2dense[s]];
}

// round-robin deal of the degree-sorted order: position i -> block i % n, rank i / n
// (blocks of equal size B; the unfilled tail slot of a block stays a padding slot)
__global__ void k_deal(const uint32_t* __restrict__ s2d, const uint32_t* __restrict__ indeg, uint64_t V, int n,
                       uint64_t B, uint32_t* s2d_out, uint32_t* indeg_out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < V; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t pos = (i % n) * B + i / n;
        s2d_out[pos] = s2d[i];
        indeg_out[pos] = indeg[i];
    }
}

static uint64_t round_up(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }

__global__ void k_pack_sw(const uint32_t* __restrict__ src, const uint32_t* __restrict__ w, uint64_t n,
                          uint32_t shift, uint32_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (src[i] << shift) | w[i];
}

__global__ void k_low32(const uint64_t* __restrict__ keys, uint64_t n, uint32_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (uint32_t)keys[i];
}

static int bits_for(uint64_t v) {
    int b = 0;
    while (b < 64 && (v >> b) != 0) ++b;
    return b;
}

static unsigned grid_e(uint64_t n) { return grid_for(n, kBlock, 148ull * 32); }

// radix sort of 64-bit keys (and optional u32 values) over [0, end_bit)
static int sort_pairs(uint64_t* keys, uint64_t* keys_alt, uint32_t* vals, uint32_t* vals_alt,
                      uint64_t n, int end_bit, cudaStream_t st, uint64_t** keys_out,
                      uint32_t** vals_out) {
    cub::DoubleBuffer<uint64_t> kb(keys, keys_alt);
    cub::DoubleBuffer<uint32_t> vb(vals, vals_alt);
    size_t temp = 0;
    // CUB's num_items is int-typed for the legacy overload; use the 64-bit
    // NumItemsT template parameter.
    if (vals) {
        GXB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, kb, vb, (int64_t)n, 0, end_bit, st));
    } else {
        GXB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, temp, kb, (int64_t)n, 0, end_bit, st));
    }
    void* tmp = nullptr;
    GXB_CHECK(dalloc(&tmp, temp));
    cudaError_t e;
    if (vals) e = cub::DeviceRadixSort::SortPairs(tmp, temp, kb, vb, (int64_t)n, 0, end_bit, st);
    else e = cub::DeviceRadixSort::SortKeys(tmp, temp, kb, (int64_t)n, 0, end_bit, st);
    cudaStreamSynchronize(st);
    dfree(tmp);
    if (e != cudaSuccess) return cuda_fail(e, "cub::DeviceRadixSort");
    *keys_out = kb.Current();
    *vals_out = vals ? vb.Current() : nullptr;
    return GXB_OK;
}

template <typename T>
static int exclusive_scan(const T* in, T* out, uint64_t n, cudaStream_t st) {
    size_t temp = 0;
    GXB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp, in, out, (int64_t)n, st));
    void* tmp = nullptr;
    GXB_CHECK(dalloc(&tmp, temp));
    cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, temp, in, out, (int64_t)n, st);
    cudaStreamSynchronize(st);
    dfree(tmp);
    if (e != cudaSuccess) return cuda_fail(e, "cub::DeviceScan");
    return GXB_OK;
}

// RAII list of scratch buffers
struct Scratch {
    std::vector<void*> ptrs;
    ~Scratch() {
        for (void* p : ptrs) dfree(p);
    }
    template <typename T>
    int get(T** p, size_t n) {
        int rc = dalloc_t(p, n);
        if (rc == GXB_OK) ptrs.push_back(*p);
        return rc;
    }
};

static void graph_release(gxb_graph* g) {
    dfree(g->d_slot2id);
    dfree(g->d_dense2slot);
    dfree(g->d_outdeg);
    dfree(g->d_remote_src);
    dfree(g->d_in_off);
    dfree(g->d_in_src);
    dfree(g->d_in_w);
    dfree(g->d_in_sw);
    dfree(g->d_owned_d2s);
    dfree(g->d_out_off);
    dfree(g->d_out_dst);
    dfree(g->d_out_w);
    dfree(g->plan.d_item_slot);
    dfree(g->plan.d_item_begin);
    dfree(g->plan.d_item_first);
    dfree(g->plan.d_item_count);
    dfree(g->plan.d_slot_arrive);
    dfree(g->tiles.d_lane_slot);
    dfree(g->d_xsend_idx);
    dfree(g->d_xrecv_idx);
    dfree(g->tiles.d_tile_start);
    dfree(g->tiles.d_lane_mask);
    dfree(g->tiles.d_tile_head);
    dfree(g->tiles.d_tile_tail);
    dfree(g->tiles.d_span_first);
    dfree(g->tiles.d_span_count);
    dfree(g->tiles.d_span_pbase);
    dfree(g->tiles.d_span_slot);
}

void shadow_graph_free(gxb_graph* g) {
    if (!g) return;
    graph_release(g);
    delete g;
}

// warp-tile plan of the edge-balanced pull merge: kTileEdges edges per warp;
// slots crossing a tile boundary ("spans") combine per-tile partials
// slot bound of exchange chunk k of K: owned * (k / K)^p (p = option xchunk_power, 1..4).
// Slots are in-degree sorted, so the first chunk is the short hub-heavy one; a pipelined
// round runs chunks hubs-last and only the last chunk's Apply is left exposed.
uint64_t xchunk_bound(uint64_t owned, int k, int K) {
    uint64_t num = 1, den = 1;
    for (int i = 0; i < options().xchunk_power; ++i) {
        num *= (uint64_t)k;
        den *= (uint64_t)K;
    }
    return (uint64_t)((unsigned __int128)owned * num / den);  // exact: peers recompute it
}

int build_tile_plan(gxb_graph* g, cudaStream_t st) {
    TilePlan& T = g->tiles;
    const std::vector<uint32_t>& deg = g->h_indeg_sorted;
    const uint64_t owned = deg.size();
    uint64_t nz = 0;
    while (nz < owned && deg[nz] > 0) ++nz;
    T.nz_slots = nz;
    // Exchange chunks (multi-GPU pipeline shuffle): the owned slots are cut into K chunks
    // at fractions (k/K)^p of the owned count (xchunk_bound), so chunk 0 holds the few hub
    // slots (most of the edges) and the last chunk the many tail slots. Every rank cuts its
    // own block with the same formula, so peers know each other's chunk ranges.
    const bool chunked = g->nparts > 1 || options().pipeline_apply;
    const int K = std::max(1, chunked ? (int)options().exchange_chunks : 1);
    T.num_xchunks = K;
    T.xchunk_slot.assign(K + 1, 0);
    for (int k = 0; k <= K; ++k) T.xchunk_slot[k] = xchunk_bound(owned, k, K);
    // Fixed tiles of kTileEdges edges restarting at every chunk (measured faster than
    // slot-aligned variable tiles: those leave lanes idle at every cut); slots crossing a
    // tile boundary become spans whose per-tile partials are folded by k_span_fold.
    std::vector<uint64_t> off(nz + 1, 0);
    for (uint64_t s = 0; s < nz; ++s) off[s + 1] = off[s] + deg[s];
    const uint64_t E = off[nz];
    std::vector<uint64_t> starts;
    starts.reserve(E / kTileEdges + K + 2);
    T.xchunk_tile.assign(K + 1, 0);
    for (int k = 0; k < K; ++k) {
        T.xchunk_tile[k] = starts.size();
        const uint64_t e0 = off[std::min<uint64_t>(T.xchunk_slot[k], nz)];
        const uint64_t e1 = off[std::min<uint64_t>(T.xchunk_slot[k + 1], nz)];
        for (uint64_t pos = e0; pos < e1; pos += kTileEdges) starts.push_back(pos);
    }
    T.num_tiles = starts.size();
    T.xchunk_tile[K] = T.num_tiles;
    starts.push_back(E);
    // span table: slots crossing a tile boundary (hubs); never across chunks
    std::vector<uint32_t> head(T.num_tiles + 1, kNone), tail(T.num_tiles + 1, kNone);
    std::vector<uint32_t> sfirst, scount, sslot;
    std::vector<uint64_t> spbase;
    T.xchunk_span.assign(K + 1, 0);
    uint64_t pbase = 0, t = 0;
    int kc = 0;
    for (uint64_t s = 0; s < nz; ++s) {
        while (kc < K && s >= T.xchunk_slot[kc + 1]) T.xchunk_span[++kc] = sfirst.size();
        while (t + 1 < T.num_tiles && starts[t + 1] <= off[s]) ++t;
        uint64_t t1 = t;
        while (t1 + 1 < T.num_tiles && starts[t1 + 1] < off[s + 1]) ++t1;
        if (t1 == t) continue;
        const uint32_t k = (uint32_t)sfirst.size();
        sfirst.push_back((uint32_t)t);
        scount.push_back((uint32_t)(t1 - t + 1));
        sslot.push_back((uint32_t)s);
        spbase.push_back(pbase);
        pbase += t1 - t + 1;
        tail[t] = k;
        for (uint64_t u = t + 1; u <= t1; ++u) head[u] = k;
        for (uint64_t u = t + 1; u < t1; ++u) tail[u] = k;
        t = t1;
    }
    while (kc < K) T.xchunk_span[++kc] = sfirst.size();
    T.num_spans = sfirst.size();
    T.num_partials = pbase;
    int rc = GXB_OK;
    auto up = [&](auto** d, const auto& h) {
        if (rc != GXB_OK) return;
        rc = dalloc_t(d, h.size() + 1);
        if (rc == GXB_OK && !h.empty() &&
            cudaMemcpyAsync(*d, h.data(), sizeof(h[0]) * h.size(), cudaMemcpyHostToDevice, st) != cudaSuccess)
            rc = fail(GXB_ECUDA, "tile plan upload");
    };
    up(&T.d_tile_start, starts);
    up(&T.d_tile_head, head);
    up(&T.d_tile_tail, tail);
    up(&T.d_span_first, sfirst);
    up(&T.d_span_count, scount);
    up(&T.d_span_pbase, spbase);
    up(&T.d_span_slot, sslot);
    GXB_CHECK(rc);
    const uint64_t nchunks = T.num_tiles * 32;
    GXB_CHECK(dalloc_t(&T.d_lane_slot, nchunks + 32));
    GXB_CHECK(dalloc_t(&T.d_lane_mask, nchunks + 32));
    if (nchunks)
        k_lane_slot<<<grid_e(nchunks), kBlock, 0, st>>>(g->d_in_off, nz, T.d_tile_start, nchunks, T.d_lane_slot,
                                                         T.d_lane_mask);
    GXB_CUDA(cudaStreamSynchronize(st));
    return GXB_OK;
}

// degree-bin plan of the pull merge (host side, from the owned in-degrees)
int build_pull_plan(gxb_graph* g, cudaStream_t st) {
    PullPlan& P = g->plan;
    const uint64_t owned = g->hi - g->lo;
    const std::vector<uint32_t>& deg = g->h_indeg_sorted;  // descending
    // first slot with degree <= t
    auto first_le = [&](uint64_t t) -> uint64_t {
        return (uint64_t)(std::lower_bound(deg.begin(), deg.end(), (uint32_t)t,
                                           [](uint32_t a, uint32_t b) { return a > b; }) -
                          deg.begin());
    };
    P.chunk_end = first_le(kChunkMinDeg);
    // group bin k (G = 1 << k) takes degrees in (2^(k+1), 2^(k+2)], k = 0 takes [0, 4]
    for (int k = kNumGroupBins - 1; k >= 0; --k) {
        const uint64_t lower = (k == 0) ? 0 : (1ull << (k + 1));
        P.group_end[k] = (k == 0) ? owned : first_le(lower);
    }
    // chunk items
    std::vector<uint32_t> islot, ifirst, icount;
    std::vector<uint64_t> ibegin;
    uint64_t off = 0;
    for (uint64_t s = 0; s < P.chunk_end; ++s) {
        const uint32_t d = deg[s];
        const uint32_t n = (d + kChunkEdges - 1) / kChunkEdges;
        const uint32_t first = (uint32_t)islot.size();
        for (uint32_t k = 0; k < n; ++k) {
            islot.push_back((uint32_t)s);
            ibegin.push_back(off + (uint64_t)k * kChunkEdges);
            ifirst.push_back(first);
            icount.push_back(n);
        }
        off += d;
    }
    P.num_items = islot.size();
    GXB_CHECK(dalloc_t(&P.d_item_slot, P.num_items));
    GXB_CHECK(dalloc_t(&P.d_item_begin, P.num_items));
    GXB_CHECK(dalloc_t(&P.d_item_first, P.num_items));
    GXB_CHECK(dalloc_t(&P.d_item_count, P.num_items));
    GXB_CHECK(dalloc_t(&P.d_slot_arrive, P.chunk_end));
    if (P.num_items) {
        GXB_CUDA(cudaMemcpyAsync(P.d_item_slot, islot.data(), 4 * P.num_items, cudaMemcpyHostToDevice, st));
        GXB_CUDA(cudaMemcpyAsync(P.d_item_begin, ibegin.data(), 8 * P.num_items, cudaMemcpyHostToDevice, st));
        GXB_CUDA(cudaMemcpyAsync(P.d_item_first, ifirst.data(), 4 * P.num_items, cudaMemcpyHostToDevice, st));
        GXB_CUDA(cudaMemcpyAsync(P.d_item_count, icount.data(), 4 * P.num_items, cudaMemcpyHostToDevice, st));
    }
    GXB_CUDA(cudaMemsetAsync(P.d_slot_arrive, 0, 4 * (P.chunk_end + 1), st));
    GXB_CUDA(cudaStreamSynchronize(st));
    return GXB_OK;
}

// ---- needed-only mirror exchange lists (per-peer need masks) ----
// send list to peer q: my owned slots that are the source of an edge into q's
// destinations; recv list from peer p: p's owned slots that are sources of my CSC.
// Both are sorted by slot, so my send list to q is exactly q's recv list from me.
__global__ void k_send_keys(const uint32_t* __restrict__ src, const uint32_t* __restrict__ dst, uint64_t n,
                            const uint64_t* __restrict__ bounds, int nparts, int part, uint64_t* keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = src[i], d = dst[i];
        const int os = owner_of(bounds, nparts, s), od = owner_of(bounds, nparts, d);
        keys[i] = (os == part && od != part) ? ((uint64_t)od << 32 | s) : ((uint64_t)nparts << 32);
    }
}

__global__ void k_recv_keys(const uint32_t* __restrict__ in_src, uint64_t n, const uint64_t* __restrict__ bounds,
                            int nparts, int part, uint64_t* keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = in_src[i];
        const int os = owner_of(bounds, nparts, s);
        keys[i] = (os != part) ? ((uint64_t)os << 32 | s) : ((uint64_t)nparts << 32);
    }
}

static int unique_segments(uint64_t* keys, uint64_t* alt, uint64_t n, int nparts, cudaStream_t st,
                           uint32_t** d_idx, std::vector<uint64_t>& off_host) {
    uint64_t* kout = nullptr;
    uint32_t* vdummy = nullptr;
    GXB_CHECK(sort_pairs(keys, alt, nullptr, nullptr, n, 32 + bits_for((uint64_t)nparts), st, &kout, &vdummy));
    uint64_t* uniq = (kout == keys) ? alt : keys;
    uint64_t* d_num = nullptr;
    GXB_CHECK(dalloc_t(&d_num, 1));
    size_t temp = 0;
    GXB_CUDA(cub::DeviceSelect::Unique(nullptr, temp, kout, uniq, d_num, (int64_t)n, st));
    void* tmp = nullptr;
    GXB_CHECK(dalloc(&tmp, temp));
    cudaError_t e = cub::DeviceSelect::Unique(tmp, temp, kout, uniq, d_num, (int64_t)n, st);
    uint64_t nu = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&nu, d_num, 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    dfree(tmp);
    dfree(d_num);
    if (e != cudaSuccess) return cuda_fail(e, "unique_segments");
    uint64_t* d_off = nullptr;
    GXB_CHECK(dalloc_t(&d_off, nparts + 1));
    k_offsets<<<grid_e(nu + 1), kBlock, 0, st>>>(uniq, nu, (uint64_t)nparts, d_off);
    off_host.assign(nparts + 1, 0);
    e = cudaMemcpyAsync(off_host.data(), d_off, 8 * (nparts + 1), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    dfree(d_off);
    if (e != cudaSuccess) return cuda_fail(e, "unique_segments offsets");
    const uint64_t nv = off_host[nparts];  // entries before the sentinel
    GXB_CHECK(dalloc_t(d_idx, nv + 1));
    if (nv) k_low32<<<grid_e(nv), kBlock, 0, st>>>(uniq, nv, *d_idx);
    GXB_CUDA(cudaStreamSynchronize(st));
    return GXB_OK;
}

static int build_sparse_exchange(gxb_graph* g, const uint32_t* src, const uint32_t* dst, uint64_t E,
                                 uint64_t* keyA, uint64_t* keyB, const uint64_t* d_bounds, cudaStream_t st) {
    k_send_keys<<<grid_e(E), kBlock, 0, st>>>(src, dst, E, d_bounds, g->nparts, g->part, keyA);
    GXB_CHECK(unique_segments(keyA, keyB, E, g->nparts, st, &g->d_xsend_idx, g->xsend_off));
    if (g->owned_edges)
        k_recv_keys<<<grid_e(g->owned_edges), kBlock, 0, st>>>(g->d_in_src, g->owned_edges, d_bounds, g->nparts,
                                                                g->part, keyA);
    GXB_CHECK(unique_segments(keyA, keyB, g->owned_edges, g->nparts, st, &g->d_xrecv_idx, g->xrecv_off));
    return GXB_OK;
}

static int graph_build_impl(gxb_graph* g, const uint32_t* src_in, const uint32_t* dst_in,
                            const uint32_t* w_in, uint64_t E, uint32_t flags, cudaStream_t st) {
    Scratch S;
    const bool host = flags & GXB_BUILD_HOST_INPUT;
    const bool want_csr = !(flags & GXB_BUILD_NO_CSR);
    g->E = E;
    g->weighted = (w_in != nullptr);
    // working copies (relabelled in place)
    uint32_t *src = nullptr, *dst = nullptr, *w = nullptr;
    GXB_CHECK(S.get(&src, E));
    GXB_CHECK(S.get(&dst, E));
    const cudaMemcpyKind kind = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    GXB_CUDA(cudaMemcpyAsync(src, src_in, 4 * E, kind, st));
    GXB_CUDA(cudaMemcpyAsync(dst, dst_in, 4 * E, kind, st));
    if (w_in) {
        GXB_CHECK(S.get(&w, E));
        GXB_CUDA(cudaMemcpyAsync(w, w_in, 4 * E, kind, st));
    }
    // largest weight (the SSSP state checks max_w * |V| < 2^32 - 1 for exact u32 sums)
    if (w && E) {
        uint32_t* d_wmax = nullptr;
        GXB_CHECK(S.get(&d_wmax, 1));
        GXB_CUDA(cudaMemsetAsync(d_wmax, 0, 4, st));
        k_max_id<<<grid_e(E), kBlock, 0, st>>>(w, w, E, d_wmax);
        GXB_CUDA(cudaMemcpyAsync(&g->max_w, d_wmax, 4, cudaMemcpyDeviceToHost, st));
    } else {
        g->max_w = E ? 1u : 0u;
    }
    // present ids
    uint32_t* d_max = nullptr;
    GXB_CHECK(S.get(&d_max, 1));
    GXB_CUDA(cudaMemsetAsync(d_max, 0, 4, st));
    if (E) k_max_id<<<grid_e(E), kBlock, 0, st>>>(src, dst, E, d_max);
    uint32_t max_id = 0;
    GXB_CUDA(cudaMemcpyAsync(&max_id, d_max, 4, cudaMemcpyDeviceToHost, st));
    GXB_CUDA(cudaStreamSynchronize(st));
    if (max_id == 0xFFFFFFFFu) return fail(GXB_ERANGE, "vertex id 4294967295 is reserved");
    g->max_id = max_id;
    const uint64_t words = E ? ((uint64_t)max_id >> 5) + 1 : 1;
    uint32_t *bm = nullptr, *wcnt = nullptr, *wpre = nullptr;
    GXB_CHECK(S.get(&bm, words));
    GXB_CHECK(S.get(&wcnt, words + 1));
    GXB_CHECK(S.get(&wpre, words + 1));
    GXB_CUDA(cudaMemsetAsync(bm, 0, 4 * words, st));
    GXB_CUDA(cudaMemsetAsync(wcnt, 0, 4 * (words + 1), st));
    if (E) k_mark_present<<<grid_e(E), kBlock, 0, st>>>(src, dst, E, bm);
    k_word_popc<<<grid_e(words), kBlock, 0, st>>>(bm, words, wcnt);
    GXB_CHECK(exclusive_scan<uint32_t>(wcnt, wpre, words + 1, st));
    uint32_t V32 = 0;
    GXB_CUDA(cudaMemcpyAsync(&V32, wpre + words, 4, cudaMemcpyDeviceToHost, st));
    GXB_CUDA(cudaStreamSynchronize(st));
    const uint64_t V = E ? V32 : 0;
    g->V = V;
    uint32_t *ids_dense = nullptr, *outdeg_d = nullptr, *indeg_d = nullptr;
    GXB_CHECK(S.get(&ids_dense, V));
    GXB_CHECK(S.get(&outdeg_d, V));
    GXB_CHECK(S.get(&indeg_d, V));
    GXB_CUDA(cudaMemsetAsync(outdeg_d, 0, 4 * V + 4, st));
    GXB_CUDA(cudaMemsetAsync(indeg_d, 0, 4 * V + 4, st));
    if (E) {
        k_emit_ids<<<grid_e(words), kBlock, 0, st>>>(bm, wpre, words, ids_dense);
        k_rank_edges<<<grid_e(E), kBlock, 0, st>>>(src, dst, E, bm, wpre, outdeg_d, indeg_d);
    }
    // slot order: in-degree descending, ties by ascending id (stable sort). With
    // GXB_BUILD_ID_RANGES the partitions are the reference's contiguous ascending-id
    // ranges (partition_graph + even_sizes, A/graph.py:169-212) and the degree sort
    // runs inside each range: key = (partition << 32) | ~in-degree.
    const bool id_ranges = (flags & GXB_BUILD_ID_RANGES) != 0;
    std::vector<uint64_t> id_bounds;
    if (id_ranges) {
        id_bounds.assign(g->nparts + 1, 0);
        if (!g->part_sizes.empty()) {
            uint64_t acc = 0;
            for (int p = 0; p < g->nparts; ++p) acc += g->part_sizes[p];
            if (acc != V) return fail(GXB_EINVAL, "partition sizes sum to " + std::to_string(acc) +
                                                      ", expected " + std::to_string(V) + " vertices");
            for (int p = 0; p < g->nparts; ++p) id_bounds[p + 1] = id_bounds[p] + g->part_sizes[p];
        } else {
            for (int p = 0; p < g->nparts; ++p) {  // even_sizes(V, m)
                const uint64_t base = V / g->nparts, rem = V % g->nparts;
                id_bounds[p + 1] = id_bounds[p] + base + ((uint64_t)p < rem ? 1 : 0);
            }
        }
    }
    uint32_t *iota = nullptr, *slot2dense = nullptr, *indeg_slot = nullptr;
    GXB_CHECK(S.get(&iota, V));
    GXB_CHECK(S.get(&slot2dense, V));
    GXB_CHECK(S.get(&indeg_slot, V));
    if (V && !id_ranges) {
        k_iota<<<grid_e(V), kBlock, 0, st>>>(iota, V);
        size_t temp = 0;
        GXB_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, temp, indeg_d, indeg_slot, iota,
                                                           slot2dense, (int64_t)V, 0, 32, st));
        void* tmp = nullptr;
        GXB_CHECK(S.get(reinterpret_cast<uint8_t**>(&tmp), temp));
        GXB_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, temp, indeg_d, indeg_slot, iota,
                                                           slot2dense, (int64_t)V, 0, 32, st));
    } else if (V) {
        uint64_t *pkey = nullptr, *pkey_out = nullptr, *d_idb = nullptr;
        GXB_CHECK(S.get(&pkey, V));
        GXB_CHECK(S.get(&pkey_out, V));
        GXB_CHECK(S.get(&d_idb, g->nparts + 1));
        GXB_CUDA(cudaMemcpyAsync(d_idb, id_bounds.data(), 8 * (g->nparts + 1), cudaMemcpyHostToDevice, st));
        k_iota<<<grid_e(V), kBlock, 0, st>>>(iota, V);
        k_part_keys<<<grid_e(V), kBlock, 0, st>>>(indeg_d, V, d_idb, g->nparts, pkey);
        size_t temp = 0;
        GXB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp, pkey, pkey_out, iota, slot2dense, (int64_t)V, 0,
                                                 32 + bits_for((uint64_t)g->nparts), st));
        void* tmp = nullptr;
        GXB_CHECK(S.get(reinterpret_cast<uint8_t**>(&tmp), temp));
        GXB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, temp, pkey, pkey_out, iota, slot2dense, (int64_t)V, 0,
                                                 32 + bits_for((uint64_t)g->nparts), st));
        k_gather_indeg<<<grid_e(V), kBlock, 0, st>>>(slot2dense, indeg_d, V, indeg_slot);
    }
    // GXB_BUILD_RANGES keeps contiguous degree-sorted ranges balanced by cost; the default
    // for nparts > 1 deals the degree-sorted order round-robin (position i -> partition
    // i mod nparts), so every partition gets 1/nparts of the hubs AND of the low-degree
    // tail: balanced edges, balanced vertices and a balanced dense exchange
    const bool dealt = !id_ranges && g->nparts > 1 && !(flags & GXB_BUILD_RANGES);
    std::vector<uint64_t> deal_bounds;
    uint64_t SL = V;  // slot count; dealt blocks are padded to equal size B = ceil(V / nparts)
    if (dealt && V) {
        const uint64_t B = (V + g->nparts - 1) / g->nparts;
        SL = B * g->nparts;
        deal_bounds.assign(g->nparts + 1, 0);
        for (int p = 0; p <= g->nparts; ++p) deal_bounds[p] = B * p;
        uint32_t *s2d = nullptr, *ind = nullptr;
        GXB_CHECK(S.get(&s2d, SL));
        GXB_CHECK(S.get(&ind, SL));
        // padding slots (one at the end of some blocks): no id, no edges
        GXB_CUDA(cudaMemsetAsync(s2d, 0xFF, 4 * SL, st));
        GXB_CUDA(cudaMemsetAsync(ind, 0, 4 * SL, st));
        k_deal<<<grid_e(V), kBlock, 0, st>>>(slot2dense, indeg_slot, V, g->nparts, B, s2d, ind);
        slot2dense = s2d;
        indeg_slot = ind;
    }
    g->S = SL;
    GXB_CHECK(dalloc_t(&g->d_dense2slot, V));
    GXB_CHECK(dalloc_t(&g->d_slot2id, SL));
    GXB_CHECK(dalloc_t(&g->d_outdeg, SL));
    if (SL)
        k_slot_tables<<<grid_e(SL), kBlock, 0, st>>>(slot2dense, SL, ids_dense, outdeg_d, g->d_dense2slot,
                                                      g->d_slot2id, g->d_outdeg);
    if (E) k_relabel<<<grid_e(E), kBlock, 0, st>>>(src, dst, E, g->d_dense2slot);

    // destination-range partition balanced by in-edge count
    std::vector<uint32_t> h_indeg(SL);
    if (SL) GXB_CUDA(cudaMemcpyAsync(h_indeg.data(), indeg_slot, 4 * SL, cudaMemcpyDeviceToHost, st));
    GXB_CUDA(cudaStreamSynchronize(st));
    uint32_t maxin = 0;
    for (uint64_t i = 0; i < SL; ++i) maxin = std::max(maxin, h_indeg[i]);
    g->max_in_degree = maxin;
    g->bounds.assign(g->nparts + 1, 0);
    g->bounds[g->nparts] = SL;
    if (id_ranges) {
        g->bounds = id_bounds;
    } else if (dealt) {
        g->bounds = deal_bounds;
    } else {
        // per-slot cost: 12 B per in-edge (index + gathered value) and 64 B-equivalent per
        // vertex (apply, stats, span folding measured at ~5 edges' worth on B200);
        // every rank computes the same bounds from the same edge list
        auto cost = [&](uint64_t s) { return 12ull * h_indeg[s] + 64ull; };
        uint64_t total = 0;
        for (uint64_t s = 0; s < V; ++s) total += cost(s);
        // heterogeneous devices: partition p's share of the cost is its capacity factor
        // over the sum (balance_data, A/balancer.py:79-98, applied to the continuous cost
        // line instead of integer units); no factors = equal shares
        std::vector<long double> cum(g->nparts + 1, 0.0L);
        for (int p = 0; p < g->nparts; ++p)
            cum[p + 1] = cum[p] + (g->part_capacity.empty() ? 1.0L : (long double)g->part_capacity[p]);
        uint64_t acc = 0, s = 0;
        for (int p = 1; p < g->nparts; ++p) {
            const uint64_t target = (uint64_t)((long double)total * cum[p] / cum[g->nparts]);
            while (s < V && acc < target) acc += cost(s++);
            g->bounds[p] = s;
        }
    }
    g->lo = g->bounds[g->part];
    g->hi = g->bounds[g->part + 1];
    const uint64_t owned = g->hi - g->lo;
    g->h_indeg_sorted.assign(h_indeg.begin() + g->lo, h_indeg.begin() + g->hi);

    uint64_t* d_bounds = nullptr;
    GXB_CHECK(S.get(&d_bounds, g->nparts + 1));
    GXB_CUDA(cudaMemcpyAsync(d_bounds, g->bounds.data(), 8 * (g->nparts + 1), cudaMemcpyHostToDevice, st));
    const uint64_t rwords = (SL >> 5) + 1;
    GXB_CHECK(dalloc_t(&g->d_remote_src, rwords));
    GXB_CUDA(cudaMemsetAsync(g->d_remote_src, 0, 4 * rwords, st));

    uint64_t *csc_key = nullptr, *key_alt = nullptr, *csr_key = nullptr;
    GXB_CHECK(S.get(&csc_key, E));
    GXB_CHECK(S.get(&key_alt, E));
    if (want_csr) GXB_CHECK(S.get(&csr_key, E));
    if (E)
        k_keys<<<grid_e(E), kBlock, 0, st>>>(src, dst, E, d_bounds, g->nparts, g->part, g->lo, owned, SL,
                                              g->d_remote_src, csc_key, csr_key);
    // owned in-edge count
    uint64_t owned_edges = 0;
    for (uint64_t s = g->lo; s < g->hi; ++s) owned_edges += h_indeg[s];
    g->owned_edges = owned_edges;

    uint32_t* w_alt = nullptr;
    if (w) GXB_CHECK(S.get(&w_alt, E));
    // CSC
    {
        uint64_t* kout = nullptr;
        uint32_t* vout = nullptr;
        // keep a pristine copy of w for the CSR sort
        uint32_t* w_csc = nullptr;
        if (w && want_csr) {
            GXB_CHECK(S.get(&w_csc, E));
            GXB_CUDA(cudaMemcpyAsync(w_csc, w, 4 * E, cudaMemcpyDeviceToDevice, st));
        } else {
            w_csc = w;
        }
        if (E) GXB_CHECK(sort_pairs(csc_key, key_alt, w_csc, w_alt, E, 32 + bits_for(owned), st, &kout, &vout));
        // offsets padded with kOffPad copies of owned_edges, edge arrays padded to whole
        // warp tiles with zeros, so the tile kernel's vector loads never leave the buffers
        const uint64_t padded = round_up(owned_edges, kTileEdges) + kTileEdges;
        GXB_CHECK(dalloc_t(&g->d_in_off, owned + 1 + kOffPad));
        GXB_CHECK(dalloc_t(&g->d_in_src, padded));
        GXB_CUDA(cudaMemsetAsync(g->d_in_src, 0, 4 * padded, st));
        if (owned_edges) k_low32<<<grid_e(owned_edges), kBlock, 0, st>>>(kout, owned_edges, g->d_in_src);
        k_offsets<<<grid_e(owned_edges + 1), kBlock, 0, st>>>(kout, owned_edges, owned, g->d_in_off);
        k_fill_u64<<<1, 32, 0, st>>>(g->d_in_off + owned + 1, kOffPad, owned_edges);
        if (w) {
            GXB_CHECK(dalloc_t(&g->d_in_w, padded));
            GXB_CUDA(cudaMemsetAsync(g->d_in_w, 0, 4 * padded, st));
            if (owned_edges)
                GXB_CUDA(cudaMemcpyAsync(g->d_in_w, vout, 4 * owned_edges, cudaMemcpyDeviceToDevice, st));
        }
        GXB_CUDA(cudaStreamSynchronize(st));  // also publishes g->max_w to the host
        if (w) {
            const int wb = std::max(1, bits_for(g->max_w));
            if (wb < 32 && bits_for(g->S ? g->S - 1 : 0) + wb <= 32) {
                g->sw_shift = (uint32_t)wb;
                GXB_CHECK(dalloc_t(&g->d_in_sw, padded));
                k_pack_sw<<<grid_e(padded), kBlock, 0, st>>>(g->d_in_src, g->d_in_w, padded, g->sw_shift, g->d_in_sw);
                GXB_CUDA(cudaStreamSynchronize(st));
            }
        }
    }
    // push CSR (sources -> owned destinations)
    if (want_csr) {
        uint64_t* kout = nullptr;
        uint32_t* vout = nullptr;
        if (E) GXB_CHECK(sort_pairs(csr_key, key_alt, w, w_alt, E, 32 + bits_for(SL), st, &kout, &vout));
        GXB_CHECK(dalloc_t(&g->d_out_off, SL + 1));
        GXB_CHECK(dalloc_t(&g->d_out_dst, owned_edges));
        if (owned_edges) k_low32<<<grid_e(owned_edges), kBlock, 0, st>>>(kout, owned_edges, g->d_out_dst);
        k_offsets<<<grid_e(owned_edges + 1), kBlock, 0, st>>>(kout, owned_edges, SL, g->d_out_off);
        if (w) {
            GXB_CHECK(dalloc_t(&g->d_out_w, owned_edges));
            if (owned_edges)
                GXB_CUDA(cudaMemcpyAsync(g->d_out_w, vout, 4 * owned_edges, cudaMemcpyDeviceToDevice, st));
        }
        g->has_csr = true;
        g->owned_out_edges = owned_edges;
        GXB_CUDA(cudaStreamSynchronize(st));
    }
    if (g->nparts > 1 && E) GXB_CHECK(build_sparse_exchange(g, src, dst, E, csc_key, key_alt, d_bounds, st));
    GXB_CUDA(cudaGetLastError());
    GXB_CHECK(build_pull_plan(g, st));
    GXB_CHECK(build_tile_plan(g, st));
    return GXB_OK;
}

}  // namespace gxb

using namespace gxb;

// ------------------------------------------------------------------ C ABI

namespace gxb {
struct InRange {
    uint32_t lo, hi;
    __host__ __device__ bool operator()(uint32_t s) const { return s >= lo && s < hi; }
};
int build_owned_order(gxb_graph* g) {
    if (g->d_owned_d2s || !g->V) return GXB_OK;
    cudaStream_t st = 0;
    uint64_t* d_num = nullptr;
    GXB_CHECK(dalloc_t(&g->d_owned_d2s, g->V));
    GXB_CHECK(dalloc_t(&d_num, 1));
    const InRange f{(uint32_t)g->lo, (uint32_t)g->hi};
    size_t tb = 0;
    GXB_CUDA(cub::DeviceSelect::If(nullptr, tb, g->d_dense2slot, g->d_owned_d2s, d_num, (int64_t)g->V, f, st));
    void* tmp = nullptr;
    GXB_CHECK(dalloc(&tmp, tb));
    GXB_CUDA(cub::DeviceSelect::If(tmp, tb, g->d_dense2slot, g->d_owned_d2s, d_num, (int64_t)g->V, f, st));
    GXB_CUDA(cudaMemcpy(&g->owned_present, d_num, 8, cudaMemcpyDeviceToHost));
    dfree(tmp);
    dfree(d_num);
    return GXB_OK;
}
}  // namespace gxb

extern "C" {

const char* gxb_last_error(void) { return gxb::g_last_error.c_str(); }
const char* gxb_version(void) { return "gxb200 0.1 sm_100a"; }

int gxb_init(int device, gxb_ctx** out) {
    if (!out) return fail(GXB_EINVAL, "gxb_init: null out");
    int n = 0;
    GXB_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) return fail(GXB_EINVAL, "gxb_init: device index out of range");
    GXB_CUDA(cudaSetDevice(device));
    gxb_ctx* c = new gxb_ctx();
    c->device = device;
    cudaError_t e = cudaGetDeviceProperties(&c->prop, device);
    if (e != cudaSuccess) {
        delete c;
        return cuda_fail(e, "cudaGetDeviceProperties");
    }
    if (c->prop.major != 10) {
        int maj = c->prop.major, min = c->prop.minor;
        delete c;
        return fail(GXB_ECUDA, "libgxb200 requires an sm_100 device, found sm_" + std::to_string(maj) +
                                   std::to_string(min));
    }
    c->init_count = 1;  // Daemon.initialize runs exactly once (A/daemon.py:148-161)
    c->alive = true;
    *out = c;
    return GXB_OK;
}

int gxb_set_option(const char* name, int64_t value) {
    if (!name) return fail(GXB_EINVAL, "gxb_set_option: null name");
    Options& o = options();
    const std::string n(name);
    if (n == "tile_minblocks") {
        if (value != 0 && value != 1 && value != 4 && value != 6 && value != 8)
            return fail(GXB_EINVAL, "tile_minblocks: 0 (auto) / 1 / 4 / 6 / 8");
        o.tile_minblocks = value;
    } else if (n == "l2_hot_mb") {
        if (value < 0) return fail(GXB_EINVAL, "l2_hot_mb must be >= 0");
        o.l2_hot_mb = value;
    } else if (n == "push_alpha") {
        if (value < 0) return fail(GXB_EINVAL, "push_alpha must be >= 0");
        o.push_alpha = value;
    } else if (n == "pull_dense_div") {
        if (value < 0) return fail(GXB_EINVAL, "pull_dense_div must be >= 0 (0 = always test active bits)");
        o.pull_dense_div = value;
    } else if (n == "pipeline_apply") {
        if (value != 0 && value != 1) return fail(GXB_EINVAL, "pipeline_apply: 0 or 1");
        o.pipeline_apply = value;
    } else if (n == "xchunk_power") {
        if (value < 1 || value > 4) return fail(GXB_EINVAL, "xchunk_power: 1..4");
        o.xchunk_power = value;
    } else if (n == "tile_async") {
        if (value != 0 && value != 1) return fail(GXB_EINVAL, "tile_async: 0 or 1");
        o.tile_async = value;
    } else if (n == "tile_async_minblocks") {
        if (value != 0 && value != 1 && value != 4 && value != 5 && value != 6 && value != 8)
            return fail(GXB_EINVAL, "tile_async_minblocks: 0 (auto) / 1 / 4 / 5 / 6 / 8");
        o.tile_async_minblocks = value;
    } else if (n == "l1_hot_kb") {
        if (value < 0) return fail(GXB_EINVAL, "l1_hot_kb must be >= 0");
        o.l1_hot_kb = value;
    } else if (n == "exchange_chunks") {
        if (value < 1 || value > 64) return fail(GXB_EINVAL, "exchange_chunks: 1..64");
        o.exchange_chunks = value;
    } else if (n == "overlap_reserve_sms") {
        if (value < 0 || value > 140) return fail(GXB_EINVAL, "overlap_reserve_sms: 0..140");
        o.overlap_reserve_sms = value;
    } else if (n == "split_overlap") {
        if (value != 0 && value != 1) return fail(GXB_EINVAL, "split_overlap: 0 or 1");
        o.split_overlap = value;
    } else if (n == "split_reserve_sms") {
        if (value < 0 || value > 140) return fail(GXB_EINVAL, "split_reserve_sms: 0..140");
        o.split_reserve_sms = value;
    } else if (n == "carveout") {
        if (value < -1 || value > 100) return fail(GXB_EINVAL, "carveout: -1 or 0..100");
        o.carveout = value;
    } else if (n == "pr_hub_slots") {
        if (value < 0 || value > 28672) return fail(GXB_EINVAL, "pr_hub_slots: 0..28672");
        o.pr_hub_slots = value;
    } else if (n == "pr_message_bits") {
        if (value != 32 && value != 64) return fail(GXB_EINVAL, "pr_message_bits: 32 or 64");
        o.pr_message_bits = value;
    } else if (n == "pull_kernel") {
        if (value != 0 && value != 1) return fail(GXB_EINVAL, "pull_kernel: 0 = tiles, 1 = binned");
        o.pull_kernel = value;
    } else {
        return fail(GXB_EINVAL, "unknown option " + n);
    }
    return GXB_OK;
}

int gxb_get_option(const char* name, int64_t* value) {
    if (!name || !value) return fail(GXB_EINVAL, "gxb_get_option: null argument");
    Options& o = options();
    const std::string n(name);
    if (n == "tile_minblocks") *value = o.tile_minblocks;
    else if (n == "l2_hot_mb") *value = o.l2_hot_mb;
    else if (n == "push_alpha") *value = o.push_alpha;
    else if (n == "pull_kernel") *value = o.pull_kernel;
    else if (n == "pull_dense_div") *value = o.pull_dense_div;
    else if (n == "tile_async") *value = o.tile_async;
    else if (n == "xchunk_power") *value = o.xchunk_power;
    else if (n == "pipeline_apply") *value = o.pipeline_apply;
    else if (n == "tile_async_minblocks") *value = o.tile_async_minblocks;
    else if (n == "pr_message_bits") *value = o.pr_message_bits;
    else if (n == "pr_hub_slots") *value = o.pr_hub_slots;
    else if (n == "carveout") *value = o.carveout;
    else if (n == "overlap_reserve_sms") *value = o.overlap_reserve_sms;
    else if (n == "split_overlap") *value = o.split_overlap;
    else if (n == "split_reserve_sms") *value = o.split_reserve_sms;
    else if (n == "exchange_chunks") *value = o.exchange_chunks;
    else if (n == "l1_hot_kb") *value = o.l1_hot_kb;
    else return fail(GXB_EINVAL, "unknown option " + n);
    return GXB_OK;
}

int gxb_reinit(gxb_ctx* ctx) {
    if (!ctx) return fail(GXB_EINVAL, "gxb_reinit: null ctx");
    return fail(GXB_EPROTO, std::string("daemon: re-initialization attempted in phase ") +
                                (ctx->alive ? "ready" : "terminated"));
}

int gxb_init_count(const gxb_ctx* ctx, int* out) {
    if (!ctx || !out) return fail(GXB_EINVAL, "gxb_init_count: null argument");
    *out = ctx->init_count;
    return GXB_OK;
}

int gxb_shutdown(gxb_ctx* ctx) {
    if (!ctx) return GXB_OK;
    if (ctx->alive) {
        ctx->alive = false;
        cudaDeviceSynchronize();
    }
    delete ctx;
    return GXB_OK;
}

int gxb_graph_build(gxb_ctx* ctx, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                    uint64_t num_edges, int part, int nparts, uint32_t flags, void* stream,
                    gxb_graph** out) {
    return gxb_graph_build_sized(ctx, src, dst, w, num_edges, part, nparts, nullptr, flags, stream, out);
}

int gxb_graph_build_sized(gxb_ctx* ctx, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                          uint64_t num_edges, int part, int nparts, const uint64_t* sizes, uint32_t flags,
                          void* stream, gxb_graph** out) {
    NvtxRange nvtx_("gxb_graph_build_sized");
    if (!ctx || !ctx->alive) return fail(GXB_ESTATE, "gxb_graph_build: daemon not initialised");
    if (!out) return fail(GXB_EINVAL, "gxb_graph_build: null out");
    if (num_edges && (!src || !dst)) return fail(GXB_EINVAL, "gxb_graph_build: null edge arrays");
    if (nparts < 1 || nparts > 64 || part < 0 || part >= nparts)
        return fail(GXB_EINVAL, "gxb_graph_build: bad partition index");
    if (num_edges >= (1ull << 32)) return fail(GXB_ERANGE, "gxb_graph_build: more than 2^32-1 edges");
    GXB_CUDA(cudaSetDevice(ctx->device));
    gxb_graph* g = new gxb_graph();
    g->ctx = ctx;
    g->part = part;
    g->nparts = nparts;
    if (sizes) {
        g->part_sizes.assign(sizes, sizes + nparts);
        flags |= GXB_BUILD_ID_RANGES;
    }
    int rc = graph_build_impl(g, src, dst, w, num_edges, flags, (cudaStream_t)stream);
    if (rc != GXB_OK) {
        graph_release(g);
        delete g;
        return rc;
    }
    *out = g;
    return GXB_OK;
}

int gxb_graph_build_balanced(gxb_ctx* ctx, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                             uint64_t num_edges, int part, int nparts, const double* capacity, uint32_t flags,
                             void* stream, gxb_graph** out) {
    NvtxRange nvtx_("gxb_graph_build_balanced");
    if (!ctx || !ctx->alive) return fail(GXB_ESTATE, "gxb_graph_build: daemon not initialised");
    if (!out) return fail(GXB_EINVAL, "gxb_graph_build: null out");
    if (!capacity) return fail(GXB_EINVAL, "gxb_graph_build_balanced: null capacity factors");
    if (nparts < 1 || nparts > 64 || part < 0 || part >= nparts)
        return fail(GXB_EINVAL, "gxb_graph_build: bad partition index");
    for (int p = 0; p < nparts; ++p)  // NodeCost's precondition (A/balancer.py:26-28)
        if (!(capacity[p] > 0.0) || !std::isfinite(capacity[p]))
            return fail(GXB_EINVAL, "gxb_graph_build_balanced: capacity factors must be positive and finite");
    if (flags & GXB_BUILD_ID_RANGES)
        return fail(GXB_EINVAL, "gxb_graph_build_balanced: capacity factors apply to degree-sorted ranges only");
    if (num_edges && (!src || !dst)) return fail(GXB_EINVAL, "gxb_graph_build: null edge arrays");
    if (num_edges >= (1ull << 32)) return fail(GXB_ERANGE, "gxb_graph_build: more than 2^32-1 edges");
    GXB_CUDA(cudaSetDevice(ctx->device));
    gxb_graph* g = new gxb_graph();
    g->ctx = ctx;
    g->part = part;
    g->nparts = nparts;
    g->part_capacity.assign(capacity, capacity + nparts);
    int rc = graph_build_impl(g, src, dst, w, num_edges, flags | GXB_BUILD_RANGES, (cudaStream_t)stream);
    if (rc != GXB_OK) {
        graph_release(g);
        delete g;
        return rc;
    }
    *out = g;
    return GXB_OK;
}

int gxb_graph_get_info(const gxb_graph* g, gxb_graph_info* o) {
    if (!g || !o) return fail(GXB_EINVAL, "gxb_graph_get_info: null argument");
    std::memset(o, 0, sizeof(*o));
    o->num_vertices = g->V;
    o->num_slots = g->S;
    o->num_edges = g->E;
    o->owned_lo = g->lo;
    o->owned_hi = g->hi;
    o->owned_edges = g->owned_edges;
    o->owned_out_edges = g->owned_out_edges;
    o->max_id = g->max_id;
    o->max_in_degree = g->max_in_degree;
    o->part = g->part;
    o->nparts = g->nparts;
    o->weighted = g->weighted;
    o->has_csr = g->has_csr;
    return GXB_OK;
}

__global__ void k_gather_by_slot(const uint32_t* __restrict__ d2s, const uint32_t* __restrict__ vals,
                                 uint64_t V, uint32_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < V;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = vals[d2s[i]];
}

static int read_dense_u32(const gxb_graph* g, const uint32_t* per_slot, uint32_t* host_out) {
    if (!g->V) return GXB_OK;
    uint32_t* tmp = nullptr;
    GXB_CHECK(dalloc_t(&tmp, g->V));
    k_gather_by_slot<<<grid_e(g->V), kBlock>>>(g->d_dense2slot, per_slot, g->V, tmp);
    cudaError_t e = cudaMemcpy(host_out, tmp, 4 * g->V, cudaMemcpyDeviceToHost);
    dfree(tmp);
    if (e != cudaSuccess) return cuda_fail(e, "read_dense_u32");
    return GXB_OK;
}

int gxb_graph_ids(const gxb_graph* g, uint32_t* host_out) {
    if (!g || (!host_out && g->V)) return fail(GXB_EINVAL, "gxb_graph_ids: null argument");
    return read_dense_u32(g, g->d_slot2id, host_out);
}

int gxb_graph_out_degree(const gxb_graph* g, uint32_t* host_out) {
    if (!g || (!host_out && g->V)) return fail(GXB_EINVAL, "gxb_graph_out_degree: null argument");
    return read_dense_u32(g, g->d_outdeg, host_out);
}


__global__ void k_gather_ids(const uint32_t* __restrict__ d2s, uint64_t n, const uint32_t* __restrict__ slot2id,
                             uint32_t* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = slot2id[d2s[i]];
}

int gxb_graph_owned_ids(gxb_graph* g, uint32_t* host_out, uint64_t* count) {
    if (!g || !count) return fail(GXB_EINVAL, "gxb_graph_owned_ids: null argument");
    GXB_CUDA(cudaSetDevice(g->ctx->device));
    GXB_CHECK(build_owned_order(g));
    *count = g->owned_present;
    if (!host_out || !g->owned_present) return GXB_OK;
    uint32_t* d = nullptr;
    GXB_CHECK(dalloc_t(&d, g->owned_present));
    k_gather_ids<<<grid_for(g->owned_present), kBlock>>>(g->d_owned_d2s, g->owned_present, g->d_slot2id, d);
    const cudaError_t e = cudaMemcpy(host_out, d, 4 * g->owned_present, cudaMemcpyDeviceToHost);
    dfree(d);
    if (e != cudaSuccess) return cuda_fail(e, "gxb_graph_owned_ids");
    return GXB_OK;
}

int gxb_graph_part_bounds(const gxb_graph* g, uint64_t* host_out) {
    if (!g || !host_out) return fail(GXB_EINVAL, "gxb_graph_part_bounds: null argument");
    std::memcpy(host_out, g->bounds.data(), 8 * g->bounds.size());
    return GXB_OK;
}

int gxb_graph_xchunks(const gxb_graph* g, int* K, uint64_t* host_bounds) {
    if (!g || !K) return fail(GXB_EINVAL, "gxb_graph_xchunks: null argument");
    *K = g->tiles.num_xchunks;
    if (host_bounds)
        for (int k = 0; k <= *K; ++k) host_bounds[k] = g->tiles.xchunk_slot[k];
    return GXB_OK;
}

int gxb_graph_free(gxb_graph* g) {
    if (!g) return GXB_OK;
    graph_release(g);
    delete g;
    return GXB_OK;
}

}  // extern "C"
