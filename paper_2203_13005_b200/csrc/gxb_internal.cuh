// gxb_internal.cuh — shared internals of libgxb200.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/gxb.h"
#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges cost nothing without a tool attached

#if !defined(__CUDA_ARCH__) || __CUDA_ARCH__ >= 1000
#else
#error "libgxb200 is built for sm_100a only"
#endif

namespace gxb {

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define GXB_CUDA(call)                                                      \
    do {                                                                    \
        cudaError_t _e = (call);                                            \
        if (_e != cudaSuccess) return ::gxb::cuda_fail(_e, #call);          \
    } while (0)

#define GXB_CHECK(call)                                                     \
    do {                                                                    \
        int _rc = (call);                                                   \
        if (_rc != GXB_OK) return _rc;                                      \
    } while (0)

// NVTX range over a host API call (visible in nsys / ncu --nvtx timelines)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr uint32_t kInf32 = 0xFFFFFFFFu;  // SSSP "inf" lane / invalid label
constexpr int kBlock = 256;               // threads per CTA for the vertex/edge kernels
constexpr int kNumSMs = 148;

// Degree bins of the pull merge (SURVEY.md §7 "workload balancing inside a GPU").
// Slots are sorted by in-degree (descending), so every bin is a contiguous slot
// range. Bin k < kNumGroupBins uses groups of (1 << k) lanes per destination;
// destinations above kChunkMinDeg are split into chunks of kChunkEdges edges,
// one warp per chunk, combined by the last-arriving warp.
constexpr int kNumGroupBins = 6;            // G = 1, 2, 4, 8, 16, 32
constexpr uint32_t kChunkMinDeg = 128;      // > this: chunked warps
constexpr uint32_t kChunkEdges = 1024;      // edges per warp work item

// Edge-balanced pull merge (the "warp tile" kernel): each warp owns kTileEdges
// consecutive CSC edges, kTileK per lane, whatever the destination degrees.
constexpr int kTileK = 8;
constexpr uint64_t kTileEdges = 32 * kTileK;
constexpr uint64_t kOffPad = 16;           // extra offset entries (= owned_edges) after the CSC offsets
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kMaxPeers = 7;  // peer replicas a PageRank Apply writes directly (8 GPUs per NVSwitch node)

struct TilePlan {
    uint64_t nz_slots = 0;       // owned slots with in-degree > 0 (a prefix: slots are degree-sorted)
    uint64_t num_tiles = 0;
    uint64_t num_spans = 0;      // slots whose edges cross a tile boundary
    uint64_t num_partials = 0;   // sum of tiles touched by spans
    int num_xchunks = 1;         // exchange chunks of the owned slots (pipeline shuffle)
    std::vector<uint64_t> xchunk_slot;  // K+1 relative slot bounds
    std::vector<uint64_t> xchunk_tile;  // K+1 tile bounds
    std::vector<uint64_t> xchunk_span;  // K+1 span bounds
    uint64_t* d_tile_start = nullptr;  // num_tiles + 1 tile boundaries (edge offsets, slot-aligned)
    uint32_t* d_lane_slot = nullptr;   // per kTileK-edge lane chunk: slot of its first edge
    uint8_t* d_lane_mask = nullptr;    // per lane chunk: bit j <=> edge kTileK*c + j closes its segment
    uint32_t* d_tile_head = nullptr;   // per tile: span id of its first slot if that slot started earlier
    uint32_t* d_tile_tail = nullptr;   // per tile: span id of its last slot if that slot continues
    uint32_t* d_span_first = nullptr;  // per span: first tile
    uint32_t* d_span_count = nullptr;  // per span: tiles touched
    uint64_t* d_span_pbase = nullptr;  // per span: first partial index
    uint32_t* d_span_slot = nullptr;   // per span: relative slot
};

struct DeviceBuffer {
    void* ptr = nullptr;
    size_t bytes = 0;
};

// device allocation helper (cudaMalloc, tracked by the owner)
int dalloc(void** p, size_t bytes);
template <typename T>
int dalloc_t(T** p, size_t n) {
    return dalloc(reinterpret_cast<void**>(p), n * sizeof(T) + 16);
}
void dfree(void* p);

struct PullPlan {
    // slot boundaries (relative to owned_lo) of the bins; bins are in
    // descending-degree order: [chunk | G32 | G16 | G8 | G4 | G2 | G1]
    uint64_t chunk_end;                 // slots [0, chunk_end) are chunked
    uint64_t group_end[kNumGroupBins];  // group bin k covers [prev_end, group_end[...]]
    // chunk work items (one warp each)
    uint64_t num_items;
    uint32_t* d_item_slot = nullptr;    // owning slot (relative) per item
    uint64_t* d_item_begin = nullptr;   // first edge of the item
    uint32_t* d_item_first = nullptr;   // first item index of the same slot
    uint32_t* d_item_count = nullptr;   // number of items of the same slot
    uint32_t* d_slot_arrive = nullptr;  // per chunked slot arrival counters (chunk_end)
};

}  // namespace gxb

struct gxb_ctx {
    int device = 0;
    int init_count = 0;
    bool alive = false;
    cudaDeviceProp prop{};
};

struct gxb_graph {
    gxb_ctx* ctx = nullptr;
    uint64_t V = 0, E = 0;
    uint64_t S = 0;                     // slot count: V, or nparts * ceil(V / nparts) when dealt (padding slots)
    uint32_t max_id = 0;
    uint32_t max_in_degree = 0;
    uint32_t max_w = 0;                 // largest edge weight (1 when unweighted)
    int part = 0, nparts = 1;
    uint64_t lo = 0, hi = 0;            // owned slot range
    uint64_t owned_edges = 0, owned_out_edges = 0;
    bool weighted = false, has_csr = false;
    std::vector<uint64_t> bounds;       // nparts + 1 slot boundaries
    std::vector<uint64_t> part_sizes;   // explicit per-partition vertex counts (id-range mode)
    std::vector<double> part_capacity;  // per-partition capacity factors (degree-sorted ranges)

    uint32_t* d_slot2id = nullptr;      // V: original id per slot
    uint32_t* d_dense2slot = nullptr;   // V: slot of the i-th smallest id
    uint32_t* d_outdeg = nullptr;       // V: global out-degree per slot
    uint32_t* d_remote_src = nullptr;   // bitmap over slots: has an out-edge into another part
    uint64_t* d_in_off = nullptr;       // owned+1 offsets into d_in_src (0-based)
    uint32_t* d_in_src = nullptr;       // source slot per owned in-edge (sorted by (dst, src))
    uint32_t* d_in_w = nullptr;         // weight per owned in-edge (nullptr = unweighted)
    // (src << sw_shift) | w per owned in-edge, when slot and weight bits fit 32 (weighted graphs):
    // the tile kernel's single index+weight stream (4 B/edge instead of 8)
    uint32_t* d_in_sw = nullptr;
    // owned present slots in ascending-id order (lazily built by gxb_attrs_scope / gxb_graph_owned_ids)
    uint32_t* d_owned_d2s = nullptr;
    uint64_t owned_present = 0;
    uint32_t sw_shift = 0;
    uint64_t* d_out_off = nullptr;      // V+1: push CSR restricted to owned destinations
    uint32_t* d_out_dst = nullptr;
    uint32_t* d_out_w = nullptr;
    std::vector<uint32_t> h_indeg_sorted;  // owned in-degrees (descending), host copy
    // needed-only exchange (nparts > 1): sorted slot lists per peer, segment offsets on host
    uint32_t* d_xsend_idx = nullptr;    // my owned slots needed by peer q: [xsend_off[q], xsend_off[q+1])
    uint32_t* d_xrecv_idx = nullptr;    // peer p's slots my CSC reads:      [xrecv_off[p], xrecv_off[p+1])
    std::vector<uint64_t> xsend_off, xrecv_off;
    gxb::PullPlan plan;
    gxb::TilePlan tiles;
};

namespace gxb {

// ---- bitmap helpers ----
__device__ __forceinline__ bool bit_test(const uint32_t* bm, uint32_t i) {
    return (__ldg(bm + (i >> 5)) >> (i & 31)) & 1u;
}
// Push rounds walk the concatenated frontier rows (rowpre = inclusive prefix of the row
// lengths, rowpre[n - 1] > g): move row cursor f to the row of edge g, the first f' >= f
// with rowpre[f'] > g. Usually the next row or two; at N > 1 a frontier holds many rows
// with no local out-edge (changed vertices whose out-edges all leave the partition), so a
// run of empty rows is crossed by galloping plus a binary search instead of one load each.
__device__ __forceinline__ uint64_t row_advance(const uint32_t* __restrict__ rowpre, uint64_t n, uint64_t f,
                                                uint64_t g) {
    if (__ldg(rowpre + f) > g) return f;
    uint64_t lo = f + 1, hi = lo, step = 1;  // every row before lo ends at or before g
    while (__ldg(rowpre + hi) <= g) {
        lo = hi + 1;
        hi = min(hi + step, n - 1);
        step <<= 1;
    }
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (__ldg(rowpre + mid) > g) hi = mid; else lo = mid + 1;
    }
    return lo;
}

__device__ __forceinline__ bool bit_set_atomic(uint32_t* bm, uint32_t i) {
    const uint32_t m = 1u << (i & 31);
    return (atomicOr(bm + (i >> 5), m) & m) == 0u;  // true if newly set
}

// ---- L2 eviction-priority hints (PTX createpolicy / ld ... L2::cache_hint) ----
// The CSC index stream is touched once per round: evict it first so the hot,
// degree-sorted prefix of the gathered value arrays stays resident in L2.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 ld_stream_v4(const void* ptr, uint64_t pol) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t ld_stream_u32(const void* ptr, uint64_t pol) {
    uint32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ uint8_t ld_stream_u8(const uint8_t* ptr, uint64_t pol) {
    uint16_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;" : "=h"(r) : "l"(ptr), "l"(pol));
    return (uint8_t)r;
}
__device__ __forceinline__ double ld_keep_f64(const double* ptr, uint64_t pol) {
    double r;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t ld_keep_u32(const uint32_t* ptr, uint64_t pol) {
    uint32_t r;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ uint4 ld_keep_v4(const uint4* ptr, uint64_t pol) {
    uint4 r;
    asm("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(ptr), "l"(pol));
    return r;
}

// hottest prefix: keep in L1 as well (evict_last); the rest bypasses L1
__device__ __forceinline__ double ld_l1_f64(const double* ptr, uint64_t pol) {
    double r;
    asm("ld.global.nc.L1::evict_last.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_nol1_f64(const double* ptr, uint64_t pol) {
    double r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ uint4 ld_l1_v4(const uint4* ptr, uint64_t pol) {
    uint4 r;
    asm("ld.global.nc.L1::evict_last.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ uint4 ld_nol1_v4(const uint4* ptr, uint64_t pol) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t ld_l1_u32(const uint32_t* ptr, uint64_t pol) {
    uint32_t r;
    asm("ld.global.nc.L1::evict_last.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t ld_nol1_u32(const uint32_t* ptr, uint64_t pol) {
    uint32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(ptr), "l"(pol));
    return r;
}

__device__ __forceinline__ float ld_l1_f32(const float* ptr, uint64_t pol) {
    float r;
    asm("ld.global.nc.L1::evict_last.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ float ld_nol1_f32(const float* ptr, uint64_t pol) {
    float r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(ptr), "l"(pol));
    return r;
}

// asynchronous gathers straight into shared memory (LDGSTS): no registers held while the
// load is in flight. .ca allocates in L1 (4/8/16 B), .cg bypasses it (16 B only).
template <int kBytes>
__device__ __forceinline__ void cp_async_ca(uint32_t saddr, const void* g, uint64_t pol) {
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], %2, %3;" ::"r"(saddr), "l"(g), "n"(kBytes),
                 "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_cg16(uint32_t saddr, const void* g, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// d + w saturating at the inf sentinel, in two instructions: min(d, ~w) + w is d + w when
// d + w <= 0xFFFFFFFF - 0 (never wraps) and exactly 0xFFFFFFFF otherwise (d = inf included)
__device__ __forceinline__ uint32_t sat_add(uint32_t d, uint32_t w) { return min(d, ~w) + w; }

inline unsigned grid_for(uint64_t n, int block = kBlock, uint64_t cap = 148ull * 64) {
    uint64_t g = (n + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

int build_pull_plan(gxb_graph* g, cudaStream_t st);
int build_tile_plan(gxb_graph* g, cudaStream_t st);  // warp-tile plan over g->h_indeg_sorted / d_in_off
void shadow_graph_free(gxb_graph* g);                // release a plan-only graph (device arrays + delete)
int build_owned_order(gxb_graph* g);  // d_owned_d2s / owned_present
uint64_t xchunk_bound(uint64_t owned, int k, int K);  // relative slot bound k of K exchange chunks

// runtime tuning knobs (gxb_set_option); defaults are the measured best on B200
struct Options {
    int64_t tile_minblocks = 0;   // __launch_bounds__ min-blocks variant of the tile kernel (0/4/6/8)
    int64_t l2_hot_mb = 64;       // L2 budget (MB) of the evict-last prefix of gathered values
    int64_t l1_hot_kb = 160;      // L1 budget (KB) of the L1-allocating prefix (others bypass L1)
    int64_t push_alpha = 10;      // push when frontier out-edges * alpha < |E| (10 vs 20: CC S24 -14%, SSSP / LP same)
    int64_t pull_dense_div = 4;   // SSSP/CC pull skips the active bitmap when frontier out-edges * div >= |E|
    int64_t pull_kernel = 0;
    int64_t pipeline_apply = 0;   // PageRank: pipelined chunk rounds even without peer replicas (N = 1)
    int64_t xchunk_power = 4;     // exchange chunk bounds owned * (k / K)^p (4 measured best at N = 2, 4)
    int64_t tile_async = 1;       // 1 = LDGSTS-gather tile kernel (k_tile_a), 0 = register gathers (k_tile_t)
    int64_t tile_async_minblocks = 0;  // its min-blocks variant (0 = auto: 5 / 6 / 4 for 4 / 8 / 16-B values)      // 0 = warp tiles, 1 = degree-binned groups
    int64_t carveout = -1;        // tile kernel shared-memory carveout in % (-1 = driver default)
    int64_t exchange_chunks = 2;  // multi-GPU: exchange chunks (pipelined peer-write rounds; 2 measured best at N = 4)
    int64_t overlap_reserve_sms = 0;  // SMs left free while a chunked round computes (0 measured best)
    int64_t split_overlap = 0;        // SSSP / CC at N > 1: the next round's local-source pass beside the exchange
    int64_t split_reserve_sms = 16;   // SMs left to the exchange kernels during that pass
    int64_t pr_message_bits = 64; // PageRank message (rank / out_deg) precision: 64 or 32 (f64 accumulation)
    int64_t pr_hub_slots = 0;     // PageRank, one partition: in-edges from the first H source slots (the
                                  // highest out-degrees) are summed from a shared-memory table (<= 28672)
};
Options& options();

}  // namespace gxb
