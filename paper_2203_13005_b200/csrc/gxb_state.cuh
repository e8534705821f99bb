// gxb_state.cuh — algorithm state, statistics and the kernel-side views.
#pragma once

#include "gxb_internal.cuh"

namespace gxb {

constexpr int kStripes = 32;
constexpr unsigned kFull = 0xffffffffu;

// striped device counters (one 64-byte stripe per blockIdx % kStripes keeps the
// end-of-kernel atomics off a single L2 address)
struct alignas(64) StatStripe {
    unsigned long long changed;
    unsigned long long next_active;
    unsigned long long next_units;
    unsigned long long targets;
    unsigned long long remote_active;
    unsigned long long max_stat_bits;  // non-negative double bits: u64 order == double order
    unsigned long long pad[2];
};

struct LocalStats {
    unsigned long long changed = 0, next_active = 0, next_units = 0, targets = 0, remote_active = 0;
    double max_stat = 0.0;
};

// what every apply needs to publish a changed vertex (A/agent.py:404-417)
struct FrontierView {
    uint64_t lo;
    const uint32_t* outdeg;        // per slot (global out-degree)
    const uint32_t* remote_src;    // per-slot bitmap: has a consumer on another partition
    uint32_t* active_next;         // per-slot bitmap
    uint32_t* frontier_next;       // list of slots
    unsigned long long* frontier_count;
};

__device__ __forceinline__ void warp_append(uint32_t* list, unsigned long long* count, uint32_t v) {
    const unsigned mask = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    unsigned long long base = 0;
    if (lane == leader) base = atomicAdd(count, (unsigned long long)__popc(mask));
    base = __shfl_sync(mask, base, leader);
    list[base + __popc(mask & ((1u << lane) - 1u))] = v;
}

// a vertex changed and becomes active next iteration
__device__ __forceinline__ void publish_changed(const FrontierView& f, uint32_t slot, LocalStats& st) {
    st.changed++;
    st.next_active++;
    st.next_units += __ldg(f.outdeg + slot);
    if (bit_test(f.remote_src, slot)) st.remote_active++;
    atomicOr(f.active_next + (slot >> 5), 1u << (slot & 31));
    warp_append(f.frontier_next, f.frontier_count, slot);
}

// publish_changed for a full warp over kU groups of 32 CONSECUTIVE slots (all lanes call
// it; `changed[u]` per lane): each group spans at most two bitmap words, so one OR per word
// replaces 32 same-word atomics, one frontier reservation covers all groups, and the
// per-slot loads are issued together — three L2 round trips per call instead of 3·kU.
template <int kU>
__device__ __forceinline__ void publish_changed_warp(const FrontierView& f, const uint32_t (&slot)[kU],
                                                     const bool (&changed)[kU], LocalStats& st) {
    unsigned m[kU];
    unsigned total = 0;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        m[u] = __ballot_sync(kFull, changed[u]);
        total += __popc(m[u]);
    }
    if (!total) return;
    const int lane = threadIdx.x & 31;
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(f.frontier_count, (unsigned long long)total);
    uint32_t od[kU];
    bool rem[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        od[u] = changed[u] ? __ldg(f.outdeg + slot[u]) : 0u;
        rem[u] = changed[u] && bit_test(f.remote_src, slot[u]);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        if (!m[u]) continue;
        const uint32_t word = slot[u] >> 5;
        const uint32_t w0 = __shfl_sync(kFull, word, 0);
        const uint32_t mybit = changed[u] ? (1u << (slot[u] & 31)) : 0u;
        const uint32_t b0 = __reduce_or_sync(kFull, word == w0 ? mybit : 0u);
        const uint32_t b1 = __reduce_or_sync(kFull, word != w0 ? mybit : 0u);
        if (lane == 0 && b0) atomicOr(f.active_next + w0, b0);
        if (lane == 31 && b1) atomicOr(f.active_next + word, b1);
    }
    base = __shfl_sync(kFull, base, 0);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
        if (changed[u]) {
            f.frontier_next[base + __popc(m[u] & ((1u << lane) - 1u))] = slot[u];
            st.changed++;
            st.next_active++;
            st.next_units += od[u];
            if (rem[u]) st.remote_active++;
        }
        base += __popc(m[u]);
    }
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// block-wide reduction of LocalStats into one stripe
__device__ __forceinline__ void flush_stats(LocalStats st, StatStripe* stripes) {
    __shared__ unsigned long long sh[kBlock / 32][6];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long v[5] = {st.changed, st.next_active, st.next_units, st.targets, st.remote_active};
    double m = st.max_stat;
    for (int i = 0; i < 5; ++i) v[i] = warp_sum(v[i]);
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(kFull, m, o));
    if (lane == 0) {
        for (int i = 0; i < 5; ++i) sh[warp][i] = v[i];
        sh[warp][5] = (unsigned long long)__double_as_longlong(m);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t[5] = {0, 0, 0, 0, 0};
        double mm = 0.0;
        for (int w = 0; w < kBlock / 32; ++w) {
            for (int i = 0; i < 5; ++i) t[i] += sh[w][i];
            mm = fmax(mm, __longlong_as_double((long long)sh[w][5]));
        }
        StatStripe* s = stripes + (blockIdx.x % kStripes);
        if (t[0]) atomicAdd(&s->changed, t[0]);
        if (t[1]) atomicAdd(&s->next_active, t[1]);
        if (t[2]) atomicAdd(&s->next_units, t[2]);
        if (t[3]) atomicAdd(&s->targets, t[3]);
        if (t[4]) atomicAdd(&s->remote_active, t[4]);
        if (mm > 0.0) atomicMax(&s->max_stat_bits, (unsigned long long)__double_as_longlong(mm));
    }
}

}  // namespace gxb

struct gxb_state {
    gxb_graph* g = nullptr;
    int algo = 0;
    int arity = 1;
    int nsrc = 0;
    uint32_t src_slot[4] = {0, 0, 0, 0};
    bool src_present[4] = {false, false, false, false};
    uint64_t iteration = 0;
    uint64_t owned_outdeg_sum = 0;   // GEN units of a full frontier of owned vertices
    uint64_t owned_targets = 0;      // owned slots with in-degree > 0 (PR targets)

    // values (full-length replica over slots)
    double* d_rank[2] = {nullptr, nullptr}; // PR: rank per slot, double-buffered like the contributions
    bool async_stats = false;               // PR: rounds leave their statistics on the device only
    double* d_contrib[2] = {nullptr, nullptr};  // PR: rank/outdeg, double-buffered
    int cur = 0;
    bool msg32 = false;                     // PR messages in float32 (gathered / exchanged at 4 B)
    uint4* d_dist_cur = nullptr;            // SSSP: 4 lanes of u32 per slot
    uint4* d_dist_next = nullptr;
    uint32_t* d_lab_cur = nullptr;          // CC / LP labels
    uint32_t* d_lab_next = nullptr;

    // frontier
    uint32_t* d_active[2] = {nullptr, nullptr};    // bitmaps over slots
    uint32_t* d_frontier[2] = {nullptr, nullptr};  // slot lists
    unsigned long long* d_fcount = nullptr;        // [2] counters
    uint32_t* d_touched = nullptr;                 // push dedup bitmap over owned slots
    uint64_t words = 0;                            // bitmap words over V
    uint64_t frontier_len = 0;                     // host copy: length of the current frontier list
    uint64_t units_cur = 0;                        // GEN units of the current frontier

    // stats
    gxb::StatStripe* d_stats = nullptr;
    gxb::StatStripe* h_stats = nullptr;    // pinned
    unsigned long long* h_fcount = nullptr; // pinned
    cudaEvent_t stats_ready = nullptr;
    bool stats_pending = false;
    bool in_round = false;
    bool committed_inline = false;  // the round's apply already wrote the current values
    int last_direction = GXB_DIR_PULL;
    gxb_iter_stats last{};

    // request path (materialised messages, lazily allocated)
    void* d_msg = nullptr;
    uint8_t* d_msg_valid = nullptr;
    void* d_merged = nullptr;

    // pull-merge partials (chunk items of the binned kernel, spans of the tile kernel)
    void* d_partials = nullptr;
    void* d_tile_partials = nullptr;
    void* d_sums = nullptr;  // per owned slot: folded accumulator of the tile kernel

    // PageRank hub split (option pr_hub_slots, one partition): in-edges from source slots
    // < hub_n form the "hub" CSC (summed from a shared-memory table), the rest the "cold"
    // CSC (LDGSTS tile kernel); both are compacted to their non-empty destinations
    uint32_t hub_n = 0;
    gxb_graph* split_g[2] = {nullptr, nullptr};   // 0 = cold, 1 = hub: CSC + tile plan only
    uint32_t* d_split_slot[2] = {nullptr, nullptr};  // compacted destination -> owned slot
    void* d_split_partials[2] = {nullptr, nullptr};
    double* d_split_sum[2] = {nullptr, nullptr};  // per owned slot (zero where no such edge)

    // push scheduling (chunk counts, their inclusive scan, CUB scratch)
    uint32_t* d_push_cpre = nullptr;
    unsigned long long* d_scan_status = nullptr;  // k_push_rowpre: tile ticket + look-back words

    // LP scratch
    void* d_lp_scratch = nullptr;
    size_t lp_scratch_bytes = 0;

    // host<->device attribute staging (ascending-id order)
    double* d_stage = nullptr;
    // peer replicas of d_contrib[0/1] (PageRank): Apply stores each new contribution into
    // every peer's next buffer over NVLink, fusing the mirror exchange into the kernel
    int npeers = 0;
    void* peer_contrib[gxb::kMaxPeers][2] = {};
    bool peer_ipc = false;  // opened with cudaIpcOpenMemHandle (closed on free)
    int round_chunks = 0;   // exchange chunks launched in the open round
    cudaStream_t aux_stream = nullptr;  // pipelined rounds: span folds + Apply beside the tiles
    // split rounds (gxb_iterate_local): the next round's local-source pass on aux_stream
    cudaEvent_t ev_local = nullptr;
    bool local_launched = false;  // ev_local pending: join before the sums are touched
    bool local_valid = false;     // its sums are the next round's pass 1
    bool last_dense = false;      // the last tile pull gathered without the active bitmap
    cudaEvent_t ev_tile = nullptr, ev_join = nullptr;
    // per-peer delta exchange over peer memory (SSSP / CC / LP, nparts <= 8): the pack kernel
    // stores each changed owned value only into the receive arenas of the peers whose CSC
    // reads it (need mask), double-buffered by round parity; the counts ride in the vote
    uint32_t* d_need = nullptr;             // per owned slot: bit q = partition q reads it
    uint32_t* d_arena = nullptr;            // my receive arena (records from every sender)
    uint64_t arena_words = 0;
    uint64_t arena_base[gxb::kMaxPeers + 1][2] = {};  // word offset of (sender p, parity) in my arena
    uint64_t peer_recv_cap[gxb::kMaxPeers + 1] = {};  // records per (sender p, parity) block
    uint32_t* peer_arena[gxb::kMaxPeers + 1] = {};    // receiver q's arena
    uint64_t peer_base[gxb::kMaxPeers + 1][2] = {};   // my block in receiver q's arena
    unsigned long long* d_peer_cnt = nullptr;         // records packed for receiver q this round
    bool delta_peers = false, delta_ipc = false;
    int delta_parity = 0;                   // parity of the last packed round
    bool lab_injective = false;  // LP: labels are still the distinct vertex ids (before round 1)
    int attrs_scope = 0;                          // async staging: 0 = every vertex, 1 = owned vertices
    uint64_t stage_n = 0;                         // vertices per staging buffer (allocated)
    double* d_stage_in[2] = {nullptr, nullptr};   // async path: double-buffered
    double* d_stage_out[2] = {nullptr, nullptr};

    // profiling: events around the main merge kernel, launch counter
    bool timing = false;
    bool timing_pending = false;
    cudaEvent_t kev[3] = {nullptr, nullptr, nullptr};
    // async-stats rounds: per-round timing events kept in a ring, read when async mode ends
    static constexpr int kRing = 512;
    cudaEvent_t* kring = nullptr;  // kRing x 3
    int kring_n = 0;               // rounds recorded since async mode began (pending)
    double kernel_ms = 0.0;
    double rest_ms = 0.0;  // device time after the main kernel until the round closes
    uint64_t kernel_launches = 0;
    uint64_t launches = 0;

    // exchange
    void* d_xsend = nullptr;  // needed-only PR exchange: packed values per peer
    void* d_xrecv = nullptr;
    void* d_send = nullptr;
    void* d_recv = nullptr;
    uint64_t recv_cap = 0;
    // [0] async pack count, [1] async unpack GEN units, [2] GEN units of installed changes,
    // [3] an install raised a distance / label (breaks the monotonicity the dense pull relies on)
    unsigned long long* d_xscratch = nullptr;
    bool packed_async = false;    // the closed round's records are packed; the vote carries their count
    bool unpack_pending = false;  // frontier_len / units_cur still to be refreshed from the device
    bool install_pending = false; // installed changes joined the frontier; refresh its length / units
    bool nonmonotone = false;     // sticky: pull rounds keep the active-bitmap test
};

// host reduction of the closed round's statistics, then refresh of the frontier after
// asynchronous unpacks and installs (gxb_algo.cu)
namespace gxb {
int state_settle(gxb_state* s);
}  // namespace gxb
