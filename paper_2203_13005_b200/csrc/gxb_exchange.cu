// gxb_exchange.cu — mirror-value exchange between destination partitions (K6).
//
// The reference's synchronisation round (A/engine.py:242-266) publishes the
// next frontier's needs (gqq), uploads dirty-and-queried values (gdq,
// A/agent.py:550-582) and installs them (A/agent.py:584-592); lazy uploading
// keeps only changed values on the wire (A/sync.py:171-198) and the skip step
// elides the whole round when no next-active vertex has a cross-partition
// consumer (A/sync.py:201-208, A/agent.py:533-535).
//
// On B200 every rank holds a full-length replica of the source values its CSC
// slice reads. The bytes move over NCCL (torch.distributed on NVLink) between
// the device buffers exposed here:
//   dense (PageRank): the owned slice of the contribution replica is
//     all-gathered in place (every vertex changes every round);
//   delta (SSSP / CC / LP): gxb_exchange_pack emits (slot, value) records of
//     the owned vertices that changed (= the next frontier), the caller
//     all-gathers them, and gxb_exchange_unpack installs peers' records into the
//     replica, marks them active and appends them to the push frontier.
#include <cstring>

#include "gxb_state.cuh"

namespace gxb {

__device__ __forceinline__ int record_words(int algo) { return algo == GXB_ALGO_SSSP ? 5 : 2; }

__global__ void k_pack(int algo, const uint32_t* __restrict__ list, const unsigned long long* count, uint64_t lo,
                       uint64_t hi, const uint4* __restrict__ dist, const uint32_t* __restrict__ lab,
                       uint32_t* out, unsigned long long* packed) {
    const uint64_t n = *count;
    const int W = record_words(algo);
    const int lane = threadIdx.x & 31;
    // warp-uniform trip count: the record slots are reserved once per warp
    for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x + (threadIdx.x & ~31u); i0 < n;
         i0 += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = i0 + lane;
        const uint32_t s = i < n ? list[i] : 0u;
        // own changes only (received slots are appended after them)
        const bool mine = i < n && s >= lo && s < hi;
        const unsigned m = __ballot_sync(0xffffffffu, mine);
        if (!m) continue;
        unsigned long long base = 0;
        if (lane == __ffs(m) - 1) base = atomicAdd(packed, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
        if (!mine) continue;
        const unsigned long long k = base + __popc(m & ((1u << lane) - 1u));
        uint32_t* r = out + k * W;
        r[0] = s;
        if (algo == GXB_ALGO_SSSP) {
            const uint4 d = dist[s];
            r[1] = d.x;
            r[2] = d.y;
            r[3] = d.z;
            r[4] = d.w;
        } else {
            r[1] = lab[s];
        }
    }
}

constexpr int kUnpackPer = 4;

// kDedupe: a record may name a vertex already in the frontier (re-sent after an install, a
// delivered mirror): list it once. The per-peer path receives each changed vertex once per
// round from its single owner and none of them is in the (own-slot) frontier yet: it sets
// the active bit with a fire-and-forget OR and writes only the current value (a mirror's
// next value is never read: pull and push rounds write next only for owned slots).
template <bool kDedupe>
__global__ void __launch_bounds__(kBlock) k_unpack(int algo, const uint32_t* __restrict__ rec, uint64_t n,
                                                   uint64_t lo, uint64_t hi, uint4* dist_cur, uint4* dist_next,
                                                   uint32_t* lab_cur, uint32_t* lab_next, uint32_t* active,
                                                   uint32_t* list, unsigned long long* count,
                                                   const uint32_t* __restrict__ outdeg, unsigned long long* units) {
    // A block takes kUnpackPer x kBlock records per step. The frontier slots of the step are
    // reserved with one atomicAdd per block (warp prefixes in shared memory) — a reservation
    // per warp on the single frontier counter serialises in L2 at millions of records.
    constexpr int kWarps = kBlock / 32;
    __shared__ uint32_t stage_all[kWarps][32 * 5];
    __shared__ uint32_t wcnt[kWarps];
    __shared__ unsigned long long bbase;
    __shared__ unsigned long long bunits[kWarps];
    const int W = record_words(algo);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t* stage = stage_all[warp];
    unsigned long long u = 0;
    for (uint64_t t0 = (uint64_t)blockIdx.x * kUnpackPer * kBlock; t0 < n;
         t0 += (uint64_t)gridDim.x * kUnpackPer * kBlock) {
        uint32_t slot[kUnpackPer];
        unsigned m[kUnpackPer];
        uint32_t c = 0;
#pragma unroll
        for (int j = 0; j < kUnpackPer; ++j) {
            const uint64_t g0 = t0 + ((uint64_t)warp * kUnpackPer + j) * 32;  // this group's first record
            const uint64_t i = g0 + lane;
            // the group's 32 records are contiguous: load them with consecutive lanes on
            // consecutive words, then each lane reads its own from shared memory
            const uint32_t words = g0 < n ? (uint32_t)min((uint64_t)32, n - g0) * (uint32_t)W : 0u;
            for (uint32_t k = lane; k < words; k += 32) stage[k] = rec[g0 * W + k];
            __syncwarp();
            const uint32_t* r = stage + lane * W;
            const uint32_t s = i < n ? r[0] : lo;
            bool take = i < n && (s < lo || s >= hi);  // skip own records echoed back by an all-gather
            if (take) {
                if (algo == GXB_ALGO_SSSP) {
                    const uint4 d = make_uint4(r[1], r[2], r[3], r[4]);
                    dist_cur[s] = d;
                    if (kDedupe) dist_next[s] = d;
                } else {
                    lab_cur[s] = r[1];
                    if (kDedupe) lab_next[s] = r[1];
                }
                if (kDedupe) {
                    take = bit_set_atomic(active, s);  // listed once
                } else {
                    atomicOr(active + (s >> 5), 1u << (s & 31));  // result unused: a reduction
                }
                if (take) u += outdeg[s];
            }
            __syncwarp();  // the stage is reloaded by the next group
            slot[j] = s;
            m[j] = __ballot_sync(0xffffffffu, take);
            c += __popc(m[j]);
        }
        if (lane == 0) wcnt[warp] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t acc = 0;
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t x = wcnt[w];
                wcnt[w] = acc;
                acc += x;
            }
            bbase = acc ? atomicAdd(count, (unsigned long long)acc) : 0ull;
        }
        __syncthreads();
        unsigned long long base = bbase + wcnt[warp];
#pragma unroll
        for (int j = 0; j < kUnpackPer; ++j) {
            if ((m[j] >> lane) & 1u) list[base + __popc(m[j] & ((1u << lane) - 1u))] = slot[j];
            base += __popc(m[j]);
        }
        __syncthreads();  // wcnt / bbase are rewritten by the next step
    }
    for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
    if (lane == 0) bunits[warp] = u;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < kWarps; ++w) t += bunits[w];
        if (t) atomicAdd(units, t);
    }
}

// the sync round's deliver (A/agent.py:584-592) from host values: (dense index, value) pairs
// of mirror vertices -> exchange records (SSSP / CC / LP), or straight into the PageRank
// contribution replica. bad: 1 = value not representable, 2 = target owned or out of range.
__global__ void k_deliver(int algo, int arity, const uint64_t* __restrict__ dense, const double* __restrict__ vals,
                          uint64_t n, uint64_t V, const uint32_t* __restrict__ d2s, uint64_t lo, uint64_t hi,
                          const uint32_t* __restrict__ outdeg, double* rank0, double* rank1, double* contrib0,
                          double* contrib1, bool msg32, uint32_t* rec, uint32_t* bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t d = dense[i];
        if (d >= V) { atomicOr(bad, 2u); continue; }
        const uint32_t s = d2s[d];
        if (s >= lo && s < hi) { atomicOr(bad, 2u); continue; }
        if (algo == GXB_ALGO_PAGERANK) {
            // both buffers: rounds alternate between them and Apply rewrites only owned slots
            const double r = vals[i];
            rank0[s] = rank1[s] = r;
            const uint32_t od = outdeg[s];
            const double c = od ? __ddiv_rn(r, (double)od) : 0.0;
            if (msg32) {
                reinterpret_cast<float*>(contrib0)[s] = reinterpret_cast<float*>(contrib1)[s] = __double2float_rn(c);
            } else {
                contrib0[s] = contrib1[s] = c;
            }
            continue;
        }
        const int W = record_words(algo);
        uint32_t* r = rec + i * W;
        r[0] = s;
        if (algo == GXB_ALGO_SSSP) {
            for (int j = 0; j < 4; ++j) {
                uint32_t x = kInf32;
                if (j < arity) {
                    const double v = vals[i * arity + j];
                    if (!(isinf(v) && v > 0)) {
                        if (!(v >= 0.0 && v < 4294967295.0 && v == floor(v))) atomicOr(bad, 1u);
                        else x = (uint32_t)v;
                    }
                }
                r[1 + j] = x;
            }
        } else {
            const double v = vals[i];
            if (!(v >= 0.0 && v < 4294967295.0 && v == floor(v))) atomicOr(bad, 1u);
            r[1] = v >= 0.0 && v < 4294967295.0 ? (uint32_t)v : 0u;
        }
    }
}

// ---- per-peer delta records over peer memory ----
// need[s - lo] |= 1 << q for every owned slot s in the sorted list of slots peer q reads
__global__ void k_need_mask(const uint32_t* __restrict__ idx, uint64_t n, uint64_t lo, uint32_t bit, uint32_t* need) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        atomicOr(need + (idx[i] - lo), bit);
}

struct PeerArenas {
    uint32_t* arena[kMaxPeers + 1];  // receiver q's arena (nullptr for myself)
    uint64_t base[kMaxPeers + 1];    // word offset of my block (this round's parity) in it
};

// the closed round's changed owned slots (frontier list, own first) -> a record in the arena
// of every peer that reads the slot. A block takes kPackPer x kBlock list entries per step;
// the per-peer record positions come from one atomicAdd per (block step, peer) plus
// shared-memory prefixes over the warps (per-warp reservations on a handful of counters
// serialised in L2). The block's records for one peer are one contiguous run of up to
// kPackPer x kBlock records: staged in shared memory, then stored by the whole block with
// consecutive threads on consecutive words, shifted so that every warp store covers one
// aligned 128-B line (full-line writes over NVLink; a run per warp and peer cut most lines
// into two partial writes).
constexpr int kPackPer = 4;

__global__ void __launch_bounds__(kBlock) k_pack_peers(int algo, const uint32_t* __restrict__ list,
                                                        const unsigned long long* count, uint64_t lo, uint64_t hi,
                                                        const uint32_t* __restrict__ need,
                                                        const uint4* __restrict__ dist,
                                                        const uint32_t* __restrict__ lab, int nparts,
                                                        const __grid_constant__ PeerArenas A,
                                                        unsigned long long* peer_cnt) {
    constexpr int kWarps = kBlock / 32;
    __shared__ uint32_t stage[kPackPer * kBlock * 5];  // one peer's records of a block step
    __shared__ uint32_t wcnt[kWarps][kMaxPeers + 1];
    __shared__ unsigned long long bbase[kMaxPeers + 1];
    __shared__ uint32_t btot[kMaxPeers + 1];
    const uint64_t n = *count;
    const int W = record_words(algo);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lower = (1u << lane) - 1u;
    for (uint64_t t0 = (uint64_t)blockIdx.x * kPackPer * kBlock; t0 < n; t0 += (uint64_t)gridDim.x * kPackPer * kBlock) {
        // this warp's kPackPer groups of 32 consecutive list entries
        uint32_t sl[kPackPer], m[kPackPer];
        uint4 val[kPackPer];
#pragma unroll
        for (int j = 0; j < kPackPer; ++j) {
            const uint64_t i = t0 + ((uint64_t)warp * kPackPer + j) * 32 + lane;
            sl[j] = i < n ? list[i] : 0u;
            const bool mine = i < n && sl[j] >= lo && sl[j] < hi;
            m[j] = mine ? __ldg(need + (sl[j] - lo)) : 0u;
        }
#pragma unroll
        for (int j = 0; j < kPackPer; ++j) {  // each value is loaded once, for every peer
            val[j] = make_uint4(0u, 0u, 0u, 0u);
            if (m[j]) {
                if (algo == GXB_ALGO_SSSP) val[j] = dist[sl[j]];
                else val[j].x = lab[sl[j]];
            }
        }
        for (int q = 0; q < nparts; ++q) {
            uint32_t c = 0;
#pragma unroll
            for (int j = 0; j < kPackPer; ++j) c += __popc(__ballot_sync(0xffffffffu, (m[j] >> q) & 1u));
            if (lane == 0) wcnt[warp][q] = c;
        }
        __syncthreads();
        if (threadIdx.x < nparts) {  // block total per peer -> one reservation; warp prefixes in place
            const int q = threadIdx.x;
            uint32_t acc = 0;
            for (int w = 0; w < kWarps; ++w) {
                const uint32_t c = wcnt[w][q];
                wcnt[w][q] = acc;
                acc += c;
            }
            btot[q] = acc;
            bbase[q] = acc ? atomicAdd(peer_cnt + q, (unsigned long long)acc) : 0ull;
        }
        __syncthreads();
        for (int q = 0; q < nparts; ++q) {
            const uint32_t total = btot[q];
            if (!total) continue;  // block-uniform
            uint32_t pos = wcnt[warp][q];
#pragma unroll
            for (int j = 0; j < kPackPer; ++j) {
                const bool to_q = (m[j] >> q) & 1u;
                const unsigned b = __ballot_sync(0xffffffffu, to_q);
                if (to_q) {
                    uint32_t* r = stage + (pos + __popc(b & lower)) * W;
                    r[0] = sl[j];
                    r[1] = val[j].x;
                    if (algo == GXB_ALGO_SSSP) {
                        r[2] = val[j].y; r[3] = val[j].z; r[4] = val[j].w;
                    }
                }
                pos += __popc(b);
            }
            __syncthreads();
            uint32_t* dst = A.arena[q] + A.base[q] + bbase[q] * W;
            const int64_t words = (int64_t)total * W;
            const int64_t mis = (int64_t)((reinterpret_cast<uintptr_t>(dst) >> 2) & 31u);  // words past a line start
            for (int64_t k = (int64_t)threadIdx.x - mis; k < words; k += kBlock)
                if (k >= 0) dst[k] = stage[k];
            __syncthreads();  // the stage is reused for the next peer
        }
    }
    // one cumulative system-scope fence per block after a barrier (not one per thread): the
    // block's records are visible to the peers before the vote collective
    if (threadIdx.x == 0) __threadfence_system();
}

// Dense mirror exchange (rounds where most vertices changed): every owner's block of the
// next-value replica was all-gathered in place; a mirror whose landed value differs from
// the current one changed in its owner's round — install it, mark it active and append it
// to the frontier (warp-aggregated over consecutive slots: one OR per bitmap word).
template <class T>
__device__ __forceinline__ bool val_ne(const T& a, const T& b);
template <>
__device__ __forceinline__ bool val_ne<uint4>(const uint4& a, const uint4& b) {
    return a.x != b.x || a.y != b.y || a.z != b.z || a.w != b.w;
}
template <>
__device__ __forceinline__ bool val_ne<uint32_t>(const uint32_t& a, const uint32_t& b) {
    return a != b;
}

template <class T>
__global__ void k_dense_install(const T* __restrict__ next, T* cur, uint64_t S, uint64_t lo, uint64_t hi,
                                uint32_t* active, uint32_t* list, unsigned long long* count,
                                const uint32_t* __restrict__ outdeg, unsigned long long* units) {
    const int lane = threadIdx.x & 31;
    unsigned long long u = 0;
    for (uint64_t b = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) & ~31ull; b < S;
         b += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = b + lane;  // a warp covers 32 consecutive slots = one bitmap word
        bool ch = false;
        if (s < S && (s < lo || s >= hi)) {
            const T n = next[s];
            if (val_ne<T>(n, cur[s])) {
                cur[s] = n;
                ch = true;
                u += outdeg[s];
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, ch);
        if (!m) continue;
        if (lane == 0) atomicOr(active + (b >> 5), m);
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(count, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (ch) list[base + __popc(m & ((1u << lane) - 1u))] = (uint32_t)s;
    }
    for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
    if (lane == 0 && u) atomicAdd(units, u);
}

// counts into the vote block (after the 6 statistics), one double per receiver
__global__ void k_peer_counts(const unsigned long long* peer_cnt, int nparts, double* d_vote) {
    const int q = threadIdx.x;
    if (q < nparts) d_vote[6 + q] = (double)peer_cnt[q];
}

// needed-only dense exchange (PageRank): gather my values for every peer / scatter theirs
template <typename T>
__global__ void k_sparse_pack(const T* __restrict__ values, const uint32_t* __restrict__ idx, uint64_t n, T* out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = values[idx[i]];
}

template <typename T>
__global__ void k_sparse_unpack(T* values, const uint32_t* __restrict__ idx, uint64_t n, const T* __restrict__ in) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        values[idx[i]] = in[i];
}

}  // namespace gxb

using namespace gxb;

extern "C" {

// ---- fused PageRank exchange over peer memory (NVLink / NVSwitch) ----
int gxb_exchange_ipc_handle(gxb_state* s, int which, void* handle_out) {
    if (!s || !handle_out || which < 0 || which > 1) return fail(GXB_EINVAL, "gxb_exchange_ipc_handle: bad argument");
    if (s->algo != GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "peer replicas are PageRank-only");
    cudaIpcMemHandle_t h;
    GXB_CUDA(cudaIpcGetMemHandle(&h, s->d_contrib[which]));
    static_assert(sizeof(h) == GXB_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle_out, &h, sizeof(h));
    return GXB_OK;
}

int gxb_exchange_close_peers(gxb_state* s) {
    if (!s) return fail(GXB_EINVAL, "gxb_exchange_close_peers: null state");
    if (s->peer_ipc) {
        cudaSetDevice(s->g->ctx->device);
        for (int q = 0; q < s->npeers; ++q)
            for (int b = 0; b < 2; ++b)
                if (s->peer_contrib[q][b]) cudaIpcCloseMemHandle(s->peer_contrib[q][b]);
    }
    for (int q = 0; q < kMaxPeers; ++q) s->peer_contrib[q][0] = s->peer_contrib[q][1] = nullptr;
    s->npeers = 0;
    s->peer_ipc = false;
    return GXB_OK;
}

int gxb_exchange_open_peers(gxb_state* s, int npeers, const void* handles) {
    if (!s || npeers < 0 || npeers > kMaxPeers || (npeers && !handles))
        return fail(GXB_EINVAL, "gxb_exchange_open_peers: bad argument");
    if (s->algo != GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "peer replicas are PageRank-only");
    GXB_CHECK(gxb_exchange_close_peers(s));
    GXB_CUDA(cudaSetDevice(s->g->ctx->device));
    const auto* hb = static_cast<const unsigned char*>(handles);
    for (int q = 0; q < npeers; ++q) {
        for (int b = 0; b < 2; ++b) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, hb + (2 * q + b) * GXB_IPC_HANDLE_BYTES, sizeof(h));
            void* p = nullptr;
            const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) {
                cudaGetLastError();
                s->npeers = q + (b ? 1 : 0);
                s->peer_ipc = true;
                gxb_exchange_close_peers(s);
                return cuda_fail(e, "gxb_exchange_open_peers: cudaIpcOpenMemHandle");
            }
            s->peer_contrib[q][b] = p;
        }
        s->npeers = q + 1;
    }
    s->peer_ipc = npeers > 0;
    return GXB_OK;
}

int gxb_exchange_set_peer_ptrs(gxb_state* s, int npeers, void* const* ptrs) {
    if (!s || npeers < 0 || npeers > kMaxPeers || (npeers && !ptrs))
        return fail(GXB_EINVAL, "gxb_exchange_set_peer_ptrs: bad argument");
    if (s->algo != GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "peer replicas are PageRank-only");
    GXB_CHECK(gxb_exchange_close_peers(s));
    for (int q = 0; q < npeers; ++q) {
        s->peer_contrib[q][0] = ptrs[2 * q];
        s->peer_contrib[q][1] = ptrs[2 * q + 1];
    }
    s->npeers = npeers;
    return GXB_OK;
}

int gxb_exchange_buffer(gxb_state* s, int which, void** dev_ptr, uint64_t* bytes) {
    if (!s || !dev_ptr || !bytes) return fail(GXB_EINVAL, "gxb_exchange_buffer: null argument");
    gxb_graph* g = s->g;
    const uint64_t V = g->S, owned = g->hi - g->lo;  // value replicas span the slot space
    const uint64_t rec = (s->algo == GXB_ALGO_SSSP) ? 20 : 8;
    switch (which) {
        case GXB_BUF_VALUES:
            if (s->algo == GXB_ALGO_PAGERANK) {
                *dev_ptr = s->d_contrib[s->cur];
                *bytes = (s->msg32 ? 4 : 8) * V;
            } else if (s->algo == GXB_ALGO_SSSP) {
                *dev_ptr = s->d_dist_cur;
                *bytes = 16 * V;
            } else {
                *dev_ptr = s->d_lab_cur;
                *bytes = 4 * V;
            }
            return GXB_OK;
        case GXB_BUF_CONTRIB0:
        case GXB_BUF_CONTRIB1:
            if (s->algo != GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "GXB_BUF_CONTRIB* are PageRank-only");
            *dev_ptr = s->d_contrib[which == GXB_BUF_CONTRIB1 ? 1 : 0];
            *bytes = (s->msg32 ? 4 : 8) * V;
            return GXB_OK;
        case GXB_BUF_VALUES_NEXT:
            // PR: the contributions being written by the open round; SSSP / CC / LP: the
            // next-value replica (after a closed round the owned block equals the current
            // values; the non-owned part is the landing area of the dense mirror exchange)
            if (s->algo == GXB_ALGO_PAGERANK) {
                *dev_ptr = s->d_contrib[s->cur ^ 1];
                *bytes = (s->msg32 ? 4 : 8) * V;
            } else if (s->algo == GXB_ALGO_SSSP) {
                *dev_ptr = s->d_dist_next;
                *bytes = 16 * V;
            } else {
                *dev_ptr = s->d_lab_next;
                *bytes = 4 * V;
            }
            return GXB_OK;
        case GXB_BUF_SPARSE_SEND:
        case GXB_BUF_SPARSE_RECV: {
            if (s->algo != GXB_ALGO_PAGERANK || g->nparts < 2)
                return fail(GXB_EINVAL, "sparse exchange buffers: PageRank on a partitioned graph only");
            const uint64_t w = s->msg32 ? 4 : 8;
            const bool snd = which == GXB_BUF_SPARSE_SEND;
            const uint64_t n = snd ? g->xsend_off[g->nparts] : g->xrecv_off[g->nparts];
            void** slot = snd ? &s->d_xsend : &s->d_xrecv;
            if (!*slot) GXB_CHECK(dalloc(slot, w * (n + 1)));
            *dev_ptr = *slot;
            *bytes = w * n;
            return GXB_OK;
        }
        case GXB_BUF_SEND: {
            // sized for the largest partition: a padded all-gather sends max-count blocks
            uint64_t mx = owned;
            for (int q = 0; q < g->nparts; ++q) mx = std::max<uint64_t>(mx, g->bounds[q + 1] - g->bounds[q]);
            if (!s->d_send) GXB_CHECK(dalloc(&s->d_send, rec * (mx + 1) + 16));
            *dev_ptr = s->d_send;
            *bytes = rec * (mx + 1);
            return GXB_OK;
        }
        case GXB_BUF_RECV:
            if (!s->d_recv) {
                // room for every record of every rank, and for the padded all-gather of
                // nparts blocks of the largest owned range
                uint64_t mx = 0;
                for (int q = 0; q < g->nparts; ++q) mx = std::max<uint64_t>(mx, g->bounds[q + 1] - g->bounds[q]);
                const uint64_t cap = std::max<uint64_t>(V + 1, (uint64_t)g->nparts * (mx + 1));
                GXB_CHECK(dalloc(&s->d_recv, rec * cap + 16));
                s->recv_cap = cap;
            }
            *dev_ptr = s->d_recv;
            *bytes = rec * s->recv_cap;
            return GXB_OK;
        case GXB_BUF_RECORD_SIZE:
            *dev_ptr = nullptr;
            *bytes = rec;
            return GXB_OK;
    }
    return fail(GXB_EINVAL, "gxb_exchange_buffer: unknown buffer");
}

int gxb_exchange_pack(gxb_state* s, void* stream, uint64_t* count_out) {
    NvtxRange nvtx_("gxb_exchange_pack");
    if (!s || !count_out) return fail(GXB_EINVAL, "gxb_exchange_pack: null argument");
    if (s->algo == GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "gxb_exchange_pack: PageRank uses the dense exchange");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_exchange_pack: round still open");
    void* p;
    uint64_t b;
    GXB_CHECK(gxb_exchange_buffer(s, GXB_BUF_SEND, &p, &b));
    cudaStream_t st = (cudaStream_t)stream;
    gxb_iter_stats tmp;
    GXB_CHECK(gxb_stats(s, stream, &tmp));  // settles frontier_len
    gxb_graph* g = s->g;
    unsigned long long* d_cnt = reinterpret_cast<unsigned long long*>(s->d_fcount);  // scratch slot [1] is free now
    GXB_CUDA(cudaMemsetAsync(d_cnt + 1, 0, 8, st));
    if (s->frontier_len)
        k_pack<<<grid_for(s->frontier_len), kBlock, 0, st>>>(s->algo, s->d_frontier[0], s->d_fcount, g->lo, g->hi,
                                                             s->d_dist_cur, s->d_lab_cur, (uint32_t*)s->d_send,
                                                             d_cnt + 1);
    unsigned long long n = 0;
    GXB_CUDA(cudaMemcpyAsync(&n, d_cnt + 1, 8, cudaMemcpyDeviceToHost, st));
    GXB_CUDA(cudaStreamSynchronize(st));
    *count_out = n;
    return GXB_OK;
}

// asynchronous delta exchange: no host synchronisation; the record count travels in the
// vote block (gxb_stats_device) and the host-side frontier length is refreshed when the
// next round starts
int gxb_exchange_pack_async(gxb_state* s, void* stream) {
    NvtxRange nvtx_("gxb_exchange_pack_async");
    if (!s) return fail(GXB_EINVAL, "gxb_exchange_pack_async: null state");
    if (s->algo == GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "gxb_exchange_pack_async: PageRank uses the dense exchange");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_exchange_pack_async: round still open");
    void* p;
    uint64_t b;
    GXB_CHECK(gxb_exchange_buffer(s, GXB_BUF_SEND, &p, &b));
    if (!s->d_xscratch) GXB_CHECK(dalloc_t(&s->d_xscratch, 4));
    cudaStream_t st = (cudaStream_t)stream;
    gxb_graph* g = s->g;
    GXB_CUDA(cudaMemsetAsync(s->d_xscratch, 0, 8, st));
    // the closed round's frontier (its length is on the device) holds exactly the changed owned slots
    k_pack<<<grid_for(std::max<uint64_t>(1, g->hi - g->lo)), kBlock, 0, st>>>(
        s->algo, s->d_frontier[0], s->d_fcount, g->lo, g->hi, s->d_dist_cur, s->d_lab_cur, (uint32_t*)s->d_send,
        s->d_xscratch);
    GXB_CUDA(cudaGetLastError());
    s->packed_async = true;
    s->launches++;
    return GXB_OK;
}

int gxb_exchange_unpack_regions(gxb_state* s, const void* d_records, const uint64_t* counts, int nblocks,
                                uint64_t block_records, uint64_t frontier_after, uint64_t units_after,
                                void* stream) {
    NvtxRange nvtx_("gxb_exchange_unpack_regions");
    if (!s || !counts || nblocks < 0) return fail(GXB_EINVAL, "gxb_exchange_unpack_regions: bad argument");
    if (s->algo == GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "gxb_exchange_unpack_regions: PageRank uses the dense exchange");
    if (!s->d_xscratch) GXB_CHECK(dalloc_t(&s->d_xscratch, 4));
    gxb_graph* g = s->g;
    cudaStream_t st = (cudaStream_t)stream;
    const uint64_t W = (s->algo == GXB_ALGO_SSSP) ? 5 : 2;
    GXB_CUDA(cudaMemsetAsync(s->d_xscratch + 1, 0, 8, st));
    for (int q = 0; q < nblocks; ++q) {
        if (!counts[q]) continue;
        if (counts[q] > block_records) return fail(GXB_EINVAL, "gxb_exchange_unpack_regions: count exceeds the block");
        if (!d_records) return fail(GXB_EINVAL, "gxb_exchange_unpack_regions: null records");
        const uint32_t* rec = (const uint32_t*)d_records + (uint64_t)q * block_records * W;
        k_unpack<true><<<grid_for((counts[q] + kUnpackPer - 1) / kUnpackPer), kBlock, 0, st>>>(s->algo, rec, counts[q], g->lo, g->hi, s->d_dist_cur,
                                                         s->d_dist_next, s->d_lab_cur, s->d_lab_next, s->d_active[0],
                                                         s->d_frontier[0], s->d_fcount, g->d_outdeg, s->d_xscratch + 1);
        s->launches++;
    }
    GXB_CUDA(cudaGetLastError());
    if (frontier_after != ~0ull && units_after != ~0ull) {
        // the caller knows both from the vote: own changed + received records, and every
        // sender's next_units (a record is a changed vertex of its sender) — no read-back
        gxb_iter_stats tmp;
        GXB_CHECK(gxb_stats(s, stream, &tmp));  // the round's own statistics are collected first
        s->frontier_len = frontier_after;
        s->units_cur = units_after;
        s->unpack_pending = false;
    } else {
        s->unpack_pending = true;
    }
    return GXB_OK;
}

int gxb_exchange_unpack(gxb_state* s, const void* d_records, uint64_t count, void* stream) {
    NvtxRange nvtx_("gxb_exchange_unpack");
    if (!s) return fail(GXB_EINVAL, "gxb_exchange_unpack: null state");
    if (s->algo == GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "gxb_exchange_unpack: PageRank uses the dense exchange");
    if (count == 0) return GXB_OK;
    if (!d_records) return fail(GXB_EINVAL, "gxb_exchange_unpack: null records");
    gxb_graph* g = s->g;
    cudaStream_t st = (cudaStream_t)stream;
    GXB_CHECK(state_settle(s));  // the closed round's frontier first, then the records on top
    unsigned long long* d_units = reinterpret_cast<unsigned long long*>(s->d_fcount) + 1;
    GXB_CUDA(cudaMemsetAsync(d_units, 0, 8, st));
    k_unpack<true><<<grid_for((count + kUnpackPer - 1) / kUnpackPer), kBlock, 0, st>>>(s->algo, (const uint32_t*)d_records, count, g->lo, g->hi,
                                                 s->d_dist_cur, s->d_dist_next, s->d_lab_cur, s->d_lab_next,
                                                 s->d_active[0], s->d_frontier[0], s->d_fcount, g->d_outdeg, d_units);
    GXB_CUDA(cudaGetLastError());
    unsigned long long u = 0, n = 0;
    GXB_CUDA(cudaMemcpyAsync(&u, d_units, 8, cudaMemcpyDeviceToHost, st));
    GXB_CUDA(cudaMemcpyAsync(&n, s->d_fcount, 8, cudaMemcpyDeviceToHost, st));
    GXB_CUDA(cudaStreamSynchronize(st));
    s->units_cur += u;
    s->frontier_len = n;
    return GXB_OK;
}

int gxb_attrs_deliver(gxb_state* s, const uint64_t* host_dense, const double* host_vals, uint64_t n,
                      void* stream) {
    NvtxRange nvtx_("gxb_attrs_deliver");
    if (!s) return fail(GXB_EINVAL, "gxb_attrs_deliver: null state");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_attrs_deliver: a round is open");
    if (n == 0) return GXB_OK;
    if (!host_dense || !host_vals) return fail(GXB_EINVAL, "gxb_attrs_deliver: null input");
    gxb_graph* g = s->g;
    GXB_CUDA(cudaSetDevice(g->ctx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int W = s->algo == GXB_ALGO_SSSP ? 5 : 2;
    uint64_t* d_dense = nullptr;
    double* d_vals = nullptr;
    uint32_t* d_rec = nullptr;
    uint32_t* d_bad = nullptr;
    int rc = GXB_OK;
    if (dalloc_t(&d_dense, n) || dalloc_t(&d_vals, n * s->arity) || dalloc_t(&d_rec, n * W + 1) ||
        dalloc_t(&d_bad, 1)) {
        rc = fail(GXB_ENOMEM, "gxb_attrs_deliver: out of device memory");
    }
    uint32_t bad = 0;
    if (rc == GXB_OK) {
        cudaMemcpyAsync(d_dense, host_dense, 8 * n, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(d_vals, host_vals, 8 * n * s->arity, cudaMemcpyHostToDevice, st);
        cudaMemsetAsync(d_bad, 0, 4, st);
        k_deliver<<<grid_for(n), kBlock, 0, st>>>(s->algo, s->arity, d_dense, d_vals, n, g->V, g->d_dense2slot,
                                                  g->lo, g->hi, g->d_outdeg, s->d_rank[0], s->d_rank[1],
                                                  s->d_contrib[0], s->d_contrib[1], s->msg32, d_rec, d_bad);
        cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) rc = fail(GXB_ECUDA, "gxb_attrs_deliver: kernel failed");
    }
    if (rc == GXB_OK && (bad & 2u)) rc = fail(GXB_EINVAL, "gxb_attrs_deliver: target is owned by this partition or absent");
    else if (rc == GXB_OK && bad) rc = fail(GXB_ERANGE, "gxb_attrs_deliver: value not representable on the device");
    // installed mirror values are active sources of the next round (records = the delta path)
    if (rc == GXB_OK && s->algo != GXB_ALGO_PAGERANK) {
        s->lab_injective = false;
        rc = gxb_exchange_unpack(s, d_rec, n, stream);
    }
    cudaStreamSynchronize(st);
    dfree(d_dense);
    dfree(d_vals);
    dfree(d_rec);
    dfree(d_bad);
    return rc;
}

// ---- per-peer delta exchange (host side) ----
static int delta_layout(gxb_state* s, const uint64_t* cap) {
    // my arena: for every sender p != me, two parity blocks of cap[p][me] records
    const gxb_graph* g = s->g;
    const int n = g->nparts, me = g->part;
    const uint64_t W = s->algo == GXB_ALGO_SSSP ? 5 : 2;
    uint64_t acc = 0;
    for (int p = 0; p < n; ++p) {
        s->peer_recv_cap[p] = p == me ? 0 : cap[(uint64_t)p * n + me];
        for (int par = 0; par < 2; ++par) {
            s->arena_base[p][par] = acc;
            acc += s->peer_recv_cap[p] * W;
        }
    }
    s->arena_words = acc;
    // my blocks in every receiver's arena, same rule applied to the receiver's column
    for (int q = 0; q < n; ++q) {
        uint64_t a = 0;
        for (int p = 0; p < n; ++p) {
            const uint64_t c = p == q ? 0 : cap[(uint64_t)p * n + q];
            for (int par = 0; par < 2; ++par) {
                if (p == me) s->peer_base[q][par] = a;
                a += c * W;
            }
        }
    }
    return GXB_OK;
}

int gxb_exchange_delta_arena(gxb_state* s, const uint64_t* cap_matrix, void* ipc_handle_out) {
    NvtxRange nvtx_("gxb_exchange_delta_arena");
    if (!s || !cap_matrix) return fail(GXB_EINVAL, "gxb_exchange_delta_arena: null argument");
    if (s->algo == GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "gxb_exchange_delta_arena: PageRank uses the dense exchange");
    gxb_graph* g = s->g;
    const int n = g->nparts, me = g->part;
    if (n < 2 || n > kMaxPeers + 1) return fail(GXB_EINVAL, "gxb_exchange_delta_arena: needs 2..8 partitions");
    if (g->xsend_off.size() != (size_t)n + 1) return fail(GXB_EINVAL, "gxb_exchange_delta_arena: no per-peer lists");
    for (int q = 0; q < n; ++q)  // my row must be my own send lists
        if (q != me && cap_matrix[(uint64_t)me * n + q] != g->xsend_off[q + 1] - g->xsend_off[q])
            return fail(GXB_EINVAL, "gxb_exchange_delta_arena: capacity row disagrees with this partition");
    GXB_CHECK(gxb_exchange_delta_close(s));
    GXB_CUDA(cudaSetDevice(g->ctx->device));
    GXB_CHECK(delta_layout(s, cap_matrix));
    const uint64_t owned = g->hi - g->lo;
    GXB_CHECK(dalloc_t(&s->d_need, owned + 1));
    GXB_CUDA(cudaMemsetAsync(s->d_need, 0, 4 * (owned + 1), 0));
    for (int q = 0; q < n; ++q) {
        const uint64_t a = g->xsend_off[q], b = g->xsend_off[q + 1];
        if (q != me && b > a)
            k_need_mask<<<grid_for(b - a), kBlock>>>(g->d_xsend_idx + a, b - a, g->lo, 1u << q, s->d_need);
    }
    GXB_CHECK(dalloc_t(&s->d_arena, s->arena_words + 1));
    GXB_CHECK(dalloc_t(&s->d_peer_cnt, kMaxPeers + 1));
    GXB_CUDA(cudaDeviceSynchronize());
    if (ipc_handle_out) {
        cudaIpcMemHandle_t h;
        GXB_CUDA(cudaIpcGetMemHandle(&h, s->d_arena));
        std::memcpy(ipc_handle_out, &h, sizeof(h));
    }
    return GXB_OK;
}

int gxb_exchange_delta_open(gxb_state* s, const void* handles) {
    if (!s || !handles || !s->d_arena) return fail(GXB_EINVAL, "gxb_exchange_delta_open: bad argument");
    const gxb_graph* g = s->g;
    GXB_CUDA(cudaSetDevice(g->ctx->device));
    const auto* hb = static_cast<const unsigned char*>(handles);
    for (int q = 0; q < g->nparts; ++q) {
        if (q == g->part) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, hb + (uint64_t)q * GXB_IPC_HANDLE_BYTES, sizeof(h));
        void* p = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
            cudaGetLastError();
            s->delta_ipc = true;
            gxb_exchange_delta_close(s);
            return cuda_fail(e, "gxb_exchange_delta_open: cudaIpcOpenMemHandle");
        }
        s->peer_arena[q] = static_cast<uint32_t*>(p);
    }
    s->delta_ipc = true;
    s->delta_peers = true;
    s->delta_parity = 1;  // the first packed round uses parity 0
    return GXB_OK;
}

int gxb_exchange_delta_set_peers(gxb_state* s, void* const* arenas) {
    if (!s || !arenas || !s->d_arena) return fail(GXB_EINVAL, "gxb_exchange_delta_set_peers: bad argument");
    const gxb_graph* g = s->g;
    for (int q = 0; q < g->nparts; ++q)
        if (q != g->part) s->peer_arena[q] = static_cast<uint32_t*>(arenas[q]);
    s->delta_ipc = false;
    s->delta_peers = true;
    s->delta_parity = 1;
    return GXB_OK;
}

int gxb_exchange_delta_buffer(gxb_state* s, void** arena) {
    if (!s || !arena) return fail(GXB_EINVAL, "gxb_exchange_delta_buffer: null argument");
    *arena = s->d_arena;
    return GXB_OK;
}

int gxb_exchange_delta_close(gxb_state* s) {
    if (!s) return fail(GXB_EINVAL, "gxb_exchange_delta_close: null state");
    if (s->delta_ipc) {
        cudaSetDevice(s->g->ctx->device);
        for (int q = 0; q <= kMaxPeers; ++q)
            if (s->peer_arena[q]) cudaIpcCloseMemHandle(s->peer_arena[q]);
    }
    for (int q = 0; q <= kMaxPeers; ++q) s->peer_arena[q] = nullptr;
    s->delta_ipc = s->delta_peers = false;
    dfree(s->d_need);
    dfree(s->d_arena);
    dfree(s->d_peer_cnt);
    s->d_need = nullptr;
    s->d_arena = nullptr;
    s->d_peer_cnt = nullptr;
    return GXB_OK;
}

int gxb_exchange_delta_pack(gxb_state* s, double* d_vote, void* stream) {
    NvtxRange nvtx_("gxb_exchange_delta_pack");
    if (!s || !d_vote) return fail(GXB_EINVAL, "gxb_exchange_delta_pack: null argument");
    if (!s->delta_peers) return fail(GXB_ESTATE, "gxb_exchange_delta_pack: peer arenas not set up");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_exchange_delta_pack: round still open");
    gxb_graph* g = s->g;
    cudaStream_t st = (cudaStream_t)stream;
    s->delta_parity ^= 1;
    PeerArenas A{};
    for (int q = 0; q < g->nparts; ++q) {
        A.arena[q] = q == g->part ? nullptr : s->peer_arena[q];
        A.base[q] = s->peer_base[q][s->delta_parity];
    }
    GXB_CUDA(cudaMemsetAsync(s->d_peer_cnt, 0, 8 * (kMaxPeers + 1), st));
    k_pack_peers<<<grid_for(std::max<uint64_t>(1, (g->hi - g->lo) / kPackPer)), kBlock, 0, st>>>(
        s->algo, s->d_frontier[0], s->d_fcount, g->lo, g->hi, s->d_need, s->d_dist_cur, s->d_lab_cur, g->nparts, A,
        s->d_peer_cnt);
    k_peer_counts<<<1, 32, 0, st>>>(s->d_peer_cnt, g->nparts, d_vote);
    GXB_CUDA(cudaGetLastError());
    s->launches += 2;
    return GXB_OK;
}

int gxb_exchange_delta_unpack(gxb_state* s, const uint64_t* counts_from, void* stream) {
    NvtxRange nvtx_("gxb_exchange_delta_unpack");
    if (!s || !counts_from) return fail(GXB_EINVAL, "gxb_exchange_delta_unpack: null argument");
    if (!s->delta_peers) return fail(GXB_ESTATE, "gxb_exchange_delta_unpack: peer arenas not set up");
    gxb_graph* g = s->g;
    cudaStream_t st = (cudaStream_t)stream;
    GXB_CHECK(state_settle(s));  // the closed round's own frontier first
    if (!s->d_xscratch) GXB_CHECK(dalloc_t(&s->d_xscratch, 4));
    GXB_CUDA(cudaMemsetAsync(s->d_xscratch + 1, 0, 8, st));
    const int par = s->delta_parity;
    for (int p = 0; p < g->nparts; ++p) {
        if (p == g->part || !counts_from[p]) continue;
        if (counts_from[p] > s->peer_recv_cap[p]) return fail(GXB_EINVAL, "gxb_exchange_delta_unpack: count exceeds the block");
        k_unpack<false><<<grid_for((counts_from[p] + kUnpackPer - 1) / kUnpackPer), kBlock, 0, st>>>(s->algo, s->d_arena + s->arena_base[p][par], counts_from[p],
                                                              g->lo, g->hi, s->d_dist_cur, s->d_dist_next, s->d_lab_cur,
                                                              s->d_lab_next, s->d_active[0], s->d_frontier[0], s->d_fcount,
                                                              g->d_outdeg, s->d_xscratch + 1);
        s->launches++;
    }
    GXB_CUDA(cudaGetLastError());
    s->lab_injective = false;
    s->unpack_pending = true;  // the next round reads the frontier's length and GEN units back
    return GXB_OK;
}

int gxb_exchange_dense_install(gxb_state* s, void* stream) {
    NvtxRange nvtx_("gxb_exchange_dense_install");
    if (!s) return fail(GXB_EINVAL, "gxb_exchange_dense_install: null state");
    if (s->algo == GXB_ALGO_PAGERANK) return fail(GXB_EINVAL, "gxb_exchange_dense_install: PageRank uses the dense exchange");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_exchange_dense_install: round still open");
    gxb_graph* g = s->g;
    cudaStream_t st = (cudaStream_t)stream;
    GXB_CHECK(state_settle(s));  // the closed round's own frontier first
    if (!s->d_xscratch) GXB_CHECK(dalloc_t(&s->d_xscratch, 4));
    GXB_CUDA(cudaMemsetAsync(s->d_xscratch + 1, 0, 8, st));
    if (g->S) {
        const unsigned grid = grid_for(g->S);
        if (s->algo == GXB_ALGO_SSSP)
            k_dense_install<uint4><<<grid, kBlock, 0, st>>>(s->d_dist_next, s->d_dist_cur, g->S, g->lo, g->hi,
                                                            s->d_active[0], s->d_frontier[0], s->d_fcount, g->d_outdeg,
                                                            s->d_xscratch + 1);
        else
            k_dense_install<uint32_t><<<grid, kBlock, 0, st>>>(s->d_lab_next, s->d_lab_cur, g->S, g->lo, g->hi,
                                                               s->d_active[0], s->d_frontier[0], s->d_fcount,
                                                               g->d_outdeg, s->d_xscratch + 1);
        s->launches++;
    }
    GXB_CUDA(cudaGetLastError());
    s->lab_injective = false;
    s->unpack_pending = true;  // the next round reads the frontier's length and GEN units back
    return GXB_OK;
}

int gxb_exchange_sparse_counts(const gxb_state* s, uint64_t* send_counts, uint64_t* recv_counts) {
    if (!s || !send_counts || !recv_counts) return fail(GXB_EINVAL, "gxb_exchange_sparse_counts: null argument");
    const gxb_graph* g = s->g;
    if (g->nparts < 2 || g->xsend_off.empty()) return fail(GXB_EINVAL, "no needed-only exchange lists (nparts < 2)");
    for (int q = 0; q < g->nparts; ++q) {
        send_counts[q] = g->xsend_off[q + 1] - g->xsend_off[q];
        recv_counts[q] = g->xrecv_off[q + 1] - g->xrecv_off[q];
    }
    return GXB_OK;
}

int gxb_exchange_sparse_pack(gxb_state* s, void* stream) {
    if (!s) return fail(GXB_EINVAL, "gxb_exchange_sparse_pack: null state");
    if (s->in_round) return fail(GXB_ESTATE, "gxb_exchange_sparse_pack: round still open");
    void* buf;
    uint64_t bytes;
    GXB_CHECK(gxb_exchange_buffer(s, GXB_BUF_SPARSE_SEND, &buf, &bytes));
    const gxb_graph* g = s->g;
    const uint64_t n = g->xsend_off[g->nparts];
    cudaStream_t st = (cudaStream_t)stream;
    if (n) {
        if (s->msg32)
            k_sparse_pack<float><<<grid_for(n), kBlock, 0, st>>>((const float*)s->d_contrib[s->cur], g->d_xsend_idx, n,
                                                              (float*)buf);
        else
            k_sparse_pack<double><<<grid_for(n), kBlock, 0, st>>>(s->d_contrib[s->cur], g->d_xsend_idx, n, (double*)buf);
    }
    GXB_CUDA(cudaGetLastError());
    return GXB_OK;
}

int gxb_exchange_sparse_unpack(gxb_state* s, void* stream) {
    if (!s) return fail(GXB_EINVAL, "gxb_exchange_sparse_unpack: null state");
    void* buf;
    uint64_t bytes;
    GXB_CHECK(gxb_exchange_buffer(s, GXB_BUF_SPARSE_RECV, &buf, &bytes));
    const gxb_graph* g = s->g;
    const uint64_t n = g->xrecv_off[g->nparts];
    cudaStream_t st = (cudaStream_t)stream;
    if (n) {
        if (s->msg32)
            k_sparse_unpack<float><<<grid_for(n), kBlock, 0, st>>>((float*)s->d_contrib[s->cur], g->d_xrecv_idx, n,
                                                                (const float*)buf);
        else
            k_sparse_unpack<double><<<grid_for(n), kBlock, 0, st>>>(s->d_contrib[s->cur], g->d_xrecv_idx, n,
                                                                 (const double*)buf);
    }
    GXB_CUDA(cudaGetLastError());
    return GXB_OK;
}

int gxb_exchange_finish(gxb_state* s, void* stream) {
    if (!s) return fail(GXB_EINVAL, "gxb_exchange_finish: null state");
    GXB_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return GXB_OK;
}

}  // extern "C"
