// dsmem_gather_probe.cu — feasibility probe (development aid, not part of libgxb200):
// random 8-B element gathers from (a) global memory through LDGSTS (k_tile_a's path),
// (b) a CTA-local shared-memory table (ld.shared), (c) a table distributed over the shared
// memory of an 8-CTA thread-block cluster (mapa + ld.shared::cluster, DSMEM). Question: can a
// cluster-wide hot-source table (8 x 192 KB = 196,608 f64 values, ~40% of R-MAT S26's edges)
// serve hub-source gathers faster than the L1 data pipe serves LDGSTS, i.e. is DSMEM a way
// to cut the gathered-from-global elements per edge of PageRank's k_tile_a?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_gather_probe tools/dsmem_gather_probe.cu
//   ./dsmem_gather_probe [num_gathers]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

constexpr int kCluster = 8;
constexpr int kSlice = 24576;                     // f64 values per CTA (192 KB)
constexpr int kTable = kSlice * kCluster;         // cluster-wide table
constexpr int kThreads = 1024;
constexpr int kPer = 8;                           // gathers per lane per step

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// (a) LDGSTS from global, same index stream (idx < table_size) — k_tile_a's gather
__global__ void __launch_bounds__(256) k_ldgsts(const double* __restrict__ vals, const uint32_t* __restrict__ idx,
                                                uint64_t n, double* out) {
    __shared__ double row[8][kPer * 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double acc = 0.0;
    const uint64_t nw = (uint64_t)gridDim.x * 8;
    for (uint64_t t = blockIdx.x * 8ull + w; t * (kPer * 32) < n; t += nw) {
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const uint32_t s = idx[t * (kPer * 32) + 32 * j + lane];
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&row[w][32 * j + lane])),
                         "l"(vals + s)
                         : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kPer; ++j) acc += row[w][32 * j + lane];
        __syncwarp();
    }
    if (acc == 12345.678) out[0] = acc;
}

// (b) CTA-local table: indices taken modulo the slice
__global__ void __launch_bounds__(kThreads) k_lds(const double* __restrict__ vals, const uint32_t* __restrict__ idx,
                                                 uint64_t n, double* out) {
    extern __shared__ double tab[];
    for (int i = threadIdx.x; i < kSlice; i += blockDim.x) tab[i] = vals[i];
    __syncthreads();
    double acc = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += stride)
        acc += tab[idx[e] % kSlice];
    if (acc == 12345.678) out[0] = acc;
}

// (c) cluster-distributed table: value i lives in CTA rank i / kSlice at offset i % kSlice
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads)
    k_dsmem(const double* __restrict__ vals, const uint32_t* __restrict__ idx, uint64_t n, double* out) {
    extern __shared__ double tab[];
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = threadIdx.x; i < kSlice; i += blockDim.x) tab[i] = vals[rank * kSlice + i];
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    const uint32_t base = smem_u32(tab);
    double acc = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += stride) {
        const uint32_t i = idx[e];
        const uint32_t r = i / kSlice, off = i - r * kSlice;
        uint32_t remote;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(base + 8 * off), "r"(r));
        double v;
        asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
        acc += v;
    }
    // keep every CTA's table alive until the whole cluster is done reading
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
    const uint64_t ng = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : (1ull << 28);
    std::vector<uint32_t> h(ng);
    uint64_t x = 88172645463325252ull;
    for (auto& v : h) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        v = (uint32_t)(x % kTable);
    }
    double *vals, *out;
    uint32_t* idx;
    CK(cudaMalloc(&vals, 8ull * kTable));
    CK(cudaMalloc(&idx, 4 * ng));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(vals, 0, 8ull * kTable));
    CK(cudaMemcpy(idx, h.data(), 4 * ng, cudaMemcpyHostToDevice));
    const size_t smem = 8ull * kSlice;
    CK(cudaFuncSetAttribute(k_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const char* names[3] = {"ldgsts_global", "lds_cta_table", "dsmem_cluster8_table"};
    for (int variant = 0; variant < 3; ++variant) {
        float best = 1e9f;
        for (int rep = 0; rep < 4; ++rep) {
            CK(cudaEventRecord(a));
            if (variant == 0) k_ldgsts<<<148 * 6, 256>>>(vals, idx, ng, out);
            else if (variant == 1) k_lds<<<148, kThreads, smem>>>(vals, idx, ng, out);
            else k_dsmem<<<144, kThreads, smem>>>(vals, idx, ng, out);  // 18 clusters of 8
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            CK(cudaGetLastError());
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (rep) best = ms < best ? ms : best;
        }
        std::printf("{\"variant\": \"%s\", \"gathers\": %llu, \"table_values\": %d, \"ms\": %.3f, "
                    "\"Ggathers_per_s\": %.1f}\n",
                    names[variant], (unsigned long long)ng, variant == 1 ? kSlice : kTable, best,
                    ng / (best * 1e-3) / 1e9);
    }
    return 0;
}
