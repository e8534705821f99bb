// tma_gather_probe.cu — feasibility probe (development aid, not part of libgxb200):
// random 8-B element gathers into shared memory through (a) LDGSTS, one per lane and
// element, and (b) the TMA unit's tile::gather4 (four 16-B rows per instruction, the
// element's row), to see whether TMA gathers escape the L1 data-pipe bound of k_tile_a.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_gather_probe tools/tma_gather_probe.cu
//   ./tma_gather_probe [num_values] [num_gathers]
#include <cuda.h>
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

constexpr int kWarps = 8;
constexpr int kTile = 256;  // elements per warp per step

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// (a) LDGSTS: lane l copies elements 32 j + l of the tile
__global__ void __launch_bounds__(256) k_ldgsts(const double* __restrict__ vals, const uint32_t* __restrict__ idx,
                                                uint64_t n, double* out) {
    __shared__ double row[kWarps][kTile];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double acc = 0.0;
    const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
    for (uint64_t t = blockIdx.x * (uint64_t)kWarps + w; t * kTile < n; t += nwarps) {
#pragma unroll
        for (int j = 0; j < kTile / 32; ++j) {
            const uint32_t s = idx[t * kTile + 32 * j + lane];
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&row[w][32 * j + lane])),
                         "l"(vals + s)
                         : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kTile / 32; ++j) acc += row[w][32 * j + lane];
        __syncwarp();
    }
    if (acc == 12345.678) out[0] = acc;
}

// (b) TMA gather4: the value array viewed as [rows = n_values / 2][2 doubles]; element s lives
// in row s >> 1. Each gather4 lands 4 rows (64 B); a tile of 256 elements is 64 gather4.
__global__ void __launch_bounds__(256) k_gather4(const __grid_constant__ CUtensorMap map,
                                                 const uint32_t* __restrict__ idx, uint64_t n, double* out) {
    constexpr int kT = kTile / 2;  // 128 elements = one gather4 per lane per step
    __shared__ alignas(128) double rows[kWarps][kT * 4];  // each gather4 lands at a 128-B boundary
    __shared__ alignas(8) uint64_t bar[kWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[w])));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    double acc = 0.0;
    uint32_t phase = 0;
    const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
    for (uint64_t t = blockIdx.x * (uint64_t)kWarps + w; t * kT < n; t += nwarps) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w])),
                         "r"(kT * 16)
                         : "memory");
        __syncwarp();
#pragma unroll
        for (int g = 0; g < kT / 4 / 32; ++g) {  // one gather4 per lane
            const uint64_t e = t * kT + (uint64_t)(g * 32 + lane) * 4;
            const int r0 = (int)(idx[e] >> 1), r1 = (int)(idx[e + 1] >> 1), r2 = (int)(idx[e + 2] >> 1),
                      r3 = (int)(idx[e + 3] >> 1);
            const uint32_t dst = smem_u32(&rows[w][(g * 32 + lane) * 16]);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
                "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(&bar[w]))
                : "memory");
        }
        // wait for the tile's bytes
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(smem_u32(&bar[w])), "r"(phase)
                : "memory");
        }
        phase ^= 1;
#pragma unroll
        for (int j = 0; j < kT / 32; ++j) {
            const uint64_t e = t * kT + 32 * j + lane;
            const uint32_t k = 32 * j + lane;  // gather k / 4, row k % 4 of it
            acc += rows[w][(k >> 2) * 16 + (k & 3) * 2 + (idx[e] & 1)];
        }
        __syncwarp();
    }
    if (acc == 12345.678) out[0] = acc;
}


// (c) hybrid: per 256-element tile, 128 elements through gather4 (one per lane) and 128
// through LDGSTS (4 per lane) — do the TMA and LSU paths add up?
__global__ void __launch_bounds__(256) k_hybrid(const __grid_constant__ CUtensorMap map, const double* __restrict__ vals,
                                                const uint32_t* __restrict__ idx, uint64_t n, double* out) {
    constexpr int kT = kTile / 2;
    __shared__ alignas(128) double rows[kWarps][kT * 4];
    __shared__ double row2[kWarps][kT];
    __shared__ alignas(8) uint64_t bar[kWarps];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[w])));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    double acc = 0.0;
    uint32_t phase = 0;
    const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
    for (uint64_t t = blockIdx.x * (uint64_t)kWarps + w; t * kTile < n; t += nwarps) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w])), "r"(kT * 16)
                         : "memory");
        __syncwarp();
        const uint64_t e = t * kTile + (uint64_t)lane * 4;
        const int r0 = (int)(idx[e] >> 1), r1 = (int)(idx[e + 1] >> 1), r2 = (int)(idx[e + 2] >> 1),
                  r3 = (int)(idx[e + 3] >> 1);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(&rows[w][lane * 16])),
            "l"(&map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(&bar[w]))
            : "memory");
#pragma unroll
        for (int j = 0; j < kT / 32; ++j) {
            const uint32_t s = idx[t * kTile + kT + 32 * j + lane];
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&row2[w][32 * j + lane])),
                         "l"(vals + s)
                         : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(smem_u32(&bar[w])), "r"(phase)
                : "memory");
        }
        phase ^= 1;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < kT / 32; ++j) {
            const uint32_t k = 32 * j + lane;
            acc += rows[w][(k >> 2) * 16 + (k & 3) * 2 + (idx[t * kTile + k] & 1)] + row2[w][k];
        }
        __syncwarp();
    }
    if (acc == 12345.678) out[0] = acc;
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const uint64_t nv = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : (1ull << 25);
    const uint64_t ng = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : (1ull << 28);
    std::vector<uint32_t> h(ng);
    uint64_t x = 88172645463325252ull;
    for (auto& v : h) {
        x ^= x << 13;
        x ^= x >> 7;
        x ^= x << 17;
        v = (uint32_t)(x % nv);
    }
    double* vals;
    uint32_t* idx;
    double* out;
    CK(cudaMalloc(&vals, 8 * nv));
    CK(cudaMalloc(&idx, 4 * ng));
    CK(cudaMalloc(&out, 8));
    CK(cudaMemset(vals, 0, 8 * nv));
    CK(cudaMemcpy(idx, h.data(), 4 * ng, cudaMemcpyHostToDevice));

    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    CUtensorMap map;
    const cuuint64_t dims[2] = {2, nv / 2};
    const cuuint64_t strides[1] = {16};
    const cuuint32_t box[2] = {2, 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = ((EncodeTiled)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, vals, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::fprintf(stderr, "cuTensorMapEncodeTiled failed: %d\n", (int)r);
        return 1;
    }
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    for (int variant = 0; variant < 3; ++variant) {
        for (int occ : {4, 6, 8}) {
            const unsigned grid = 148 * occ;
            float best = 1e9f;
            for (int rep = 0; rep < 4; ++rep) {
                CK(cudaEventRecord(a));
                if (variant == 0) k_ldgsts<<<grid, 256>>>(vals, idx, ng, out);
                else if (variant == 1) k_gather4<<<grid, 256>>>(map, idx, ng, out);
                else k_hybrid<<<grid, 256>>>(map, vals, idx, ng, out);
                CK(cudaEventRecord(b));
                CK(cudaEventSynchronize(b));
                CK(cudaGetLastError());
                float ms;
                CK(cudaEventElapsedTime(&ms, a, b));
                if (rep) best = ms < best ? ms : best;
            }
            std::printf("{\"variant\": \"%s\", \"ctas_per_sm\": %d, \"gathers\": %llu, \"values\": %llu, "
                        "\"ms\": %.3f, \"Ggathers_per_s\": %.1f}\n",
                        variant == 2 ? "hybrid" : variant ? "tma_gather4" : "ldgsts", occ, (unsigned long long)ng, (unsigned long long)nv,
                        best, ng / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}
