// gxb_rmat.cu — device R-MAT edge stream (include/gxb_rmat.h), the ingest path
// that feeds scale-26 graphs without a host round trip.
#include "gxb_internal.cuh"
#include "../../include/gxb_rmat.h"

namespace gxb {

__global__ void k_rmat(gxb_rmat_params p, uint64_t seedmix, uint64_t wseedmix, uint64_t m, uint32_t* src,
                       uint32_t* dst, uint32_t* w) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s, d;
        gxb_rmat_edge(&p, seedmix, i, &s, &d);
        src[i] = s;
        dst[i] = d;
        uint32_t ww = 0;
        if (w) w[i] = ww = gxb_rmat_weight(&p, wseedmix, i);
        if (p.symmetric) {
            src[m + i] = d;
            dst[m + i] = s;
            if (w) w[m + i] = ww;
        }
    }
}

}  // namespace gxb

extern "C" int gxb_rmat_generate(gxb_ctx* ctx, const gxb_rmat_args* a, uint32_t* d_src, uint32_t* d_dst,
                                 uint32_t* d_w, void* stream) {
    using namespace gxb;
    if (!ctx || !ctx->alive) return fail(GXB_ESTATE, "gxb_rmat_generate: daemon not initialised");
    if (!a || !d_src || !d_dst) return fail(GXB_EINVAL, "gxb_rmat_generate: null argument");
    if (a->scale < 1 || a->scale > 32) return fail(GXB_EINVAL, "gxb_rmat_generate: scale must be in [1, 32]");
    if ((uint64_t)a->a + a->b + a->c > 0xFFFFFFFFull)
        return fail(GXB_EINVAL, "gxb_rmat_generate: a + b + c must be < 1");
    gxb_rmat_params p;
    p.scale = a->scale;
    p.edge_factor = a->edge_factor;
    p.seed = a->seed;
    p.a = a->a;
    p.b = a->b;
    p.c = a->c;
    p.wmax = a->wmax;
    p.scramble = a->scramble;
    p.symmetric = a->symmetric;
    const uint64_t m = (uint64_t)a->edge_factor << a->scale;
    GXB_CUDA(cudaSetDevice(ctx->device));
    k_rmat<<<grid_for(m, kBlock, 148ull * 16), kBlock, 0, (cudaStream_t)stream>>>(
        p, gxb_rmat_seedmix(a->seed), gxb_rmat_wseedmix(a->seed), m, d_src, d_dst, a->wmax ? d_w : nullptr);
    GXB_CUDA(cudaGetLastError());
    return GXB_OK;
}
