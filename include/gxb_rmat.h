/*
 * gxb_rmat.h — the seeded R-MAT edge generator shared by the device store
 * (libgxb200.so), the CPU oracle and the bench.
 *
 * The reference ships no R-MAT generator ("Corpus generators":
 * `A/generators.py:1-98` has path/cycle/star/random/components only), so this
 * header FIXES one formulation (SURVEY.md Appendix B asks the build to "fix
 * one formulation and seed"):
 *
 *   edge i in [0, m), m = edge_factor << scale
 *   for level l in [0, scale):
 *       u = 32-bit draw (l even: low half, l odd: high half of
 *           splitmix64(seedmix + (i << 4 | l >> 1)))
 *       quadrant: u < A -> (0,0); u < A+B -> (0,1); u < A+B+C -> (1,0); else (1,1)
 *       src |= row << l; dst |= col << l
 *   optional: src = scramble(src), dst = scramble(dst)   (bijection on [0, 2^scale))
 *   weight   = 1 + splitmix64(wseedmix + i) % wmax        (integers in [1, wmax])
 *
 * Probabilities are integer thresholds (p * 2^32, rounded down), so every
 * implementation — CUDA, C, numpy — produces bit-identical edges. Duplicate
 * edges and self-loops are kept, exactly as `load_edge_list` keeps them
 * (`A/graph.py:131-166`).
 */
#ifndef GXB_RMAT_H
#define GXB_RMAT_H

#include <stdint.h>

#if defined(__CUDACC__)
#define GXB_HD __host__ __device__ __forceinline__
#else
#define GXB_HD static inline
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct gxb_rmat_params {
    uint32_t scale;        /* id space = 2^scale, scale in [1, 32] */
    uint32_t edge_factor;  /* m = edge_factor << scale */
    uint64_t seed;
    uint32_t a, b, c;      /* quadrant thresholds in units of 2^-32; d = 2^32 - a - b - c */
    uint32_t wmax;         /* weights uniform in [1, wmax]; 0 = unweighted (weight 1) */
    uint32_t scramble;     /* 1 = apply the seeded id bijection (Graph500-style) */
    uint32_t symmetric;    /* 1 = append the reversed copy of every edge (CC input) */
} gxb_rmat_params;

GXB_HD uint64_t gxb_splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

GXB_HD uint64_t gxb_rmat_seedmix(uint64_t seed) { return gxb_splitmix64(seed ^ 0xD1B54A32D192ED03ull); }
GXB_HD uint64_t gxb_rmat_wseedmix(uint64_t seed) { return gxb_splitmix64(seed ^ 0x8CB92BA72F3D8DD7ull); }

/* Bijection on [0, 2^scale): xor with a seed mask, two odd multiplies and
 * xor-shifts, all modulo 2^scale (each step is invertible). */
GXB_HD uint64_t gxb_rmat_scramble(uint64_t x, uint32_t scale, uint64_t seedmix) {
    const uint64_t mask = (scale >= 64) ? ~0ull : ((1ull << scale) - 1ull);
    const uint32_t sh = (scale + 1u) / 2u;
    x = (x ^ (seedmix >> 7)) & mask;
    x = (x * 0x9E3779B97F4A7C15ull) & mask;   /* odd multiplier */
    x ^= x >> sh;
    x = (x * 0xC2B2AE3D27D4EB4Full) & mask;   /* odd multiplier */
    x ^= x >> sh;
    return x & mask;
}

/* Edge i of the (non-symmetrised) stream. */
GXB_HD void gxb_rmat_edge(const gxb_rmat_params* p, uint64_t seedmix, uint64_t i,
                          uint32_t* src_out, uint32_t* dst_out) {
    uint64_t src = 0, dst = 0, r = 0;
    const uint32_t tab = p->a + p->b, tabc = p->a + p->b + p->c;
    for (uint32_t l = 0; l < p->scale; ++l) {
        if ((l & 1u) == 0u) r = gxb_splitmix64(seedmix + ((i << 4) | (uint64_t)(l >> 1)));
        const uint32_t u = (l & 1u) ? (uint32_t)(r >> 32) : (uint32_t)r;
        uint64_t row, col;
        if (u < p->a)       { row = 0; col = 0; }
        else if (u < tab)   { row = 0; col = 1; }
        else if (u < tabc)  { row = 1; col = 0; }
        else                { row = 1; col = 1; }
        src |= row << l;
        dst |= col << l;
    }
    if (p->scramble) {
        src = gxb_rmat_scramble(src, p->scale, seedmix);
        dst = gxb_rmat_scramble(dst, p->scale, seedmix);
    }
    *src_out = (uint32_t)src;
    *dst_out = (uint32_t)dst;
}

GXB_HD uint32_t gxb_rmat_weight(const gxb_rmat_params* p, uint64_t wseedmix, uint64_t i) {
    if (p->wmax == 0u) return 1u;
    return 1u + (uint32_t)(gxb_splitmix64(wseedmix + i) % (uint64_t)p->wmax);
}

/* Number of edges in the emitted stream (2m when symmetrised). */
GXB_HD uint64_t gxb_rmat_num_edges(const gxb_rmat_params* p) {
    const uint64_t m = (uint64_t)p->edge_factor << p->scale;
    return p->symmetric ? 2ull * m : m;
}

#ifdef __cplusplus
}
#endif

#endif /* GXB_RMAT_H */
