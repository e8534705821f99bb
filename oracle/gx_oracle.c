/*
 * gx_oracle.c — TEST INFRASTRUCTURE ONLY; see gx_oracle.h for the contract.
 * CPU restatement of `run_reference` (pkg/src/accelgraph/algorithms.py:298-342).
 * Compile with -ffp-contract=off so `0.15 + 0.85 * s` keeps the reference's two
 * roundings (PageRank.apply_one, algorithms.py:157-159).
 */
#include "gx_oracle.h"
#include "../include/gxb_rmat.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

struct gxo_graph {
    uint64_t V, E;
    uint32_t* ids;        /* ascending present ids (dense index -> id) */
    uint32_t* outdeg;     /* per dense vertex */
    uint64_t* in_off;     /* CSC offsets, V+1 */
    uint32_t* in_src;     /* dense source per in-edge, ordered (src asc, file order) */
    double* in_w;         /* weight per in-edge */
};

typedef struct { uint32_t s; double w; } gxo_sw;

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

static uint64_t lower_bound_u32(const uint32_t* a, uint64_t n, uint32_t key) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (a[mid] < key) lo = mid + 1; else hi = mid;
    }
    return lo;
}

void gxo_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int gxo_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void gxo_graph_free(gxo_graph* g) {
    if (!g) return;
    free(g->ids); free(g->outdeg); free(g->in_off); free(g->in_src); free(g->in_w);
    free(g);
}

static int cmp_sw(const void* a, const void* b) {
    const gxo_sw* x = (const gxo_sw*)a;
    const gxo_sw* y = (const gxo_sw*)b;
    if (x->s != y->s) return (x->s > y->s) - (x->s < y->s);
    return (x->w > y->w) - (x->w < y->w);
}

/* Ingest in parallel. Within one destination the in-edges end up ordered by
 * (source, weight): the reference's order is (source asc, file order), and
 * in-edges that share both source and destination carry the same message for
 * PageRank / LP / CC and are folded by min for SSSP, so the order among them
 * never changes a result — every fold stays the reference's. */
gxo_graph* gxo_graph_new(uint64_t E, const uint32_t* src, const uint32_t* dst, const double* w) {
    gxo_graph* g = (gxo_graph*)calloc(1, sizeof(gxo_graph));
    if (!g) return NULL;
    g->E = E;
    uint32_t max_id = 0;
    #pragma omp parallel for schedule(static) reduction(max:max_id)
    for (int64_t e = 0; e < (int64_t)E; ++e) {
        if (src[e] > max_id) max_id = src[e];
        if (dst[e] > max_id) max_id = dst[e];
    }
    uint32_t* sidx = (uint32_t*)malloc(sizeof(uint32_t) * (E ? E : 1));
    uint32_t* didx = (uint32_t*)malloc(sizeof(uint32_t) * (E ? E : 1));
    if (!sidx || !didx) { free(sidx); free(didx); gxo_graph_free(g); return NULL; }

    /* vertex set = ids present in any edge (graph.py:163-164) */
    const uint64_t dense_limit = 4ull * E + (1ull << 26);
    if ((uint64_t)max_id + 1 <= dense_limit) {
        const int64_t n = (int64_t)max_id + 1;
        uint32_t* map = (uint32_t*)calloc((size_t)n, sizeof(uint32_t));
        if (!map) { free(sidx); free(didx); gxo_graph_free(g); return NULL; }
        #pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < (int64_t)E; ++e) { map[src[e]] = 1; map[dst[e]] = 1; }
        /* blocked exclusive scan of the presence flags: dense index = rank of the id */
        const int64_t nb = 4096, bs = (n + nb - 1) / nb;
        uint64_t* bsum = (uint64_t*)calloc(nb + 1, sizeof(uint64_t));
        #pragma omp parallel for schedule(static)
        for (int64_t b = 0; b < nb; ++b) {
            uint64_t c = 0;
            for (int64_t i = b * bs; i < n && i < (b + 1) * bs; ++i) c += (E && map[i]);
            bsum[b + 1] = c;
        }
        for (int64_t b = 0; b < nb; ++b) bsum[b + 1] += bsum[b];
        const uint64_t V = bsum[nb];
        g->V = V;
        g->ids = (uint32_t*)malloc(sizeof(uint32_t) * (V ? V : 1));
        #pragma omp parallel for schedule(static)
        for (int64_t b = 0; b < nb; ++b) {
            uint64_t k = bsum[b];
            for (int64_t i = b * bs; i < n && i < (b + 1) * bs; ++i)
                if (E && map[i]) { g->ids[k] = (uint32_t)i; map[i] = (uint32_t)k++; }
        }
        free(bsum);
        #pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < (int64_t)E; ++e) { sidx[e] = map[src[e]]; didx[e] = map[dst[e]]; }
        free(map);
    } else {
        uint32_t* all = (uint32_t*)malloc(sizeof(uint32_t) * 2 * E);
        if (!all) { free(sidx); free(didx); gxo_graph_free(g); return NULL; }
        memcpy(all, src, sizeof(uint32_t) * E);
        memcpy(all + E, dst, sizeof(uint32_t) * E);
        qsort(all, 2 * E, sizeof(uint32_t), cmp_u32);
        uint64_t V = 0;
        for (uint64_t i = 0; i < 2 * E; ++i) if (i == 0 || all[i] != all[i - 1]) all[V++] = all[i];
        g->V = V;
        g->ids = (uint32_t*)realloc(all, sizeof(uint32_t) * (V ? V : 1));
        #pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < (int64_t)E; ++e) {
            sidx[e] = (uint32_t)lower_bound_u32(g->ids, V, src[e]);
            didx[e] = (uint32_t)lower_bound_u32(g->ids, V, dst[e]);
        }
    }
    const uint64_t V = g->V;
    g->outdeg = (uint32_t*)calloc(V ? V : 1, sizeof(uint32_t));
    g->in_off = (uint64_t*)calloc(V + 1, sizeof(uint64_t));
    g->in_src = (uint32_t*)malloc(sizeof(uint32_t) * (E ? E : 1));
    g->in_w = w ? (double*)malloc(sizeof(double) * (E ? E : 1)) : NULL;
    uint64_t* cur = (uint64_t*)malloc(sizeof(uint64_t) * (V + 1));
    if (!g->outdeg || !g->in_off || !g->in_src || (w && !g->in_w) || !cur) {
        free(cur); free(sidx); free(didx); gxo_graph_free(g); return NULL;
    }
    /* out-degree counts duplicates and self-loops (graph.py:203-210) */
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)E; ++e) {
        #pragma omp atomic
        g->outdeg[sidx[e]]++;
        #pragma omp atomic
        g->in_off[didx[e] + 1]++;
    }
    for (uint64_t v = 0; v < V; ++v) g->in_off[v + 1] += g->in_off[v];
    memcpy(cur, g->in_off, sizeof(uint64_t) * (V + 1));
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < (int64_t)E; ++e) {
        uint64_t pos;
        #pragma omp atomic capture
        pos = cur[didx[e]]++;
        g->in_src[pos] = sidx[e];
        if (w) g->in_w[pos] = w[e];
    }
    free(cur); free(sidx); free(didx);
    /* each destination's in-edges in source order (see above) */
    #pragma omp parallel
    {
        gxo_sw* tmp = NULL;
        uint64_t tcap = 0;
        #pragma omp for schedule(dynamic, 256)
        for (int64_t d = 0; d < (int64_t)V; ++d) {
            const uint64_t a = g->in_off[d], n = g->in_off[d + 1] - a;
            if (n < 2) continue;
            if (!w) { qsort(g->in_src + a, n, sizeof(uint32_t), cmp_u32); continue; }
            if (n > tcap) { free(tmp); tcap = n; tmp = (gxo_sw*)malloc(sizeof(gxo_sw) * tcap); }
            for (uint64_t k = 0; k < n; ++k) { tmp[k].s = g->in_src[a + k]; tmp[k].w = g->in_w[a + k]; }
            qsort(tmp, n, sizeof(gxo_sw), cmp_sw);
            for (uint64_t k = 0; k < n; ++k) { g->in_src[a + k] = tmp[k].s; g->in_w[a + k] = tmp[k].w; }
        }
        free(tmp);
    }
    return g;
}

uint64_t gxo_graph_num_vertices(const gxo_graph* g) { return g->V; }
uint64_t gxo_graph_num_edges(const gxo_graph* g) { return g->E; }
void gxo_graph_ids(const gxo_graph* g, uint32_t* out) { memcpy(out, g->ids, sizeof(uint32_t) * g->V); }
void gxo_graph_out_degree(const gxo_graph* g, uint32_t* out) { memcpy(out, g->outdeg, sizeof(uint32_t) * g->V); }

static void record(int64_t it, int64_t cap, int64_t* tu, int64_t* tc, double* tm,
                   int64_t units, int64_t changed, double max_stat) {
    if (it >= cap) return;
    if (tu) tu[it] = units;
    if (tc) tc[it] = changed;
    if (tm) tm[it] = max_stat;
}

/* LP mode of a label multiset: max count, ties to the smallest label
 * (LabelPropagation.apply_one, algorithms.py:194-199). */
static uint32_t lp_mode(uint32_t* buf, uint64_t n) {
    qsort(buf, n, sizeof(uint32_t), cmp_u32);
    uint32_t best = buf[0];
    uint64_t best_cnt = 0, i = 0;
    while (i < n) {
        uint64_t j = i;
        while (j < n && buf[j] == buf[i]) ++j;
        if (j - i > best_cnt) { best_cnt = j - i; best = buf[i]; }
        i = j;
    }
    return best;
}

int gxo_run(const gxo_graph* g, int algo, int nsrc, const uint32_t* sources,
            int64_t max_iterations, int nthreads,
            double* attrs_out, int* arity_out, int64_t* iterations_out, int* converged_out,
            int64_t* trace_units, int64_t* trace_changed, double* trace_max_stat,
            int64_t trace_cap) {
    const uint64_t V = g->V;
    const uint64_t* off = g->in_off;
    const uint32_t* isrc = g->in_src;
    const double* iw = g->in_w;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    int64_t cap;
    int arity = 1;
    uint32_t* src_dense = NULL;
    if (algo == GXO_SSSP) {
        if (sources && nsrc > 0) {
            if (nsrc > 64) return -3;
            arity = nsrc;
            src_dense = (uint32_t*)malloc(sizeof(uint32_t) * nsrc);
            for (int j = 0; j < nsrc; ++j) {
                uint64_t p = lower_bound_u32(g->ids, V, sources[j]);
                src_dense[j] = (p < V && g->ids[p] == sources[j]) ? (uint32_t)p : UINT32_MAX;
            }
        } else {
            /* sources = sorted(vertex_ids)[:4] (algorithms.py:219-222) */
            arity = V < 4 ? (int)V : 4;
            if (arity == 0) return -1; /* SsspBellmanFord raises on no sources (algorithms.py:91-92) */
            src_dense = (uint32_t*)malloc(sizeof(uint32_t) * arity);
            for (int j = 0; j < arity; ++j) src_dense[j] = (uint32_t)j;
        }
        cap = (int64_t)V + 1;
    } else if (algo == GXO_PAGERANK) {
        cap = 100;
    } else if (algo == GXO_LP) {
        cap = 15;
    } else if (algo == GXO_CC) {
        cap = (int64_t)V + 1;
    } else {
        return -2;
    }
    if (max_iterations >= 0) cap = max_iterations;
    if (arity_out) *arity_out = arity;

    uint8_t* active = (uint8_t*)calloc(V ? V : 1, 1);
    uint8_t* next_active = (uint8_t*)calloc(V ? V : 1, 1);
    int64_t it = 0;
    int converged = 0;

    if (algo == GXO_PAGERANK) {
        double* rank = (double*)malloc(sizeof(double) * (V ? V : 1));
        double* contrib = (double*)malloc(sizeof(double) * (V ? V : 1));
        double* newrank = (double*)malloc(sizeof(double) * (V ? V : 1));
        for (uint64_t v = 0; v < V; ++v) rank[v] = 1.0;          /* initial_attr (141-142) */
        for (; it < cap; ) {
            /* gen: rank / out_deg (147-149); every vertex is active (144-145) */
            #pragma omp parallel for schedule(static)
            for (int64_t v = 0; v < (int64_t)V; ++v)
                contrib[v] = g->outdeg[v] ? rank[v] / (double)g->outdeg[v] : 0.0;
            double max_stat = 0.0;
            int64_t changed = 0;
            #pragma omp parallel for schedule(dynamic, 1024) reduction(max:max_stat) reduction(+:changed)
            for (int64_t d = 0; d < (int64_t)V; ++d) {
                double s = 0.0;                                   /* merged.get(vid, 0.0) */
                for (uint64_t k = off[d]; k < off[d + 1]; ++k) s += contrib[isrc[k]];
                const double nr = 0.15 + 0.85 * s;                /* apply_one (157-159) */
                newrank[d] = nr;
                if (nr != rank[d]) {
                    const double st = fabs(nr - rank[d]);         /* convergence_stat (161-162) */
                    if (st > max_stat) max_stat = st;
                    changed++;
                }
            }
            double* t = rank; rank = newrank; newrank = t;
            record(it, trace_cap, trace_units, trace_changed, trace_max_stat, (int64_t)g->E, changed, max_stat);
            ++it;
            if (max_stat < 1e-9) { converged = 1; break; }        /* vote (164-165) */
        }
        for (uint64_t v = 0; v < V; ++v) attrs_out[v] = rank[v];
        free(rank); free(contrib); free(newrank);
    } else if (algo == GXO_SSSP) {
        const int K = arity;
        double* dist = (double*)malloc(sizeof(double) * (V ? V : 1) * K);
        double* ndist = (double*)malloc(sizeof(double) * (V ? V : 1) * K);
        for (uint64_t v = 0; v < V * (uint64_t)K; ++v) dist[v] = INFINITY;
        for (int j = 0; j < K; ++j)
            if (src_dense[j] != UINT32_MAX) { dist[(uint64_t)src_dense[j] * K + j] = 0.0; active[src_dense[j]] = 1; }
        memcpy(ndist, dist, sizeof(double) * V * K);
        for (; it < cap; ) {
            int64_t units = 0, changed = 0;
            #pragma omp parallel for schedule(static) reduction(+:units)
            for (int64_t v = 0; v < (int64_t)V; ++v) if (active[v]) units += g->outdeg[v];
            #pragma omp parallel for schedule(dynamic, 1024) reduction(+:changed)
            for (int64_t d = 0; d < (int64_t)V; ++d) {
                double m[64];
                int has = 0;
                const int kk = K;
                for (int j = 0; j < kk; ++j) m[j] = INFINITY;
                for (uint64_t k = off[d]; k < off[d + 1]; ++k) {
                    const uint32_t s = isrc[k];
                    if (!active[s]) continue;
                    has = 1;
                    for (int j = 0; j < kk; ++j) {               /* gen d + w (102-105), merge min (107-108) */
                        const double c = dist[(uint64_t)s * K + j] + (iw ? iw[k] : 1.0);
                        if (c < m[j]) m[j] = c;
                    }
                }
                next_active[d] = 0;
                if (!has) continue;
                int ch = 0;
                for (int j = 0; j < kk; ++j) {                   /* apply min (113-115) */
                    const double o = dist[(uint64_t)d * K + j];
                    const double n = m[j] < o ? m[j] : o;
                    ndist[(uint64_t)d * K + j] = n;
                    if (n != o) ch = 1;
                }
                next_active[d] = (uint8_t)ch;
                changed += ch;
            }
            #pragma omp parallel for schedule(static)
            for (int64_t d = 0; d < (int64_t)V; ++d)
                if (next_active[d]) memcpy(dist + (uint64_t)d * K, ndist + (uint64_t)d * K, sizeof(double) * K);
            uint8_t* t = active; active = next_active; next_active = t;
            record(it, trace_cap, trace_units, trace_changed, trace_max_stat, units, changed, changed ? 1.0 : 0.0);
            ++it;
            if (changed == 0) { converged = 1; break; }           /* vote: not next_active (70-72) */
        }
        memcpy(attrs_out, dist, sizeof(double) * V * K);
        free(dist); free(ndist);
    } else {
        /* LP (174-205) and CC: labels start at the vertex id */
        uint32_t* label = (uint32_t*)malloc(sizeof(uint32_t) * (V ? V : 1));
        uint32_t* nlabel = (uint32_t*)malloc(sizeof(uint32_t) * (V ? V : 1));
        for (uint64_t v = 0; v < V; ++v) { label[v] = g->ids[v]; active[v] = 1; }
        uint32_t maxdeg = 0;
        for (uint64_t v = 0; v < V; ++v) if (off[v + 1] - off[v] > maxdeg) maxdeg = (uint32_t)(off[v + 1] - off[v]);
        for (; it < cap; ) {
            int64_t units = 0, changed = 0;
            #pragma omp parallel for schedule(static) reduction(+:units)
            for (int64_t v = 0; v < (int64_t)V; ++v) if (active[v]) units += g->outdeg[v];
            #pragma omp parallel reduction(+:changed)
            {
                uint32_t* buf = (algo == GXO_LP) ? (uint32_t*)malloc(sizeof(uint32_t) * (maxdeg ? maxdeg : 1)) : NULL;
                #pragma omp for schedule(dynamic, 256)
                for (int64_t d = 0; d < (int64_t)V; ++d) {
                    uint64_t n = 0;
                    uint32_t mn = UINT32_MAX;
                    for (uint64_t k = off[d]; k < off[d + 1]; ++k) {
                        const uint32_t s = isrc[k];
                        if (!active[s]) continue;
                        if (algo == GXO_LP) buf[n] = label[s];
                        else if (label[s] < mn) mn = label[s];
                        n++;
                    }
                    nlabel[d] = label[d];
                    next_active[d] = 0;
                    if (n == 0) continue;                          /* no messages: keep, inactive (195-196) */
                    const uint32_t nl = (algo == GXO_LP) ? lp_mode(buf, n) : (mn < label[d] ? mn : label[d]);
                    if (nl != label[d]) { nlabel[d] = nl; next_active[d] = 1; changed++; }
                }
                free(buf);
            }
            uint32_t* t = label; label = nlabel; nlabel = t;
            uint8_t* ta = active; active = next_active; next_active = ta;
            record(it, trace_cap, trace_units, trace_changed, trace_max_stat, units, changed, changed ? 1.0 : 0.0);
            ++it;
            if (changed == 0) { converged = 1; break; }
        }
        for (uint64_t v = 0; v < V; ++v) attrs_out[v] = (double)label[v];
        free(label); free(nlabel);
    }
    free(active); free(next_active); free(src_dense);
    if (iterations_out) *iterations_out = it;
    if (converged_out) *converged_out = converged;
    return 0;
}

int gxo_rmat(uint32_t scale, uint32_t edge_factor, uint64_t seed, uint32_t a, uint32_t b,
             uint32_t c, uint32_t wmax, uint32_t scramble, uint32_t symmetric,
             uint32_t* src_out, uint32_t* dst_out, uint32_t* w_out) {
    if (scale < 1 || scale > 32) return -1;
    gxb_rmat_params p;
    p.scale = scale; p.edge_factor = edge_factor; p.seed = seed;
    p.a = a; p.b = b; p.c = c; p.wmax = wmax; p.scramble = scramble; p.symmetric = symmetric;
    const uint64_t m = (uint64_t)edge_factor << scale;
    const uint64_t sm = gxb_rmat_seedmix(seed), wm = gxb_rmat_wseedmix(seed);
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)m; ++i) {
        uint32_t s, d;
        gxb_rmat_edge(&p, sm, (uint64_t)i, &s, &d);
        src_out[i] = s; dst_out[i] = d;
        if (w_out) w_out[i] = gxb_rmat_weight(&p, wm, (uint64_t)i);
        if (symmetric) {
            src_out[m + i] = d; dst_out[m + i] = s;
            if (w_out) w_out[m + i] = w_out[i];
        }
    }
    return 0;
}
