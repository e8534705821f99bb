/*
 * gx_oracle.h — TEST INFRASTRUCTURE ONLY (the parity checker, never the
 * product path). Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so.
 *
 * A plain-C restatement of the reference's ground-truth loop
 * `run_reference` (`pkg/src/accelgraph/algorithms.py:298-342`) for the three
 * reference algorithms (`SsspBellmanFord` 81-122, `PageRank` 125-171,
 * `LabelPropagation` 174-205) plus the build-defined CC plug-in
 * (SURVEY.md Appendix A).
 *
 * Parity pin: tests/test_oracle_golden.py checks this file against golden
 * vectors produced by running the reference itself
 * (tests/golden/make_golden.py imports /root/reference/pkg/src).
 *
 * Exactness: the per-destination fold visits in-edges ordered by
 * (source id ascending, file order), which is exactly the order in which
 * `run_reference` emits messages for one target (`sorted(active)` then the
 * source's out-edges in file order, algorithms.py:320-324) and folds them
 * (`msg_merge`, algorithms.py:243-251). So PageRank sums are bit-identical to
 * the reference's, and SSSP/LP/CC are exact by construction. Parallelism is
 * over destinations only (OpenMP), which does not change any fold order.
 */
#ifndef GX_ORACLE_H
#define GX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { GXO_SSSP = 0, GXO_PAGERANK = 1, GXO_LP = 2, GXO_CC = 3 };

typedef struct gxo_graph gxo_graph;

/* Ingest an edge list (duplicates and self-loops kept, A/graph.py:131-166).
 * w may be NULL (every weight 1.0, A/graph.py:155). Vertex set = ids present
 * in any edge (A/graph.py:163-164). Returns NULL on allocation failure. */
gxo_graph* gxo_graph_new(uint64_t num_edges, const uint32_t* src, const uint32_t* dst,
                         const double* w);
void gxo_graph_free(gxo_graph* g);
uint64_t gxo_graph_num_vertices(const gxo_graph* g);
uint64_t gxo_graph_num_edges(const gxo_graph* g);
/* ascending present ids (length = num_vertices) */
void gxo_graph_ids(const gxo_graph* g, uint32_t* out);
/* out-degree per present id, in ascending-id order (A/graph.py:203-210) */
void gxo_graph_out_degree(const gxo_graph* g, uint32_t* out);

/* Run one algorithm like run_reference.
 *   sources: original ids (SSSP only); NULL/nsrc<=0 = the 4 lowest present ids
 *            (make_algorithm, algorithms.py:219-222)
 *   max_iterations < 0 = the algorithm's default cap (algorithms.py:117-119,
 *            167-168, 201-202; CC: |V|+1)
 *   nthreads <= 0 = OpenMP default
 *   attrs_out: num_vertices * arity doubles, ascending-id order
 *            (SSSP: one distance per source, +inf unreachable; PR: rank;
 *             LP/CC: label)
 *   trace_*: optional per-iteration records (length trace_cap):
 *            units = GEN work items (frontier out-edges, A/daemon.py:102),
 *            changed = vertices whose attribute changed,
 *            max_stat = convergence statistic (algorithms.py:335)
 * Returns 0 on success, negative on bad arguments. */
int gxo_run(const gxo_graph* g, int algo, int nsrc, const uint32_t* sources,
            int64_t max_iterations, int nthreads,
            double* attrs_out, int* arity_out, int64_t* iterations_out, int* converged_out,
            int64_t* trace_units, int64_t* trace_changed, double* trace_max_stat,
            int64_t trace_cap);

/* The shared R-MAT generator (include/gxb_rmat.h) on the host, OpenMP. */
int gxo_rmat(uint32_t scale, uint32_t edge_factor, uint64_t seed, uint32_t a, uint32_t b,
             uint32_t c, uint32_t wmax, uint32_t scramble, uint32_t symmetric,
             uint32_t* src_out, uint32_t* dst_out, uint32_t* w_out /* may be NULL */);

int gxo_max_threads(void);
/* OpenMP threads of every later call (torchrun exports OMP_NUM_THREADS=1 to its ranks) */
void gxo_set_threads(int n);

#ifdef __cplusplus
}
#endif

#endif
