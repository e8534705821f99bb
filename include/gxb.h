/*
 * gxb.h — C ABI of libgxb200.so, the B200-native daemon for GX-Plug's
 * per-iteration graph compute path (MSGGen -> MSGMerge -> MSGApply plus the
 * per-iteration mirror exchange).
 *
 * Every entry point returns an int status: GXB_OK (0) or a negative GXB_E*
 * code; gxb_last_error() returns a thread-local message for the last failure.
 * Plain pointers and sizes only. Streams are passed as `void*` (a
 * cudaStream_t; NULL = the legacy default stream). Calls on one gxb_ctx must be
 * serialised by the caller — the role the agent<->daemon region queue plays in
 * the reference (`A/channel.py:74-130`).
 *
 * Reference interfaces replaced (A/ = pkg/src/accelgraph/):
 *   gxb_init / gxb_shutdown / gxb_init_count ..... Daemon.initialize / shutdown /
 *                                                   init_count (A/daemon.py:133-168),
 *                                                   daemon_init (A/daemon.py:207-212)
 *   gxb_graph_build .............................. partition_graph (A/graph.py:175-212)
 *                                                   + Agent._remote_dsts (A/agent.py:156-166)
 *   gxb_graph_get_info / gxb_graph_ids ............... PartitionedGraph.num_vertices /
 *                                                   vertex_ids / out_degree (A/graph.py:109-128)
 *   gxb_state_create ............................. make_algorithm + initial_attr /
 *                                                   initially_active (A/algorithms.py:208-229,
 *                                                   96-100, 141-145, 179-183)
 *   gxb_request(GXB_OP_GEN|MERGE|APPLY) .......... execute_request (A/daemon.py:86-130) over a
 *                                                   WorkItem range descriptor; Agent.request
 *                                                   (A/agent.py:234-276)
 *   gxb_iterate .................................. one BSP iteration Gen∘Merge∘Apply
 *                                                   (A/agent.py:469-498, A/algorithms.py:318-341)
 *   gxb_stats .................................... round_closed / vote inputs, max_stat,
 *                                                   next frontier (A/agent.py:404-417, 533-540)
 *   gxb_exchange_* ............................... sync round gqq/gdq + skip
 *                                                   (A/engine.py:242-266, A/sync.py:163-208,
 *                                                   A/agent.py:542-592)
 *   gxb_read_attrs ............................... dump of Engine.store / run_reference attrs
 *                                                   (A/engine.py:370, 430-433)
 */
#ifndef GXB_H
#define GXB_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes */
#define GXB_OK            0
#define GXB_EINVAL       -22   /* bad argument (Python: ValueError) */
#define GXB_EPROTO       -71   /* protocol violation, e.g. re-init (Python: ProtocolError) */
#define GXB_ENOMEM       -12   /* device allocation failed (Python: MemoryError) */
#define GXB_ECUDA        -5    /* CUDA runtime error (Python: RuntimeError) */
#define GXB_ERANGE       -34   /* value outside the device representation (Python: ValueError) */
#define GXB_ENOTOWNED    -66   /* apply target not owned by this partition (Python: ValueError) */
#define GXB_ESTATE       -77   /* call out of order for the current phase (Python: ProtocolError) */

/* algorithms (A/algorithms.py:81-205; CC per SURVEY.md Appendix A) */
#define GXB_ALGO_SSSP      0
#define GXB_ALGO_PAGERANK  1
#define GXB_ALGO_LP        2
#define GXB_ALGO_CC        3

/* template operations (A/channel.py:25-28) */
#define GXB_OP_GEN    0
#define GXB_OP_MERGE  1
#define GXB_OP_APPLY  2

/* gxb_graph_build flags */
#define GXB_BUILD_HOST_INPUT   0x1u  /* src/dst/w are host pointers (else device pointers) */
#define GXB_BUILD_NO_CSR       0x2u  /* skip the push-mode CSR (PR/LP never push) */
#define GXB_BUILD_ID_RANGES    0x4u  /* partitions = contiguous ascending-id ranges of even
                                        vertex counts, as partition_graph(even_sizes) does
                                        (A/graph.py:169-212); default = ranges balanced by
                                        in-edges over the degree-sorted order */
#define GXB_BUILD_RANGES       0x8u  /* contiguous degree-sorted ranges balanced by in-edge
                                        cost instead of the default round-robin deal of the
                                        degree-sorted order (nparts > 1) */

/* gxb_iterate direction policy */
#define GXB_DIR_AUTO  0
#define GXB_DIR_PULL  1
#define GXB_DIR_PUSH  2

typedef struct gxb_ctx gxb_ctx;
typedef struct gxb_graph gxb_graph;
typedef struct gxb_state gxb_state;

typedef struct gxb_graph_info {
    uint64_t num_vertices;     /* present ids (A/graph.py:163-164) */
    uint64_t num_edges;        /* all edges of the graph (duplicates, self-loops kept) */
    uint64_t owned_lo;         /* owned slot range [owned_lo, owned_hi) in device order */
    uint64_t owned_hi;
    uint64_t owned_edges;      /* in-edges of the owned destinations (CSC slice) */
    uint64_t owned_out_edges;  /* out-edges of owned sources (push CSR slice), 0 if not built */
    uint32_t max_id;           /* largest present original id */
    uint32_t max_in_degree;
    int32_t  part;             /* partition index / world size */
    int32_t  nparts;
    int32_t  weighted;
    int32_t  has_csr;
    uint64_t num_slots;        /* device slot space: num_vertices, or padded to equal
                                  partition blocks (dealt layout); value buffers are
                                  num_slots long */
} gxb_graph_info;

typedef struct gxb_iter_stats {
    uint64_t iteration;        /* apply rounds completed */
    uint64_t changed;          /* owned vertices whose attribute changed (A/agent.py:406-409) */
    uint64_t next_active;      /* owned vertices active next iteration (A/agent.py:416) */
    uint64_t next_units;       /* out-edges of the next frontier = next GEN units (A/daemon.py:102) */
    uint64_t units;            /* GEN units processed in the last iteration */
    uint64_t targets;          /* vertices that received >= 1 message (|merged|, A/algorithms.py:327) */
    uint64_t remote_active;    /* next-active vertices with a cross-partition consumer (A/agent.py:533-535) */
    double   max_stat;         /* max convergence_stat over changed vertices (A/algorithms.py:335) */
    int32_t  voted;            /* local convergence vote (A/algorithms.py:70-72, 164-165) */
    int32_t  direction;        /* GXB_DIR_PULL / GXB_DIR_PUSH used by the last iteration */
} gxb_iter_stats;

typedef struct gxb_rmat_args {
    uint32_t scale, edge_factor;
    uint64_t seed;
    uint32_t a, b, c;          /* quadrant thresholds * 2^32 (include/gxb_rmat.h) */
    uint32_t wmax, scramble, symmetric;
} gxb_rmat_args;

/* ---- errors / lifecycle (A/daemon.py:133-212) ---- */
const char* gxb_last_error(void);
const char* gxb_version(void);
int gxb_init(int device, gxb_ctx** out);            /* Daemon.initialize: exactly once */
int gxb_reinit(gxb_ctx* ctx);                       /* always GXB_EPROTO (A/daemon.py:150-154) */
int gxb_init_count(const gxb_ctx* ctx, int* out);
int gxb_shutdown(gxb_ctx* ctx);                     /* idempotent (A/daemon.py:163-168) */

/* ---- tuning knobs (process-wide): "tile_minblocks" (0/4/6/8), "l2_hot_mb", "l1_hot_kb",
 * "push_alpha" (push when frontier out-edges * alpha < |E|), "pull_dense_div" (SSSP/CC
 * pull gathers every source, no active-bitmap test, when frontier out-edges * div >= |E|;
 * 0 = always test), "pull_kernel" (0 = edge-balanced warp tiles, 1 = degree-binned groups),
 * "carveout", "exchange_chunks", "overlap_reserve_sms", "pr_message_bits" (64 / 32) ---- */
int gxb_set_option(const char* name, int64_t value);
int gxb_get_option(const char* name, int64_t* value);

/* ---- device R-MAT ingest ---- */
/* Fills device arrays src/dst[/w] (num = gxb_rmat_num_edges) on `stream`. */
int gxb_rmat_generate(gxb_ctx* ctx, const gxb_rmat_args* args, uint32_t* d_src,
                      uint32_t* d_dst, uint32_t* d_w, void* stream);

/* ---- graph store (A/graph.py:175-212) ----
 * Builds the device store from E edges (src[i] -> dst[i], weight w[i] or 1).
 * Default partitioning for nparts > 1: the in-degree-sorted order is dealt
 * round-robin (each partition gets every nparts-th vertex, hence the same share of
 * hubs and of the tail) and each partition's share is one contiguous slot range.
 * Weights are non-negative integers (u32); the float64 reference weights are
 * accepted by the Python layer only when integral.
 * nparts/part: destination-range partition (part in [0, nparts)); every rank
 * passes the SAME full edge list and receives the in-edges of its own
 * destination range, balanced by in-edge count (Lemma 2 with equal c_j,
 * A/balancer.py:79-98). nparts = 1 for a single GPU. */
int gxb_graph_build(gxb_ctx* ctx, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                    uint64_t num_edges, int part, int nparts, uint32_t flags, void* stream,
                    gxb_graph** out);
/* as gxb_graph_build with explicit per-partition vertex counts over ascending ids
 * (the `sizes` argument of partition_graph, A/graph.py:175-191); sum must equal the
 * number of present ids, else GXB_EINVAL */
int gxb_graph_build_sized(gxb_ctx* ctx, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                          uint64_t num_edges, int part, int nparts, const uint64_t* sizes, uint32_t flags,
                          void* stream, gxb_graph** out);
/* heterogeneous devices: contiguous degree-sorted ranges (GXB_BUILD_RANGES) whose in-edge
 * cost is split in proportion to per-partition capacity factors (units per unit time =
 * 1 / unit_cost): the data-resizing planner balance_data (A/balancer.py:79-98) applied to
 * the graph's cost line; every factor must be > 0 and finite, else GXB_EINVAL; combining
 * with GXB_BUILD_ID_RANGES is GXB_EINVAL */
int gxb_graph_build_balanced(gxb_ctx* ctx, const uint32_t* src, const uint32_t* dst, const uint32_t* w,
                             uint64_t num_edges, int part, int nparts, const double* capacity, uint32_t flags,
                             void* stream, gxb_graph** out);
int gxb_graph_get_info(const gxb_graph* g, gxb_graph_info* out);
/* ascending present ids (host buffer of num_vertices) */
int gxb_graph_ids(const gxb_graph* g, uint32_t* host_out);
/* global out-degree per present id in ascending-id order (host, num_vertices) */
int gxb_graph_out_degree(const gxb_graph* g, uint32_t* host_out);
/* partition boundaries in device slot order (host, nparts+1) */
int gxb_graph_part_bounds(const gxb_graph* g, uint64_t* host_out);
/* owned present ids of this partition in ascending order (host, *count entries; host_out
 * may be NULL to query the count) */
int gxb_graph_owned_ids(gxb_graph* g, uint32_t* host_out, uint64_t* count);
int gxb_graph_free(gxb_graph* g);

/* ---- algorithm state ---- */
/* sources: original ids for SSSP (NULL/nsrc=0 = 4 lowest present ids,
 * A/algorithms.py:219-222), at most 4. */
int gxb_state_create(gxb_graph* g, int algo, const uint32_t* sources, int nsrc,
                     gxb_state** out);
int gxb_state_free(gxb_state* s);
int gxb_state_arity(const gxb_state* s, int* out);

/* One fused BSP iteration over the owned partition: Gen∘Merge∘Apply in one
 * pull pass (or push over the CSR for sparse SSSP/CC frontiers). Leaves the
 * stats on the device; gxb_stats() synchronises `stream` and reads them. */
int gxb_iterate(gxb_state* s, int direction, void* stream);

/* Split rounds (option split_overlap, SSSP / CC at N > 1): launch the NEXT round's
 * local-source pass (in-edges from this partition's own slots) on an internal stream
 * ordered after `stream`, so it runs while the closed round's records travel to and from
 * the peers (SURVEY.md §8(e) overlap; the reference's sync round A/engine.py:247-266 sits
 * between two rounds the same way). The next gxb_iterate, if it is a tile pull, gathers
 * only the remote sources and combines. A no-op unless the last round was a dense pull;
 * *launched (optional) = 1 when the pass was launched. */
int gxb_iterate_local(gxb_state* s, void* stream, int* launched);

/* API-faithful template ops over a WorkItem range descriptor (A/daemon.py:86-130):
 *   GEN:   [lo, hi) = owned CSC edge range; materialises one message per edge
 *          whose source is active (A/algorithms.py:232-240)
 *   MERGE: [lo, hi) = owned destination slots; folds each slot's messages
 *          (A/algorithms.py:243-263)
 *   APPLY: [lo, hi) = owned destination slots; applies, detects changes, builds
 *          the next frontier (A/algorithms.py:266-295). Targets outside the owned
 *          range fail with GXB_ENOTOWNED (A/daemon.py:121-122).
 * After all APPLY ranges of an iteration, gxb_commit() closes the round. */
int gxb_request(gxb_state* s, int op, uint64_t lo, uint64_t hi, void* stream);
int gxb_commit(gxb_state* s, void* stream);

int gxb_stats(gxb_state* s, void* stream, gxb_iter_stats* out);
/* the last closed round's vote block written on the device, no host synchronisation:
 * d_out[0..5] = changed, next_active, next_units, remote_active, records packed by
 * gxb_exchange_pack_async (else 0), max_stat (doubles) —
 * what the sync round all-gathers (A/engine.py:267-285) */
int gxb_stats_device(gxb_state* s, double* d_out, void* stream);
/* PageRank back-to-back rounds: in async mode a round leaves its statistics on the device
 * (read them with gxb_stats_device), so the host can launch round k+1 before it has read
 * round k's vote; rank and contributions are double-buffered, so a round launched after
 * the converged one is undone exactly by gxb_round_rollback (A/algorithms.py:318-341:
 * the reference stops at the first converged round) */
int gxb_stats_async(gxb_state* s, int on);  /* gxb_stats keeps reporting the last synchronous round */
int gxb_round_rollback(gxb_state* s);

/* ---- mirror exchange (A/engine.py:242-266) ----
 * Multi-partition runs keep a full-length replica of every source value. After
 * an iteration each rank publishes its changed owned values; the caller moves
 * the bytes with NCCL (torch.distributed) between these device buffers:
 *   dense (PR): the owned slice of the value replica is all-gathered in place;
 *   delta (SSSP/CC/LP): gxb_exchange_pack writes (slot, value) records of
 *     changed owned vertices; gxb_exchange_unpack installs received records
 *     into the replica and marks them active for the next iteration. */
int gxb_exchange_buffer(gxb_state* s, int which, void** dev_ptr, uint64_t* bytes);

/* fused PageRank exchange over peer memory: every rank exports the IPC handles of its
 * two contribution buffers (which = 0 / 1), opens its peers' handles, and from then on
 * the Apply kernel stores each new contribution of an owned vertex into every peer's
 * replica over NVLink / NVSwitch — no separate all-gather (the reference's gqq/gdq
 * mirror shuffle, A/engine.py:248-285, fused into MSGApply). All ranks must iterate in
 * lockstep (the round's vote collective orders the stores before the next gather).
 * set_peer_ptrs takes device pointers directly (same-process peers). */
#define GXB_IPC_HANDLE_BYTES 64
int gxb_exchange_ipc_handle(gxb_state* s, int which, void* handle_out);
int gxb_exchange_open_peers(gxb_state* s, int npeers, const void* handles);   /* npeers x 2 handles */
int gxb_exchange_set_peer_ptrs(gxb_state* s, int npeers, void* const* ptrs);  /* npeers x 2 pointers */
int gxb_exchange_close_peers(gxb_state* s);
int gxb_exchange_pack(gxb_state* s, void* stream, uint64_t* count_out);
int gxb_exchange_unpack(gxb_state* s, const void* d_records, uint64_t count, void* stream);
/* asynchronous delta exchange (no host synchronisation): pack_async writes the records into
 * GXB_BUF_SEND and leaves their count for the vote block (gxb_stats_device, entry 4); after
 * a padded all-gather of nblocks blocks of block_records records, unpack_regions installs
 * counts[q] records of block q (the caller passes 0 for its own block); frontier_after /
 * units_after are the next frontier's length and GEN units when the caller knows them from
 * the vote (own changed + received records; the sum of every rank's next_units) */
int gxb_exchange_pack_async(gxb_state* s, void* stream);
int gxb_exchange_unpack_regions(gxb_state* s, const void* d_records, const uint64_t* counts, int nblocks,
                                uint64_t block_records, uint64_t frontier_after, uint64_t units_after,
                                void* stream);  /* *_after = ~0: read back from the device */
int gxb_exchange_finish(gxb_state* s, void* stream);
#define GXB_BUF_VALUES      0   /* the value replica (contributions / distances / labels) */
#define GXB_BUF_SEND        1   /* packed (slot, value) records of this rank */
#define GXB_BUF_RECV        2   /* receive area for peers' records */
#define GXB_BUF_RECORD_SIZE 3   /* bytes per record in *bytes */
#define GXB_BUF_VALUES_NEXT 4   /* PageRank: the contribution array the open round writes */
#define GXB_BUF_SPARSE_SEND 5   /* PageRank needed-only exchange: my values, grouped by peer */
#define GXB_BUF_SPARSE_RECV 6   /* PageRank needed-only exchange: peers' values, grouped by peer */
#define GXB_BUF_CONTRIB0    7   /* PageRank: contribution buffer 0 (absolute, not rotating) */
#define GXB_BUF_CONTRIB1    8   /* PageRank: contribution buffer 1 */

/* Needed-only dense exchange (PageRank, nparts > 1): peer q receives exactly my owned
 * slots that are sources of edges into q's destinations (static lists built with the
 * graph, sorted by slot on both sides). pack: values -> GXB_BUF_SPARSE_SEND grouped by
 * peer (send_counts); the caller runs an all-to-all into GXB_BUF_SPARSE_RECV
 * (recv_counts); unpack scatters them into the replica. */
int gxb_exchange_sparse_counts(const gxb_state* s, uint64_t* send_counts, uint64_t* recv_counts);

/* per-peer delta exchange over peer memory (SSSP / CC / LP, 2..8 partitions): the lazy
 * upload of "dirty and queried" values (A/agent.py:550-582, A/sync.py:171-198) with the
 * query set static — a changed owned value goes only to the peers whose CSC reads it.
 *   arena:  cap_matrix[p * nparts + q] = records partition p may send to q (= p's
 *           gxb_exchange_sparse_counts send_counts[q], all-gathered by the caller; this
 *           partition's row must match its own lists). Allocates this partition's receive
 *           arena (two round-parity blocks per sender) and its need mask; writes the arena's
 *           IPC handle when ipc_handle_out != NULL.
 *   open:   nparts IPC handles (this partition's own entry ignored) -> peers' arenas;
 *   set_peers: same-process peers' arenas (gxb_exchange_delta_buffer), nparts pointers.
 *   pack:   after a closed round, stores every changed owned value into the arena of each
 *           peer that reads it (NVLink / NVSwitch stores, fenced system-wide) and writes the
 *           per-receiver record counts into d_vote[6 + q] (doubles) — the vote collective
 *           that follows orders the stores before any peer reads them.
 *   unpack: counts_from[p] = records partition p packed for this one (from the vote);
 *           installs them, marks them active and appends them to the frontier.
 * Round parities alternate, so a sender never overwrites a block its receiver has not
 * unpacked (the receiver unpacks round k before it joins vote k + 1). */
int gxb_exchange_delta_arena(gxb_state* s, const uint64_t* cap_matrix, void* ipc_handle_out);
int gxb_exchange_delta_open(gxb_state* s, const void* handles);
int gxb_exchange_delta_set_peers(gxb_state* s, void* const* arenas);
int gxb_exchange_delta_buffer(gxb_state* s, void** arena);
int gxb_exchange_delta_close(gxb_state* s);
int gxb_exchange_delta_pack(gxb_state* s, double* d_vote, void* stream);
int gxb_exchange_delta_unpack(gxb_state* s, const uint64_t* counts_from, void* stream);

/* dense mirror exchange for the rounds where most vertices changed (SSSP / CC / LP): the
 * caller all-gathers every owner's block of GXB_BUF_VALUES_NEXT in place (equal blocks:
 * the dealt partitioning), then dense_install installs every mirror whose landed value
 * differs from its current one (it changed in its owner's round), marks it active and
 * appends it to the frontier — coalesced passes instead of per-record scatter. */
int gxb_exchange_dense_install(gxb_state* s, void* stream);
int gxb_exchange_sparse_pack(gxb_state* s, void* stream);
int gxb_exchange_sparse_unpack(gxb_state* s, void* stream);

/* ---- pipeline shuffle (Alg. 1-2 realised as stream overlap) ----
 * A PageRank pull round split into K exchange chunks of the owned slots (chunk k =
 * relative slots [b[k], b[k+1]), b from gxb_graph_xchunks; every rank cuts its block
 * with b[k] = owned * k^2 / K^2, so chunk 0 holds the hubs). After gxb_iterate_chunk(k)
 * the chunk's new contributions (GXB_BUF_VALUES_NEXT) are final and can be sent while
 * later chunks compute; gxb_iterate_end closes the round (stats, buffer rotation).
 * Equivalent to gxb_iterate when all chunks are run. */
int gxb_graph_xchunks(const gxb_graph* g, int* K, uint64_t* host_bounds);
int gxb_iterate_begin(gxb_state* s, void* stream);
int gxb_iterate_chunk(gxb_state* s, int k, void* stream);
int gxb_iterate_end(gxb_state* s, void* stream);

/* attributes in ascending original-id order (host buffer num_vertices * arity;
 * SSSP: float64 distances, +inf unreachable; PR: float64 rank; LP/CC: float64 label).
 * Only owned vertices are meaningful on a partitioned run (owned_only = 1
 * writes NaN elsewhere). */
int gxb_read_attrs(gxb_state* s, double* host_out, int owned_only, void* stream);

/* install attribute values from the host (ascending original-id order, same
 * encoding as gxb_read_attrs) — the agent's update("pull_from_upper")
 * (A/agent.py:224-232, 433-443). Does not change the active frontier.
 * SSSP distances / labels must be non-negative integers < 2^32-1 (+inf allowed
 * for distances), else GXB_ERANGE. */
int gxb_write_attrs(gxb_state* s, const double* host_in, void* stream);

/* the sync round's deliver from host values (Agent.deliver, A/agent.py:584-592; the
 * values come from the upper system's gdq, A/engine.py:255-266): install n mirror values
 * (vertices owned by OTHER partitions, given as dense indices = rank of the id among the
 * present ids, same value encoding as gxb_read_attrs) into this partition's source
 * replica. SSSP / CC / LP: the delivered vertices become active sources of the next
 * round (changed set = next frontier), exactly like received exchange records.
 * An owned or absent target is GXB_EINVAL; a non-representable value GXB_ERANGE. */
int gxb_attrs_deliver(gxb_state* s, const uint64_t* host_dense, const double* host_vals, uint64_t n,
                      void* stream);

/* asynchronous staging for a pipelined agent loop (no host synchronisation; the
 * caller orders the copy and compute streams with events): h2d copies pinned host
 * attributes into staging buffer `buf` (0/1), install scatters them into the state,
 * extract gathers the state into output buffer `buf`, d2h copies it to pinned host
 * memory. install does not validate values (use gxb_write_attrs for checked input). */
int gxb_attrs_h2d(gxb_state* s, const double* host_in, int buf, void* stream);
/* staging scope: 0 = every present vertex (default), 1 = this partition's owned vertices
 * only, ascending id order (gxb_graph_owned_ids) — the agent of one partition moves only
 * its own vertices (A/agent.py:224-232, 433-443) */
int gxb_attrs_scope(gxb_state* s, int owned_only);
int gxb_attrs_install(gxb_state* s, int buf, void* stream);
int gxb_attrs_extract(gxb_state* s, int buf, void* stream);
int gxb_attrs_d2h(gxb_state* s, double* host_out, int buf, void* stream);

/* ---- profiling: CUDA events around the main merge kernel of every fused
 * iteration, and a count of every kernel the library launched ---- */
typedef struct gxb_profile {
    double   main_kernel_ms;       /* summed device time of the main merge kernel */
    uint64_t main_kernel_launches;
    uint64_t kernels_launched;     /* all kernels launched by gxb_iterate since the last reset */
    uint64_t iterations;
    double   rest_ms;              /* device time of the round after the main kernel (apply, folds, commit) */
} gxb_profile;
int gxb_profile_enable(gxb_state* s, int on);
int gxb_profile_read(gxb_state* s, gxb_profile* out, int reset);

#ifdef __cplusplus
}
#endif

#endif /* GXB_H */
