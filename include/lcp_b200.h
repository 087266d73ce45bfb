/*
 * lcp_b200.h — C ABI of the B200-native LCP top-k retrieval library.
 *
 * This is the drop-in boundary for the hot path of arXiv 2602.04936's
 * reference package `lcpsearch` (/root/reference/pkg/src/lcpsearch).  The
 * reference has no FFI: its boundary is the Python API re-exported from
 * `src/__init__.py:21-24,44-79`.  Each entry point below names the reference
 * function it replaces (paths relative to pkg/src/lcpsearch/).  The Python
 * package `paper_2602_04936_b200` binds these symbols with ctypes and keeps
 * the reference's names, argument meanings and exception types.
 *
 * Conventions
 *  - Every function returns an lcp_status; it never throws across the ABI.
 *    On failure lcp_last_error() returns a thread-local message whose text
 *    matches the reference's exception message where one exists.
 *  - `stream` is a cudaStream_t passed as void* (NULL = the workspace's own
 *    stream for *_host calls, legacy default stream otherwise).
 *  - "_host" entry points take host pointers (pinned or pageable) and are
 *    synchronous: they include the host<->device copies.  The others take
 *    device pointers and are asynchronous on `stream`.
 *  - A built lcp_index is immutable; concurrent queries are safe as long as
 *    each thread uses its own lcp_workspace (reference: trie.py:19-20,
 *    SPEC.md:197-198 "queried concurrently without synchronization").
 *    A workspace's scratch (packed queries, unrequested matched_depth / aux
 *    outputs, full-scan lists) is shared by every call made with it, so
 *    calls in flight at the same time on different streams need different
 *    workspaces.
 */
#ifndef LCP_B200_H
#define LCP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LCP_ABI_VERSION 1

/* Status codes.  3/4 mirror the reference CLI exit codes for
 * InvalidInputError / InternalInvariantError (cli.py:55-58, 418-431). */
typedef enum lcp_status {
  LCP_OK = 0,
  LCP_ERR_INVALID_INPUT = 3, /* core.InvalidInputError  (core.py:29-30) */
  LCP_ERR_INTERNAL = 4,      /* core.InternalInvariantError (core.py:41-42) */
  LCP_ERR_CUDA = 5,          /* CUDA runtime failure (no reference counterpart) */
  LCP_ERR_STATE = 6          /* core.InvalidStateError (core.py:37-38) */
} lcp_status;

/* Query modes; numeric values equal trie.MODE_CODES (trie.py:49). */
typedef enum lcp_mode {
  LCP_MODE_STRICT = 0,
  LCP_MODE_COMPLETE = 1,
  LCP_MODE_TAL = 2
} lcp_mode;

typedef struct lcp_index lcp_index;
typedef struct lcp_workspace lcp_workspace;

typedef struct lcp_index_info {
  int64_t n;              /* items                                   */
  int32_t length;         /* L, symbols per item                     */
  int32_t sigma;          /* alphabet size                           */
  int32_t bits;           /* bits per packed symbol (power of two)   */
  int32_t syms_per_word;  /* 64 / bits                               */
  int32_t words;          /* u64 words per packed key                */
  int32_t search_levels;  /* levels of the k-ary search tree         */
  int32_t tal_depth;      /* TAL bucket depth d, -1 if none          */
  int32_t has_directory;  /* dense TAL directory present             */
  int64_t tal_buckets;    /* sigma**d (0 if no TAL structure)        */
  int64_t device_bytes;   /* bytes of device memory held by the index */
} lcp_index_info;

int lcp_abi_version(void);
const char* lcp_last_error(void);

/* ---- index build ---------------------------------------------------------
 * Replaces trie.build (trie.py:397-431): core.lexicographic_order
 * (core.py:162-174) + core.adjacent_lcp (core.py:177-184) + the per-depth
 * boundary tables; and, when tal_depth >= 0, the TalEngine constructor
 * (tal.py:42-82) for bucket depth tal_depth (directory when
 * sigma**d <= 2**24, tal.py:26).
 * rows: n*length uint16 row-major, host or device pointer.  Synchronous.
 * Errors: symbol >= sigma, length not in [1, 65535], sigma not in
 * [2, 65536], n >= 2**31  ->  LCP_ERR_INVALID_INPUT.                      */
int lcp_index_build(const uint16_t* rows, int64_t n, int32_t length, int32_t sigma,
                    int32_t tal_depth, lcp_index** out);
int lcp_index_free(lcp_index* index);
int lcp_index_get_info(const lcp_index* index, lcp_index_info* info);

/* Parity / introspection exports (host or device destination, synchronous).
 * order         : n int32   == TrieIndex.order (trie.py:425) / TalEngine.item_index
 * sorted_keys   : n*words u64 packed keys in sorted order
 * adjacent_lcp  : n-1 uint16 == core.adjacent_lcp(rows[order]) (core.py:177-184)
 * directory     : sigma**d + 1 int64 == TalEngine.directory (tal.py:76-82)
 * level_offset  : length+2 int64 == TrieIndex.level_offset (trie.py:405-421)
 * trie tables   : node_count int32 row_lo + uint16 edge_symbol (trie.py:409-419) */
int lcp_index_export_order(const lcp_index* index, int32_t* order);
int lcp_index_export_sorted_keys(const lcp_index* index, uint64_t* keys);
/* rows [first, first + count) of sorted_keys (e.g. a shard's first / last key) */
int lcp_index_export_sorted_key_range(const lcp_index* index, int64_t first, int64_t count,
                                      uint64_t* keys);
int lcp_index_export_adjacent_lcp(const lcp_index* index, uint16_t* adj);
int lcp_index_export_directory(const lcp_index* index, int64_t* directory);
int lcp_index_trie_level_offsets(const lcp_index* index, int64_t* level_offset);
int lcp_index_export_trie(const lcp_index* index, int32_t* row_lo, uint16_t* edge_symbol);
/* LCPI index snapshot (storage.index_snapshot_bytes, storage.py:155-210),
 * generated on the GPU and byte-identical to the reference.  Call with
 * out == NULL to get the size in *size; then with a buffer of *size bytes
 * (host or device).  Synchronous. */
int lcp_index_snapshot(const lcp_index* index, uint8_t* out, int64_t* size);
/* Load an LCPI snapshot (storage.index_from_snapshot_bytes,
 * storage.py:226-389): validates the stream (bad magic / version / widths,
 * truncation, level order, child ids, posting permutation, trailing bytes ->
 * LCP_ERR_INVALID_INPUT), recovers the rows, rebuilds on the GPU and checks
 * the rebuilt snapshot is byte-identical.  raw is a host buffer. */
int lcp_index_from_snapshot(const uint8_t* raw, int64_t size, lcp_index** out);
/* TalEngine.bucket_range_search (tal.py:124-136): binary search on the packed
 * d-prefixes, independent of the directory. q: `count` host queries; lo/hi host. */
int lcp_index_bucket_range_search(const lcp_index* index, const uint16_t* queries,
                                  int32_t count, int64_t* lo, int64_t* hi);

/* ---- workspace -------------------------------------------------------- */
int lcp_workspace_create(lcp_workspace** out);
int lcp_workspace_free(lcp_workspace* ws);
/* The workspace's own CUDA stream (cudaStream_t as void*). */
void* lcp_workspace_stream(lcp_workspace* ws);

/* ---- batched top-k query ------------------------------------------------
 * Replaces TrieIndex.query (trie.py:290-342) for mode strict/complete and
 * TalEngine.query (tal.py:155-194) for mode tal, over `count` queries.
 * queries      : count*length uint16
 * ids, lcps    : count*out_stride; row q holds hits[q] results ordered by
 *                (lcp desc, id asc).  out_stride >= min(k, n).
 * hits         : count int32
 * matched_depth: count uint16 (descent depth d_max; bucket depth for tal)
 * aux          : count*2 uint64 work counters, so the host can rebuild the
 *                reference WorkReport exactly (work.py:36-81):
 *                strict/complete: aux[2q] = d_max | (d_star << 32),
 *                                 aux[2q+1] = |R(d*)| | (first row of R(d*) << 32)
 *                                 (R(d*) = sorted rows sharing q's d*-prefix)
 *                tal            : aux[2q] = items_scanned,
 *                                 aux[2q+1] = symbols_compared
 * Errors: k < 1, bad mode, no TAL structure for tal, query symbol >= sigma. */
int lcp_query(const lcp_index* index, lcp_workspace* ws, const uint16_t* queries,
              int32_t count, int32_t k, int32_t mode, int32_t out_stride, uint32_t* ids,
              uint16_t* lcps, int32_t* hits, uint16_t* matched_depth, uint64_t* aux,
              void* stream);
int lcp_query_host(const lcp_index* index, lcp_workspace* ws, const uint16_t* queries,
                   int32_t count, int32_t k, int32_t mode, int32_t out_stride, uint32_t* ids,
                   uint16_t* lcps, int32_t* hits, uint16_t* matched_depth, uint64_t* aux);
/* Single-copy variant of lcp_query_host: every output lands in one host
 * block (ideally page-locked) with the byte layout lcp_packed_layout_for()
 * reports, so a batch costs one H2D and one D2H transfer. */
typedef struct lcp_packed_layout {
  int64_t ids, lcps, hits, matched_depth, aux; /* byte offsets */
  int64_t total;                               /* block size in bytes */
  int64_t err; /* byte offset of the int32 invalid-query flag (between hits and
                  matched_depth, so the LCP_PACKED_NO_WORK copy carries it) */
} lcp_packed_layout;
int lcp_packed_layout_for(int32_t count, int32_t out_stride, lcp_packed_layout* layout);
int lcp_query_host_packed(const lcp_index* index, lcp_workspace* ws, const uint16_t* queries,
                          int32_t count, int32_t k, int32_t mode, int32_t out_stride,
                          void* out_block);
/* Asynchronous lcp_query_host_packed: enqueues the H2D copy, the query kernel
 * and the single D2H copy on the workspace's stream and returns at once.  The
 * host buffers must stay untouched until lcp_workspace_wait(ws) returns.  At
 * most one batch in flight per workspace; use several workspaces to overlap
 * consecutive batches (transfers, kernels and host work run concurrently).
 * Batches of up to 1024 queries (LCP_DIRECT_IO_MAX) whose query rows and
 * output block both lie in lcp_pinned_alloc blocks skip the copies: the
 * kernel reads the rows from and writes the results into host memory
 * directly, which halves a small batch's round trip.  lcp_query_host_packed
 * is this call followed by lcp_workspace_wait. */
#define LCP_PACKED_NO_WORK 1 /* flags: skip matched_depth/aux in the D2H copy */
int lcp_query_host_packed_async(const lcp_index* index, lcp_workspace* ws,
                                const uint16_t* queries, int32_t count, int32_t k, int32_t mode,
                                int32_t out_stride, void* out_block, int32_t flags);
/* Wait for the workspace's in-flight batch; LCP_ERR_INVALID_INPUT if it had
 * a query symbol >= sigma.  A no-op when nothing is in flight. */
int lcp_workspace_wait(lcp_workspace* ws);
/* Device-side error flag raised by lcp_query (invalid query symbol); reading
 * it synchronises `stream`.  Returns LCP_OK or LCP_ERR_INVALID_INPUT and clears it. */
int lcp_workspace_check(lcp_workspace* ws, void* stream);

/* ---- brute-force full scan ----------------------------------------------
 * Replaces oracle.oracle_top_k (oracle.py:38-59): top-min(k,n) over every
 * item in original row order, (lcp desc, id asc).  Same buffers as lcp_query
 * minus matched_depth/aux. */
int lcp_fullscan(const lcp_index* index, lcp_workspace* ws, const uint16_t* queries,
                 int32_t count, int32_t k, int32_t out_stride, uint32_t* ids, uint16_t* lcps,
                 int32_t* hits, void* stream);
int lcp_fullscan_host(const lcp_index* index, lcp_workspace* ws, const uint16_t* queries,
                      int32_t count, int32_t k, int32_t out_stride, uint32_t* ids,
                      uint16_t* lcps, int32_t* hits);

/* ---- shard merge (multi-GPU; no reference counterpart) ------
 * encode: per-shard results -> candidates ((length-lcp) << 32 | (id+id_offset)),
 *         padded with UINT64_MAX: cand[count*k].
 * merge : cand[shards][count][k] -> global top-min(k, n_total) per query,
 *         optionally keeping only lcp == max lcp across shards (strict). */
int lcp_encode_candidates(const uint32_t* ids, const uint16_t* lcps, const int32_t* hits,
                          int32_t count, int32_t k, int32_t in_stride, int32_t length,
                          int64_t id_offset, uint64_t* cand, void* stream);
int lcp_merge_candidates(const uint64_t* cand, int32_t shards, int32_t count, int32_t k,
                         int32_t take, int32_t length, int32_t strict, uint32_t* ids,
                         uint16_t* lcps, int32_t* hits, void* stream);
/* (ids/lcps of lcp_merge_candidates have row stride max(1, take); take <= 32
 *  merges with one warp per query, larger take with one CTA per query for
 *  shards * k <= 8192.) */

/* ---- device-side routing for sharded query steps (no reference
 * counterpart; SURVEY §8e lexicographic range sharding).  Every entry point
 * is asynchronous on `stream` with device buffers and never synchronises the
 * host, so a whole sharded step can be captured in one CUDA graph.
 *
 * pack_queries : rows (count*length u16) -> packed keys (count*words u64),
 *                the index's key encoding (order-preserving).
 * route_queries: owner(q) = #splitters <= q (splitters: nsplit sorted packed
 *                keys, nsplit = world - 1), on `qkeys` (count*words packed
 *                keys) or, when qkeys is NULL, on the rows packed here.
 *                consult == 0: select the queries this `rank` owns and, when
 *                given, reset thresholds[q] = -1 and reset_cand[q*cand_k ..
 *                q*cand_k + cand_k) = UINT64_MAX for every q (the step's state).
 *                consult == 1: select the queries another rank owns for which
 *                this rank is nonempty and max(lcp(q, first[rank]),
 *                lcp(q, last[rank])) >= thresholds[q] (first/last: world packed
 *                keys).  Selected rows are written densely to out_rows
 *                (count*length u16 capacity), their batch positions to
 *                out_sel, their number to *d_count (device int; reset by the
 *                call).  Selection order within the dense batch is
 *                unspecified; results are scattered back by out_sel, so
 *                outputs are deterministic.
 * query_counted: lcp_query over `capacity` rows of which *d_count (device)
 *                are live; grids are sized for `expected` rows.
 * shard_thresholds: thresholds[sel[i]] = the lcp of hit need-1 (complete;
 *                -1 if fewer hits) or matched_depth (strict; -1 if none), for
 *                i < *d_count.
 * encode_candidates_sel: cand[sel[i]*k + j] = (length - lcp) << 32 |
 *                (gids ? gids[id] : id) + id_offset for j < hits[i], else
 *                UINT64_MAX, for i < *d_count (rows not selected untouched). */
int lcp_pack_queries(const lcp_index* index, lcp_workspace* ws, const uint16_t* rows, int32_t count,
                     uint64_t* keys, void* stream);
int lcp_route_queries(const lcp_index* index, lcp_workspace* ws, const uint16_t* queries,
                      const uint64_t* qkeys, int32_t count, const uint64_t* splitters,
                      int32_t nsplit, const uint64_t* first, const uint64_t* last,
                      const int32_t* nonempty, int32_t rank, int32_t* thresholds,
                      int32_t consult, uint16_t* out_rows, int32_t* out_sel, int32_t* d_count,
                      uint64_t* reset_cand, int32_t cand_k, void* stream);
int lcp_query_counted(const lcp_index* index, lcp_workspace* ws, const uint16_t* queries,
                      int32_t capacity, const int32_t* d_count, int32_t expected, int32_t k,
                      int32_t mode, int32_t out_stride, uint32_t* ids, uint16_t* lcps,
                      int32_t* hits, uint16_t* matched_depth, uint64_t* aux, void* stream);
int lcp_shard_thresholds(const uint16_t* lcps, const int32_t* hits, const uint16_t* matched_depth,
                         const int32_t* sel, const int32_t* d_count, int32_t capacity, int32_t stride,
                         int32_t need, int32_t strict, int32_t* thresholds, void* stream);
int lcp_encode_candidates_sel(const uint32_t* ids, const uint16_t* lcps, const int32_t* hits,
                              const int32_t* sel, const int32_t* d_count, int32_t capacity, int32_t k,
                              int32_t in_stride, int32_t length, const int64_t* gids,
                              int64_t id_offset, uint64_t* cand, void* stream);

/* Candidate exchange over NVLink peer memory (symmetric allocations mapped
 * into every rank; replaces the all-to-all + merge of a sharded step).
 * peer_signals / peer_cand: device arrays of `world` device pointers (rank
 * s's signal array of world u32 / candidate buffer of batch rows x k u64).
 * signal_peers : bump *epoch (device u32) and store it, behind a system fence,
 *                into slot [rank] of every peer's signal array.
 * merge_candidates_peers: wait until my_signals[s] >= *epoch for every s, then
 *                merge rows [rank*m, (rank+1)*m) of every peer's candidates
 *                (read over NVLink) into ids/lcps (row stride out_stride) and
 *                hits, like lcp_merge_candidates (take <= 32). */
int lcp_signal_peers(uint32_t* const* peer_signals, int32_t world, int32_t rank, uint32_t* epoch,
                     void* stream);
int lcp_merge_candidates_peers(const uint64_t* const* peer_cand, int32_t world, int32_t rank, int32_t m,
                               int32_t k, int32_t take, int32_t length, int32_t strict,
                               const uint32_t* my_signals, const uint32_t* epoch, uint32_t* ids,
                               uint16_t* lcps, int32_t* hits, int32_t out_stride, void* stream);

/* ---- single-query server (latency mode; the reference answers one query
 * per call, trie.py:290-342, and its GNC loop calls it back to back,
 * bench.py:353) ------------------------------------------------------------
 * One resident warp answers single queries through two mailboxes in
 * page-locked host memory (serve_kernels.cuh): lcp_server_query copies the
 * row at `query_row` into the request mailbox, the warp answers it with the
 * batch kernel's per-query code and sends the packed answer back in one
 * burst, and lcp_server_query unpacks it into `out_block`
 * (lcp_packed_layout_for(1, out_stride), work counters included): no launch,
 * copy or event per query.  `query_row` and `out_block` are ordinary host
 * memory.  W == 1, strict, complete or TAL, k <= 32 and out_stride <= 32
 * (else LCP_ERR_STATE: use the batch path).  lcp_server_query spins until
 * the answer is in; LCP_ERR_INVALID_INPUT for a symbol >= sigma.  The warp
 * exits after 100 ms without a request (so a device-wide synchronisation
 * never waits on it for long) and is relaunched on the next query.  One
 * server per thread; lcp_server_stop ends and frees it. */
typedef struct lcp_server lcp_server;
int lcp_server_start(const lcp_index* index, int32_t k, int32_t mode, int32_t out_stride,
                     const uint16_t* query_row, void* out_block, lcp_server** out);
int lcp_server_query(lcp_server* server);
/* lcp_server_query with the query read from `row` (L symbols) instead of the
 * row given at start. */
int lcp_server_query_row(lcp_server* server, const uint16_t* row);
int lcp_server_stop(lcp_server* server);

/* ---- host staging (no reference counterpart) -----------------------------
 * Page-locked, device-mapped host buffers (cudaHostAlloc): *_host calls DMA
 * directly, and small packed batches in them use direct host I/O. */
int lcp_pinned_alloc(int64_t bytes, void** out);
int lcp_pinned_free(void* p);
/* Synchronise a stream (cudaStream_t as void*). */
int lcp_stream_sync(void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LCP_B200_H */
