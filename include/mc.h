/* ===========================================================================
 * mc.h — C-ABI of the B200-native MetaCache-GPU hot path (libmc.so).
 *
 * The library implements the data-parallel hot path of MetaCache-GPU
 * (Kobus et al., arXiv 2106.08150; /root/reference/PAPER.md cited as P:<line>):
 *   build : encode -> window -> canonical k-mers -> h1 -> minhash sketch ->
 *           warp-aggregated insert into a multi-bucket hash table ->
 *           per-feature cap + condensed layout
 *   query : read (+ mate) sketch -> table probe -> gather -> sort ->
 *           window counts -> contiguous-range top hits -> partition merge ->
 *           hit threshold / LCA classification
 * Every step runs in hand-written sm_100a CUDA kernels; there is no CPU
 * fallback.  Readings of points the paper leaves open are listed in
 * DESIGN.md ("Readings", S1..S24).
 *
 * Conventions for every entry point
 *  - Return 0 (MC_OK) on success, a negative MC_ERR_* code otherwise; the
 *    message of the last failure on the calling thread is mc_last_error().
 *    No C++ exception crosses the ABI.
 *  - The caller owns every input and output buffer.  Sequence / read inputs
 *    and outputs may be HOST memory (pageable or pinned) or DEVICE memory on
 *    the handle's GPU; the library detects which (cudaPointerGetAttributes).
 *    Offsets arrays are always read as given (host or device).
 *  - Calls are synchronous: outputs are complete when the call returns.
 *  - Sequences are ASCII: A/C/G/T in either case are bases (A=0 C=1 G=2 T=3),
 *    every other byte is ambiguous and excludes the k-mers containing it
 *    (reading S3/S4).
 *  - A handle is used by one host thread at a time.
 * ======================================================================== */
#ifndef MC_H_
#define MC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MC_OK 0
#define MC_ERR_INVALID_ARG (-1) /* bad argument / config / duplicate id / unknown taxon */
#define MC_ERR_STATE (-2)       /* call not allowed in the handle's lifecycle state       */
#define MC_ERR_CAPACITY (-3)    /* static capacity exceeded (table, windows, read size)   */
#define MC_ERR_CUDA (-4)        /* CUDA runtime / kernel failure                          */
#define MC_ERR_OOM (-5)         /* device or pinned allocation failed                     */
#define MC_ERR_PEER (-6)        /* inter-GPU transport failed: peer access between two of a
                                   multi-GPU handle's devices unavailable, or a peer copy
                                   failed (the exchange runs over NVLink peer memory)      */
#define MC_ERR_NCCL MC_ERR_PEER /* SURVEY §8(b)'s name for the inter-GPU error class      */

typedef struct mc_db mc_db; /* opaque; owned by the library */


/* Sketching / classification parameters (P:699-705 defaults: k=16, s=16,
 * w=127 -> stride 112; cap 254 per feature and partition P:465-466;
 * m=4 candidates P:596-598).  Constraints checked by mc_db_create:
 *   1 <= k <= 16, 1 <= sketch_size <= 16, k <= window_len,
 *   stride = window_len-k+1 <= 128 (one warp covers a window),
 *   1 <= max_locations_per_feature <= 1023, 1 <= max_candidates <= 8,
 *   n_partitions >= 1, partition_begin + n_local_partitions <= n_partitions. */
typedef struct {
  uint32_t k;                         /* k-mer length                      (16)  */
  uint32_t sketch_size;               /* s, features per window            (16)  */
  uint32_t window_len;                /* w, window length in bases         (127) */
  uint32_t max_locations_per_feature; /* cap per (feature, partition)      (254) */
  uint32_t max_candidates;            /* m, top candidates per read        (4)   */
  uint32_t hits_min;                  /* classification hit threshold      (5)   */
  uint32_t hits_diff;                 /* near-tie distance for the LCA rule (4)  */
  uint32_t n_partitions;              /* P: total logical DB partitions    (1)   */
  uint32_t partition_begin;           /* first partition held by this handle (0) */
  uint32_t n_local_partitions;        /* partitions held here; 0 -> all P  (0)   */
  int32_t device;                     /* CUDA device ordinal; -1 -> current (-1) */
  uint32_t flags;                     /* reserved, must be 0                (0)   */
  uint64_t capacity_bp;               /* static allocation: max reference bp held
                                         by this handle       (2^30) */
  uint64_t max_targets;               /* static allocation: max targets; 0 -> auto */
  uint64_t read_batch;                /* read records per internal batch (2^20) */
  double table_slots_per_location;    /* build-table slots per location of capacity
                                         (1.25 -> load <= 0.8 in the worst case)   */
  uint32_t insert_size_max;           /* paired records: the window range of the
                                         contiguous-range top hits spans at least
                                         this many bases of the fragment (SURVEY
                                         §8(f) NEXT rank 1; reading S25):
                                         sws = 2 + max(|r1|+|r2|, insert_size_max)
                                         / stride for pairs; 0 -> S10 (0).
                                         Must be <= (1022 * stride).               */
  uint32_t reserved2;                 /* must be 0                           (0)   */
  /* Multi-GPU database (P:444-452 partitions by target; P:604-618 query chain;
   * P:673-679 per-GPU batch pipeline).  n_gpus = G > 1: ONE handle drives G
   * devices; it must hold every partition (n_local_partitions 0 or
   * n_partitions, partition_begin 0) and n_partitions % G == 0.  Shard g holds
   * partitions [g P/G, (g+1) P/G) on device devices[g] (-1 -> ordinal g).
   * Ordinals may repeat: several shards then share one GPU (the exchange
   * degenerates to same-device copies; results are identical).  G <= 1: one
   * device, `device` above.                                                  */
  uint32_t n_gpus;                    /* G, 0 or 1 -> single device       (1)   */
  int32_t devices[8];                 /* device of shard g; -1 -> g       (-1)  */
} mc_config;

/* Taxonomy: parent array over taxon ids 0..n_taxa-1.  Id 0 is invalid; a root
 * has parent[root] == root.  rank may be NULL.      */
typedef struct {
  uint32_t n_taxa;
  const uint32_t* parent;
  const uint8_t* rank;
} mc_taxonomy;

/* Final candidate (D8, Fig. 1): target id, hits in its best
 * contiguous window range, range [win_beg, win_end] (0-based window ids).
 * tgt == UINT32_MAX marks an empty slot (other fields 0).                  */
typedef struct {
  uint32_t tgt, hits, win_beg, win_end;
} mc_candidate;

/* Per-partition candidate with its taxon: the record exchanged between
 * ranks before mc_merge_classify.  Same empty convention.     */
typedef struct {
  uint32_t tgt, hits, win_beg, win_end, taxon, reserved;
} mc_hit;

/* Fill *cfg with the paper's defaults (values in parentheses above). */
void mc_config_init(mc_config* cfg);

/* Create a handle.  Validates cfg and the taxonomy (ids < n_taxa, no cycles,
 * depth <= 64), builds the lineage table on the device and
 * allocates every partition's static build table from capacity_bp
 * (P:650-652).  On failure *out is NULL.
 * Multi-GPU (n_gpus = G > 1): every shard gets its partitions' share of
 * capacity_bp / max_targets (+1/8 slack for the S9 imbalance), its own
 * lineage table and streams; peer access is enabled between every pair of
 * distinct devices (MC_ERR_PEER if the platform refuses it).               */
int mc_db_create(const mc_config* cfg, const mc_taxonomy* tax, mc_db** out);

/* Insert n reference targets (§5.2 build pipeline): every window
 * is sketched on the GPU and its (feature, location) pairs are appended to
 * the partition's region-partitioned pair store; the multi-value hash table
 * itself is filled by mc_db_finalize.
 *   seqs        ASCII bases, target i = seqs[offsets[i] .. offsets[i+1])
 *   offsets     uint64[n+1], non-decreasing
 *   target_ids  uint32[n], unique across all inserts, != UINT32_MAX
 *   taxa        uint32[n], each 1 <= taxon < n_taxa
 *   partition_ids  NULL -> the library assigns each target to the local
 *               partition with the fewest bp so far (reading S9, ties to the
 *               lowest index, state kept across calls); otherwise uint32[n]
 *               global partition ids that must lie in this handle's range.
 * Targets shorter than k are accepted and contribute no windows.
 * Every (feature, target, window) location is stored (no cap at this stage).
 * Errors: INVALID_ARG, STATE (after finalize), CAPACITY (static allocation
 * exceeded; the handle is then unusable except for destroy/clear).          */
int mc_db_insert_targets(mc_db* db, uint32_t n, const char* seqs, const uint64_t* offsets,
                         const uint32_t* target_ids, const uint32_t* taxa,
                         const uint32_t* partition_ids);

/* Several target batches in one call (same per-batch semantics as
 * mc_db_insert_targets, batches in order; S9 state carries across them).  On
 * a multi-GPU handle every device sketches its partitions' targets of all
 * batches concurrently with the others (targets are distributed
 * to the GPUs' partitions); a device-resident batch is best placed on the
 * device of its targets' partitions (others read it over NVLink).  Host
 * batches: each device copies only the byte runs holding its own targets
 * (runs split where more than 1 MiB of foreign bytes separate them).       */
typedef struct {
  uint32_t n;
  const char* seqs;
  const uint64_t* offsets;        /* [n+1] */
  const uint32_t* target_ids;     /* [n]   */
  const uint32_t* taxa;           /* [n]   */
  const uint32_t* partition_ids;  /* [n] or NULL (S9) */
} mc_target_batch;
int mc_db_insert_target_batches(mc_db* db, uint32_t n_batches, const mc_target_batch* batches);

/* Finalize: fill the multi-value hash
 * table with warp-aggregated inserts (one atomic per distinct key per warp),
 * lay every feature's locations out contiguously (the condensed layout: value
 * array + key -> (count, offset) table), and for a feature with more than
 * max_locations_per_feature locations in the partition keep the smallest by
 * (target id, window id) (reading S7).  Bucket order inside a feature is not
 * specified (dumps return it sorted).  STATE if already finalized; CAPACITY
 * if the table is full.                                                      */
int mc_db_finalize(mc_db* db);

/* Classify n_reads read records (Fig. 1).  Record i is
 * reads[read_offsets[i] .. read_offsets[i+1]) plus, if mates != NULL, its
 * mate mates[mate_offsets[i] .. mate_offsets[i+1]) (one taxon per pair).
 *   out_taxon       uint32[n_reads]; 0 = unclassified
 *   out_candidates  mc_candidate[n_reads * max_candidates] or NULL
 * Requires every partition in the handle, i.e. n_local_partitions ==
 * n_partitions (multi-process callers use mc_query_partials + exchange +
 * mc_merge_classify).  Multi-GPU handle: per batch of read_batch records,
 * device g copies record slice g (host input) and pulls the other slices
 * from its peers (all-gather over NVLink), every device scores all records
 * against its partitions, and device h merges + classifies slice h reading
 * the other devices' per-partition hits straight from their memory (the
 * exchange fused into the merge kernel); batches are double-buffered so the
 * copies of batch b+1 overlap the scoring of batch b.
 * Errors: STATE (not finalized), INVALID_ARG (offsets decrease), CAPACITY (a
 * record hits more than 16384 distinct 4-window blocks or has more than 64
 * windows in one partition, or spans more than the 1022-window range limit),
 * PEER (multi-GPU transport).                                                */
int mc_classify(mc_db* db, uint64_t n_reads, const char* reads, const uint64_t* read_offsets,
                const char* mates, const uint64_t* mate_offsets, uint32_t* out_taxon,
                mc_candidate* out_candidates);

/* Multi-rank query half 1: top-m candidates of every record in
 * each LOCAL partition.  out_hits: mc_hit[n_reads * n_local * m], record-
 * major (record r, local partition q, rank i at [(r*n_local + q)*m + i]).
 * On a multi-GPU handle n_local = n_partitions (every shard's lists).       */
int mc_query_partials(mc_db* db, uint64_t n_reads, const char* reads, const uint64_t* read_offsets,
                      const char* mates, const uint64_t* mate_offsets, mc_hit* out_hits);

/* Multi-rank query half 2 (reading S12/S13): merge n_lists
 * per-partition lists per record into the global top-m (hits desc, target
 * asc) and classify (hits_min / hits_diff / LCA).
 *   hits: mc_hit[n_reads * n_lists * m] laid out as mc_query_partials'.     */
int mc_merge_classify(mc_db* db, uint64_t n_reads, uint32_t n_lists, const mc_hit* hits,
                      uint32_t* out_taxon, mc_candidate* out_candidates);

/* Release the handle and all device memory.  NULL is a no-op. */
void mc_db_destroy(mc_db* db);

/* Back to the freshly created state (no targets), keeping all allocations. */
int mc_db_clear(mc_db* db);

/* Launch all work of this handle on the given cudaStream_t (NULL -> the
 * library's own stream).  Lets callers time the path with CUDA events.
 * Single-device handles only (STATE on a multi-GPU handle).               */
int mc_db_set_stream(mc_db* db, void* cuda_stream);

/* Message of the last failed call on this thread ("" if none). */
const char* mc_last_error(void);

/* ---- diagnostics (test / bench support; not part of the method) -------- */

/* Deterministic partition plan used when partition_ids == NULL (S9):
 * target i -> argmin_q running_bp[q] (ties lowest q); running_bp[P] in/out. */
int mc_plan_partitions(uint32_t P, uint32_t n, const uint64_t* lengths, uint64_t* running_bp,
                       uint32_t* out_part);

/* Sketch every window of n sequences on the GPU (build-side kernel path).
 *   out_window_offsets uint64[n+1]: first window of sequence i (host)
 *   out_features       uint32[total_windows * sketch_size], row padded with 0
 *   out_counts         uint32[total_windows]
 * Call with out_features == NULL to obtain out_window_offsets only.         */
int mc_debug_sketch(const mc_config* cfg, uint32_t n, const char* seqs, const uint64_t* offsets,
                    uint32_t* out_features, uint32_t* out_counts, uint64_t* out_window_offsets);

/* Global partition that holds target_id (INVALID_ARG if unknown here). */
int mc_db_partition_of(const mc_db* db, uint32_t target_id, uint32_t* out_partition);

/* Sorted, capped location list ((tgt<<32)|window) of one feature in one
 * global partition held by this handle (after finalize).  Writes at most
 * cap entries; *out_n = full list length.                                   */
int mc_db_feature_locations(const mc_db* db, uint32_t partition, uint32_t feature, uint64_t* out,
                            uint32_t cap, uint32_t* out_n);

/* Dump one finalized partition in ascending key order: keys[n_keys],
 * counts[n_keys], values[n_values] ((tgt<<32)|window, grouped by key).
 * Pass NULL arrays to query *n_keys / *n_values only.                        */
int mc_db_dump_partition(const mc_db* db, uint32_t partition, uint32_t* keys, uint32_t* counts,
                         uint64_t* values, uint64_t* n_keys, uint64_t* n_values);

/* JSON statistics: counts (bp, windows, locations, keys, values, truncated,
 * table slots/bytes), kernel launch counts and per-stage device times
 * (CUDA events) accumulated since create / the last mc_db_reset_stats.
 * Writes a NUL-terminated string; INVALID_ARG if buf_len is too small.     */
int mc_db_stats(const mc_db* db, char* out_json, uint64_t buf_len);
int mc_db_reset_stats(mc_db* db);

/* Condensed database dump / load (the paper writes
 * database.meta + one cache file per partition and reloads a condensed
 * layout, Fig. 2, §4.2; its on-the-fly mode skips this,
 * P:307-313).  mc_db_save writes a FINALIZED handle's
 * configuration, taxonomy and, per local partition, the target metadata,
 * the condensed key table (the used slot prefix), the sub-region value
 * bases, the value array and the ranked-target tables to one file at
 * `path` (host byte order; overwritten).  mc_db_load creates a handle on
 * `device` (-1: current) from such a file -- the same static allocation as
 * mc_db_create with the saved configuration -- and leaves it FINALIZED:
 * queries on it give the saved handle's results bit for bit.
 * Errors: STATE (save before finalize), INVALID_ARG (NULL, bad or truncated
 * file), CUDA / OOM as elsewhere.  The caller owns the path string.        */
int mc_db_save(const mc_db* db, const char* path);   /* single-device handles (STATE otherwise) */
int mc_db_load(const char* path, int32_t device, mc_db** out);
/* The handle's configuration (as created or loaded) -> *out. */
int mc_db_get_config(const mc_db* db, mc_config* out);

#ifdef __cplusplus
}
#endif
#endif /* MC_H_ */
