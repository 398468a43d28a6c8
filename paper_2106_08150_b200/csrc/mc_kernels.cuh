// Kernel-launch interface shared by the CUDA translation units of libmc.so
// (build_kernels.cu, query_kernels.cu, runtime.cu).  Internal to the library.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "mc_device.cuh"

namespace mc {

// Gap (in window ids) between consecutive targets in the ranked window-index
// space, so that "same target and within sws windows" is a single integer
// comparison.  Requires sws <= kRankGap (checked on the host).
constexpr uint32_t kRankGap = 1024;

// ---- build -------------------------------------------------------------------
struct BuildBatch {
  const uint8_t* chars;      // device bytes
  const uint64_t* win_base;  // [nt+1] cumulative window counts in this batch
  const uint64_t* seq_off;   // [nt] byte offset of each target in chars
  const uint64_t* seq_len;   // [nt]
  const uint32_t* bwi_base;  // [nt] build window index of each target's window 0
  uint32_t nt;
  uint64_t total_windows;
};

void launch_debug_sketch(const BuildBatch& b, SketchCfg c, uint32_t* feats, uint32_t* counts, int grid,
                         cudaStream_t st);

// ---- region-partitioned pair store ------------------------------------------
// Insert calls only sketch and append (key, value) pairs to per-region
// buckets (region = home slot >> shift of the table); finalize fills the
// table region by region so that the active table lines stay in L2.
struct PairStore {
  uint2* pairs;                 // [nreg * rcap + spill_cap] (feature, gapped window index)
  unsigned long long* cursor;   // [nreg + 2]: region fills, [nreg] spill fill, [nreg + 1] work counter
  uint64_t rcap, spill_cap;     // bucket capacity per region, spill capacity
  uint64_t nslots;              // table slots (the home-slot range)
  uint32_t nreg, shift;
  int* err;                     // [0] table full, [1] spill overflow
  uint32_t* hll;                // [kHllRegs] HyperLogLog registers of the distinct features
};
constexpr uint32_t kHllBits = 10, kHllRegs = 1u << kHllBits;
// the HyperLogLog sees a 1 / 2^kHllSampleBits sample of the hash space (the
// features whose next kHllSampleBits hash bits are 0); the estimate is scaled
// back at finalize.  (Saves the per-pair register update on most pairs.)
constexpr uint32_t kHllSampleBits = 4;
size_t sketch_partition_smem(uint32_t nreg);
void launch_sketch_partition(const BuildBatch& b, SketchCfg c, const PairStore& ps, int sms, cudaStream_t st);

// ---- finalize ----------------------------------------------------------------
// The table is cut into SUB-REGIONS of kSubSlots slots; linear probing wraps
// inside a key's sub-region, so one CTA can build a sub-region entirely in
// shared memory.  The pair store (by region) is first regrouped by sub-region.
struct FinalizeArgs {
  PairStore ps;
  KSlot* T;
  unsigned long long* vbase;   // [nsub] first value of each sub-region (slot offsets are relative)
  uint64_t nslots;             // slots in use: a multiple of kSubSlots
  uint32_t cap;
  const uint4* gcoarse;        // per 1024 gapped window ids: (delta of the target at the block start,
                               // first gapped id of the next target if it starts in the block else ~0,
                               // delta of that next target, 0); delta = ranked - gapped window index
  bool identity;               // targets were inserted in id order: ranked == gapped
  uint32_t* values;            // condensed values: per key min(count, cap) ranked window ids
  uint32_t* side;              // keys with count > cap: all their values before selection
  ulonglong2* heavy;           // keys with count > cap: (side fill cursor, final offset | count << 40)
  unsigned long long* counters;  // [0] keys [1] locations [2] truncated [3] heavy keys [4] values
                                 // [5] side cursor [6] sub-region ticket
  uint2* sorted;               // the pairs regrouped by sub-region
  uint32_t* subcnt;            // [nsub] pairs per sub-region, then regroup cursors
  uint64_t* subbase;           // [nsub + 1] first pair of each sub-region in `sorted`
  uint64_t nsub;
};
uint32_t split_bins(const FinalizeArgs& a);
void launch_sub_count(const FinalizeArgs& a, int sms, cudaStream_t st);
void launch_sub_scatter(const FinalizeArgs& a, int sms, cudaStream_t st);
void launch_sub_finalize(const FinalizeArgs& a, int sms, cudaStream_t st);
void launch_heavy_select(const FinalizeArgs& a, int grid, cudaStream_t st);

// exclusive scan of min(in, clamp): uint32 -> uint64 (total in *total_dev)
uint64_t scan_scratch_bytes(uint64_t n);
void launch_exclusive_scan(const uint32_t* in, uint64_t* out, uint64_t n, uint32_t clamp, void* scratch,
                           uint64_t* total_dev, cudaStream_t st, int* launches);

// ---- query ---------------------------------------------------------------------
struct ReadBatch {
  const uint8_t* r1;
  const uint64_t* o1;  // [n+1] absolute offsets into r1 (minus base1)
  uint64_t base1;
  const uint8_t* r2;   // nullable
  const uint64_t* o2;
  uint64_t base2;
  uint64_t n;
};

struct PartView {
  const KSlot* T;  // finalized table: key -> (count, sub-region-relative offset)
  const unsigned long long* vbase;  // [nslots >> kSubLg] first value of each sub-region
  uint64_t nslots;
  const uint32_t* values;
  const uint32_t* rank_base;  // [nt+1]
  const uint32_t* tgt_id;     // [nt] by rank
  const uint32_t* taxon;      // [nt] by rank
  uint32_t nt;
  const uint2* coarse;        // [(rank_base[nt] >> 10) + 1] per 1024 ranked windows: (target rank at the
                              // block start, first window of the next target if it starts in the block)
};

// target rank of ranked window id b: one 8-byte lookup (targets are >= kRankGap
// apart, so a 1024-window block holds at most one target start)
__device__ __forceinline__ uint32_t target_of(const PartView& pv, uint32_t b) {
  const uint2 c = pv.coarse[b >> 10];
  return b >= c.y ? c.x + 1 : c.x;
}

struct HitRec {  // == mc_hit
  uint32_t tgt, hits, win_beg, win_end, taxon, reserved;
};

struct QueryArgs {
  ReadBatch rb;
  PartView pv;
  SketchCfg c;
  uint32_t m;
  uint32_t insert_size_max;  // pairs: sws from max(|r1| + |r2|, insert_size_max) (S25; 0 = S10)
  HitRec* out;      // [n * n_lists * m]
  uint32_t n_lists, list;
  uint32_t* qM;     // deferred to the medium bin
  uint32_t* qL;     // deferred to the large bin
  unsigned int* qcount;  // [0] medium [1] large
  int* err;         // [0] 1: record exceeds the large bin, [1] its index; [2] bad input kind, [3] its record
  unsigned long long* stats;  // [0] features probed, [1] locations gathered, [2] read bp, [3..5] locations per
                              // bin, [6] records deferred to medium, [7] to large, [8] probes that found a
                              // (non-empty) list
  const uint64_t* wbase;      // [n+1] first window of each record (exclusive scan of windows)
  const uint64_t* qfeat;      // [windows * s] probe result: bucket offset << 24 | list length
};

// Q1: per-record window counts + input checks; Q2-Q3: sketch + probe of
// every window of the batch (one thread per window)
void launch_query_plan(const QueryArgs& a, uint32_t* nwt, uint64_t lim_bp, cudaStream_t st);
void launch_query_sketch_probe(const QueryArgs& a, uint64_t n_windows, uint64_t* qfeat, int sms, cudaStream_t st);

// per-record window-count hash capacity H (uniques <= 3H/4), windows and
// gathered locations per record
#ifndef MC_SMALL_H
#define MC_SMALL_H 512
#endif
#ifndef MC_SMALL_L
#define MC_SMALL_L 4096
#endif
#ifndef MC_MED_T
#define MC_MED_T 128
#endif
constexpr uint32_t kSmallH = MC_SMALL_H, kSmallW = 4, kSmallL = MC_SMALL_L;   // warp per record
constexpr uint32_t kMedH = 2048, kMedW = 16, kMedL = 16384, kMedT = MC_MED_T;  // CTA per record
constexpr uint32_t kLargeH = 16384, kLargeW = 64;    // 512-thread CTA per record

void launch_query_small(const QueryArgs& a, int grid, cudaStream_t st);
void launch_query_medium(const QueryArgs& a, int grid, cudaStream_t st);
void launch_query_large(const QueryArgs& a, int grid, cudaStream_t st);
void query_kernels_init();
void launch_key_lookup(const PartView& pv, uint32_t key, unsigned long long* out, cudaStream_t st);

constexpr uint32_t kMaxGpus = 8;
struct MergeArgs {
  const HitRec* in;  // [n * n_lists * m]  (n_src == 0)
  uint64_t n;
  uint32_t n_lists, m;
  uint32_t hits_min, hits_diff;
  const uint32_t* anc;    // lineage table [n_taxa * (maxd+1)]
  const uint32_t* depth;  // [n_taxa]
  uint32_t maxd, n_taxa;
  uint32_t* out_taxon;
  uint32_t* out_cand;     // mc_candidate [n * m] as 4 x u32
  const int* err = nullptr;  // the batch's status words: err[2] != 0 -> invalid input, nothing to merge
  // multi-GPU exchange fused into the merge (n_src > 0): the lists of record r
  // are read straight from the n_src devices' hit buffers (peer memory over
  // NVLink): source g holds lists_per_src lists of every record of the batch,
  // record R at src[g] + R * lists_per_src * m; this launch merges records
  // R = r0 .. r0 + n - 1 (n_lists = n_src * lists_per_src)
  const HitRec* src[kMaxGpus] = {};
  uint32_t n_src = 0, lists_per_src = 0;
  uint64_t r0 = 0;
};
void launch_merge_classify(const MergeArgs& a, cudaStream_t st);

int num_sms();

}  // namespace mc
