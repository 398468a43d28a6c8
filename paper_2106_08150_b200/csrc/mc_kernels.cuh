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

void launch_sketch_insert(const BuildBatch& b, SketchCfg c, Slot* T, uint64_t nslots,
                          unsigned long long* n_locations, int* err, int grid, cudaStream_t st);
// region-partitioned insert: regions of 2^shift slots (>= 2^20 slots = 32 MiB
// of table; larger for huge tables so that nreg <= 2048)
struct PartitionArgs {
  uint2* pairs;                 // [nreg * rcap] (key, value) buckets, one per region
  unsigned long long* cursor;   // [nreg] bucket fill (zeroed)
  unsigned long long* work;     // insert work counter (zeroed)
  int* overflow;                // set if a bucket overflows
  uint64_t rcap;                // bucket capacity (pairs)
  uint64_t nslots;
  uint32_t nreg, shift;
};
size_t sketch_partition_smem(uint32_t nreg);
void launch_sketch_partition(const BuildBatch& b, SketchCfg c, const PartitionArgs& pa, int grid, cudaStream_t st);
void launch_insert_pairs(const PartitionArgs& pa, Slot* T, uint64_t nslots, int* err, int grid, cudaStream_t st);
void launch_debug_sketch(const BuildBatch& b, SketchCfg c, uint32_t* feats, uint32_t* counts, int grid,
                         cudaStream_t st);

// finalize
struct FinalizeArgs {
  Slot* T;  // primaries of finalized keys become the condensed key table: v[0] = count, v[1..2] = offset
  uint64_t nslots;
  uint32_t cap;
  uint32_t* cnt;               // [nslots] full location count, accumulated at each primary (zeroed)
  uint32_t* spos;              // [nslots] position of a slot's first value inside its key's list
  uint64_t* off;               // [nslots] exclusive scan of min(cnt, cap)
  const uint32_t* ins_base;    // [nt] gapped window base of each target (insertion order, ascending)
  const uint32_t* delta;       // [nt] ranked - gapped window index for each target
  uint32_t nt;
  bool identity;               // targets were inserted in id order: ranked == gapped
  uint32_t* values;            // condensed values (ranked window ids)
  uint64_t* heavy;             // primaries of keys with more than cap locations
  uint64_t* sortq;             // segments 2 <= n <= cap to sort: offset | n << 48
  unsigned long long* counters;  // [0] keys [1] locations [2] truncated [3] heavy [4] sortq
  int* err;
};
constexpr uint32_t kLight = 16;
void launch_fin_count(const FinalizeArgs& a, int grid, cudaStream_t st);
void launch_fin_scatter(const FinalizeArgs& a, int grid, cudaStream_t st);
void launch_fin_sort_light(const FinalizeArgs& a, int grid, cudaStream_t st);
void launch_fin_sort_warp(const FinalizeArgs& a, int grid, cudaStream_t st);
void launch_fin_heavy(const FinalizeArgs& a, int grid, cudaStream_t st);

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
  const Slot* T;  // finalized table: a key's first slot in probe order holds (count, offset)
  uint64_t nslots;
  const uint32_t* values;
  const uint32_t* rank_base;  // [nt+1]
  const uint32_t* tgt_id;     // [nt] by rank
  const uint32_t* taxon;      // [nt] by rank
  uint32_t nt;
};

struct HitRec {  // == mc_hit
  uint32_t tgt, hits, win_beg, win_end, taxon, reserved;
};

struct QueryArgs {
  ReadBatch rb;
  PartView pv;
  SketchCfg c;
  uint32_t m;
  HitRec* out;      // [n * n_lists * m]
  uint32_t n_lists, list;
  uint32_t* qM;     // deferred to the medium bin
  uint32_t* qL;     // deferred to the large bin
  unsigned int* qcount;  // [0] medium [1] large
  int* err;         // 1: record exceeds the large bin; err[1] = record index
  unsigned long long* stats;  // [0] features with a non-empty list, [1] locations gathered
};

// per-record window-count hash capacity H (uniques <= 3H/4), windows and
// gathered locations per record
constexpr uint32_t kSmallH = 256, kSmallW = 4, kSmallL = 1024;   // warp per record
constexpr uint32_t kMedH = 2048, kMedW = 16, kMedL = 16384;      // 128-thread CTA per record
constexpr uint32_t kLargeH = 16384, kLargeW = 64;    // 512-thread CTA per record

void launch_query_small(const QueryArgs& a, int grid, cudaStream_t st);
void launch_query_medium(const QueryArgs& a, int grid, cudaStream_t st);
void launch_query_large(const QueryArgs& a, int grid, cudaStream_t st);
void query_kernels_init();

struct MergeArgs {
  const HitRec* in;  // [n * n_lists * m]
  uint64_t n;
  uint32_t n_lists, m;
  uint32_t hits_min, hits_diff;
  const uint32_t* anc;    // lineage table [n_taxa * (maxd+1)]
  const uint32_t* depth;  // [n_taxa]
  uint32_t maxd, n_taxa;
  uint32_t* out_taxon;
  uint32_t* out_cand;     // mc_candidate [n * m] as 4 x u32
};
void launch_merge_classify(const MergeArgs& a, cudaStream_t st);

int num_sms();

}  // namespace mc
