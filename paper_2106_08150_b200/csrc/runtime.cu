// Host runtime of libmc.so: the C-ABI declared in include/mc.h.
//
// Owns the per-partition static allocations, the target
// registry, partition assignment (S9), the stream and per-stage CUDA-event
// timers, and drives the kernels of build_kernels.cu / query_kernels.cu.
// All method arithmetic runs on the device; the host only validates,
// plans (window counts, target ranking) and moves bytes.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <numeric>
#include <string>
#include <new>
#include <stdexcept>
#include <thread>
#include <unordered_map>
#include <vector>

#include "mc.h"
#include "mc_kernels.cuh"

using namespace mc;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(x)                                                                                              \
  do {                                                                                                     \
    cudaError_t e_ = (x);                                                                                  \
    if (e_ != cudaSuccess) {                                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? MC_ERR_OOM : MC_ERR_CUDA, "%s:%d %s: %s", __FILE__, \
                  __LINE__, #x, cudaGetErrorString(e_));                                                   \
    }                                                                                                      \
  } while (0)

#define TRY(x)              \
  do {                      \
    int rc_ = (x);          \
    if (rc_ != MC_OK) return rc_; \
  } while (0)

// MC_TRACE=1: host wall time of each phase of an insert / finalize call, so
// host work between kernels (GPU idle) is visible (stderr, one JSON line per call)
struct HostPhases {
  using clk = std::chrono::steady_clock;
  const char* call;
  bool on;
  clk::time_point t0, last;
  std::string out;
  HostPhases* prev;
  static HostPhases*& cur() {
    static thread_local HostPhases* p = nullptr;
    return p;
  }
  explicit HostPhases(const char* c) : call(c), on(getenv("MC_TRACE") != nullptr), prev(cur()) {
    t0 = last = clk::now();
    cur() = this;
  }
  void mark(const char* what) {
    if (!on) return;
    const auto t = clk::now();
    char b[96];
    snprintf(b, sizeof b, ", \"%s\": %.3f", what, std::chrono::duration<double, std::milli>(t - last).count());
    out += b;
    last = t;
  }
  ~HostPhases() {
    cur() = prev;
    if (on)
      fprintf(stderr, "{\"mc_host_ms\": {\"call\": \"%s\"%s, \"total\": %.3f}}\n", call, out.c_str(),
              std::chrono::duration<double, std::milli>(clk::now() - t0).count());
  }
};
static void phase(const char* what) {
  if (HostPhases* p = HostPhases::cur()) p->mark(what);
}

// no C++ exception (a failed host allocation, std::bad_alloc) ever crosses
// the ABI (mc.h conventions): host-heavy entry points run through this
template <class F>
static int no_throw(F&& f) {
  try {
    return f();
  } catch (const std::bad_alloc&) {
    return fail(MC_ERR_OOM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(MC_ERR_INVALID_ARG, "internal error: %s", e.what());
  } catch (...) {
    return fail(MC_ERR_INVALID_ARG, "internal error");
  }
}


template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;  // capacity in elements
  int ensure(size_t cnt) {
    if (cnt <= n && p) return MC_OK;
    release();
    size_t bytes = std::max<size_t>(cnt, 1) * sizeof(T);
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      n = 0;
      return fail(MC_ERR_OOM, "cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
    }
    n = std::max<size_t>(cnt, 1);
    return MC_OK;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// device ordinal holding p, -1 for host memory (pageable, pinned or unknown)
int ptr_device(const void* p) {
  if (!p) return -1;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) ? at.device : -1;
}

template <class T>
int to_host(const T* p, size_t n, std::vector<T>& out) {
  out.resize(n);
  if (n == 0) return MC_OK;
  if (is_device_ptr(p)) {
    CK(cudaMemcpy(out.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost));
  } else {
    std::memcpy(out.data(), p, n * sizeof(T));
  }
  return MC_OK;
}

// A caller array readable on the host: the caller's own memory when it is
// host memory (no copy), else a host copy of the device array.
template <class T>
struct HostView {
  const T* p = nullptr;
  std::vector<T> copy;
  int load(const T* src, size_t n) {
    if (src && is_device_ptr(src)) {
      TRY(to_host(src, n, copy));
      p = copy.data();
    } else {
      p = src;
    }
    return MC_OK;
  }
  const T& operator[](size_t i) const { return p[i]; }
  const T* data() const { return p; }
};

uint64_t n_windows_host(uint64_t L, uint32_t k, uint32_t stride) {
  return L < k ? 0 : (L - k + stride) / stride;
}

int validate_cfg(const mc_config* c) {
  if (!c) return fail(MC_ERR_INVALID_ARG, "config is NULL");
  if (c->k < 1 || c->k > 16) return fail(MC_ERR_INVALID_ARG, "k=%u outside [1,16]", c->k);
  if (c->sketch_size < 1 || c->sketch_size > 16)
    return fail(MC_ERR_INVALID_ARG, "sketch_size=%u outside [1,16]", c->sketch_size);
  if (c->window_len < c->k) return fail(MC_ERR_INVALID_ARG, "window_len=%u < k=%u", c->window_len, c->k);
  if (c->window_len - c->k + 1 > 128)
    return fail(MC_ERR_INVALID_ARG, "window stride w-k+1=%u > 128", c->window_len - c->k + 1);
  return MC_OK;
}

// ---- per-stage device timers (CUDA events on the handle's stream) -----------
struct Pending {
  std::string name;
  cudaEvent_t a, b;
};

}  // namespace

struct Part {
  uint32_t gid = 0;
  KSlot* T = nullptr;  // multi-value hash table: key -> (count, bucket offset)
  uint64_t nslots = 0, cap_windows = 0, cap_targets = 0;
  // region-partitioned pair store (filled by inserts, consumed by finalize)
  DevBuf<uint2> pairs;
  DevBuf<unsigned long long> cursor, cursor_bak;  // (bak: rollback copy of an insert call)
  DevBuf<uint32_t> hll, hll_bak;
  uint64_t rcap = 0, spill_cap = 0, nslots_max = 0;  // nslots = slots in use after finalize
  uint32_t nreg = 0, shift = 20;
  std::vector<uint32_t> tid, taxon;
  std::vector<uint64_t> nwin;
  std::vector<uint32_t> gbase;  // gapped window base of each target (insertion order)
  uint64_t windows = 0, bp = 0, gwin = 0;  // gwin = windows + kRankGap * targets
  // finalized state

  DevBuf<uint32_t> values;
  DevBuf<unsigned long long> vbase;  // first value of each table sub-region
  uint64_t n_value_slots = 0;  // extent of `values` (>= n_values: truncated keys leave gaps)
  uint64_t n_values = 0, n_keys = 0, n_locations = 0, truncated = 0;
  DevBuf<uint32_t> rank_base, tgt_id, taxon_rank;
  DevBuf<uint2> coarse;
  std::vector<uint32_t> rank_base_h, tgt_by_rank_h;
};

// Target id -> (local partition, index) registry: open addressing, linear
// probing, power-of-two capacity at load <= 0.5.  UINT32_MAX (a reserved id)
// marks empty slots.  A std::unordered_map cost ~30 ms of host time per build
// (insert + duplicate check + clear) at 2.4e5 targets (AFS31-shaped shard).
struct IdMap {
  std::vector<uint32_t> key;
  std::vector<std::pair<uint32_t, uint32_t>> val;
  size_t n = 0;
  size_t slot(uint32_t id) const {
    const size_t mask = key.size() - 1;
    size_t h = (size_t)(((uint64_t)id * 0x9E3779B97F4A7C15ull) >> 32) & mask;
    while (key[h] != id && key[h] != 0xffffffffu) h = (h + 1) & mask;
    return h;
  }
  void reserve(size_t m) {
    if ((n + m) * 2 <= key.size()) return;
    size_t cap = 1024;
    while (cap < (n + m) * 2) cap <<= 1;
    std::vector<uint32_t> ok(std::move(key));
    std::vector<std::pair<uint32_t, uint32_t>> ov(std::move(val));
    key.assign(cap, 0xffffffffu);
    val.resize(cap);
    for (size_t i = 0; i < ok.size(); ++i)
      if (ok[i] != 0xffffffffu) {
        const size_t h = slot(ok[i]);
        key[h] = ok[i];
        val[h] = ov[i];
      }
  }
  // (UINT32_MAX is the empty marker and never a stored id: it is never found)
  size_t count(uint32_t id) const { return id != 0xffffffffu && !key.empty() && key[slot(id)] == id; }
  const std::pair<uint32_t, uint32_t>* find(uint32_t id) const {
    if (key.empty() || id == 0xffffffffu) return nullptr;
    const size_t h = slot(id);
    return key[h] == id ? &val[h] : nullptr;
  }
  bool put(uint32_t id, uint32_t a, uint32_t b) {  // false: id already present (or the reserved UINT32_MAX)
    if (id == 0xffffffffu) return false;
    reserve(1);
    const size_t h = slot(id);
    if (key[h] == id) return false;
    key[h] = id;
    val[h] = {a, b};
    ++n;
    return true;
  }
  void clear() {
    key.clear();
    val.clear();
    n = 0;
  }
};

struct mc_db {
  mc_config cfg{};
  SketchCfg sc{};
  int device = 0;
  cudaStream_t own = nullptr, stream = nullptr;
  uint32_t pbegin = 0, n_local = 1;
  uint32_t n_taxa = 0, maxd = 0;
  DevBuf<uint32_t> anc, depth;
  std::vector<uint32_t> parent_h;  // the taxonomy as given (kept for mc_db_save)
  std::vector<uint8_t> rank_h;     // (empty: no ranks given)
  std::vector<Part> parts;
  IdMap where;
  std::vector<uint64_t> running_bp;
  int state = 0;  // 0 building, 1 finalized, -1 broken
  // scratch
  DevBuf<uint8_t> chars, rbuf1, rbuf2, scan_scratch, stage[2];
  cudaStream_t copy_stream = nullptr;
  // staging slots (3: a query's copy of batch b+2 proceeds while batches b, b+1 compute)
  cudaEvent_t stage_ready[3] = {nullptr, nullptr, nullptr}, stage_free[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t qstat_ev[3] = {nullptr, nullptr, nullptr};  // a query batch's status copy is complete
  // results go back on their own stream (PCIe is full duplex: the D2H of batch b
  // overlaps the H2D of batch b+1 and the compute of batch b+1); double-buffered
  cudaStream_t d2h_stream = nullptr;
  cudaEvent_t out_ready[2] = {nullptr, nullptr}, out_free[2] = {nullptr, nullptr};
  DevBuf<uint32_t> otx[2], ocd[2];
  DevBuf<HitRec> ohits[2];
  DevBuf<unsigned long long> cursor;
  DevBuf<uint2> pairs;
  DevBuf<uint64_t> meta64, roff1, roff2, heavy, total, wbase, qfeat, subbase;
  DevBuf<uint2> sorted;
  DevBuf<uint32_t> meta32, side, qM, qL, otaxon, ocand, nwt, subcnt;
  DevBuf<uint4> gcoarse;  // finalize: gapped -> ranked window ids
  DevBuf<unsigned long long> counters, qstats;
  DevBuf<unsigned int> qcount;
  DevBuf<int> err;
  int* herr_pin = nullptr;  // pinned copy of err (per-batch status, read without stalling the pipeline)
  uint8_t* pin = nullptr;   // pinned host staging for host-built tables (async uploads)
  size_t pin_cap = 0;
  int ensure_pin(size_t bytes) {
    if (bytes <= pin_cap) return MC_OK;
    if (pin) {
      cudaStreamSynchronize(stream);  // (an upload from the old buffer may be in flight)
      cudaFreeHost(pin);
    }
    pin = nullptr;
    pin_cap = 0;
    const size_t cap = std::max<size_t>(bytes + bytes / 4, 1 << 20);
    if (cudaMallocHost(&pin, cap) != cudaSuccess) {
      cudaGetLastError();
      pin = nullptr;
      return fail(MC_ERR_OOM, "pinned staging of %zu bytes failed", cap);
    }
    pin_cap = cap;
    return MC_OK;
  }
  DevBuf<uint8_t> qbuf1[3], qbuf2[3];  // host-read staging slots (query)
  DevBuf<uint64_t> qoff1[3], qoff2[3];
  DevBuf<HitRec> hits;
  // per-batch query scratch, double-buffered: consecutive batches run on two
  // compute streams so one batch's kernel tails overlap the next one's start
  struct QSlot {
    DevBuf<uint32_t> qM, qL, nwt;
    DevBuf<uint64_t> wbase, qfeat;
    DevBuf<uint8_t> scan;
    DevBuf<unsigned int> qcount;
    DevBuf<HitRec> hits;
    void release() {
      qM.release(), qL.release(), nwt.release(), wbase.release(), qfeat.release(), scan.release(), qcount.release(),
          hits.release();
    }
  } qs[2];
  cudaStream_t own2 = nullptr;  // the second compute stream of a pipelined query
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  // multi-GPU handle (cfg.n_gpus > 1): the shards (single-device handles) it
  // drives; empty for a single-device handle.  Per-batch exchange events of a
  // shard in a group query (double-buffered like the staging slots).
  std::vector<mc_db*> shards;
  cudaEvent_t own_ready[2] = {nullptr, nullptr}, part_done[2] = {nullptr, nullptr},
              merge_done[2] = {nullptr, nullptr};
  // stats
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  // host scratch of an insert call, kept across calls (no re-allocation and
  // page-faulting of per-target arrays at 10^5 targets)
  std::vector<uint64_t> h_nwin, h_soff;
  std::vector<uint32_t> h_bwi, h_sel, h_loc, h_part;
  std::map<std::string, double> stage_ms;
  std::map<std::string, uint64_t> launches;
  uint64_t st_bp = 0, st_windows = 0, st_locations = 0, st_reads = 0, st_qfeat = 0, st_qloc = 0, st_read_bp = 0;
  uint64_t st_qfeat_hit = 0;  // probes that found a list
  uint64_t st_qoverlap = 0;   // query calls whose batches ran on two compute streams (stage times overlap)
  uint64_t st_qmed = 0, st_qlarge = 0, st_qloc_bin[3] = {0, 0, 0};
  int sms = 148;

  cudaEvent_t ev() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void begin(const char* name, cudaStream_t s = nullptr) {
    Pending p{name, ev(), ev()};
    cudaEventRecord(p.a, s ? s : stream);
    pending.push_back(p);
  }
  void end(cudaStream_t s = nullptr) { cudaEventRecord(pending.back().b, s ? s : stream); }
  void launched(const char* name, uint64_t n = 1) { launches[name] += n; }
  void collect() {  // call after a stream sync
    for (auto& p : pending) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, p.a, p.b) == cudaSuccess) stage_ms[p.name] += ms;
      cudaGetLastError();
      event_pool.push_back(p.a);
      event_pool.push_back(p.b);
    }
    pending.clear();
  }
  int sync() {
    CK(cudaStreamSynchronize(stream));
    CK(cudaGetLastError());
    collect();
    return MC_OK;
  }
};

namespace mc {
int num_sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}
}  // namespace mc

extern "C" {

const char* mc_last_error(void) { return g_err.c_str(); }

void mc_config_init(mc_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->k = 16;
  c->sketch_size = 16;
  c->window_len = 127;
  c->max_locations_per_feature = 254;
  c->max_candidates = 4;
  c->hits_min = 5;
  c->hits_diff = 4;
  c->n_partitions = 1;
  c->partition_begin = 0;
  c->n_local_partitions = 0;
  c->device = -1;
  c->capacity_bp = 1ull << 30;
  c->max_targets = 0;
  c->read_batch = 1ull << 20;
  c->table_slots_per_location = 1.25;
  c->n_gpus = 1;
  for (int g = 0; g < 8; ++g) c->devices[g] = -1;
}

int mc_plan_partitions(uint32_t P, uint32_t n, const uint64_t* lengths, uint64_t* running_bp, uint32_t* out_part) {
  if (P == 0 || (n && (!lengths || !out_part)) || !running_bp) return fail(MC_ERR_INVALID_ARG, "bad arguments");
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t best = 0;
    for (uint32_t q = 1; q < P; ++q)
      if (running_bp[q] < running_bp[best]) best = q;
    out_part[i] = best;
    running_bp[best] += lengths[i];
  }
  return MC_OK;
}

static int select_device(const mc_config* c, int* dev) {
  if (c->device >= 0) {
    CK(cudaSetDevice(c->device));
    *dev = c->device;
  } else {
    CK(cudaGetDevice(dev));
  }
  return MC_OK;
}

static int create_impl(const mc_config* cfg, const mc_taxonomy* tax, mc_db* db) {
  TRY(validate_cfg(cfg));
  const mc_config& c = *cfg;
  if (c.max_locations_per_feature < 1 || c.max_locations_per_feature > kMaxCap)
    return fail(MC_ERR_INVALID_ARG, "max_locations_per_feature=%u outside [1,%u]", c.max_locations_per_feature, kMaxCap);
  if (c.max_candidates < 1 || c.max_candidates > 8)
    return fail(MC_ERR_INVALID_ARG, "max_candidates=%u outside [1,8]", c.max_candidates);
  if (c.n_partitions < 1) return fail(MC_ERR_INVALID_ARG, "n_partitions must be >= 1");
  if (c.reserved2 != 0) return fail(MC_ERR_INVALID_ARG, "reserved2 must be 0");
  if (c.n_gpus > kMaxGpus) return fail(MC_ERR_INVALID_ARG, "n_gpus=%u exceeds %u", c.n_gpus, kMaxGpus);
  if (c.k >= 1 && c.window_len >= c.k && (uint64_t)c.insert_size_max > (uint64_t)(kRankGap - 2) * (c.window_len - c.k + 1))
    return fail(MC_ERR_INVALID_ARG, "insert_size_max=%u exceeds %u windows", c.insert_size_max, kRankGap - 2);
  const uint32_t n_local = c.n_local_partitions ? c.n_local_partitions : c.n_partitions;
  if ((uint64_t)c.partition_begin + n_local > c.n_partitions)
    return fail(MC_ERR_INVALID_ARG, "local partitions [%u,%u) exceed n_partitions=%u", c.partition_begin,
                c.partition_begin + n_local, c.n_partitions);
  if ((uint64_t)n_local * c.max_candidates > 64)
    return fail(MC_ERR_INVALID_ARG, "n_local_partitions * max_candidates must be <= 64");
  if (!(c.table_slots_per_location >= 0.05)) return fail(MC_ERR_INVALID_ARG, "table_slots_per_location too small");
  if (!tax || !tax->parent || tax->n_taxa < 2) return fail(MC_ERR_INVALID_ARG, "taxonomy needs n_taxa >= 2");

  db->cfg = c;
  db->cfg.n_local_partitions = n_local;
  if (db->cfg.read_batch == 0) db->cfg.read_batch = 1ull << 20;
  db->sc = make_sketch_cfg(c.k, c.sketch_size, c.window_len);
  db->pbegin = c.partition_begin;
  db->n_local = n_local;
  TRY(select_device(&c, &db->device));
  db->sms = num_sms();

  // ---- taxonomy -> depth + lineage table ----
  const uint32_t nt = tax->n_taxa;
  std::vector<uint32_t> parent(tax->parent, tax->parent + nt);
  db->parent_h = parent;
  if (tax->rank) db->rank_h.assign(tax->rank, tax->rank + nt);
  for (uint32_t i = 1; i < nt; ++i)
    if (parent[i] >= nt || parent[i] == 0) return fail(MC_ERR_INVALID_ARG, "taxon %u has invalid parent %u", i, parent[i]);
  std::vector<int32_t> depth(nt, -1);
  depth[0] = 0;
  std::vector<uint32_t> path;
  uint32_t maxd = 0;
  for (uint32_t i = 1; i < nt; ++i) {
    path.clear();
    uint32_t x = i;
    while (depth[x] < 0) {
      path.push_back(x);
      if (path.size() > 65) return fail(MC_ERR_INVALID_ARG, "taxonomy deeper than 64 or cyclic at taxon %u", i);
      if (parent[x] == x) break;
      x = parent[x];
    }
    int32_t d = (parent[x] == x && depth[x] < 0) ? -1 : depth[x];
    for (size_t j = path.size(); j-- > 0;) {
      uint32_t y = path[j];
      depth[y] = (parent[y] == y) ? 0 : d + 1;
      d = depth[y];
      if (d > 64) return fail(MC_ERR_INVALID_ARG, "taxonomy deeper than 64");
      maxd = std::max<uint32_t>(maxd, d);
    }
  }
  const uint32_t D = maxd + 1;
  std::vector<uint32_t> anc((size_t)nt * D, 0), dep(nt, 0);
  for (uint32_t i = 1; i < nt; ++i) {
    dep[i] = (uint32_t)depth[i];
    uint32_t x = i;
    for (int32_t d = depth[i]; d >= 0; --d) {
      anc[(size_t)i * D + d] = x;
      x = parent[x];
    }
  }
  db->n_taxa = nt;
  db->maxd = maxd;
  TRY(db->anc.ensure(anc.size()));
  TRY(db->depth.ensure(nt));
  CK(cudaMemcpy(db->anc.p, anc.data(), anc.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(db->depth.p, dep.data(), nt * 4, cudaMemcpyHostToDevice));

  CK(cudaStreamCreateWithFlags(&db->own, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&db->copy_stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&db->d2h_stream, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&db->own2, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&db->fork_ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&db->join_ev, cudaEventDisableTiming));
  for (int i = 0; i < 2; ++i) {
    CK(cudaEventCreateWithFlags(&db->out_ready[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&db->out_free[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&db->stage_ready[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&db->stage_free[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&db->qstat_ev[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&db->own_ready[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&db->part_done[i], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&db->merge_done[i], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&db->stage_ready[2], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&db->qstat_ev[2], cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&db->stage_free[2], cudaEventDisableTiming));
  db->stream = db->own;
  query_kernels_init();

  // ---- static per-partition build tables ----
  db->parts.resize(n_local);
  db->running_bp.assign(n_local, 0);
  const uint64_t bp_cap = n_local == 1 ? c.capacity_bp : c.capacity_bp / n_local + c.capacity_bp / (8 * n_local) + (64ull << 20);
  const uint64_t t_cap = c.max_targets ? (n_local == 1 ? c.max_targets : c.max_targets / n_local + c.max_targets / 4 + 64)
                                       : bp_cap / 512 + 1024;
  for (uint32_t q = 0; q < n_local; ++q) {
    Part& p = db->parts[q];
    p.gid = c.partition_begin + q;
    p.cap_targets = t_cap;
    p.cap_windows = bp_cap / db->sc.stride + t_cap;
    const uint64_t cap_loc = p.cap_windows * c.sketch_size;
    p.nslots = ((uint64_t)((double)cap_loc * c.table_slots_per_location) + 64 + kSubSlots - 1) & ~(uint64_t)(kSubSlots - 1);
    cudaError_t e = cudaMalloc(&p.T, p.nslots * sizeof(KSlot));
    if (e != cudaSuccess) {
      cudaGetLastError();
      p.T = nullptr;
      return fail(MC_ERR_OOM, "hash table of %llu slots (%.2f GB) does not fit", (unsigned long long)p.nslots,
                  p.nslots * (double)sizeof(KSlot) / 1e9);
    }
    // pair store: <= 1024 table regions of >= 2^20 slots; buckets 1.15x the mean + slack, shared spill
    p.shift = 20;
    while ((p.nslots >> p.shift) >= 1024) ++p.shift;
    p.nreg = (uint32_t)((p.nslots + (1ull << p.shift) - 1) >> p.shift);
    p.rcap = (uint64_t)((double)cap_loc / p.nreg * 1.15) + 4096;
    p.spill_cap = cap_loc / 32 + 65536;
    if (const char* e2 = getenv("MC_TEST_BUCKET_CAP")) {  // test knob: tiny buckets exercise the spill path
      p.rcap = strtoull(e2, nullptr, 10);
      p.spill_cap = cap_loc + 65536;
    }
    p.rcap = (p.rcap + 1) & ~1ull;  // even: every chunk starts 16-byte aligned (bulk copies in k_sub_scatter)
    p.spill_cap = (p.spill_cap + 1) & ~1ull;
    TRY(p.pairs.ensure(p.rcap * p.nreg + p.spill_cap));
    TRY(p.cursor.ensure(p.nreg + 2));
    TRY(p.hll.ensure(kHllRegs));
    CK(cudaMemsetAsync(p.cursor.p, 0, (p.nreg + 2) * 8, db->stream));
    CK(cudaMemsetAsync(p.hll.p, 0, kHllRegs * 4, db->stream));
    p.nslots_max = p.nslots;
  }
  TRY(db->counters.ensure(8));
  TRY(db->qstats.ensure(16));
  TRY(db->err.ensure(12));  // 3 status slots of 4 words (a query batch's slot is bi % 3)
  CK(cudaMallocHost(&db->herr_pin, 12 * sizeof(int)));
  TRY(db->qcount.ensure(4));
  TRY(db->total.ensure(2));
  return db->sync();
}

static int group_create(const mc_config* cfg, const mc_taxonomy* tax, mc_db* grp);

int mc_db_create(const mc_config* cfg, const mc_taxonomy* tax, mc_db** out) {
  if (!out) return fail(MC_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  mc_db* db = new mc_db();
  int rc = no_throw([&] { return cfg && cfg->n_gpus > 1 ? group_create(cfg, tax, db) : create_impl(cfg, tax, db); });
  if (rc != MC_OK) {
    std::string msg = g_err;
    mc_db_destroy(db);
    g_err = msg;
    return rc;
  }
  *out = db;
  return MC_OK;
}

void mc_db_destroy(mc_db* db) {
  if (!db) return;
  if (!db->shards.empty()) {  // multi-GPU handle: its shards own every resource
    for (mc_db* sh : db->shards) mc_db_destroy(sh);
    delete db;
    return;
  }
  cudaSetDevice(db->device);
  if (db->stream) cudaStreamSynchronize(db->stream);
  for (auto& p : db->parts) {
    if (p.T) cudaFree(p.T);
    p.pairs.release();
    p.cursor.release();
    p.cursor_bak.release();
    p.hll.release();
    p.hll_bak.release();
    p.values.release();
    p.rank_base.release();
    p.coarse.release();
    p.tgt_id.release();
    p.taxon_rank.release();
  }
  for (auto* b : {&db->chars, &db->rbuf1, &db->rbuf2, &db->scan_scratch, &db->stage[0], &db->stage[1], &db->qbuf1[0],
                  &db->qbuf1[1], &db->qbuf1[2], &db->qbuf2[0], &db->qbuf2[1], &db->qbuf2[2]})
    b->release();
  for (auto* b : {&db->qoff1[0], &db->qoff1[1], &db->qoff1[2], &db->qoff2[0], &db->qoff2[1], &db->qoff2[2]}) b->release();
  if (db->herr_pin) cudaFreeHost(db->herr_pin);
  if (db->pin) cudaFreeHost(db->pin);
  if (db->copy_stream) cudaStreamSynchronize(db->copy_stream), cudaStreamDestroy(db->copy_stream);
  if (db->d2h_stream) cudaStreamSynchronize(db->d2h_stream), cudaStreamDestroy(db->d2h_stream);
  if (db->own2) cudaStreamSynchronize(db->own2), cudaStreamDestroy(db->own2);
  for (cudaEvent_t e : {db->fork_ev, db->join_ev})
    if (e) cudaEventDestroy(e);
  db->qs[0].release();
  db->qs[1].release();
  for (int i = 0; i < 2; ++i) {
    if (db->out_ready[i]) cudaEventDestroy(db->out_ready[i]);
    if (db->out_free[i]) cudaEventDestroy(db->out_free[i]);
    db->otx[i].release();
    db->ocd[i].release();
    db->ohits[i].release();
    if (db->stage_ready[i]) cudaEventDestroy(db->stage_ready[i]);
    if (db->stage_free[i]) cudaEventDestroy(db->stage_free[i]);
    if (i == 1) {
      if (db->stage_ready[2]) cudaEventDestroy(db->stage_ready[2]);
      if (db->stage_free[2]) cudaEventDestroy(db->stage_free[2]);
      if (db->qstat_ev[2]) cudaEventDestroy(db->qstat_ev[2]);
    }
    if (db->qstat_ev[i]) cudaEventDestroy(db->qstat_ev[i]);
    for (cudaEvent_t e : {db->own_ready[i], db->part_done[i], db->merge_done[i]})
      if (e) cudaEventDestroy(e);
  }
  db->cursor.release();
  db->pairs.release();
  for (auto* b : {&db->meta64, &db->roff1, &db->roff2, &db->heavy, &db->total, &db->wbase, &db->qfeat, &db->subbase}) b->release();
  db->sorted.release();
  db->gcoarse.release();
  for (auto* b : {&db->meta32, &db->side, &db->qM, &db->qL, &db->otaxon, &db->ocand, &db->nwt, &db->subcnt, &db->anc,
                  &db->depth})
    b->release();
  db->counters.release();
  db->qstats.release();
  db->qcount.release();
  db->err.release();
  db->hits.release();
  for (auto& p : db->pending) db->event_pool.push_back(p.a), db->event_pool.push_back(p.b);
  for (auto e : db->event_pool) cudaEventDestroy(e);
  if (db->own) cudaStreamDestroy(db->own);
  delete db;
}

int mc_db_set_stream(mc_db* db, void* s) {
  if (!db) return fail(MC_ERR_INVALID_ARG, "db is NULL");
  if (!db->shards.empty()) return fail(MC_ERR_STATE, "mc_db_set_stream: not on a multi-GPU handle");
  CK(cudaSetDevice(db->device));
  CK(cudaStreamSynchronize(db->stream));
  db->collect();
  db->stream = s ? static_cast<cudaStream_t>(s) : db->own;
  return MC_OK;
}

int mc_db_clear(mc_db* db) {
  if (!db) return fail(MC_ERR_INVALID_ARG, "db is NULL");
  if (!db->shards.empty()) {
    for (mc_db* sh : db->shards) TRY(mc_db_clear(sh));
    db->where.clear();
    std::fill(db->running_bp.begin(), db->running_bp.end(), 0);
    db->state = 0;
    return MC_OK;
  }
  CK(cudaSetDevice(db->device));
  db->begin("clear");
  for (auto& p : db->parts) {
    CK(cudaMemsetAsync(p.cursor.p, 0, (p.nreg + 2) * 8, db->stream));
    CK(cudaMemsetAsync(p.hll.p, 0, kHllRegs * 4, db->stream));
    p.nslots = p.nslots_max;
    p.tid.clear();
    p.taxon.clear();
    p.nwin.clear();
    p.gbase.clear();
    p.windows = p.bp = p.gwin = 0;
    p.n_values = p.n_keys = p.n_locations = p.truncated = p.n_value_slots = 0;
    p.rank_base_h.clear();
    p.tgt_by_rank_h.clear();
  }
  db->end();
  db->where.clear();
  std::fill(db->running_bp.begin(), db->running_bp.end(), 0);
  db->state = 0;
  return db->sync();
}

// ---------------------------------------------------------------------------
// build: B1-B5
// ---------------------------------------------------------------------------
// One device's share of an insert call: caller targets sel[j] (in order) go
// to this handle's local partitions loc[j].  The caller validated ids, taxa
// and offsets.  Host bytes are staged in chunks of up to kStage bytes made of
// RUNS (consecutive own targets plus foreign gaps under kRunGap), one copy per
// run, double-buffered on the copy stream against the sketch of the previous
// chunk; device bytes (this or a peer GPU) are read in place.
// `before_commit` (may be empty) runs on the host while the GPU sketches: the
// caller's duplicate-id check of the call.  If it fails, the pair store's
// cursors and HyperLogLog registers are restored from a copy taken before the
// launch and the handle stays usable (nothing of the call is kept).
static int shard_insert(mc_db* db, const char* seqs, bool dev, const uint64_t* offs, const uint32_t* ids,
                        const uint32_t* tx, const std::vector<uint32_t>& sel, const std::vector<uint32_t>& loc,
                        const std::function<int()>& before_commit = {},
                        const std::function<int(uint32_t, uint32_t)>& assign = {}) {
  const uint32_t n = (uint32_t)sel.size();
  if (n == 0) return MC_OK;
  CK(cudaSetDevice(db->device));
  const uint32_t k = db->sc.k, stride = db->sc.stride;
  // per target: windows, gapped build window index of window 0 (filled chunk
  // by chunk, right before the chunk's launch; committed at the end)
  std::vector<uint64_t>& nwin = db->h_nwin;
  nwin.resize(n);
  std::vector<uint32_t>& bwi = db->h_bwi;
  bwi.resize(n);
  // running per-partition counters of the capacity check (committed at the end)
  std::vector<uint64_t> gw(db->n_local), win(db->n_local), ntg(db->n_local);
  for (uint32_t q = 0; q < db->n_local; ++q)
    gw[q] = db->parts[q].gwin, win[q] = db->parts[q].windows, ntg[q] = db->parts[q].tid.size();
  const double inv_stride = 1.0 / stride;
  // validation + window counts + capacity of targets [j0, j1) (MC_OK or the error)
  auto prepare = [&](uint32_t j0, uint32_t j1) -> int {
    for (uint32_t j = j0; j < j1; ++j) {
      const uint32_t i = sel[j], q = loc[j];
      if (offs[i + 1] < offs[i]) return fail(MC_ERR_INVALID_ARG, "offsets decrease at target %u", i);
      const uint64_t L = offs[i + 1] - offs[i];
      uint64_t w = 0;  // ceil((L - k + 1) / stride), by a reciprocal (exact after the correction)
      if (L >= k) {
        const uint64_t x = L - k + stride;
        w = (uint64_t)((double)x * inv_stride);
        while (w * stride > x) --w;
        while ((w + 1) * stride <= x) ++w;
      }
      nwin[j] = w;
      bwi[j] = (uint32_t)gw[q];
      gw[q] += w + kRankGap;
      win[q] += w;
      ntg[q] += 1;
      Part& p = db->parts[q];
      if (win[q] > p.cap_windows || ntg[q] > p.cap_targets || gw[q] >= 0xffffffffull)
        return fail(MC_ERR_CAPACITY, "partition %u: %llu windows / %llu targets exceed the static capacity (%llu / %llu); raise capacity_bp / max_targets",
                    p.gid, (unsigned long long)win[q], (unsigned long long)ntg[q], (unsigned long long)p.cap_windows,
                    (unsigned long long)p.cap_targets);
    }
    return MC_OK;
  };
  // ---- plan: chunks of up to kStage bytes (host) / 32 k targets (device).  Host bytes are staged chunk by
  // chunk in RUNS (consecutive own targets plus foreign gaps under kRunGap),
  // one copy per run; device bytes are read in place.  Each chunk's batch
  // metadata is built right before its launch (the GPU sketches chunk c while
  // the host prepares chunk c + 1) and goes up through pinned staging.
  uint64_t kStage = 1ull << 30;
  if (const char* e2 = getenv("MC_TEST_STAGE_BYTES")) kStage = strtoull(e2, nullptr, 10);  // test knob
  constexpr uint64_t kRunGap = 1ull << 20;
  constexpr uint32_t kDevChunkTargets = 1u << 15;
  struct Run {
    uint64_t src, bytes, dst;  // caller bytes [src, src + bytes) -> staging offset dst
  };
  struct Chunk {
    uint32_t j0, j1, r0, r1;
    uint64_t bytes, base;  // bytes staged (host) / spanned (device); device: first byte in the caller's buffer
  };
  std::vector<Run> runs;
  std::vector<Chunk> chunks;
  std::vector<uint64_t>& soff = db->h_soff;  // target sel[j]'s first byte, relative to its chunk's base
  soff.resize(n);
  if (dev) {  // device chunks only bound the host's planning ahead of the GPU (32 k targets); their
              // byte span and offsets are taken when the chunk is prepared
    for (uint32_t j0 = 0; j0 < n; j0 += kDevChunkTargets) chunks.push_back({j0, std::min(n, j0 + kDevChunkTargets), 0, 0, 0, 0});
  } else {
    Chunk cur{0, 0, 0, 0, 0, 0};
    for (uint32_t j = 0; j < n; ++j) {
      const uint64_t b = offs[sel[j]], e = offs[sel[j] + 1];
      if (e < b) return fail(MC_ERR_INVALID_ARG, "offsets decrease at target %u", sel[j]);
      const bool have = cur.r1 > cur.r0;
      const uint64_t rend = have ? runs.back().src + runs.back().bytes : 0;
      bool extend = have && b >= rend && b - rend <= kRunGap;
      uint64_t add = extend ? e - rend : e - b;
      if (cur.j1 > cur.j0 && cur.bytes + add > kStage) {  // close the chunk
        chunks.push_back(cur);
        cur = Chunk{j, j, (uint32_t)runs.size(), (uint32_t)runs.size(), 0, 0};
        extend = false;
        add = e - b;
      }
      if (extend) {
        runs.back().bytes = e - runs.back().src;
      } else {
        runs.push_back({b, e - b, cur.bytes});
        cur.r1 = (uint32_t)runs.size();
      }
      soff[j] = runs.back().dst + (b - runs.back().src);
      cur.bytes += add;
      cur.j1 = j + 1;
    }
    chunks.push_back(cur);
  }
  // metadata of all batches: per batch win_base[nt+1] | seq_off[nt] | seq_len[nt] (u64), bwi_base[nt] (u32)
  const size_t cap64 = 3 * (size_t)n + (size_t)db->n_local * chunks.size(), cap32 = n;
  TRY(db->meta64.ensure(cap64));
  TRY(db->meta32.ensure(cap32));
  TRY(db->ensure_pin(cap64 * 8 + cap32 * 4));
  uint64_t* m64 = reinterpret_cast<uint64_t*>(db->pin);
  uint32_t* m32 = reinterpret_cast<uint32_t*>(m64 + cap64);
  size_t o64 = 0, o32 = 0;
  phase("plan");
  cudaStream_t st = db->stream;
  // From the first launch on, a failure leaves the pair store partly written:
  // the handle is broken unless the call completes or rolls back cleanly.
  struct BrokenUnlessDone {
    mc_db* db;
    bool done = false;
    ~BrokenUnlessDone() {
      if (!done) db->state = -1;
    }
  } guard{db};
  // rollback point: the region cursors and HyperLogLog registers.  A call
  // that fails validation, capacity or the duplicate check (all found while
  // earlier chunks already run) restores them: nothing of the call is kept
  // and the handle stays usable.
  for (auto& p : db->parts) {
    TRY(p.cursor_bak.ensure(p.nreg + 2));
    TRY(p.hll_bak.ensure(kHllRegs));
    CK(cudaMemcpyAsync(p.cursor_bak.p, p.cursor.p, (p.nreg + 2) * 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(p.hll_bak.p, p.hll.p, kHllRegs * 4, cudaMemcpyDeviceToDevice, st));
  }
  auto rollback = [&](int rc) -> int {
    const std::string msg = g_err;
    for (auto& p : db->parts) {
      CK(cudaMemcpyAsync(p.cursor.p, p.cursor_bak.p, (p.nreg + 2) * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(p.hll.p, p.hll_bak.p, kHllRegs * 4, cudaMemcpyDeviceToDevice, st));
    }
    TRY(db->sync());
    CK(cudaStreamSynchronize(db->copy_stream));
    guard.done = true;
    g_err = msg;
    return rc;
  };
  CK(cudaMemsetAsync(db->err.p, 0, sizeof(int) * 4, st));
  CK(cudaMemsetAsync(db->counters.p, 0, sizeof(unsigned long long), st));
  auto store_of = [&](Part& p) {
    PairStore ps{};
    ps.pairs = p.pairs.p;
    ps.cursor = p.cursor.p;
    ps.rcap = p.rcap;
    ps.spill_cap = p.spill_cap;
    ps.nslots = p.nslots_max;
    ps.nreg = p.nreg;
    ps.shift = p.shift;
    ps.err = db->err.p;
    ps.hll = p.hll.p;
    return ps;
  };
  if (!dev) {  // size both staging buffers up front (no reallocation while kernels read them)
    uint64_t mx = 0;
    for (auto& ch : chunks) mx = std::max<uint64_t>(mx, ch.bytes);
    for (int i = 0; i < 2 && i < (int)chunks.size(); ++i) TRY(db->stage[i].ensure(mx + 64));
  }
  // ---- stream the chunks: sketch every window, append its pairs to the store ----
  std::vector<uint32_t> pick;
  for (uint32_t c = 0; c < chunks.size(); ++c) {
    Chunk& ch = chunks[c];
    if (assign)
      if (const int rc = assign(ch.j0, ch.j1)) return rollback(rc);
    if (const int rc = prepare(ch.j0, ch.j1)) return rollback(rc);
    if (dev) {  // (offsets validated by prepare)
      ch.base = offs[sel[ch.j0]];
      for (uint32_t j = ch.j0; j < ch.j1; ++j) soff[j] = offs[sel[j]] - ch.base;
    }
    const uint8_t* dchars;
    const int sb = c & 1;
    if (dev) {
      dchars = reinterpret_cast<const uint8_t*>(seqs) + ch.base;
    } else {
      CK(cudaStreamWaitEvent(db->copy_stream, db->stage_free[sb], 0));
      db->begin("h2d_refs", db->copy_stream);
      for (uint32_t r = ch.r0; r < ch.r1; ++r)
        CK(cudaMemcpyAsync(db->stage[sb].p + runs[r].dst, seqs + runs[r].src, runs[r].bytes, cudaMemcpyHostToDevice,
                           db->copy_stream));
      db->end(db->copy_stream);
      // (the sketch reads whole aligned words: define the padding after the chunk)
      CK(cudaMemsetAsync(db->stage[sb].p + ch.bytes, 'N', 64, db->copy_stream));
      CK(cudaEventRecord(db->stage_ready[sb], db->copy_stream));
      dchars = db->stage[sb].p;
    }
    // this chunk's batches (one per local partition): metadata -> pinned -> device
    const size_t c64 = o64, c32 = o32;
    struct B {
      uint32_t q, nt;
      size_t o64, o32;
      uint64_t windows;
    };
    B bl[64];
    uint32_t nbl = 0;
    for (uint32_t q = 0; q < db->n_local; ++q) {
      pick.clear();
      for (uint32_t j = ch.j0; j < ch.j1; ++j)
        if (loc[j] == q && nwin[j] > 0) pick.push_back(j);
      if (pick.empty()) continue;
      B bt{q, (uint32_t)pick.size(), o64, o32, 0};
      uint64_t acc = 0;
      for (uint32_t x = 0; x < bt.nt; ++x) {
        const uint32_t j = pick[x], i = sel[j];
        m64[bt.o64 + x] = acc;
        acc += nwin[j];
        m64[bt.o64 + bt.nt + 1 + x] = soff[j];
        m64[bt.o64 + 2 * (size_t)bt.nt + 1 + x] = offs[i + 1] - offs[i];
        m32[bt.o32 + x] = bwi[j];
      }
      m64[bt.o64 + bt.nt] = acc;
      bt.windows = acc;
      o64 += 3 * (size_t)bt.nt + 1;
      o32 += bt.nt;
      bl[nbl++] = bt;
    }
    if (o64 > c64) {
      CK(cudaMemcpyAsync(db->meta64.p + c64, m64 + c64, (o64 - c64) * 8, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(db->meta32.p + c32, m32 + c32, (o32 - c32) * 4, cudaMemcpyHostToDevice, st));
    }
    if (!dev) CK(cudaStreamWaitEvent(st, db->stage_ready[sb], 0));
    for (uint32_t x = 0; x < nbl; ++x) {
      const B& bt = bl[x];
      Part& p = db->parts[bt.q];
      const BuildBatch bb{dchars, db->meta64.p + bt.o64, db->meta64.p + bt.o64 + bt.nt + 1,
                          db->meta64.p + bt.o64 + 2 * (size_t)bt.nt + 1, db->meta32.p + bt.o32, bt.nt, bt.windows};
      db->begin("sketch_partition");
      launch_sketch_partition(bb, db->sc, store_of(p), db->sms, st);
      db->end();
      db->launched("k_sketch_partition");
    }
    if (!dev) CK(cudaEventRecord(db->stage_free[sb], st));
    CK(cudaGetLastError());
  }
  phase("enqueue");
  // ---- while the GPU sketches: the caller's checks, then the registry commit ----
  if (before_commit) {
    if (const int rc = before_commit()) return rollback(rc);
    phase("check_ids");
  }
  db->where.reserve(n);
  for (uint32_t j = 0; j < n; ++j) {
    const uint32_t i = sel[j];
    Part& p = db->parts[loc[j]];
    db->where.put(ids[i], loc[j], (uint32_t)p.tid.size());
    p.tid.push_back(ids[i]);
    p.taxon.push_back(tx[i]);
    p.nwin.push_back(nwin[j]);
    p.gbase.push_back(bwi[j]);
    p.windows += nwin[j];
    p.gwin += nwin[j] + kRankGap;
    p.bp += offs[i + 1] - offs[i];
    db->running_bp[loc[j]] += offs[i + 1] - offs[i];
  }
  phase("commit");
  int herr[4];
  CK(cudaMemcpyAsync(herr, db->err.p, sizeof herr, cudaMemcpyDeviceToHost, db->stream));
  TRY(db->sync());
  phase("gpu_wait");
  if (herr[1]) return fail(MC_ERR_CAPACITY, "pair store spill area full (skewed features; raise capacity_bp)");
  for (uint32_t j = 0; j < n; ++j) db->st_bp += offs[sel[j] + 1] - offs[sel[j]], db->st_windows += nwin[j];
  guard.done = true;
  return MC_OK;
}

// Host copies of one caller batch's arrays + checks that need no handle state.
struct TargetIn {
  uint32_t n = 0;
  const char* seqs = nullptr;
  bool dev = false;
  HostView<uint64_t> offs;
  HostView<uint32_t> ids, tx, pids;
  bool has_pids = false;
};

static int read_target_batch(const mc_target_batch& b, uint32_t n_taxa, TargetIn& t) {
  t.n = b.n;
  t.seqs = b.seqs;
  if (b.n == 0) return MC_OK;
  if (!b.seqs || !b.offsets || !b.target_ids || !b.taxa) return fail(MC_ERR_INVALID_ARG, "NULL input array");
  TRY(t.offs.load(b.offsets, (size_t)b.n + 1));
  TRY(t.ids.load(b.target_ids, b.n));
  TRY(t.tx.load(b.taxa, b.n));
  t.has_pids = b.partition_ids != nullptr;
  if (t.has_pids) TRY(t.pids.load(b.partition_ids, b.n));
  t.dev = is_device_ptr(b.seqs);
  return MC_OK;
}

// ids and taxa of batch t valid (offsets are checked where the windows are counted)
static int check_ids_taxa(const TargetIn& t, uint32_t n_taxa) {
  for (uint32_t i = 0; i < t.n; ++i) {
    if (t.ids[i] == 0xffffffffu) return fail(MC_ERR_INVALID_ARG, "target id UINT32_MAX is reserved");
    if (t.tx[i] == 0 || t.tx[i] >= n_taxa) return fail(MC_ERR_INVALID_ARG, "taxon %u of target %u invalid", t.tx[i], t.ids[i]);
  }
  return MC_OK;
}

// Ids of all batches: unique among themselves and new to `reg`.
static int check_new_ids(const IdMap& reg, const std::vector<TargetIn>& in) {
  IdMap seen;
  size_t tot = 0;
  for (auto& t : in) tot += t.n;
  seen.reserve(tot);
  for (auto& t : in)
    for (uint32_t i = 0; i < t.n; ++i) {
      if (reg.count(t.ids[i])) return fail(MC_ERR_INVALID_ARG, "duplicate target id %u", t.ids[i]);
      if (!seen.put(t.ids[i], 0, 0)) return fail(MC_ERR_INVALID_ARG, "duplicate target id %u in the call", t.ids[i]);
    }
  return MC_OK;
}

// S9: partition of every target, global ids in [pbegin, pbegin + np);
// `run` (running bp per partition) is advanced.
static int assign_range(const TargetIn& t, uint32_t i0, uint32_t i1, uint32_t pbegin, uint32_t np,
                        std::vector<uint64_t>& run, std::vector<uint32_t>& part) {
  for (uint32_t i = i0; i < i1; ++i) {
    const uint64_t L = t.offs[i + 1] - t.offs[i];
    uint32_t q;
    if (t.has_pids) {
      if (t.pids[i] < pbegin || t.pids[i] >= pbegin + np)
        return fail(MC_ERR_INVALID_ARG, "partition id %u of target %u is not held by this handle", t.pids[i], t.ids[i]);
      q = t.pids[i] - pbegin;
    } else {
      q = 0;
      for (uint32_t r = 1; r < np; ++r)
        if (run[r] < run[q]) q = r;
    }
    part[i] = pbegin + q;
    run[q] += L;
  }
  return MC_OK;
}
static int assign_partitions(const TargetIn& t, uint32_t pbegin, uint32_t np, std::vector<uint64_t>& run,
                             std::vector<uint32_t>& part) {
  part.resize(t.n);
  return assign_range(t, 0, t.n, pbegin, np, run, part);
}

static int group_insert(mc_db* grp, const std::vector<TargetIn>& in);

static int insert_batches_impl(mc_db* db, uint32_t nb, const mc_target_batch* b) {
  if (!db) return fail(MC_ERR_INVALID_ARG, "db is NULL");
  if (db->state != 0) return fail(MC_ERR_STATE, db->state == 1 ? "insert after finalize" : "handle is broken");
  if (nb && !b) return fail(MC_ERR_INVALID_ARG, "NULL batches");
  HostPhases ph("insert");
  std::vector<TargetIn> in(nb);
  for (uint32_t x = 0; x < nb; ++x) TRY(read_target_batch(b[x], db->n_taxa, in[x]));
  phase("read_validate");
  if (!db->shards.empty()) {
    for (auto& t : in) {
      TRY(check_ids_taxa(t, db->n_taxa));
      for (uint32_t i = 0; i < t.n; ++i)
        if (t.offs[i + 1] < t.offs[i]) return fail(MC_ERR_INVALID_ARG, "offsets decrease at target %u", i);
    }
    TRY(check_new_ids(db->where, in));
    return group_insert(db, in);
  }
  for (auto& t : in)
    if (t.dev && ptr_device(t.seqs) != db->device)
      return fail(MC_ERR_INVALID_ARG, "device-resident targets must be on the handle's device %d", db->device);
  // the duplicate-id check of the whole call runs on the host while the GPU
  // sketches the first non-empty batch (which is rolled back if it fails)
  bool checked = false;
  for (auto& t : in) {
    if (t.n == 0) continue;
    std::vector<uint64_t> run = db->running_bp;
    std::vector<uint32_t>&part = db->h_part, &sel = db->h_sel, &loc = db->h_loc;
    sel.resize(t.n);
    loc.resize(t.n);
    part.resize(t.n);
    for (uint32_t i = 0; i < t.n; ++i) sel[i] = i;
    // S9 assignment chunk by chunk, right before each chunk's launch (in order:
    // the running bp carries over), so the GPU starts after the first chunk
    auto assign = [&](uint32_t j0, uint32_t j1) -> int {
      TRY(assign_range(t, j0, j1, db->pbegin, db->n_local, run, part));
      for (uint32_t j = j0; j < j1; ++j) loc[j] = part[j] - db->pbegin;
      return MC_OK;
    };
    std::function<int()> check;
    if (!checked)
      check = [&]() -> int {
        for (auto& tt : in) TRY(check_ids_taxa(tt, db->n_taxa));
        return check_new_ids(db->where, in);
      };
    checked = true;
    TRY(shard_insert(db, t.seqs, t.dev, t.offs.data(), t.ids.data(), t.tx.data(), sel, loc, check, assign));
  }
  return MC_OK;
}

// ---------------------------------------------------------------------------
// finalize: B6
// ---------------------------------------------------------------------------
static int finalize_part(mc_db* db, Part& p) {
  HostPhases ph("finalize");
  const uint32_t nt = (uint32_t)p.tid.size();
  cudaStream_t st = db->stream;
  // The target ranking and its tables (rank -> window base / id / taxon, the
  // gapped -> ranked conversion for finalize, the coarse index for queries) are
  // built on the host WHILE the GPU regroups the pairs (k_sub_count /
  // k_sub_scatter do not read them); they go up through pinned staging.
  const uint64_t nblk_g = ((uint64_t)p.gwin >> 10) + 1;
  TRY(p.rank_base.ensure(nt + 1));
  TRY(p.tgt_id.ensure(std::max(nt, 1u)));
  TRY(p.taxon_rank.ensure(std::max(nt, 1u)));
  TRY(db->gcoarse.ensure(nblk_g));
  bool identity = true;
  auto rank_tables = [&]() -> int {
    // rank targets by id; ranked window space with gaps (kRankGap) between targets
    std::vector<uint32_t> order(nt);
    std::iota(order.begin(), order.end(), 0u);
    if (!std::is_sorted(p.tid.begin(), p.tid.end()))  // (ids in insertion order: order is the identity)
      std::sort(order.begin(), order.end(), [&](uint32_t x, uint32_t y) { return p.tid[x] < p.tid[y]; });
    std::vector<uint32_t> rank_of(nt);
    p.rank_base_h.assign(nt + 1, 0);
    p.tgt_by_rank_h.resize(nt);
    uint64_t acc = 0;
    for (uint32_t r = 0; r < nt; ++r) {
      rank_of[order[r]] = r;
      p.rank_base_h[r] = (uint32_t)acc;
      p.tgt_by_rank_h[r] = p.tid[order[r]];
      acc += p.nwin[order[r]] + kRankGap;
      if (acc >= 0xffffffffull) return fail(MC_ERR_CAPACITY, "partition %u: ranked window space exceeds 32 bits", p.gid);
    }
    p.rank_base_h[nt] = (uint32_t)acc;
    const uint64_t nblk_c = (acc >> 10) + 1;
    const size_t bytes = nblk_g * sizeof(uint4) + nblk_c * sizeof(uint2) + ((size_t)nt + 1) * 4 + 2 * (size_t)nt * 4;
    TRY(db->ensure_pin(bytes));
    uint4* gc = reinterpret_cast<uint4*>(db->pin);
    uint2* coarse = reinterpret_cast<uint2*>(gc + nblk_g);
    uint32_t* rb = reinterpret_cast<uint32_t*>(coarse + nblk_c);
    uint32_t* tg = rb + nt + 1;
    uint32_t* tx = tg + nt;
    std::memcpy(rb, p.rank_base_h.data(), ((size_t)nt + 1) * 4);
    if (nt) std::memcpy(tg, p.tgt_by_rank_h.data(), (size_t)nt * 4);
    for (uint32_t r = 0; r < nt; ++r) tx[r] = p.taxon[order[r]];
    phase("rank");
    std::vector<uint32_t> delta(std::max(nt, 1u), 0);
    for (uint32_t i = 0; i < nt; ++i) {
      delta[i] = p.rank_base_h[rank_of[i]] - p.gbase[i];
      identity &= delta[i] == 0;
    }
    {  // gapped -> ranked window conversion table for finalize (see to_ranked)
      uint32_t t = 0;
      for (uint64_t j = 0; j < nblk_g; ++j) {
        while (t + 1 < nt && p.gbase[t + 1] <= (j << 10)) ++t;
        const uint64_t nxt = t + 1 < nt ? p.gbase[t + 1] : 0xffffffffull;
        const bool in = nxt < ((j + 1) << 10);
        gc[j] = make_uint4(nt ? delta[t] : 0u, in ? (uint32_t)nxt : 0xffffffffu, in ? delta[t + 1] : 0u, 0u);
      }
    }
    {  // coarse index: target rank at the start of every 1024 ranked windows
       // (targets are >= kRankGap apart, so a block holds at most one target start)
      uint32_t t = 0;
      for (uint64_t j = 0; j < nblk_c; ++j) {
        while (t + 1 < nt && p.rank_base_h[t + 1] <= (j << 10)) ++t;
        const uint64_t nxt = t + 1 < nt ? p.rank_base_h[t + 1] : 0xffffffffull;
        coarse[j] = make_uint2(t, nxt < ((j + 1) << 10) ? (uint32_t)nxt : 0xffffffffu);
      }
    }
    TRY(p.coarse.ensure(nblk_c));
    CK(cudaMemcpyAsync(db->gcoarse.p, gc, nblk_g * sizeof(uint4), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(p.coarse.p, coarse, nblk_c * sizeof(uint2), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(p.rank_base.p, rb, ((size_t)nt + 1) * 4, cudaMemcpyHostToDevice, st));
    if (nt) {
      CK(cudaMemcpyAsync(p.tgt_id.p, tg, (size_t)nt * 4, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(p.taxon_rank.p, tx, (size_t)nt * 4, cudaMemcpyHostToDevice, st));
    }
    phase("coarse_tables");
    return MC_OK;
  };
  const uint32_t cap = db->cfg.max_locations_per_feature;
  // table size from the HyperLogLog estimate of distinct features (load ~0.4);
  // fastrange keeps every region of the pair store a contiguous slot range
  std::vector<uint32_t> hreg(kHllRegs);
  CK(cudaMemcpyAsync(hreg.data(), p.hll.p, kHllRegs * 4, cudaMemcpyDeviceToHost, st));
  TRY(db->sync());
  phase("hll_read");
  double z = 0;
  uint32_t zeros = 0;
  for (uint32_t v : hreg) z += std::ldexp(1.0, -(int)v), zeros += v == 0;
  const double mreg = kHllRegs, alpha = 0.7213 / (1 + 1.079 / mreg);
  double est = alpha * mreg * mreg / z;
  if (est <= 2.5 * mreg && zeros) est = mreg * std::log(mreg / zeros);
  est *= (double)(1u << kHllSampleBits);  // (the registers saw a 1 / 2^kHllSampleBits hash-space sample)
  auto round_sub = [](uint64_t x) { return (x + kSubSlots - 1) & ~(uint64_t)(kSubSlots - 1); };
  p.nslots = std::min<uint64_t>(p.nslots_max, round_sub((uint64_t)(est * 2.5) + 4096));
  if (const char* e2 = getenv("MC_TEST_TABLE_SLOTS"))  // test knob: an undersized table exercises the retry
    p.nslots = std::min<uint64_t>(p.nslots_max, round_sub(strtoull(e2, nullptr, 10)));
  // pairs in the store (exact: region fills, spill fill)
  std::vector<unsigned long long> cur(p.nreg + 1);
  CK(cudaMemcpyAsync(cur.data(), p.cursor.p, (p.nreg + 1) * 8, cudaMemcpyDeviceToHost, st));
  TRY(db->sync());
  phase("cursor_read");
  uint64_t n_pairs = 0;
  for (uint32_t r = 0; r < p.nreg; ++r) n_pairs += std::min<uint64_t>(cur[r], p.rcap);
  n_pairs += std::min<uint64_t>(cur[p.nreg], p.spill_cap);
  FinalizeArgs a{};
  a.ps.pairs = p.pairs.p;
  a.ps.cursor = p.cursor.p;
  a.ps.rcap = p.rcap;
  a.ps.spill_cap = p.spill_cap;
  a.ps.nslots = p.nslots_max;
  a.ps.nreg = p.nreg;
  a.ps.shift = p.shift;
  a.ps.err = db->err.p;
  a.ps.hll = p.hll.p;
  a.T = p.T;
  a.cap = cap;
  a.gcoarse = db->gcoarse.p;
  a.identity = true;  // (set once the rank tables exist, before k_sub_finalize)
  a.counters = db->counters.p;
  TRY(db->sorted.ensure(std::max<uint64_t>(n_pairs, 1)));
  TRY(p.values.ensure(std::max<uint64_t>(n_pairs, 1)));
  TRY(db->heavy.ensure(2 * (n_pairs / (cap + 1) + 1)));
  a.sorted = db->sorted.p;
  a.values = p.values.p;
  TRY(db->side.ensure(std::max<uint64_t>(n_pairs, 1)));  // upper bound; only heavy keys' values land here
  a.side = db->side.p;
  a.heavy = reinterpret_cast<ulonglong2*>(db->heavy.p);
  // B5 + B6: regroup the pairs by table sub-region, then build every
  // sub-region in shared memory; if the HyperLogLog estimate was too small a
  // sub-region fills up and finalize reruns at the static maximum
  for (int attempt = 0;; ++attempt) {
    a.nslots = p.nslots;
    a.nsub = p.nslots >> kSubLg;
    TRY(p.vbase.ensure(a.nsub));
    a.vbase = p.vbase.p;
    TRY(db->subcnt.ensure(a.nsub));
    TRY(db->subbase.ensure(a.nsub + 1));
    a.subcnt = db->subcnt.p;
    a.subbase = db->subbase.p;
    CK(cudaMemsetAsync(db->err.p, 0, 4 * sizeof(int), st));
    CK(cudaMemsetAsync(db->counters.p, 0, 8 * sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(a.subcnt, 0, a.nsub * 4, st));
    db->begin("sub_count");
    launch_sub_count(a, db->sms, st);
    TRY(db->scan_scratch.ensure(scan_scratch_bytes(a.nsub)));
    int nl = 0;
    launch_exclusive_scan(a.subcnt, a.subbase, a.nsub, 0xffffffffu, db->scan_scratch.p, a.subbase + a.nsub, st, &nl);
    db->end();
    db->launched("k_sub_count");
    db->launched("k_scan", nl);
    CK(cudaMemsetAsync(a.subcnt, 0, a.nsub * 4, st));
    db->begin("sub_scatter");
    launch_sub_scatter(a, db->sms, st);
    db->end();
    db->launched("k_sub_scatter");
    if (attempt == 0) {  // (host work overlapping the regroup kernels)
      TRY(rank_tables());
      a.identity = identity;
    }
    db->begin("sub_finalize");
    launch_sub_finalize(a, db->sms, st);
    db->end();
    db->launched("k_sub_finalize");
    int herr[4];
    CK(cudaMemcpyAsync(herr, db->err.p, sizeof herr, cudaMemcpyDeviceToHost, st));
    TRY(db->sync());
    if (herr[2]) return fail(MC_ERR_CUDA, "internal: sub-region bound violated");
    if (!herr[0]) break;
    if (p.nslots == p.nslots_max) return fail(MC_ERR_CAPACITY, "hash table full (raise capacity_bp or table_slots_per_location)");
    p.nslots = p.nslots_max;
  }
  phase("kernels");
  unsigned long long ctr[8];
  CK(cudaMemcpyAsync(ctr, db->counters.p, sizeof ctr, cudaMemcpyDeviceToHost, st));
  TRY(db->sync());
  p.n_keys = ctr[0];
  p.n_locations = ctr[1];
  p.truncated = ctr[2];
  p.n_values = ctr[4];
  p.n_value_slots = n_pairs;
  if (ctr[3]) {
    db->begin("heavy_select");
    launch_heavy_select(a, db->sms * 4, st);
    db->end();
    db->launched("k_heavy_select");
  }
  TRY(db->sync());
  phase("heavy");
  db->st_locations += p.n_locations;
  return MC_OK;
}

static int group_finalize(mc_db* grp);

int mc_db_finalize(mc_db* db) {
  if (!db) return fail(MC_ERR_INVALID_ARG, "db is NULL");
  if (db->state != 0) return fail(MC_ERR_STATE, db->state == 1 ? "already finalized" : "handle is broken");
  if (!db->shards.empty()) return group_finalize(db);
  CK(cudaSetDevice(db->device));
  for (auto& p : db->parts) {
    int rc = finalize_part(db, p);
    if (rc != MC_OK) {
      db->state = -1;
      return rc;
    }
  }
  db->state = 1;
  return MC_OK;
}

// ---------------------------------------------------------------------------
// query: Q1-Q9
// ---------------------------------------------------------------------------
struct ReadSide {
  std::vector<uint64_t> copy;       // host copy of device-resident offsets (only when the bytes are not)
  const uint64_t* offs = nullptr;   // host-readable offsets: the caller's host array (no copy) or `copy`;
                                    // null when reads and offsets are both device-resident
  bool dev = false, dev_offs = false;
  bool on_device() const { return dev && dev_offs; }
};

// Every record's offsets and length are checked on the device (k_query_plan;
// the error names the record, reported one batch later).  The host only needs
// the byte range of each batch to stage host reads, so host offsets are read
// in place (no copy, no per-record host loop) and device offsets come to the
// host only when the bytes do not live on the device.
static int check_reads(mc_db* db, uint64_t n, const char* reads, const uint64_t* ro, const char* mates,
                       const uint64_t* mo, ReadSide& r1, ReadSide& r2) {
  (void)db;
  if (!reads || !ro) return fail(MC_ERR_INVALID_ARG, "NULL reads");
  if (mates && !mo) return fail(MC_ERR_INVALID_ARG, "mates without mate_offsets");
  r1.dev = is_device_ptr(reads);
  r1.dev_offs = is_device_ptr(ro);
  if (mates) {
    r2.dev = is_device_ptr(mates);
    r2.dev_offs = is_device_ptr(mo);
  }
  if (r1.on_device() && (!mates || r2.on_device())) return MC_OK;
  auto view = [&](const uint64_t* p, ReadSide& r) -> int {
    if (r.dev_offs) {
      TRY(to_host(p, n + 1, r.copy));
      r.offs = r.copy.data();
    } else {
      r.offs = p;
    }
    return MC_OK;
  };
  TRY(view(ro, r1));
  if (mates) TRY(view(mo, r2));
  return MC_OK;
}

// Q1-Q7 of one batch on db->stream, no host synchronisation when the batch's
// window total W is known on the host (host offsets); W = UINT64_MAX: read it
// back from the device (device-resident offsets).
static int run_partials(mc_db* db, const ReadBatch& rb, HitRec* hits, uint64_t W, int* err, int k,
                        cudaStream_t st) {
  auto& q = db->qs[k];  // this batch's scratch slot
  const uint64_t nb = rb.n;
  TRY(q.qM.ensure(nb));
  TRY(q.qL.ensure(nb));
  TRY(q.nwt.ensure(nb));
  TRY(q.wbase.ensure(nb + 1));
  TRY(q.qcount.ensure(4));
  QueryArgs a{};
  a.rb = rb;
  a.c = db->sc;
  a.m = db->cfg.max_candidates;
  a.insert_size_max = db->cfg.insert_size_max;
  a.out = hits;
  a.n_lists = db->n_local;
  a.qM = q.qM.p;
  a.qL = q.qL.p;
  a.qcount = q.qcount.p;
  a.err = err;
  a.stats = db->qstats.p;
  a.wbase = q.wbase.p;
  // Q1: windows per record -> first window of each record, and the batch total
  db->begin("query_plan", st);
  launch_query_plan(a, q.nwt.p, (uint64_t)(kRankGap - 2) * db->sc.stride, st);
  TRY(q.scan.ensure(scan_scratch_bytes(nb)));
  int nl = 0;
  launch_exclusive_scan(q.nwt.p, q.wbase.p, nb, 0xffffffffu, q.scan.p, q.wbase.p + nb, st, &nl);
  db->end(st);
  db->launched("k_query_plan");
  db->launched("k_scan", nl);
  if (W == UINT64_MAX) {
    CK(cudaMemcpyAsync(&W, q.wbase.p + nb, sizeof W, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  TRY(q.qfeat.ensure(std::max<uint64_t>(W * db->sc.s, 1)));
  a.qfeat = q.qfeat.p;
  for (uint32_t qi = 0; qi < db->n_local; ++qi) {
    Part& p = db->parts[qi];
    CK(cudaMemsetAsync(q.qcount.p, 0, 4 * sizeof(unsigned), st));
    a.pv = PartView{p.T, p.vbase.p, p.nslots, p.values.p, p.rank_base.p, p.tgt_id.p, p.taxon_rank.p, (uint32_t)p.tid.size(),
                    p.coarse.p};
    a.list = qi;
    db->begin("query_sketch_probe", st);
    launch_query_sketch_probe(a, W, q.qfeat.p, db->sms, st);
    db->end(st);
    const uint64_t want = (nb + 7) / 8;
    const int gs = (int)std::min<uint64_t>(std::max<uint64_t>(want, 1), (uint64_t)db->sms * 16);
    db->begin("query_small", st);
    launch_query_small(a, gs, st);
    db->end(st);
    db->begin("query_medium", st);
    launch_query_medium(a, db->sms * (7 * 128 / kMedT), st);
    db->end(st);
    db->begin("query_large", st);
    launch_query_large(a, db->sms, st);
    db->end(st);
    if (W) db->launched("k_query_sketch_probe");
    db->launched("k_query_small");
    db->launched("k_query_medium");
    db->launched("k_query_large");
    CK(cudaGetLastError());
  }
  return MC_OK;
}

// error status of one batch (pinned copy of its err slot) -> MC_* code
static int batch_status(mc_db* db, const int* herr, uint64_t b0) {
  if (herr[2] == 1)
    return fail(MC_ERR_INVALID_ARG, "read offsets decrease at record %llu", (unsigned long long)(b0 + (uint64_t)herr[3]));
  if (herr[2] == 2)
    return fail(MC_ERR_CAPACITY, "record %llu is longer than the contiguous-range scan supports (<= %llu bp)",
                (unsigned long long)(b0 + (uint64_t)herr[3]), (unsigned long long)(kRankGap - 2) * db->sc.stride);
  if (herr[0])
    return fail(MC_ERR_CAPACITY, "record %llu hits more than %u distinct 4-window blocks (or has more than %u windows) in one partition",
                (unsigned long long)(b0 + (uint64_t)herr[1]), kLargeH, kLargeW);
  return MC_OK;
}

// Batches of read_batch records, pipelined: host reads of batch b+1 are copied
// on the copy stream (double-buffered staging) while batch b computes on the
// main stream; results go back with asynchronous copies; each batch's status
// lands in pinned memory and is checked one batch later (no per-batch stall).
static int query_impl(mc_db* db, uint64_t n, const char* reads, const uint64_t* ro, const char* mates,
                      const uint64_t* mo, mc_hit* out_hits, uint32_t* out_taxon, mc_candidate* out_cand) {
  if (!db) return fail(MC_ERR_INVALID_ARG, "db is NULL");
  if (db->state != 1) return fail(MC_ERR_STATE, "database is not finalized");
  if (n == 0) return MC_OK;
  CK(cudaSetDevice(db->device));
  ReadSide s1, s2;
  TRY(check_reads(db, n, reads, ro, mates, mo, s1, s2));
  const uint32_t m = db->cfg.max_candidates;
  const bool dev_hits = out_hits && is_device_ptr(out_hits);
  const bool dev_tax = out_taxon && is_device_ptr(out_taxon);
  const bool dev_cand = out_cand && is_device_ptr(out_cand);
  // device-resident reads and offsets have no copies to overlap: they run in
  // batches of 2^19 .. 2^20 records -- at least two when there are more than
  // 2^19, so the two compute streams overlap one batch's kernels (the small
  // bin's issue-bound gather) with the next one's (the sketch / probe); the
  // subset's 1M pairs: 11.72 ms as one batch, 11.29 ms as two (r02s).  Host
  // inputs use read_batch so copies overlap compute.
  const bool all_dev = s1.on_device() && (!mates || s2.on_device());
  const uint64_t dev_b = n <= (1ull << 19) ? n : std::min<uint64_t>(1ull << 20, std::max<uint64_t>(1ull << 19, (n + 1) / 2));
  const uint64_t B = std::min<uint64_t>(all_dev ? std::max<uint64_t>(db->cfg.read_batch, dev_b) : db->cfg.read_batch, n);
  // batch boundaries: host inputs ramp up (B/8, B/4, B/2, then B), so the
  // first copy -- the one nothing overlaps -- is short and the GPU starts early
  std::vector<uint64_t> bnd{0};
  // (ramp of 3 steps: 13.56 ms on the subset e2e, 2 steps 13.87, 4 steps 13.82, a single B/4: 13.82)
  if (!all_dev && n > B)
    for (int r = 3; r >= 1 && bnd.back() < n; --r) bnd.push_back(std::min(n, bnd.back() + std::max<uint64_t>(B >> r, 1)));
  while (bnd.back() < n) bnd.push_back(std::min(n, bnd.back() + B));
  const uint64_t nbat = bnd.size() - 1;
  cudaStream_t st = db->stream, cs = db->copy_stream;
  // batch bi computes on stream cst[bi & 1]: the second stream starts after
  // everything queued on the caller's stream so far, and the caller's stream
  // waits for it before the call returns
  const cudaStream_t cst[2] = {st, nbat > 1 ? db->own2 : st};
  const bool host_offs = s1.offs != nullptr;
  CK(cudaMemsetAsync(db->qstats.p, 0, 16 * sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(db->err.p, 0, 12 * sizeof(int), st));
  if (cst[1] != st) {
    CK(cudaEventRecord(db->fork_ev, st));
    CK(cudaStreamWaitEvent(cst[1], db->fork_ev, 0));
  }
  // staging of one side of batch b into slot k (copy stream for host bytes)
  auto stage = [&](const char* data, const uint64_t* offs_user, const ReadSide& sd, uint64_t b0, uint64_t b1, int k,
                   DevBuf<uint8_t>* bufs, DevBuf<uint64_t>* obufs, const uint8_t** dptr, const uint64_t** doff,
                   uint64_t* base) -> int {
    if (!sd.offs) {  // device reads + device offsets: offsets index the caller's buffer directly
      *base = 0;
      *dptr = reinterpret_cast<const uint8_t*>(data);
      *doff = offs_user + b0;
      return MC_OK;
    }
    const uint64_t lo = sd.offs[b0], bytes = sd.offs[b1] - lo;
    *base = lo;
    if (sd.dev) {
      *dptr = reinterpret_cast<const uint8_t*>(data) + lo;
    } else {
      CK(cudaMemcpyAsync(bufs[k].p, data + lo, bytes, cudaMemcpyHostToDevice, cs));
      CK(cudaMemsetAsync(bufs[k].p + bytes, 'N', 64, cs));  // defined padding after the batch (aligned-word reads)
      *dptr = bufs[k].p;
    }
    if (is_device_ptr(offs_user)) {
      *doff = offs_user + b0;
    } else {
      CK(cudaMemcpyAsync(obufs[k].p, sd.offs + b0, (b1 - b0 + 1) * 8, cudaMemcpyHostToDevice, cs));
      *doff = obufs[k].p;
    }
    return MC_OK;
  };
  // size both staging slots for the largest batch before anything is in flight
  if (host_offs) {
    uint64_t mx1 = 0, mx2 = 0;
    for (uint64_t bi = 0; bi < nbat; ++bi) {
      const uint64_t b0 = bnd[bi], b1 = bnd[bi + 1];
      if (s1.offs[b1] < s1.offs[b0] || (mates && s2.offs[b1] < s2.offs[b0]))
        return fail(MC_ERR_INVALID_ARG, "read offsets decrease within records [%llu, %llu)", (unsigned long long)b0,
                    (unsigned long long)b1);
      mx1 = std::max(mx1, s1.offs[b1] - s1.offs[b0]);
      if (mates) mx2 = std::max(mx2, s2.offs[b1] - s2.offs[b0]);
    }
    for (int k = 0; k < 3; ++k) {
      if (!s1.dev) TRY(db->qbuf1[k].ensure(mx1 + 64));
      if (mates && !s2.dev) TRY(db->qbuf2[k].ensure(mx2 + 64));
      if (!is_device_ptr(ro)) TRY(db->qoff1[k].ensure(B + 1));
      if (mates && !is_device_ptr(mo)) TRY(db->qoff2[k].ensure(B + 1));
    }
  }
  std::vector<ReadBatch> rbs(nbat);
  // MC_TRACE=1: per-batch timeline of the copy / compute / result streams (stderr)
  static const bool trace = getenv("MC_TRACE") != nullptr;
  std::vector<std::pair<std::string, cudaEvent_t>> tr;
  auto mark = [&](const char* what, uint64_t bi, cudaStream_t s) {
    if (!trace) return;
    cudaEvent_t e = db->ev();  // (timing events from the handle's pool)
    cudaEventRecord(e, s);
    tr.push_back({std::string(what) + " " + std::to_string(bi), e});
  };
  struct TraceDump {
    mc_db* db;
    std::vector<std::pair<std::string, cudaEvent_t>>& tr;
    ~TraceDump() {
      if (tr.empty()) return;
      for (cudaStream_t s : {db->copy_stream, db->stream, db->d2h_stream}) cudaStreamSynchronize(s);
      std::string out = "{\"mc_trace_ms\": {";
      for (size_t i = 0; i < tr.size(); ++i) {
        float ms = -1;
        const cudaError_t e = cudaEventElapsedTime(&ms, tr[0].second, tr[i].second);
        char b[160];
        snprintf(b, sizeof b, "%s\"%s\": %.3f%s", i ? ", " : "", tr[i].first.c_str(), ms,
                 e == cudaSuccess ? "" : cudaGetErrorString(e));
        out += b;
        db->event_pool.push_back(tr[i].second);
      }
      cudaGetLastError();
      fprintf(stderr, "%s}}\n", out.c_str());
    }
  } trace_dump{db, tr};
  mark("call", 0, st);
  auto issue_copy = [&](uint64_t bi) -> int {
    const int k = (int)(bi % 3);  // staging slot
    const uint64_t b0 = bnd[bi], b1 = bnd[bi + 1];
    ReadBatch& rb = rbs[bi];
    rb.n = b1 - b0;
    CK(cudaStreamWaitEvent(cs, db->stage_free[k], 0));  // slot k's previous batch is done with it
    mark("h2d_start", bi, cs);
    TRY(stage(reads, ro, s1, b0, b1, k, db->qbuf1, db->qoff1, &rb.r1, &rb.o1, &rb.base1));
    if (mates) TRY(stage(mates, mo, s2, b0, b1, k, db->qbuf2, db->qoff2, &rb.r2, &rb.o2, &rb.base2));
    mark("h2d_end", bi, cs);
    CK(cudaEventRecord(db->stage_ready[k], cs));
    return MC_OK;
  };
  // whatever way the call ends, no copy into the caller's buffers is still in flight
  struct StreamsIdle {
    mc_db* db;
    ~StreamsIdle() {
      cudaStreamSynchronize(db->d2h_stream);
      cudaStreamSynchronize(db->copy_stream);
      cudaStreamSynchronize(db->own2);
      cudaStreamSynchronize(db->stream);
    }
  } idle{db};
  // the first use of the staging / output events in this call must not wait on stale records
  for (int k = 0; k < 3; ++k) CK(cudaEventRecord(db->stage_free[k], st));
  for (int k = 0; k < 2; ++k) CK(cudaEventRecord(db->out_free[k], db->d2h_stream));
  db->begin("h2d_reads");
  TRY(issue_copy(0));
  db->end();
  for (uint64_t bi = 0; bi < nbat; ++bi) {
    const int k = (int)(bi & 1);
    const uint64_t b0 = bnd[bi], b1 = bnd[bi + 1], nb = b1 - b0;
    const int ks = (int)(bi % 3);    // (this batch's staging slot)
    const cudaStream_t st = cst[k];  // (this batch's compute stream)
    CK(cudaStreamWaitEvent(st, db->stage_ready[ks], 0));
    // host offsets: an O(1) upper bound of the batch's windows (windows(L) <= L / stride + 1)
    // sizes the launch; the sketch kernel clamps to the exact device-side total
    uint64_t W = UINT64_MAX;
    if (host_offs) {
      W = (s1.offs[b1] - s1.offs[b0]) / db->sc.stride + nb;
      if (mates) W += (s2.offs[b1] - s2.offs[b0]) / db->sc.stride + nb;
    }
    HitRec* hits;
    const size_t nh = nb * db->n_local * m;
    const bool host_hits = out_hits && !dev_hits;
    const bool host_res = out_taxon && (!dev_tax || (out_cand && !dev_cand));
    if (host_hits) CK(cudaStreamWaitEvent(st, db->out_free[k], 0));  // slot k's hits have left (D2H of batch bi-2)
    if (dev_hits) {
      hits = reinterpret_cast<HitRec*>(out_hits) + b0 * db->n_local * m;
    } else if (host_hits) {
      TRY(db->ohits[k].ensure(nh));
      hits = db->ohits[k].p;
    } else {
      TRY(db->qs[k].hits.ensure(nh));
      hits = db->qs[k].hits.p;
    }
    int* err = db->err.p + 4 * ks;  // (status slot bi % 3: checked two batches later)
    mark("compute_start", bi, st);
    TRY(run_partials(db, rbs[bi], hits, W, err, k, st));
    mark("partials_end", bi, st);
    CK(cudaEventRecord(db->stage_free[ks], st));  // staging slot ks's input is consumed
    if (bi + 1 < nbat) TRY(issue_copy(bi + 1));   // overlaps this batch's compute
    if (host_hits) {
      CK(cudaEventRecord(db->out_ready[k], st));
      CK(cudaStreamWaitEvent(db->d2h_stream, db->out_ready[k], 0));
      CK(cudaMemcpyAsync(out_hits + b0 * db->n_local * m, hits, nh * sizeof(HitRec), cudaMemcpyDeviceToHost,
                         db->d2h_stream));
      CK(cudaEventRecord(db->out_free[k], db->d2h_stream));
    }
    if (out_taxon) {
      uint32_t* tx = dev_tax ? out_taxon + b0 : nullptr;
      uint32_t* cd = dev_cand ? reinterpret_cast<uint32_t*>(out_cand + b0 * m) : nullptr;
      if (!tx) {
        TRY(db->otx[k].ensure(B));
        tx = db->otx[k].p;
      }
      if (out_cand && !cd) {
        TRY(db->ocd[k].ensure(B * m * 4));
        cd = db->ocd[k].p;
      }
      MergeArgs ma{hits, nb, db->n_local, m, db->cfg.hits_min, db->cfg.hits_diff, db->anc.p, db->depth.p,
                   db->maxd, db->n_taxa, tx, cd, err};
      // only the merge writes slot k's outputs: it (not the scoring) waits for their D2H of batch bi-2
      if (host_res) CK(cudaStreamWaitEvent(st, db->out_free[k], 0));
      db->begin("merge_classify", st);
      launch_merge_classify(ma, st);
      db->end(st);
      db->launched("k_merge_classify");
      if (host_res) {
        CK(cudaEventRecord(db->out_ready[k], st));
        CK(cudaStreamWaitEvent(db->d2h_stream, db->out_ready[k], 0));
        if (!dev_tax) CK(cudaMemcpyAsync(out_taxon + b0, tx, nb * 4, cudaMemcpyDeviceToHost, db->d2h_stream));
        if (out_cand && !dev_cand)
          CK(cudaMemcpyAsync(out_cand + b0 * m, cd, nb * m * sizeof(mc_candidate), cudaMemcpyDeviceToHost,
                             db->d2h_stream));
        mark("d2h_end", bi, db->d2h_stream);
        CK(cudaEventRecord(db->out_free[k], db->d2h_stream));
      }
    }
    // the batch's status words follow its results on the result stream (a D2H
    // copy on the compute stream would queue behind the results' copies on the
    // copy engine and hold up the next batch)
    CK(cudaEventRecord(db->out_ready[k], st));
    CK(cudaStreamWaitEvent(db->d2h_stream, db->out_ready[k], 0));
    CK(cudaMemcpyAsync(db->herr_pin + 4 * ks, err, 4 * sizeof(int), cudaMemcpyDeviceToHost, db->d2h_stream));
    CK(cudaEventRecord(db->qstat_ev[ks], db->d2h_stream));
    if (bi >= 2) {  // status of batch bi - 2: the host stays two batches ahead of the GPU
      const int kp = (int)((bi - 2) % 3);
      CK(cudaEventSynchronize(db->qstat_ev[kp]));
      TRY(batch_status(db, db->herr_pin + 4 * kp, bnd[bi - 2]));
    }
  }
  if (cst[1] != st) {  // the caller's stream joins the second compute stream
    ++db->st_qoverlap;
    CK(cudaEventRecord(db->join_ev, cst[1]));
    CK(cudaStreamWaitEvent(st, db->join_ev, 0));
  }
  CK(cudaStreamSynchronize(db->d2h_stream));  // every result copy has landed
  TRY(db->sync());
  for (uint64_t bi = nbat >= 2 ? nbat - 2 : 0; bi < nbat; ++bi)  // the last two batches' status
    TRY(batch_status(db, db->herr_pin + 4 * (bi % 3), bnd[bi]));
  unsigned long long qs[16];
  CK(cudaMemcpy(qs, db->qstats.p, sizeof qs, cudaMemcpyDeviceToHost));
  db->st_qfeat += qs[0];
  db->st_qfeat_hit += qs[8];
  db->st_qloc += qs[1];
  for (int b = 0; b < 3; ++b) db->st_qloc_bin[b] += qs[3 + b];
  db->st_qmed += qs[6];
  db->st_qlarge += qs[7];
  db->st_reads += n;
  db->st_read_bp += qs[2];
  return MC_OK;
}

static int group_query(mc_db* grp, uint64_t n, const char* reads, const uint64_t* ro, const char* mates,
                       const uint64_t* mo, mc_hit* out_hits, uint32_t* out_taxon, mc_candidate* out_cand);

int mc_classify(mc_db* db, uint64_t n_reads, const char* reads, const uint64_t* read_offsets, const char* mates,
                const uint64_t* mate_offsets, uint32_t* out_taxon, mc_candidate* out_candidates) {
  if (!db) return fail(MC_ERR_INVALID_ARG, "db is NULL");
  if (!out_taxon && n_reads) return fail(MC_ERR_INVALID_ARG, "out_taxon is NULL");
  if (!db->shards.empty())
    return no_throw([&] {
      return group_query(db, n_reads, reads, read_offsets, mates, mate_offsets, nullptr, out_taxon, out_candidates);
    });
  if (db->n_local != db->cfg.n_partitions)
    return fail(MC_ERR_STATE, "mc_classify needs all partitions in one handle; use mc_query_partials + mc_merge_classify");
  if (!out_taxon && n_reads) return fail(MC_ERR_INVALID_ARG, "out_taxon is NULL");
  return query_impl(db, n_reads, reads, read_offsets, mates, mate_offsets, nullptr, out_taxon, out_candidates);
}

int mc_query_partials(mc_db* db, uint64_t n_reads, const char* reads, const uint64_t* read_offsets, const char* mates,
                      const uint64_t* mate_offsets, mc_hit* out_hits) {
  if (!db) return fail(MC_ERR_INVALID_ARG, "db is NULL");
  if (!out_hits && n_reads) return fail(MC_ERR_INVALID_ARG, "out_hits is NULL");
  if (!db->shards.empty())
    return no_throw([&] {
      return group_query(db, n_reads, reads, read_offsets, mates, mate_offsets, out_hits, nullptr, nullptr);
    });
  return query_impl(db, n_reads, reads, read_offsets, mates, mate_offsets, out_hits, nullptr, nullptr);
}

int mc_merge_classify(mc_db* db, uint64_t n, uint32_t n_lists, const mc_hit* hits, uint32_t* out_taxon,
                      mc_candidate* out_cand) {
  if (!db) return fail(MC_ERR_INVALID_ARG, "db is NULL");
  if (!db->shards.empty()) return mc_merge_classify(db->shards[0], n, n_lists, hits, out_taxon, out_cand);
  if (n == 0) return MC_OK;
  if (!hits || !out_taxon) return fail(MC_ERR_INVALID_ARG, "NULL hits / out_taxon");
  const uint32_t m = db->cfg.max_candidates;
  if (n_lists == 0 || (uint64_t)n_lists * m > 64) return fail(MC_ERR_INVALID_ARG, "n_lists * m must be in [1, 64]");
  CK(cudaSetDevice(db->device));
  cudaStream_t st = db->stream;
  const bool dh = is_device_ptr(hits), dt = is_device_ptr(out_taxon), dc = out_cand && is_device_ptr(out_cand);
  const uint64_t B = db->cfg.read_batch;
  for (uint64_t b0 = 0; b0 < n; b0 += B) {
    const uint64_t nb = std::min(n, b0 + B) - b0;
    const HitRec* h = reinterpret_cast<const HitRec*>(hits) + b0 * n_lists * m;
    if (!dh) {
      TRY(db->hits.ensure(nb * n_lists * m));
      CK(cudaMemcpyAsync(db->hits.p, h, nb * n_lists * m * sizeof(HitRec), cudaMemcpyHostToDevice, st));
      h = db->hits.p;
    }
    uint32_t* tx = dt ? out_taxon + b0 : nullptr;
    uint32_t* cd = dc ? reinterpret_cast<uint32_t*>(out_cand + b0 * m) : nullptr;
    if (!tx) {
      TRY(db->otaxon.ensure(nb));
      tx = db->otaxon.p;
    }
    if (out_cand && !cd) {
      TRY(db->ocand.ensure(nb * m * 4));
      cd = db->ocand.p;
    }
    MergeArgs ma{h, nb, n_lists, m, db->cfg.hits_min, db->cfg.hits_diff, db->anc.p, db->depth.p, db->maxd,
                 db->n_taxa, tx, cd};
    db->begin("merge_classify");
    launch_merge_classify(ma, st);
    db->end();
    db->launched("k_merge_classify");
    if (!dt) CK(cudaMemcpyAsync(out_taxon + b0, tx, nb * 4, cudaMemcpyDeviceToHost, st));
    if (out_cand && !dc) CK(cudaMemcpyAsync(out_cand + b0 * m, cd, nb * m * 16, cudaMemcpyDeviceToHost, st));
    TRY(db->sync());
  }
  return MC_OK;
}

// ---------------------------------------------------------------------------
// diagnostics
// ---------------------------------------------------------------------------
int mc_debug_sketch(const mc_config* cfg, uint32_t n, const char* seqs, const uint64_t* offsets,
                    uint32_t* out_features, uint32_t* out_counts, uint64_t* out_window_offsets) {
  TRY(validate_cfg(cfg));
  if (!offsets || !out_window_offsets || (n && !seqs)) return fail(MC_ERR_INVALID_ARG, "NULL argument");
  int dev;
  TRY(select_device(cfg, &dev));
  const SketchCfg sc = make_sketch_cfg(cfg->k, cfg->sketch_size, cfg->window_len);
  std::vector<uint64_t> offs;
  TRY(to_host(offsets, (size_t)n + 1, offs));
  out_window_offsets[0] = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (offs[i + 1] < offs[i]) return fail(MC_ERR_INVALID_ARG, "offsets decrease");
    out_window_offsets[i + 1] = out_window_offsets[i] + n_windows_host(offs[i + 1] - offs[i], sc.k, sc.stride);
  }
  const uint64_t W = out_window_offsets[n];
  if (!out_features || W == 0) return MC_OK;
  if (!out_counts) return fail(MC_ERR_INVALID_ARG, "out_counts is NULL");
  std::vector<uint32_t> sel;
  for (uint32_t i = 0; i < n; ++i)
    if (out_window_offsets[i + 1] > out_window_offsets[i]) sel.push_back(i);
  const uint32_t nt = (uint32_t)sel.size();
  std::vector<uint64_t> m64(3 * (size_t)nt + 1);
  std::vector<uint32_t> m32(nt, 0);
  for (uint32_t j = 0; j < nt; ++j) {
    m64[j] = out_window_offsets[sel[j]];
    m64[nt + 1 + j] = offs[sel[j]] - offs[0];
    m64[2 * (size_t)nt + 1 + j] = offs[sel[j] + 1] - offs[sel[j]];
  }
  m64[nt] = W;
  DevBuf<uint8_t> chars;
  DevBuf<uint64_t> d64;
  DevBuf<uint32_t> d32, feats, counts;
  const uint64_t bytes = offs[n] - offs[0];
  const uint8_t* dchars;
  cudaStream_t st = cudaStreamPerThread;
  int rc = MC_OK;
  do {
    if (is_device_ptr(seqs)) {
      dchars = reinterpret_cast<const uint8_t*>(seqs) + offs[0];
    } else {
      if ((rc = chars.ensure(bytes + 64)) != MC_OK) break;
      if (cudaMemcpy(chars.p, seqs + offs[0], bytes, cudaMemcpyHostToDevice) != cudaSuccess) { rc = MC_ERR_CUDA; break; }
      cudaMemset(chars.p + bytes, 'N', 64);
      dchars = chars.p;
    }
    if ((rc = d64.ensure(m64.size())) != MC_OK || (rc = d32.ensure(m32.size())) != MC_OK ||
        (rc = feats.ensure(W * sc.s)) != MC_OK || (rc = counts.ensure(W)) != MC_OK)
      break;
    cudaMemcpy(d64.p, m64.data(), m64.size() * 8, cudaMemcpyHostToDevice);
    BuildBatch b{dchars, d64.p, d64.p + nt + 1, d64.p + 2 * (size_t)nt + 1, d32.p, nt, W};
    launch_debug_sketch(b, sc, feats.p, counts.p, num_sms() * 8, st);
    if (cudaStreamSynchronize(st) != cudaSuccess || cudaGetLastError() != cudaSuccess) { rc = MC_ERR_CUDA; break; }
    const bool df = is_device_ptr(out_features), dcn = is_device_ptr(out_counts);
    cudaMemcpy(out_features, feats.p, W * sc.s * 4, df ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost);
    cudaMemcpy(out_counts, counts.p, W * 4, dcn ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost);
  } while (0);
  chars.release();
  d64.release();
  d32.release();
  feats.release();
  counts.release();
  if (rc == MC_ERR_CUDA) return fail(rc, "debug sketch failed: %s", cudaGetErrorString(cudaGetLastError()));
  return rc;
}

int mc_db_partition_of(const mc_db* db, uint32_t target_id, uint32_t* out) {
  if (!db || !out) return fail(MC_ERR_INVALID_ARG, "NULL argument");
  const auto* it = db->where.find(target_id);
  if (!it) return fail(MC_ERR_INVALID_ARG, "unknown target id %u", target_id);
  if (!db->shards.empty()) {  // (a group's registry holds global partitions)
    *out = it->first;
    return MC_OK;
  }
  *out = db->parts[it->first].gid;
  return MC_OK;
}

// the shard of a multi-GPU handle holding global partition gid (db itself otherwise)
static const mc_db* shard_of(const mc_db* db, uint32_t gid) {
  if (db->shards.empty() || gid >= db->cfg.n_partitions) return db;
  return db->shards[gid / (db->cfg.n_partitions / (uint32_t)db->shards.size())];
}

static int part_of_gid(const mc_db* db, uint32_t gid, const Part** p) {
  if (gid < db->pbegin || gid >= db->pbegin + db->n_local) return fail(MC_ERR_INVALID_ARG, "partition %u not held here", gid);
  *p = &db->parts[gid - db->pbegin];
  return MC_OK;
}

static uint64_t ranked_to_location(const Part& p, uint32_t rwi) {
  const uint32_t r = (uint32_t)(std::upper_bound(p.rank_base_h.begin(), p.rank_base_h.end() - 1, rwi) -
                                p.rank_base_h.begin()) - 1;
  return ((uint64_t)p.tgt_by_rank_h[r] << 32) | (uint64_t)(rwi - p.rank_base_h[r]);
}

// finalized partition on the host: (key, count, offset) of every primary + values
struct HostEntry {
  uint32_t key, cnt;
  uint64_t off;
};
static int download_part(const mc_db* db, const Part& p, std::vector<HostEntry>& E, std::vector<uint32_t>& V) {
  std::vector<KSlot> T(p.nslots);
  std::vector<unsigned long long> vb(p.nslots >> kSubLg);
  CK(cudaMemcpy(T.data(), p.T, p.nslots * sizeof(KSlot), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(vb.data(), p.vbase.p, vb.size() * 8, cudaMemcpyDeviceToHost));
  V.resize(p.n_value_slots);
  if (p.n_value_slots) CK(cudaMemcpy(V.data(), p.values.p, p.n_value_slots * 4, cudaMemcpyDeviceToHost));
  E.clear();
  for (uint64_t i = 0; i < p.nslots; ++i) {
    const unsigned long long w = T[i].kc;
    if (!slot_cnt(w)) continue;
    const uint64_t off = vb[i >> kSubLg] + slot_loff(w);
    E.push_back({slot_key(w), slot_cnt(w), off});
    std::sort(V.begin() + off, V.begin() + off + slot_cnt(w));  // buckets are unordered on the GPU
  }
  std::sort(E.begin(), E.end(), [](const HostEntry& a, const HostEntry& b) { return a.key < b.key; });
  return MC_OK;
}

int mc_db_feature_locations(const mc_db* cdb, uint32_t partition, uint32_t feature, uint64_t* out, uint32_t cap,
                            uint32_t* out_n) {
  if (!cdb || !out_n || (cap && !out)) return fail(MC_ERR_INVALID_ARG, "NULL argument");
  mc_db* db = const_cast<mc_db*>(shard_of(cdb, partition));
  if (db->state != 1) return fail(MC_ERR_STATE, "database is not finalized");
  const Part* p;
  TRY(part_of_gid(db, partition, &p));
  CK(cudaSetDevice(db->device));
  // one key: device-side probe, then only its bucket comes to the host
  TRY(db->meta64.ensure(2));
  const PartView pv{p->T, p->vbase.p, p->nslots, p->values.p, p->rank_base.p, p->tgt_id.p, p->taxon_rank.p,
                    (uint32_t)p->tid.size(), p->coarse.p};
  launch_key_lookup(pv, feature, reinterpret_cast<unsigned long long*>(db->meta64.p), db->stream);
  unsigned long long r[2];
  CK(cudaMemcpyAsync(r, db->meta64.p, sizeof r, cudaMemcpyDeviceToHost, db->stream));
  TRY(db->sync());
  *out_n = (uint32_t)r[0];
  if (r[0] && cap) {
    std::vector<uint32_t> V(r[0]);
    CK(cudaMemcpy(V.data(), p->values.p + r[1], r[0] * 4, cudaMemcpyDeviceToHost));
    std::sort(V.begin(), V.end());  // buckets are unordered on the GPU
    for (uint32_t i = 0; i < r[0] && i < cap; ++i) out[i] = ranked_to_location(*p, V[i]);
  }
  return MC_OK;
}

int mc_db_dump_partition(const mc_db* db, uint32_t partition, uint32_t* keys, uint32_t* counts, uint64_t* values,
                         uint64_t* n_keys, uint64_t* n_values) {
  if (!db || !n_keys || !n_values) return fail(MC_ERR_INVALID_ARG, "NULL argument");
  db = shard_of(db, partition);
  if (db->state != 1) return fail(MC_ERR_STATE, "database is not finalized");
  const Part* p;
  TRY(part_of_gid(db, partition, &p));
  *n_keys = p->n_keys;
  *n_values = p->n_values;
  if (!keys && !counts && !values) return MC_OK;
  CK(cudaSetDevice(db->device));
  std::vector<HostEntry> E;
  std::vector<uint32_t> V;
  TRY(download_part(db, *p, E, V));
  uint64_t nv = 0;
  for (size_t i = 0; i < E.size(); ++i) {
    if (keys) keys[i] = E[i].key;
    if (counts) counts[i] = E[i].cnt;
    if (values)
      for (uint32_t j = 0; j < E[i].cnt; ++j) values[nv + j] = ranked_to_location(*p, V[E[i].off + j]);
    nv += E[i].cnt;
  }
  return MC_OK;
}

int mc_db_reset_stats(mc_db* db) {
  if (!db) return fail(MC_ERR_INVALID_ARG, "db is NULL");
  for (mc_db* sh : db->shards) TRY(mc_db_reset_stats(sh));
  if (!db->shards.empty()) return MC_OK;
  TRY(db->sync());
  db->stage_ms.clear();
  db->launches.clear();
  db->st_bp = db->st_windows = db->st_locations = db->st_reads = db->st_qfeat = db->st_qloc = db->st_read_bp = 0;
  db->st_qfeat_hit = 0;
  db->st_qoverlap = 0;
  db->st_qmed = db->st_qlarge = 0;
  db->st_qloc_bin[0] = db->st_qloc_bin[1] = db->st_qloc_bin[2] = 0;
  return MC_OK;
}

int mc_db_stats(const mc_db* cdb, char* out, uint64_t len) {
  mc_db* db = const_cast<mc_db*>(cdb);
  if (!db || !out) return fail(MC_ERR_INVALID_ARG, "NULL argument");
  // a multi-GPU handle reports its shards' sums (build counters, launches),
  // shard 0's query counters (every shard scores every record) and per stage
  // the maximum over shards (they run concurrently) + each shard's stage times
  std::vector<mc_db*> all = db->shards.empty() ? std::vector<mc_db*>{db} : db->shards;
  uint64_t bp = 0, win = 0, locs = 0;
  std::map<std::string, double> stage;
  std::map<std::string, uint64_t> launches;
  for (mc_db* d : all) {
    CK(cudaSetDevice(d->device));
    TRY(d->sync());
    bp += d->st_bp;
    win += d->st_windows;
    locs += d->st_locations;
    for (auto& kv : d->stage_ms) stage[kv.first] = std::max(stage[kv.first], kv.second);
    for (auto& kv : d->launches) launches[kv.first] += kv.second;
  }
  const mc_db* q = all[0];
  std::string s = "{";
  char b[1024];
  snprintf(b, sizeof b,
           "\"state\": %d, \"n_gpus\": %zu, \"bp\": %llu, \"windows\": %llu, \"locations_inserted\": %llu, \"reads\": %llu, "
           "\"read_bp\": %llu, \"query_features\": %llu, \"query_locations\": %llu, \"sms\": %d, "
           "\"query_medium_bin\": %llu, \"query_large_bin\": %llu, \"query_locations_by_bin\": [%llu, %llu, %llu], "
           "\"query_features_found\": %llu, \"query_overlapped_calls\": %llu, ",
           db->state, all.size(), (unsigned long long)bp, (unsigned long long)win, (unsigned long long)locs,
           (unsigned long long)q->st_reads, (unsigned long long)q->st_read_bp, (unsigned long long)q->st_qfeat,
           (unsigned long long)q->st_qloc, q->sms, (unsigned long long)q->st_qmed, (unsigned long long)q->st_qlarge,
           (unsigned long long)q->st_qloc_bin[0], (unsigned long long)q->st_qloc_bin[1],
           (unsigned long long)q->st_qloc_bin[2], (unsigned long long)q->st_qfeat_hit,
           (unsigned long long)q->st_qoverlap);
  s += b;
  s += "\"partitions\": [";
  bool first = true;
  for (mc_db* d : all)
    for (size_t i = 0; i < d->parts.size(); ++i) {
      const Part& p = d->parts[i];
      snprintf(b, sizeof b,
               "%s{\"partition\": %u, \"device\": %d, \"targets\": %zu, \"bp\": %llu, \"windows\": %llu, "
               "\"table_slots\": %llu, \"table_bytes\": %llu, \"keys\": %llu, \"locations\": %llu, \"values\": %llu, "
               "\"truncated\": %llu}",
               first ? "" : ", ", p.gid, d->device, p.tid.size(), (unsigned long long)p.bp, (unsigned long long)p.windows,
               (unsigned long long)p.nslots, (unsigned long long)(p.nslots * sizeof(KSlot)),
               (unsigned long long)p.n_keys, (unsigned long long)p.n_locations, (unsigned long long)p.n_values,
               (unsigned long long)p.truncated);
      s += b;
      first = false;
    }
  auto put_map = [&](const char* name, const std::map<std::string, double>& mp) {
    s += std::string(", \"") + name + "\": {";
    bool f = true;
    for (auto& kv : mp) {
      snprintf(b, sizeof b, "%s\"%s\": %.6f", f ? "" : ", ", kv.first.c_str(), kv.second);
      s += b;
      f = false;
    }
    s += "}";
  };
  s += "]";
  put_map("stage_ms", stage);
  s += ", \"launches\": {";
  first = true;
  for (auto& kv : launches) {
    snprintf(b, sizeof b, "%s\"%s\": %llu", first ? "" : ", ", kv.first.c_str(), (unsigned long long)kv.second);
    s += b;
    first = false;
  }
  s += "}";
  if (!db->shards.empty()) {
    s += ", \"shard_stage_ms\": [";
    for (size_t g = 0; g < all.size(); ++g) {
      if (g) s += ", ";
      std::string one;
      std::swap(one, s);
      put_map("x", all[g]->stage_ms);
      std::swap(one, s);
      s += one.substr(one.find('{'));
    }
    s += "]";
  }
  s += "}";
  if (s.size() + 1 > len) return fail(MC_ERR_INVALID_ARG, "stats buffer too small (%zu bytes needed)", s.size() + 1);
  std::memcpy(out, s.c_str(), s.size() + 1);
  return MC_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// condensed dump / load
// ---------------------------------------------------------------------------
namespace {
constexpr char kMagic[8] = {'M', 'C', 'D', 'B', 0, 0, 0, 2};
constexpr uint64_t kIoChunk = 64ull << 20;

struct File {
  FILE* f = nullptr;
  bool ok = true;
  uint64_t size = 0;  // bytes in the file (reads: array counts are checked against what is left)
  uint64_t left() {
    const long pos = ftell(f);
    return pos < 0 || (uint64_t)pos > size ? 0 : size - (uint64_t)pos;
  }
  ~File() {
    if (f) fclose(f);
  }
  void put(const void* p, size_t n) { ok = ok && (n == 0 || fwrite(p, 1, n, f) == n); }
  void get(void* p, size_t n) { ok = ok && (n == 0 || fread(p, 1, n, f) == n); }
  template <class T> void put_v(const std::vector<T>& v) {
    const uint64_t n = v.size();
    put(&n, 8);
    put(v.data(), n * sizeof(T));
  }
  template <class T> void get_v(std::vector<T>& v, uint64_t max_n) {
    uint64_t n = 0;
    get(&n, 8);
    if (!ok || n > max_n || n > left() / sizeof(T)) { ok = false; return; }  // corrupt / truncated count
    v.resize(n);
    get(v.data(), n * sizeof(T));
  }
};

// device array <-> file through a host chunk
int dev_to_file(File& F, const void* d, uint64_t bytes) {
  F.put(&bytes, 8);
  std::vector<uint8_t> h(std::min(bytes, kIoChunk));
  for (uint64_t o = 0; o < bytes && F.ok; o += kIoChunk) {
    const uint64_t n = std::min(kIoChunk, bytes - o);
    CK(cudaMemcpy(h.data(), static_cast<const uint8_t*>(d) + o, n, cudaMemcpyDeviceToHost));
    F.put(h.data(), n);
  }
  return F.ok ? MC_OK : fail(MC_ERR_INVALID_ARG, "write failed");
}
int file_to_dev(File& F, void* d, uint64_t expect) {
  uint64_t bytes = 0;
  F.get(&bytes, 8);
  if (!F.ok || bytes != expect || bytes > F.left()) return fail(MC_ERR_INVALID_ARG, "database file: bad array size");
  std::vector<uint8_t> h(std::min(bytes, kIoChunk));
  for (uint64_t o = 0; o < bytes && F.ok; o += kIoChunk) {
    const uint64_t n = std::min(kIoChunk, bytes - o);
    F.get(h.data(), n);
    if (F.ok) CK(cudaMemcpy(static_cast<uint8_t*>(d) + o, h.data(), n, cudaMemcpyHostToDevice));
  }
  return F.ok ? MC_OK : fail(MC_ERR_INVALID_ARG, "database file truncated");
}
}  // namespace

int mc_db_get_config(const mc_db* db, mc_config* out) {
  if (!db || !out) return fail(MC_ERR_INVALID_ARG, "NULL argument");
  *out = db->cfg;
  return MC_OK;
}

static int save_file(const mc_db* cdb, const char* path) {
  mc_db* db = const_cast<mc_db*>(cdb);
  if (!db || !path) return fail(MC_ERR_INVALID_ARG, "NULL argument");
  if (!db->shards.empty()) return fail(MC_ERR_STATE, "mc_db_save: single-device handles only");
  if (db->state != 1) return fail(MC_ERR_STATE, "database is not finalized");
  CK(cudaSetDevice(db->device));
  TRY(db->sync());
  File F;
  F.f = fopen(path, "wb");
  if (!F.f) return fail(MC_ERR_INVALID_ARG, "cannot open %s for writing", path);
  F.put(kMagic, 8);
  const uint64_t csz = sizeof(mc_config);
  F.put(&csz, 8);
  F.put(&db->cfg, csz);
  F.put_v(db->parent_h);
  F.put_v(db->rank_h);
  const uint32_t nl = (uint32_t)db->parts.size();
  F.put(&nl, 4);
  for (const Part& p : db->parts) {
    const uint32_t nt = (uint32_t)p.tid.size();
    F.put(&p.gid, 4);
    F.put_v(p.tid);
    F.put_v(p.taxon);
    F.put_v(p.nwin);
    F.put_v(p.gbase);
    const uint64_t sc[9] = {p.windows, p.bp, p.gwin, p.nslots, p.n_value_slots, p.n_values, p.n_keys,
                            p.n_locations, p.truncated};
    F.put(sc, sizeof sc);
    F.put_v(p.rank_base_h);
    F.put_v(p.tgt_by_rank_h);
    TRY(dev_to_file(F, p.T, p.nslots * sizeof(KSlot)));
    TRY(dev_to_file(F, p.vbase.p, (p.nslots >> kSubLg) * 8));
    TRY(dev_to_file(F, p.values.p, p.n_value_slots * 4));
    TRY(dev_to_file(F, p.taxon_rank.p, (uint64_t)nt * 4));
    const uint64_t ncoarse = ((uint64_t)(p.rank_base_h.empty() ? 0 : p.rank_base_h.back()) >> 10) + 1;
    F.put(&ncoarse, 8);
    TRY(dev_to_file(F, p.coarse.p, ncoarse * sizeof(uint2)));
  }
  if (!F.ok || fflush(F.f) != 0) return fail(MC_ERR_INVALID_ARG, "write to %s failed", path);
  return MC_OK;
}

static int load_impl(mc_db* db, File& F) {
  const uint32_t nl = (uint32_t)db->parts.size();
  uint32_t fnl = 0;
  F.get(&fnl, 4);
  if (!F.ok || fnl != nl) return fail(MC_ERR_INVALID_ARG, "database file: partition count mismatch");
  for (uint32_t q = 0; q < nl; ++q) {
    Part& p = db->parts[q];
    uint32_t gid = 0;
    F.get(&gid, 4);
    if (!F.ok || gid != p.gid) return fail(MC_ERR_INVALID_ARG, "database file: partition id mismatch");
    const uint64_t lim = db->cfg.max_targets ? db->cfg.max_targets + 1 : (1ull << 32);
    F.get_v(p.tid, lim);
    F.get_v(p.taxon, lim);
    F.get_v(p.nwin, lim);
    F.get_v(p.gbase, lim);
    uint64_t sc[9];
    F.get(sc, sizeof sc);
    if (!F.ok) return fail(MC_ERR_INVALID_ARG, "database file truncated");
    const uint32_t nt = (uint32_t)p.tid.size();
    if (p.taxon.size() != nt || p.nwin.size() != nt || p.gbase.size() != nt)
      return fail(MC_ERR_INVALID_ARG, "database file: target tables disagree");
    p.windows = sc[0], p.bp = sc[1], p.gwin = sc[2], p.nslots = sc[3], p.n_value_slots = sc[4];
    p.n_values = sc[5], p.n_keys = sc[6], p.n_locations = sc[7], p.truncated = sc[8];
    if (p.nslots > p.nslots_max || (p.nslots & (kSubSlots - 1)))
      return fail(MC_ERR_INVALID_ARG, "database file: table of %llu slots does not fit this configuration",
                  (unsigned long long)p.nslots);
    F.get_v(p.rank_base_h, (uint64_t)nt + 1);
    F.get_v(p.tgt_by_rank_h, nt);
    if (!F.ok || p.rank_base_h.size() != (uint64_t)nt + 1 || p.tgt_by_rank_h.size() != nt)
      return fail(MC_ERR_INVALID_ARG, "database file: ranked target tables disagree");
    TRY(file_to_dev(F, p.T, p.nslots * sizeof(KSlot)));
    TRY(p.vbase.ensure(std::max<uint64_t>(p.nslots >> kSubLg, 1)));
    TRY(file_to_dev(F, p.vbase.p, (p.nslots >> kSubLg) * 8));
    TRY(p.values.ensure(std::max<uint64_t>(p.n_value_slots, 1)));
    TRY(file_to_dev(F, p.values.p, p.n_value_slots * 4));
    TRY(p.rank_base.ensure(nt + 1));
    CK(cudaMemcpy(p.rank_base.p, p.rank_base_h.data(), ((uint64_t)nt + 1) * 4, cudaMemcpyHostToDevice));
    TRY(p.tgt_id.ensure(std::max(nt, 1u)));
    if (nt) CK(cudaMemcpy(p.tgt_id.p, p.tgt_by_rank_h.data(), (uint64_t)nt * 4, cudaMemcpyHostToDevice));
    TRY(p.taxon_rank.ensure(std::max(nt, 1u)));
    TRY(file_to_dev(F, p.taxon_rank.p, (uint64_t)nt * 4));
    uint64_t ncoarse = 0;
    F.get(&ncoarse, 8);
    if (!F.ok || ncoarse != ((uint64_t)p.rank_base_h.back() >> 10) + 1)
      return fail(MC_ERR_INVALID_ARG, "database file: coarse index size mismatch");
    TRY(p.coarse.ensure(ncoarse));
    TRY(file_to_dev(F, p.coarse.p, ncoarse * sizeof(uint2)));
    for (uint32_t i = 0; i < nt; ++i) {
      if (!db->where.put(p.tid[i], q, i)) return fail(MC_ERR_INVALID_ARG, "database file: duplicate target id");
    }
    db->running_bp[q] = p.bp;
  }
  db->state = 1;
  return db->sync();
}

static int load_file(const char* path, int32_t device, mc_db** out) {
  if (!path || !out) return fail(MC_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  File F;
  F.f = fopen(path, "rb");
  if (!F.f) return fail(MC_ERR_INVALID_ARG, "cannot open %s", path);
  if (fseek(F.f, 0, SEEK_END) == 0) {
    const long sz = ftell(F.f);
    F.size = sz > 0 ? (uint64_t)sz : 0;
  }
  if (fseek(F.f, 0, SEEK_SET) != 0) return fail(MC_ERR_INVALID_ARG, "cannot read %s", path);
  char magic[8];
  uint64_t csz = 0;
  F.get(magic, 8);
  F.get(&csz, 8);
  if (!F.ok || std::memcmp(magic, kMagic, 8) != 0 || csz != sizeof(mc_config))
    return fail(MC_ERR_INVALID_ARG, "%s is not a database file of this version", path);
  mc_config cfg;
  F.get(&cfg, csz);
  std::vector<uint32_t> parent;
  std::vector<uint8_t> rank;
  F.get_v(parent, 1ull << 32);
  F.get_v(rank, 1ull << 32);
  if (!F.ok || parent.size() < 2 || (!rank.empty() && rank.size() != parent.size()))
    return fail(MC_ERR_INVALID_ARG, "database file: bad taxonomy");
  cfg.device = device;
  const mc_taxonomy tax{(uint32_t)parent.size(), parent.data(), rank.empty() ? nullptr : rank.data()};
  mc_db* db = nullptr;
  TRY(mc_db_create(&cfg, &tax, &db));
  const int rc = load_impl(db, F);
  if (rc != MC_OK) {
    const std::string msg = g_err;
    mc_db_destroy(db);
    g_err = msg;
    return rc;
  }
  *out = db;
  return MC_OK;
}

extern "C" {
int mc_db_insert_targets(mc_db* db, uint32_t n, const char* seqs, const uint64_t* offsets, const uint32_t* target_ids,
                         const uint32_t* taxa, const uint32_t* partition_ids) {
  const mc_target_batch b{n, seqs, offsets, target_ids, taxa, partition_ids};
  return no_throw([&] { return insert_batches_impl(db, 1, &b); });
}
int mc_db_insert_target_batches(mc_db* db, uint32_t n_batches, const mc_target_batch* batches) {
  return no_throw([&] { return insert_batches_impl(db, n_batches, batches); });
}
int mc_db_save(const mc_db* db, const char* path) { return no_throw([&] { return save_file(db, path); }); }
int mc_db_load(const char* path, int32_t device, mc_db** out) {
  return no_throw([&] { return load_file(path, device, out); });
}
}  // extern "C"

// ===========================================================================
// Multi-GPU handle (cfg.n_gpus = G > 1): one handle, G single-device shards.
//
// The database is partitioned by target: shard g holds global
// partitions [g P/G, (g+1) P/G) on its own device and builds them with no
// communication.  A query batch is distributed like the paper's read chain
// but as an all-gather over NVLink peer memory: device g copies
// record slice g from the host and pulls the other slices from its peers'
// staging buffers; every device scores all records against its partitions;
// device h then merges + classifies slice h, its merge kernel reading the
// per-partition top-m lists straight from the other devices' memory (the
// paper's GPU-to-GPU merge, fused into one kernel).  Batches are
// double-buffered with cross-device events (the paper's per-GPU batch arenas,
// P:673-679).  Ordinals may repeat: the same code then runs same-device copies.
// ===========================================================================
template <class F>
static int on_shards(mc_db* grp, F&& f) {
  const size_t G = grp->shards.size();
  std::vector<int> rc(G, MC_OK);
  std::vector<std::string> msg(G);
  std::vector<std::thread> th;
  th.reserve(G);
  for (size_t g = 0; g < G; ++g)
    th.emplace_back([&, g] {
      rc[g] = no_throw([&] {
        CK(cudaSetDevice(grp->shards[g]->device));
        return f((uint32_t)g, grp->shards[g]);
      });
      if (rc[g] != MC_OK) msg[g] = g_err;
    });
  for (auto& t : th) t.join();
  for (size_t g = 0; g < G; ++g)
    if (rc[g] != MC_OK) {
      g_err = msg[g];
      return rc[g];
    }
  return MC_OK;
}

static int group_create(const mc_config* cfg, const mc_taxonomy* tax, mc_db* grp) {
  TRY(validate_cfg(cfg));
  const mc_config& c = *cfg;
  const uint32_t G = c.n_gpus, P = c.n_partitions;
  if (G > kMaxGpus) return fail(MC_ERR_INVALID_ARG, "n_gpus=%u exceeds %u", G, kMaxGpus);
  if (P < G || P % G != 0) return fail(MC_ERR_INVALID_ARG, "n_partitions=%u must be a multiple of n_gpus=%u", P, G);
  if (c.partition_begin != 0 || (c.n_local_partitions != 0 && c.n_local_partitions != P))
    return fail(MC_ERR_INVALID_ARG, "a multi-GPU handle holds every partition (partition_begin 0, n_local_partitions 0 or P)");
  if (!tax || !tax->parent || tax->n_taxa < 2) return fail(MC_ERR_INVALID_ARG, "taxonomy needs n_taxa >= 2");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  std::vector<int> dev(G);
  for (uint32_t g = 0; g < G; ++g) {
    dev[g] = c.devices[g] >= 0 ? c.devices[g] : (int)g;
    if (dev[g] >= ndev) return fail(MC_ERR_INVALID_ARG, "shard %u: device %d does not exist (%d visible)", g, dev[g], ndev);
  }
  // peer access between every pair of distinct devices (NVLink / NVSwitch)
  for (uint32_t a = 0; a < G; ++a)
    for (uint32_t b = 0; b < G; ++b) {
      if (dev[a] == dev[b]) continue;
      int ok = 0;
      CK(cudaDeviceCanAccessPeer(&ok, dev[a], dev[b]));
      if (!ok) return fail(MC_ERR_PEER, "device %d cannot access device %d's memory (no peer path)", dev[a], dev[b]);
      CK(cudaSetDevice(dev[a]));
      const cudaError_t e = cudaDeviceEnablePeerAccess(dev[b], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(MC_ERR_PEER, "enabling peer access %d -> %d: %s", dev[a], dev[b], cudaGetErrorString(e));
      }
    }
  grp->cfg = c;
  grp->cfg.n_local_partitions = P;
  if (grp->cfg.read_batch == 0) grp->cfg.read_batch = 1ull << 20;
  grp->sc = make_sketch_cfg(c.k, c.sketch_size, c.window_len);
  grp->pbegin = 0;
  grp->n_local = P;
  grp->device = dev[0];
  grp->running_bp.assign(P, 0);
  const uint32_t Pg = P / G;
  for (uint32_t g = 0; g < G; ++g) {
    mc_config cg = c;
    cg.n_gpus = 1;
    cg.device = dev[g];
    cg.partition_begin = g * Pg;
    cg.n_local_partitions = Pg;
    // the shard's share of the static allocation, + 1/8 for the S9 imbalance
    cg.capacity_bp = c.capacity_bp / G + c.capacity_bp / (8 * G) + (64ull << 20);
    if (c.max_targets) cg.max_targets = c.max_targets / G + c.max_targets / 8 + 64;
    mc_db* sh = new mc_db();
    grp->shards.push_back(sh);
    TRY(create_impl(&cg, tax, sh));
  }
  grp->n_taxa = grp->shards[0]->n_taxa;
  grp->sms = grp->shards[0]->sms;
  return MC_OK;
}

static int group_insert(mc_db* grp, const std::vector<TargetIn>& in) {
  const uint32_t G = (uint32_t)grp->shards.size(), P = grp->cfg.n_partitions, Pg = P / G;
  for (auto& t : in)
    if (t.dev) {
      const int d = ptr_device(t.seqs);
      bool ok = false;
      for (mc_db* sh : grp->shards) ok |= sh->device == d;
      if (!ok) return fail(MC_ERR_INVALID_ARG, "device-resident targets must be on one of the handle's devices");
    }
  std::vector<uint64_t> run = grp->running_bp;
  std::vector<std::vector<uint32_t>> part(in.size());
  std::vector<std::vector<std::vector<uint32_t>>> sel(in.size(), std::vector<std::vector<uint32_t>>(G)),
      loc(in.size(), std::vector<std::vector<uint32_t>>(G));
  for (size_t x = 0; x < in.size(); ++x) {
    TRY(assign_partitions(in[x], 0, P, run, part[x]));
    for (uint32_t i = 0; i < in[x].n; ++i) {
      const uint32_t g = part[x][i] / Pg;
      sel[x][g].push_back(i);
      loc[x][g].push_back(part[x][i] - g * Pg);
    }
  }
  // every device sketches its partitions' targets of all batches, concurrently
  const int rc = on_shards(grp, [&](uint32_t g, mc_db* sh) {
    for (size_t x = 0; x < in.size(); ++x)
      TRY(shard_insert(sh, in[x].seqs, in[x].dev, in[x].offs.data(), in[x].ids.data(), in[x].tx.data(), sel[x][g],
                       loc[x][g]));
    return MC_OK;
  });
  if (rc != MC_OK) {
    grp->state = -1;  // some shards may hold their share: the handle is broken
    return rc;
  }
  grp->running_bp = run;
  size_t tot = 0;
  for (auto& t : in) tot += t.n;
  grp->where.reserve(tot);
  for (size_t x = 0; x < in.size(); ++x)
    for (uint32_t i = 0; i < in[x].n; ++i) grp->where.put(in[x].ids[i], part[x][i], 0);
  return MC_OK;
}

static int group_finalize(mc_db* grp) {
  const int rc = on_shards(grp, [&](uint32_t, mc_db* sh) { return mc_db_finalize(sh); });
  grp->state = rc == MC_OK ? 1 : -1;
  return rc;
}

static int group_query(mc_db* grp, uint64_t n, const char* reads, const uint64_t* ro, const char* mates,
                       const uint64_t* mo, mc_hit* out_hits, uint32_t* out_taxon, mc_candidate* out_cand) {
  if (grp->state != 1) return fail(MC_ERR_STATE, "database is not finalized");
  if (n == 0) return MC_OK;
  if (!reads || !ro) return fail(MC_ERR_INVALID_ARG, "NULL reads");
  if (mates && !mo) return fail(MC_ERR_INVALID_ARG, "mates without mate_offsets");
  const uint32_t G = (uint32_t)grp->shards.size(), P = grp->cfg.n_partitions, Pg = P / G;
  const uint32_t m = grp->cfg.max_candidates;
  auto& S = grp->shards;
  // host views of the offsets (device offsets come to the host once: every
  // batch's byte ranges and window bounds are then planned without a sync)
  std::vector<uint64_t> c1, c2;
  const uint64_t* o1 = ro;
  const uint64_t* o2 = mo;
  if (is_device_ptr(ro)) {
    TRY(to_host(ro, n + 1, c1));
    o1 = c1.data();
  }
  if (mates && is_device_ptr(mo)) {
    TRY(to_host(mo, n + 1, c2));
    o2 = c2.data();
  }
  const int src1 = ptr_device(reads), src2 = mates ? ptr_device(mates) : -1;  // -1: host bytes
  for (int sd : {src1, src2}) {
    if (sd < 0) continue;
    bool ok = false;
    for (mc_db* sh : S) ok |= sh->device == sd;
    if (!ok) return fail(MC_ERR_INVALID_ARG, "device-resident reads must be on one of the handle's devices");
  }
  const uint64_t B = std::min<uint64_t>(grp->cfg.read_batch, n), nbat = (n + B - 1) / B;
  uint64_t mx1 = 0, mx2 = 0;
  for (uint64_t b0 = 0; b0 < n; b0 += B) {
    const uint64_t b1 = std::min(n, b0 + B);
    if (o1[b1] < o1[b0] || (mates && o2[b1] < o2[b0]))
      return fail(MC_ERR_INVALID_ARG, "read offsets decrease within records [%llu, %llu)", (unsigned long long)b0,
                  (unsigned long long)b1);
    mx1 = std::max(mx1, o1[b1] - o1[b0]);
    if (mates) mx2 = std::max(mx2, o2[b1] - o2[b0]);
  }
  // per shard: staging slots, offsets, hits and slice outputs (double-buffered)
  for (uint32_t h = 0; h < G; ++h) {
    mc_db* d = S[h];
    CK(cudaSetDevice(d->device));
    for (int k = 0; k < 2; ++k) {
      if (src1 != d->device) TRY(d->qbuf1[k].ensure(mx1 + 64));
      if (mates && src2 != d->device) TRY(d->qbuf2[k].ensure(mx2 + 64));
      TRY(d->qoff1[k].ensure(B + 1));
      if (mates) TRY(d->qoff2[k].ensure(B + 1));
      TRY(d->ohits[k].ensure(B * Pg * m));
      if (out_taxon) TRY(d->otx[k].ensure(B));
      if (out_cand) TRY(d->ocd[k].ensure(B * m * 4));
    }
    CK(cudaMemsetAsync(d->qstats.p, 0, 16 * sizeof(unsigned long long), d->stream));
    CK(cudaMemsetAsync(d->err.p, 0, 8 * sizeof(int), d->stream));
    // the first waits of this call must not see stale records
    for (int k = 0; k < 2; ++k) {
      for (cudaEvent_t e : {d->stage_free[k], d->part_done[k], d->merge_done[k]}) CK(cudaEventRecord(e, d->stream));
      for (cudaEvent_t e : {d->stage_ready[k], d->own_ready[k]}) CK(cudaEventRecord(e, d->copy_stream));
      CK(cudaEventRecord(d->out_free[k], d->d2h_stream));
    }
  }
  // whatever way the call ends, nothing still reads or writes the caller's buffers
  struct AllIdle {
    std::vector<mc_db*>& S;
    ~AllIdle() {
      for (mc_db* d : S) {
        cudaSetDevice(d->device);
        cudaStreamSynchronize(d->copy_stream);
        cudaStreamSynchronize(d->stream);
        cudaStreamSynchronize(d->d2h_stream);
      }
    }
  } idle{S};
  auto slice = [&](uint64_t b0, uint64_t nb, uint32_t g) { return b0 + nb * g / G; };
  for (uint64_t bi = 0; bi < nbat; ++bi) {
    const int k = (int)(bi & 1);
    const uint64_t b0 = bi * B, b1 = std::min(n, b0 + B), nb = b1 - b0;
    // ---- distribution: own slice (host) or broadcast (device bytes) ----------
    for (uint32_t g = 0; g < G; ++g) {
      mc_db* d = S[g];
      CK(cudaSetDevice(d->device));
      cudaStream_t cs = d->copy_stream;
      CK(cudaStreamWaitEvent(cs, d->stage_free[k], 0));   // own scoring of batch bi-2 is done with slot k
      for (uint32_t h = 0; h < G; ++h)                      // peers finished pulling from slot k
        if (h != g) CK(cudaStreamWaitEvent(cs, S[h]->stage_ready[k], 0));
      const uint64_t lo = slice(b0, nb, g), hi = slice(b0, nb, g + 1);
      auto put = [&](const char* data, const uint64_t* off, int src, DevBuf<uint8_t>* buf) -> int {
        if (src == d->device) return MC_OK;  // read in place
        if (src < 0) {                       // host: own slice only
          if (off[hi] > off[lo])
            CK(cudaMemcpyAsync(buf[k].p + (off[lo] - off[b0]), data + off[lo], off[hi] - off[lo], cudaMemcpyHostToDevice, cs));
        } else if (off[b1] > off[b0]) {      // a peer device's bytes: the whole batch over NVLink
          CK(cudaMemcpyPeerAsync(buf[k].p, d->device, data + off[b0], src, off[b1] - off[b0], cs));
        }
        return MC_OK;
      };
      TRY(put(reads, o1, src1, d->qbuf1));
      if (mates) TRY(put(mates, o2, src2, d->qbuf2));
      CK(cudaMemcpyAsync(d->qoff1[k].p, o1 + b0, (nb + 1) * 8, cudaMemcpyHostToDevice, cs));
      if (mates) CK(cudaMemcpyAsync(d->qoff2[k].p, o2 + b0, (nb + 1) * 8, cudaMemcpyHostToDevice, cs));
      CK(cudaEventRecord(d->own_ready[k], cs));
    }
    // ---- all-gather of host slices: pull every peer's slice over NVLink -------
    for (uint32_t h = 0; h < G; ++h) {
      mc_db* d = S[h];
      CK(cudaSetDevice(d->device));
      cudaStream_t cs = d->copy_stream;
      for (int side = 0; side < (mates ? 2 : 1); ++side) {
        const uint64_t* off = side ? o2 : o1;
        const int src = side ? src2 : src1;
        if (src == d->device) continue;  // read in place
        for (uint32_t g = 0; g < G && src < 0; ++g) {
          if (g == h) continue;
          const uint64_t lo = slice(b0, nb, g), hi = slice(b0, nb, g + 1);
          if (off[hi] == off[lo]) continue;
          DevBuf<uint8_t>& mine = side ? d->qbuf2[k] : d->qbuf1[k];
          DevBuf<uint8_t>& theirs = side ? S[g]->qbuf2[k] : S[g]->qbuf1[k];
          CK(cudaStreamWaitEvent(cs, S[g]->own_ready[k], 0));
          CK(cudaMemcpyPeerAsync(mine.p + (off[lo] - off[b0]), d->device, theirs.p + (off[lo] - off[b0]),
                                 S[g]->device, off[hi] - off[lo], cs));
        }
        DevBuf<uint8_t>& mine = side ? d->qbuf2[k] : d->qbuf1[k];
        CK(cudaMemsetAsync(mine.p + (off[b1] - off[b0]), 'N', 64, cs));  // defined padding (aligned-word reads)
      }
      CK(cudaEventRecord(d->stage_ready[k], cs));
    }
    // ---- scoring: every device, every record, its partitions -------------------
    for (uint32_t h = 0; h < G; ++h) {
      mc_db* d = S[h];
      CK(cudaSetDevice(d->device));
      cudaStream_t st = d->stream;
      CK(cudaStreamWaitEvent(st, d->stage_ready[k], 0));
      for (uint32_t g = 0; g < G; ++g) CK(cudaStreamWaitEvent(st, S[g]->merge_done[k], 0));  // hits slot k is free
      ReadBatch rb{};
      rb.n = nb;
      rb.base1 = o1[b0];
      rb.r1 = src1 == d->device ? reinterpret_cast<const uint8_t*>(reads) + o1[b0] : d->qbuf1[k].p;
      rb.o1 = d->qoff1[k].p;
      if (mates) {
        rb.base2 = o2[b0];
        rb.r2 = src2 == d->device ? reinterpret_cast<const uint8_t*>(mates) + o2[b0] : d->qbuf2[k].p;
        rb.o2 = d->qoff2[k].p;
      }
      uint64_t W = (o1[b1] - o1[b0]) / d->sc.stride + nb;
      if (mates) W += (o2[b1] - o2[b0]) / d->sc.stride + nb;
      TRY(run_partials(d, rb, d->ohits[k].p, W, d->err.p + 4 * k, k, st));
      CK(cudaEventRecord(d->stage_free[k], st));
      CK(cudaEventRecord(d->part_done[k], st));
      if (out_hits) {  // this device's Pg lists of every record -> their columns of out_hits
        CK(cudaStreamWaitEvent(d->d2h_stream, d->part_done[k], 0));
        CK(cudaMemcpy2DAsync(out_hits + (b0 * P + (uint64_t)h * Pg) * m, (size_t)P * m * sizeof(mc_hit), d->ohits[k].p,
                             (size_t)Pg * m * sizeof(HitRec), (size_t)Pg * m * sizeof(HitRec), nb, cudaMemcpyDefault,
                             d->d2h_stream));
        CK(cudaEventRecord(d->merge_done[k], d->d2h_stream));  // (slot k's hits are read)
      }
    }
    // ---- merge + classify slice h, reading every device's lists (peer memory) --
    if (out_taxon) {
      for (uint32_t h = 0; h < G; ++h) {
        mc_db* d = S[h];
        CK(cudaSetDevice(d->device));
        cudaStream_t st = d->stream;
        const uint64_t lo = slice(b0, nb, h), hi = slice(b0, nb, h + 1), ns = hi - lo;
        for (uint32_t g = 0; g < G; ++g) CK(cudaStreamWaitEvent(st, S[g]->part_done[k], 0));
        CK(cudaStreamWaitEvent(st, d->out_free[k], 0));  // slot k's outputs of batch bi-2 have left
        if (ns) {
          MergeArgs ma{nullptr, ns, P, m, grp->cfg.hits_min, grp->cfg.hits_diff, d->anc.p, d->depth.p, d->maxd,
                       d->n_taxa, d->otx[k].p, out_cand ? d->ocd[k].p : nullptr, d->err.p + 4 * k};
          for (uint32_t g = 0; g < G; ++g) ma.src[g] = S[g]->ohits[k].p;
          ma.n_src = G;
          ma.lists_per_src = Pg;
          ma.r0 = lo - b0;
          d->begin("merge_classify");
          launch_merge_classify(ma, st);
          d->end();
          d->launched("k_merge_classify");
        }
        CK(cudaEventRecord(d->merge_done[k], st));
        CK(cudaEventRecord(d->out_ready[k], st));
        CK(cudaStreamWaitEvent(d->d2h_stream, d->out_ready[k], 0));
        if (ns) {
          CK(cudaMemcpyAsync(out_taxon + lo, d->otx[k].p, ns * 4, cudaMemcpyDefault, d->d2h_stream));
          if (out_cand)
            CK(cudaMemcpyAsync(out_cand + lo * m, d->ocd[k].p, ns * m * sizeof(mc_candidate), cudaMemcpyDefault,
                               d->d2h_stream));
        }
        CK(cudaEventRecord(d->out_free[k], d->d2h_stream));
      }
    }
    // ---- status of this batch on every device (checked one batch later) ------
    for (uint32_t h = 0; h < G; ++h) {
      mc_db* d = S[h];
      CK(cudaSetDevice(d->device));
      CK(cudaMemcpyAsync(d->herr_pin + 4 * k, d->err.p + 4 * k, 4 * sizeof(int), cudaMemcpyDeviceToHost, d->stream));
      if (bi >= 1) {
        const int kp = (int)((bi - 1) & 1);
        CK(cudaEventSynchronize(d->qstat_ev[kp]));
        TRY(batch_status(d, d->herr_pin + 4 * kp, (bi - 1) * B));
      }
      CK(cudaEventRecord(d->qstat_ev[k], d->stream));
    }
  }
  for (uint32_t h = 0; h < G; ++h) {
    mc_db* d = S[h];
    CK(cudaSetDevice(d->device));
    CK(cudaStreamSynchronize(d->d2h_stream));
    CK(cudaStreamSynchronize(d->copy_stream));
    TRY(d->sync());
    TRY(batch_status(d, d->herr_pin + 4 * ((nbat - 1) & 1), (nbat - 1) * B));
    unsigned long long qs[16];
    CK(cudaMemcpy(qs, d->qstats.p, sizeof qs, cudaMemcpyDeviceToHost));
    d->st_qfeat += qs[0];
    d->st_qfeat_hit += qs[8];
    d->st_qloc += qs[1];
    for (int b = 0; b < 3; ++b) d->st_qloc_bin[b] += qs[3 + b];
    d->st_qmed += qs[6];
    d->st_qlarge += qs[7];
    d->st_reads += n;
    d->st_read_bp += qs[2];
  }
  return MC_OK;
}
