// Device building blocks of the B200 MetaCache path (sm_100a).
//
// Paper: arXiv 2106.08150, /root/reference/PAPER.md (P:<line>).  Readings of
// silent points (S1..S24) are listed in DESIGN.md.  Nothing here is shared
// with oracle/: the oracle is an independent CPU program.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mc {

constexpr uint32_t kFull = 0xffffffffu;

// ---------------------------------------------------------------------------
// Sketch parameters: k-mer length, sketch size s, window stride
// w-k+1.  One warp covers one window: lane i owns k-mer starts 4i..4i+3
// (P:709-727), so stride <= 128.
// ---------------------------------------------------------------------------
struct SketchCfg {
  uint32_t k, s, stride;
  // 2^16, 2^8 and 2^24 at run time: multiplies by them stand in for shifts
  // in the sketch loop (IMAD / IMAD.HI issue on the FMA pipe, which idles
  // while the loop saturates the ALU pipe); being kernel parameters, ptxas
  // cannot turn them back into shifts
  uint32_t p16, p8, p24;
  // candidate threshold of the filtered build sketch (sketch_slot_filter):
  // a fixed quantile of the 32-bit feature range, tuned, not a result input
  uint32_t thr0;
};
#ifndef MC_THR0
#define MC_THR0 0x40000000u  // 1/4 of the range
#endif
inline SketchCfg make_sketch_cfg(uint32_t k, uint32_t s, uint32_t w) {
  return SketchCfg{k, s, w - k + 1, 1u << 16, 1u << 8, 1u << 24, MC_THR0};
}

// S1: h1 = 32-bit bijective integer mixer (P:331, P:683 name it, never define it).
__device__ __forceinline__ uint32_t h1(uint32_t x) {
  x = ((x >> 16) ^ x) * 0x45d9f3bu;
  x = ((x >> 16) ^ x) * 0x45d9f3bu;
  return (x >> 16) ^ x;
}

// S2: slot hash ("h2") -- internal to the table (no effect on
// results).  Fibonacci (multiplicative) hashing: minhash keys are h1 outputs
// concentrated in the low ~15 % of the 32-bit range, and key * 2^64/phi
// spreads them evenly over the high bits that fastrange maps to [0, n)
// (three-distance theorem); 2 multiply-adds instead of a 64-bit mixer's ~20
// instructions, on a path that hashes every location five times.
__device__ __forceinline__ uint64_t slot_hash(uint32_t key) { return (uint64_t)key * 0x9e3779b97f4a7c15ull; }
// fastrange: floor(h * n / 2^64).  For n < 2^32 (tables of < 4.3 G slots) it
// is hi * n + umulhi(lo, n) >> 32 -- exact (the dropped fraction cannot carry)
// and 3 multiply-adds instead of a 64 x 64 multiply-high
#ifndef MC_FASTRANGE32
#define MC_FASTRANGE32 1
#endif
__device__ __forceinline__ uint64_t fastrange64(uint64_t h, uint64_t n) {
  if (MC_FASTRANGE32 && n <= 0xffffffffull)
    return ((uint64_t)(uint32_t)(h >> 32) * (uint32_t)n + __umulhi((uint32_t)h, (uint32_t)n)) >> 32;
  return __umul64hi(h, n);
}
__device__ __forceinline__ uint64_t home_slot(uint32_t key, uint64_t n) { return fastrange64(slot_hash(key), n); }
// Linear probing wraps inside the key's table SUB-REGION of kSubSlots slots
// (the table size is a multiple of it), so finalize can build each
// sub-region in shared memory.
constexpr uint32_t kSubLg = 13, kSubSlots = 1u << kSubLg;
__device__ __forceinline__ uint64_t next_slot(uint64_t s) {
  return (s & ~(uint64_t)(kSubSlots - 1)) | ((s + 1) & (kSubSlots - 1));
}

// ---------------------------------------------------------------------------
// §5.2 step (1) / §5.3: encode 4 ASCII chars (byte 0 = first char)
// into 2-bit codes A0 C1 G2 T3 (S3) with an ambiguity nibble (S4).
// Result bits [7:0]: codes, first char in bits 7:6; bits [11:8]: N-mask,
// first char in bit 11.  Case-insensitive; any other byte is ambiguous.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t encode4(uint32_t w) {
  const uint32_t v = w | 0x20202020u;
  const uint32_t ok = __vcmpeq4(v, 0x61616161u) | __vcmpeq4(v, 0x63636363u) | __vcmpeq4(v, 0x67676767u) |
                      __vcmpeq4(v, 0x74747474u);
  const uint32_t x = (w >> 1) & 0x03030303u;      // A0 C1 G3 T2 (either case)
  const uint32_t c = x ^ ((x >> 1) & 0x01010101u);  // -> A0 C1 G2 T3, one code per byte
  // gather the 4 byte-codes (first char most significant) with one multiply:
  // bytes reversed, then x * (2^18 + 2^12 + 2^6 + 1) puts c0..c3 at bits 24..18
  const uint32_t code = ((__byte_perm(c, 0, 0x0123) * 0x41041u) >> 18) & 0xffu;
  const uint32_t bad = (~ok >> 7) & 0x01010101u;  // 1 per ambiguous byte
  const uint32_t nm = ((__byte_perm(bad, 0, 0x0123) * 0x204081u) >> 21) & 0xfu;
  return code | (nm << 8);
}

// position of the r-th (0-based) set bit of m (m must have more than r set bits)
__device__ __forceinline__ uint32_t nth_set_bit(uint32_t m, uint32_t r) {
  uint32_t p = 0;
#pragma unroll
  for (uint32_t w = 16; w; w >>= 1) {
    const uint32_t c = __popc(m & ((1u << w) - 1u));
    if (r >= c) { r -= c; m >>= w; p += w; }
  }
  return p;
}

// reverse complement of a k-mer held in the low 2k bits (first base most significant)
__device__ __forceinline__ uint32_t revcomp(uint32_t fwd, uint32_t k) {
  uint32_t r = __brev(~fwd);                                   // complement, reverse bits
  r = ((r >> 1) & 0x55555555u) | ((r & 0x55555555u) << 1);      // restore order inside each base
  return r >> (32 - 2 * k);
}

// ---------------------------------------------------------------------------
// Warp-cooperative minhash sketch of ONE window (§4.1).
//   p  : the window's first char (device, any alignment)
//   nk : number of k-mer starts in the window (1..stride).
// Lane i loads one aligned 32-bit word (+ one more for lanes < 5), encodes it
// and gathers the 6 words covering its 4 k-mers with 5 shuffles.  The s
// smallest UNIQUE features are then extracted by s rounds of a warp-wide
// min-reduction (REDUX) -- duplicates drop out because every copy of the
// minimum is retired in the same round.
// Returns the sketch size (warp-uniform); lane l < size receives feature l
// (ascending) in *feat.  Must be called by all 32 lanes.
// ---------------------------------------------------------------------------
// Window loads, separated from the arithmetic so a warp can prefetch the next
// window while it sketches the current one.
struct WinWords {
  uint32_t wA, wB, sh;
};

__device__ __forceinline__ WinWords load_window(const uint8_t* p, uint32_t nk, const SketchCfg& c, uint32_t lane) {
  const uint32_t nchars = nk + c.k - 1;
  const uintptr_t addr = reinterpret_cast<uintptr_t>(p);
  WinWords w;
  w.sh = (uint32_t)(addr & 3u);
  const uint32_t nwords = (w.sh + nchars + 3) >> 2;  // <= 37; aligned words never cross a page
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(addr & ~(uintptr_t)3);
  w.wA = lane < nwords ? __ldg(wp + lane) : 0x4e4e4e4eu;
  w.wB = lane + 32 < nwords ? __ldg(wp + 32 + lane) : 0x4e4e4e4eu;
  return w;
}

// Sketch of one window from its loaded words.  kToSmem: lane 0 writes feature
// i to sout[i] (ascending); otherwise lane i receives feature i in *feat.
// Returns the sketch size (warp-uniform).  Must be called by all 32 lanes.
// K: compile-time k-mer length (0 = runtime c.k); K = 16, the paper's default,
// folds every shift and mask into constants.
template <bool kToSmem, uint32_t K = 0>
__device__ __forceinline__ int sketch_words(const WinWords& ww, uint32_t nk, const SketchCfg& c, uint32_t lane,
                                            uint32_t& feat, uint32_t* sout) {
  const uint32_t sh = ww.sh;
  const uint32_t k = K ? K : c.k;
  const uint32_t pk = encode4(ww.wA) | (encode4(ww.wB) << 16);

  // this lane's 24-char stream: 2-bit codes, char 0 most significant
  // (Shi = chars 0..7, Slo = chars 8..23) and the 24-bit ambiguity mask
  uint32_t Shi = 0, Slo = 0, N = 0;
#pragma unroll
  for (uint32_t d = 0; d < 6; ++d) {
    const uint32_t src = lane + d;
    const uint32_t v = d == 0 ? pk : __shfl_sync(kFull, pk, src & 31);
    const uint32_t u = src < 32 ? (v & 0xffffu) : (v >> 16);
    if (d < 2) Shi = (Shi << 8) | (u & 0xffu);
    else Slo = (Slo << 8) | (u & 0xffu);
    N = (N << 4) | ((u >> 8) & 0xfu);
  }

  const uint32_t kmask = k == 16 ? 0xffffffffu : ((1u << (2 * k)) - 1u);
  const uint32_t nmask = (1u << k) - 1u;
  // reverse complement of the whole 24-char stream (R char i = comp(S char 23-i)),
  // so each k-mer's reverse complement is one funnel shift of R
  const uint32_t rlo = revcomp(Slo, 16);
  const uint32_t Rhi = rlo >> 16, Rlo = (rlo << 16) | revcomp(Shi, 8);
  uint32_t v0, v1, v2, v3;  // the lane's 4 features; invalid k-mers -> 0xffffffff
  bool has_max = false;      // a VALID feature equal to 0xffffffff (h1 is a bijection)
  {
    uint32_t val[4];
#pragma unroll
    for (uint32_t j = 0; j < 4; ++j) {
      const uint32_t t = 4 * lane + j;  // k-mer start inside the window
      const uint32_t q0 = sh + j;       // its char position inside this lane's stream
      // bits [47 - 2*q0, 48 - 2*(q0 + k)) of the 48-bit stream Shi:Slo
      const uint32_t sft = 48 - 2 * (q0 + k);
      const uint32_t fwd = (K == 16 ? __funnelshift_r(Slo, Shi, sft)
                                    : sft >= 32 ? (Shi >> (sft - 32)) : __funnelshift_r(Slo, Shi, sft)) & kmask;
      const uint32_t nb = (N >> (24 - q0 - k)) & nmask;
      const uint32_t rc = __funnelshift_r(Rlo, Rhi, 2 * q0) & kmask;  // chars [24-q0-k, 24-q0) of R
      const uint32_t f = h1(min(fwd, rc));  // canonical k-mer -> feature
      const bool ok = t < nk && nb == 0;
      has_max |= ok && f == 0xffffffffu;
      val[j] = ok ? f : 0xffffffffu;
    }
    v0 = val[0]; v1 = val[1]; v2 = val[2]; v3 = val[3];
  }
  // sort the lane's 4 values, drop in-lane duplicates, sort again
#define MC_CE(a, b) { const uint32_t lo_ = min(a, b), hi_ = max(a, b); a = lo_; b = hi_; }
  MC_CE(v0, v1) MC_CE(v2, v3) MC_CE(v0, v2) MC_CE(v1, v3) MC_CE(v1, v2)
  {
    const bool d1 = v1 == v0, d2 = v2 == v1, d3 = v3 == v2;
    v1 = d1 ? 0xffffffffu : v1;
    v2 = d2 ? 0xffffffffu : v2;
    v3 = d3 ? 0xffffffffu : v3;
  }
  MC_CE(v0, v1) MC_CE(v2, v3) MC_CE(v0, v2) MC_CE(v1, v3) MC_CE(v1, v2)
#undef MC_CE
  const uint32_t s = c.s;
  feat = 0;

  // s rounds of a warp-wide minimum (REDUX) over the lanes' sorted queues;
  // every lane retires its (single, deduplicated) copy of the minimum, so the
  // selected features are the s smallest UNIQUE ones, in ascending order
  // (branch-free: all s rounds run; a round whose minimum is 0xffffffff found
  // no value left, and the count is taken afterwards)
#define MC_ROUND(I)                                              \
  {                                                              \
    const uint32_t m = __reduce_min_sync(kFull, v0);             \
    if (kToSmem) {                                               \
      if (lane == 0) sout[I] = m;                                \
    } else if (lane == (uint32_t)(I)) {                          \
      feat = m;                                                  \
    }                                                            \
    const bool e0 = v0 == m;                                     \
    v0 = e0 ? v1 : v0;                                           \
    v1 = e0 ? v2 : v1;                                           \
    v2 = e0 ? v3 : v2;                                           \
    v3 = e0 ? 0xffffffffu : v3;                                  \
  }
  if (s == 16) {  // the paper's default: fully unrolled
#pragma unroll
    for (int i = 0; i < 16; ++i) MC_ROUND(i)
  } else {
    for (int i = 0; i < (int)s; ++i) MC_ROUND(i)
  }
#undef MC_ROUND
  if (kToSmem) {
    __syncwarp();
    feat = lane < s ? sout[lane] : 0xffffffffu;
  }
  int cnt = __popc(__ballot_sync(kFull, lane < s && feat != 0xffffffffu));
  // 0xffffffff is the largest feature: it is in the sketch iff it is valid
  // somewhere and fewer than s smaller unique features exist (slot cnt holds it)
  if (cnt < (int)s && __any_sync(kFull, has_max)) ++cnt;
  return cnt;
}


__device__ __forceinline__ int sketch_window(const uint8_t* p, uint32_t nk, const SketchCfg& c, uint32_t lane,
                                             uint32_t& feat) {
  const WinWords ww = load_window(p, nk, c, lane);
  return c.k == 16 ? sketch_words<false, 16>(ww, nk, c, lane, feat, nullptr)
                   : sketch_words<false, 0>(ww, nk, c, lane, feat, nullptr);
}

// ---------------------------------------------------------------------------
// Thread-per-window sketch (the build path; same result as sketch_words).
//
// The warp-per-window form above spends most of its ~550 instructions per
// window on lane plumbing (shuffles, 16 warp-wide REDUX rounds).  Here each
// thread rolls over its own window, 4 chars (one word) at a time, and keeps
// the 16 smallest features in a register-resident sorted list updated by a
// min/max insertion network -- ~50 thread instructions per k-mer, all ALU.
// The list is filled WITHOUT de-duplication; that is exact whenever the 16
// smallest of the multiset are pairwise distinct (they are then the 16
// smallest distinct features).  Windows where they are not (repeats) and
// windows that produced the value 0xffffffff (it doubles as the invalid
// marker) are re-sketched by the exact warp-per-window routine.
// ---------------------------------------------------------------------------
constexpr uint32_t kSlotWords = 36;  // staged window: <= 144 chars, 144-B stride (LDS.128 conflict-free)

struct Enc4 {
  uint32_t f32;  // bits 31..24 = codes c0 c1 c2 c3 (c0 most significant), bits below are don't-care
  uint32_t r8;   // bits 7..0 = comp(c0) | comp(c1) << 2 | comp(c2) << 4 | comp(c3) << 6
  uint32_t inv;  // bit 28 + i set: char i is not one of ACGTacgt (S4)
};

// 4 ASCII chars (byte i = char i) -> codes A0 C1 G2 T3 (S3), either case.
__device__ __forceinline__ Enc4 enc_word(uint32_t w) {
  Enc4 e;
  const uint32_t x = (w >> 1) ^ (w >> 2);  // bits 1:0 of each byte = code of A/C/G/T/a/c/g/t
  const uint32_t code = x & 0x03030303u;
  e.f32 = code * 0x40100401u;                       // gathers byte codes at bits 31..24
  e.r8 = ((~x & 0x03030303u) * 0x01041040u) >> 24;  // complements, c0 lowest
  // validity: re-spell each byte from its code and compare (case folded);
  // PRMT takes the selector nibbles in the order c0 c2 c1 c3
  const uint32_t expect = __byte_perm(0x54474341u, 0u, code | (code >> 12));
  const uint32_t d = (__byte_perm(w, 0u, 0x3120u) & 0xdfdfdfdfu) ^ expect;
  const uint32_t bad = (((d & 0x7f7f7f7fu) + 0x7f7f7f7fu) | d) & 0x80808080u;  // bits 7,15,23,31 = c0 c2 c1 c3
  e.inv = (bad * 0x00208041u) & 0xf0000000u;
  return e;
}

// 16-entry ascending list, insertion without de-duplication
__device__ __forceinline__ void bottom16_insert(uint32_t (&v)[16], uint32_t x) {
#pragma unroll
  for (int i = 15; i > 0; --i) v[i] = min(v[i], max(v[i - 1], x));
  v[0] = min(v[0], x);
}

#define MC_CE(a, b) { const uint32_t lo_ = min(a, b), hi_ = max(a, b); a = lo_; b = hi_; }
// Compare-exchange with the max on the FMA pipe: hi = a + b - min(a, b)
// (exact mod 2^32) as two IMADs by an opaque 1, so the min is the only ALU
// instruction.  The fast sketch loop is ALU-pipe bound (min/max, xor, LOP3)
// while the FMA pipe runs at half its rate; moving ~half the network's max
// operations across balances the two pipes.
#define MC_CEF(a, b) { const uint32_t lo_ = min(a, b), s_ = (a) * one + (b); b = s_ - lo_ * one; a = lo_; }
#ifndef MC_CE_FMA
#define MC_CE_FMA 1
#endif
// v (ascending) <- the 16 smallest of v and b[0..8): sort b (19-comparator
// network), bitonic half-cleaner against v, bitonic merge -- 110 min/max for
// 8 values instead of 8 x 31 for one-by-one insertion.  one: a run-time 1.
__device__ __forceinline__ void bottom16_merge8(uint32_t (&v)[16], uint32_t (&b)[8], uint32_t one) {
#if MC_CE_FMA & 2
#define MC_CEB MC_CEF
#else
#define MC_CEB MC_CE
#endif
  MC_CEB(b[0], b[2]) MC_CEB(b[1], b[3]) MC_CEB(b[4], b[6]) MC_CEB(b[5], b[7])
  MC_CEB(b[0], b[4]) MC_CEB(b[1], b[5]) MC_CEB(b[2], b[6]) MC_CEB(b[3], b[7])
  MC_CEB(b[0], b[1]) MC_CEB(b[2], b[3]) MC_CEB(b[4], b[5]) MC_CEB(b[6], b[7])
  MC_CEB(b[2], b[4]) MC_CEB(b[3], b[5])
  MC_CEB(b[1], b[4]) MC_CEB(b[3], b[6])
  MC_CEB(b[1], b[2]) MC_CEB(b[3], b[4]) MC_CEB(b[5], b[6])
#undef MC_CEB
#pragma unroll
  for (int i = 0; i < 8; ++i) v[8 + i] = min(v[8 + i], b[7 - i]);  // v is now bitonic
#pragma unroll
  for (int d = 8; d > 0; d >>= 1) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (!(i & d)) {
        if ((MC_CE_FMA & 1) && !((MC_CE_FMA & 4) && d == 8)) MC_CEF(v[i], v[i + d])
        else MC_CE(v[i], v[i + d])
      }
  }
}
#ifndef MC_MERGE16
#define MC_MERGE16 0
#endif
#ifndef MC_HALF_ITER
#define MC_HALF_ITER 1  // fast sketch loop of 8 chars per iteration (sketch_slot_fast)
#endif
#ifndef MC_HALF_ITER_SLOT
#define MC_HALF_ITER_SLOT 0  // 1: the same for the checked path (sketch_slot; read windows in the query)
#endif
// v (ascending) <- the 16 smallest of v and b[0..16): sort b (60-comparator,
// 10-layer network; checked on all 2^16 0-1 inputs), half-cleaner against v,
// bitonic merge -- 200 min/max for 16 values (12.5 per value, 13.75 for
// bottom16_merge8).  one: a run-time 1.
#ifndef MC_SORT_FMA_N
#define MC_SORT_FMA_N ((MC_CE_FMA & 2) ? 60 : 0)  // sort comparators [0, N) take the FMA-pipe form
#endif
__device__ __forceinline__ void bottom16_merge16(uint32_t (&v)[16], uint32_t (&b)[16], uint32_t one) {
  constexpr uint8_t kNet[60][2] = {  // 10 layers
      {0, 13}, {1, 12}, {2, 15}, {3, 14}, {4, 8}, {5, 6}, {7, 11}, {9, 10},
      {0, 5}, {1, 7}, {2, 9}, {3, 4}, {6, 13}, {8, 14}, {10, 15}, {11, 12},
      {0, 1}, {2, 3}, {4, 5}, {6, 8}, {7, 9}, {10, 11}, {12, 13}, {14, 15},
      {0, 2}, {1, 3}, {4, 10}, {5, 11}, {6, 7}, {8, 9}, {12, 14}, {13, 15},
      {1, 2}, {3, 12}, {4, 6}, {5, 7}, {8, 10}, {9, 11}, {13, 14},
      {1, 4}, {2, 6}, {5, 8}, {7, 10}, {9, 13}, {11, 14},
      {2, 4}, {3, 6}, {9, 12}, {11, 13},
      {3, 5}, {6, 8}, {7, 9}, {10, 12},
      {3, 4}, {5, 6}, {7, 8}, {9, 10}, {11, 12},
      {6, 7}, {8, 9},
  };
#pragma unroll
  for (int i = 0; i < 60; ++i) {
    if (i < MC_SORT_FMA_N) MC_CEF(b[kNet[i][0]], b[kNet[i][1]])
    else MC_CE(b[kNet[i][0]], b[kNet[i][1]])
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = min(v[i], b[15 - i]);  // v is now bitonic
#pragma unroll
  for (int d = 8; d > 0; d >>= 1) {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (!(i & d)) {
        if ((MC_CE_FMA & 1) && !((MC_CE_FMA & 4) && d == 8)) MC_CEF(v[i], v[i + d])
        else MC_CE(v[i], v[i + d])
      }
  }
}
#undef MC_CE

// One word of the window: chars 4q..4q+3.  State: fwd = last 16 codes (newest
// lowest), rc = reverse complement of the last 16 chars (newest highest),
// nm = ambiguity bits of the last 32 chars (newest at bit 31).  out[j] = the
// feature of the k-mer ending at char j of the word (0xffffffff: invalid),
// for j >= J0.
template <uint32_t K, int J0>
__device__ __forceinline__ void tw_word(uint32_t w, uint32_t k, uint32_t& fwd, uint32_t& rc, uint32_t& nm,
                                        uint32_t* out, uint32_t& hmax) {
  const Enc4 e = enc_word(w);
  nm = (nm >> 4) | e.inv;
#pragma unroll
  for (int j = J0; j < 4; ++j) {
    const uint32_t n = 2 * (j + 1);
    uint32_t fw = __funnelshift_l(e.f32, fwd, n);  // chars ending at char j, last one lowest
    uint32_t rv = __funnelshift_r(rc, e.r8, n);
    bool ok;
    if (K == 16) {
      ok = (nm & (0xffffu << (13 + j))) == 0;
    } else {
      fw &= k == 16 ? 0xffffffffu : ((1u << (2 * k)) - 1u);
      rv >>= 32 - 2 * k;
      ok = (nm & (((1u << k) - 1u) << (29 + j - k))) == 0;
    }
    const uint32_t h = h1(min(fw, rv));  // canonical k-mer -> feature
    hmax = max(hmax, h);
    out[j] = ok ? h : 0xffffffffu;
  }
  fwd = __funnelshift_l(e.f32, fwd, 8);
  rc = __funnelshift_r(rc, e.r8, 8);
}

// ---- fast path: k = 16, full windows of 127 chars, no ambiguous char --------
// Shifts become multiplies on the FMA pipe: x >> 16 == umulhi(x, 2^16); the
// rolling k-mers fw = fwd << n | top n bits of the word's codes and
// rc = rc >> n | complements << (32 - n) are two multiply-adds each.
__device__ __forceinline__ uint32_t h1_fma(uint32_t x, uint32_t p16) {
  x = (__umulhi(x, p16) ^ x) * 0x45d9f3bu;
  x = (__umulhi(x, p16) ^ x) * 0x45d9f3bu;
  return __umulhi(x, p16) ^ x;
}

// One word (chars 4q..4q+3) without ambiguity tracking: inv accumulates the
// word's ambiguity bits (a window with any is recomputed by the checked path).
// mj = 4^(j+1) multipliers, qj = 2^(32 - 2(j+1)); derived from the opaque
// kernel parameters so they stay multiplies.
template <int J0, bool kLastKmerOut>
__device__ __forceinline__ void tw_word_fast(uint32_t w, uint32_t& fwd, uint32_t& rc, uint32_t& inv, uint32_t* out,
                                             const uint32_t (&mj)[4], const uint32_t (&qj)[4], uint32_t p16) {
  const Enc4 e = enc_word(w);
  inv |= e.inv;
#pragma unroll
  for (int j = J0; j < 4; ++j) {
    const uint32_t fw = fwd * mj[j] + __umulhi(e.f32, mj[j]);  // chars ending at char j, last one lowest
    const uint32_t rv = e.r8 * qj[j] + __umulhi(rc, qj[j]);
    out[j] = h1_fma(min(fw, rv), p16);  // canonical k-mer -> feature
  }
  if (kLastKmerOut) out[3] = 0xffffffffu;  // the 128th char starts the next window's k-mers
  fwd = fwd * mj[3] + __umulhi(e.f32, mj[3]);
  rc = e.r8 * qj[3] + __umulhi(rc, qj[3]);
}

// Sketch of a full 127-char window staged at `slot` (k = 16, 112 k-mers, 8
// iterations of 16 chars); returns false if the window must be recomputed:
// an ambiguous char, a duplicate among the 16 smallest, or fewer than 16
// features below 0xffffffff (the value doubles as the invalid marker).
__device__ __forceinline__ bool sketch_slot_fast(const uint32_t* __restrict__ slot, const SketchCfg& c,
                                                 uint32_t (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = 0xffffffffu;
  const uint32_t p2 = c.p8 >> 6;  // 4
  const uint32_t one = c.p8 >> 8;  // opaque 1 (bottom16_merge8)
  const uint32_t mj[4] = {p2, p2 * p2, p2 * p2 * p2, c.p8};
  const uint32_t qj[4] = {c.p24 << 6, c.p24 << 4, c.p24 << 2, c.p24};
  uint32_t fwd = 0, rc = 0, inv = 0;
  const uint4* q = reinterpret_cast<const uint4*>(slot);
#if MC_MERGE16 && !MC_HALF_ITER
  uint32_t b[16];
#else
  uint32_t b[8];
#endif
  {
    const uint4 a = q[0];  // no 16-mer ends before char 15
    tw_word_fast<4, false>(a.x, fwd, rc, inv, b, mj, qj, c.p16);
    tw_word_fast<4, false>(a.y, fwd, rc, inv, b, mj, qj, c.p16);
    tw_word_fast<4, false>(a.z, fwd, rc, inv, b, mj, qj, c.p16);
    tw_word_fast<3, false>(a.w, fwd, rc, inv, b, mj, qj, c.p16);
    v[0] = b[3];
  }
#if MC_HALF_ITER
  // 14 iterations of 8 chars (two words, one merge8): a loop body of ~250
  // instructions fits the SMSP's L0 instruction cache (~6 KB); the 16-char
  // body did not, and the kernel stalled ~20 % of the time on instruction
  // fetch (ncu s2b).  The window's last word is masked in the loop
  {
    const uint2* q2 = reinterpret_cast<const uint2*>(slot);
#pragma unroll 1
    for (uint32_t it = 2; it < 16; ++it) {
      const uint2 a = q2[it];
      const bool last = it == 15;  // chars 120..127: the 127th char is byte 2 of .y, byte 3 is padding
      tw_word_fast<0, false>(a.x, fwd, rc, inv, b, mj, qj, c.p16);
      tw_word_fast<0, false>(last ? (a.y & 0x00ffffffu) | 0x41000000u : a.y, fwd, rc, inv, b + 4, mj, qj, c.p16);
      b[7] = last ? 0xffffffffu : b[7];
      bottom16_merge8(v, b, one);
    }
  }
#elif MC_MERGE16
#pragma unroll 1
  for (uint32_t it = 1; it < 7; ++it) {
    const uint4 a = q[it];
    tw_word_fast<0, false>(a.x, fwd, rc, inv, b, mj, qj, c.p16);
    tw_word_fast<0, false>(a.y, fwd, rc, inv, b + 4, mj, qj, c.p16);
    tw_word_fast<0, false>(a.z, fwd, rc, inv, b + 8, mj, qj, c.p16);
    tw_word_fast<0, false>(a.w, fwd, rc, inv, b + 12, mj, qj, c.p16);
    bottom16_merge16(v, b, one);
  }
  {
    const uint4 a = q[7];
    tw_word_fast<0, false>(a.x, fwd, rc, inv, b, mj, qj, c.p16);
    tw_word_fast<0, false>(a.y, fwd, rc, inv, b + 4, mj, qj, c.p16);
    tw_word_fast<0, false>(a.z, fwd, rc, inv, b + 8, mj, qj, c.p16);
    // the window's last char (127th) is this word's byte 2; byte 3 is padding
    tw_word_fast<0, true>(a.w & 0x00ffffffu | 0x41000000u, fwd, rc, inv, b + 12, mj, qj, c.p16);
    bottom16_merge16(v, b, one);
  }
#else
#pragma unroll 1
  for (uint32_t it = 1; it < 7; ++it) {
    const uint4 a = q[it];
    tw_word_fast<0, false>(a.x, fwd, rc, inv, b, mj, qj, c.p16);
    tw_word_fast<0, false>(a.y, fwd, rc, inv, b + 4, mj, qj, c.p16);
    bottom16_merge8(v, b, one);
    tw_word_fast<0, false>(a.z, fwd, rc, inv, b, mj, qj, c.p16);
    tw_word_fast<0, false>(a.w, fwd, rc, inv, b + 4, mj, qj, c.p16);
    bottom16_merge8(v, b, one);
  }
  {
    const uint4 a = q[7];
    tw_word_fast<0, false>(a.x, fwd, rc, inv, b, mj, qj, c.p16);
    tw_word_fast<0, false>(a.y, fwd, rc, inv, b + 4, mj, qj, c.p16);
    bottom16_merge8(v, b, one);
    tw_word_fast<0, false>(a.z, fwd, rc, inv, b, mj, qj, c.p16);
    // the window's last char (127th) is this word's byte 2; byte 3 is padding
    tw_word_fast<0, true>(a.w & 0x00ffffffu | 0x41000000u, fwd, rc, inv, b + 4, mj, qj, c.p16);
    bottom16_merge8(v, b, one);
  }
#endif
  bool exact = inv == 0 && v[15] != 0xffffffffu;
#pragma unroll
  for (int i = 0; i < 15; ++i) exact &= v[i] != v[i + 1];
  return exact;
}

// ---- candidate-filtered fast path (build; k = 16, full 127-char windows) ----
// Only a feature below the running threshold thr can still enter the bottom
// 16, so each k-mer's feature is a CANDIDATE iff it is below thr: candidates
// are appended to the lane's column of a shared-memory buffer (rows of 32
// lanes, conflict-free) and merged into v 16 at a time, when some lane of
// the warp holds 16 (a warp-uniform decision: every lane merges its rows,
// the rows beyond a lane's count hold 0xffffffff).  thr starts at
// c.thr0 (a fixed hash quantile: P(fewer than 16 of a window's 112 features
// below it) is ~0.2 % at 1/4 of the range) and drops to v[15] after each
// merge.  The result is the 16 smallest of the multiset whenever the window
// has >= 16 features below thr0 (v[15] != 0xffffffff); otherwise the window
// is re-sketched exactly like any other inexact one.  A window merges ~3
// times (200 min/max each) instead of running 7 merges over all 112
// features: the selection work drops from ~12.5 to ~5.5 ALU operations per
// k-mer plus ~2 for the filter.
constexpr uint32_t kCandRows = 24;  // 15 held + 8 appended between checks, rounded up

struct CandBuf {
  uint32_t* col;  // the lane's column: row i at col[32 i]
  uint32_t* wp;   // next free row (col + 32 x candidates held)
  uint32_t thr;   // running threshold
  __device__ __forceinline__ void push(uint32_t h) {
    if (h < thr) {
      *wp = h;
      wp += 32;
    }
  }
  __device__ __forceinline__ bool full() const { return wp >= col + 16 * 32; }
  __device__ __forceinline__ bool empty() const { return wp == col; }
};

// v <- bottom 16 of v and the lane's first 16 rows; rows 16.. move down,
// the vacated rows are refilled with 0xffffffff.  Warp-uniform.
__device__ __forceinline__ void cand_merge(CandBuf& cb, uint32_t (&v)[16], uint32_t one) {
  uint32_t b[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) b[i] = cb.col[i << 5];
#pragma unroll
  for (int i = 0; i < (int)kCandRows - 16; ++i) {
    cb.col[i << 5] = cb.col[(16 + i) << 5];
    cb.col[(16 + i) << 5] = 0xffffffffu;
  }
#pragma unroll
  for (int i = kCandRows - 16; i < 16; ++i) cb.col[i << 5] = 0xffffffffu;
  cb.wp = cb.full() ? cb.wp - 16 * 32 : cb.col;
  bottom16_merge16(v, b, one);
  cb.thr = min(cb.thr, v[15]);
}

template <int J0, bool kLastKmerOut>
__device__ __forceinline__ void tw_word_filt(uint32_t w, uint32_t& fwd, uint32_t& rc, uint32_t& inv, CandBuf& cb,
                                             const uint32_t (&mj)[4], const uint32_t (&qj)[4], uint32_t p16) {
  const Enc4 e = enc_word(w);
  inv |= e.inv;
#pragma unroll
  for (int j = J0; j < (kLastKmerOut ? 3 : 4); ++j) {
    const uint32_t fw = fwd * mj[j] + __umulhi(e.f32, mj[j]);  // chars ending at char j, last one lowest
    const uint32_t rv = e.r8 * qj[j] + __umulhi(rc, qj[j]);
    cb.push(h1_fma(min(fw, rv), p16));  // canonical k-mer -> feature
  }
  fwd = fwd * mj[3] + __umulhi(e.f32, mj[3]);
  rc = e.r8 * qj[3] + __umulhi(rc, qj[3]);
}

// Same contract as sketch_slot_fast; `col` = the lane's candidate column
// (kCandRows rows, any contents).
__device__ __forceinline__ bool sketch_slot_filter(const uint32_t* __restrict__ slot, const SketchCfg& c,
                                                   uint32_t* col, uint32_t (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < (int)kCandRows; ++i) col[i << 5] = 0xffffffffu;
  const uint32_t p2 = c.p8 >> 6;   // 4
  const uint32_t one = c.p8 >> 8;  // opaque 1 (bottom16_merge16)
  const uint32_t mj[4] = {p2, p2 * p2, p2 * p2 * p2, c.p8};
  const uint32_t qj[4] = {c.p24 << 6, c.p24 << 4, c.p24 << 2, c.p24};
  uint32_t fwd = 0, rc = 0, inv = 0;
  CandBuf cb{col, col, c.thr0};
  const uint4* q = reinterpret_cast<const uint4*>(slot);
  {
    const uint4 a = q[0];  // no 16-mer ends before char 15
    tw_word_filt<4, false>(a.x, fwd, rc, inv, cb, mj, qj, c.p16);
    tw_word_filt<4, false>(a.y, fwd, rc, inv, cb, mj, qj, c.p16);
    tw_word_filt<4, false>(a.z, fwd, rc, inv, cb, mj, qj, c.p16);
    tw_word_filt<3, false>(a.w, fwd, rc, inv, cb, mj, qj, c.p16);
  }
#pragma unroll 1
  for (uint32_t it = 1; it < 8; ++it) {
    const uint4 a = q[it];
    tw_word_filt<0, false>(a.x, fwd, rc, inv, cb, mj, qj, c.p16);
    tw_word_filt<0, false>(a.y, fwd, rc, inv, cb, mj, qj, c.p16);
    if (__any_sync(kFull, cb.full())) cand_merge(cb, v, one);
    tw_word_filt<0, false>(a.z, fwd, rc, inv, cb, mj, qj, c.p16);
    if (it < 7) {
      tw_word_filt<0, false>(a.w, fwd, rc, inv, cb, mj, qj, c.p16);
    } else {  // the window's last char (127th) is this word's byte 2; byte 3 is padding
      tw_word_filt<0, true>(a.w & 0x00ffffffu | 0x41000000u, fwd, rc, inv, cb, mj, qj, c.p16);
    }
    if (__any_sync(kFull, cb.full())) cand_merge(cb, v, one);
  }
  while (__any_sync(kFull, !cb.empty())) cand_merge(cb, v, one);
  bool exact = inv == 0 && v[15] != 0xffffffffu;
#pragma unroll
  for (int i = 0; i < 15; ++i) exact &= v[i] != v[i + 1];
  return exact;
}

// Sketch of the window staged at `slot` (chars beyond the window are 'N'):
// v = 16 smallest features of the multiset, ascending, padded with
// 0xffffffff; returns false if the result must be recomputed exactly.
template <uint32_t K>
__device__ __forceinline__ bool sketch_slot(const uint32_t* __restrict__ slot, uint32_t niter, uint32_t k,
                                            uint32_t one, uint32_t (&v)[16]) {
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = 0xffffffffu;
  uint32_t fwd = 0, rc = 0, nm = 0xffffffffu, hmax = 0;
  const uint4* q = reinterpret_cast<const uint4*>(slot);
  uint32_t it = 0;
  uint32_t b[8];
  if (K == 16) {  // no 16-mer ends before char 15: the first 15 chars only build state
    const uint4 a = q[0];
    tw_word<K, 4>(a.x, k, fwd, rc, nm, b, hmax);
    tw_word<K, 4>(a.y, k, fwd, rc, nm, b, hmax);
    tw_word<K, 4>(a.z, k, fwd, rc, nm, b, hmax);
    tw_word<K, 3>(a.w, k, fwd, rc, nm, b, hmax);
    v[0] = b[3];
    it = 1;
  }
#if MC_HALF_ITER_SLOT
  // (8 chars per iteration, as in sketch_slot_fast: a loop body that fits the
  // L0 instruction cache)
  const uint2* q2 = reinterpret_cast<const uint2*>(slot);
#pragma unroll 1
  for (uint32_t i2 = 2 * it; i2 < 2 * niter; ++i2) {
    const uint2 a = q2[i2];
    tw_word<K, 0>(a.x, k, fwd, rc, nm, b, hmax);
    tw_word<K, 0>(a.y, k, fwd, rc, nm, b + 4, hmax);
    bottom16_merge8(v, b, one);
  }
#else
#pragma unroll 1
  for (; it < niter; ++it) {
    const uint4 a = q[it];
    tw_word<K, 0>(a.x, k, fwd, rc, nm, b, hmax);
    tw_word<K, 0>(a.y, k, fwd, rc, nm, b + 4, hmax);
    bottom16_merge8(v, b, one);
    tw_word<K, 0>(a.z, k, fwd, rc, nm, b, hmax);
    tw_word<K, 0>(a.w, k, fwd, rc, nm, b + 4, hmax);
    bottom16_merge8(v, b, one);
  }
#endif
  bool exact = hmax != 0xffffffffu;
#pragma unroll
  for (int i = 0; i < 15; ++i) exact &= v[i] != v[i + 1] || v[i] == 0xffffffffu;
  return exact;
}

// Stage the warp's 32 windows (lane i: window start p, nch chars, 0 = none)
// into 32 consecutive slots, realigned to char 0 and padded with 'N' up to
// nwords (<= kSlotWords) words.  Lane l moves aligned source word l (lanes
// 0..4 also word 32 + l); 8 windows' loads are in flight at a time.
__device__ __forceinline__ uint32_t pad_tail(uint32_t x, int rem) {  // chars >= rem of the word -> 'N'
  if (rem >= 4) return x;
  return rem <= 0 ? 0x4e4e4e4eu : (x & (0xffffffffu >> (32 - 8 * rem))) | (0x4e4e4e4eu << (8 * rem));
}

__device__ __forceinline__ void stage_windows(uint32_t* __restrict__ wslots, const uint8_t* p, uint32_t nch,
                                              uint32_t nwords, uint32_t lane) {
  constexpr int kB = 8;
#pragma unroll 1
  for (uint32_t w0 = 0; w0 < 32; w0 += kB) {
    uint32_t lo[kB], lo1[kB], sh[kB], n[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      n[u] = __shfl_sync(kFull, nch, w0 + u);
      const uintptr_t a = (uintptr_t)__shfl_sync(kFull, (unsigned long long)(uintptr_t)p, w0 + u);
      const uint32_t* src = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
      sh[u] = (uint32_t)(a & 3u) * 8u;
      const uint32_t have = ((uint32_t)(a & 3u) + n[u] + 3) >> 2;  // aligned words holding the window
      lo[u] = lane < have ? __ldg(src + lane) : 0x4e4e4e4eu;
      lo1[u] = lane + 32 < have ? __ldg(src + 32 + lane) : 0x4e4e4e4eu;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      uint32_t* dst = wslots + (w0 + u) * kSlotWords;
      uint32_t hi = __shfl_down_sync(kFull, lo[u], 1);
      const uint32_t w32 = __shfl_sync(kFull, lo1[u], 0);
      if (lane == 31) hi = w32;
      dst[lane] = pad_tail(__funnelshift_r(lo[u], hi, sh[u]), (int)n[u] - (int)(4 * lane));
      if (nwords > 32) {  // windows longer than 128 chars
        const uint32_t hi1 = __shfl_down_sync(kFull, lo1[u], 1);
        if (lane < nwords - 32)
          dst[32 + lane] = pad_tail(__funnelshift_r(lo1[u], hi1, sh[u]), (int)n[u] - (int)(4 * (32 + lane)));
      }
    }
  }
}

// Bulk prefetch of [p, p + bytes) into L2 (TMA engine; no registers held),
// rounded out to 16-byte bounds.
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p);
  const uintptr_t lo = a & ~(uintptr_t)15;
  const uint32_t n = (uint32_t)(((a + bytes + 15) & ~(uintptr_t)15) - lo);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"(n) : "memory");
}

// ---- TMA bulk copies (global -> shared) completing on an mbarrier ----------
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one arrival that also expects `bytes` of transaction count
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "MC_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra MC_WAIT_%=;\n}\n" ::"r"(
          smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// dst, src 16-byte aligned; bytes a multiple of 16.  Orders the CTA's earlier
// generic-proxy accesses of dst before the async-proxy write.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

// Stage nchars contiguous chars starting at p0 (any alignment) into dst,
// realigned to char 0: word w = chars 4w..4w+3 (coalesced, 2 loads per word,
// the second an L1 hit).  Reads no aligned word beyond the span's last char.
__device__ __forceinline__ void stage_span(uint32_t* __restrict__ dst, const uint8_t* p0, uint32_t nchars,
                                           uint32_t lane) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p0);
  const uint32_t* src = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
  const uint32_t sh = (uint32_t)(a & 3u) * 8u;
  const uint32_t nsrc = ((uint32_t)(a & 3u) + nchars + 3) >> 2;  // aligned source words holding the span
  const uint32_t nout = (nchars + 3) >> 2;
#pragma unroll 4
  for (uint32_t w = lane; w < nout; w += 32) {
    const uint32_t lo = __ldg(src + w);
    const uint32_t hi = w + 1 < nsrc ? __ldg(src + w + 1) : 0x4e4e4e4eu;
    dst[w] = __funnelshift_r(lo, hi, sh);
  }
}

// Same result as stage_span for nchars <= 8 * 512 - 15, with every load in
// flight at once: lane l loads 16-byte chunks l, l + 32, ... (<= 8) of the
// aligned superset of the span, then realigns them with the next chunk's
// first word (shuffled from lane l + 1).  The chunk holding the span's last
// char is loaded word by word (no aligned word beyond the last char is read).
// One load round trip per span instead of one per 4 words per lane.
#ifndef MC_STAGE_WIDE
#define MC_STAGE_WIDE 1
#endif
__device__ __forceinline__ void stage_span_wide(uint32_t* __restrict__ dst, const uint8_t* p0, uint32_t nchars,
                                                uint32_t lane) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p0);
  const uint4* src = reinterpret_cast<const uint4*>(a & ~(uintptr_t)15);
  const uint32_t b0 = (uint32_t)(a & 15u);
  const uint32_t last = (b0 + nchars - 1) >> 4;           // chunk of the last char
  const uint32_t nsrcw = (b0 + nchars + 3) >> 2;          // aligned source words holding the span
  const int nout = (int)((nchars + 3) >> 2);
  uint4 ch[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t c = lane + 32u * k;
    if (c < last) {
      ch[k] = __ldg(src + c);
    } else {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(src + c);
      ch[k].x = c == last && 4 * c + 0 < nsrcw ? __ldg(w + 0) : 0x4e4e4e4eu;
      ch[k].y = c == last && 4 * c + 1 < nsrcw ? __ldg(w + 1) : 0x4e4e4e4eu;
      ch[k].z = c == last && 4 * c + 2 < nsrcw ? __ldg(w + 2) : 0x4e4e4e4eu;
      ch[k].w = c == last && 4 * c + 3 < nsrcw ? __ldg(w + 3) : 0x4e4e4e4eu;
    }
  }
  const uint32_t sh = (b0 & 3u) * 8u;
  const int wo = (int)(b0 >> 2);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    uint32_t nx = __shfl_down_sync(kFull, ch[k].x, 1);
    const uint32_t wrap = k < 7 ? __shfl_sync(kFull, ch[k < 7 ? k + 1 : k].x, 0) : 0x4e4e4e4eu;
    if (lane == 31) nx = wrap;
    const int base = 4 * (int)(lane + 32u * k) - wo;  // dst word of this chunk's first output word
    if (base >= nout) continue;
    const uint32_t o0 = __funnelshift_r(ch[k].x, ch[k].y, sh), o1 = __funnelshift_r(ch[k].y, ch[k].z, sh);
    const uint32_t o2 = __funnelshift_r(ch[k].z, ch[k].w, sh), o3 = __funnelshift_r(ch[k].w, nx, sh);
    if (wo == 0) {
      *reinterpret_cast<uint4*>(dst + base) = make_uint4(o0, o1, o2, o3);
    } else {
      if (base >= 0) dst[base] = o0;
      if (base + 1 >= 0) dst[base + 1] = o1;
      if (base + 2 >= 0) dst[base + 2] = o2;
      dst[base + 3] = o3;  // (base + 3 >= 0: wo <= 3)
    }
  }
}

// The warp's 32 windows (lane = window; nch = 0: none) -> v (ascending, first
// n valid).  `myslot` = this lane's staged slot, reused as scratch.
// kFilter: full windows take the candidate-filtered fast path with the
// warp's buffer `cand` (kCandRows x 32 words); otherwise the merge network
// over every feature (the query kernel, whose shared memory holds no buffer).
template <uint32_t K, bool kFilter = false>
__device__ __forceinline__ int sketch_warp_windows(uint32_t* wslots, const uint8_t* p, uint32_t nk,
                                                   const SketchCfg& c, uint32_t lane, uint32_t (&v)[16],
                                                   uint32_t* cand = nullptr) {
  const uint32_t nch = nk ? nk + c.k - 1 : 0u;
  const uint32_t niter = (c.stride + c.k - 1 + 15) >> 4;
  bool exact;
  const uint8_t* p0 = reinterpret_cast<const uint8_t*>(__shfl_sync(kFull, (unsigned long long)(uintptr_t)p, 0));
  if (K == 16 && c.stride == 112 && __all_sync(kFull, nch == 127 && p == p0 + 112 * lane)) {
    // 32 consecutive full windows of one target (the common case): stage their
    // contiguous span once; window i then starts 16-B aligned at byte 112 i
    if (MC_STAGE_WIDE) stage_span_wide(wslots, p0, 31 * 112 + 127, lane);
    else stage_span(wslots, p0, 31 * 112 + 127, lane);
    __syncwarp();
    exact = kFilter ? sketch_slot_filter(wslots + 28 * lane, c, cand + lane, v) : sketch_slot_fast(wslots + 28 * lane, c, v);
    __syncwarp();  // (the span is dead; the exact fallback below reuses the slots)
  } else {
    stage_windows(wslots, p, nch, niter * 4, lane);
    __syncwarp();
    if (K == 16 && c.stride == 112 && __all_sync(kFull, nch == 127 || nch == 0))  // full windows (warp-uniform)
      exact = (kFilter ? sketch_slot_filter(wslots + lane * kSlotWords, c, cand + lane, v)
                    : sketch_slot_fast(wslots + lane * kSlotWords, c, v)) || nch == 0;
    else
      exact = sketch_slot<K>(wslots + lane * kSlotWords, niter, c.k, c.p8 >> 8, v) || nch == 0;
  }
  uint32_t* myslot = wslots + lane * kSlotWords;
  int n = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) n += (uint32_t)i < c.s && v[i] != 0xffffffffu;
  if (nch == 0) n = 0;
  uint32_t redo = __ballot_sync(kFull, !exact);
  if (redo) {  // rare: re-sketch those windows with the exact warp routine
    const uint32_t mine = redo;
    while (redo) {
      const uint32_t o = __ffs(redo) - 1;
      redo &= redo - 1;
      const uint8_t* po = reinterpret_cast<const uint8_t*>(__shfl_sync(kFull, (unsigned long long)(uintptr_t)p, o));
      const uint32_t nko = __shfl_sync(kFull, nk, o);
      uint32_t f;
      const int cnt = sketch_words<true, K>(load_window(po, nko, c, lane), nko, c, lane, f,
                                            wslots + o * kSlotWords);
      if (lane == o) n = cnt;
    }
    __syncwarp();
    if (mine >> lane & 1u) {
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = (uint32_t)i < c.s ? myslot[i] : 0xffffffffu;
    }
  }
  return n;
}

// ---------------------------------------------------------------------------
// Multi-value hash table (D3/D4, Fig. 3; B200 redesign).
// Open addressing, one 8-byte slot per distinct feature:
//   key (bits 0..31) | count (bits 32..41, the key's bucket length <= cap)
//   | loff (bits 42..63, the bucket's offset from the first value of the
//   slot's sub-region; vbase[sub-region] holds that first value)
// -- the paper's condensed layout with sub-region-relative
// offsets so a slot fits one 8-byte word (four per 32 B sector).
// A slot is empty iff its count is 0 (a claimed slot has count >= 1), so every
// 32-bit key value is legal.  Built sub-region by sub-region in shared memory
// (finalize_kernels.cu); probing wraps inside the sub-region.
// ---------------------------------------------------------------------------
struct __align__(8) KSlot {
  unsigned long long kc;
};
constexpr uint32_t kSlotCntBits = 10, kSlotOffBits = 22;
constexpr uint32_t kMaxCap = (1u << kSlotCntBits) - 1u;               // cap <= 1023
constexpr uint64_t kMaxSubValues = (1ull << kSlotOffBits) - 1ull;     // values per sub-region
__host__ __device__ __forceinline__ uint32_t slot_key(unsigned long long w) { return (uint32_t)w; }
__host__ __device__ __forceinline__ uint32_t slot_cnt(unsigned long long w) {
  return (uint32_t)(w >> 32) & kMaxCap;
}
__host__ __device__ __forceinline__ uint32_t slot_loff(unsigned long long w) { return (uint32_t)(w >> 42); }
__host__ __device__ __forceinline__ unsigned long long make_slot(uint32_t key, uint32_t cnt, uint32_t loff) {
  return (unsigned long long)key | ((unsigned long long)cnt << 32) | ((unsigned long long)loff << 42);
}

// Condensed lookup: count of `key`'s bucket (0 if absent) and its offset.
__device__ __forceinline__ uint32_t keytable_find(const KSlot* __restrict__ T, const unsigned long long* vbase,
                                                  uint64_t n, uint32_t key, uint64_t* off) {
  uint64_t s = home_slot(key, n);
  for (uint32_t probes = 0; probes < kSubSlots; ++probes, s = next_slot(s)) {
    const unsigned long long e = __ldg(&T[s].kc);
    if (slot_cnt(e) == 0) return 0;
    if (slot_key(e) == key) {
      *off = vbase[s >> kSubLg] + slot_loff(e);
      return slot_cnt(e);
    }
  }
  return 0;
}

// index of the last element <= x in a sorted array a[0..n) (a[0] <= x assumed)
template <typename T>
__device__ __forceinline__ uint32_t upper_index(const T* __restrict__ a, uint32_t n, T x) {
  uint32_t lo = 0, hi = n;  // invariant: a[lo] <= x, answer in [lo, hi)
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}


// Segment of element g0 + lane, for a warp whose 32 lanes take consecutive
// elements: B[0..nseg] are the segments' first elements (B[nseg] = total).
// s0 (warp-uniform, carried between calls, never past g0's segment) is
// advanced to g0's segment -- a short walk, else a binary search -- and the
// lanes then add the boundaries that fall inside the warp's 32 elements.
template <typename T>
__device__ __forceinline__ uint32_t warp_segment(const T* __restrict__ B, uint32_t nseg, uint64_t total, uint64_t g0,
                                                 uint32_t& s0, uint32_t lane) {
  int steps = 0;
  while (s0 + 1 < nseg && B[s0 + 1] <= g0) {
    if (++steps > 8) {
      s0 += upper_index(B + s0, nseg - s0, (T)g0);
      break;
    }
    ++s0;
  }
  const uint64_t g = g0 + lane;
  const uint64_t bj = s0 + 1 + lane < nseg ? (uint64_t)B[s0 + 1 + lane] : ~0ull;
  uint32_t m = __ballot_sync(kFull, bj <= g0 + 31);
  if (m == kFull) return g < total ? upper_index(B, nseg + 1, (T)g) : s0;  // tiny segments
  uint32_t t = s0;
  while (m) {
    const uint32_t j = __ffs(m) - 1;
    m &= m - 1;
    t += __shfl_sync(kFull, bj, j) <= g;
  }
  return t;
}

// tiles [first, end) of CTA blockIdx.x: contiguous, so segments advance monotonically
__device__ __forceinline__ void cta_tiles(uint64_t ntiles, uint64_t* first, uint64_t* end) {
  *first = ntiles * blockIdx.x / gridDim.x;
  *end = ntiles * (blockIdx.x + 1) / gridDim.x;
}

}  // namespace mc
