// Fast CTC prefix beam-search decode kernel for beam <= 16 (the paper's and
// BASELINE.json's beam 10 configurations).  Same semantics as the generic
// kernel (ctcb_generic.cu) and the reference (ctcforge decoder.py:102-817),
// re-organised so that a frame step is a few hundred warp instructions:
//
//   * the beam lives in registers: lane e (< 16) holds entry e (rank order =
//     trellis slot), lanes 16..31 mirror the entries' parent hashes;
//   * one match.any over {prefix hash, parent hash} gives, per entry, the
//     other blank-flag variant of its prefix, its flag-0 children and its
//     parent prefix's entries (the merge structure of decoder.py:595-613);
//   * top-k: lane maxima -> bitonic sort -> threshold -> compaction ->
//     register bitonic sort of (log-prob desc, index asc) keys;
//   * selection: lanes 0..15 own <= 3 "special" groups each (blank, repeat,
//     last-token append), lanes 16..31 own one sorted append list per distinct
//     prefix; the next beam is popped with redux.sync.max on 32-bit
//     fixed-point keys (score - (best - beam_threshold)), exact fp64 compare
//     and token-sequence order on key ties (decoder.py:651-681);
//   * back-pointers go to the global trellis plus a 32-step shared-memory ring
//     that yields per-checkpoint ancestor slots, so the n-best backtrace is a
//     short coarse walk followed by 32-step walks in parallel lanes.
#include <cfloat>
#include <cmath>

#include "ctcb_common.cuh"
#include "ctcb_internal.h"
#include <cstdio>
// Debug builds (-DCTCB_FAST_CHECK): bounds / invariant checks that print the
// first few failures (compute-sanitizer is not available on the GPU pool).
#ifdef CTCB_FAST_CHECK
__device__ int g_fchk_count;
#define FCHK(c, a, b)                                                                                       \
  do {                                                                                                     \
    if (!(c) && atomicAdd(&g_fchk_count, 1) < 16)                                                          \
      printf("ctcb_fast check failed: %s (line %d, block %d, lane %d) %d %d\n", #c, __LINE__, blockIdx.x,     \
             (int)(threadIdx.x & 31), (int)(a), (int)(b));                                                 \
  } while (0)
#else
#define FCHK(c, a, b) do { } while (0)
#endif
// Diagnostics (-DCTCB_PHASES, with CTCB_UTT_TRACE set): lane 0 accumulates
// clock() cycles per frame phase; summed per launch after the utterance trace
// (tools/phase_cycles.py).
#ifdef CTCB_PHASES
#define PH(n)                                          \
  do {                                                 \
    if (P.utt_trace && lane == 0) {                    \
      const uint32_t t_ = (uint32_t)clock();           \
      ph_cyc[ph_cur] += t_ - ph_t;                     \
      ph_t = t_;                                       \
      ph_cur = (n);                                    \
    }                                                  \
  } while (0)
#else
#define PH(n) do { } while (0)
#endif

namespace ctcb {

namespace {

constexpr uint64_t kDummy = 0xa5a5a5a55a5a5a5aull;
constexpr uint32_t kSentinel = 0xffffffffu;  // a NaN whose order key is 0

// Order key of an fp32 log-prob: float order, -0 == +0, sentinel -> 0.
__device__ __forceinline__ uint32_t okey(float x) {
  uint32_t u = __float_as_uint(x);
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ double unord64(uint64_t k) {
  uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}
__device__ __forceinline__ uint64_t shfl64(uint64_t x, int src) {
  uint32_t lo = __shfl_sync(FULL, (uint32_t)x, src);
  uint32_t hi = __shfl_sync(FULL, (uint32_t)(x >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t shflx64(uint64_t x, int m) {
  uint32_t lo = __shfl_xor_sync(FULL, (uint32_t)x, m);
  uint32_t hi = __shfl_xor_sync(FULL, (uint32_t)(x >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}
// Register bitonic sorts across the warp, descending.
__device__ __forceinline__ uint32_t sort_desc32(uint32_t x, int lane) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      uint32_t y = __shfl_xor_sync(FULL, x, j);
      bool take_max = ((lane & j) == 0) == ((lane & size) == 0);
      x = take_max ? max(x, y) : min(x, y);
    }
  return x;
}
__device__ __forceinline__ uint64_t sort_desc64(uint64_t x, int lane) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1)
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      uint64_t y = shflx64(x, j);
      bool take_max = ((lane & j) == 0) == ((lane & size) == 0);
      x = take_max ? (x > y ? x : y) : (x < y ? x : y);
    }
  return x;
}
// Descending sort of 32 keys by rank counting through shared memory
// (`sc`: 64 words): every lane reads all keys with 8 broadcast LDS.128,
// counts the larger ones and scatters its key to that rank.  About as many
// instructions as the 15-stage shuffle network but ~1/3 of its latency; the
// latency-bound small-batch walks (precomputed top-k mode) use it.  Nonzero
// keys must be distinct (they carry slot tags); zero keys sort last.
__device__ __forceinline__ uint32_t sort_desc32_rank(uint32_t x, int lane, uint32_t* sc) {
  sc[lane] = x;
  __syncwarp();
  const uint4* s4 = (const uint4*)sc;
  int r0 = 0, r1 = 0, r2 = 0, r3 = 0;
#pragma unroll
  for (int q = 0; q < 8; q++) {
    const uint4 v = s4[q];
    r0 += v.x > x ? 1 : 0;
    r1 += v.y > x ? 1 : 0;
    r2 += v.z > x ? 1 : 0;
    r3 += v.w > x ? 1 : 0;
  }
  sc[32 + lane] = 0u;
  __syncwarp();
  if (x) sc[32 + ((r0 + r1) + (r2 + r3))] = x;
  __syncwarp();
  const uint32_t y = sc[32 + lane];
  __syncwarp();
  return y;
}
// Sort a bitonic sequence descending.
__device__ __forceinline__ uint64_t merge_desc64(uint64_t x, int lane) {
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) {
    uint64_t y = shflx64(x, j);
    x = ((lane & j) == 0) ? (x > y ? x : y) : (x < y ? x : y);
  }
  return x;
}
__device__ __forceinline__ int warp_incl_scan(int x, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  return x;
}

struct FastSmem {
  uint8_t* rows;
  uint64_t* mbar;
  uint64_t* cand;
  double* tie_sc;
  uint64_t* hs;
  float* sval;
  int *stok, *rec_i, *tie_i, *hl;
  uint32_t *excl, *tring, *hist;
  uint8_t* posmap;
  uint64_t* tc_h;
  int* tc_r;
  uint32_t* gkey;
  double* hsc;
  int* hp2;
  int* dlane;
  double* dA;
  uint32_t* dgv;
  long long* wp;
  uint32_t* ckey;
  uint16_t* cidx;
  int* slot_rec;
  long long* dG;
};

// Tie-order cache: prefix hashes identify token sequences globally, so a
// cached "seq(h1) vs seq(h2)" stays valid for the whole decode (and across
// utterances).  Sibling prefixes with identical scores (a duplicated fp32
// value in some row) tie again every frame; the cache answers those without
// re-reading their sequences.
// 4-way set associative (kTieCache / 4 sets): the set of a pair is a
// symmetric hash of the two prefix hashes, so a lookup is four probes (a
// persistent exact tie asks every frame); each set replaces round-robin
// (2-bit cursors packed in tc_r[kTieCache]).
__device__ __forceinline__ int tc_set(uint64_t ha, uint64_t hb) {
  const uint64_t x = (ha ^ hb) * 0x9e3779b97f4a7c15ull;
  return (int)(x >> 59) & (kTieCache / 4 - 1);
}
__device__ int tc_lookup(const FastSmem& S, uint64_t ha, uint64_t hb) {
  const int s0 = 4 * tc_set(ha, hb);
#pragma unroll
  for (int w = 0; w < 4; w++) {
    const uint64_t a = S.tc_h[2 * (s0 + w)], b = S.tc_h[2 * (s0 + w) + 1];
    if (a == ha && b == hb) return S.tc_r[s0 + w];
    if (a == hb && b == ha) return -S.tc_r[s0 + w];
  }
  return 0;
}
__device__ void tc_insert(const FastSmem& S, uint64_t ha, uint64_t hb, int r) {
  if (tc_lookup(S, ha, hb)) return;
  const int set = tc_set(ha, hb);
  const uint32_t cur = (uint32_t)S.tc_r[kTieCache];
  const int w = (int)((cur >> (2 * set)) & 3u);
  const int i = 4 * set + w;
  S.tc_h[2 * i] = ha;
  S.tc_h[2 * i + 1] = hb;
  S.tc_r[i] = r;
  S.tc_r[kTieCache] = (int)((cur & ~(3u << (2 * set))) | ((uint32_t)((w + 1) & 3) << (2 * set)));
}
__device__ int fast_seq_cmp_full(const Params& P, const FastSmem& S, int u, int steps_done, int ea, int xa, int eb,
                                 int xb, bool* strict);
// Python tuple order of seq(ea)+[xa] vs seq(eb)+[xb]; hs/hl hold the hashes and
// lengths of the current entries.  Orders of sequence pairs that differ
// before the end of the shorter one ("strict") are cached: every extension of
// such a pair keeps the order, so a tie that recurs on the next frame between
// their descendants is answered from the cache.
__device__ int fast_seq_cmp(const Params& P, const FastSmem& S, int u, int steps_done, int ea, int xa, int eb,
                            int xb) {
  const uint64_t hba = S.hs[ea], hbb = S.hs[eb];
  const int lba = S.hl[ea], lbb = S.hl[eb];
  if (hba == hbb && lba == lbb) {  // same base prefix: compare the extra tokens
    if (xa == xb) return 0;
    return xa < xb ? -1 : 1;
  }
  const uint64_t ha = xa >= 0 ? child_hash(hba, xa) : hba, hb = xb >= 0 ? child_hash(hbb, xb) : hbb;
  const int la = lba + (xa >= 0), lb = lbb + (xb >= 0);
  if (ha == hb && la == lb) return 0;  // identical sequences (e.g. (R,c) vs (R+c))
  int r = tc_lookup(S, hba, hbb);
  if (r) {
    tc_insert(S, ha, hb, r);
    return r;
  }
  r = tc_lookup(S, ha, hb);
  if (r) return r;
  bool strict = false;
  r = fast_seq_cmp_full(P, S, u, steps_done, ea, -1, eb, -1, &strict);
  if (strict) {
    tc_insert(S, hba, hbb, r);
    tc_insert(S, ha, hb, r);
    return r;
  }
  r = fast_seq_cmp_full(P, S, u, steps_done, ea, xa, eb, xb, &strict);
  if (strict) tc_insert(S, ha, hb, r);
  return r;
}
__device__ int fast_seq_cmp_full(const Params& P, const FastSmem& S, int u, int steps_done, int ea, int xa, int eb,
                                 int xb, bool* strict) {
  int* A = P.seqbuf + (size_t)u * 3 * (P.T_max + 1);
  const uint32_t* tr = P.trellis + (size_t)u * P.T_max * P.beam;
  auto rec = [&](int i, int slot) {
    const uint32_t r = tr[(size_t)i * P.beam + slot];
    return make_int2(trel_tok(r), trel_src(r));
  };
  return trellis_seq_cmp(rec, steps_done, ea, xa, eb, xb, A, A + P.T_max + 1, strict, P.dbg);
}
// a precedes b in the reference's rank order: score desc, sequence asc, flag asc.
__device__ bool fast_precedes(const Params& P, const FastSmem& S, int u, int sd, double sa, int ba, int xa, int fa,
                              double sb, int bb, int xb, int fb) {
  if (sa != sb) return sa > sb;
  atomicAdd(&P.dbg[kDbgExactTies], 1ull);
  int c = fast_seq_cmp(P, S, u, sd, ba, xa, bb, xb);
  if (c) return c < 0;
  return fa < fb;
}

// Exact top-k fallback (rows with > 64 candidates above the lane-max
// threshold, e.g. many exactly tied values): 8-bit radix select on the order
// keys, ordered compaction, register sort.  Returns this lane's S key.
template <class KeyOf>
__device__ uint64_t topk_radix_f(const FastSmem& S, KeyOf key_of, int V, int k, int lane) {
  uint32_t prefix = 0, pmask = 0;
  int need = k;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = lane; b < 256; b += 32) S.hist[b] = 0;
    __syncwarp();
    for (int c = lane; c < V; c += 32) {
      uint32_t key = key_of(c);
      if (key && (key & pmask) == prefix) atomicAdd(&S.hist[(key >> shift) & 255u], 1u);
    }
    __syncwarp();
    uint32_t h[8], s = 0;
#pragma unroll
    for (int q = 0; q < 8; q++) { h[q] = S.hist[lane * 8 + q]; s += h[q]; }
    uint32_t incl = s;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      uint32_t v = __shfl_down_sync(FULL, incl, off);
      if (lane + off < 32) incl += v;
    }
    uint32_t cum = incl - s;
    int found = -1;
    uint32_t cgt = 0;
#pragma unroll
    for (int q = 7; q >= 0; q--) {
      if (found < 0 && cum < (uint32_t)need && cum + h[q] >= (uint32_t)need) { found = lane * 8 + q; cgt = cum; }
      cum += h[q];
    }
    unsigned bal = __ballot_sync(FULL, found >= 0);
    int src = __ffs(bal) - 1;
    int digit = __shfl_sync(FULL, found, src);
    cgt = __shfl_sync(FULL, cgt, src);
    need -= (int)cgt;
    prefix |= (uint32_t)digit << shift;
    pmask |= 0xffu << shift;
    __syncwarp();
  }
  const uint32_t kth = prefix;
  int n = 0, eq_taken = 0;
  const unsigned lt = lanemask_lt();
  for (int c0 = 0; c0 < V; c0 += 32) {
    int c = c0 + lane;
    uint32_t key = c < V ? key_of(c) : 0u;
    bool gt = key > kth, eq = key != 0u && key == kth;
    unsigned beq = __ballot_sync(FULL, eq);
    bool acc = gt || (eq && eq_taken + __popc(beq & lt) < need);
    unsigned bsel = __ballot_sync(FULL, acc);
    if (acc) S.cand[n + __popc(bsel & lt)] = ((uint64_t)key << 32) | (uint64_t)(0xffffffffu - (uint32_t)c);
    n += __popc(bsel);
    eq_taken += __popc(beq);
  }
  __syncwarp();
  uint64_t x = lane < n ? S.cand[lane] : 0ull;
  __syncwarp();
  return sort_desc64(x, lane);
}
__device__ uint64_t topk_radix(const FastSmem& S, const float* row, int V, int k, int lane) {
  return topk_radix_f(S, [&](int c) { return okey(row[c]); }, V, k, lane);
}
// The same for the SMALL kernels, out of line (rows with > 64 values above the
// lane-maximum threshold, e.g. many exact ties): scalar / pointer arguments
// only, so the hot frame loop keeps its registers and loses ~0.5k instructions
// of code it almost never runs.
__device__ __noinline__ uint64_t topk_radix_ool(const float* row, uint32_t* hist, uint64_t* cand, int V, int k,
                                                int lane) {
  FastSmem T{};
  T.hist = hist;
  T.cand = cand;
  return topk_radix_f(T, [&](int c) { return okey(row[c]); }, V, k, lane);
}

}  // namespace

// Blank-skip compaction of one utterance by one warp: ballot + prefix
// popcount over the blank column (emissions.py:298-306).  Returns the kept count.
__device__ __forceinline__ int frame_map_warp(const Params& P, const float* ubase, int len_u, int32_t* fmap, int lane) {
  int kept = 0;
  for (int t0 = 0; t0 < len_u; t0 += 32) {
    int t = t0 + lane;
    bool keep = t < len_u;
    if (keep && P.skip) keep = !(__ldg(ubase + (size_t)t * P.stride_t + P.blank) >= P.cutoff);
    unsigned bal = __ballot_sync(FULL, keep);
    if (keep) fmap[kept + __popc(bal & lanemask_lt())] = t;
    kept += __popc(bal);
  }
  return kept;
}

// Top-k of one staged row (blank and padding hold kSentinel), general path:
// threshold = k-th largest lane maximum (>= k elements reach it),
// compaction of the <= 64 elements above it, register bitonic sort of
// (log-prob desc, index asc) 64-bit keys; > 64 survivors take the radix
// select.  Returns this lane's key of S (lanes < k).
__device__ __forceinline__ uint64_t topk_key(const FastSmem& S, const float* row, int V, int k, int lane, bool small_v,
                                             int nch4, unsigned long long* dbg) {
  const float4* row4 = (const float4*)row;
  float lmax = __uint_as_float(kSentinel);
  for (int c = lane; c < nch4; c += 32) {
    float4 q = row4[c];
    lmax = fmaxf(lmax, fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w)));
  }
  const uint32_t t0 = __shfl_sync(FULL, sort_desc32(isnan(lmax) ? 0u : okey(lmax), lane), k - 1);
  const float tf = t0 == 0u ? -INFINITY : unord32(t0);
  uint32_t pm = 0u;  // predicate bits (V <= 1024: chunk j of this lane -> bits 4j..4j+3)
  int cl = 0;
  if (small_v) {
    int j = 0;
    for (int c = lane; c < nch4; c += 32, j += 4) {
      float4 q = row4[c];
      pm |= ((uint32_t)(q.x >= tf) | ((uint32_t)(q.y >= tf) << 1) | ((uint32_t)(q.z >= tf) << 2) |
             ((uint32_t)(q.w >= tf) << 3)) << j;
    }
    cl = __popc(pm);
  } else {
    for (int c = lane; c < nch4; c += 32) {
      float4 q = row4[c];
      cl += (q.x >= tf) + (q.y >= tf) + (q.z >= tf) + (q.w >= tf);
    }
  }
  const int cnt = __reduce_add_sync(FULL, cl);
  uint64_t skey;
  // cnt < k only when NaN values (invalid input, never >= tf) leave too few
  // survivors: the radix select then keeps every index in range
  if (cnt <= 64 && cnt >= k) {
    int off = warp_incl_scan(cl, lane) - cl;
    if (small_v) {
      while (pm) {
        const int bt = __ffs(pm) - 1;
        pm &= pm - 1u;
        const int e = 4 * (lane + 32 * (bt >> 2)) + (bt & 3);
        S.cand[off++] = ((uint64_t)okey(row[e]) << 32) | (uint64_t)(0xffffffffu - (uint32_t)e);
      }
    } else {
      for (int c = lane; c < nch4; c += 32) {
        float4 q = row4[c];
        float vv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int z = 0; z < 4; z++)
          if (vv[z] >= tf)
            S.cand[off++] = ((uint64_t)okey(vv[z]) << 32) | (uint64_t)(0xffffffffu - (uint32_t)(4 * c + z));
      }
    }
    __syncwarp();
    uint64_t a = lane < cnt ? S.cand[lane] : 0ull;
    uint64_t b = lane + 32 < cnt ? S.cand[lane + 32] : 0ull;
    __syncwarp();
    a = sort_desc64(a, lane);
    if (cnt > 32) {
      b = sort_desc64(b, lane);
      uint64_t br = shfl64(b, 31 - lane);
      a = a > br ? a : br;
      a = merge_desc64(a, lane);
    }
    skey = a;
  } else {
    if (lane == 0 && dbg) atomicAdd(&dbg[kDbgRadix], 1ull);
    skey = topk_radix(S, row, V, k, lane);
  }
  return skey;
}
// Top-k of one row read straight from global memory (large V, frame-parallel
// kernel): the passes of topk_key with the blank column masked on the fly, so
// nothing is staged in shared memory and many more warps fit per SM (the
// passes after the first hit L1/L2).  Requires V % 4 == 0 and a 16-B aligned row.
__device__ __forceinline__ uint64_t topk_key_g(const FastSmem& S, const float* __restrict__ grow, int V, int blank,
                                               int k, int lane, unsigned long long* dbg) {
  const float4* g4 = (const float4*)grow;
  const int nch4 = V >> 2;
  const float sent = __uint_as_float(kSentinel);
  auto ld = [&](int c) -> float4 {
    float4 q = __ldg(g4 + c);
    const int b = blank - 4 * c;
    if (b == 0) q.x = sent;
    if (b == 1) q.y = sent;
    if (b == 2) q.z = sent;
    if (b == 3) q.w = sent;
    return q;
  };
  float lmax = sent;
  for (int c = lane; c < nch4; c += 32) {
    const float4 q = ld(c);
    lmax = fmaxf(lmax, fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w)));
  }
  const uint32_t t0 = __shfl_sync(FULL, sort_desc32(isnan(lmax) ? 0u : okey(lmax), lane), k - 1);
  const float tf = t0 == 0u ? -INFINITY : unord32(t0);
  int cl = 0;
  for (int c = lane; c < nch4; c += 32) {
    const float4 q = ld(c);
    cl += (q.x >= tf) + (q.y >= tf) + (q.z >= tf) + (q.w >= tf);
  }
  const int cnt = __reduce_add_sync(FULL, cl);
  if (cnt > 64 || cnt < k) {  // cnt < k: NaN input (see topk_key)
    if (lane == 0 && dbg) atomicAdd(&dbg[kDbgRadix], 1ull);
    return topk_radix_f(S, [&](int c) { return c == blank ? 0u : okey(__ldg(grow + c)); }, V, k, lane);
  }
  int off = warp_incl_scan(cl, lane) - cl;
  for (int c = lane; c < nch4; c += 32) {
    const float4 q = ld(c);
    const float vv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int z = 0; z < 4; z++)
      if (vv[z] >= tf) S.cand[off++] = ((uint64_t)okey(vv[z]) << 32) | (uint64_t)(0xffffffffu - (uint32_t)(4 * c + z));
  }
  __syncwarp();
  uint64_t a = lane < cnt ? S.cand[lane] : 0ull;
  uint64_t bq = lane + 32 < cnt ? S.cand[lane + 32] : 0ull;
  __syncwarp();
  a = sort_desc64(a, lane);
  if (cnt > 32) {
    bq = sort_desc64(bq, lane);
    const uint64_t br = shfl64(bq, 31 - lane);
    a = a > br ? a : br;
    a = merge_desc64(a, lane);
  }
  return a;
}
__device__ __forceinline__ int skey_tok(uint64_t skey) { return (int)(0xffffffffu - (uint32_t)(skey & 0xffffffffu)); }

// Sort a bitonic sequence of 32-bit keys descending.
__device__ __forceinline__ uint32_t merge_desc32(uint32_t x, int lane) {
#pragma unroll
  for (int j = 16; j > 0; j >>= 1) {
    uint32_t y = __shfl_xor_sync(FULL, x, j);
    x = ((lane & j) == 0) ? max(x, y) : min(x, y);
  }
  return x;
}

// Top-k of one staged row for V <= 512 (<= 4 float4 chunks per lane) and
// k <= 31, with 32-bit sort keys.  The chunks stay in registers between the
// lane-maximum pass and the predicate pass; survivors (>= threshold) are
// compacted in token-index order (per-chunk counts packed into one scan), so a
// survivor's slot q orders ties by index.  Sort key = (order key with its low
// 6 bits cleared) | (63 - q): value desc, then index asc, exact unless two
// values collide after truncation; adjacent collisions in the top k+1 take the
// exact 64-bit path (~1-2 % of rows).  Returns the token of rank `lane`
// (lanes < k).
__device__ __forceinline__ int topk_small(const FastSmem& S, const float* row, int V, int k, int lane, int nch4,
                                          unsigned long long* dbg) {
  const float4* row4 = (const float4*)row;
  const float sent = __uint_as_float(kSentinel);
  float4 q[4];
  float lmax = sent;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    q[j] = row4[lane + 32 * j];  // rows are padded to 512 floats
    lmax = fmaxf(lmax, fmaxf(fmaxf(q[j].x, q[j].y), fmaxf(q[j].z, q[j].w)));
  }
  const uint32_t t0 = __shfl_sync(FULL, sort_desc32(isnan(lmax) ? 0u : okey(lmax), lane), k - 1);
  const float tf = t0 == 0u ? -INFINITY : unord32(t0);
  uint32_t pm = 0u, packed = 0u;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const uint32_t nib = (uint32_t)(q[j].x >= tf) | ((uint32_t)(q[j].y >= tf) << 1) |
                         ((uint32_t)(q[j].z >= tf) << 2) | ((uint32_t)(q[j].w >= tf) << 3);
    pm |= nib << (4 * j);
    packed |= (uint32_t)__popc(nib) << (8 * j);
  }
  const int cnt = __reduce_add_sync(FULL, __popc(pm));
  if (cnt > 64 || cnt < k) {  // cnt < k: NaN input (see topk_key)
    if (lane == 0 && dbg) atomicAdd(&dbg[kDbgRadix], 1ull);
    const uint64_t sk = topk_radix_ool(row, S.hist, S.cand, V, k, lane);
    return skey_tok(sk);
  }
  // per-chunk exclusive offsets: chunk j of lane l starts after all survivors
  // of chunks < j (every lane) and of chunk j in lanes < l
  uint32_t incl = packed;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t tot = __shfl_sync(FULL, incl, 31);
  uint32_t offs = tot * 0x01010100u + (incl - packed);
  uint16_t* cidx = S.cidx;
  while (pm) {
    const int bt = __ffs(pm) - 1;
    pm &= pm - 1u;
    const int sh = 8 * (bt >> 2);
    const uint32_t off = (offs >> sh) & 0xffu;
    offs += 1u << sh;
    cidx[off] = (uint16_t)(4 * (lane + 32 * (bt >> 2)) + (bt & 3));
  }
  __syncwarp();
  // slot q holds the q-th survivor in index order: key = truncated value | 63 - q
  uint32_t a = lane < cnt ? ((okey(row[cidx[lane]]) & ~63u) | (uint32_t)(63 - lane)) : 0u;
  a = sort_desc32(a, lane);
  if (cnt > 32) {
    uint32_t b = lane + 32 < cnt ? ((okey(row[cidx[lane + 32]]) & ~63u) | (uint32_t)(31 - lane)) : 0u;
    b = sort_desc32(b, lane);
    a = max(a, __shfl_sync(FULL, b, 31 - lane));
    a = merge_desc32(a, lane);
  }
  // exactness: keys that differ after truncation are ordered exactly
  const uint32_t an = __shfl_down_sync(FULL, a, 1);
  const bool bad = lane < k && a != 0u && (a >> 6) == (an >> 6);
  int tok;
  if (__any_sync(FULL, bad)) {
    if (lane == 0 && dbg) atomicAdd(&dbg[kDbgTopkFix], 1ull);
    const int ia = lane < cnt ? cidx[lane] : 0, ib = lane + 32 < cnt ? cidx[lane + 32] : 0;
    uint64_t x = lane < cnt ? (((uint64_t)okey(row[ia]) << 32) | (uint64_t)(0xffffffffu - (uint32_t)ia)) : 0ull;
    x = sort_desc64(x, lane);
    if (cnt > 32) {
      uint64_t y = lane + 32 < cnt ? (((uint64_t)okey(row[ib]) << 32) | (uint64_t)(0xffffffffu - (uint32_t)ib)) : 0ull;
      y = sort_desc64(y, lane);
      const uint64_t yr = shfl64(y, 31 - lane);
      x = x > yr ? x : yr;
      x = merge_desc64(x, lane);
    }
    tok = skey_tok(x);
  } else {
    tok = cidx[63u - (a & 63u)];
  }
  __syncwarp();
  return tok;
}

#ifndef CTCB_FAST_MIN_BLOCKS
#define CTCB_FAST_MIN_BLOCKS 4
#endif

// Rank keys are 32-bit fixed point: key(x) ~ (x - (best - R)) * 2^32 / R,
// R = beam_threshold (2^20 when infinite); 0 = dropped (-inf), 1 = at or below
// the floor.  Append keys are the clamped sum of a per-list term floor((A -
// base) * 2^32/R) and a per-position term floor(v * 2^32/R) (64-bit integer
// add instead of fp64 per candidate), so a key can be off by up to 2 units:
// heads within kTol of the maximum are resolved exactly (fp64 fold, then
// token-sequence order), as are keys within kTol of the floor (the exact
// threshold test, decoder.py:621-623).
constexpr uint32_t kTol = 3u;


__device__ __forceinline__ uint32_t f2u_sat(double z) {
  uint32_t r;
  asm("cvt.rzi.u32.f64 %0, %1;" : "=r"(r) : "d"(z));  // saturating: < 0 -> 0, >= 2^32 -> 2^32 - 1
  return r;
}
__device__ __forceinline__ long long f2ll_floor(double z) {
  long long r;
  asm("cvt.rmi.s64.f64 %0, %1;" : "=l"(r) : "d"(z));  // saturating; -inf -> INT64_MIN
  return r;
}

// Exact order of close-key runs with exactly equal scores: token sequence,
// then flag (decoder.py:651-681), by lane 0 (insertion sort with
// fast_precedes); lanes < beam then write the new beam's merge records.
__device__ __forceinline__ void serial_runs(const Params& P, const FastSmem& S, int u, int i, int beam, int lane,
                                         uint64_t h, int len, double es, int ba, int xa, int fa, int rec,
                                         unsigned cm, int bmax) {
  int* pi = (int*)S.cand;
  if (lane <= bmax) {
    S.tie_sc[lane] = es;
    S.tie_i[lane * 4 + 0] = ba;
    S.tie_i[lane * 4 + 1] = xa;
    S.tie_i[lane * 4 + 2] = fa;
    S.tie_i[lane * 4 + 3] = rec;
    pi[lane] = lane;
  }
  if (lane < 16) { S.hs[lane] = h; S.hl[lane] = len; }
  __syncwarp();
  if (lane == 0) {
    for (int a = 0; a <= bmax;) {
      int b = a;
      while (b < bmax && ((cm >> b) & 1u)) b++;
      for (int q = a + 1; q <= b; q++) {  // insertion sort of positions a..b
        const int x = pi[q];
        int r = q;
        while (r > a) {
          const int y = pi[r - 1];
          if (!fast_precedes(P, S, u, i, S.tie_sc[x], S.tie_i[x * 4], S.tie_i[x * 4 + 1], S.tie_i[x * 4 + 2],
                             S.tie_sc[y], S.tie_i[y * 4], S.tie_i[y * 4 + 1], S.tie_i[y * 4 + 2]))
            break;
          pi[r] = y;
          r--;
        }
        pi[r] = x;
      }
      a = b + 1;
    }
  }
  __syncwarp();
  if (lane < beam) S.rec_i[lane] = lane <= bmax ? S.tie_i[pi[lane] * 4 + 3] : rec;
  __syncwarp();
}

// Exact order inside runs of close keys (rare; a persistent near-tie between
// two beam entries recurs every frame).  Lane p holds the p-th largest sorted
// key; `cl` marks (p, p+1) as possibly misordered and `es` is the exact fp64
// score of lane p's candidate.  Keys of different runs are ordered exactly, so
// only the runs up to the beam cut are re-ranked by exact score
// (decoder.py:651-681).  Returns 1 with `pos` = the candidate's exact rank,
// 0 when the run at the cut reaches lane 31 (candidates beyond the warp are
// not visible), 2 when a run holds exactly equal scores (token-sequence
// order needed).  cm / bmax: run links and the last position that matters.
__device__ __forceinline__ int close_runs_rank(bool cl, double es, int beam, int lane, int& pos, unsigned& cm,
                                               int& bmax) {
  cm = __ballot_sync(FULL, cl);
  bmax = beam - 1 + (__ffs(~(cm >> (beam - 1))) - 1);  // end of the run holding beam - 1
  const unsigned starts = ~(cm << 1);
  const int rs = 31 - __clz(starts & (0xffffffffu >> (31 - lane)));
  const unsigned after = lane < 31 ? starts & (0xfffffffeu << lane) : 0u;
  const int re = after ? __ffs(after) - 2 : 31;
  int rank = 0;
  bool tie = false;
#pragma unroll 1
  for (int q = 0; q < 32; q++) {
    const double eq = __shfl_sync(FULL, es, q);
    if (q <= bmax && q != lane && q >= rs && q <= re) {
      rank += eq > es ? 1 : 0;
      tie |= eq == es;
    }
  }
  const bool any_tie = __any_sync(FULL, tie && lane <= bmax);
  pos = lane <= bmax ? rs + rank : lane;
  return bmax >= 31 ? 0 : (any_tie ? 2 : 1);
}

// SMALL: V <= 512, ring 2, rows of 2048 B -- the shared-memory layout is a
// compile-time constant (immediate offsets from one base register).
template <bool PRE, bool SMALL>
__device__ __forceinline__ void fast_decode(const Params& P) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int me = lane & 15;
  const FastLayout L = SMALL ? make_fast_layout(kSmallV, 2, kSmallRowBytes) : make_fast_layout(P.V, P.ring, P.row_bytes);
  uint8_t* wbase = smem + (size_t)wid * (SMALL ? L.total : (size_t)P.smem_per_warp);
  FastSmem S;
  S.rows = wbase + L.rows;
  S.mbar = (uint64_t*)(wbase + L.mbar);
  S.cand = (uint64_t*)(wbase + L.cand);
  S.tie_sc = (double*)(wbase + L.tie_sc);
  S.hs = (uint64_t*)(wbase + L.hs);
  S.sval = (float*)(wbase + L.sval);
  S.stok = (int*)(wbase + L.stok);
  S.excl = (uint32_t*)(wbase + L.excl);
  S.rec_i = (int*)(wbase + L.rec_i);
  S.tie_i = (int*)(wbase + L.tie_i);
  S.hl = (int*)(wbase + L.hl);
  S.tring = (uint32_t*)(wbase + L.ring);
  S.hist = (uint32_t*)(wbase + L.hist);
  S.posmap = wbase + L.posmap;
  S.tc_h = (uint64_t*)(wbase + L.tc_h);
  S.tc_r = (int*)(wbase + L.tc_r);
  S.hsc = (double*)(wbase + L.hsc);
  S.hp2 = (int*)(wbase + L.hp2);
  S.dlane = (int*)(wbase + L.dlane);
  S.dA = (double*)(wbase + L.dA);
  S.dgv = (uint32_t*)(wbase + L.dgv);
  S.wp = (long long*)(wbase + L.wp);
  S.ckey = (uint32_t*)(wbase + L.ckey);
  S.cidx = (uint16_t*)(wbase + L.cidx);
  S.slot_rec = (int*)(wbase + L.slot_rec);
  S.dG = (long long*)(wbase + L.dG);
  for (int i = lane; i < 2 * kTieCache; i += 32) S.tc_h[i] = 0ull;
  for (int i = lane; i <= kTieCache; i += 32) S.tc_r[i] = 0;

  const int V = P.V, k = P.k, beam = P.beam, ring = SMALL ? 2 : P.ring;
  // rows staged by TMA (16-B aligned rows): the host picks SMALL only then
  const bool bulk = SMALL || P.bulk_ok;
  const bool MX = P.merge_max != 0;  // merge_mode="max" (decoder.py:610-613)
  // beam_size_token < V runs on the general-layout kernels only (the host never
  // picks a SMALL variant for it), so its code is compiled out of SMALL
  const int tokK = SMALL ? 0 : P.tokK;
  const int row_bytes = SMALL ? kSmallRowBytes : P.row_bytes;
  const int nch4 = (V + 3) >> 2;
  const bool small_v = SMALL || nch4 <= 256;      // general path: predicate bits fit one register
  // topk_small (<= 4 chunks per lane, k <= 31): the host picks SMALL only for
  // k <= 31, so this is a compile-time constant (no per-frame test, and the
  // general top-k is compiled out of the SMALL kernels)
  const bool tiny_v = SMALL;
  const uint32_t fullk = k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
  const double kR = P.threshold_inf ? 1048576.0 : fmin(P.beam_threshold, 1048576.0);
  const double kScale = 4294967296.0 / kR;
  // one-shot selection quota table: append slot `lane` -> (prefix d, j-th valid position)
  int ldj = 0xff;
  for (int d = 0, off = 0; d < beam && beam <= 10; d++) {
    const int q = beam / (d + 1);
    if (lane >= off && lane < off + q) ldj = d | ((lane - off) << 4);
    off += q;
  }

  if (lane == 0)
    for (int s = 0; s < ring; s++) mbar_init(&S.mbar[s], 1);
  for (int c = lane; c < V; c += 32) S.posmap[c] = 0xff;
  // padding beyond V is never written by the row copies: sentinel it once
  // (SMALL with V > 384: -FLT_MAX, below every log-prob and neutral for the
  // input screen, so the screen needs no bounds checks; every lane holds real
  // values for the top-k threshold and the radix fallback reads only c < V)
  // (V <= 384 keeps the NaN sentinel: whole lanes of padding must not feed
  // the top-k threshold)
  const bool padded = SMALL && P.V > 384;
  const uint32_t pad = padded ? __float_as_uint(-FLT_MAX) : kSentinel;
  for (int s = 0; s < ring; s++)
    for (int c = V + lane; c < row_bytes / 4; c += 32) ((uint32_t*)(S.rows + (size_t)s * row_bytes))[c] = pad;
  fence_mbar_init();
  __syncwarp();
  int slot_i = 0, slot_c = 0;     // ring slots of the next issue / consume
  uint32_t par_c = 0u;            // mbarrier phase parity of the consume slot
  const uint32_t row_copy = (uint32_t)V * 4u;

  int tr_u = -1;  // diagnostics timeline (P.utt_trace): utterance in progress
#ifdef CTCB_PHASES
  unsigned long long ph_cyc[16] = {};
  uint32_t ph_t = 0;
  int ph_cur = 15;
#endif
  auto tr_end = [&]() {
    if (P.utt_trace && tr_u >= 0 && lane == 0) P.utt_trace[2 * (size_t)tr_u + 1] = globaltimer_ns();
#ifdef CTCB_PHASES
    if (P.utt_trace && tr_u >= 0 && lane == 0)
      for (int q = 0; q < 16; q++) atomicAdd(&P.utt_trace[2 * (size_t)P.B + q], ph_cyc[q]);
    if (lane == 0)
      for (int q = 0; q < 16; q++) ph_cyc[q] = 0;
#endif
  };
  for (;;) {
    tr_end();
    int item = 0;
    if (lane == 0) item = atomicAdd(P.counter, 1);
    item = __shfl_sync(FULL, item, 0);
    if (item >= P.B) {
      // overlapped top-k: this grid completes only after the top-k grid has
      // (its validation keys and lists are then visible to later stream work)
      if (PRE && P.ready != nullptr) pdl_wait_primary();
      break;
    }
    const int u = P.order[item];
    const int len_u = P.lens[u];
    if (P.utt_trace && lane == 0) {
      tr_u = u;
      P.utt_trace[2 * (size_t)u] = ((unsigned long long)smid() << 48) |
                                   ((unsigned long long)(blockIdx.x * (blockDim.x >> 5) + wid) << 32) |
                                   (globaltimer_ns() & 0xffffffffull);
    }
    if (len_u <= 0 || len_u > P.T_max) {
      if (lane == 0) {
        P.status[u] = len_u == 0 ? kUttEmpty : kUttBadLen;
        P.out_count[u] = 0;
        P.kept[u] = 0;
      }
      continue;
    }
    // SMALL: the host guarantees stride_b < 2^32 elements, so the offsets are
    // 32 x 32 -> 64-bit products (one IMAD.WIDE instead of 64-bit multiplies
    // the compiler rematerialises every frame)
    const float* ubase = P.lp + (SMALL ? (size_t)(uint32_t)u * (uint32_t)P.stride_b : (size_t)u * P.stride_b);
    int32_t* fmap = P.frame_map + (size_t)(uint32_t)u * (uint32_t)P.T_max;
    const uint32_t st32 = (uint32_t)P.stride_t;
    auto row_of = [&](int fr) -> const float* {  // row fr of this utterance
      return ubase + (SMALL ? (size_t)((uint32_t)fr * st32) : (size_t)fr * P.stride_t);
    };

    // -- A. blank-skip compaction (emissions.py:298-306); in precomputed-top-k
    //    mode ctcb_framemap_kernel already did it
    //    Otherwise frames are classified 32 at a time just ahead of the row
    //    prefetch, so the blank values read here are still in L2 when the TMA
    //    fetches the rows (a pass over the whole utterance first costs an extra
    //    DRAM burst per frame: 6 % of cfg4's traffic)
    int kept = 0;  // !PRE: kept frames classified so far
    int ct = 0;    // !PRE: next frame to classify
    if (PRE) kept = P.kept[u];
    auto classify_to = [&](int idx) {  // classify until kept frame `idx` is known or frames run out
      while (!PRE && idx >= kept && ct < len_u) {
        const int t = ct + lane;
        bool keep = t < len_u;
        if (keep && P.skip) keep = !(__ldg(row_of(t) + P.blank) >= P.cutoff);
        const unsigned bal = __ballot_sync(FULL, keep);
        if (keep) fmap[kept + __popc(bal & lanemask_lt())] = t;
        kept += __popc(bal);
        ct += 32;
        __syncwarp();
      }
    };
    // precomputed top-k lists, prefetched one frame ahead
    const size_t tk_base = (size_t)u * P.T_max * k;
    int pre_st = 0;
    float pre_sv = 0.0f;
    // overlapped top-k (P.ready): list j is read only once its flag is
    // published; flags are polled 32 frames at a time (one poll per 32 frames
    // while the top-k kernel runs ahead), lists are read through L2 (__ldcg)
    int rdy = 0;
    // Invalid input rows (emissions.py:128-150) are never walked in
    // precomputed mode: the top-k kernel screens every row before its list
    // exists, so an utterance with an offender key ends as a dead beam before
    // its first frame (lists complete) or before the frames of the poll that
    // saw it (overlapped); ctcb_validate_post_kernel then reports the
    // offender.  (NaN / +inf scores could otherwise reach the selection.)
    bool vbad = PRE && P.validate && P.ready == nullptr && kept > 0 &&
                __shfl_sync(FULL, (int)(__ldcg(P.vkey + u) != ~0ull), 0);
    auto await_list = [&](int j) {
      if (!PRE || P.ready == nullptr || j < rdy) return;
      const uint32_t* fl = P.ready + (size_t)(uint32_t)u * (uint32_t)P.T_max;
      for (;;) {
        const int f = rdy + lane;
        const bool ok = f >= kept || ld_acquire_gpu(fl + f) != 0u;
        const unsigned bal = __ballot_sync(FULL, ok);
        rdy += bal == FULL ? 32 : __ffs(~bal) - 1;
        if (j < rdy) break;
        __nanosleep(128);
      }
      fence_acq_rel_gpu();
      __syncwarp();
      if (P.validate && __shfl_sync(FULL, (int)(__ldcg(P.vkey + u) != ~0ull), 0)) vbad = true;  // lane 0's view: warp-uniform
    };
    auto load_list = [&](int j) {
      if (P.ready != nullptr) {
        pre_st = __ldcg(P.topk_tok + tk_base + (size_t)j * k + lane);
        pre_sv = __ldcg(P.topk_val + tk_base + (size_t)j * k + lane);
      } else {
        pre_st = P.topk_tok[tk_base + (size_t)j * k + lane];
        pre_sv = P.topk_val[tk_base + (size_t)j * k + lane];
      }
    };
    if (PRE && kept > 0) await_list(0);
    if (PRE && kept > 0 && lane < k) load_list(0);

    // row staging: lane 0 issues the bulk copy of kept frame `idx`; frame-map
    // entries are read 32 at a time into registers
    int fm_blk = -1, fm_reg = 0, fm_hi = 0;
    auto issue = [&](int idx) {
      if ((idx >> 5) != fm_blk || idx >= fm_hi) {  // (re)load: the block may have grown since
        fm_blk = idx >> 5;
        const int t = (fm_blk << 5) + lane;
        fm_reg = t < kept ? fmap[t] : 0;
        fm_hi = kept < (fm_blk << 5) + 32 ? kept : (fm_blk << 5) + 32;
      }
      const int fr = __shfl_sync(FULL, fm_reg, idx & 31);
      if (lane == 0) {
        const float* src = row_of(fr);
        fence_proxy_async();
        mbar_arrive_expect_tx(&S.mbar[slot_i], row_copy);
        tma_bulk_g2s(S.rows + (size_t)slot_i * row_bytes, src, row_copy, &S.mbar[slot_i]);
      }
      slot_i = slot_i + 1 == ring ? 0 : slot_i + 1;
    };
    int n_out = 0;  // issued, not yet consumed
    classify_to(ring - 1);
    if (bulk) {
      const int pre = kept < ring - 1 ? kept : ring - 1;
      for (int i = 0; i < pre; i++) { issue(i); n_out++; }
    }

    // beam state (decoder.py:358-370): the empty prefix, blank flag set, score 0
    double s = 0.0;
    uint64_t h = kEmptyPrefixHash, ph = 0ull;
    int last = -1, len = 0, fl = 1;
    int H = 1;
    bool died = false;
    int died_at = 0;

    int i = 0;
    for (;; i++) {
      PH(0);
      classify_to(i + ring - 1);
      if (i >= kept) break;
      if (PRE && vbad) { died = true; died_at = i; break; }
      float* row;
      if (bulk) {
        if (i + ring - 1 < kept) { issue(i + ring - 1); n_out++; }
        mbar_wait(&S.mbar[slot_c], par_c);
        PH(1);
        row = (float*)(S.rows + (size_t)slot_c * row_bytes);
        n_out--;
        slot_c++;
        if (slot_c == ring) { slot_c = 0; par_c ^= 1u; }
      } else {
        row = (float*)S.rows;
        const float* src = row_of(fmap[i]);
        for (int c = lane; c < V; c += 32) row[c] = __ldg(src + c);
        __syncwarp();
      }
      // input validation fused into the staging (emissions.py:128-150): lane
      // partials now, the warp verdict at the end of the frame (off the
      // critical path); suspicious rows get the exact check from global memory
      // (precomputed mode: ctcb_topk_kernel already screened every kept row)
      // The shortcut pass below provides the non-blank maximum (vmax), so the
      // screen skips its own (max = max(vmax, blank value)).
      const bool v_scmax = !tokK && tiny_v;  // == sc_on && !PRE
      RowPart vpart{0u, 0xffffffffu, 0u};
      if (!PRE && P.validate)
        vpart = v_scmax ? (padded ? row_partials<4, false, true>(row, V, lane)
                                  : row_partials<SMALL ? 4 : 0, false>(row, V, lane))
                        : row_partials<SMALL ? 4 : 0>(row, V, lane);
      double vmax = -INFINITY;
      const float eb_f = row[P.blank];
      auto vfinish = [&]() {
        if (!PRE && P.validate && v_scmax) vpart.kmx = max(vpart.kmx, ord32(fmaxf((float)vmax, eb_f)));
        if (!PRE && P.validate && !row_verdict(vpart, P.validate == 1)) {
          const int fr = fmap[i];
          const unsigned long long vk = row_check_exact(row_of(fr), V, fr, lane, P.validate == 1);
          if (lane == 0 && vk != ~0ull) atomicMin(&P.vkey[u], vk);
        }
      };
      const double eb = (double)eb_f;
      __syncwarp();
      if (!PRE) {
        if (lane == 0) ((uint32_t*)row)[P.blank] = kSentinel;
        __syncwarp();
      }

      // ---- blank-frame shortcut (full vocabulary).  Every append group
      // (R+c, 0), including the last-token append from (R,1), scores at most
      // A_R + max_c v_c <= U = max_R A_R + vmax.  When at least `beam` blank /
      // repeat groups score above U, the new beam is made of those groups
      // alone and the frame needs no top-k, append lists or list selection
      // (~60 % of cfg4 frames).  vmax comes from a lane-max pass over the
      // staged row (blank holds the sentinel).
      const bool sc_on = !tokK && (PRE || tiny_v);
      if (sc_on && !PRE) {
        const float4* r4 = (const float4*)row;
        float lm = __uint_as_float(kSentinel);
#pragma unroll
        for (int j = 0; j < 4; j++) {
          const float4 q = r4[lane + 32 * j];
          lm = fmaxf(lm, fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w)));
        }
        const uint32_t mk = __reduce_max_sync(FULL, isnan(lm) ? 0u : okey(lm));
        vmax = mk ? (double)unord32(mk) : -INFINITY;
      }
      int st = 0;
      float sv = 0.0f;
      uint32_t selk = fullk;
      bool has_blank = true, wide = false;
      int mS = k;
      uint32_t tv = 0u;
      int ti = 0;
      // ================= top-k (k <= 32) =================
      auto full_topk = [&]() {
        if (PRE) {
          st = pre_st;
          sv = pre_sv;
          if (i + 1 < kept) await_list(i + 1);
          if (i + 1 < kept && lane < k) load_list(i + 1);
        } else {
          if (tiny_v) st = topk_small(S, row, V, k, lane, nch4, P.dbg);
          else st = skey_tok(topk_key(S, row, V, k, lane, small_v, nch4, P.dbg));
          st = lane < k ? st : 0;
          sv = lane < k ? row[st] : 0.0f;
        }
        // per-position key term: floor(v_p * 2^32 / R) (64-bit)
        if (lane < k) {
          S.sval[lane] = sv;
          S.stok[lane] = st;
          S.posmap[st] = (uint8_t)lane;
          S.wp[lane] = f2ll_floor((double)sv * kScale);
        }
        __syncwarp();
        // beam_size_token = K < V (decoder.py:440-458): the selected non-blank
        // tokens are a prefix (mS) of S when K <= k; otherwise all of S plus
        // tokens beyond it, tested against the K-th key (kth_token)
        if (tokK) {
          const uint32_t kb = ord32((float)eb);
          if (tokK <= k) {
            const bool above = lane < k && (ord32(sv) > kb || (ord32(sv) == kb && st < P.blank));
            has_blank = __popc(__ballot_sync(FULL, above)) < tokK;
            mS = has_blank ? tokK - 1 : tokK;
            selk = mS >= 32 ? 0xffffffffu : ((1u << mS) - 1u);
          } else {
            kth_token(row, V, P.blank, (float)eb, tokK, S.hist, lane, tv, ti);
            has_blank = token_selected(kb, P.blank, tv, ti);
            wide = true;
          }
        }
      };
      if (!sc_on || PRE) full_topk();
      if (sc_on && PRE) {  // precomputed lists: vmax is the top entry
        const float v0 = __shfl_sync(FULL, sv, 0);
        vmax = k > 0 ? (double)v0 : -INFINITY;
      }

      PH(2);
      // ================= merge structure =================
      const bool ent = lane < H;
      const uint64_t ph_m = shfl64(ph, me);
      const int len_m = __shfl_sync(FULL, len, me);
      uint64_t mkey;
      if (lane < 16) mkey = ent ? h : (kDummy ^ (uint64_t)lane);
      else mkey = (me < H && len_m > 0) ? ph_m : (kDummy ^ (uint64_t)lane);
      const unsigned m = __match_any_sync(FULL, mkey);
      const unsigned same = m & 0xffffu;
      const unsigned parents = __shfl_sync(FULL, m & 0xffffu, me + 16);
      const bool isfirst = ent && (__ffs(same) - 1) == lane;
      const unsigned firstmask = __ballot_sync(FULL, isfirst);
      const int nD = __popc(firstmask);
      const unsigned pmask = same & ~(1u << lane);
      const int p2 = (ent && pmask) ? __ffs(pmask) - 1 : -1;
      const double s_p2 = __shfl_sync(FULL, s, p2 >= 0 ? p2 : lane);
      const int fl_p2 = __shfl_sync(FULL, fl, p2 >= 0 ? p2 : lane);
      const int pa = (ent && parents) ? __ffs(parents) - 1 : -1;
      const unsigned pr2 = parents & (parents - 1);
      const int pb = (ent && pr2) ? __ffs(pr2) - 1 : -1;
      const double s_pa = __shfl_sync(FULL, s, pa >= 0 ? pa : lane);
      const int fl_pa = __shfl_sync(FULL, fl, pa >= 0 ? pa : lane);
      const int last_pa = __shfl_sync(FULL, last, pa >= 0 ? pa : lane);
      const double s_pb = __shfl_sync(FULL, s, pb >= 0 ? pb : lane);
      const int fl_pb = __shfl_sync(FULL, fl, pb >= 0 ? pb : lane);
      const int last_pb = __shfl_sync(FULL, last, pb >= 0 ? pb : lane);
      // A = logaddexp of the prefix's entries (append-list base)
      const double A = isfirst ? (p2 >= 0 ? merge2(s, s_p2, MX) : s) : 0.0;

      // blank / repeat groups need only the staged row (decoder.py:513-530);
      // with beam_size_token they are computed after the top-k (selection)
      double c_blank = -INFINITY, c_rep = -INFINITY, c_single = -INFINITY;
      int rep_src = lane, rep_tok = -1, single_src = lane;
      auto blank_repeat = [&](bool mem_last) {
        if (isfirst && has_blank) {  // blank group (R,1): entries of R in rank order (decoder.py:513-521)
          c_blank = s + eb;
          if (p2 >= 0) c_blank = merge2(c_blank, s_p2 + eb, MX);
        }
        if (ent && fl == 0 && mem_last) {  // repeat group (R',0): repeat first, then parent appends (:522-543)
          const double ec = (double)row[last];
          double sc = s + ec, bst = sc;
          if (pa >= 0 && !(fl_pa == 0 && last_pa == last)) {
            double x = s_pa + ec;
            sc = merge2(sc, x, MX);
            if (x > bst) { bst = x; rep_src = pa; rep_tok = last; }
          }
          if (pb >= 0 && !(fl_pb == 0 && last_pb == last)) {
            double x = s_pb + ec;
            sc = merge2(sc, x, MX);
            if (x > bst) { bst = x; rep_src = pb; rep_tok = last; }
          }
          c_rep = sc;
        }
      };
      if (!tokK) blank_repeat(true);

      // Exact order inside runs of close keys (rare; a persistent near-tie
      // between two beam entries recurs every frame).  Lane p holds the p-th
      // largest sorted key (slot tag in the low 6 bits); `cl` marks (p, p+1) as
      // possibly misordered.  Keys of different runs are ordered exactly, so
      // only the runs up to the beam cut are re-ranked, by exact fp64 score
      // (decoder.py:651-681); exact_of(slot, es, ba, xa, fa) is
      // warp-collective.  Exactly equal scores inside a run are ordered by
      // token sequence and flag by lane 0 when `serial` (the shortcut path);
      // otherwise, or when the run at the cut reaches lane 31, returns false
      // and the caller takes the exact k-way merge.
      PH(3);
      bool shortcut = false;
      int Hn = 0;
      if (sc_on) {
        // U: bound of every append score this frame
        // (an upper bound is enough: the high half of the largest order key
        // with all-ones low bits, one redux instead of two)
        const uint64_t ak = (isfirst && A > -INFINITY) ? ord64(A) : 0ull;
        const uint32_t ahi = __reduce_max_sync(FULL, (uint32_t)(ak >> 32));
        const uint64_t ab = ahi ? (((uint64_t)ahi << 32) | 0xffffffffull) : 0ull;
        const double U = (ab == 0ull || !(vmax > -INFINITY)) ? -INFINITY : unord64(ab) + vmax;
        const double Um = U + 1e-9 * (1.0 + fabs(U));  // appends are scored ~A + v: fp64 rounding margin
        const bool above_b = lane < 16 && c_blank > Um, above_r = lane < 16 && c_rep > Um;
        shortcut = __popc(__ballot_sync(FULL, above_b)) + __popc(__ballot_sync(FULL, above_r)) >= beam;
        if (shortcut) {
          // candidates: repeat group of entry e on lane e, blank group of
          // entry e on lane 16 + e (both exact fp64); frame best among them
          const double cb = __shfl_sync(FULL, c_blank, me), cr = c_rep;
          const double mine = lane < 16 ? cr : cb;
          const uint64_t o64 = (mine > -INFINITY && (lane < 16 ? lane < H : me < H)) ? ord64(mine) : 0ull;
          const uint32_t bhi = __reduce_max_sync(FULL, (uint32_t)(o64 >> 32));
          const uint32_t blo = __reduce_max_sync(FULL, (uint32_t)(o64 >> 32) == bhi ? (uint32_t)o64 : 0u);
          const double sbest = unord64(((uint64_t)bhi << 32) | blo);
          const double sbase = sbest - kR;
          // merge record of each candidate: (entry lane | item << 8), item =
          // the group's index in the entry's local order (repeat before
          // blank on equal scores; no last-token append in this frame)
          const int rf = __shfl_sync(FULL, (c_rep >= c_blank) ? 1 : 0, me);
          S.slot_rec[lane] = lane < 16 ? (lane | ((rf ? 0 : 1) << 8)) : (me | ((rf ? 1 : 0) << 8));
          uint32_t key = 0u;
          if (o64) {
            const uint32_t t = f2u_sat((mine - sbase) * kScale);
            key = ((t > 1u ? t : 1u) & ~63u) | (uint32_t)(63 - lane);
          }
          key = PRE ? sort_desc32_rank(key, lane, (uint32_t*)S.cand) : sort_desc32(key, lane);
          const uint32_t nxt = __shfl_down_sync(FULL, key, 1);
          // not separated by a truncated unit, or near the threshold floor:
          // the full path decides this frame
          const bool cl = lane < 31 && key != 0u && nxt != 0u && (key >> 6) - (nxt >> 6) <= 1u;
          const bool bad = lane < beam && key != 0u && (cl || key < 256u);
          __syncwarp();
          Hn = __popc(__ballot_sync(FULL, lane < beam && key != 0u));
          if (!__any_sync(FULL, bad)) {
            if (lane < Hn) S.rec_i[lane] = S.slot_rec[63 - (int)(key & 63u)];
          } else {
            // rare: keys near the threshold floor -> the full path; close keys
            // -> exact order inside their runs (candidate of slot g = 63 - tag:
            // repeat group of entry g < 16 or blank group of entry g - 16)
            int rr = 0;
            if (!__any_sync(FULL, lane < beam && key != 0u && key < 256u)) {
              const int g = key ? 63 - (int)(key & 63u) : 0;
              const double r_es = __shfl_sync(FULL, mine, g);
              const int r_rec = S.slot_rec[g];
              int r_pos, r_bmax;
              unsigned r_cm;
              rr = close_runs_rank(cl, r_es, beam, lane, r_pos, r_cm, r_bmax);
              if (rr == 1) {
                if (r_pos < beam) S.rec_i[r_pos] = r_rec;
              } else if (rr == 2) {
                serial_runs(P, S, u, i, beam, lane, h, len, r_es, g & 15, -1, g >= 16 ? 1 : 0, r_rec, r_cm, r_bmax);
                rr = 1;
              }
            }
            if (rr == 0) {
              shortcut = false;
              Hn = 0;
              if (lane == 0) atomicAdd(&P.dbg[kDbgOneshotFallback], 1ull);
            }
          }
          __syncwarp();
        }
      }
      // local order of an entry's groups: score desc; ties repeat (R,0) <
      // blank (R,1) < single (R+c,0)
      double q0, q1, q2;
      int kpack;
      auto local_order = [&]() {
        q0 = c_rep; q1 = c_blank; q2 = c_single;
        int k0 = 1, k1 = 0, k2 = 2;
        if (q1 > q0) { double t = q0; q0 = q1; q1 = t; int x = k0; k0 = k1; k1 = x; }
        if (q2 > q1) {
          double t = q1; q1 = q2; q2 = t; int x = k1; k1 = k2; k2 = x;
          if (q1 > q0) { t = q0; q0 = q1; q1 = t; x = k0; k0 = k1; k1 = x; }
        }
        kpack = k0 | (k1 << 2) | (k2 << 4);
      };
      int gsrc = lane;
      if (shortcut) local_order();
#ifdef CTCB_PHASES
      if (P.utt_trace && lane == 0) ph_cyc[14] += shortcut ? 1 : 0;
#endif
      if (!shortcut) {
        PH(4);
        if (sc_on && !PRE) full_topk();
        PH(5);
        // S positions of last tokens; flag-0 children exclude their token from
        // the parent's append list (they become repeat groups)
        const int mypos = (ent && last >= 0) ? (int)S.posmap[last] : 0xff;
        const uint32_t mybit = mypos < 32 ? (1u << mypos) : 0u;
        if (lane < 16) S.excl[lane] = 0u;
        __syncwarp();
        if (ent && fl == 0 && pa >= 0 && mybit) atomicOr(&S.excl[pa], mybit);
        __syncwarp();
        const uint32_t childx = lane < 16 ? S.excl[lane] : 0u;
        // last(R) selected this frame (repeat groups and the last-token append need it)
        const bool mem_last = !tokK || (ent && last >= 0 &&
                                          (wide ? token_selected(ord32(row[last]), last, tv, ti) : mypos < mS));
        if (tokK) blank_repeat(mem_last);
        if (isfirst && mybit && mem_last && !(childx & mybit)) {  // (R+last(R),0) from (R,1) only (blocked repeat)
          const int f1 = fl == 1 ? lane : ((p2 >= 0 && fl_p2 == 1) ? p2 : -1);
          if (f1 >= 0) {
            c_single = (f1 == lane ? s : s_p2) + (double)S.sval[mypos];
            single_src = f1;
          }
        }
        local_order();

        // ================= append lists (lanes 16..16+nD) =================
        // first lanes publish (lane, A, valid positions) at their distinct index
        if (isfirst) {
          const int d = __popc(firstmask & lanemask_lt());
          S.dlane[d] = lane;
          S.dA[d] = A;
          S.dgv[d] = selk & ~(childx | mybit);
        }
        __syncwarp();
        const bool gen = lane >= 16 && me < nD;
        gsrc = gen ? S.dlane[me] : lane;
        const double gA = gen ? S.dA[me] : 0.0;
        uint32_t gv = gen ? S.dgv[me] : 0u;
        const int gf = gv ? __ffs(gv) - 1 : 0;  // first valid position of the list

      // frame best (approximate append scores A + v; exact on key ties)
      const double hsc0 = lane < 16 ? q0 : (gv ? gA + (double)S.sval[gf] : -INFINITY);
      const uint64_t ok64 = hsc0 > -INFINITY ? ord64(hsc0) : 0ull;
      const uint32_t mhi = __reduce_max_sync(FULL, (uint32_t)(ok64 >> 32));
      const uint32_t mlo = __reduce_max_sync(FULL, (uint32_t)(ok64 >> 32) == mhi ? (uint32_t)ok64 : 0u);
      const uint64_t bk = ((uint64_t)mhi << 32) | mlo;
      if (bk == 0ull) { vfinish(); died = true; died_at = i; break; }  // every extension is -inf (decoder.py:616-620)
      const double best = unord64(bk);
      // keep iff score >= best - beam_threshold and score > -inf (decoder.py:621-623)
      const double lo_thr = P.threshold_inf ? -DBL_MAX : best - P.beam_threshold;
      const double kbase = best - kR;
      auto keyof = [&](double sc) -> uint32_t {
        if (!(sc > -INFINITY)) return 0u;
        const uint32_t t = f2u_sat((sc - kbase) * kScale);
        return t > 1u ? t : 1u;
      };
      // list keys: 64-bit fixed point (A - base) + v, both floored, clamped to
      // [1, 2^32 - 1] for a live list (A > -inf), 0 otherwise
      const long long gG = gv ? f2ll_floor((gA - kbase) * kScale) : 0ll;
      const uint32_t gLow = (gv && gA > -INFINITY) ? 1u : 0u;
      PH(6);
      // ---- one-shot selection (beam <= 10): when the distinct prefixes are
      // ordered by A with a margin, append (d, j) (j-th valid S position of
      // the d-th prefix) is beaten by the (d+1)(j+1)-1 appends (d' <= d,
      // j' <= j), so only j < beam/(d+1) can enter the beam: <= 27 append
      // slots + <= 30 specials, one 64-key sort.  Keys carry the slot in their
      // low 6 bits; adjacent keys within 2 truncated units, or keys near the
      // floor, fall back to the exact k-way merge below.
      bool oneshot = beam <= 10;
      int ldj_f = ldj;
      if (oneshot) {
        // the dominance count needs every list to hold >= beam valid positions
        // (true with k = 2 beam <= V-1 and the full vocabulary; small V or
        // beam_size_token can leave shorter lists)
        const double gA_prev = __shfl_up_sync(FULL, gA, 1);
        const bool shortl = gen && __popc(gv) < beam;
        const bool unsorted = gen && me > 0 && !(gA_prev > gA + 1e-9 * (1.0 + fabs(gA)));
        if (__any_sync(FULL, shortl)) {
          oneshot = false;
        } else if (__any_sync(FULL, unsorted)) {
          // prefixes not ordered by A (or tied): the same dominance count with
          // tiers -- list d keeps beam / (1 + lists whose A exceeds A_d by the
          // margin) positions; the slots are laid out by a prefix sum
          int tier = 0;
          for (int d2 = 0; d2 < nD; d2++) {
            const double a2 = __shfl_sync(FULL, gA, 16 + d2);
            tier += (gen && a2 > gA + 1e-9 * (1.0 + fabs(gA))) ? 1 : 0;
          }
          const int q = gen ? beam / (tier + 1) : 0;
          const int qi = warp_incl_scan(q, lane);
          const int tot = __shfl_sync(FULL, qi, 31);
          if (tot > 32) {
            oneshot = false;
          } else {
            const int off = qi - q;
            const unsigned starts = __reduce_or_sync(FULL, q > 0 ? 1u << off : 0u);
            if (q > 0) S.hist[off] = (uint32_t)me;
            __syncwarp();
            ldj_f = 0xff;
            if (lane < tot) {
              const int st0 = 31 - __clz(starts & (0xffffffffu >> (31 - lane)));
              ldj_f = (int)S.hist[st0] | ((lane - st0) << 4);
            }
            __syncwarp();
          }
        }
        if (!oneshot && lane == 0) atomicAdd(&P.dbg[kDbgFrames], 1ull);  // diagnostics: fallback by order/length
      }
      if (oneshot) {
        if (gen) S.dG[me] = gG;
        // specials -> slots [0, nS) in lane order
        const uint32_t s0 = lane < 16 ? keyof(q0) : 0u, s1 = lane < 16 ? keyof(q1) : 0u,
                       s2 = lane < 16 ? keyof(q2) : 0u;
        const int cS = (s0 != 0u) + (s1 != 0u) + (s2 != 0u);  // q0 >= q1 >= q2: a prefix
        // slot offsets: exclusive prefix sum of cS in {0..3} from its two bits
        const unsigned cb0 = __ballot_sync(FULL, cS & 1), cb1 = __ballot_sync(FULL, cS & 2);
        const unsigned lt_ = lanemask_lt();
        const int sb = __popc(cb0 & lt_) + 2 * __popc(cb1 & lt_);
        const int nS = __popc(cb0) + 2 * __popc(cb1);
        bool nearfloor = (s0 != 0u && s0 < 128u) || (s1 != 0u && s1 < 128u) || (s2 != 0u && s2 < 128u);
        if (cS > 0) { S.ckey[sb] = (s0 & ~63u) | (uint32_t)(63 - sb); S.slot_rec[sb] = lane; }
        if (cS > 1) { S.ckey[sb + 1] = (s1 & ~63u) | (uint32_t)(62 - sb); S.slot_rec[sb + 1] = lane | (1 << 8); }
        if (cS > 2) { S.ckey[sb + 2] = (s2 & ~63u) | (uint32_t)(61 - sb); S.slot_rec[sb + 2] = lane | (2 << 8); }
        __syncwarp();
        // append slot 32 + lane: (d, j) from the quota table
        uint32_t bkey = 0u;
        const int qd = ldj_f & 15, qj = ldj_f >> 4;
        if (ldj_f != 0xff && qd < nD) {
          // j-th valid position: j plus the excluded positions at or below it
          // (exclusions are the few flag-0 children and last(R))
          uint32_t ex = ~S.dgv[qd] & fullk;
          int pp = qj;
          while (ex) {
            const int e = __ffs(ex) - 1;
            if (e > pp) break;
            pp++;
            ex &= ex - 1u;
          }
          if (pp < k) {
            const long long t = S.dG[qd] + S.wp[pp];
            const uint32_t kk = t < 1ll ? 1u : (t > 0xffffffffll ? 0xffffffffu : (uint32_t)t);
            const bool live = S.dA[qd] > -INFINITY;
            nearfloor |= live && kk < 128u;
            bkey = live ? ((kk & ~63u) | (uint32_t)(31 - lane)) : 0u;
            S.slot_rec[32 + lane] = (16 + qd) | (pp << 8);
          }
        }
        uint32_t akey = lane < nS ? S.ckey[lane] : 0u;
        if (PRE) {  // latency-bound small batches: rank-count sorts (the fused
                    // kernel at 16 warps/SM is faster with the shuffle network: 5.25 vs 5.43 ms)
          akey = sort_desc32_rank(akey, lane, (uint32_t*)S.cand);
          bkey = sort_desc32_rank(bkey, lane, (uint32_t*)S.cand);
        } else {
          akey = sort_desc32(akey, lane);
          bkey = sort_desc32(bkey, lane);
        }
        akey = max(akey, __shfl_sync(FULL, bkey, 31 - lane));
        akey = merge_desc32(akey, lane);
        const uint32_t nxt = __shfl_down_sync(FULL, akey, 1);
        const bool cl = lane < 31 && akey != 0u && nxt != 0u && (akey >> 6) - (nxt >> 6) <= 1u;
        Hn = __popc(__ballot_sync(FULL, lane < beam && akey != 0u));
        if (!__any_sync(FULL, (cl && lane < beam) || nearfloor)) {
          if (lane < Hn) S.rec_i[lane] = S.slot_rec[63 - (int)(akey & 63u)];
        } else if (__any_sync(FULL, nearfloor)) {
          oneshot = false;
        } else {
          // rare: close keys -> exact order inside their runs; the exact score
          // of slot sl's candidate as the commit below computes it
          const int sl = akey ? 63 - (int)(akey & 63u) : 0;
          const int rec = akey != 0u ? S.slot_rec[sl] : (lane & 15);
          const int wl = rec & 0xff, it = rec >> 8;
          const int wk = __shfl_sync(FULL, kpack, wl);
          const double w0 = __shfl_sync(FULL, q0, wl), w1 = __shfl_sync(FULL, q1, wl), w2 = __shfl_sync(FULL, q2, wl);
          const int bse = __shfl_sync(FULL, gsrc, wl);
          const double bs1 = __shfl_sync(FULL, s, bse), bs2 = __shfl_sync(FULL, s_p2, bse);
          const int bp2 = __shfl_sync(FULL, p2, bse), blst = __shfl_sync(FULL, last, bse);
          double r_es;
          int r_ba, r_xa, r_fa;
          if (wl >= 16) {  // append group (R+c, 0)
            const int itc = it < 32 ? it : 0;
            const double v = (double)S.sval[itc];
            r_es = bs1 + v;
            if (bp2 >= 0) r_es = merge2(r_es, bs2 + v, MX);
            r_ba = bse;
            r_xa = S.stok[itc];
            r_fa = 0;
          } else {  // special group: blank (R,1), repeat (R,0), last-token append (R+last,0)
            const int kind = (wk >> (2 * (it & 3))) & 3;
            r_es = it == 0 ? w0 : (it == 1 ? w1 : w2);
            r_ba = wl;
            r_xa = kind == 2 ? blst : -1;
            r_fa = kind == 0 ? 1 : 0;
          }
          int r_pos, r_bmax;
          unsigned r_cm;
          const int rr = close_runs_rank(cl, r_es, beam, lane, r_pos, r_cm, r_bmax);
          if (rr == 1) {
            if (r_pos < beam) S.rec_i[r_pos] = rec;
          } else if (rr == 2) {
            serial_runs(P, S, u, i, beam, lane, h, len, r_es, r_ba, r_xa, r_fa, rec, r_cm, r_bmax);
          } else {
            oneshot = false;
          }
        }
        if (!oneshot) {
          Hn = 0;
          if (lane == 0) atomicAdd(&P.dbg[kDbgOneshotFallback], 1ull);
        }
        __syncwarp();
      }
      if (!oneshot) {
      PH(7);
      // rank-key queues: each lane pops its candidates in order.  Lanes < 16
      // queue their <= 3 special groups (items 0..2 = local sorted order);
      // lanes 16.. queue the next four valid positions of their append list
      // (gq = queued positions), refilled on demand.
      uint32_t kq0, kq1, kq2, kq3;
      uint32_t gq = 0u;  // queued items (specials: local ranks 0..2; lists: S positions)
      auto refill = [&]() {
        uint32_t kk[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
          kk[q] = 0u;
          if (gv) {
            const int p = __ffs(gv) - 1;
            gv &= gv - 1u;
            gq |= 1u << p;
            const long long t = gG + S.wp[p];
            kk[q] = t < 1ll ? gLow : (t > 0xffffffffll ? 0xffffffffu : (uint32_t)t);
          }
        }
        kq0 = kk[0]; kq1 = kk[1]; kq2 = kk[2]; kq3 = kk[3];
      };
      if (lane < 16) {
        kq0 = keyof(q0); kq1 = keyof(q1); kq2 = keyof(q2); kq3 = 0u;
        gq = 7u;
      } else {
        refill();
      }
      int recw = lane | ((__ffs(gq) - 1) << 8);  // record of the queue head
#ifdef CTCB_FAST_CHECK
      {
        FCHK((kq0 == 0u) == (gq == 0u) || lane < 16, i, (int)gq);
      }
#endif

      // ================= k-way merge (decoder.py:651-681) =================
      for (int r = 0; r < beam; r++) {
        const uint32_t mk = __reduce_max_sync(FULL, kq0);
        if (mk == 0u) break;
        // the unique head within kTol of the maximum wins outright (predicated
        // pop below); several such heads, or a head near the floor, take the
        // exact path
        bool win = kq0 != 0u && mk - kq0 <= kTol;
        const unsigned tied = __ballot_sync(FULL, win);
        if ((tied & (tied - 1)) || mk <= kTol + 1u) {
          int w = __ffs(tied) - 1;
          // exact resolution: fp64 score, then token sequence, then flag;
          // near the floor also the exact threshold test
          if (tied & (1u << lane)) {
            double esc;
            int eb_, ex, ef, pos;
            if (lane < 16) {
              const int npop = __ffs(gq) - 1;
              const int kind = (kpack >> (2 * npop)) & 3;
              esc = npop == 0 ? q0 : (npop == 1 ? q1 : q2);
              eb_ = lane;
              ex = kind == 2 ? last : -1;
              ef = kind == 0 ? 1 : 0;
              pos = -1;
            } else {
              pos = __ffs(gq) - 1;
              esc = 0.0;  // exact fold below
              eb_ = gsrc;
              ex = S.stok[pos];
              ef = 0;
            }
            S.tie_sc[lane] = esc;
            S.tie_i[lane * 4 + 0] = eb_;
            S.tie_i[lane * 4 + 1] = ex;
            S.tie_i[lane * 4 + 2] = ef;
            S.tie_i[lane * 4 + 3] = pos;
          }
          if (lane < 16) { S.hs[lane] = h; S.hl[lane] = len; S.hsc[lane] = s; S.hp2[lane] = p2; }
          __syncwarp();
          if (lane == 0) {
            atomicAdd(&P.dbg[kDbgTies], 1ull);
            // exact append-group scores for tied list heads
            unsigned tl = tied;
            while (tl) {
              const int c = __ffs(tl) - 1;
              tl &= tl - 1;
              const int pos = S.tie_i[c * 4 + 3];
              if (pos >= 0) {
                const int f = S.tie_i[c * 4];
                const double v = (double)S.sval[pos];
                double e = S.hsc[f] + v;
                if (S.hp2[f] >= 0) e = merge2(e, S.hsc[S.hp2[f]] + v, MX);
                S.tie_sc[c] = e;
              }
            }
            unsigned rest = tied & (tied - 1);
            while (rest) {
              const int c = __ffs(rest) - 1;
              rest &= rest - 1;
              if (fast_precedes(P, S, u, i, S.tie_sc[c], S.tie_i[c * 4], S.tie_i[c * 4 + 1], S.tie_i[c * 4 + 2],
                                S.tie_sc[w], S.tie_i[w * 4], S.tie_i[w * 4 + 1], S.tie_i[w * 4 + 2]))
                w = c;
            }
            const double wsc = S.tie_sc[w];
            if (!(wsc > -INFINITY) || !(wsc >= lo_thr)) w = -1;  // below the threshold: the beam is complete
          }
          w = __shfl_sync(FULL, w, 0);
          __syncwarp();
          if (w < 0) break;
          win = lane == w;
        }
        // pop: the record of the head (lane | item << 8) goes to the new rank;
        // losers write their own scratch slot instead of branching
        FCHK(!win || gq != 0u, i, r * 1000 + (int)kq0);
        S.rec_i[win ? r : 16 + lane] = recw;
        gq = win ? (gq & (gq - 1u)) : gq;
        recw = lane | ((__ffs(gq) - 1) << 8);
        kq0 = win ? kq1 : kq0;
        kq1 = win ? kq2 : kq1;
        kq2 = win ? kq3 : kq2;
        kq3 = win ? 0u : kq3;
        const bool need = win && kq0 == 0u && gv != 0u;
        if (__any_sync(FULL, need)) {
          if (need) {
            refill();
            recw = lane | ((__ffs(gq) - 1) << 8);
          }
        }
        Hn = r + 1;
      }
      }  // !oneshot
      }  // !shortcut
      __syncwarp();
      if (Hn == 0) { vfinish(); died = true; died_at = i; break; }

      PH(8);
      // ================= commit (decoder.py:683-744) =================
      // lane r builds new entry r from the winning lane's registers
      const bool nent = lane < Hn;
      const int rec = S.rec_i[nent ? lane : 0];
#ifdef CTCB_FAST_CHECK
      {
        FCHK(Hn <= beam, Hn, beam);
        const int wl_ = rec & 0xff, it_ = rec >> 8;
        FCHK(!nent || (wl_ < 32 && (wl_ >= 16 ? it_ < k : it_ < 3)), rec, i);
        const unsigned mm = __match_any_sync(FULL, nent ? rec : -1 - lane);
        FCHK(!nent || __popc(mm) == 1, rec, (int)mm);
      }
#endif
      const int wl = nent ? (rec & 0xff) : lane, item2 = rec >> 8;
      const int wk = __shfl_sync(FULL, kpack, wl);
      const double w_q0 = __shfl_sync(FULL, q0, wl), w_q1 = __shfl_sync(FULL, q1, wl), w_q2 = __shfl_sync(FULL, q2, wl);
      const int w_src = __shfl_sync(FULL, rep_src | (single_src << 8), wl);
      const int w_rtok = __shfl_sync(FULL, rep_tok, wl);
      const int w_gsrc = __shfl_sync(FULL, gsrc, wl);
      const bool wgen = wl >= 16;
      const int base = wgen ? w_gsrc : wl;
      const uint64_t bh = shfl64(h, base), bph = shfl64(ph, base);
      const int blast = __shfl_sync(FULL, last, base), blen = __shfl_sync(FULL, len, base);
      const double b_s1 = __shfl_sync(FULL, s, base), b_s2 = __shfl_sync(FULL, s_p2, base);
      const int b_p2 = __shfl_sync(FULL, p2, base);
      double nsc;
      int x, src, tok, nfl;
      if (wgen) {  // append group (R+c,0): exact fold of R's entries in rank order
        const int c = S.stok[item2];
        const double v = (double)S.sval[item2];
        nsc = b_s1 + v;
        if (b_p2 >= 0) nsc = merge2(nsc, b_s2 + v, MX);
        x = c; src = base; tok = c; nfl = 0;
      } else {
        const int kind = (wk >> (2 * item2)) & 3;
        nsc = item2 == 0 ? w_q0 : (item2 == 1 ? w_q1 : w_q2);
        if (kind == 0) { x = -1; src = wl; tok = -1; nfl = 1; }                  // blank group
        else if (kind == 1) { x = -1; src = w_src & 0xff; tok = w_rtok; nfl = 0; }  // repeat group
        else { x = blast; src = w_src >> 8; tok = blast; nfl = 0; }               // last-token append
      }
      const uint32_t trel = pack_trel(src, tok);
      __syncwarp();
      // reset the token -> S rank map
      if (lane < k) S.posmap[st] = 0xff;
      if (nent) {
        s = nsc;
        h = x >= 0 ? child_hash(bh, x) : bh;
        ph = x >= 0 ? bh : bph;
        last = x >= 0 ? x : blast;
        len = x >= 0 ? blen + 1 : blen;
        fl = nfl;
        P.trellis[(size_t)(uint32_t)u * (uint32_t)(P.T_max * beam) + (uint32_t)(i * beam + lane)] = trel;
        S.tring[(i % kChunk) * 16 + lane] = trel;
      }
      H = Hn;
      PH(9);
      vfinish();
      __syncwarp();
      // trellis checkpoint: ancestor slot at the chunk start for every entry
      if ((i % kChunk) == kChunk - 1) {
        if (lane < H) {
          int slot = lane;
          for (int t = i % kChunk; t >= 0; --t) slot = trel_src(S.tring[t * 16 + slot]);
          P.anc[((size_t)u * P.n_chunks + i / kChunk) * 16 + lane] = (uint8_t)slot;
        }
        __syncwarp();
      }
    }
    if (!PRE && lane == 0) P.kept[u] = kept;  // (partial if the beam died: later frames unclassified)
    if (!died && kept % kChunk != 0) {  // checkpoint of the last, partial chunk
      const int il = kept - 1;
      if (lane < H) {
        int slot = lane;
        for (int t = il % kChunk; t >= 0; --t) slot = trel_src(S.tring[t * 16 + slot]);
        P.anc[((size_t)u * P.n_chunks + il / kChunk) * 16 + lane] = (uint8_t)slot;
      }
      __syncwarp();
    }

    if (lane == 0) P.vdone[u] = (PRE || !died) ? kept : died_at + 1;  // rows screened (here or by the top-k kernel)
    if (died) {
      while (n_out > 0) {
        mbar_wait(&S.mbar[slot_c], par_c);
        n_out--;
        slot_c++;
        if (slot_c == ring) { slot_c = 0; par_c ^= 1u; }
      }
      for (int c = lane; c < V; c += 32) S.posmap[c] = 0xff;
      if (lane == 0) {  // the dying frame (kept-frame index) goes to out_len[u][0]
        P.status[u] = kUttBeamDied;
        P.out_count[u] = 0;
        P.out_len[(size_t)u * P.nbest] = died_at;
      }
      __syncwarp();
      continue;
    }

    // ================= finalize (decoder.py:753-817) =================
    {
      const bool ent = lane < H;
      const unsigned fm = __match_any_sync(FULL, ent ? h : (kDummy ^ (uint64_t)lane));
      const bool isf = ent && (__ffs(fm) - 1) == lane;
      const unsigned pm = fm & ~(1u << lane);
      const int p2 = (ent && pm) ? __ffs(pm) - 1 : -1;
      const double s_p2 = __shfl_sync(FULL, s, p2 >= 0 ? p2 : lane);
      const double gsc = isf ? (p2 >= 0 ? merge2(s, s_p2, MX) : s) : -INFINITY;
      // order groups: (score desc, lane asc) by register sort, then exact tie runs
      uint64_t key = isf ? ord64(gsc) : 0ull;
      int pay = lane;
#pragma unroll 1
      for (int size = 2; size <= 32; size <<= 1)
#pragma unroll 1
        for (int j = size >> 1; j > 0; j >>= 1) {
          uint64_t ky = shflx64(key, j);
          int py = __shfl_xor_sync(FULL, pay, j);
          bool mine_first = key > ky || (key == ky && pay < py);
          bool take_first = ((lane & j) == 0) == ((lane & size) == 0);
          if (take_first != mine_first) { key = ky; pay = py; }
        }
      const int nF = __popc(__ballot_sync(FULL, isf));
      const double srt_sc = __shfl_sync(FULL, gsc, pay);
      // exact tie runs (identical fp64 scores): token-sequence order
      S.tie_i[lane] = pay;
      S.tie_sc[lane] = srt_sc;
      if (lane < 16) { S.hs[lane] = h; S.hl[lane] = len; }
      __syncwarp();
      if (lane == 0) {
        for (int a = 1; a < nF; a++) {
          int j = a;
          while (j > 0 && S.tie_sc[j] == S.tie_sc[j - 1] &&
                 fast_seq_cmp(P, S, u, kept, S.tie_i[j], -1, S.tie_i[j - 1], -1) < 0) {
            int t = S.tie_i[j]; S.tie_i[j] = S.tie_i[j - 1]; S.tie_i[j - 1] = t;
            j--;
          }
        }
      }
      __syncwarp();
      const int nOut = nF < P.nbest ? nF : P.nbest;
      const int nchk = (kept + kChunk - 1) / kChunk;
      int* ends = P.seqbuf + (size_t)u * 3 * (P.T_max + 1);
      int* tmp_tok = ends + (P.T_max + 1);
      int* tmp_fr = tmp_tok + (P.T_max + 1);
      for (int r = 0; r < nOut; r++) {
        const int e = S.tie_i[r];
        const double sc = __shfl_sync(FULL, gsc, e);
        const int L_e = __shfl_sync(FULL, len, e);
        const size_t o = (size_t)u * P.nbest + r;
        if (lane == 0) { P.out_score[o] = sc; P.out_len[o] = L_e; }
        int* tok_out = P.out_tokens + o * P.T_max;
        int* ts_out = P.out_ts ? P.out_ts + o * P.T_max : nullptr;
        if (L_e == 0 || nchk == 0) continue;
        // coarse walk over checkpoints
        if (lane == 0) {
          int slot = e;
          for (int c = nchk - 1; c >= 0; --c) {
            ends[c] = slot;
            slot = P.anc[((size_t)u * P.n_chunks + c) * 16 + slot];
          }
        }
        __syncwarp();
        // fine walks, one chunk per lane
        for (int c = lane; c < nchk; c += 32) {
          int slot = ends[c], cntc = 0;
          const int i_end = min(kept, (c + 1) * kChunk) - 1;
          for (int ii = i_end; ii >= c * kChunk; --ii) {
            uint32_t rec = P.trellis[((size_t)u * P.T_max + ii) * beam + slot];
            int tok = trel_tok(rec);
            if (tok >= 0) {
              tmp_tok[c * kChunk + cntc] = tok;
              tmp_fr[c * kChunk + cntc] = fmap[ii];
              cntc++;
            }
            slot = trel_src(rec);
          }
          ends[c] = cntc;
        }
        __syncwarp();
        int running = 0;
        for (int b0 = 0; b0 < nchk; b0 += 32) {
          const int c = b0 + lane;
          const int cnt_c = c < nchk ? ends[c] : 0;
          const int incl = warp_incl_scan(cnt_c, lane);
          const int off = running + incl - cnt_c;
          for (int q = 0; q < cnt_c; q++) {
            tok_out[off + q] = tmp_tok[c * kChunk + cnt_c - 1 - q];
            if (ts_out) ts_out[off + q] = tmp_fr[c * kChunk + cnt_c - 1 - q];
          }
          running += __shfl_sync(FULL, incl, 31);
        }
        __syncwarp();
      }
      if (lane == 0) { P.out_count[u] = nOut; P.status[u] = kUttOk; }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(128, CTCB_FAST_MIN_BLOCKS) ctcb_decode_fast_kernel(const __grid_constant__ Params P) {
  fast_decode<false, false>(P);
}
__global__ void __launch_bounds__(128, CTCB_FAST_MIN_BLOCKS)
    ctcb_decode_fast_small_kernel(const __grid_constant__ Params P) {
  fast_decode<false, true>(P);
}
__global__ void __launch_bounds__(128, CTCB_FAST_MIN_BLOCKS)
    ctcb_decode_fast_pre_kernel(const __grid_constant__ Params P) {
  fast_decode<true, false>(P);
}
__global__ void __launch_bounds__(128, CTCB_FAST_MIN_BLOCKS)
    ctcb_decode_fast_pre_small_kernel(const __grid_constant__ Params P) {
  fast_decode<true, true>(P);
}

// Precomputed-top-k mode (small batches, where one warp per utterance leaves
// the GPU latency-bound): frame maps first, then the top-k of every kept frame
// of every utterance in parallel, then the beam kernel walks the frames with
// the top-k lists prefetched.
__global__ void __launch_bounds__(256) ctcb_framemap_kernel(const __grid_constant__ Params P) {
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (u >= P.B) return;
  int len_u = P.lens[u];
  if (len_u < 0 || len_u > P.T_max) len_u = 0;
  const int kept = frame_map_warp(P, P.lp + (size_t)u * P.stride_b, len_u, P.frame_map + (size_t)u * P.T_max, lane);
  if (lane == 0) P.kept[u] = kept;
}

// Exclusive prefix sums of the kept-frame counts (one block): row offsets of
// the flattened (utterance, kept frame) space the top-k kernel splits evenly.
__global__ void __launch_bounds__(1024) ctcb_rowoff_kernel(const __grid_constant__ Params P) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < P.B; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    const int v = b < P.B ? P.kept[b] : 0;
    const int incl = warp_incl_scan(v, lane);
    if (lane == 31) warp_tot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      const int t = warp_tot[lane];
      warp_tot[lane] = warp_incl_scan(t, lane) - t;
    }
    __syncthreads();
    if (b < P.B) P.rowoff[b] = carry + warp_tot[wid] + incl - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += warp_tot[31] + incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) P.rowoff[P.B] = carry;
}

// Frame-parallel top-k (precomputed mode; the per-frame token selection of
// decoder.py:431-466): the kept rows of all utterances, split over the warps
// (contiguous flattened ranges when it runs before the walk, frame-major with
// per-list ready flags when it runs beside it); rows are staged by TMA bulk
// copies into a per-warp 2-deep ring one row ahead of use (V <= 512) or read
// straight from global memory (V > 512).
#ifndef CTCB_TOPK_MIN_BLOCKS
#define CTCB_TOPK_MIN_BLOCKS 4
#endif
#ifndef CTCB_TOPK_RING
#define CTCB_TOPK_RING 2
#endif
__global__ void __launch_bounds__(256, CTCB_TOPK_MIN_BLOCKS) ctcb_topk_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int kRing = CTCB_TOPK_RING;
  uint8_t* wbase = smem + (size_t)wid * P.smem_per_warp;
  FastSmem S{};
  S.rows = wbase;
  uint64_t* mbar = (uint64_t*)(wbase + (size_t)kRing * P.row_bytes);
  S.cand = (uint64_t*)(wbase + (size_t)kRing * P.row_bytes + 64);
  S.hist = (uint32_t*)((uint8_t*)S.cand + 64 * 8);
  S.ckey = (uint32_t*)((uint8_t*)S.hist + 256 * 4);
  S.cidx = (uint16_t*)((uint8_t*)S.ckey + 64 * 4);
  const int V = P.V, k = P.k, nch4 = (V + 3) >> 2;
  const bool small_v = nch4 <= 256;
  const bool tiny_v = nch4 <= 128 && k <= 31;
  const uint32_t sdir = 0u;
  (void)sdir;
  for (int r = 0; r < kRing; r++)
    for (int c = V + lane; c < P.row_bytes / 4; c += 32) ((uint32_t*)(S.rows + (size_t)r * P.row_bytes))[c] = kSentinel;
  if (lane == 0)
    for (int r = 0; r < kRing; r++) mbar_init(&mbar[r], 1);
  fence_mbar_init();
  fence_proxy_async();
  __syncwarp();
  // overlapped mode (P.ready): the walk is a programmatic dependent of this
  // grid; it may launch once every CTA here is running (no CTA of this grid
  // ever waits on it, so the pair cannot deadlock)
  pdl_launch_dependents();
  const bool fm = P.ready != nullptr;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + wid;
  // Row cursors.  Flattened split (fm = false): warp w takes the contiguous
  // range [g0, g1) of the utterance-major (u, kept frame) space.  Frame-major
  // (fm = true, overlapped with the walk): position p = frame * B + slot,
  // utterance order[slot] (the walk's longest-first order), warp w takes
  // p = w, w + nw, ...: the lists of frame i of every utterance are written
  // before those of frame i + 1, in the order the walks consume them.
  struct Cur {
    int u, i;
    long long p;
  };
  const long long G = fm ? (long long)P.B * P.T_max : 0;
  auto fm_settle = [&](Cur& c) {  // first valid position >= c.p on this warp's stride
    for (; c.p < G; c.p += nw) {
      const int uu = P.order[(int)(c.p % P.B)], ii = (int)(c.p / P.B);
      if (ii < P.kept[uu]) { c.u = uu; c.i = ii; return; }
    }
    c.u = P.B;
  };
  Cur c0{0, 0, w};
  long long n = 0;
  if (fm) {
    fm_settle(c0);
    if (c0.u >= P.B) return;
  } else {
    const long long total = P.rowoff[P.B];
    const long long g0 = total * w / nw, g1 = total * (w + 1) / nw;
    if (g0 >= g1) return;
    n = g1 - g0;
    int lo = 0, hi = P.B - 1;  // utterance of the first row: last u with rowoff[u] <= g0
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (P.rowoff[mid] <= g0) lo = mid; else hi = mid - 1;
    }
    c0.u = lo;
    c0.i = (int)(g0 - P.rowoff[lo]);
    while (c0.u < P.B && c0.i >= P.kept[c0.u]) { c0.u++; c0.i = 0; }
  }
  auto advance = [&](Cur& c) {
    if (fm) {
      c.p += nw;
      fm_settle(c);
    } else {
      c.i++;
      while (c.u < P.B && c.i >= P.kept[c.u]) { c.u++; c.i = 0; }
    }
  };
  auto more = [&](const Cur& c, long long cnt) { return fm ? c.u < P.B : cnt < n; };
  auto src_of = [&](int u, int i) -> const float* {
    return P.lp + (size_t)u * P.stride_b + (size_t)P.frame_map[(size_t)u * P.T_max + i] * P.stride_t;
  };
  // list (u, i) written by lanes < k: every lane fences its stores, then lane 0
  // publishes the flag (release, gpu scope)
  auto publish = [&](const Cur& c) {
    if (!fm) return;
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release_gpu(P.ready + (size_t)c.u * P.T_max + c.i, 1u);
  };
  if (P.row_bytes == 0) {
    // large vocabulary: rows read straight from global memory (topk_key_g)
    Cur c = c0;
    for (long long g = 0; more(c, g); g++) {
      const int fr = P.frame_map[(size_t)c.u * P.T_max + c.i];
      const float* src = P.lp + (size_t)c.u * P.stride_b + (size_t)fr * P.stride_t;
      if (P.validate && !row_screen_scalar(src, V, lane, P.validate == 1)) {  // emissions.py:128-150
        const unsigned long long vk = row_check_exact(src, V, fr, lane, P.validate == 1);
        if (lane == 0 && vk != ~0ull) atomicMin(&P.vkey[c.u], vk);
      }
      const int st = skey_tok(topk_key_g(S, src, V, P.blank, k, lane, nullptr));
      if (lane < k) {
        const size_t o = ((size_t)c.u * P.T_max + c.i) * k + lane;
        P.topk_tok[o] = st;
        P.topk_val[o] = __ldg(src + st);
      }
      __syncwarp();
      publish(c);
      advance(c);
    }
    return;
  }
  // staged rows: issue cursor ic runs kRing - 1 rows ahead of consume cursor cc
  const uint32_t row_copy = (uint32_t)V * 4u;
  Cur ic = c0, cc = c0;
  int slot_i = 0, slot_c = 0;
  uint32_t par = 0u;
  long long issued = 0;
  auto issue = [&]() {
    if (P.bulk_ok) {
      if (lane == 0) {
        mbar_arrive_expect_tx(&mbar[slot_i], row_copy);
        tma_bulk_g2s(S.rows + (size_t)slot_i * P.row_bytes, src_of(ic.u, ic.i), row_copy, &mbar[slot_i]);
      }
    }
    slot_i = slot_i + 1 == kRing ? 0 : slot_i + 1;
    issued++;
    advance(ic);
  };
  for (int r = 0; r < kRing - 1 && more(ic, issued); r++) issue();
  for (long long g = 0; more(cc, g); g++) {
    if (more(ic, issued)) issue();
    float* row = (float*)(S.rows + (size_t)slot_c * P.row_bytes);
    const float* src = src_of(cc.u, cc.i);
    if (P.bulk_ok) {
      mbar_wait(&mbar[slot_c], par);
    } else {
      for (int c = lane; c < V; c += 32) row[c] = __ldg(src + c);
    }
    __syncwarp();
    // input validation of every kept row (emissions.py:128-150): the beam walk
    // of precomputed mode leaves it to this frame-parallel pass
    if (P.validate && !row_screen(row, V, lane, P.validate == 1)) {
      const int fr = P.frame_map[(size_t)cc.u * P.T_max + cc.i];
      const unsigned long long vk = row_check_exact(src, V, fr, lane, P.validate == 1);
      if (lane == 0 && vk != ~0ull) atomicMin(&P.vkey[cc.u], vk);
    }
    if (lane == 0) ((uint32_t*)row)[P.blank] = kSentinel;
    __syncwarp();
    const int st = tiny_v ? topk_small(S, row, V, k, lane, nch4, nullptr)
                          : skey_tok(topk_key(S, row, V, k, lane, small_v, nch4, nullptr));
    if (lane < k) {
      const size_t o = ((size_t)cc.u * P.T_max + cc.i) * k + lane;
      P.topk_tok[o] = st;
      P.topk_val[o] = row[st];
    }
    __syncwarp();
    publish(cc);
    fence_proxy_async();  // generic writes to the slot (blank sentinel) before it is refilled by TMA
    slot_c++;
    if (slot_c == kRing) { slot_c = 0; par ^= 1u; }
    advance(cc);
  }
}

}  // namespace ctcb
