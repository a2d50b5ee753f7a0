// Headline decode kernel: CTC prefix beam search for beam <= 16, V <= 512,
// blank = 0, full vocabulary (the paper's and BASELINE.json's V=500 / beam 10
// configurations), TWO utterances per warp.
//
// Same semantics as the other search kernels and the reference (ctcforge
// decoder.py:102-817); what changes is the mapping onto the warp.  The
// one-utterance-per-warp kernel (ctcb_fast.cu) keeps <= 16 useful lanes for
// most of a frame step and pays a 15-stage 32-lane sorting network several
// times per frame.  Here each 16-lane half-warp owns one utterance:
//
//   * lane e of a half holds beam entry e (score f64, prefix hash, parent
//     hash, last token, length, blank flag) AND, when it is the first entry of
//     its prefix, that prefix's sorted append list -- so the whole frame step
//     runs on 16 lanes and one warp instruction advances two utterances;
//   * rows are staged speculatively by TMA (cp.async.bulk, one frame ahead);
//     blank skipping (emissions.py:298-306) is decided on the staged row's
//     blank value, so there is no separate strided pass over the blank column;
//   * top-k (k = 2 beam): 2 group maxima per lane -> a 2-per-lane 32-element
//     bitonic sort gives a threshold reached by >= k values -> index-ordered
//     compaction -> a 2- (or 4-) per-lane register sort of truncated keys;
//   * merge structure: two warp-wide match.any calls over {h of one half,
//     parent hashes of the same utterance mirrored from the other half} give
//     both utterances' flag variants and parent entries (decoder.py:595-613);
//   * selection: a k-way merge over the lanes' (specials, append list) queues
//     with per-half redux.sync on 32-bit fixed-point keys; heads within the
//     key tolerance are resolved exactly (fp64 fold, token sequence, flag:
//     decoder.py:651-681);
//   * back-pointers: a 16-bit trellis (source slot << 12 | token + 1) plus a
//     16-step shared-memory ring for checkpoint ancestors (n-best backtrace).
#include <cfloat>
#include <cmath>

#include "ctcb_common.cuh"
#include "ctcb_internal.h"
#include <cstdio>

#ifdef CTCB_PAIR_CHECK
#define PCHK(c)                                                                                   \
  do {                                                                                            \
    if (!(c)) {                                                                                   \
      printf("ctcb_pair check failed: %s (line %d, block %d, thread %d)\n", #c, __LINE__, blockIdx.x, threadIdx.x); \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define PCHK(c) do { } while (0)
#endif
#ifdef CTCB_PAIR_DIVCHK
#define PDIV(id)                                                                   \
  do {                                                                             \
    const unsigned am_ = __activemask();                                           \
    if (am_ != FULL && (__ffs(am_) - 1) == (int)(threadIdx.x & 31)) atomicAdd(&P.dbg[id], 1ull); \
  } while (0)
#else
#define PDIV(id) do { } while (0)
#endif

namespace ctcb {

namespace {

constexpr uint64_t kPDummy = 0xa5a5a5a55a5a5a5aull;
constexpr uint32_t kPSent = 0xffffffffu;  // NaN sentinel: order key 0
constexpr uint32_t kPTol = 3u;            // rank-key tolerance (keys are within 2 units of exact)

__device__ __forceinline__ uint32_t pkey(float x) {
  uint32_t u = __float_as_uint(x);
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ double punord64(uint64_t k) {
  uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}
__device__ __forceinline__ uint32_t pf2u_sat(double z) {
  uint32_t r;
  asm("cvt.rzi.u32.f64 %0, %1;" : "=r"(r) : "d"(z));
  return r;
}
__device__ __forceinline__ long long pf2ll_floor(double z) {
  long long r;
  asm("cvt.rmi.s64.f64 %0, %1;" : "=l"(r) : "d"(z));
  return r;
}
// shuffles inside a 16-lane half (src relative to the half)
__device__ __forceinline__ int hsh(int v, int src, unsigned m = FULL) { return __shfl_sync(m, v, src, 16); }
__device__ __forceinline__ uint32_t hshu(uint32_t v, int src, unsigned m = FULL) { return __shfl_sync(m, v, src, 16); }
__device__ __forceinline__ double hshd(double v, int src, unsigned m = FULL) { return __shfl_sync(m, v, src, 16); }
__device__ __forceinline__ uint64_t hsh64(uint64_t v, int src, unsigned m = FULL) {
  const uint32_t lo = __shfl_sync(m, (uint32_t)v, src, 16), hi = __shfl_sync(m, (uint32_t)(v >> 32), src, 16);
  return ((uint64_t)hi << 32) | lo;
}

// Per-half reductions with full-warp (uniform-mask) redux: a non-uniform
// member mask makes the compiler wrap the collective in a loop.
__device__ __forceinline__ uint32_t seg_max(uint32_t v, int hf) {
  const uint32_t a = __reduce_max_sync(FULL, hf ? 0u : v), b = __reduce_max_sync(FULL, hf ? v : 0u);
  return hf ? b : a;
}
__device__ __forceinline__ uint32_t seg_sum(uint32_t v, int hf) {
  const uint32_t a = __reduce_add_sync(FULL, hf ? 0u : v), b = __reduce_add_sync(FULL, hf ? v : 0u);
  return hf ? b : a;
}
__device__ __forceinline__ bool seg_any(bool p, unsigned seg) { return (__ballot_sync(FULL, p) & seg) != 0u; }

__device__ __forceinline__ uint64_t hsh64x(uint64_t v, int m) {
  const uint32_t lo = __shfl_xor_sync(FULL, (uint32_t)v, m, 16), hi = __shfl_xor_sync(FULL, (uint32_t)(v >> 32), m, 16);
  return ((uint64_t)hi << 32) | lo;
}

// One non-blocking probe of an mbarrier phase (the caller loops warp-uniformly).
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0u;
}

// 16-bit trellis record: source slot (4 bits) | token + 1 (12 bits)
__device__ __forceinline__ uint16_t ptrel(int src, int tok) { return (uint16_t)((src << 12) | (tok + 1)); }
__device__ __forceinline__ int ptrel_src(uint32_t r) { return (int)(r >> 12); }
__device__ __forceinline__ int ptrel_tok(uint32_t r) { return (int)(r & 0xfffu) - 1; }

// 32 keys held two per lane (element 2*hl + r) over a 16-lane half: bitonic
// sort, descending.
__device__ __forceinline__ void sort2_desc(uint32_t& x0, uint32_t& x1, int hl, unsigned msk = FULL) {
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      if (j == 1) {
        const bool desc = ((2 * hl) & size) == 0;
        const uint32_t a = max(x0, x1), b = min(x0, x1);
        x0 = desc ? a : b;
        x1 = desc ? b : a;
      } else {
        const int m = j >> 1;
        const uint32_t y0 = __shfl_xor_sync(msk, x0, m, 16), y1 = __shfl_xor_sync(msk, x1, m, 16);
        const bool tmax = ((hl & m) == 0) == (((2 * hl) & size) == 0);
        x0 = tmax ? max(x0, y0) : min(x0, y0);
        x1 = tmax ? max(x1, y1) : min(x1, y1);
      }
    }
  }
}
// 64 keys held four per lane (element 4*hl + r), descending.
__device__ __forceinline__ void sort4_desc(uint32_t (&x)[4], int hl, unsigned msk = FULL) {
#pragma unroll
  for (int size = 2; size <= 64; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      if (j <= 2) {
#pragma unroll
        for (int lo = 0; lo < 4; lo++) {
          if (lo & j) continue;
          const int hi = lo | j;
          const bool desc = ((4 * hl + lo) & size) == 0;
          const uint32_t a = max(x[lo], x[hi]), b = min(x[lo], x[hi]);
          x[lo] = desc ? a : b;
          x[hi] = desc ? b : a;
        }
      } else {
        const int m = j >> 2;
        const bool tmax = ((hl & m) == 0) == (((4 * hl) & size) == 0);
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const uint32_t y = __shfl_xor_sync(msk, x[r], m, 16);
          x[r] = tmax ? max(x[r], y) : min(x[r], y);
        }
      }
    }
  }
}

// Per-half shared memory.
struct PairSmem {
  float* rows;        // [kPairRing][kSmallV]
  uint64_t* mbar;     // [kPairRing]
  float* sval;        // [32] sorted top-k values
  int* stok;          // [32] sorted top-k tokens
  long long* wp;      // [32] floor(v * 2^32 / R)
  uint16_t* cidx;     // [64] top-k survivors (index order)
  uint8_t* posmap;    // [kSmallV] token -> top-k rank (0xff: none)
  uint32_t* excl;     // [16] flag-0 children positions per prefix owner
  int* rec;           // [32] merge record per new entry (+ scratch)
  uint64_t* hs;       // [16] entry hashes (exact slow paths)
  int* hl;            // [16] entry lengths
  double* hsc;        // [16] entry scores
  int* hp2;           // [16] flag partner
  double* tie_sc;     // [32] exact scores of tied heads (also 64-bit keys of the top-k fix)
  int* tie_i;         // [32 * 4]
  uint64_t* tc_h;     // [2 * kTieCache] tie-order cache keys
  int* tc_r;          // [kTieCache + 1]
  uint16_t* tring;    // [kChunk][16] trellis ring for checkpoints
};

__device__ PairSmem pair_smem(uint8_t* base) {
  const PairLayout L = make_pair_layout();
  PairSmem S;
  S.rows = (float*)(base + L.rows);
  S.mbar = (uint64_t*)(base + L.mbar);
  S.sval = (float*)(base + L.sval);
  S.stok = (int*)(base + L.stok);
  S.wp = (long long*)(base + L.wp);
  S.cidx = (uint16_t*)(base + L.cidx);
  S.posmap = base + L.posmap;
  S.excl = (uint32_t*)(base + L.excl);
  S.rec = (int*)(base + L.rec);
  S.hs = (uint64_t*)(base + L.hs);
  S.hl = (int*)(base + L.hl);
  S.hsc = (double*)(base + L.hsc);
  S.hp2 = (int*)(base + L.hp2);
  S.tie_sc = (double*)(base + L.tie_sc);
  S.tie_i = (int*)(base + L.tie_i);
  S.tc_h = (uint64_t*)(base + L.tc_h);
  S.tc_r = (int*)(base + L.tc_r);
  S.tring = (uint16_t*)(base + L.tring);
  return S;
}

// ---------------------------------------------------------------- exact ties
__device__ int ptc_lookup(const PairSmem& S, uint64_t ha, uint64_t hb) {
#pragma unroll 1
  for (int i = 0; i < kTieCache; i++) {
    if (S.tc_h[2 * i] == ha && S.tc_h[2 * i + 1] == hb) return S.tc_r[i];
    if (S.tc_h[2 * i] == hb && S.tc_h[2 * i + 1] == ha) return -S.tc_r[i];
  }
  return 0;
}
__device__ void ptc_insert(const PairSmem& S, uint64_t ha, uint64_t hb, int r) {
  if (ptc_lookup(S, ha, hb)) return;
  const int i = S.tc_r[kTieCache];
  S.tc_h[2 * i] = ha;
  S.tc_h[2 * i + 1] = hb;
  S.tc_r[i] = r;
  S.tc_r[kTieCache] = (i + 1) % kTieCache;
}
__device__ int pair_seq_cmp_full(const Params& P, const PairSmem& S, int u, int sd, int ea, int xa, int eb, int xb,
                                 bool* strict) {
  int* A = P.seqbuf + (size_t)u * 3 * (P.T_max + 1);
  const uint16_t* tr = (const uint16_t*)P.trellis + (size_t)u * P.T_max * P.beam;  // 16-bit records
  auto rec = [&](int i, int slot) {
    const uint32_t r = tr[(size_t)i * P.beam + slot];
    return make_int2(ptrel_tok(r), ptrel_src(r));
  };
  return trellis_seq_cmp(rec, sd, ea, xa, eb, xb, A, A + P.T_max + 1, strict, P.dbg);
}
// Python tuple order of seq(ea)+[xa] vs seq(eb)+[xb] (x < 0: no extra token).
__device__ int pair_seq_cmp(const Params& P, const PairSmem& S, int u, int sd, int ea, int xa, int eb, int xb) {
  const uint64_t hba = S.hs[ea], hbb = S.hs[eb];
  const int lba = S.hl[ea], lbb = S.hl[eb];
  if (hba == hbb && lba == lbb) {
    if (xa == xb) return 0;
    return xa < xb ? -1 : 1;
  }
  const uint64_t ha = xa >= 0 ? child_hash(hba, xa) : hba, hb = xb >= 0 ? child_hash(hbb, xb) : hbb;
  const int la = lba + (xa >= 0), lb = lbb + (xb >= 0);
  if (ha == hb && la == lb) return 0;
  int r = ptc_lookup(S, hba, hbb);
  if (r) {
    ptc_insert(S, ha, hb, r);
    return r;
  }
  r = ptc_lookup(S, ha, hb);
  if (r) return r;
  bool strict = false;
  r = pair_seq_cmp_full(P, S, u, sd, ea, -1, eb, -1, &strict);
  if (strict) {
    ptc_insert(S, hba, hbb, r);
    ptc_insert(S, ha, hb, r);
    return r;
  }
  r = pair_seq_cmp_full(P, S, u, sd, ea, xa, eb, xb, &strict);
  if (strict) ptc_insert(S, ha, hb, r);
  return r;
}
// a precedes b: score desc, token sequence asc, flag asc (decoder.py:651-681).
__device__ bool pair_precedes(const Params& P, const PairSmem& S, int u, int sd, double sa, int ba, int xa, int fa,
                              double sb, int bb, int xb, int fb) {
  if (sa != sb) return sa > sb;
  atomicAdd(&P.dbg[kDbgExactTies], 1ull);
  const int c = pair_seq_cmp(P, S, u, sd, ba, xa, bb, xb);
  if (c) return c < 0;
  return fa < fb;
}

// ---------------------------------------------------------------- top-k
// Sorted top-k (k <= 32) of one staged row (V <= 512, padding = sentinel,
// blank = 0 masked) for each active half of the warp; writes stok / sval /
// wp / posmap of the half.  All 32 lanes call it; collectives use the half's
// lane mask, so the halves may take different (rare) fallback branches.
__device__ __forceinline__ void pair_topk(const PairSmem& S, const float* row, bool act, int V, int k, double kScale,
                                          int hl, unsigned seg, unsigned long long* dbg) {
  const float4* row4 = (const float4*)row;
  const float sent = __uint_as_float(kPSent);
  float4 q[8];
#pragma unroll
  for (int j = 0; j < 8; j++) q[j] = act ? row4[hl + 16 * j] : make_float4(sent, sent, sent, sent);
  if (hl == 0) q[0].x = sent;  // blank (index 0) is not a candidate
  auto m4 = [](float4 a) { return fmaxf(fmaxf(a.x, a.y), fmaxf(a.z, a.w)); };
  const float g0 = fmaxf(fmaxf(m4(q[0]), m4(q[1])), fmaxf(m4(q[2]), m4(q[3])));
  const float g1 = fmaxf(fmaxf(m4(q[4]), m4(q[5])), fmaxf(m4(q[6]), m4(q[7])));
  // threshold: k-th largest of the 32 group maxima (>= k values reach it)
  uint32_t a0 = isnan(g0) ? 0u : pkey(g0), a1 = isnan(g1) ? 0u : pkey(g1);
  sort2_desc(a0, a1, hl);
  const uint32_t t0 = hshu(((k - 1) & 1) ? a1 : a0, (k - 1) >> 1);
  const float tf = t0 == 0u ? -INFINITY : unord32(t0);
  // survivors: predicate nibbles of the 8 chunks, per-chunk counts packed in bytes
  uint32_t pm = 0u, c0 = 0u, c1 = 0u;
#pragma unroll
  for (int j = 0; j < 8; j++) {
    const uint32_t nib = (uint32_t)(q[j].x >= tf) | ((uint32_t)(q[j].y >= tf) << 1) |
                         ((uint32_t)(q[j].z >= tf) << 2) | ((uint32_t)(q[j].w >= tf) << 3);
    pm |= nib << (4 * j);
    if (j < 4) c0 |= (uint32_t)__popc(nib) << (8 * j);
    else c1 |= (uint32_t)__popc(nib) << (8 * (j - 4));
  }
  const int hf = (threadIdx.x >> 4) & 1;
  const int cnt = (int)seg_sum((unsigned)__popc(pm), hf);
  const bool big = __any_sync(FULL, cnt > 32);  // warp-uniform sort width
  if (__any_sync(FULL, cnt > 64 || cnt < k)) {  // cnt < k: NaN input leaves too few survivors
    // many exact ties above the threshold: exact selection by k rounds of a
    // segmented max over (value desc, index asc) keys (rare)
    // (both halves take this path; it is exact for any row)
    if (hl == 0 && dbg && cnt > 64) atomicAdd(&dbg[kDbgRadix], 1ull);
    uint32_t taken = 0u;
    for (int p = 0; p < k; p++) {
      uint64_t bestk = 0ull;
      int bj = -1;
      for (int bt = 0; bt < 32; bt++) {
        const int idx = 4 * (hl + 16 * (bt >> 2)) + (bt & 3);
        if ((taken & (1u << bt)) || idx == 0 || idx >= V) continue;
        const uint32_t kk = pkey(row[idx]);
        if (kk == 0u) continue;
        const uint64_t key = ((uint64_t)kk << 32) | (uint64_t)(0xffffffffu - (uint32_t)idx);
        if (key > bestk) { bestk = key; bj = bt; }
      }
      const uint32_t hi = seg_max((uint32_t)(bestk >> 32), hf);
      const uint32_t lo = seg_max((uint32_t)(bestk >> 32) == hi ? (uint32_t)bestk : 0u, hf);
      if (bj >= 0 && (uint32_t)(bestk >> 32) == hi && (uint32_t)bestk == lo) taken |= 1u << bj;
      if (hl == 0 && act) S.stok[p] = (int)(0xffffffffu - lo);
    }
    __syncwarp();
  } else {
    // index-ordered compaction: chunk j of lane l starts after the survivors
    // of chunks < j (all lanes) and of chunk j in lanes < l
    uint32_t i0 = c0, i1 = c1;
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) {
      const uint32_t y0 = __shfl_up_sync(FULL, i0, o, 16), y1 = __shfl_up_sync(FULL, i1, o, 16);
      if (hl >= o) { i0 += y0; i1 += y1; }
    }
    const uint32_t tot0 = hshu(i0, 15), tot1 = hshu(i1, 15);
    uint32_t offs0 = tot0 * 0x01010100u + (i0 - c0);
    const uint32_t base1 = (tot0 * 0x01010101u) >> 24;
    uint32_t offs1 = tot1 * 0x01010100u + (i1 - c1) + base1 * 0x01010101u;
    // (loop bounds are warp-uniform everywhere in the frame step: lane-dependent
    // trip counts can leave the warp split into groups the compiler never
    // re-merges, and the full-mask collectives below then misbehave)
    uint32_t bits = pm;
    const int nit = (int)__reduce_max_sync(FULL, (unsigned)__popc(pm));
    for (int it = 0; it < nit; it++) {
      if (bits) {
        const int bt = __ffs(bits) - 1;
        bits &= bits - 1u;
        const bool lo = bt < 16;
        const int sh = 8 * ((bt >> 2) & 3);
        const uint32_t off = ((lo ? offs0 : offs1) >> sh) & 0xffu;
        if (lo) offs0 += 1u << sh;
        else offs1 += 1u << sh;
        PCHK(off < 64);
        S.cidx[off] = (uint16_t)(4 * (hl + 16 * (bt >> 2)) + (bt & 3));
      }
    }
    __syncwarp();
    // key = (order key with the low 6 bits cleared) | (63 - slot): value desc,
    // then index asc (slots are in index order); the lane holding rank p
    // writes stok[p]
    bool bad = false;
    if (!big) {
      uint32_t x0 = 2 * hl < cnt ? ((pkey(row[S.cidx[2 * hl]]) & ~63u) | (uint32_t)(63 - 2 * hl)) : 0u;
      uint32_t x1 = 2 * hl + 1 < cnt ? ((pkey(row[S.cidx[2 * hl + 1]]) & ~63u) | (uint32_t)(62 - 2 * hl)) : 0u;
      sort2_desc(x0, x1, hl);
      const uint32_t nx = __shfl_down_sync(FULL, x0, 1, 16);
      const uint32_t x2 = hl < 15 ? nx : 0u;
      bad = (2 * hl < k && x0 != 0u && (x0 >> 6) == (x1 >> 6)) ||
            (2 * hl + 1 < k && x1 != 0u && (x1 >> 6) == (x2 >> 6));
      PCHK(!act || 2 * hl >= k || (x0 != 0u && 63 - (x0 & 63u) < cnt));
      if (act && 2 * hl < k) S.stok[2 * hl] = S.cidx[63 - (x0 & 63u)];
      if (act && 2 * hl + 1 < k) S.stok[2 * hl + 1] = S.cidx[63 - (x1 & 63u)];
    } else {
      uint32_t x[4];
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const int e = 4 * hl + r;
        x[r] = e < cnt ? ((pkey(row[S.cidx[e]]) & ~63u) | (uint32_t)(63 - e)) : 0u;
      }
      sort4_desc(x, hl);
      const uint32_t nx = __shfl_down_sync(FULL, x[0], 1, 16);
      const uint32_t x4 = hl < 15 ? nx : 0u;
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const uint32_t nb = r < 3 ? x[r + 1] : x4;
        bad |= 4 * hl + r < k && x[r] != 0u && (x[r] >> 6) == (nb >> 6);
        PCHK(!act || 4 * hl + r >= k || (x[r] != 0u && 63 - (x[r] & 63u) < cnt));
        if (act && 4 * hl + r < k) S.stok[4 * hl + r] = S.cidx[63 - (x[r] & 63u)];
      }
    }
    __syncwarp();
    if (__any_sync(FULL, bad)) {
      // truncated keys collide: exact ranks of 64-bit keys by counting (rare;
      // both halves take this path, it is exact for any row)
      const bool mine = seg_any(bad, seg);
      if (hl == 0 && dbg && mine) atomicAdd(&dbg[kDbgTopkFix], 1ull);
      uint64_t* k64 = (uint64_t*)S.tie_sc;  // 64 x 8 B (tie_sc + tie_i)
#pragma unroll
      for (int e0 = 0; e0 < 64; e0 += 16) {
        const int e = e0 + hl;
        if (e < cnt) {
          const int idx = S.cidx[e];
          k64[e] = ((uint64_t)pkey(row[idx]) << 32) | (uint64_t)(0xffffffffu - (uint32_t)idx);
        }
      }
      __syncwarp();
      const int cmax = max(cnt, __shfl_xor_sync(FULL, cnt, 16));
#pragma unroll
      for (int e0 = 0; e0 < 64; e0 += 16) {
        const int e = e0 + hl;
        const uint64_t me = e < cnt ? k64[e] : 0ull;
        int rank = 0;
        for (int f = 0; f < cmax; f++) rank += (f < cnt && k64[f] > me) ? 1 : 0;
        if (act && e < cnt && rank < k) S.stok[rank] = S.cidx[e];
      }
      __syncwarp();
    }
  }
#pragma unroll
  for (int p0 = 0; p0 < 32; p0 += 16) {
    const int p = p0 + hl;
    if (act && p < k) {
      const int tok = S.stok[p];
      PCHK(tok > 0 && tok < V);
      const float v = row[tok];
      S.sval[p] = v;
      S.wp[p] = pf2ll_floor((double)v * kScale);
      S.posmap[tok] = (uint8_t)p;
    }
  }
  __syncwarp();
}

}  // namespace

#ifndef CTCB_PAIR_MIN_BLOCKS
#define CTCB_PAIR_MIN_BLOCKS 3
#endif

__global__ void __launch_bounds__(128, CTCB_PAIR_MIN_BLOCKS) ctcb_decode_pair_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int hf = lane >> 4, hl = lane & 15;
  const unsigned seg = 0xffffu << (16 * hf);
  const PairLayout PL = make_pair_layout();
  uint8_t* hbase = smem + (size_t)(2 * wid + hf) * PL.total;
  const PairSmem S = pair_smem(hbase);
  uint16_t* tr16 = (uint16_t*)P.trellis;

  const int V = P.V, k = P.k, beam = P.beam;
  const bool MX = P.merge_max != 0;
  const uint32_t fullk = k >= 32 ? 0xffffffffu : ((1u << k) - 1u);
  const double kR = P.threshold_inf ? 1048576.0 : fmin(P.beam_threshold, 1048576.0);
  const double kScale = 4294967296.0 / kR;
  const uint32_t row_copy = (uint32_t)V * 4u;

  // one-time init of this half's shared memory
  for (int c0 = 0; c0 < 2 * kTieCache + 16; c0 += 16) {
    const int c = c0 + hl;
    if (c < 2 * kTieCache) S.tc_h[c] = 0ull;
    if (c <= kTieCache) S.tc_r[c] = 0;
  }
  for (int c0 = 0; c0 < kSmallV; c0 += 16) {
    const int c = c0 + hl;
    S.posmap[c] = 0xff;
    if (c >= V)
      for (int s = 0; s < kPairRing; s++) ((uint32_t*)(S.rows + s * kSmallV))[c] = kPSent;
  }
  if (hl == 0)
    for (int s = 0; s < kPairRing; s++) mbar_init(&S.mbar[s], 1);
  fence_mbar_init();
  __syncwarp();

  // per-half utterance state
  int u = -1, len_u = 0, t = 0, i = 0;  // utterance, length, next frame, kept frames so far
  bool exhausted = false;
  uint32_t n_iss = 0, n_cons = 0;       // rows issued / consumed by this half (ring slot = n & 1)
  const float* ubase = nullptr;
  // beam state (decoder.py:358-370)
  double s = 0.0;
  uint64_t h = kEmptyPrefixHash, ph = 0ull;
  int last = -1, len = 0, fl = 1, H = 0;
  bool died = false;
  int died_at = 0;

  auto issue = [&](int fr) {  // TMA row fr of the current utterance into slot n_iss & 1
    if (hl == 0) {
      const int sl = n_iss & 1;
      fence_proxy_async();
      mbar_arrive_expect_tx(&S.mbar[sl], row_copy);
      tma_bulk_g2s(S.rows + sl * kSmallV, ubase + (size_t)fr * P.stride_t, row_copy, &S.mbar[sl]);
    }
    n_iss++;
  };

  // Control flow is warp-uniform throughout: both halves execute every
  // collective with the full mask (a half-mask warpsync on one half while the
  // other waits at a full-mask one is undefined), and per-half work is
  // predicated on the half's own state.
  bool have_row = false;
  for (;;) {
    // ---------------- utterance bookkeeping: claim, finalize, next kept row
    for (;;) {
      const bool need = !exhausted && u < 0;
      if (__any_sync(FULL, need)) {  // claim the next utterance (longest first)
        int item = 0;
        if (need && hl == 0) item = atomicAdd(P.counter, 1);
        item = hsh(item, 0);
        if (need) {
          if (item >= P.B) {
            exhausted = true;
          } else {
            u = P.order[item];
            len_u = P.lens[u];
            if (len_u <= 0 || len_u > P.T_max) {
              if (hl == 0) {
                P.status[u] = len_u == 0 ? kUttEmpty : kUttBadLen;
                P.out_count[u] = 0;
                P.kept[u] = 0;
              }
              u = -1;
            } else {
              ubase = P.lp + (size_t)u * P.stride_b;
              t = 0;
              i = 0;
              s = 0.0;
              h = kEmptyPrefixHash;
              ph = 0ull;
              last = -1;
              len = 0;
              fl = 1;
              H = 1;
              died = false;
              have_row = false;
              issue(0);
              if (len_u > 1) issue(1);
            }
          }
        }
        continue;
      }
      const bool fin = !exhausted && (t >= len_u || died);
      if (__any_sync(FULL, fin)) {
        // ---------------- finalize (decoder.py:753-817) of the halves in `fin`
        if (fin && hl == 0) P.kept[u] = i;
        if (fin && !died && (i % kChunk) != 0 && hl < H) {  // checkpoint of the partial last chunk
          int slot = hl;
#pragma unroll
          for (int tt = kChunk - 1; tt >= 0; --tt)
            if (tt <= (i - 1) % kChunk) slot = ptrel_src(S.tring[tt * 16 + slot]);
          P.anc[((size_t)u * P.n_chunks + (i - 1) / kChunk) * 16 + hl] = (uint8_t)slot;
        }
        for (;;) {  // died: drain rows still in flight (warp-uniform polling)
          const bool more = fin && died && n_cons < n_iss;
          if (!__any_sync(FULL, more)) break;
          if (more && mbar_try(&S.mbar[n_cons & 1], (n_cons >> 1) & 1u)) n_cons++;
        }
        if (fin && died) {
          if (hl == 0) {
            P.status[u] = kUttBeamDied;
            P.out_count[u] = 0;
            P.out_len[(size_t)u * P.nbest] = died_at;
          }
        }
        const bool fo = fin && !died;  // this half emits its n-best
        const bool ent = fo && hl < H;
        // flag variants of one prefix (decoder.py:789-791); keys of the two
        // halves may coincide, the half's own bits are kept
        const unsigned fm = __match_any_sync(FULL, ent ? h : (kPDummy ^ (uint64_t)lane));
        const unsigned fmh = (fm >> (16 * hf)) & 0xffffu;
        const bool isf = ent && (__ffs(fmh) - 1) == hl;
        const unsigned pmk = fmh & ~(1u << hl);
        const int p2 = (ent && pmk) ? __ffs(pmk) - 1 : -1;
        const double s_p2 = hshd(s, p2 >= 0 ? p2 : hl);
        const double gsc = isf ? (p2 >= 0 ? merge2(s, s_p2, MX) : s) : -INFINITY;
        // order groups: (score desc, lane asc) by a 16-lane register sort
        uint64_t key = isf ? ord64(gsc) : 0ull;
        int pay = hl;
#pragma unroll 1
        for (int size = 2; size <= 16; size <<= 1)
#pragma unroll 1
          for (int j = size >> 1; j > 0; j >>= 1) {
            const uint64_t ky = hsh64x(key, j);
            const int py = __shfl_xor_sync(FULL, pay, j, 16);
            const bool mine_first = key > ky || (key == ky && pay < py);
            const bool take_first = ((hl & j) == 0) == ((hl & size) == 0);
            if (take_first != mine_first) { key = ky; pay = py; }
          }
        const int nF = __popc((__ballot_sync(FULL, isf) >> (16 * hf)) & 0xffffu);
        const double srt_sc = hshd(gsc, pay);
        S.tie_i[hl] = pay;
        S.tie_sc[hl] = srt_sc;
        S.hs[hl] = h;
        S.hl[hl] = len;
        __syncwarp();
        if (fo && hl == 0) {  // exact tie runs (identical fp64 scores): token-sequence order
          for (int a = 1; a < nF; a++) {
            int j = a;
            while (j > 0 && S.tie_sc[j] == S.tie_sc[j - 1] &&
                   pair_seq_cmp(P, S, u, i, S.tie_i[j], -1, S.tie_i[j - 1], -1) < 0) {
              const int tt = S.tie_i[j];
              S.tie_i[j] = S.tie_i[j - 1];
              S.tie_i[j - 1] = tt;
              j--;
            }
          }
        }
        __syncwarp();
        const int nOut = fo ? (nF < P.nbest ? nF : P.nbest) : 0;
        const int nchk = fo ? (i + kChunk - 1) / kChunk : 0;
        const int nOutMax = max(nOut, __shfl_xor_sync(FULL, nOut, 16));
        const int nchkMax = max(nchk, __shfl_xor_sync(FULL, nchk, 16));
        int* ends = fo ? P.seqbuf + (size_t)u * 3 * (P.T_max + 1) : nullptr;
        int* tmp_tok = ends + (P.T_max + 1);
        int* tmp_fr = tmp_tok + (P.T_max + 1);
        const int32_t* fmap = P.frame_map + (size_t)(fo ? u : 0) * P.T_max;
        for (int r = 0; r < nOutMax; r++) {
          const bool on = r < nOut;
          const int e = on ? S.tie_i[r] : 0;
          const double sc = hshd(gsc, e);
          const int L_e = hsh(len, e);
          const size_t o = (size_t)(on ? u : 0) * P.nbest + r;
          if (on && hl == 0) { P.out_score[o] = sc; P.out_len[o] = L_e; }
          int* tok_out = P.out_tokens + o * P.T_max;
          int* ts_out = P.out_ts ? P.out_ts + o * P.T_max : nullptr;
          const bool walk = on && L_e > 0 && nchk > 0;
          if (walk && hl == 0) {  // coarse walk over checkpoints
            int slot = e;
            for (int c = nchk - 1; c >= 0; --c) {
              ends[c] = slot;
              slot = P.anc[((size_t)u * P.n_chunks + c) * 16 + slot];
            }
          }
          __syncwarp();
          for (int c0 = 0; c0 < nchkMax; c0 += 16) {  // fine walks, one chunk per lane
            const int c = c0 + hl;
            if (walk && c < nchk) {
              int slot = ends[c], cntc = 0;
              const int i_end = min(i, (c + 1) * kChunk) - 1;
              for (int d = kChunk - 1; d >= 0; --d) {
                const int ii = c * kChunk + d;
                if (ii > i_end) continue;
                PCHK(slot >= 0 && slot < beam && ii >= 0 && ii < P.T_max);
                const uint32_t rec = tr16[((size_t)u * P.T_max + ii) * beam + slot];
                const int tok = ptrel_tok(rec);
                if (tok >= 0) {
                  tmp_tok[c * kChunk + cntc] = tok;
                  tmp_fr[c * kChunk + cntc] = fmap[ii];
                  cntc++;
                }
                slot = ptrel_src(rec);
              }
              ends[c] = cntc;
            }
          }
          __syncwarp();
          int running = 0;
          for (int b0 = 0; b0 < nchkMax; b0 += 16) {
            const int c = b0 + hl;
            const int cnt_c = (walk && c < nchk) ? ends[c] : 0;
            int incl = cnt_c;
#pragma unroll
            for (int o2 = 1; o2 < 16; o2 <<= 1) {
              const int y = __shfl_up_sync(FULL, incl, o2, 16);
              if (hl >= o2) incl += y;
            }
            const int off = running + incl - cnt_c;
            for (int q = 0; q < kChunk; q++) {
              if (q < cnt_c) {
                tok_out[off + q] = tmp_tok[c * kChunk + cnt_c - 1 - q];
                if (ts_out) ts_out[off + q] = tmp_fr[c * kChunk + cnt_c - 1 - q];
              }
            }
            running += hsh(incl, 15);
          }
          __syncwarp();
        }
        if (fo && hl == 0) { P.out_count[u] = nOut; P.status[u] = kUttOk; }
        if (fin) u = -1;
        __syncwarp();
        continue;
      }
      // next frame: speculative row, skip decided on its blank value (emissions.py:298-306)
      const bool wantr = !exhausted && !have_row;
      bool ready = !wantr;
      while (!__all_sync(FULL, ready))  // warp-uniform polling of the halves' row barriers
        if (!ready) ready = mbar_try(&S.mbar[n_cons & 1], (n_cons >> 1) & 1u);
      if (wantr) {
        const float ebf = S.rows[(n_cons & 1) * kSmallV];
        if (P.skip && ebf >= P.cutoff) {  // dropped frame: the slot is free again
          n_cons++;
          if (t + 2 < len_u) issue(t + 2);
          t++;
        } else {
          have_row = true;
        }
      }
      if (__any_sync(FULL, !exhausted && !have_row)) continue;
      break;
    }
    if (__all_sync(FULL, exhausted)) break;
    const bool act = !exhausted;
    PDIV(0);
    float* row = S.rows + (n_cons & 1) * kSmallV;
    if (act) {
      n_cons++;
      have_row = false;
    }

    // ---------------- frame step, both halves (warp-uniform control flow)
    const double eb = act ? (double)row[0] : 0.0;
    pair_topk(S, row, act, V, k, kScale, hl, seg, P.dbg);
    PDIV(1);

    // merge structure: call A = utterance of half 0 (h on lanes 0-15, parent
    // hashes on 16-31), call B = half 1 (parents on 0-15, h on 16-31)
    const bool ent = act && hl < H;
    const uint64_t xph = ((uint64_t)__shfl_xor_sync(FULL, (uint32_t)(ph >> 32), 16) << 32) |
                         __shfl_xor_sync(FULL, (uint32_t)ph, 16);
    const int xok = __shfl_xor_sync(FULL, (ent && len > 0) ? 1 : 0, 16);
    const uint64_t dum = kPDummy ^ (uint64_t)lane;
    const uint64_t kA = hf == 0 ? (ent ? h : dum) : (xok ? xph : dum);
    const uint64_t kB = hf == 1 ? (ent ? h : dum) : (xok ? xph : dum);
    const unsigned mA = __match_any_sync(FULL, kA);
    const unsigned mB = __match_any_sync(FULL, kB);
    const unsigned same = hf ? (mB >> 16) : (mA & 0xffffu);
    const unsigned pout = hf ? (mA & 0xffffu) : (mB >> 16);
    const unsigned pin = __shfl_xor_sync(FULL, pout, 16);
    const unsigned parents = ent ? pin : 0u;
    const bool isfirst = ent && (__ffs(same) - 1) == hl;
    const unsigned pmask = same & ~(1u << hl);
    const int p2 = (ent && pmask) ? __ffs(pmask) - 1 : -1;
    const double s_p2 = hshd(s, p2 >= 0 ? p2 : hl);
    const int fl_p2 = hsh(fl, p2 >= 0 ? p2 : hl);

    PCHK(!ent || (last >= -1 && last < V));
    const int mypos = (ent && last >= 0) ? (int)S.posmap[last] : 0xff;
    const uint32_t mybit = mypos < 32 ? (1u << mypos) : 0u;
    S.excl[hl] = 0u;
    __syncwarp();
    const int pa = (ent && parents) ? __ffs(parents) - 1 : -1;
#ifdef CTCB_PAIR_CHECK
    if (pa >= 16) printf("pa %d lane %d hf %d H %d parents %08x pin %08x pout %08x mA %08x mB %08x same %08x xok %d ent %d\n", pa, lane, hf, H, parents, pin, pout, mA, mB, same, xok, (int)ent);
#endif
    PCHK(pa < 16);
    if (ent && fl == 0 && pa >= 0 && mybit) atomicOr(&S.excl[pa], mybit);
    __syncwarp();
    const uint32_t childx = S.excl[hl];

    PDIV(2);
    // ---------------- special groups
    const unsigned pr2 = parents & (parents - 1);
    const int pb = (ent && pr2) ? __ffs(pr2) - 1 : -1;
    const double s_pa = hshd(s, pa >= 0 ? pa : hl);
    const int fl_pa = hsh(fl, pa >= 0 ? pa : hl);
    const int last_pa = hsh(last, pa >= 0 ? pa : hl);
    const double s_pb = hshd(s, pb >= 0 ? pb : hl);
    const int fl_pb = hsh(fl, pb >= 0 ? pb : hl);
    const int last_pb = hsh(last, pb >= 0 ? pb : hl);
    double c_blank = -INFINITY, c_rep = -INFINITY, c_single = -INFINITY;
    int rep_src = hl, rep_tok = -1, single_src = hl;
    if (isfirst) {  // blank group (R,1): entries of R in rank order (decoder.py:513-521)
      c_blank = s + eb;
      if (p2 >= 0) c_blank = merge2(c_blank, s_p2 + eb, MX);
    }
    if (ent && fl == 0) {  // repeat group (R',0): repeat first, then parent appends (:522-543)
      PCHK(last > 0 && last < V);
      const double ec = (double)row[last];
      double sc = s + ec, bst = sc;
      if (pa >= 0 && !(fl_pa == 0 && last_pa == last)) {
        const double x = s_pa + ec;
        sc = merge2(sc, x, MX);
        if (x > bst) { bst = x; rep_src = pa; rep_tok = last; }
      }
      if (pb >= 0 && !(fl_pb == 0 && last_pb == last)) {
        const double x = s_pb + ec;
        sc = merge2(sc, x, MX);
        if (x > bst) { bst = x; rep_src = pb; rep_tok = last; }
      }
      c_rep = sc;
    }
    if (isfirst && mybit && !(childx & mybit)) {  // (R+last(R),0) from (R,1) only
      const int f1 = fl == 1 ? hl : ((p2 >= 0 && fl_p2 == 1) ? p2 : -1);
      if (f1 >= 0) {
        PCHK(mypos < k);
        c_single = (f1 == hl ? s : s_p2) + (double)S.sval[mypos];
        single_src = f1;
      }
    }
    // local order: score desc; ties repeat (R,0) < blank (R,1) < single (R+c,0)
    double q0 = c_rep, q1 = c_blank, q2 = c_single;
    int k0 = 1, k1 = 0, k2 = 2;
    if (q1 > q0) { double tq = q0; q0 = q1; q1 = tq; int x = k0; k0 = k1; k1 = x; }
    if (q2 > q1) {
      double tq = q1; q1 = q2; q2 = tq; int x = k1; k1 = k2; k2 = x;
      if (q1 > q0) { tq = q0; q0 = q1; q1 = tq; x = k0; k0 = k1; k1 = x; }
    }
    const int kpack = k0 | (k1 << 2) | (k2 << 4);

    // ---------------- append list of this lane's prefix (owner = first entry)
    const double A = isfirst ? (p2 >= 0 ? merge2(s, s_p2, MX) : s) : 0.0;
    uint32_t gv = isfirst ? (fullk & ~(childx | mybit)) : 0u;
    const int gf = gv ? __ffs(gv) - 1 : 0;

    // frame best (appends approximated by A + v; exact on key ties)
    const double hsc0 = fmax(q0, gv ? A + (double)S.sval[gf] : -INFINITY);
    const uint64_t ok64 = (ent && hsc0 > -INFINITY) ? ord64(hsc0) : 0ull;
    const uint32_t mhi = seg_max((uint32_t)(ok64 >> 32), hf);
    const uint32_t mlo = seg_max((uint32_t)(ok64 >> 32) == mhi ? (uint32_t)ok64 : 0u, hf);
    const uint64_t bk = ((uint64_t)mhi << 32) | mlo;
    bool live = act && bk != 0ull;
    if (act && bk == 0ull) { died = true; died_at = i; }  // every extension is -inf (decoder.py:616-620)
    const double best = live ? punord64(bk) : 0.0;
    const double lo_thr = P.threshold_inf ? -DBL_MAX : best - P.beam_threshold;
    const double kbase = best - kR;
    auto keyof = [&](double sc) -> uint32_t {
      if (!(sc > -INFINITY)) return 0u;
      const uint32_t tt = pf2u_sat((sc - kbase) * kScale);
      return tt > 1u ? tt : 1u;
    };
    const long long gG = gv ? pf2ll_floor((A - kbase) * kScale) : 0ll;
    const uint32_t gLow = (gv && A > -INFINITY) ? 1u : 0u;
    PDIV(3);
    // ---------------- k-way merge (decoder.py:651-681)
    // Each lane pops from two queues: its <= 3 special groups (exact fp64,
    // locally sorted) and, as a prefix owner, its append list (head position
    // lp0 = lowest valid top-k rank).  One round = one new beam entry.
    uint32_t sp0 = ent ? keyof(q0) : 0u, sp1 = ent ? keyof(q1) : 0u, sp2 = ent ? keyof(q2) : 0u;
    int spi = 0;  // specials popped
    auto lkey = [&](int p) -> uint32_t {
      const long long tt = gG + S.wp[p];
      return tt < 1ll ? gLow : (tt > 0xffffffffll ? 0xffffffffu : (uint32_t)tt);
    };
    // ---- one-shot selection: each lane's local top-4 of (specials, list),
    // one 64-key register sort per half.  Keys carry (lane, item) in their low
    // 7 bits; adjacent keys within one truncated unit, keys near the floor, or
    // a lane whose next local candidate may still reach the beam fall back to
    // the exact k-way merge below.
    uint32_t lkk[5];
    int lpk = 0;  // first four valid list positions, 5 bits each
    {
      uint32_t g2 = gv;
#pragma unroll
      for (int j = 0; j < 5; j++) {
        const int p = g2 ? __ffs(g2) - 1 : 0;
        lkk[j] = g2 ? lkey(p) : 0u;
        if (j < 4) lpk |= p << (5 * j);
        g2 &= g2 - 1u;
      }
    }
    auto tagk = [&](uint32_t key, int item) -> uint32_t {
      return key ? (((key < 128u ? 128u : key) & ~127u) | (uint32_t)(hl << 3) | (uint32_t)item) : 0u;
    };
    uint32_t xs[4];
    {
      const uint32_t a0 = tagk(sp0, 0), a1 = tagk(sp1, 1), a2 = tagk(sp2, 2);
      xs[0] = max(a0, tagk(lkk[3], 6));
      xs[1] = max(a1, tagk(lkk[2], 5));
      xs[2] = max(a2, tagk(lkk[1], 4));
      xs[3] = tagk(lkk[0], 3);  // (a3 = 0)
      // bitonic sequence -> descending
      uint32_t t0 = max(xs[0], xs[2]), t2 = min(xs[0], xs[2]), t1 = max(xs[1], xs[3]), t3 = min(xs[1], xs[3]);
      xs[0] = max(t0, t1); xs[1] = min(t0, t1); xs[2] = max(t2, t3); xs[3] = min(t2, t3);
    }
    // largest local candidate left out: next special / next list key
    uint32_t U;
    {
      int cA = 0;
#pragma unroll
      for (int r = 0; r < 4; r++) cA += (xs[r] != 0u && (xs[r] & 7u) <= 2u) ? 1 : 0;
      int nz = 0;
#pragma unroll
      for (int r = 0; r < 4; r++) nz += xs[r] != 0u ? 1 : 0;
      const int cB = nz - cA;
      const uint32_t nA = cA == 0 ? sp0 : (cA == 1 ? sp1 : (cA == 2 ? sp2 : 0u));
      const uint32_t nB = cB == 0 ? lkk[0] : (cB == 1 ? lkk[1] : (cB == 2 ? lkk[2] : (cB == 3 ? lkk[3] : lkk[4])));
      U = max(nA, nB);
    }
    sort4_desc(xs, hl);
    int Hn = 0;
    bool fb;
    {
      // rank rho = 4 * hl + r; the beam is ranks < beam
      const uint32_t nx0 = __shfl_down_sync(FULL, xs[0], 1, 16);
      const uint32_t nxt = hl < 15 ? nx0 : 0u;
      const int cl = (beam - 1) >> 2, cr = (beam - 1) & 3;
      const uint32_t kc0 = hshu(xs[0], cl), kc1 = hshu(xs[1], cl), kc2 = hshu(xs[2], cl), kc3 = hshu(xs[3], cl);
      const uint32_t kcut = cr == 0 ? kc0 : (cr == 1 ? kc1 : (cr == 2 ? kc2 : kc3));
      bool bad = U != 0u && (kcut == 0u || (U >> 7) + 1u >= (kcut >> 7));
      int cnt = 0;
#pragma unroll
      for (int r = 0; r < 4; r++) {
        const int rho = 4 * hl + r;
        const uint32_t a = xs[r], b = r < 3 ? xs[r + 1] : nxt;
        if (rho < beam) {
          cnt += a != 0u ? 1 : 0;
          bad |= a != 0u && (a >> 7) <= 1u;                              // near the floor
          bad |= a != 0u && b != 0u && (a >> 7) - (b >> 7) <= 1u;         // not separated
        }
      }
      const bool anybad = seg_any(bad, seg);
      const int hcnt = (int)seg_sum((unsigned)cnt, hf);
      fb = live && anybad;
      Hn = live ? hcnt : 0;
      if (live && !fb) {
#pragma unroll
        for (int r = 0; r < 4; r++) {
          const int rho = 4 * hl + r;
          const uint32_t a = xs[r];
          if (rho < beam && a != 0u) {
            const int id = (int)(a & 7u), wl = (int)((a >> 3) & 15u);
            S.rec[rho] = wl | ((id <= 2 ? id : (0x40 | (id - 3))) << 8);
          }
        }
      }
    }
    PDIV(4);
    if (fb) Hn = 0;
    live = fb;  // the exact k-way merge runs only for halves whose one-shot failed
    if (__any_sync(FULL, fb) && hl == 0 && fb) atomicAdd(&P.dbg[kDbgOneshotFallback], 1ull);
    int lp0 = gv ? __ffs(gv) - 1 : 0;
    uint32_t lk0 = gv ? lkey(lp0) : 0u;
    for (int r = 0; r < beam; r++) {
      if (!__any_sync(FULL, live)) break;
      const uint32_t hd = live ? max(sp0, lk0) : 0u;
      const uint32_t mk = seg_max(hd, hf);
      live = live && mk != 0u;  // no candidate left: the beam is complete
      const bool w_sp = live && sp0 != 0u && mk - sp0 <= kPTol;
      const bool w_lk = live && lk0 != 0u && mk - lk0 <= kPTol;
      const unsigned tw = (__ballot_sync(FULL, w_sp || w_lk) >> (16 * hf)) & 0xffffu;
      const unsigned tb = (__ballot_sync(FULL, w_sp && w_lk) >> (16 * hf)) & 0xffffu;
      // several heads within the key tolerance, or a head near the floor:
      // exact resolution (fp64 score, token sequence, flag; threshold test)
      const bool exact = live && ((tw & (tw - 1u)) != 0u || tb != 0u || mk <= kPTol + 1u);
      bool pop_sp = w_sp, pop_lk = w_lk;
      if (__any_sync(FULL, exact)) {
#pragma unroll
        for (int wq = 0; wq < 2; wq++) {
          const bool in = exact && (wq == 0 ? w_sp : w_lk);
          const int slot = 2 * hl + wq;
          S.tie_i[slot * 4 + 0] = in ? hl : -1;
          if (in && wq == 0) {
            const int kind = (kpack >> (2 * spi)) & 3;
            S.tie_sc[slot] = spi == 0 ? q0 : (spi == 1 ? q1 : q2);
            S.tie_i[slot * 4 + 1] = kind == 2 ? last : -1;
            S.tie_i[slot * 4 + 2] = kind == 0 ? 1 : 0;
            S.tie_i[slot * 4 + 3] = -1;
          }
          if (in && wq == 1) {
            S.tie_sc[slot] = 0.0;
            S.tie_i[slot * 4 + 1] = S.stok[lp0];
            S.tie_i[slot * 4 + 2] = 0;
            S.tie_i[slot * 4 + 3] = lp0;
          }
        }
        S.hs[hl] = h;
        S.hl[hl] = len;
        S.hsc[hl] = s;
        S.hp2[hl] = p2;
        __syncwarp();
        int w = -1;
        if (hl == 0 && exact) {
          atomicAdd(&P.dbg[kDbgTies], 1ull);
          for (int c = 0; c < 32; c++) {
            if (S.tie_i[c * 4] < 0) continue;
            const int pos = S.tie_i[c * 4 + 3];
            if (pos >= 0) {  // exact append-group score: fold of the prefix's entries
              const int f = S.tie_i[c * 4];
              const double v = (double)S.sval[pos];
              double e = S.hsc[f] + v;
              if (S.hp2[f] >= 0) e = merge2(e, S.hsc[S.hp2[f]] + v, MX);
              S.tie_sc[c] = e;
            }
            if (w < 0 || pair_precedes(P, S, u, i, S.tie_sc[c], S.tie_i[c * 4], S.tie_i[c * 4 + 1],
                                       S.tie_i[c * 4 + 2], S.tie_sc[w], S.tie_i[w * 4], S.tie_i[w * 4 + 1],
                                       S.tie_i[w * 4 + 2]))
              w = c;
          }
          const double wsc = S.tie_sc[w];
          if (!(wsc > -INFINITY) || !(wsc >= lo_thr)) w = -1;  // below the threshold: the beam is complete
        }
        w = __shfl_sync(FULL, w, 0, 16);
        __syncwarp();
        if (exact) {
          live = w >= 0;
          pop_sp = live && (w >> 1) == hl && (w & 1) == 0;
          pop_lk = live && (w >> 1) == hl && (w & 1) == 1;
        }
      }
      // pop: the record (lane | item << 8) goes to rank r
      PCHK(!(pop_sp && pop_lk) && spi < 3 && lp0 < 32);
      if (pop_sp || pop_lk) S.rec[r] = hl | ((pop_sp ? spi : (0x80 | lp0)) << 8);
      if (pop_sp) { sp0 = sp1; sp1 = sp2; sp2 = 0u; spi++; }
      if (pop_lk) {
        gv &= gv - 1u;
        lp0 = gv ? __ffs(gv) - 1 : 0;
        lk0 = gv ? lkey(lp0) : 0u;
      }
      if (live) Hn = r + 1;
    }
    __syncwarp();
    if (act && !died && Hn == 0) { died = true; died_at = i; }
    const bool step = act && !died;
    PDIV(5);
    // ---------------- commit (decoder.py:683-744): lane r builds new entry r
    const bool nent = step && hl < Hn;
    const int rec = S.rec[nent ? hl : 0];
    const int wl = nent ? (rec & 0xff) : hl, item = rec >> 8;
    PCHK(!nent || (wl < 16 && ((item & 0xc0) ? true : item < 3)));
    const int wk = hsh(kpack, wl);
    const double w_q0 = hshd(q0, wl), w_q1 = hshd(q1, wl), w_q2 = hshd(q2, wl);
    const int w_src = hsh(rep_src | (single_src << 8), wl);
    const int w_rtok = hsh(rep_tok, wl);
    const uint64_t bh = hsh64(h, wl), bph = hsh64(ph, wl);
    const int blast = hsh(last, wl), blen = hsh(len, wl);
    const double b_s1 = hshd(s, wl), b_s2 = hshd(s_p2, wl);
    const int b_p2 = hsh(p2, wl);
    const int w_lpk = hsh(lpk, wl);
    double nsc;
    int x, src, tok, nfl;
    if (item & 0xc0) {  // append group (R+c,0): exact fold of R's entries in rank order
      const int pos = (item & 0x80) ? (item & 0x1f) : ((w_lpk >> (5 * (item & 3))) & 0x1f);
      const int c = S.stok[pos];
      const double v = (double)S.sval[pos];
      nsc = b_s1 + v;
      if (b_p2 >= 0) nsc = merge2(nsc, b_s2 + v, MX);
      x = c; src = wl; tok = c; nfl = 0;
    } else {
      const int kind = (wk >> (2 * item)) & 3;
      nsc = item == 0 ? w_q0 : (item == 1 ? w_q1 : w_q2);
      if (kind == 0) { x = -1; src = wl; tok = -1; nfl = 1; }                      // blank group
      else if (kind == 1) { x = -1; src = w_src & 0xff; tok = w_rtok; nfl = 0; }  // repeat group
      else { x = blast; src = w_src >> 8; tok = blast; nfl = 0; }                 // last-token append
    }
    __syncwarp();
    // reset the token -> rank map of this frame
#pragma unroll
    for (int p0 = 0; p0 < 32; p0 += 16)
      if (act && p0 + hl < k) S.posmap[S.stok[p0 + hl]] = 0xff;
    if (nent) {
      s = nsc;
      h = x >= 0 ? child_hash(bh, x) : bh;
      ph = x >= 0 ? bh : bph;
      last = x >= 0 ? x : blast;
      len = x >= 0 ? blen + 1 : blen;
      fl = nfl;
      PCHK(src >= 0 && src < 16 && tok >= -1 && tok < V && u >= 0 && u < P.B && i < P.T_max);
      const uint16_t tr = ptrel(src, tok);
      tr16[((size_t)u * P.T_max + i) * beam + hl] = tr;
      S.tring[(i % kChunk) * 16 + hl] = tr;
    }
    PDIV(6);
    if (step) {
      H = Hn;
      if (hl == 0) P.frame_map[(size_t)u * P.T_max + i] = t;
    }
    __syncwarp();
    if (step && (i % kChunk) == kChunk - 1) {
      // trellis checkpoint: ancestor slot at the chunk start for every entry
      if (hl < H) {
        int slot = hl;
#pragma unroll
        for (int tt = kChunk - 1; tt >= 0; --tt) slot = ptrel_src(S.tring[tt * 16 + slot]);
        PCHK(slot >= 0 && slot < 16 && i / kChunk < P.n_chunks);
        P.anc[((size_t)u * P.n_chunks + i / kChunk) * 16 + hl] = (uint8_t)slot;
      }
    }
    __syncwarp();
    PDIV(7);
    if (act) {
      if (step) i++;
      if (!died && t + 2 < len_u) issue(t + 2);
      t++;
    }
  }
}

}  // namespace ctcb
