// Large-beam decode kernel (16 < beam <= 128, V <= 2048, full vocabulary, no
// LM): one 256-thread CTA per utterance.  Same semantics as the generic
// one-warp kernel (ctcb_generic.cu) and the reference (ctcforge
// decoder.py:102-817); every stage of a frame step runs on the whole block:
//
//   * top-k (k = min(2 beam, V-1)): 8-bit radix select with a block histogram,
//     index-ordered compaction, block bitonic sort of (value desc, index asc);
//   * merge structure: prefix groups and parent links through a shared-memory
//     hash table keyed by (prefix hash, length) (decoder.py:595-613);
//   * special groups (blank, repeat, last-token append) exact in fp64;
//   * selection WITHOUT a sequential k-way merge: the append (d, j) -- the j-th
//     valid top-k position of prefix d -- is preceded by its own list's first
//     j positions and, for every prefix d' whose A = logaddexp of its entries
//     exceeds A_d by a margin, by >= j candidates of d' (its appends at the
//     same or better positions, or the repeat groups that replace excluded
//     ones; at most one position per prefix, its last token, is lost).  So
//     (d, j) can enter the beam only if (d_eff + 1) j < beam, d_eff = number of
//     such prefixes.  Those appends plus all specials get 64-bit keys (32-bit
//     fixed-point score | candidate id) and one block sort ranks them; runs of
//     keys within the rounding tolerance around ranks [0, beam] are re-ordered
//     exactly (fp64 fold, then token sequence, then flag: decoder.py:651-681)
//     and the beam threshold is applied on exact scores (:615-626).
#include <cfloat>
#include <cmath>

#include "ctcb_common.cuh"
#include "ctcb_internal.h"
#include <cstdio>
#ifdef CTCB_BLOCK_CHECK
#define BCHK(c)                                                                                    \
  do {                                                                                             \
    if (!(c)) { printf("ctcb_block check failed: %s (line %d, block %d, thread %d)\n", #c, __LINE__, blockIdx.x, threadIdx.x); __trap(); } \
  } while (0)
#else
#define BCHK(c) do { } while (0)
#endif

namespace ctcb {

namespace {

constexpr int NT = 256;          // threads per CTA (one utterance)
constexpr int kTolB = 2;         // rank-key tolerance (fixed-point units)
constexpr uint32_t kSpecial = 0x80000000u;

// Dynamic shared memory of the block kernel: one fixed layout for the largest
// supported beam / vocabulary, so every array base below is a link-time
// constant (an immediate offset in the shared-memory instructions) instead of
// a pointer held in registers or spilled to the stack.
extern __shared__ __align__(128) uint8_t blk_smem[];

struct Blk {
  static constexpr BlockLayout L = make_block_layout(kBlockMaxBeam, 256, kBlockMaxV, kBlockMaxV * 4);
  static constexpr int kw = L.kw, kpad = L.kpad, ts = L.ts, ncap = L.ncap;
  static constexpr size_t row_bytes = kBlockMaxV * 4;
  const Params* P;
  int tid, u, steps_done;
  int par;  // which half of the double-buffered entry state is current
  __device__ uint8_t* rows() const { return (uint8_t*)(blk_smem + L.rows); }
  __device__ uint64_t* mbar() const { return (uint64_t*)(blk_smem + L.mbar); }
  __device__ double* lA() const { return (double*)(blk_smem + L.lA); }
  __device__ double* spsc() const { return (double*)(blk_smem + L.spsc); }
  __device__ uint64_t* skey() const { return (uint64_t*)(blk_smem + L.skey); }
  __device__ uint64_t* ckey() const { return (uint64_t*)(blk_smem + L.ckey); }
  __device__ uint64_t* htk() const { return (uint64_t*)(blk_smem + L.htk); }
  __device__ uint64_t* tc_h() const { return (uint64_t*)(blk_smem + L.tc_h); }
  __device__ int* htf() const { return (int*)(blk_smem + L.htf); }
  __device__ int* hslot() const { return (int*)(blk_smem + L.hslot); }
  __device__ int* first() const { return (int*)(blk_smem + L.first); }
  __device__ int* dpi() const { return (int*)(blk_smem + L.dpi); }
  __device__ int* pd() const { return (int*)(blk_smem + L.pd); }
  __device__ int* e1() const { return (int*)(blk_smem + L.e1); }
  __device__ int* e2() const { return (int*)(blk_smem + L.e2); }
  __device__ int* qoff() const { return (int*)(blk_smem + L.qoff); }
  __device__ int* spbase() const { return (int*)(blk_smem + L.spbase); }
  __device__ int* spx() const { return (int*)(blk_smem + L.spx); }
  __device__ int* spflag() const { return (int*)(blk_smem + L.spflag); }
  __device__ int* spsrc() const { return (int*)(blk_smem + L.spsrc); }
  __device__ int* sptok() const { return (int*)(blk_smem + L.sptok); }
  __device__ int* misc() const { return (int*)(blk_smem + L.misc); }
  __device__ int8_t* tc_r() const { return (int8_t*)(blk_smem + L.tc_r); }
  __device__ int* rec() const { return (int*)(blk_smem + L.rec); }
  __device__ int* ord() const { return (int*)(blk_smem + L.ord); }
  __device__ int* runbuf() const { return (int*)(blk_smem + L.runbuf); }
  __device__ double* runsc() const { return (double*)(blk_smem + L.runsc); }
  __device__ uint32_t* ntrel() const { return (uint32_t*)(blk_smem + L.ntrel); }
  __device__ uint32_t* excl() const { return (uint32_t*)(blk_smem + L.excl); }
  __device__ uint32_t* hist() const { return (uint32_t*)(blk_smem + L.hist); }
  __device__ uint32_t* crec() const { return (uint32_t*)(blk_smem + L.crec); }
  __device__ float* sval() const { return (float*)(blk_smem + L.sval); }
  __device__ int* stok() const { return (int*)(blk_smem + L.stok); }
  __device__ uint16_t* pos() const { return (uint16_t*)(blk_smem + L.pos); }
  __device__ double* cs() const { return (double*)(blk_smem + (par ? L.ns : L.cs)); }
  __device__ double* ns() const { return (double*)(blk_smem + (par ? L.cs : L.ns)); }
  __device__ uint64_t* ch() const { return (uint64_t*)(blk_smem + (par ? L.nh : L.ch)); }
  __device__ uint64_t* nh() const { return (uint64_t*)(blk_smem + (par ? L.ch : L.nh)); }
  __device__ uint64_t* cph() const { return (uint64_t*)(blk_smem + (par ? L.nph : L.cph)); }
  __device__ uint64_t* nph() const { return (uint64_t*)(blk_smem + (par ? L.cph : L.nph)); }
  __device__ int* cl() const { return (int*)(blk_smem + (par ? L.nl : L.cl)); }
  __device__ int* nl() const { return (int*)(blk_smem + (par ? L.cl : L.nl)); }
  __device__ int* cn() const { return (int*)(blk_smem + (par ? L.nn : L.cn)); }
  __device__ int* nn() const { return (int*)(blk_smem + (par ? L.cn : L.nn)); }
  __device__ int* cf() const { return (int*)(blk_smem + (par ? L.nf : L.cf)); }
  __device__ int* nf() const { return (int*)(blk_smem + (par ? L.cf : L.nf)); }

  __device__ void swap_state() { par ^= 1; }
};

// ------------------------------------------------------------------ block helpers
__device__ __forceinline__ void bsync() { __syncthreads(); }

// Block bitonic sort of n (power of two, >= 2) u64 keys, descending.
__device__ __forceinline__ void block_sort_desc(uint64_t* key, int n, int tid) {
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = tid; t < (n >> 1); t += NT) {
        const int i = ((t & ~(stride - 1)) << 1) | (t & (stride - 1));
        const int j = i + stride;
        const uint64_t a = key[i], b = key[j];
        const bool desc = (i & size) == 0;
        if (desc ? (a < b) : (a > b)) { key[i] = b; key[j] = a; }
      }
      bsync();
    }
}

// One-warp bitonic sort of 32 R u64 keys held in registers, descending; key
// i = lane R + r.  Strides >= R exchange across lanes (two shuffles per key),
// smaller ones inside a lane: no barriers, unlike block_sort_desc.
__device__ __forceinline__ uint64_t shfl_xor64(uint64_t x, int m) {
  const uint32_t lo = __shfl_xor_sync(FULL, (uint32_t)x, m), hi = __shfl_xor_sync(FULL, (uint32_t)(x >> 32), m);
  return ((uint64_t)hi << 32) | lo;
}
template <int R>
__device__ __forceinline__ void warp_sort_desc(uint64_t (&k)[R], int lane) {
  constexpr int N = 32 * R;
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= R) {
        const int lm = stride / R;
        const bool lower = (lane & lm) == 0;
#pragma unroll
        for (int r = 0; r < R; r++) {
          const uint64_t o = shfl_xor64(k[r], lm);
          const bool desc = ((lane * R + r) & size) == 0;
          k[r] = (lower == desc) ? (k[r] > o ? k[r] : o) : (k[r] < o ? k[r] : o);
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; r++) {
          const int p = r ^ stride;
          if (p > r) {
            const bool desc = ((lane * R + r) & size) == 0;
            const uint64_t a = k[r], b = k[p];
            if (desc ? a < b : a > b) { k[r] = b; k[p] = a; }
          }
        }
      }
    }
  }
}
// Block sort of n <= 512 keys (nonzero keys distinct; zeros are padding and
// are dropped): each warp sorts a 64-key chunk in registers, then every key's
// rank is its chunk position plus, per other chunk, the number of larger keys
// (binary search).  dst[0 .. #nonzero) receives the nonzero keys descending.
// Two barriers instead of the 45 of a block bitonic network.  tmp: 512 keys.
__device__ __forceinline__ void block_sort512(const uint64_t* src, int n, uint64_t* tmp, uint64_t* dst, int tid) {
  const int wid = tid >> 5, lane = tid & 31;
  const int nch = (n + 63) >> 6;
  uint64_t k[2] = {0ull, 0ull};
  if (wid < nch) {
#pragma unroll
    for (int r = 0; r < 2; r++) {
      const int i = wid * 64 + r * 32 + lane;
      k[r] = i < n ? src[i] : 0ull;
    }
    warp_sort_desc<2>(k, lane);
#pragma unroll
    for (int r = 0; r < 2; r++) tmp[wid * 64 + lane * 2 + r] = k[r];
  }
  __syncthreads();
  if (wid < nch) {
#pragma unroll
    for (int r = 0; r < 2; r++) {
      const uint64_t key = k[r];
      if (key == 0ull) continue;
      int rank = lane * 2 + r;
#pragma unroll
      for (int c = 0; c < 8; c++) {
        if (c == wid || c >= nch) continue;
        const uint64_t* ch = tmp + c * 64;
        int lo = 0;  // number of keys > key in the descending chunk
#pragma unroll
        for (int step = 32; step > 0; step >>= 1)
          if (ch[lo + step - 1] > key) lo += step;
        lo += ch[lo] > key ? 1 : 0;  // lo <= 63 here; all 64 larger
        rank += lo;
      }
      dst[rank] = key;
    }
  }
  __syncthreads();
}

// Exclusive block scan of one int per thread (NT = 256).
// kTail = false: the caller guarantees a barrier before tmp is written again.
template <bool kTail = true>
__device__ __forceinline__ int block_excl_scan(int v, int tid, int* tmp, int* total) {
  const int lane = tid & 31, wid = tid >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) tmp[wid] = incl;
  bsync();
  if (wid == 0) {
    const int t = lane < NT / 32 ? tmp[lane] : 0;
    int x = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane < NT / 32) tmp[lane] = x - t;
    if (lane == NT / 32 - 1) tmp[NT / 32] = x;
  }
  bsync();
  const int r = tmp[wid] + incl - v;
  *total = tmp[NT / 32];
  if (kTail) bsync();  // tmp reusable at once
  return r;
}

// ------------------------------------------------------------------ token sequences (single-thread slow path)
// Token-sequence order of two entries (trellis_seq_cmp: lockstep walk back to
// the merge point of their trellis paths).
__device__ __forceinline__ int bseq_cmp_full(const Blk& w, int ea, int xa, int eb, int xb, bool* strict) {
  const Params& P = *w.P;
  int* A = P.seqbuf + (size_t)w.u * 3 * (P.T_max + 1);
  const uint32_t* tr = P.trellis + (size_t)w.u * P.T_max * P.beam;
  auto rec = [&](int i, int slot) {
    const uint32_t r = tr[(size_t)i * P.beam + slot];
    return make_int2(trel_tok(r), trel_src(r));
  };
  return trellis_seq_cmp(rec, w.steps_done, ea, xa, eb, xb, A, A + P.T_max + 1, strict, P.dbg);
}
// Sequence-order cache: direct-mapped on the unordered pair of sequence
// hashes, holding the order of the lower hash's sequence against the other.
// Results hold across utterances (a hash names one token sequence).
__device__ __forceinline__ int btc_slot(uint64_t lo, uint64_t hi) {
  return (int)(mix64(lo * 0x9e3779b97f4a7c15ull ^ hi) & (uint64_t)(kBlockTieCache - 1));
}
__device__ __forceinline__ int btc_lookup(const Blk& w, uint64_t ha, uint64_t hb) {
  const uint64_t lo = ha < hb ? ha : hb, hi = ha < hb ? hb : ha;
  const int i = btc_slot(lo, hi);
  if (w.tc_h()[2 * i] != lo || w.tc_h()[2 * i + 1] != hi) return 0;
  const int r = w.tc_r()[i];
  return ha < hb ? r : -r;
}
__device__ __forceinline__ void btc_insert(const Blk& w, uint64_t ha, uint64_t hb, int r) {
  const uint64_t lo = ha < hb ? ha : hb, hi = ha < hb ? hb : ha;
  const int i = btc_slot(lo, hi);
  w.tc_h()[2 * i] = lo;
  w.tc_h()[2 * i + 1] = hi;
  w.tc_r()[i] = (int8_t)(ha < hb ? r : -r);
}
// Python tuple order of seq(ea)+[xa] vs seq(eb)+[xb] (x < 0: no extra token).
__device__ __forceinline__ int bseq_cmp(const Blk& w, int ea, int xa, int eb, int xb) {
  const uint64_t hba = w.ch()[ea], hbb = w.ch()[eb];
  const int lba = w.cn()[ea], lbb = w.cn()[eb];
  if (hba == hbb && lba == lbb) {
    if (xa == xb) return 0;
    return xa < xb ? -1 : 1;
  }
  const uint64_t ha = xa >= 0 ? child_hash(hba, xa) : hba, hb = xb >= 0 ? child_hash(hbb, xb) : hbb;
  const int la = lba + (xa >= 0), lb = lbb + (xb >= 0);
  if (ha == hb && la == lb) return 0;
  int r = btc_lookup(w, hba, hbb);
  if (r) {
    btc_insert(w, ha, hb, r);
    return r;
  }
  r = btc_lookup(w, ha, hb);
  if (r) return r;
  bool strict = false;
  r = bseq_cmp_full(w, ea, -1, eb, -1, &strict);
  if (strict) {
    btc_insert(w, hba, hbb, r);
    btc_insert(w, ha, hb, r);
    return r;
  }
  r = bseq_cmp_full(w, ea, xa, eb, xb, &strict);
  if (strict) btc_insert(w, ha, hb, r);
  return r;
}
struct BDesc { double sc; int base, x, flag; };
// out of line: the exact tie path is rare and would otherwise be inlined at
// every call site
__device__ __noinline__ bool bprecedes(const Blk w, const BDesc a, const BDesc b) {
  if (a.sc != b.sc) return a.sc > b.sc;
  atomicAdd(&w.P->dbg[kDbgExactTies], 1ull);
  const int c = bseq_cmp(w, a.base, a.x, b.base, b.x);
  if (c) return c < 0;
  return a.flag < b.flag;
}

// ------------------------------------------------------------------ top-k
// S = the k best non-blank tokens of `row` by (value desc, index asc), sorted
// into sval / stok; pos[token] = rank in S.
__device__ __forceinline__ void btopk(Blk& w, const float* row) {
  const Params& P = *w.P;
  const int V = P.V, blank = P.blank, k = P.k, tid = w.tid;
  if (V <= 512) {
    // whole row: block sort by (value desc, index asc); the first k are S
    // (same order as select + compaction + sort below)
    for (int c = tid; c < V; c += NT)
      w.skey()[c] = c != blank ? (((uint64_t)ord32(row[c]) << 32) | (uint64_t)(0xffffffffu - (uint32_t)c)) : 0ull;
    bsync();
    block_sort512(w.skey(), V, w.ckey(), w.ckey() + 512, tid);
    for (int j = tid; j < k; j += NT) {
      const int c = (int)(0xffffffffu - (uint32_t)(w.ckey()[512 + j] & 0xffffffffu));
      w.stok()[j] = c;
      w.sval()[j] = row[c];
      w.pos()[c] = (uint16_t)j;
    }
    bsync();
    return;
  }
  uint32_t kth = 0;
  int need = V;
  if (k < V - 1) {
    uint32_t prefix = 0, pmask = 0;
    need = k;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int b = tid; b < 256; b += NT) w.hist()[b] = 0;
      bsync();
      for (int c = tid; c < V; c += NT) {
        if (c == blank) continue;
        const uint32_t key = ord32(row[c]);
        if ((key & pmask) == prefix) atomicAdd(&w.hist()[(key >> shift) & 255u], 1u);
      }
      bsync();
      if (tid < 32) {  // digit holding the need-th largest key
        const int lane = tid;
        uint32_t h[8], s = 0;
#pragma unroll
        for (int q = 0; q < 8; q++) { h[q] = w.hist()[lane * 8 + q]; s += h[q]; }
        uint32_t incl = s;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t v = __shfl_down_sync(FULL, incl, off);
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
        const unsigned bal = __ballot_sync(FULL, found >= 0);
        const int src = __ffs(bal) - 1;
        const int digit = __shfl_sync(FULL, found, src);
        cgt = __shfl_sync(FULL, cgt, src);
        if (lane == 0) { w.misc()[4] = digit; w.misc()[5] = (int)cgt; }
      }
      bsync();
      need -= w.misc()[5];
      prefix |= (uint32_t)w.misc()[4] << shift;
      pmask |= 0xffu << shift;
      bsync();
    }
    kth = prefix;
  }
  // ordered compaction: keys > kth, then the `need` lowest-index keys == kth;
  // thread t owns tokens [t*cpt, (t+1)*cpt)
  const int cpt = (V + NT - 1) / NT;
  int ngt = 0, neq = 0;
  for (int q = 0; q < cpt; q++) {
    const int c = tid * cpt + q;
    if (c >= V || c == blank) continue;
    const uint32_t key = ord32(row[c]);
    ngt += key > kth;
    neq += key == kth;
  }
  int tot_eq = 0, tot = 0;
  const int eq_before = block_excl_scan(neq, tid, w.qoff(), &tot_eq);
  int eq_take = need - eq_before;
  eq_take = eq_take < 0 ? 0 : (eq_take > neq ? neq : eq_take);
  const int off = block_excl_scan<false>(ngt + eq_take, tid, w.qoff(), &tot);
  int o = off, taken = 0;
  for (int q = 0; q < cpt; q++) {
    const int c = tid * cpt + q;
    if (c >= V || c == blank) continue;
    const uint32_t key = ord32(row[c]);
    const bool acc = key > kth || (key == kth && taken++ < eq_take);
    if (acc) w.skey()[o++] = ((uint64_t)key << 32) | (uint64_t)(0xffffffffu - (uint32_t)c);
  }
  bsync();
  block_sort512(w.skey(), tot, w.ckey(), w.ckey() + 512, tid);  // tot = k <= 256
  for (int j = tid; j < k; j += NT) {
    const int c = (int)(0xffffffffu - (uint32_t)(w.ckey()[512 + j] & 0xffffffffu));
    w.stok()[j] = c;
    w.sval()[j] = row[c];
    w.pos()[c] = (uint16_t)j;
  }
  bsync();
}

__device__ __forceinline__ bool bexcl(const Blk& w, int d, int j) {
  return (w.excl()[d * w.kw + (j >> 5)] >> (j & 31)) & 1u;
}
// j-th valid (non-excluded) top-k position of list d, or k
__device__ __forceinline__ int jth_valid(const Blk& w, int d, int j, int k) {
  const uint32_t* ex = w.excl() + d * w.kw;
  for (int wd = 0; wd < w.kw; wd++) {
    const int lo = wd * 32;
    if (lo >= k) break;
    const int nbits = k - lo < 32 ? k - lo : 32;
    const uint32_t live = ~ex[wd] & (nbits == 32 ? 0xffffffffu : ((1u << nbits) - 1u));
    const int c = __popc(live);
    if (j < c) {
      uint32_t m = live;  // position of its (j+1)-th set bit: binary search on popcounts
      int p = 0;
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) {
        const int h = __popc(m & ((1u << s) - 1u));
        if (j >= h) { j -= h; m >>= s; p += s; }
      }
      return lo + p;
    }
    j -= c;
  }
  return k;
}
__device__ __forceinline__ double bgen_score(const Blk& w, int d, int j) {
  const double v = (double)w.sval()[j];
  const int a = w.e1()[d], b = w.e2()[d];
  double s = w.cs()[a] + v;
  if (b >= 0) s = merge2_exact(s, w.cs()[b] + v, w.P->merge_max != 0);
  return s;
}
__device__ __forceinline__ BDesc cand_desc(const Blk& w, uint32_t rec) {
  if (rec & kSpecial) {
    const int s = (int)(rec & ~kSpecial);
    return BDesc{w.spsc()[s], w.spbase()[s], w.spx()[s], w.spflag()[s]};
  }
  const int d = (int)(rec >> 12), j = (int)(rec & 0xfff);
  return BDesc{bgen_score(w, d, j), w.e1()[d], w.stok()[j], 0};
}

// Descriptor of candidate record `rec` with its exact score already known.
__device__ __forceinline__ BDesc desc_sc(const Blk& w, uint32_t rec, double sc) {
  if (rec & kSpecial) {
    const int s = (int)(rec & ~kSpecial);
    return BDesc{sc, w.spbase()[s], w.spx()[s], w.spflag()[s]};
  }
  return BDesc{sc, w.e1()[(int)(rec >> 12)], w.stok()[(int)(rec & 0xfff)], 0};
}

// One frame step; returns the new beam size (0: beam died).
__device__ __forceinline__ int bstep(Blk& w, const float* row, int H) {
  const Params& P = *w.P;
  const int tid = w.tid, beam = P.beam, k = P.k;
  const bool MX = P.merge_max != 0;
  const double eb = (double)row[P.blank];

  // -- prefix groups (flag 0 / flag 1 entries of one token sequence)
  const int TS = w.ts;
  for (int i = tid; i < TS; i += NT) { w.htk()[i] = 0ull; w.htf()[i] = 0x7fffffff; }
  if (tid == 0) { w.misc()[0] = 0; w.misc()[1] = 0; }
  bsync();
  for (int e = tid; e < H; e += NT) {
    const uint64_t key = (w.ch()[e] ^ ((uint64_t)w.cn()[e] * 0x9e3779b97f4a7c15ull)) | 1ull;
    uint32_t i = (uint32_t)mix64(key) & (uint32_t)(TS - 1);
    for (;;) {
      const unsigned long long prev = atomicCAS((unsigned long long*)&w.htk()[i], 0ull, (unsigned long long)key);
      if (prev == 0ull || prev == key) break;
      i = (i + 1) & (uint32_t)(TS - 1);
    }
    atomicMin(&w.htf()[i], e);
    w.hslot()[e] = (int)i;
  }
  bsync();
  for (int e = tid; e < H; e += NT) w.first()[e] = w.htf()[w.hslot()[e]];
  bsync();
  // distinct prefixes numbered in entry order (d = rank of its first entry)
  int nD = 0;
  {
    const bool isf = tid < H && w.first()[tid] == tid;
    int tot = 0;
    const int d = block_excl_scan<false>(isf ? 1 : 0, tid, w.qoff(), &tot);
    nD = tot;
    if (isf) { w.dpi()[tid] = d; w.e1()[d] = tid; w.e2()[d] = -1; }
  }
  bsync();
  for (int e = tid; e < H; e += NT)
    if (w.first()[e] != e) { const int d = w.dpi()[w.first()[e]]; w.dpi()[e] = d; w.e2()[d] = e; }
  for (int i = tid; i < nD * w.kw; i += NT) w.excl()[i] = 0u;
  bsync();
  // -- parent links of flag-0 entries; children exclude their token from the
  //    parent's list (they become repeat groups)
  for (int e = tid; e < H; e += NT) {
    int p = -1;
    if (w.cf()[e] == 0) {
      const uint64_t key = (w.cph()[e] ^ ((uint64_t)(w.cn()[e] - 1) * 0x9e3779b97f4a7c15ull)) | 1ull;
      uint32_t i = (uint32_t)mix64(key) & (uint32_t)(TS - 1);
      for (;;) {
        const uint64_t k2 = w.htk()[i];
        if (k2 == 0ull) break;
        if (k2 == key) { p = w.dpi()[w.htf()[i]]; break; }
        i = (i + 1) & (uint32_t)(TS - 1);
      }
      if (p >= 0) {
        const int j = w.pos()[w.cl()[e]];
        if (j != 0xffff) atomicOr(&w.excl()[p * w.kw + (j >> 5)], 1u << (j & 31));
      }
    }
    w.pd()[e] = p;
  }
  bsync();
  // -- specials: blank groups, last-token appends (per prefix), repeat groups (per flag-0 entry)
  for (int d = tid; d < nD; d += NT) {
    const int a = w.e1()[d], b = w.e2()[d];
    double sc = w.cs()[a] + eb;
    if (b >= 0) sc = merge2_exact(sc, w.cs()[b] + eb, MX);
    int s = atomicAdd(&w.misc()[0], 1);
    BCHK(s < 3 * beam);
    w.spsc()[s] = sc; w.spbase()[s] = a; w.spx()[s] = -1; w.spflag()[s] = 1; w.spsrc()[s] = a; w.sptok()[s] = -1;
    const int c = w.cl()[a];
    if (c >= 0) {
      const int j = w.pos()[c];
      if (j != 0xffff && !bexcl(w, d, j)) {
        const int f = w.cf()[a] == 1 ? a : ((b >= 0 && w.cf()[b] == 1) ? b : -1);
        if (f >= 0) {
          s = atomicAdd(&w.misc()[0], 1);
          w.spsc()[s] = w.cs()[f] + (double)w.sval()[j];
          w.spbase()[s] = a; w.spx()[s] = c; w.spflag()[s] = 0; w.spsrc()[s] = f; w.sptok()[s] = c;
        }
        atomicOr(&w.excl()[d * w.kw + (j >> 5)], 1u << (j & 31));
      }
    }
    // A = logaddexp of the prefix's entries (list base)
    w.lA()[d] = b >= 0 ? merge2_exact(w.cs()[a], w.cs()[b], MX) : w.cs()[a];
  }
  for (int e = tid; e < H; e += NT) {
    if (w.cf()[e] != 0) continue;
    const int c = w.cl()[e];
    BCHK(c >= 0 && c < P.V);
    const double ec = (double)row[c];
    double sc = w.cs()[e] + ec, best = sc;  // repeat candidate first (decoder.py:522-530)
    int src = e, tok = -1;
    const int p = w.pd()[e];
    if (p >= 0) {
      const int srcs[2] = {w.e1()[p], w.e2()[p]};
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int h = srcs[q];
        if (h < 0 || (w.cf()[h] == 0 && w.cl()[h] == c)) continue;  // blocked repeat (decoder.py:495)
        const double x = w.cs()[h] + ec;
        sc = merge2_exact(sc, x, MX);
        if (x > best) { best = x; src = h; tok = c; }
      }
    }
    const int s = atomicAdd(&w.misc()[0], 1);
    BCHK(s < 3 * beam);
    w.spsc()[s] = sc; w.spbase()[s] = e; w.spx()[s] = -1; w.spflag()[s] = 0; w.spsrc()[s] = src; w.sptok()[s] = tok;
  }
  bsync();
  const int nS = w.misc()[0];

  // -- append quotas: d_eff = prefixes whose A exceeds A_d by a margin;
  //    (d, j) can reach the beam only if (d_eff + 1) j < beam
  int q = 0;
  if (tid < nD) {
    const double Ad = w.lA()[tid];
    int deff = 0;
    if (Ad > -INFINITY) {
      const double thr = Ad + 1e-9 * (1.0 + fabs(Ad));
      for (int d2 = 0; d2 < nD; d2++) deff += w.lA()[d2] > thr;
      q = (beam - 1) / (deff + 1) + 1;
    }
  }
  int nA = 0;
  const int qo = block_excl_scan<false>(q, tid, w.rec(), &nA);
  if (tid < nD) { w.qoff()[tid] = qo; }
  if (tid == 0) w.qoff()[nD] = nA;
  bsync();
  const int N = nS + nA;
  int ncap = 2;
  while (ncap < N) ncap <<= 1;

  // -- frame best on approximate scores (specials exact, list heads A + v)
  double lb = -INFINITY;
  for (int s = tid; s < nS; s += NT) lb = fmax(lb, w.spsc()[s]);
  for (int d = tid; d < nD; d += NT) {
    const int j0 = jth_valid(w, d, 0, k);
    if (j0 < k) lb = fmax(lb, w.lA()[d] + (double)w.sval()[j0]);
  }
  {
    const uint64_t o64 = lb > -INFINITY ? ord64(lb) : 0ull;
    const uint32_t hi = __reduce_max_sync(FULL, (uint32_t)(o64 >> 32));
    const uint32_t lo = __reduce_max_sync(FULL, (uint32_t)(o64 >> 32) == hi ? (uint32_t)o64 : 0u);
    if ((tid & 31) == 0) w.skey()[tid >> 5] = ((uint64_t)hi << 32) | lo;  // skey: free after the top-k
  }
  bsync();
  uint64_t bk = 0ull;
  for (int i = 0; i < NT / 32; i++) bk = bk > w.skey()[i] ? bk : w.skey()[i];
  if (bk == 0ull) return 0;  // every extension is -inf (decoder.py:616-620)

  // more candidates than the key buffer holds (exactly tied prefixes defeat
  // the quotas): exact serial selection below; misc[10] is also raised by an
  // absurdly long tie run and read only after the barriers that follow
  const bool big = ncap > w.ncap;
  if (tid == 0) w.misc()[10] = big ? 1 : 0;
  if (!big) {
    const double best_a = __longlong_as_double((long long)((bk >> 63) ? (bk & 0x7fffffffffffffffull) : ~bk));
    const double kR = P.threshold_inf ? 1048576.0 : fmin(P.beam_threshold, 1048576.0);
    const double kScale = 4294967294.0 / kR, koff = -(best_a - kR) * kScale;
    auto keyof = [&](double sc) -> uint32_t {
      if (!(sc > -INFINITY)) return 0u;
      const double z = fmin(fmax(fma(sc, kScale, koff), 0.0), 4294967294.0);
      return 1u + (uint32_t)z;
    };
    // -- candidate keys: (fixed-point score | candidate id); id -> record in crec
    for (int c = tid; c < ncap; c += NT) {
      uint64_t key = 0ull;
      if (c < nS) {
        const uint32_t kk = keyof(w.spsc()[c]);
        w.crec()[c] = kSpecial | (uint32_t)c;
        key = kk ? (((uint64_t)kk << 32) | (uint64_t)(0xffffffffu - (uint32_t)c)) : 0ull;
      } else if (c < N) {
        const int g = c - nS;
        int lo = 0, hi = nD - 1;  // list of append slot g: last d with qoff[d] <= g
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (w.qoff()[mid] <= g) lo = mid; else hi = mid - 1;
        }
        const int d = lo, j = g - w.qoff()[d];
        BCHK(d >= 0 && d < nD && j >= 0);
        const int p = jth_valid(w, d, j, k);
        if (p < k && w.lA()[d] > -INFINITY) {
          const uint32_t kk = keyof(w.lA()[d] + (double)w.sval()[p]);
          w.crec()[c] = ((uint32_t)d << 12) | (uint32_t)p;
          key = kk ? (((uint64_t)kk << 32) | (uint64_t)(0xffffffffu - (uint32_t)c)) : 0ull;
        }
      }
      w.ckey()[c] = key;
    }
    bsync();
    // -- survivors: keys within a margin of the beam-th, exactly ranked.
    //    Warps sort strided 64-key chunks of ckey in registers (chunk c =
    //    slots c, c + nch, ...; at most 4 per warp).  Each chunk's q-th key,
    //    q = ceil((beam + 1) / nch), bounds the (beam + 1)-th key from below;
    //    keys under that bound minus the margin cannot reach the beam or its
    //    tie runs.  The survivors (a prefix of every sorted chunk) are
    //    compacted and ranked by counting: four barriers in all.
    const int need = beam + 1;
    const int nch = (ncap + 63) >> 6;
    const int q = (need + nch - 1) / nch;
    const int lane = tid & 31, wid = tid >> 5;
    uint64_t kk[4][2];
#pragma unroll
    for (int h = 0; h < 4; h++) {
      const int c = wid + h * (NT / 32);
      kk[h][0] = kk[h][1] = 0ull;
      if (c < nch) {
#pragma unroll
        for (int r = 0; r < 2; r++) {
          const int i = c + nch * (r * 32 + lane);
          kk[h][r] = i < ncap ? w.ckey()[i] : 0ull;
        }
        const int nz = __popc(__ballot_sync(FULL, kk[h][0] != 0ull)) + __popc(__ballot_sync(FULL, kk[h][1] != 0ull));
        warp_sort_desc<2>(kk[h], lane);
#pragma unroll
        for (int r = 0; r < 2; r++)
          if (lane * 2 + r == q - 1) w.hist()[32 + c] = (uint32_t)(kk[h][r] >> 32);
        if (lane == 0) w.hist()[c] = (uint32_t)nz;
      }
    }
    bsync();
    uint32_t tau = 0xffffffffu;
    bool fb = false;
    for (int c = 0; c < nch; c++) {
      if ((int)w.hist()[c] < q) fb = true;
      tau = min(tau, w.hist()[32 + c]);
    }
    const uint32_t lim = fb ? 1u : (tau > 64u ? tau - 64u : 1u);
    auto surv = [&](uint64_t x) { return x != 0ull && (uint32_t)(x >> 32) >= lim; };
#pragma unroll
    for (int h = 0; h < 4; h++) {
      const int c = wid + h * (NT / 32);
      if (c < nch) {
        const int sc = __popc(__ballot_sync(FULL, surv(kk[h][0]))) + __popc(__ballot_sync(FULL, surv(kk[h][1])));
        if (lane == 0) w.hist()[64 + c] = (uint32_t)sc;
      }
    }
    bsync();
    uint64_t* dst = (uint64_t*)w.ord();  // [0, 512): ranked survivors, [512, 1024): compacted
    int nsurv = 0;
    for (int c = 0; c < nch; c++) nsurv += (int)w.hist()[64 + c];
    uint64_t* sk = dst;
    int nsk = nsurv;
    bool trunc = lim > 1u;
    if (nsurv <= 512) {
#pragma unroll
      for (int h = 0; h < 4; h++) {
        const int c = wid + h * (NT / 32);
        if (c < nch) {
          int off = 0;
          for (int c2 = 0; c2 < c; c2++) off += (int)w.hist()[64 + c2];
#pragma unroll
          for (int r = 0; r < 2; r++)
            if (surv(kk[h][r])) dst[512 + off + lane * 2 + r] = kk[h][r];
        }
      }
      bsync();
      for (int t = tid; t < nsurv; t += NT) {
        const uint64_t x = dst[512 + t];
        int rank = 0;
        int i = 0;
        for (; i + 1 < nsurv; i += 2) {
          const ulonglong2 y = *(const ulonglong2*)&dst[512 + i];  // 16-B aligned pair
          rank += (y.x > x) + (y.y > x);
        }
        if (i < nsurv) rank += dst[512 + i] > x;
        dst[rank] = x;
      }
      bsync();
    } else {  // (almost) every candidate survives: full sort
#pragma unroll
      for (int h = 0; h < 4; h++) {
        const int c = wid + h * (NT / 32);
        if (c < nch)
#pragma unroll
          for (int r = 0; r < 2; r++) {
            const int i = c + nch * (lane * 2 + r);
            if (i < ncap) w.ckey()[i] = kk[h][r];
          }
      }
      bsync();
      block_sort_desc(w.ckey(), ncap, tid);
      sk = w.ckey();
      nsk = ncap;
      trunc = false;
    }
    if (tid == 0) {  // selection statistics (debug counters)
      atomicAdd(&P.dbg[kDbgRadix], (unsigned long long)N);
      atomicAdd(&P.dbg[kDbgTopkFix], (unsigned long long)nsurv);
    }
    // -- exact order where keys are within the tolerance: runs of adjacent
    //    keys (differences <= kTolB) in ranks [0, beam] are re-sorted on exact
    //    descriptors (fp64 fold, token sequence, flag)
    for (int attempt = 0; attempt < 2; attempt++) {
      bool tie = false;
      for (int r = tid; r < beam && r + 1 < nsk; r += NT) {
        const uint64_t x = sk[r], y = sk[r + 1];
        tie |= x != 0ull && y != 0ull && (uint32_t)(x >> 32) - (uint32_t)(y >> 32) <= (uint32_t)kTolB;
      }
      const int anytie = __syncthreads_or(tie ? 1 : 0);
      for (int r = tid; r < beam; r += NT) {
        const uint64_t x = r < nsk ? sk[r] : 0ull;
        w.rec()[r] = x ? (int)w.crec()[0xffffffffu - (uint32_t)(x & 0xffffffffu)] : -1;
      }
      if (tid == 0) w.misc()[9] = 0;
      bsync();
      if (anytie) {
        if (tid == 0) {
          atomicAdd(&P.dbg[kDbgTies], 1ull);
          int end = beam < nsk ? beam : nsk;  // extend over keys within the tolerance of the cut
          while (end > 0 && sk[end - 1] == 0ull) end--;  // fewer live candidates than beam
          while (end < nsk && sk[end] != 0ull &&
                 (uint32_t)(sk[end - 1] >> 32) - (uint32_t)(sk[end] >> 32) <= (uint32_t)kTolB)
            end++;
          // the run may continue below the margin: redo on all candidates
          w.misc()[9] = (trunc && (end >= nsk || sk[end] == 0ull)) ? 1 : 0;
          w.misc()[12] = end;
          w.misc()[13] = 0;
        }
        bsync();
        const int end = w.misc()[12];
        if (!w.misc()[9]) {
          // exact fp64 scores of ranks [0, end) in parallel, then thread 0
          // insertion-sorts each run (token sequences only on exact ties)
          if (end <= kBlockRun)
            for (int r = tid; r < end; r += NT) {
              const uint32_t id = w.crec()[0xffffffffu - (uint32_t)(sk[r] & 0xffffffffu)];
              w.runbuf()[r] = (int)id;
              w.runsc()[r] = cand_desc(w, id).sc;
            }
          bsync();
          // each run's first rank sorts it by exact score; runs holding
          // exactly equal scores (token-sequence order, shared scratch) are
          // left to thread 0
          auto near = [&](int r) {  // ranks r - 1 and r within the key tolerance
            return (uint32_t)(sk[r - 1] >> 32) - (uint32_t)(sk[r] >> 32) <= (uint32_t)kTolB;
          };
          int* run = w.runbuf();
          double* rsc = w.runsc();
          if (end <= kBlockRun)
            for (int r0 = tid; r0 + 1 < end; r0 += NT) {
              if ((r0 > 0 && near(r0)) || !near(r0 + 1)) continue;  // not the start of a run of >= 2
              int b0 = r0 + 2;
              while (b0 < end && near(b0)) b0++;
              bool eq = false;
              for (int i = r0 + 1; i < b0; i++) {
                const int x = run[i];
                const double xs = rsc[i];
                int j = i;
                while (j > r0 && xs >= rsc[j - 1]) {
                  if (xs == rsc[j - 1]) { eq = true; break; }
                  run[j] = run[j - 1];
                  rsc[j] = rsc[j - 1];
                  j--;
                }
                run[j] = x;
                rsc[j] = xs;
              }
              if (eq) {
                const int f = atomicAdd(&w.misc()[13], 1);
                if (f < 64) { w.hist()[128 + 2 * f] = (uint32_t)r0; w.hist()[129 + 2 * f] = (uint32_t)b0; }
              } else {
                for (int i = r0; i < b0 && i < beam; i++) w.rec()[i] = run[i];
              }
            }
          bsync();
          const int nflag = w.misc()[13];
          if (tid == 0 && (nflag || end > kBlockRun)) {
            if (end > kBlockRun) {
              w.misc()[10] = 1;  // absurd tie run: exact serial path
            } else {
              for (int f = 0; f < nflag; f++) {
                int a0, b0;
                if (nflag <= 64) {
                  a0 = (int)w.hist()[128 + 2 * f];
                  b0 = (int)w.hist()[129 + 2 * f];
                } else {  // too many to list: rescan every run
                  if (f > 0) break;
                  a0 = 0;
                  b0 = end;
                }
                for (int i = a0 + 1; i < b0; i++) {
                  const int x = run[i];
                  const double xs = rsc[i];
                  int j = i;
                  while (j > a0) {
                    const double ys = rsc[j - 1];
                    bool prec = xs > ys;
                    if (xs == ys) prec = bprecedes(w, desc_sc(w, (uint32_t)x, xs), desc_sc(w, (uint32_t)run[j - 1], ys));
                    if (!prec) break;
                    run[j] = run[j - 1];
                    rsc[j] = ys;
                    j--;
                  }
                  run[j] = x;
                  rsc[j] = xs;
                }
                for (int i = a0; i < b0 && i < beam; i++) w.rec()[i] = run[i];
              }
            }
          }
          bsync();
        }
      }
      if (!w.misc()[9]) break;
      if (tid == 0) atomicAdd(&P.dbg[kDbgOneshotFallback], 1ull);  // redo count
      // redo with every candidate (rare): full sort of the candidate keys
      bsync();
      block_sort_desc(w.ckey(), ncap, tid);
      sk = w.ckey();
      nsk = ncap;
      trunc = false;
    }
  }
  if (big || w.misc()[10]) {
    // exactly tied prefixes can exceed the candidate buffer (d_eff counts
    // strictly better prefixes only): exact serial selection for this frame
    if (tid == 0) {
      atomicAdd(&P.dbg[kDbgFrames], 1ull);
      int* head = w.dpi();  // per list: next valid position (dpi is free after grouping)
      for (int d = 0; d < nD; d++) head[d] = jth_valid(w, d, 0, k);
      int* sord = w.ord();  // specials in exact order
      for (int i = 0; i < nS; i++) {
        int j = i;
        const BDesc di{w.spsc()[i], w.spbase()[i], w.spx()[i], w.spflag()[i]};
        while (j > 0) {
          const int y = sord[j - 1];
          if (!bprecedes(w, di, BDesc{w.spsc()[y], w.spbase()[y], w.spx()[y], w.spflag()[y]})) break;
          sord[j] = y;
          j--;
        }
        sord[j] = i;
      }
      int sp = 0;
      for (int r = 0; r < beam; r++) {
        int wd = -2;  // -1: special, >= 0: list
        BDesc best{};
        if (sp < nS) { const int x = sord[sp]; best = BDesc{w.spsc()[x], w.spbase()[x], w.spx()[x], w.spflag()[x]}; wd = -1; }
        for (int d = 0; d < nD; d++) {
          if (head[d] >= k || !(w.lA()[d] > -INFINITY)) continue;
          const BDesc dd{bgen_score(w, d, head[d]), w.e1()[d], w.stok()[head[d]], 0};
          if (wd == -2 || bprecedes(w, dd, best)) { best = dd; wd = d; }
        }
        if (wd == -2 || !(best.sc > -INFINITY)) { w.rec()[r] = -1; continue; }
        if (wd == -1) {
          w.rec()[r] = (int)(kSpecial | (uint32_t)sord[sp]);
          sp++;
        } else {
          w.rec()[r] = (wd << 12) | head[wd];
          int nx = head[wd] + 1;
          while (nx < k && bexcl(w, wd, nx)) nx++;
          head[wd] = nx;
        }
      }
    }
    bsync();
  }
  // -- new entries (exact scores), then the exact beam threshold
  for (int r = tid; r < beam; r += NT) {
    const int rc = w.rec()[r];
    if (rc == -1) continue;
    const uint32_t rec = (uint32_t)rc;
    BCHK((rec & kSpecial) ? (int)(rec & ~kSpecial) < nS : ((int)(rec >> 12) < nD && (int)(rec & 0xfff) < k));
    if (!(rec & kSpecial)) {
      const int d = (int)(rec >> 12), j = (int)(rec & 0xfff);
      const int a = w.e1()[d], c = w.stok()[j];
      w.ns()[r] = bgen_score(w, d, j); w.nh()[r] = child_hash(w.ch()[a], c); w.nph()[r] = w.ch()[a];
      w.nl()[r] = c; w.nn()[r] = w.cn()[a] + 1; w.nf()[r] = 0; w.ntrel()[r] = pack_trel(a, c);
    } else {
      const int sx = (int)(rec & ~kSpecial);
      const int a = w.spbase()[sx], x = w.spx()[sx];
      w.ns()[r] = w.spsc()[sx];
      if (x >= 0) {
        w.nh()[r] = child_hash(w.ch()[a], x); w.nph()[r] = w.ch()[a]; w.nl()[r] = x; w.nn()[r] = w.cn()[a] + 1;
      } else {
        w.nh()[r] = w.ch()[a]; w.nph()[r] = w.cph()[a]; w.nl()[r] = w.cl()[a]; w.nn()[r] = w.cn()[a];
      }
      w.nf()[r] = w.spflag()[sx];
      w.ntrel()[r] = pack_trel(w.spsrc()[sx], w.sptok()[sx]);
    }
  }
  bsync();
  // winners are in exact rank order, ns[0] is the exact frame best; the kept
  // ones (decoder.py:621-623) form a prefix
  int c2 = 0;
  for (int r = tid; r < beam; r += NT)
    c2 += (w.rec()[r] != -1 && w.ns()[r] > -INFINITY && (P.threshold_inf || w.ns()[r] >= w.ns()[0] - P.beam_threshold)) ? 1 : 0;
  const int Hn = __syncthreads_count(c2);
  // reset the token -> S rank map for the next frame
  for (int j = tid; j < k; j += NT) w.pos()[w.stok()[j]] = 0xffff;
  bsync();
  return Hn;
}

// ------------------------------------------------------------------ finalize (decoder.py:753-817)
__device__ __forceinline__ void bfinalize(Blk& w, int H, int kept) {
  const Params& P = *w.P;
  const int tid = w.tid, u = w.u;
  for (int e = tid; e < H; e += NT) {
    int f = e;
    for (int q = 0; q < e; q++)
      if (w.ch()[q] == w.ch()[e] && w.cn()[q] == w.cn()[e]) { f = q; break; }
    w.first()[e] = f;
  }
  if (tid == 0) w.misc()[0] = 0;
  bsync();
  for (int e = tid; e < H; e += NT) {
    if (w.first()[e] != e) continue;
    double sc = w.cs()[e];  // entries are in rank order: the first is the payload (decoder.py:794-797)
    for (int q = e + 1; q < H; q++)
      if (w.first()[q] == e) sc = merge2_exact(sc, w.cs()[q], w.P->merge_max != 0);
    const int s = atomicAdd(&w.misc()[0], 1);
    w.spsc()[s] = sc; w.spbase()[s] = e; w.spx()[s] = -1; w.spflag()[s] = 0;
  }
  bsync();
  const int nF = w.misc()[0];
  int pad = 2;
  while (pad < nF) pad <<= 1;
  for (int s = tid; s < pad; s += NT)
    w.ckey()[s] = s < nF ? ((ord64(w.spsc()[s]) & ~0x3ffull) | (uint64_t)(0x3ff - s)) : 0ull;
  bsync();
  block_sort_desc(w.ckey(), pad, tid);
  // exact order: scores (full precision) then token sequences (tie runs)
  if (tid == 0) {
    int* ord = w.rec();
    for (int r = 0; r < nF; r++) ord[r] = 0x3ff - (int)(w.ckey()[r] & 0x3ffull);
    for (int i = 1; i < nF; i++) {
      const int x = ord[i];
      const BDesc dx{w.spsc()[x], w.spbase()[x], -1, 0};
      int j = i;
      while (j > 0) {
        const int y = ord[j - 1];
        const BDesc dy{w.spsc()[y], w.spbase()[y], -1, 0};
        if (!bprecedes(w, dx, dy)) break;
        ord[j] = y;
        j--;
      }
      ord[j] = x;
    }
  }
  bsync();
  const int nOut = nF < P.nbest ? nF : P.nbest;
  for (int r = tid; r < nOut; r += NT) {
    const int s = w.rec()[r];
    BCHK(s >= 0 && s < 3 * P.beam);
    const int e = w.spbase()[s];
    const int len = w.cn()[e];
    const size_t o = ((size_t)u * P.nbest + r);
    P.out_score[o] = w.spsc()[s];
    P.out_len[o] = len;
    int* tok_out = P.out_tokens + o * P.T_max;
    int* ts_out = P.out_ts ? P.out_ts + o * P.T_max : nullptr;
    int pos = len, slot = e;
    for (int i = kept - 1; i >= 0 && pos > 0; --i) {
      BCHK(slot >= 0 && slot < P.beam);
      const uint32_t rec = P.trellis[((size_t)u * P.T_max + i) * P.beam + slot];
      const int tok = trel_tok(rec);
      if (tok >= 0) {
        --pos;
        tok_out[pos] = tok;
        if (ts_out) ts_out[pos] = P.frame_map[(size_t)u * P.T_max + i];
      }
      slot = trel_src(rec);
    }
  }
  if (tid == 0) P.out_count[u] = nOut;
}

}  // namespace

__global__ void __launch_bounds__(NT) ctcb_decode_block_kernel(const __grid_constant__ Params P) {
  Blk w;
  w.P = &P;
  w.tid = threadIdx.x;
  const int tid = w.tid;
  w.par = 0;
  if (tid == 0)
    for (int s = 0; s < 2; s++) mbar_init(&w.mbar()[s], 1);
  for (int c = tid; c < P.V; c += NT) w.pos()[c] = 0xffff;
  for (int i = tid; i < 2 * kBlockTieCache; i += NT) w.tc_h()[i] = 0ull;
  for (int i = tid; i < kBlockTieCache; i += NT) w.tc_r()[i] = 0;
  fence_mbar_init();
  __syncthreads();
  uint32_t n_issue = 0, n_cons = 0;
  const uint32_t row_copy = (uint32_t)P.V * 4u;

  for (;;) {
    if (tid == 0) w.misc()[2] = atomicAdd(P.counter, 1);
    __syncthreads();
    const int item = w.misc()[2];
    __syncthreads();
    if (item >= P.B) {
      if (P.ready != nullptr) pdl_wait_primary();  // complete only after the top-k grid
      break;
    }
    const int u = P.order[item];
    w.u = u;
    const int len = P.lens[u];
    if (len <= 0 || len > P.T_max) {
      if (tid == 0) {
        P.status[u] = len == 0 ? kUttEmpty : kUttBadLen;
        P.out_count[u] = 0;
        P.kept[u] = 0;
      }
      continue;
    }
    const float* ubase = P.lp + (size_t)u * P.stride_b;
    int32_t* fmap = P.frame_map + (size_t)u * P.T_max;
    // -- A. blank-skip compaction (warp 0: ballot + prefix popcount); in
    //    precomputed mode ctcb_framemap_kernel already did it
    if (P.precomp) {
      if (tid == 0) w.misc()[3] = P.kept[u];
    } else if (tid < 32) {
      int kept = 0;
      for (int t0 = 0; t0 < len; t0 += 32) {
        const int t = t0 + tid;
        bool keep = t < len;
        if (keep && P.skip) keep = !(__ldg(ubase + (size_t)t * P.stride_t + P.blank) >= P.cutoff);
        const unsigned bal = __ballot_sync(FULL, keep);
        if (keep) fmap[kept + __popc(bal & lanemask_lt())] = t;
        kept += __popc(bal);
      }
      if (tid == 0) { P.kept[u] = kept; w.misc()[3] = kept; }
    }
    __syncthreads();
    const int kept = w.misc()[3];
    // -- B. frame loop
    if (tid == 0) { w.cs()[0] = 0.0; w.ch()[0] = kEmptyPrefixHash; w.cph()[0] = 0ull; w.cl()[0] = -1; w.cn()[0] = 0; w.cf()[0] = 1; }
    int H = 1;
    w.steps_done = 0;
    auto issue = [&](int i) {
      const uint32_t slot = n_issue & 1u;
      if (tid == 0 && P.bulk_ok) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&w.mbar()[slot], row_copy);
        tma_bulk_g2s(w.rows() + (size_t)slot * Blk::row_bytes, ubase + (size_t)fmap[i] * P.stride_t, row_copy,
                     &w.mbar()[slot]);
      }
      n_issue++;
    };
    if (kept > 0) issue(0);
    // precomputed top-k lists (ctcb_topk_wide_kernel), one frame ahead in registers
    const int k = P.k;
    const size_t tk_base = (size_t)u * P.T_max * k;
    int pre_t = 0;
    float pre_v = 0.0f;
    // overlapped top-k (P.ready): list j is read only after its flag is
    // published (warp 0 polls 32 flags per ballot, the block learns the new
    // bound through misc[15]); lists are read through L2 (__ldcg)
    int rdy = 0;
    // invalid input rows are never walked (see fast_decode): an utterance with
    // an offender key from the top-k kernel's screen ends as a dead beam before
    // its first frame / before the frames of the poll that saw it; misc[14]
    // makes the verdict block-uniform
    bool vbad = false;
    if (tid == 0) w.misc()[14] = (P.precomp && P.validate && P.ready == nullptr && kept > 0 && __ldcg(P.vkey + u) != ~0ull) ? 1 : 0;
    __syncthreads();
    vbad = w.misc()[14] != 0;
    __syncthreads();
    auto await_list = [&](int j) {  // block-uniform
      if (P.ready == nullptr || j < rdy) return;
      if (tid < 32) {
        const uint32_t* fl = P.ready + (size_t)u * P.T_max;
        int r = rdy;
        for (;;) {
          const int f = r + tid;
          const bool ok = f >= kept || ld_acquire_gpu(fl + f) != 0u;
          const unsigned bal = __ballot_sync(FULL, ok);
          r += bal == FULL ? 32 : __ffs(~bal) - 1;
          if (j < r) break;
          __nanosleep(128);
        }
        fence_acq_rel_gpu();
        if (tid == 0) {
          w.misc()[15] = r;
          if (P.validate && __ldcg(P.vkey + u) != ~0ull) w.misc()[14] = 1;
        }
      }
      __syncthreads();
      rdy = w.misc()[15];
      vbad = w.misc()[14] != 0;
      __syncthreads();
    };
    auto load_list = [&](int j) {
      if (P.ready != nullptr) {
        pre_t = __ldcg(P.topk_tok + tk_base + (size_t)j * k + tid);
        pre_v = __ldcg(P.topk_val + tk_base + (size_t)j * k + tid);
      } else {
        pre_t = P.topk_tok[tk_base + (size_t)j * k + tid];
        pre_v = P.topk_val[tk_base + (size_t)j * k + tid];
      }
    };
    if (P.precomp && kept > 0) await_list(0);
    if (P.precomp && kept > 0 && tid < k) load_list(0);
    __syncthreads();
    bool died = false;
    for (int i = 0; i < kept; i++) {
      if (vbad) { died = true; break; }
      if (i + 1 < kept) issue(i + 1);
      const uint32_t slot = n_cons & 1u;
      if (P.bulk_ok) {
        mbar_wait(&w.mbar()[slot], (n_cons >> 1) & 1u);
      } else {  // rows that are not 16-B multiples: plain copy (no TMA)
        float* dst = (float*)(w.rows() + (size_t)slot * Blk::row_bytes);
        const float* src = ubase + (size_t)fmap[i] * P.stride_t;
        for (int c = tid; c < P.V; c += NT) dst[c] = __ldg(src + c);
        __syncthreads();
      }
      n_cons++;
      const float* row = (const float*)(w.rows() + (size_t)slot * Blk::row_bytes);
      // input validation fused into the staging (emissions.py:128-150): warp 0
      // takes lane partials now and the verdict after the step (no extra
      // barrier); suspicious rows get the exact check from global memory
      // (precomputed mode: ctcb_topk_wide_kernel already screened every kept row)
      const bool vscreen = P.validate && !P.precomp;
      RowPart vpart{0u, 0xffffffffu, 0u};
      if (vscreen && tid < 32) vpart = row_partials(row, P.V, tid);
      auto vfinish = [&]() {
        if (vscreen && tid < 32 && !row_verdict(vpart, P.validate == 1)) {
          const int fr = fmap[i];
          const unsigned long long vk = row_check_exact(ubase + (size_t)fr * P.stride_t, P.V, fr, tid, P.validate == 1);
          if (tid == 0 && vk != ~0ull) atomicMin(&P.vkey[u], vk);
        }
      };
      if (P.precomp) {
        if (i + 1 < kept) await_list(i + 1);
        // S of this frame; bstep's first barrier publishes it
        if (tid < k) {
          w.stok()[tid] = pre_t;
          w.sval()[tid] = pre_v;
          w.pos()[pre_t] = (uint16_t)tid;
          if (i + 1 < kept) load_list(i + 1);
        }
      } else {
        btopk(w, row);
      }
      const int Hn = bstep(w, row, H);
      vfinish();
      if (Hn == 0) { died = true; break; }
      // ntrel / the row slot are rewritten only after later barriers
      uint32_t* trow = P.trellis + ((size_t)u * P.T_max + i) * P.beam;
      for (int r = tid; r < Hn; r += NT) trow[r] = w.ntrel()[r];
      w.swap_state();
      H = Hn;
      w.steps_done = i + 1;
    }
    if (tid == 0) P.vdone[u] = (P.precomp || !died) ? kept : w.steps_done + 1;  // rows screened
    if (died) {
      while (n_cons < n_issue) {
        if (P.bulk_ok) mbar_wait(&w.mbar()[n_cons & 1u], (n_cons >> 1) & 1u);
        n_cons++;
      }
      if (tid == 0) {
        P.status[u] = kUttBeamDied;
        P.out_count[u] = 0;
        P.out_len[(size_t)u * P.nbest] = w.steps_done;
      }
      __syncthreads();
      continue;
    }
    bfinalize(w, H, kept);
    if (tid == 0) P.status[u] = kUttOk;
    __syncthreads();
  }
}

// Frame-parallel top-k for the block kernel (V <= 512, k <= 256): one warp
// per kept row of the flattened (utterance, kept frame) space.  The k-th
// largest value key is found by a bitwise radix select (one warp reduction
// per bit), the keys above it plus the lowest-index ones equal to it are
// ballot-compacted into shared memory and sorted in registers (value desc,
// index asc); they go to topk_tok / topk_val[u, i, :].  Same S as btopk.
template <int R>
__device__ __forceinline__ void topk_sort_write(const uint64_t* buf, int k, const float* src, int32_t* tok,
                                                float* val, int lane) {
  uint64_t kk[R];
#pragma unroll
  for (int r = 0; r < R; r++) {
    const int i = r * 32 + lane;
    kk[r] = i < k ? buf[i] : 0ull;
  }
  warp_sort_desc<R>(kk, lane);
#pragma unroll
  for (int r = 0; r < R; r++) {
    const int j = lane * R + r;
    if (j < k) {
      const int c = (int)(0xffffffffu - (uint32_t)(kk[r] & 0xffffffffu));
      tok[j] = c;
      val[j] = __ldg(src + c);  // the row's own bits (signed zeros)
    }
  }
}
__global__ void __launch_bounds__(256, 3) ctcb_topk_wide_kernel(const __grid_constant__ Params P) {
  __shared__ uint64_t sbuf[8][256];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint64_t* buf = sbuf[wid];
  // overlapped mode (P.ready): the block walk is a programmatic dependent of
  // this grid (see ctcb_topk_kernel); rows go frame-major, g = frame * B + slot
  // with utterance order[slot], and each list is published by its ready flag
  pdl_launch_dependents();
  const bool fm = P.ready != nullptr;
  const long long nw = (long long)gridDim.x * (blockDim.x >> 5);
  const long long total = fm ? (long long)P.B * P.T_max : P.rowoff[P.B];
  const int V = P.V, k = P.k, blank = P.blank;
  for (long long g = (long long)blockIdx.x * (blockDim.x >> 5) + wid; g < total; g += nw) {
    int u, i;
    if (fm) {
      u = P.order[(int)(g % P.B)];
      i = (int)(g / P.B);
      if (i >= P.kept[u]) continue;
    } else {
      int lo = 0, hi = P.B - 1;  // utterance: last u with rowoff[u] <= g
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (P.rowoff[mid] <= g) lo = mid; else hi = mid - 1;
      }
      u = lo;
      i = (int)(g - P.rowoff[u]);
    }
    const float* src = P.lp + (size_t)u * P.stride_b + (size_t)P.frame_map[(size_t)u * P.T_max + i] * P.stride_t;
    uint32_t key[16];  // ord32 (0: absent), token r * 32 + lane
    float vs = 0.0f, vmn = INFINITY, vmx = -INFINITY;  // validation screen partials
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int c = r * 32 + lane;
      const float x = c < V ? __ldg(src + c) : -1e30f;
      key[r] = (c < V && c != blank) ? ord32(x) : 0u;
      vmn = fminf(vmn, x);
      vmx = fmaxf(vmx, x);
      vs += ex2_ftz(x * 1.4426950408889634f);
    }
    if (P.validate) {  // input validation of every kept row (emissions.py:128-150)
      const RowPart vp{vs <= 2.0f ? ord32(vmx) : 0xffffffffu, ord32(vmn), (uint32_t)(fminf(vs, 2.0f) * 33554432.0f)};
      if (!row_verdict(vp, P.validate == 1)) {
        const int fr = P.frame_map[(size_t)u * P.T_max + i];
        const unsigned long long vk = row_check_exact(src, V, fr, lane, P.validate == 1);
        if (lane == 0 && vk != ~0ull) atomicMin(&P.vkey[u], vk);
      }
    }
    // largest T with #{key >= T} >= k
    uint32_t T = 0u;
    for (int bit = 31; bit >= 0; bit--) {
      const uint32_t cand = T | (1u << bit);
      int n = 0;
#pragma unroll
      for (int r = 0; r < 16; r++) n += key[r] >= cand;
      if (__reduce_add_sync(FULL, n) >= k) T = cand;
    }
    // keys > T, then the lowest-index keys == T up to k, compacted in token order
    int ngt = 0;
#pragma unroll
    for (int r = 0; r < 16; r++) ngt += key[r] > T;
    int need_eq = k - (int)__reduce_add_sync(FULL, ngt);
    int o = 0;
#pragma unroll
    for (int r = 0; r < 16; r++) {
      const int c = r * 32 + lane;
      const bool eq = key[r] == T && (c < V && c != blank);
      const unsigned beq = __ballot_sync(FULL, eq);
      const int rank_eq = __popc(beq & lanemask_lt());
      const bool take = key[r] > T || (eq && rank_eq < need_eq);
      need_eq -= __popc(beq) < need_eq ? __popc(beq) : need_eq;
      const unsigned bt = __ballot_sync(FULL, take);
      if (take) buf[o + __popc(bt & lanemask_lt())] = ((uint64_t)key[r] << 32) | (uint64_t)(0xffffffffu - (uint32_t)c);
      o += __popc(bt);
    }
    __syncwarp();
    const size_t ob = ((size_t)u * P.T_max + i) * k;
    if (k <= 64) topk_sort_write<2>(buf, k, src, P.topk_tok + ob, P.topk_val + ob, lane);
    else if (k <= 128) topk_sort_write<4>(buf, k, src, P.topk_tok + ob, P.topk_val + ob, lane);
    else topk_sort_write<8>(buf, k, src, P.topk_tok + ob, P.topk_val + ob, lane);
    __syncwarp();
    if (fm) {  // every lane fences its list stores, lane 0 publishes
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_gpu(P.ready + (size_t)u * P.T_max + i, 1u);
    }
  }
}

}  // namespace ctcb
