// Generic CTC prefix beam-search decode kernel: one warp per utterance,
// any beam <= 1024, any vocabulary.  Semantics follow the reference CPU
// decoder (ctcforge, decoder.py:102-817; emissions.py:284-306) exactly; see
// DESIGN.md for the derivation of the reduced candidate set.
//
// Per utterance (one warp, persistent loop over a longest-first work queue):
//   A. blank-skip compaction: warp ballot + prefix popcount over the blank
//      column builds the kept-frame map (emissions.py:298-306);
//   B. per kept frame, the row is staged into shared memory by a TMA bulk copy
//      (ring of `ring` rows, prefetched ahead), then
//      1. top-k: radix select of the k = min(2*beam, V-1) best non-blank
//         tokens by (log-prob desc, index asc) + bitonic sort;
//      2. merge groups are formed analytically:
//         blank groups (R,1), repeat groups (R',0) for beam entries, and
//         append groups (R+c,0) as one sorted list per distinct prefix R;
//      3. the next beam is a k-way merge of those sorted lists under the
//         reference's total order (score desc, token sequence asc, flag asc)
//         with the beam_threshold cut (decoder.py:615-681);
//      4. back-pointers go to a device-resident trellis;
//   C. finalize: log-add the flag variants of each prefix, order, backtrace
//      the n-best through the trellis (decoder.py:753-817).
#include <cfloat>
#include <cmath>

#include "ctcb_common.cuh"
#include "ctcb_internal.h"

namespace ctcb {

namespace {

struct Warp {
  const Params* P;
  int lane, u, steps_done;
  int keff;  // valid top-k positions this frame (beam_size_token: the selected prefix of S)
  uint8_t* rows;
  uint64_t* mbar;
  double *cs, *ns, *headsc, *spsc;
  uint64_t *ch, *cph, *nh, *nph, *skey, *spkey;
  int *cl, *cn, *cf, *nl, *nn, *nf;
  uint32_t *ntrel, *excl, *hist;
  int *first, *dpi, *pd, *e1, *e2, *headj;
  float* sval;
  int *stok, *spord, *spbase, *spx, *spflag, *spsrc, *sptok, *misc;
  uint16_t* pos;
  uint64_t* tc_h;
  int* tc_r;
  uint64_t* htk;
  int *htf, *hslot, *rec, *rec2;
  uint32_t* hkey;
  double* lA;
  int kw, ts;

  __device__ void swap_state() {
    double* d = cs; cs = ns; ns = d;
    uint64_t* h = ch; ch = nh; nh = h;
    h = cph; cph = nph; nph = h;
    int* x = cl; cl = nl; nl = x;
    x = cn; cn = nn; nn = x;
    x = cf; cf = nf; nf = x;
  }
};

__device__ void carve(Warp& w, uint8_t* base, const Params& P) {
  int kpad = P.kpad;
  WarpLayout L = make_layout(P.beam, kpad, P.V, P.ring, P.row_bytes);
  w.rows = base + L.rows;
  w.mbar = (uint64_t*)(base + L.mbar);
  w.cs = (double*)(base + L.cur_score);
  w.ch = (uint64_t*)(base + L.cur_hash);
  w.cph = (uint64_t*)(base + L.cur_phash);
  w.ns = (double*)(base + L.nxt_score);
  w.nh = (uint64_t*)(base + L.nxt_hash);
  w.nph = (uint64_t*)(base + L.nxt_phash);
  w.headsc = (double*)(base + L.head_sc);
  w.skey = (uint64_t*)(base + L.skey);
  w.spsc = (double*)(base + L.sp_sc);
  w.spkey = (uint64_t*)(base + L.sp_key);
  w.cl = (int*)(base + L.cur_last);
  w.cn = (int*)(base + L.cur_len);
  w.cf = (int*)(base + L.cur_flag);
  w.nl = (int*)(base + L.nxt_last);
  w.nn = (int*)(base + L.nxt_len);
  w.nf = (int*)(base + L.nxt_flag);
  w.ntrel = (uint32_t*)(base + L.nxt_trel);
  w.first = (int*)(base + L.first);
  w.dpi = (int*)(base + L.dpi);
  w.pd = (int*)(base + L.pd);
  w.e1 = (int*)(base + L.dp_e1);
  w.e2 = (int*)(base + L.dp_e2);
  w.headj = (int*)(base + L.head_j);
  w.excl = (uint32_t*)(base + L.excl);
  w.sval = (float*)(base + L.sval);
  w.stok = (int*)(base + L.stok);
  w.spord = (int*)(base + L.sp_ord);
  w.spbase = (int*)(base + L.sp_base);
  w.spx = (int*)(base + L.sp_x);
  w.spflag = (int*)(base + L.sp_flag);
  w.spsrc = (int*)(base + L.sp_src);
  w.sptok = (int*)(base + L.sp_tok);
  w.hist = (uint32_t*)(base + L.hist);
  w.misc = (int*)(base + L.misc);
  w.pos = (uint16_t*)(base + L.pos);
  w.tc_h = (uint64_t*)(base + L.tc_h);
  w.tc_r = (int*)(base + L.tc_r);
  w.htk = (uint64_t*)(base + L.htk);
  w.htf = (int*)(base + L.htf);
  w.hslot = (int*)(base + L.hslot);
  w.rec = (int*)(base + L.rec);
  w.rec2 = (int*)(base + L.rec2);
  w.hkey = (uint32_t*)(base + L.hkey);
  w.lA = (double*)(base + L.lA);
  w.kw = L.kw;
  w.ts = L.ts;
}

// ------------------------------------------------------------------ sorting
// Warp bitonic sort of u64 keys, descending.
__device__ void bitonic_desc_u64(uint64_t* key, int n, int lane) {
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = lane; t < (n >> 1); t += 32) {
        int i = ((t & ~(stride - 1)) << 1) | (t & (stride - 1));
        int j = i + stride;
        uint64_t a = key[i], b = key[j];
        bool desc = (i & size) == 0;
        if (desc ? (a < b) : (a > b)) { key[i] = b; key[j] = a; }
      }
      __syncwarp();
    }
}
// Warp bitonic sort of (key desc, idx asc) pairs.
__device__ void bitonic_pairs(uint64_t* key, int* idx, int n, int lane) {
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = lane; t < (n >> 1); t += 32) {
        int i = ((t & ~(stride - 1)) << 1) | (t & (stride - 1));
        int j = i + stride;
        uint64_t a = key[i], b = key[j];
        int ia = idx[i], ib = idx[j];
        bool a_first = a > b || (a == b && ia < ib);
        bool desc = (i & size) == 0;
        if (desc ? !a_first : a_first) { key[i] = b; key[j] = a; idx[i] = ib; idx[j] = ia; }
      }
      __syncwarp();
    }
}

// ------------------------------------------------------------------ token sequences
// Full comparison through the trellis (trellis_seq_cmp); *strict: the
// sequences differ before the shorter one ends (then every extension keeps
// the order).
__device__ int seq_cmp_full(const Warp& w, int ea, int xa, int eb, int xb, bool* strict) {
  const Params& P = *w.P;
  int* A = P.seqbuf + (size_t)w.u * 3 * (P.T_max + 1);
  const uint32_t* tr = P.trellis + (size_t)w.u * P.T_max * P.beam;
  auto rec = [&](int i, int slot) {
    const uint32_t r = tr[(size_t)i * P.beam + slot];
    return make_int2(trel_tok(r), trel_src(r));
  };
  return trellis_seq_cmp(rec, w.steps_done, ea, xa, eb, xb, A, A + P.T_max + 1, strict, P.dbg);
}
// Strict-order cache keyed by prefix hashes (see the fast kernel): orders of
// sibling lineages with identical scores are computed once.
__device__ int gtc_lookup(const Warp& w, uint64_t ha, uint64_t hb) {
#pragma unroll 1
  for (int i = 0; i < kTieCache; i++) {
    if (w.tc_h[2 * i] == ha && w.tc_h[2 * i + 1] == hb) return w.tc_r[i];
    if (w.tc_h[2 * i] == hb && w.tc_h[2 * i + 1] == ha) return -w.tc_r[i];
  }
  return 0;
}
__device__ void gtc_insert(const Warp& w, uint64_t ha, uint64_t hb, int r) {
  if (gtc_lookup(w, ha, hb)) return;
  int i = w.tc_r[kTieCache];
  w.tc_h[2 * i] = ha;
  w.tc_h[2 * i + 1] = hb;
  w.tc_r[i] = r;
  w.tc_r[kTieCache] = (i + 1) % kTieCache;
}
// Python tuple order of seq(ea)+[xa] vs seq(eb)+[xb] (x < 0: no extra token).
__device__ int seq_cmp(const Warp& w, int ea, int xa, int eb, int xb) {
  const uint64_t hba = w.ch[ea], hbb = w.ch[eb];
  const int lba = w.cn[ea], lbb = w.cn[eb];
  if (hba == hbb && lba == lbb) {
    if (xa == xb) return 0;
    return xa < xb ? -1 : 1;
  }
  const uint64_t ha = xa >= 0 ? child_hash(hba, xa) : hba, hb = xb >= 0 ? child_hash(hbb, xb) : hbb;
  const int la = lba + (xa >= 0), lb = lbb + (xb >= 0);
  if (ha == hb && la == lb) return 0;
  int r = gtc_lookup(w, hba, hbb);
  if (r) {
    gtc_insert(w, ha, hb, r);
    return r;
  }
  r = gtc_lookup(w, ha, hb);
  if (r) return r;
  bool strict = false;
  r = seq_cmp_full(w, ea, -1, eb, -1, &strict);
  if (strict) {
    gtc_insert(w, hba, hbb, r);
    gtc_insert(w, ha, hb, r);
    return r;
  }
  r = seq_cmp_full(w, ea, xa, eb, xb, &strict);
  if (strict) gtc_insert(w, ha, hb, r);
  return r;
}
// Candidate descriptor: (score, base entry, extra token, blank flag).
struct Desc { double sc; int base, x, flag; };
// true if a precedes b in the reference's rank order (decoder.py:651-681).
__device__ bool precedes(const Warp& w, const Desc& a, const Desc& b) {
  if (a.sc != b.sc) return a.sc > b.sc;
  atomicAdd(&w.P->dbg[kDbgExactTies], 1ull);
  int c = seq_cmp(w, a.base, a.x, b.base, b.x);
  if (c) return c < 0;
  return a.flag < b.flag;
}
__device__ Desc spec_desc(const Warp& w, int s) { return Desc{w.spsc[s], w.spbase[s], w.spx[s], w.spflag[s]}; }

// Re-sort runs of exactly equal scores in a sorted specials order (lane 0;
// only when the parallel check finds a run).
__device__ void fix_tie_runs(const Warp& w, int n) {
  bool run = false;
  for (int s = w.lane; s + 1 < n; s += 32) run |= w.spkey[s] == w.spkey[s + 1];
  if (!__any_sync(FULL, run)) return;
  if (w.lane == 0) {
    int a = 0;
    while (a < n) {
      int b = a + 1;
      while (b < n && w.spkey[b] == w.spkey[a]) b++;
      if (b - a > 1)
        for (int i = a + 1; i < b; i++) {
          int x = w.spord[i], j = i;
          Desc dx = spec_desc(w, x);
          while (j > a && precedes(w, dx, spec_desc(w, w.spord[j - 1]))) { w.spord[j] = w.spord[j - 1]; j--; }
          w.spord[j] = x;
        }
      a = b;
    }
  }
  __syncwarp();
}

// ------------------------------------------------------------------ top-k
// S = the k best non-blank tokens of `row` by (value desc, index asc),
// written sorted to sval/stok; pos[token] = rank in S.
__device__ void topk(Warp& w, const float* row) {
  const Params& P = *w.P;
  const int V = P.V, blank = P.blank, k = P.k, lane = w.lane;
  uint32_t kth = 0;
  int need = V;
  if (k < V - 1) {
    uint32_t prefix = 0, pmask = 0;
    need = k;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int b = lane; b < 256; b += 32) w.hist[b] = 0;
      __syncwarp();
      for (int c = lane; c < V; c += 32) {
        if (c == blank) continue;
        uint32_t key = ord32(row[c]);
        if ((key & pmask) == prefix) atomicAdd(&w.hist[(key >> shift) & 255u], 1u);
      }
      __syncwarp();
      uint32_t h[8], s = 0;
#pragma unroll
      for (int q = 0; q < 8; q++) { h[q] = w.hist[lane * 8 + q]; s += h[q]; }
      uint32_t incl = s;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        uint32_t v = __shfl_down_sync(FULL, incl, off);
        if (lane + off < 32) incl += v;
      }
      uint32_t cum = incl - s;  // tokens in digits owned by higher lanes
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
    kth = prefix;
  }
  // ordered compaction: keys > kth, then the `need` lowest-index keys == kth
  int n = 0, eq_taken = 0;
  const unsigned lt = lanemask_lt();
  for (int c0 = 0; c0 < V; c0 += 32) {
    int c = c0 + lane;
    bool valid = c < V && c != blank;
    uint32_t key = valid ? ord32(row[c]) : 0u;
    bool gt = valid && key > kth, eq = valid && key == kth;
    unsigned beq = __ballot_sync(FULL, eq);
    bool acc = gt || (eq && eq_taken + __popc(beq & lt) < need);
    unsigned bsel = __ballot_sync(FULL, acc);
    if (acc) w.skey[n + __popc(bsel & lt)] = ((uint64_t)key << 32) | (uint64_t)(0xffffffffu - (uint32_t)c);
    n += __popc(bsel);
    eq_taken += __popc(beq);
  }
  for (int j = n + lane; j < P.kpad; j += 32) w.skey[j] = 0;
  __syncwarp();
  bitonic_desc_u64(w.skey, P.kpad, lane);
  for (int j = lane; j < k; j += 32) {
    int c = (int)(0xffffffffu - (uint32_t)(w.skey[j] & 0xffffffffu));
    w.stok[j] = c;
    w.sval[j] = row[c];
    w.pos[c] = (uint16_t)j;
  }
  __syncwarp();
}

// ------------------------------------------------------------------ beam step
__device__ __forceinline__ bool excl_bit(const Warp& w, int d, int j) {
  return (w.excl[d * w.kw + (j >> 5)] >> (j & 31)) & 1u;
}
__device__ __forceinline__ int next_valid(const Warp& w, int d, int j) {
  const int k = w.keff;
  for (++j; j < k; ++j)
    if (!excl_bit(w, d, j)) break;
  return j;
}
// score of the append group (R_d + S[j], 0): fold of the prefix's entries in
// rank order (candidate order is hypothesis-major, decoder.py:531-543).
__device__ __forceinline__ double gen_score(const Warp& w, int d, int j) {
  double v = (double)w.sval[j];
  int a = w.e1[d], b = w.e2[d];
  double s = w.cs[a] + v;
  if (b >= 0) s = merge2_exact(s, w.cs[b] + v, w.P->merge_max != 0);
  return s;
}

// One frame-synchronous step over the current beam (H entries) with emission
// row `row`.  Returns the new beam size (0: beam died).
__device__ int beam_step(Warp& w, const float* row, int H) {
  const Params& P = *w.P;
  const int lane = w.lane, beam = P.beam;
  const double eb = (double)row[P.blank];
  // beam_size_token = K < V (decoder.py:440-458): blank / repeats / appends
  // only for selected tokens; the selected non-blank tokens are a prefix of S
  // when K <= k, else every S token plus those above the K-th key
  int k = P.k;
  bool has_blank = true, wide = false;
  uint32_t tv = 0u;
  int ti = 0;
  if (P.tokK) {
    const uint32_t kb = ord32((float)eb);
    if (P.tokK <= P.k) {
      int above = 0;
      for (int j = lane; j < P.k; j += 32) {
        const uint32_t kv = ord32(w.sval[j]);
        above += (kv > kb || (kv == kb && w.stok[j] < P.blank)) ? 1 : 0;
      }
      above = __reduce_add_sync(FULL, above);
      has_blank = above < P.tokK;
      k = has_blank ? P.tokK - 1 : P.tokK;
    } else {
      kth_token(row, P.V, P.blank, (float)eb, P.tokK, w.hist, lane, tv, ti);
      has_blank = token_selected(kb, P.blank, tv, ti);
      wide = true;
    }
  }
  w.keff = k;
  auto selected = [&](int c) -> bool {
    if (!P.tokK) return true;
    if (wide) return token_selected(ord32(row[c]), c, tv, ti);
    const int j = w.pos[c];
    return j != 0xffff && j < k;
  };

  // -- prefix grouping: entries sharing a token sequence (flag 0 / flag 1),
  //    through a shared-memory hash table keyed by (prefix hash, length)
  const int TS = w.ts;
  for (int i = lane; i < TS; i += 32) { w.htk[i] = 0ull; w.htf[i] = 0x7fffffff; }
  __syncwarp();
  for (int e = lane; e < H; e += 32) {
    const uint64_t key = (w.ch[e] ^ ((uint64_t)w.cn[e] * 0x9e3779b97f4a7c15ull)) | 1ull;
    uint32_t i = (uint32_t)mix64(key) & (uint32_t)(TS - 1);
    for (;;) {
      const unsigned long long prev = atomicCAS((unsigned long long*)&w.htk[i], 0ull, (unsigned long long)key);
      if (prev == 0ull || prev == key) break;
      i = (i + 1) & (uint32_t)(TS - 1);
    }
    atomicMin(&w.htf[i], e);
    w.hslot[e] = (int)i;
  }
  __syncwarp();
  for (int e = lane; e < H; e += 32) w.first[e] = w.htf[w.hslot[e]];
  __syncwarp();
  int nD = 0;
  for (int b0 = 0; b0 < H; b0 += 32) {
    int e = b0 + lane;
    bool isf = e < H && w.first[e] == e;
    unsigned bal = __ballot_sync(FULL, isf);
    if (isf) {
      int d = nD + __popc(bal & lanemask_lt());
      w.dpi[e] = d; w.e1[d] = e; w.e2[d] = -1;
    }
    nD += __popc(bal);
  }
  __syncwarp();
  for (int e = lane; e < H; e += 32)
    if (w.first[e] != e) { int d = w.dpi[w.first[e]]; w.dpi[e] = d; w.e2[d] = e; }
  for (int i = lane; i < nD * w.kw; i += 32) w.excl[i] = 0u;
  if (lane == 0) w.misc[0] = 0;
  __syncwarp();
  // -- parent links of flag-0 entries; children exclude their token from the
  //    parent's generic list (they become repeat groups)
  for (int e = lane; e < H; e += 32) {
    int p = -1;
    if (w.cf[e] == 0) {
      const uint64_t key = (w.cph[e] ^ ((uint64_t)(w.cn[e] - 1) * 0x9e3779b97f4a7c15ull)) | 1ull;
      uint32_t i = (uint32_t)mix64(key) & (uint32_t)(TS - 1);
      for (;;) {
        const uint64_t k2 = w.htk[i];
        if (k2 == 0ull) break;
        if (k2 == key) { p = w.dpi[w.htf[i]]; break; }
        i = (i + 1) & (uint32_t)(TS - 1);
      }
      if (p >= 0) {
        int j = w.pos[w.cl[e]];
        if (j != 0xffff) atomicOr(&w.excl[p * w.kw + (j >> 5)], 1u << (j & 31));
      }
    }
    w.pd[e] = p;
  }
  __syncwarp();
  // -- specials: blank groups, repeat groups, last-token appends
  for (int d = lane; d < nD; d += 32) {
    int a = w.e1[d], b = w.e2[d];
    if (has_blank) {
      double sc = w.cs[a] + eb;
      if (b >= 0) sc = merge2_exact(sc, w.cs[b] + eb, w.P->merge_max != 0);
      int s = atomicAdd(&w.misc[0], 1);
      w.spsc[s] = sc; w.spbase[s] = a; w.spx[s] = -1; w.spflag[s] = 1; w.spsrc[s] = a; w.sptok[s] = -1;
    }
    int c = w.cl[a];
    if (c >= 0) {
      int j = w.pos[c];
      if (j != 0xffff && !excl_bit(w, d, j)) {
        int f = w.cf[a] == 1 ? a : ((b >= 0 && w.cf[b] == 1) ? b : -1);
        if (f >= 0 && selected(c)) {
          int s2 = atomicAdd(&w.misc[0], 1);
          w.spsc[s2] = w.cs[f] + (double)w.sval[j];
          w.spbase[s2] = a; w.spx[s2] = c; w.spflag[s2] = 0; w.spsrc[s2] = f; w.sptok[s2] = c;
        }
        w.excl[d * w.kw + (j >> 5)] |= 1u << (j & 31);
      }
    }
  }
  for (int e = lane; e < H; e += 32) {
    if (w.cf[e] != 0) continue;
    int c = w.cl[e];
    if (!selected(c)) continue;  // no repeat and no parent append of an unselected token
    double ec = (double)row[c];
    double sc = w.cs[e] + ec, best = sc;  // repeat candidate comes first (decoder.py:522-530)
    int src = e, tok = -1;
    int p = w.pd[e];
    if (p >= 0) {
      int srcs[2] = {w.e1[p], w.e2[p]};
#pragma unroll
      for (int q = 0; q < 2; q++) {
        int h = srcs[q];
        if (h < 0 || (w.cf[h] == 0 && w.cl[h] == c)) continue;  // blocked repeat (decoder.py:495)
        double x = w.cs[h] + ec;
        sc = merge2_exact(sc, x, w.P->merge_max != 0);
        if (x > best) { best = x; src = h; tok = c; }
      }
    }
    int s = atomicAdd(&w.misc[0], 1);
    w.spsc[s] = sc; w.spbase[s] = e; w.spx[s] = -1; w.spflag[s] = 0; w.spsrc[s] = src; w.sptok[s] = tok;
  }
  __syncwarp();
  const int nS = w.misc[0];
  const int sp_pad = pow2_at_least(nS);
  for (int s = lane; s < sp_pad; s += 32) {
    w.spkey[s] = s < nS ? ord64(w.spsc[s]) : 0ull;
    w.spord[s] = s < nS ? s : 0x7fffffff;
  }
  __syncwarp();
  bitonic_pairs(w.spkey, w.spord, sp_pad, lane);
  fix_tie_runs(w, nS);
  // -- append-list heads.  Lists are ranked by A(R) + v with A = logaddexp of
  //    R's entries (a few ulps from the exact per-candidate fold); exact
  //    scores are computed for key ties and, in parallel, for the winners.
  for (int d = lane; d < nD; d += 32) {
    const int a = w.e1[d], b = w.e2[d];
    w.lA[d] = b >= 0 ? merge2_exact(w.cs[a], w.cs[b], w.P->merge_max != 0) : w.cs[a];
    w.headj[d] = next_valid(w, d, -1);
  }
  __syncwarp();
  const int nH = nD + 1;  // lists 0..nD-1, then the sorted specials
  auto head_approx = [&](int i, int sp) -> double {
    if (i < nD) return w.headj[i] < k ? w.lA[i] + (double)w.sval[w.headj[i]] : -INFINITY;
    return sp < nS ? w.spsc[w.spord[sp]] : -INFINITY;
  };
  double lbest = -INFINITY;
  for (int i = lane; i < nH; i += 32) lbest = fmax(lbest, head_approx(i, 0));
  const uint64_t ok64 = lbest > -INFINITY ? ord64(lbest) : 0ull;
  const uint32_t mhi = __reduce_max_sync(FULL, (uint32_t)(ok64 >> 32));
  const uint32_t mlo = __reduce_max_sync(FULL, (uint32_t)(ok64 >> 32) == mhi ? (uint32_t)ok64 : 0u);
  const uint64_t bk = ((uint64_t)mhi << 32) | mlo;
  if (bk == 0ull) return 0;  // every extension is -inf (decoder.py:616-620)
  const uint64_t bu = (bk >> 63) ? (bk & 0x7fffffffffffffffull) : ~bk;
  const double best = __longlong_as_double((long long)bu);
  const double lo_thr = P.threshold_inf ? -DBL_MAX : best - P.beam_threshold;  // decoder.py:621-623
  const double kR = P.threshold_inf ? 1048576.0 : fmin(P.beam_threshold, 1048576.0);
  const double kScale = 4294967294.0 / kR, koff = -(best - kR) * kScale;
  auto keyof = [&](double sc) -> uint32_t {
    const double z = fmin(fmax(fma(sc, kScale, koff), 0.0), 4294967294.0);
    const uint32_t t = (uint32_t)__double_as_longlong(__dadd_rz(z, 4503599627370496.0));
    // approximate list scores may sit an ulp below the threshold: keep a
    // margin here, the exact post-filter below applies decoder.py:621-623
    if (!(sc > -INFINITY)) return 0u;
    return (P.threshold_inf || sc >= lo_thr - 1e-9 * (1.0 + fabs(lo_thr))) ? 1u + t : 0u;
  };
  for (int i = lane; i < nH; i += 32) w.hkey[i] = keyof(head_approx(i, 0));
  __syncwarp();

  // -- k-way merge under the reference order (decoder.py:651-681): one
  //    redux per round; each lane keeps the best key of the heads it owns
  //    (i = lane + 32 j); the winner's lane pops and rescans its own heads.
  int sp_ptr = 0;  // owned by lane (nD & 31); mirrored to misc[1] for the tie path
  if (lane == 0) w.misc[1] = 0;
  uint32_t lk = 0u, lk2 = 0u;  // best and second-best key of the heads this lane owns
  int li = -1;
  auto rescan = [&]() {
    lk = 0u; lk2 = 0u; li = -1;
    for (int i = lane; i < nH; i += 32) {
      const uint32_t kk = w.hkey[i];
      if (kk > lk) { lk2 = lk; lk = kk; li = i; }
      else if (kk > lk2) lk2 = kk;
    }
  };
  rescan();
  int Hn = 0;
  // list keys come from A + v, a few ulps from the exact fold, and every key
  // is floored: heads within kTolG units of the maximum are resolved exactly
  constexpr uint32_t kTolG = 2u;
  for (int r = 0; r < beam; r++) {
    const uint32_t mk = __reduce_max_sync(FULL, lk);
    if (mk == 0u) break;
    const unsigned tl = __ballot_sync(FULL, mk - lk <= kTolG);
    const int first_lane = __ffs(tl) - 1;
    const uint32_t second = __shfl_sync(FULL, lk2, first_lane);
    int win;
    if ((tl & (tl - 1)) == 0u && (second == 0u || mk - second > kTolG)) {
      win = __shfl_sync(FULL, li, first_lane);
    } else {
      // (near-)equal keys: exact scores, then token sequence, then flag
      win = -1;
      __syncwarp();
      if (lane == 0) {
        const int sp = w.misc[1];
        Desc dw{};
        for (int i = 0; i < nH; i++) {
          if (w.hkey[i] == 0u || mk - w.hkey[i] > kTolG) continue;
          Desc di = i < nD ? Desc{gen_score(w, i, w.headj[i]), w.e1[i], w.stok[w.headj[i]], 0}
                           : spec_desc(w, w.spord[sp]);
          if (win < 0 || precedes(w, di, dw)) { win = i; dw = di; }
        }
      }
      win = __shfl_sync(FULL, win, 0);
    }
    if ((win & 31) == lane) {
      if (win < nD) {
        const int j = w.headj[win];
        w.rec[r] = (win << 12) | j;
        const int jn = next_valid(w, win, j);
        w.headj[win] = jn;
        w.hkey[win] = jn < k ? keyof(w.lA[win] + (double)w.sval[jn]) : 0u;
      } else {
        w.rec[r] = (win << 12) | 0xfff;
        w.rec2[r] = sp_ptr;
        sp_ptr++;
        w.misc[1] = sp_ptr;
        w.hkey[win] = sp_ptr < nS ? keyof(w.spsc[w.spord[sp_ptr]]) : 0u;
      }
      rescan();
    }
    Hn = r + 1;
  }
  __syncwarp();
  // -- new entries in parallel (exact scores: fold of R's entries in rank order)
  for (int r = lane; r < Hn; r += 32) {
    const int win = w.rec[r] >> 12, j = w.rec[r] & 0xfff;
    if (win < nD) {
      const int a = w.e1[win], c = w.stok[j];
      w.ns[r] = gen_score(w, win, j); w.nh[r] = child_hash(w.ch[a], c); w.nph[r] = w.ch[a];
      w.nl[r] = c; w.nn[r] = w.cn[a] + 1; w.nf[r] = 0; w.ntrel[r] = pack_trel(a, c);
    } else {
      const int s = w.spord[w.rec2[r]];
      const int a = w.spbase[s], x = w.spx[s];
      w.ns[r] = w.spsc[s];
      if (x >= 0) {
        w.nh[r] = child_hash(w.ch[a], x); w.nph[r] = w.ch[a]; w.nl[r] = x; w.nn[r] = w.cn[a] + 1;
      } else {
        w.nh[r] = w.ch[a]; w.nph[r] = w.cph[a]; w.nl[r] = w.cl[a]; w.nn[r] = w.cn[a];
      }
      w.nf[r] = w.spflag[s];
      w.ntrel[r] = pack_trel(w.spsrc[s], w.sptok[s]);
    }
  }
  // threshold on exact scores (winners are in exact rank order): drop a tail
  // whose exact score falls below best_exact - beam_threshold
  __syncwarp();
  if (Hn > 0 && !P.threshold_inf) {
    const double bex = w.ns[0];
    int keepn = 0;
    for (int r0 = 0; r0 < Hn; r0 += 32) {
      const int r = r0 + lane;
      const bool ok = r < Hn && w.ns[r] >= bex - P.beam_threshold && w.ns[r] > -INFINITY;
      keepn += __popc(__ballot_sync(FULL, ok));
    }
    Hn = keepn;
  }
  // reset the token -> S rank map for the next frame
  for (int j = lane; j < P.k; j += 32) w.pos[w.stok[j]] = 0xffff;
  __syncwarp();
  return Hn;
}

// ------------------------------------------------------------------ finalize
__device__ void finalize(Warp& w, int H, int kept) {
  const Params& P = *w.P;
  const int lane = w.lane, u = w.u;
  for (int e = lane; e < H; e += 32) {
    int f = e;
    for (int q = 0; q < e; q++)
      if (w.ch[q] == w.ch[e] && w.cn[q] == w.cn[e]) { f = q; break; }
    w.first[e] = f;
  }
  if (lane == 0) w.misc[0] = 0;
  __syncwarp();
  for (int e = lane; e < H; e += 32) {
    if (w.first[e] != e) continue;
    double sc = w.cs[e];  // entries are in rank order: the first is the payload (decoder.py:794-797)
    for (int q = e + 1; q < H; q++)
      if (w.first[q] == e) sc = merge2_exact(sc, w.cs[q], w.P->merge_max != 0);
    int s = atomicAdd(&w.misc[0], 1);
    w.spsc[s] = sc; w.spbase[s] = e; w.spx[s] = -1; w.spflag[s] = 0;
  }
  __syncwarp();
  const int nF = w.misc[0];
  const int pad = pow2_at_least(nF);
  for (int s = lane; s < pad; s += 32) {
    w.spkey[s] = s < nF ? ord64(w.spsc[s]) : 0ull;
    w.spord[s] = s < nF ? s : 0x7fffffff;
  }
  __syncwarp();
  bitonic_pairs(w.spkey, w.spord, pad, lane);
  fix_tie_runs(w, nF);
  const int nOut = nF < P.nbest ? nF : P.nbest;
  for (int r = lane; r < nOut; r += 32) {
    int s = w.spord[r], e = w.spbase[s];
    int len = w.cn[e];
    size_t o = ((size_t)u * P.nbest + r);
    P.out_score[o] = w.spsc[s];
    P.out_len[o] = len;
    int* tok_out = P.out_tokens + o * P.T_max;
    int* ts_out = P.out_ts ? P.out_ts + o * P.T_max : nullptr;
    int pos = len, slot = e;
    for (int i = kept - 1; i >= 0 && pos > 0; --i) {
      uint32_t rec = P.trellis[((size_t)u * P.T_max + i) * P.beam + slot];
      int tok = trel_tok(rec);
      if (tok >= 0) {
        --pos;
        tok_out[pos] = tok;
        if (ts_out) ts_out[pos] = P.frame_map[(size_t)u * P.T_max + i];
      }
      slot = trel_src(rec);
    }
  }
  if (lane == 0) P.out_count[u] = nOut;
}

}  // namespace

// ------------------------------------------------------------------ kernel
__global__ void __launch_bounds__(256) ctcb_decode_generic_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  Warp w;
  w.P = &P;
  w.lane = lane;
  carve(w, smem + (size_t)wid * P.smem_per_warp, P);
  if (lane == 0)
    for (int s = 0; s < P.ring; s++) mbar_init(&w.mbar[s], 1);
  for (int c = lane; c < P.V; c += 32) w.pos[c] = 0xffff;
  for (int i = lane; i < 2 * kTieCache; i += 32) w.tc_h[i] = 0ull;
  for (int i = lane; i <= kTieCache; i += 32) w.tc_r[i] = 0;
  fence_mbar_init();
  __syncwarp();
  uint32_t n_issue = 0, n_cons = 0;  // ring bookkeeping across utterances
  const uint32_t row_bytes_copy = (uint32_t)P.V * 4u;

  for (;;) {
    int item = 0;
    if (lane == 0) item = atomicAdd(P.counter, 1);
    item = __shfl_sync(FULL, item, 0);
    if (item >= P.B) break;
    const int u = P.order[item];
    w.u = u;
    const int len = P.lens[u];
    if (len <= 0 || len > P.T_max) {
      if (lane == 0) {
        P.status[u] = len == 0 ? kUttEmpty : kUttBadLen;
        P.out_count[u] = 0;
        P.kept[u] = 0;
      }
      continue;
    }
    const float* ubase = P.lp + (size_t)u * P.stride_b;
    int32_t* fmap = P.frame_map + (size_t)u * P.T_max;
    // -- A. blank-skip compaction (warp ballot + prefix popcount)
    int kept = 0;
    for (int t0 = 0; t0 < len; t0 += 32) {
      int t = t0 + lane;
      bool keep = t < len;
      if (keep && P.skip) keep = !(__ldg(ubase + (size_t)t * P.stride_t + P.blank) >= P.cutoff);
      unsigned bal = __ballot_sync(FULL, keep);
      if (keep) fmap[kept + __popc(bal & lanemask_lt())] = t;
      kept += __popc(bal);
    }
    if (lane == 0) P.kept[u] = kept;
    __syncwarp();

    // -- B. frame loop
    if (lane == 0) { w.cs[0] = 0.0; w.ch[0] = kEmptyPrefixHash; w.cph[0] = 0ull; w.cl[0] = -1; w.cn[0] = 0; w.cf[0] = 1; }
    int H = 1;
    w.steps_done = 0;
    auto issue = [&](int i) {
      uint32_t slot = n_issue % (uint32_t)P.ring;
      const float* src = ubase + (size_t)fmap[i] * P.stride_t;
      fence_proxy_async();
      mbar_arrive_expect_tx(&w.mbar[slot], row_bytes_copy);
      tma_bulk_g2s(w.rows + (size_t)slot * P.row_bytes, src, row_bytes_copy, &w.mbar[slot]);
      n_issue++;
    };
    if (P.bulk_ok) {
      const int pre = kept < P.ring - 1 ? kept : P.ring - 1;
      for (int i = 0; i < pre; i++)
        if (lane == 0) issue(i); else n_issue++;
    }
    __syncwarp();
    bool died = false;
    for (int i = 0; i < kept; i++) {
      const float* row;
      if (P.bulk_ok) {
        if (i + P.ring - 1 < kept) {
          if (lane == 0) issue(i + P.ring - 1); else n_issue++;
        }
        uint32_t slot = n_cons % (uint32_t)P.ring;
        mbar_wait(&w.mbar[slot], (n_cons / (uint32_t)P.ring) & 1u);
        n_cons++;
        row = (const float*)(w.rows + (size_t)slot * P.row_bytes);
      } else {
        float* dst = (float*)w.rows;
        const float* src = ubase + (size_t)fmap[i] * P.stride_t;
        for (int c = lane; c < P.V; c += 32) dst[c] = __ldg(src + c);
        __syncwarp();
        row = dst;
      }
      topk(w, row);
      int Hn = beam_step(w, row, H);
      if (Hn == 0) { died = true; break; }
      uint32_t* trow = P.trellis + ((size_t)u * P.T_max + i) * P.beam;
      for (int r = lane; r < Hn; r += 32) trow[r] = w.ntrel[r];
      w.swap_state();
      H = Hn;
      w.steps_done = i + 1;
      __syncwarp();
    }
    if (died) {
      // drain outstanding row copies of this utterance before moving on
      while (n_cons < n_issue) {
        uint32_t slot = n_cons % (uint32_t)P.ring;
        mbar_wait(&w.mbar[slot], (n_cons / (uint32_t)P.ring) & 1u);
        n_cons++;
      }
      if (lane == 0) {  // the dying frame (kept-frame index) goes to out_len[u][0]
        P.status[u] = kUttBeamDied;
        P.out_count[u] = 0;
        P.out_len[(size_t)u * P.nbest] = w.steps_done;
      }
      __syncwarp();
      continue;
    }
    // -- C. finalize
    finalize(w, H, kept);
    if (lane == 0) P.status[u] = kUttOk;
    __syncwarp();
  }
}

// Minimum-slice debug entry: blank-skip compaction + per-frame top-k only
// (one warp per utterance; rows loaded directly).
__global__ void __launch_bounds__(32) ctcb_debug_kernel(const __grid_constant__ Params P, int32_t* out_topk_tok,
                                                        float* out_topk_val, float* out_blank) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x;
  Warp w;
  w.P = &P;
  w.lane = lane;
  w.u = u;
  carve(w, smem, P);
  for (int c = lane; c < P.V; c += 32) w.pos[c] = 0xffff;
  __syncwarp();
  int len = P.lens[u];
  if (len < 0 || len > P.T_max) len = 0;
  const float* ubase = P.lp + (size_t)u * P.stride_b;
  int32_t* fmap = P.frame_map + (size_t)u * P.T_max;
  int kept = 0;
  for (int t0 = 0; t0 < len; t0 += 32) {
    int t = t0 + lane;
    bool keep = t < len;
    if (keep && P.skip) keep = !(__ldg(ubase + (size_t)t * P.stride_t + P.blank) >= P.cutoff);
    unsigned bal = __ballot_sync(FULL, keep);
    if (keep) fmap[kept + __popc(bal & lanemask_lt())] = t;
    kept += __popc(bal);
  }
  if (lane == 0) P.kept[u] = kept;
  __syncwarp();
  float* row = (float*)w.rows;
  for (int i = 0; i < kept; i++) {
    const float* src = ubase + (size_t)fmap[i] * P.stride_t;
    for (int c = lane; c < P.V; c += 32) row[c] = __ldg(src + c);
    __syncwarp();
    topk(w, row);
    size_t o = ((size_t)u * P.T_max + i) * P.k;
    for (int j = lane; j < P.k; j += 32) {
      out_topk_tok[o + j] = w.stok[j];
      out_topk_val[o + j] = w.sval[j];
      w.pos[w.stok[j]] = 0xffff;
    }
    if (lane == 0) out_blank[(size_t)u * P.T_max + i] = row[P.blank];
    __syncwarp();
  }
}

// Longest-first processing order (LPT within one GPU): one block sorts
// (len desc, index asc); falls back to index order for very large batches.
__global__ void ctcb_order_kernel(const int32_t* lens, int B, int32_t* order, int32_t* counter) {
  extern __shared__ uint64_t keys[];
  int n = 1;
  while (n < B) n <<= 1;
  if (threadIdx.x == 0) *counter = 0;
  if (n > 8192) {
    for (int i = threadIdx.x; i < B; i += blockDim.x) order[i] = i;
    return;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (i < B) {
      int l = lens[i];
      uint32_t inv = 0x7fffffffu - (uint32_t)(l < 0 ? 0 : l);
      keys[i] = ((uint64_t)inv << 32) | (uint32_t)i;
    } else {
      keys[i] = ~0ull;
    }
  }
  __syncthreads();
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
        int i = ((t & ~(stride - 1)) << 1) | (t & (stride - 1));
        int j = i + stride;
        uint64_t a = keys[i], b = keys[j];
        bool asc = (i & size) == 0;
        if (asc ? (a > b) : (a < b)) { keys[i] = b; keys[j] = a; }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < B; i += blockDim.x) order[i] = (int32_t)(keys[i] & 0xffffffffu);
}

}  // namespace ctcb
