// Internal launch parameters and the per-warp shared-memory layout, shared by
// the host side (ctcb_api.cu) and the kernels.
#pragma once
#include <cstddef>
#include <cstdint>

namespace ctcb {

// Per-utterance status codes written by the kernels (host maps them to the
// reference's ValueError messages).
enum UttStatus : int32_t {
  kUttOk = 0,
  kUttEmpty = 1,      // len_b == 0: "empty emissions" (decoder.py:117-118)
  kUttBadLen = 2,     // len_b < 0 or len_b > T_max
  kUttBeamDied = 3,   // "beam died" (decoder.py:616-620)
  // input validation (emissions.py:128-150): out_len[u][0] = frame, out_count[u] = token (-1 for 7)
  kUttNonFinite = 5,
  kUttAboveZero = 6,
  kUttNotNormalized = 7,
};

struct Params {
  // input [B, T_max, V] with element strides
  const float* lp;
  long long stride_b, stride_t;
  const int32_t* lens;
  int B, T_max, V, blank;
  // decoder options
  int beam, nbest, k, kpad;  // k = min(2*beam, V-1) kept tokens per frame, kpad = pow2 >= k
  float cutoff;              // drop frame iff lp[t, blank] >= cutoff (+inf: no skipping)
  int skip;                  // cutoff finite
  double beam_threshold;
  int threshold_inf;
  int merge_max;             // merge_mode="max": group max instead of the logadd fold
  int tokK;                  // beam_size_token K (0: full vocabulary; else 1 <= K < V)
  // workspace
  int32_t* frame_map;   // [B, T_max]
  int32_t* kept;        // [B]
  uint32_t* trellis;    // [B, T_max, beam]
  int32_t* status;      // [B]
  int32_t* order;       // [B] utterance processing order (longest first)
  int32_t* counter;     // [1] work claim counter
  int32_t* seqbuf;      // [B, 3, T_max + 1] scratch: exact-tie token sequences, backtrace staging
  uint8_t* anc;         // [B, n_chunks, 16] fast path: ancestor slot at each trellis checkpoint
  // outputs
  int32_t* out_tokens;  // [B, nbest, T_max]
  int32_t* out_ts;      // [B, nbest, T_max] or null
  int32_t* out_len;     // [B, nbest]
  double* out_score;    // [B, nbest]
  int32_t* out_count;   // [B]
  // staging
  int ring;             // row ring depth
  int row_bytes;        // smem bytes per staged row (multiple of 16)
  int bulk_ok;          // rows may be staged with cp.async.bulk
  int warps_per_block;
  int smem_per_warp;
  int n_chunks;         // ceil(T_max / kChunk)
  unsigned long long* dbg;  // [8] debug counters (kDbg*)
  int precomp;              // top-k lists precomputed by ctcb_topk_kernel
  int32_t* topk_tok;        // [B, T_max, k] (precomp mode)
  float* topk_val;          // [B, T_max, k]
  int32_t* rowoff;          // [B + 1] exclusive prefix sums of kept (precomp mode)
  // overlapped precomp mode: per-list ready flags [B, T_max] (zeroed before the
  // top-k kernel, set with release semantics after each list is written); the walk
  // is launched as a programmatic dependent and waits on them.  null = the lists
  // are complete before the walk starts (flattened split, plain stream order).
  uint32_t* ready;
  // fused search (ctcb_set_lm / ctcb_set_silence): token-level LM and silence bonus
  const double* lm_score;   // [S, V] natural-log LM score of token c after context s, or null (no LM)
  const int32_t* lm_next;   // [S, V] successor context
  const double* lm_fin;     // [S] score of "</s>"
  const double* lm_wmax;    // [S] max_c weight * lm_score[s, c] (pruning bound)
  const double* lm_wx;      // [S] the same maximum over the explicit tokens of s
  const double* lm_A;       // [S] accumulated backoff: other tokens score A_s + lm_score[0, c]
  const double* lm_wu;      // [V] weight * lm_score[0, c] (-inf: blank / silence)
  const uint32_t* lm_xbits; // [S, ceil(V/32)] explicit-token bitmap
  int lm_start;             // start context
  double lm_weight;
  int sil;                  // silence token (-1: none)
  double sil_score;
  double* out_lm;           // [B, nbest] LM total of each hypothesis, or null
  // input validation fused into the row staging (ctcb_set_validate)
  int validate;             // 0 off, 1 strict (normalisation too), 2 finite / <= 1e-4 only
  unsigned long long* vkey; // [B] smallest offender key (vkey_make) seen, ~0 = none
  int32_t* vdone;           // [B] leading kept frames the decode kernel checked
  int vfused;               // the decode kernel wrote vdone (else every frame is checked after it)
  unsigned long long* utt_trace;  // diagnostics (CTCB_UTT_TRACE): [B, 2] {smid << 48 | global warp, start ns}, end ns
};

// Fused search limits.
constexpr int kFusedMaxBeam = 128;
constexpr int kUttOverflow = 4;  // fused search: too many near-tied candidates at the beam cut

// Device copy of a flattened backoff n-gram model (ctcb_lm_t).
struct LmModel {
  int order, device;
  int64_t n, cap, n_states;
  int32_t *words, *lengths;     // [n, order], [n]
  double *logprob, *backoff;    // [n]
  int32_t* slots;               // [cap] open-addressing table: entry index or -1
  int32_t* state_entry;         // [n_states] entry of context state s (-1: the empty context)
  int32_t* entry_state;         // [n] context state of an entry (-1: top-order n-gram)
  int start_state, eos;
};
// Dense fusion tables of one handle: S x V scores / successors, finish scores, bounds.
struct LmTables {
  double* score;
  int32_t* next;
  double* fin;
  double* wmax;
  double* wx;
  double* A;
  double* wu;
  uint32_t* xbits;
  int64_t n_states;
  int start;
};
int lm_model_create(int order, int64_t n, const int32_t* words, const int32_t* lengths, const double* logprob,
                    const double* backoff, const int32_t* start, int start_len, int eos, int device, LmModel** out,
                    const char** err);
void lm_model_destroy(LmModel* m);
int lm_tables_build(const LmModel* m, const int32_t* token_word, int V, double weight, LmTables* t, const char** err);
void lm_tables_free(LmTables* t);
size_t fused_smem_per_warp(int beam, int V, int ring, int row_bytes);
const void* fused_kernel_fn();

// Record the error message of a failing C-ABI call (ctcb_last_error).
int set_error(int code, const char* msg);

enum DbgCounter {
  kDbgTies = 0, kDbgExactTies = 1, kDbgMaterialize = 2, kDbgMatSteps = 3, kDbgRadix = 4, kDbgFrames = 5, kDbgTopkFix = 6, kDbgOneshotFallback = 7
};

// Fast path (beam <= kFastBeam): trellis checkpoint interval.
constexpr int kFastBeam = 16;
constexpr int kChunk = 16;
constexpr int kTieCache = 32;
// Fast path with a compile-time shared-memory layout: V <= kSmallV, ring 2.
constexpr int kSmallV = 512;
constexpr int kSmallRowBytes = kSmallV * 4;
#ifndef CTCB_TOPK_RING
#define CTCB_TOPK_RING 2
#endif
constexpr int kTopkRing = CTCB_TOPK_RING;  // row ring depth of ctcb_topk_kernel

// Byte offsets of the per-warp shared memory of the fast decode kernel.
struct FastLayout {
  size_t rows, mbar, cand, sval, stok, excl, rec_i, tie_sc, tie_i, hs, hl, tc_h, tc_r, gkey, hsc, hp2, dlane, dA, dgv, ring, hist,
      posmap, wp, ckey, cidx, slot_rec, dG, total;
};
__host__ __device__ constexpr inline FastLayout make_fast_layout(int V, int ring, int row_bytes) {
  FastLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes, size_t align) {
    o = (o + align - 1) / align * align;
    size_t r = o;
    o += bytes;
    return r;
  };
  L.rows = take((size_t)ring * row_bytes, 128);
  L.mbar = take((size_t)ring * 8, 8);
  L.cand = take(64 * 8, 16);  // 16-B aligned: also the rank-sort scratch (uint4 reads)
  L.tie_sc = take(32 * 8, 8);
  L.hs = take(16 * 8, 8);
  L.sval = take(32 * 4, 4);
  L.stok = take(32 * 4, 4);
  L.excl = take(16 * 4, 4);
  L.rec_i = take(48 * 4, 4);       // merge record per new entry: winning lane | item << 8 (+32 scratch)
  L.tie_i = take(32 * 4 * 4, 4);   // 4 ints per tie candidate
  L.hl = take(16 * 4, 4);          // entry lengths (tie slow path)
  L.tc_h = take(2 * kTieCache * 8, 8);  // tie-order cache: (seq hash a, seq hash b)
  L.tc_r = take((kTieCache + 1) * 4, 4);  // cached order (-1/+1) + replacement cursor
  L.gkey = take(256 * 4, 4);       // radix-select histogram (fallback only)
  L.hsc = take(16 * 8, 8);         // entry scores (tie slow path)
  L.hp2 = take(16 * 4, 4);         // partner entry of each first entry (tie slow path)
  L.dA = take(16 * 8, 8);          // per distinct prefix: A = logaddexp of its entries
  L.dlane = take(16 * 4, 4);       // per distinct prefix: its first entry lane
  L.dgv = take(16 * 4, 4);         // per distinct prefix: valid append positions in S
  L.ring = take((size_t)kChunk * 16 * 4, 4);
  L.hist = L.gkey;
  L.wp = take(32 * 8, 8);          // per S position: floor(v * 2^32 / R)
  L.ckey = take(64 * 4, 4);        // top-k survivors: 32-bit sort keys
  L.cidx = take(64 * 2, 2);        //                  token indices (index order)
  L.slot_rec = take(64 * 4, 4);    // one-shot selection: merge record per candidate slot
  L.dG = take(16 * 8, 8);          // per distinct prefix: floor((A - base) * 2^32 / R)
  L.posmap = take((size_t)V, 1);
  L.total = (o + 127) / 128 * 128;
  return L;
}

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Large-beam block kernel (ctcb_block.cu): one CTA per utterance.
constexpr int kBlockMaxBeam = 128;
constexpr int kBlockMaxV = 2048;
constexpr int kBlockCands = 2048;  // candidate keys per frame (specials + quota appends)
constexpr int kBlockRun = 512;     // longest near-tie run re-sorted exactly
constexpr int kBlockTieCache = 512;  // hashed sequence-order cache entries (power of 2)
struct BlockLayout {
  size_t rows, mbar, cs, ns, lA, spsc, ch, cph, nh, nph, skey, ckey, htk, tc_h, cl, cn, cf, nl, nn, nf, htf, hslot,
      first, dpi, pd, e1, e2, qoff, spbase, spx, spflag, spsrc, sptok, misc, tc_r, rec, ord, runbuf, runsc, ntrel, excl, hist, crec,
      sval, stok, pos, total;
  int kw, kpad, ts, ncap;
};
__host__ __device__ constexpr inline BlockLayout make_block_layout(int beam, int kpad, int V, int row_bytes) {
  BlockLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes, size_t align) {
    o = (o + align - 1) / align * align;
    size_t r = o;
    o += bytes;
    return r;
  };
  const size_t B = (size_t)beam, S = 3 * B;
  int ts = 1;
  while (ts < 2 * beam) ts <<= 1;
  L.kpad = kpad;
  L.kw = (kpad + 31) / 32;
  L.ts = ts;
  L.ncap = kBlockCands;
  const size_t small = B + 1 > 16 ? B + 1 : 16;
  L.rows = take(2 * (size_t)row_bytes, 128);
  L.mbar = take(16, 8);
  L.cs = take(8 * B, 8); L.ns = take(8 * B, 8); L.lA = take(8 * B, 8); L.spsc = take(8 * S, 8);
  L.ch = take(8 * B, 8); L.cph = take(8 * B, 8); L.nh = take(8 * B, 8); L.nph = take(8 * B, 8);
  L.skey = take(8 * (size_t)(kpad > 512 ? kpad : 512), 8);  // also sort scratch
  L.ckey = take(8 * (size_t)L.ncap, 8); L.htk = take(8 * (size_t)ts, 8);
  L.tc_h = take(8 * 2 * kBlockTieCache, 8);
  L.cl = take(4 * B, 4); L.cn = take(4 * B, 4); L.cf = take(4 * B, 4);
  L.nl = take(4 * B, 4); L.nn = take(4 * B, 4); L.nf = take(4 * B, 4);
  L.htf = take(4 * (size_t)ts, 4); L.hslot = take(4 * B, 4); L.first = take(4 * B, 4); L.dpi = take(4 * B, 4);
  L.pd = take(4 * B, 4); L.e1 = take(4 * B, 4); L.e2 = take(4 * B, 4); L.qoff = take(4 * small, 4);
  L.spbase = take(4 * S, 4); L.spx = take(4 * S, 4); L.spflag = take(4 * S, 4); L.spsrc = take(4 * S, 4);
  L.sptok = take(4 * S, 4); L.misc = take(4 * 16, 4); L.tc_r = take(kBlockTieCache, 4);
  L.rec = take(4 * small, 4);
  L.ord = take(4 * (size_t)L.ncap, 16);  // also the survivor key buffer (u64, read in 16-B pairs)
  L.runbuf = take(4 * kBlockRun, 4); L.runsc = take(8 * kBlockRun, 8);
  L.ntrel = take(4 * B, 4); L.excl = take(4 * B * (size_t)L.kw, 4); L.hist = take(4 * 256, 4);
  L.crec = take(4 * (size_t)L.ncap, 4);
  L.sval = take(4 * (size_t)kpad, 4); L.stok = take(4 * (size_t)kpad, 4); L.pos = take(2 * (size_t)V, 2);
  L.total = (o + 127) / 128 * 128;
  return L;
}

// Two-utterances-per-warp kernel (ctcb_pair.cu): per-half shared memory.
constexpr int kPairRing = 2;
struct PairLayout {
  size_t rows, mbar, sval, stok, wp, cidx, posmap, excl, rec, hs, hl, hsc, hp2, tie_sc, tie_i, tc_h, tc_r, tring, total;
};
__host__ __device__ constexpr inline PairLayout make_pair_layout() {
  PairLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes, size_t align) {
    o = (o + align - 1) / align * align;
    size_t r = o;
    o += bytes;
    return r;
  };
  L.rows = take((size_t)kPairRing * kSmallRowBytes, 128);
  L.mbar = take((size_t)kPairRing * 8, 8);
  L.wp = take(32 * 8, 8);
  L.hs = take(16 * 8, 8);
  L.hsc = take(16 * 8, 8);
  L.tie_sc = take(64 * 8, 8);      // also the 64-bit keys of the top-k exactness fix
  L.tc_h = take(2 * kTieCache * 8, 8);
  L.sval = take(32 * 4, 4);
  L.stok = take(32 * 4, 4);
  L.excl = take(16 * 4, 4);
  L.rec = take(32 * 4, 4);
  L.hl = take(16 * 4, 4);
  L.hp2 = take(16 * 4, 4);
  L.tie_i = take(32 * 4 * 4, 4);
  L.tc_r = take((kTieCache + 1) * 4, 4);
  L.cidx = take(64 * 2, 2);
  L.tring = take((size_t)kChunk * 16 * 2, 2);
  L.posmap = take((size_t)kSmallV, 1);
  L.total = (o + 127) / 128 * 128;
  return L;
}


// Byte offsets of the per-warp shared-memory arrays of the generic decode kernel.
struct WarpLayout {
  size_t rows, mbar;
  size_t cur_score, cur_hash, cur_phash, cur_last, cur_len, cur_flag;
  size_t nxt_score, nxt_hash, nxt_phash, nxt_last, nxt_len, nxt_flag, nxt_trel;
  size_t first, dpi, pd, dp_e1, dp_e2, excl, head_j, head_sc;
  size_t skey, sval, stok, pos;
  size_t sp_sc, sp_key, sp_ord, sp_base, sp_x, sp_flag, sp_src, sp_tok;
  size_t hist, misc, tc_h, tc_r, htk, htf, hslot, rec, rec2, hkey, lA;
  size_t total;
  int kw, sp_cap, sp_pad, ts;
};

__host__ __device__ inline int pow2_at_least(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

__host__ __device__ inline WarpLayout make_layout(int beam, int kpad, int V, int ring, int row_bytes) {
  WarpLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes, size_t align) {
    o = align_up(o, align);
    size_t r = o;
    o += bytes;
    return r;
  };
  L.kw = (kpad + 31) / 32;
  L.sp_cap = 3 * beam;
  L.sp_pad = pow2_at_least(L.sp_cap);
  L.rows = take((size_t)ring * row_bytes, 128);
  L.mbar = take((size_t)ring * 8, 8);
  L.cur_score = take(8 * (size_t)beam, 8);
  L.cur_hash = take(8 * (size_t)beam, 8);
  L.cur_phash = take(8 * (size_t)beam, 8);
  L.nxt_score = take(8 * (size_t)beam, 8);
  L.nxt_hash = take(8 * (size_t)beam, 8);
  L.nxt_phash = take(8 * (size_t)beam, 8);
  L.head_sc = take(8 * (size_t)beam, 8);
  L.skey = take(8 * (size_t)kpad, 8);
  L.sp_sc = take(8 * (size_t)L.sp_cap, 8);
  L.sp_key = take(8 * (size_t)L.sp_pad, 8);
  L.cur_last = take(4 * (size_t)beam, 4);
  L.cur_len = take(4 * (size_t)beam, 4);
  L.cur_flag = take(4 * (size_t)beam, 4);
  L.nxt_last = take(4 * (size_t)beam, 4);
  L.nxt_len = take(4 * (size_t)beam, 4);
  L.nxt_flag = take(4 * (size_t)beam, 4);
  L.nxt_trel = take(4 * (size_t)beam, 4);
  L.first = take(4 * (size_t)beam, 4);
  L.dpi = take(4 * (size_t)beam, 4);
  L.pd = take(4 * (size_t)beam, 4);
  L.dp_e1 = take(4 * (size_t)beam, 4);
  L.dp_e2 = take(4 * (size_t)beam, 4);
  L.head_j = take(4 * (size_t)beam, 4);
  L.excl = take(4 * (size_t)beam * L.kw, 4);
  L.sval = take(4 * (size_t)kpad, 4);
  L.stok = take(4 * (size_t)kpad, 4);
  L.sp_ord = take(4 * (size_t)L.sp_pad, 4);
  L.sp_base = take(4 * (size_t)L.sp_cap, 4);
  L.sp_x = take(4 * (size_t)L.sp_cap, 4);
  L.sp_flag = take(4 * (size_t)L.sp_cap, 4);
  L.sp_src = take(4 * (size_t)L.sp_cap, 4);
  L.sp_tok = take(4 * (size_t)L.sp_cap, 4);
  L.hist = take(4 * 256, 4);
  L.misc = take(4 * 16, 4);
  L.tc_h = take(2 * kTieCache * 8, 8);
  L.tc_r = take((kTieCache + 1) * 4, 4);
  L.ts = pow2_at_least(2 * beam);
  L.htk = take(8 * (size_t)L.ts, 8);
  L.htf = take(4 * (size_t)L.ts, 4);
  L.hslot = take(4 * (size_t)beam, 4);
  L.rec = take(4 * (size_t)beam, 4);
  L.rec2 = take(4 * (size_t)beam, 4);
  L.hkey = take(4 * ((size_t)beam + 1), 4);
  L.lA = take(8 * (size_t)beam, 8);
  L.pos = take(2 * (size_t)V, 2);
  L.total = align_up(o, 128);
  return L;
}

}  // namespace ctcb
