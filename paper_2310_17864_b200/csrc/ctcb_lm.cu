// Token-level LM fusion and the silence bonus on the GPU (ctcforge
// decoder.py:178-259, :467-486, :753-817; lm.py:229-270).
//
// 1. Model upload (lm_model_create): the flattened backoff model (n-gram word
//    ids, natural-log logprob / backoff) plus an open-addressing table over
//    n-gram tuples, built on the host and copied to the device.  Contexts are
//    interned as states: 0 = (), then every n-gram shorter than the order.
// 2. Table build (lm_tables_build): one thread per (context state, token)
//    evaluates the Katz backoff score and the shrunk successor context with
//    device hash probes (lm.py:247-270), giving the dense S x V score /
//    successor tables that the reference builds lazily per context
//    (_TokenContexts, decoder.py:178-259); then finish scores ("</s>") and
//    per-context bounds max_c w * score.
// 3. Fused search (ctcb_decode_fused_kernel): one warp per utterance.  With an
//    LM the best appends of a prefix are no longer the best emissions, so every
//    (prefix, token) pair is a candidate: lanes scan the tokens of each prefix
//    with a per-prefix emission cut derived from the current beam bound (the
//    LM table row is read only for candidates that can still enter the beam),
//    keep a per-lane top-`beam` list, and a k-way extraction over the lane
//    lists finds the beam cut.  Candidates within a tolerance of the cut get
//    exact scores (the reference's per-candidate sums and left logaddexp fold)
//    and are ranked exactly (score desc, token sequence asc, flag asc).
//    Blank / repeat merges are formed analytically as in the generic kernel.
#include <cfloat>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/ctcb.h"
#include "ctcb_common.cuh"
#include "ctcb_internal.h"

namespace ctcb {

// ------------------------------------------------------------------ n-gram table
namespace {
constexpr double kOovPenalty = -20.0;  // lm.py:22-24
constexpr int kMaxOrder = 8;

__host__ __device__ inline uint64_t ng_mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33; return x;
}
__host__ __device__ inline uint64_t ng_hash(const int32_t* ids, int n) {
  uint64_t h = 0x84222325cbf29ce4ull ^ (uint64_t)n;
  for (int i = 0; i < n; i++) h = ng_mix(h ^ ((uint64_t)(uint32_t)ids[i] * 0x9e3779b97f4a7c15ull));
  return h;
}

struct NgView {
  int order;
  uint64_t mask;
  const int32_t *words, *lengths, *slots, *entry_state, *state_entry;
  const double *logprob, *backoff;
};

__device__ int ng_find(const NgView& m, const int32_t* ids, int n) {
  if (n == 0) return -1;
  uint64_t i = ng_hash(ids, n) & m.mask;
  for (;;) {
    const int e = m.slots[i];
    if (e < 0) return -1;
    if (m.lengths[e] == n) {
      bool eq = true;
      for (int j = 0; j < n && eq; j++) eq = m.words[(size_t)e * m.order + j] == ids[j];
      if (eq) return e;
    }
    i = (i + 1) & m.mask;
  }
}

// lm.py:247-262 (ctx already holds at most order-1 words)
__device__ double ng_backoff(const NgView& m, const int32_t* ctx_in, int n, int32_t wid) {
  int32_t ng[kMaxOrder];
  double acc = 0.0;
  int off = 0;
  for (;;) {
    for (int j = 0; j < n; j++) ng[j] = ctx_in[off + j];
    ng[n] = wid;
    const int e = ng_find(m, ng, n + 1);
    if (e >= 0) return acc + m.logprob[e];
    if (n == 0) return acc + kOovPenalty;
    const int ce = ng_find(m, ctx_in + off, n);
    if (ce >= 0) acc += m.backoff[ce];
    off++;
    n--;
  }
}

__global__ void ctcb_lm_table_kernel(NgView m, const int32_t* __restrict__ token_word, int V, long long S,
                                     double* __restrict__ score, int32_t* __restrict__ next) {
  const long long total = S * V;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int s = (int)(i / V), c = (int)(i % V);
    const int wid = token_word[c];
    if (wid == -2) { score[i] = 0.0; next[i] = s; continue; }    // blank / silence: identity rows
    if (wid < 0) { score[i] = kOovPenalty; next[i] = 0; continue; }  // OOV without <unk>: ((), -20)
    int32_t ctx[kMaxOrder];
    int n = 0;
    const int e0 = m.state_entry[s];
    if (e0 >= 0) {
      n = m.lengths[e0];
      for (int j = 0; j < n; j++) ctx[j] = m.words[(size_t)e0 * m.order + j];
    }
    score[i] = ng_backoff(m, ctx, n, wid);
    if (m.order == 1) { next[i] = 0; continue; }
    // successor: (ctx + (wid,))[-(order-1):], shrunk to a known context (lm.py:239-241, :265-270)
    ctx[n] = wid;
    int len = n + 1, off = 0;
    if (len > m.order - 1) { off = len - (m.order - 1); len = m.order - 1; }
    int st = 0;
    while (len > 0) {
      const int e = ng_find(m, ctx + off, len);
      if (e >= 0) { st = m.entry_state[e]; break; }
      off++;
      len--;
    }
    next[i] = st;
  }
}

__global__ void ctcb_lm_finish_kernel(NgView m, int eos, long long S, double* __restrict__ fin) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < S; s += (long long)gridDim.x * blockDim.x) {
    if (eos < 0) { fin[s] = kOovPenalty; continue; }
    int32_t ctx[kMaxOrder];
    int n = 0;
    const int e0 = m.state_entry[s];
    if (e0 >= 0) {
      n = m.lengths[e0];
      for (int j = 0; j < n; j++) ctx[j] = m.words[(size_t)e0 * m.order + j];
    }
    fin[s] = ng_backoff(m, ctx, n, eos);
  }
}

// per context: max_c weight * score[s, c] over word tokens (the products the
// search adds; blank and silence, identity columns, are handled separately)
__global__ void ctcb_lm_bound_kernel(const double* __restrict__ score, const int32_t* __restrict__ token_word, int V,
                                     double w, double* __restrict__ wmax) {
  const long long s = blockIdx.x;
  double mx = -INFINITY;
  for (int c = threadIdx.x; c < V; c += blockDim.x)
    if (token_word[c] != -2) mx = fmax(mx, w * score[s * V + c]);
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    if (threadIdx.x == 0) wmax[s] = mx;
  }
}

// per context: the accumulated backoff A_s of a token with no explicit n-gram
// above the unigram (the _backoff_score walk with no early hit, lm.py:247-262).
// Such a token scores exactly A_s + U[c] (U = the empty context's row).
__global__ void ctcb_lm_backoff_kernel(NgView m, long long S, double* __restrict__ A) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < S; s += (long long)gridDim.x * blockDim.x) {
    int32_t ctx[kMaxOrder];
    int n = 0;
    const int e0 = m.state_entry[s];
    if (e0 >= 0) {
      n = m.lengths[e0];
      for (int j = 0; j < n; j++) ctx[j] = m.words[(size_t)e0 * m.order + j];
    }
    double acc = 0.0;
    for (int off = 0; off < n; off++) {
      const int ce = ng_find(m, ctx + off, n - off);
      if (ce >= 0) acc += m.backoff[ce];
    }
    A[s] = acc;
  }
}

// explicit-token bitmap (bit c of context s: a word token whose score is not
// A_s + U[c]), the maximum of weight * score over those tokens, and
// weight * U[c] (-inf for blank / silence)
__global__ void ctcb_lm_explicit_kernel(const double* __restrict__ score, const int32_t* __restrict__ token_word,
                                        const double* __restrict__ A, int V, double w, uint32_t* __restrict__ xbits,
                                        double* __restrict__ wx) {
  const long long s = blockIdx.x;
  const int W = (V + 31) / 32;
  const double as = A[s];
  double mx = -INFINITY;
  for (int wi = threadIdx.x >> 5; wi < W; wi += blockDim.x >> 5) {
    const int c = wi * 32 + (threadIdx.x & 31);
    bool x = false;
    if (c < V && token_word[c] != -2) {
      const double l = score[s * V + c];
      x = l != as + score[c];
      if (x) mx = fmax(mx, w * l);
    }
    const unsigned bits = __ballot_sync(FULL, x);
    if ((threadIdx.x & 31) == 0) xbits[s * W + wi] = bits;
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
    if (threadIdx.x == 0) wx[s] = mx;
  }
}

__global__ void ctcb_lm_wu_kernel(const double* __restrict__ score, const int32_t* __restrict__ token_word, int V,
                                  double w, double* __restrict__ wu) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < V; c += gridDim.x * blockDim.x)
    wu[c] = token_word[c] == -2 ? -INFINITY : w * score[c];
}

NgView view_of(const LmModel* m) {
  NgView v;
  v.order = m->order;
  v.mask = (uint64_t)m->cap - 1;
  v.words = m->words;
  v.lengths = m->lengths;
  v.slots = m->slots;
  v.entry_state = m->entry_state;
  v.state_entry = m->state_entry;
  v.logprob = m->logprob;
  v.backoff = m->backoff;
  return v;
}
}  // namespace

int lm_model_create(int order, int64_t n, const int32_t* words, const int32_t* lengths, const double* logprob,
                    const double* backoff, const int32_t* start, int start_len, int eos, int device, LmModel** out,
                    const char** err) {
  *out = nullptr;
  if (order < 1 || order > kMaxOrder) { *err = "LM order must be in [1, 8]"; return CTCB_ERR_UNSUPPORTED; }
  if (n < 0 || n > (int64_t)1 << 30) { *err = "invalid n-gram count"; return CTCB_ERR_ARG; }
  if (n > 0 && (!words || !lengths || !logprob || !backoff)) { *err = "NULL n-gram arrays"; return CTCB_ERR_ARG; }
  if (start_len < 0 || start_len > order - 1 || (start_len > 0 && !start)) { *err = "invalid start context"; return CTCB_ERR_ARG; }
  for (int64_t i = 0; i < n; i++) {
    if (lengths[i] < 1 || lengths[i] > order) { *err = "n-gram length out of range [1, order]"; return CTCB_ERR_ARG; }
    for (int j = 0; j < lengths[i]; j++)
      if (words[i * order + j] < 0) { *err = "negative word id"; return CTCB_ERR_ARG; }
  }
  // host open-addressing table over tuples; a repeated tuple keeps its last row (dict assignment)
  int64_t cap = 16;
  while (cap < 2 * n + 16) cap <<= 1;
  std::vector<int32_t> slots((size_t)cap, -1);
  std::vector<int32_t> entry_state((size_t)(n > 0 ? n : 1), -1);
  const uint64_t mask = (uint64_t)cap - 1;
  auto find_slot = [&](const int32_t* ids, int len) -> int64_t {
    uint64_t i = ng_hash(ids, len) & mask;
    for (;;) {
      const int32_t e = slots[i];
      if (e < 0) return (int64_t)i;
      if (lengths[e] == len && memcmp(words + (size_t)e * order, ids, (size_t)len * 4) == 0) return (int64_t)i;
      i = (i + 1) & mask;
    }
  };
  for (int64_t i = 0; i < n; i++) slots[find_slot(words + i * order, lengths[i])] = (int32_t)i;
  std::vector<int32_t> state_entry(1, -1);
  for (int64_t i = 0; i < n; i++) {
    if (lengths[i] >= order) continue;
    if (slots[find_slot(words + i * order, lengths[i])] != (int32_t)i) continue;  // superseded duplicate
    entry_state[i] = (int32_t)state_entry.size();
    state_entry.push_back((int32_t)i);
  }
  int start_state = 0;
  for (int len = start_len, off = 0; len > 0; len--, off++) {  // _shrink_to_known of the start context
    const int32_t e = slots[find_slot(start + off, len)];
    if (e >= 0) { start_state = entry_state[e]; break; }
  }
  LmModel* m = new LmModel();
  m->order = order;
  m->device = device;
  m->n = n;
  m->cap = cap;
  m->n_states = (int64_t)state_entry.size();
  m->start_state = start_state;
  m->eos = eos;
  const size_t nn = (size_t)(n > 0 ? n : 1);
  cudaError_t e = cudaSetDevice(device);
  auto up = [&](void** dst, const void* src, size_t bytes) {
    if (e != cudaSuccess) return;
    e = cudaMalloc(dst, bytes > 0 ? bytes : 16);
    if (e == cudaSuccess && bytes && src) e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
  };
  up((void**)&m->words, words, (size_t)n * order * 4);
  up((void**)&m->lengths, lengths, (size_t)n * 4);
  up((void**)&m->logprob, logprob, (size_t)n * 8);
  up((void**)&m->backoff, backoff, (size_t)n * 8);
  up((void**)&m->slots, slots.data(), (size_t)cap * 4);
  up((void**)&m->entry_state, entry_state.data(), nn * 4);
  up((void**)&m->state_entry, state_entry.data(), state_entry.size() * 4);
  if (e != cudaSuccess) {
    lm_model_destroy(m);
    *err = cudaGetErrorString(e);
    return CTCB_ERR_CUDA;
  }
  *out = m;
  return CTCB_OK;
}

void lm_model_destroy(LmModel* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  cudaFree(m->words);
  cudaFree(m->lengths);
  cudaFree(m->logprob);
  cudaFree(m->backoff);
  cudaFree(m->slots);
  cudaFree(m->entry_state);
  cudaFree(m->state_entry);
  delete m;
}

int lm_tables_build(const LmModel* m, const int32_t* token_word, int V, double weight, LmTables* t, const char** err) {
  memset(t, 0, sizeof(*t));
  const long long S = m->n_states;
  const size_t need = (size_t)S * V * 12 + (size_t)S * ((V + 31) / 32) * 4 + (size_t)S * 32 + (size_t)V * 12;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) { *err = "cudaMemGetInfo failed"; return CTCB_ERR_CUDA; }
  if (need > free_b / 2) { *err = "LM tables (contexts x tokens) do not fit in half the free device memory"; return CTCB_ERR_UNSUPPORTED; }
  int32_t* dtw = nullptr;
  cudaError_t e = cudaMalloc(&t->score, (size_t)S * V * 8);
  if (e == cudaSuccess) e = cudaMalloc(&t->next, (size_t)S * V * 4);
  if (e == cudaSuccess) e = cudaMalloc(&t->fin, (size_t)S * 8);
  if (e == cudaSuccess) e = cudaMalloc(&t->wmax, (size_t)S * 8);
  if (e == cudaSuccess) e = cudaMalloc(&t->wx, (size_t)S * 8);
  if (e == cudaSuccess) e = cudaMalloc(&t->A, (size_t)S * 8);
  if (e == cudaSuccess) e = cudaMalloc(&t->wu, (size_t)V * 8);
  if (e == cudaSuccess) e = cudaMalloc(&t->xbits, (size_t)S * ((V + 31) / 32) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&dtw, (size_t)V * 4);
  if (e == cudaSuccess) e = cudaMemcpy(dtw, token_word, (size_t)V * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    const NgView v = view_of(m);
    long long blocks = (S * V + 255) / 256;
    if (blocks > 65536) blocks = 65536;
    ctcb_lm_table_kernel<<<(int)blocks, 256>>>(v, dtw, V, S, t->score, t->next);
    e = cudaGetLastError();
    if (e == cudaSuccess) {
      long long fb = (S + 255) / 256;
      ctcb_lm_finish_kernel<<<(int)(fb > 65536 ? 65536 : fb), 256>>>(v, m->eos, S, t->fin);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
      ctcb_lm_bound_kernel<<<(unsigned)S, 256>>>(t->score, dtw, V, weight, t->wmax);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
      long long fb = (S + 255) / 256;
      ctcb_lm_backoff_kernel<<<(int)(fb > 65536 ? 65536 : fb), 256>>>(v, S, t->A);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
      ctcb_lm_explicit_kernel<<<(unsigned)S, 256>>>(t->score, dtw, t->A, V, weight, t->xbits, t->wx);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) {
      ctcb_lm_wu_kernel<<<(V + 255) / 256, 256>>>(t->score, dtw, V, weight, t->wu);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  cudaFree(dtw);
  if (e != cudaSuccess) {
    lm_tables_free(t);
    *err = cudaGetErrorString(e);
    return CTCB_ERR_CUDA;
  }
  t->n_states = S;
  t->start = m->start_state;
  return CTCB_OK;
}

void lm_tables_free(LmTables* t) {
  cudaFree(t->score);
  cudaFree(t->next);
  cudaFree(t->fin);
  cudaFree(t->wmax);
  cudaFree(t->wx);
  cudaFree(t->A);
  cudaFree(t->wu);
  cudaFree(t->xbits);
  memset(t, 0, sizeof(*t));
}

// ------------------------------------------------------------------ fused search
namespace {

struct FusedLayout {
  size_t rows, mbar, cs, clm, ch, cph, cn, cl, cf, cst, ns, nlm, nh, nph, nn, nl, nf, nst, ntrel;
  size_t first, dpi, e1, e2, f1, pd, lA, vmin, vo1, vo2, exd, exc;
  size_t sp_sc, sp_lm, sp_base, sp_x, sp_flag, sp_src, sp_tok, sp_st;
  size_t lk, li, c_key, c_ord, c_id, c_sc, c_lm, c_src, c_st, excl, plist, seed, hist, misc;
  size_t total;
  int cc, cc_pad, sp_cap, excl_words;
};

__host__ __device__ inline FusedLayout make_fused_layout(int beam, int V, int ring, int row_bytes) {
  FusedLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes, size_t align) {
    o = (o + align - 1) / align * align;
    size_t r = o;
    o += bytes;
    return r;
  };
  const size_t B = (size_t)beam;
  L.sp_cap = 3 * beam;
  L.cc = 2 * beam + 32;
  L.cc_pad = pow2_at_least(L.cc);
  L.excl_words = (V + 31) / 32;
  L.rows = take((size_t)ring * row_bytes, 128);
  L.mbar = take((size_t)ring * 8, 8);
  L.cs = take(8 * B, 8); L.clm = take(8 * B, 8); L.ch = take(8 * B, 8); L.cph = take(8 * B, 8);
  L.ns = take(8 * B, 8); L.nlm = take(8 * B, 8); L.nh = take(8 * B, 8); L.nph = take(8 * B, 8);
  L.lA = take(8 * B, 8); L.vmin = take(8 * B, 8); L.vo1 = take(8 * B, 8); L.vo2 = take(8 * B, 8);
  L.sp_sc = take(8 * (size_t)L.sp_cap, 8); L.sp_lm = take(8 * (size_t)L.sp_cap, 8);
  L.lk = take(8 * 32 * B, 8);
  L.c_key = take(8 * (size_t)L.cc_pad, 8);
  L.c_sc = take(8 * (size_t)L.cc, 8);
  L.c_lm = take(8 * (size_t)L.cc, 8);
  L.cn = take(4 * B, 4); L.cl = take(4 * B, 4); L.cf = take(4 * B, 4); L.cst = take(4 * B, 4);
  L.nn = take(4 * B, 4); L.nl = take(4 * B, 4); L.nf = take(4 * B, 4); L.nst = take(4 * B, 4);
  L.ntrel = take(4 * B, 4);
  L.first = take(4 * B, 4); L.dpi = take(4 * B, 4); L.e1 = take(4 * B, 4); L.e2 = take(4 * B, 4);
  L.f1 = take(4 * B, 4); L.pd = take(4 * B, 4); L.exd = take(4 * B, 4); L.exc = take(4 * B, 4);
  L.sp_base = take(4 * (size_t)L.sp_cap, 4); L.sp_x = take(4 * (size_t)L.sp_cap, 4);
  L.sp_flag = take(4 * (size_t)L.sp_cap, 4); L.sp_src = take(4 * (size_t)L.sp_cap, 4);
  L.sp_tok = take(4 * (size_t)L.sp_cap, 4); L.sp_st = take(4 * (size_t)L.sp_cap, 4);
  L.li = take(4 * 32 * B, 4);
  L.c_ord = take(4 * (size_t)L.cc_pad, 4);
  L.c_id = take(4 * (size_t)L.cc, 4);
  L.c_src = take(4 * (size_t)L.cc, 4);
  L.c_st = take(4 * (size_t)L.cc, 4);
  L.excl = take(4 * (size_t)L.excl_words, 4);
  L.plist = take(4 * (size_t)V, 4);
  L.seed = take(4 * 32, 4);
  L.hist = take(4 * 256, 4);
  L.misc = take(4 * 16, 4);
  L.total = (o + 127) / 128 * 128;
  return L;
}

// candidate id: bit 31 set = special s; else prefix d * V + token c
constexpr uint32_t kSpecialBit = 0x80000000u;

struct FW {
  const Params* P;
  int lane, u, steps_done, V;
  uint8_t* rows;
  uint64_t* mbar;
  double *cs, *clm, *ns, *nlm, *lA, *vmin, *vo1, *vo2, *sp_sc, *sp_lm, *c_sc, *c_lm;
  uint64_t *ch, *cph, *nh, *nph, *lk, *c_key;
  int *cn, *cl, *cf, *cst, *nn, *nl, *nf, *nst, *first, *dpi, *e1, *e2, *f1, *pd, *exd, *exc;
  int *sp_base, *sp_x, *sp_flag, *sp_src, *sp_tok, *sp_st, *c_ord, *c_src, *c_st, *misc, *seed, *plist;
  uint32_t *ntrel, *li, *c_id, *excl, *hist;
  int cc, cc_pad;

  __device__ void swap_state() {
    double* d = cs; cs = ns; ns = d;
    d = clm; clm = nlm; nlm = d;
    uint64_t* h = ch; ch = nh; nh = h;
    h = cph; cph = nph; nph = h;
    int* x = cn; cn = nn; nn = x;
    x = cl; cl = nl; nl = x;
    x = cf; cf = nf; nf = x;
    x = cst; cst = nst; nst = x;
  }
};

__device__ void fcarve(FW& w, uint8_t* base, const Params& P) {
  const FusedLayout L = make_fused_layout(P.beam, P.V, P.ring, P.row_bytes);
  w.rows = base + L.rows;
  w.mbar = (uint64_t*)(base + L.mbar);
  w.cs = (double*)(base + L.cs); w.clm = (double*)(base + L.clm);
  w.ch = (uint64_t*)(base + L.ch); w.cph = (uint64_t*)(base + L.cph);
  w.ns = (double*)(base + L.ns); w.nlm = (double*)(base + L.nlm);
  w.nh = (uint64_t*)(base + L.nh); w.nph = (uint64_t*)(base + L.nph);
  w.lA = (double*)(base + L.lA); w.vmin = (double*)(base + L.vmin);
  w.vo1 = (double*)(base + L.vo1); w.vo2 = (double*)(base + L.vo2);
  w.sp_sc = (double*)(base + L.sp_sc); w.sp_lm = (double*)(base + L.sp_lm);
  w.lk = (uint64_t*)(base + L.lk);
  w.c_key = (uint64_t*)(base + L.c_key);
  w.c_sc = (double*)(base + L.c_sc); w.c_lm = (double*)(base + L.c_lm);
  w.cn = (int*)(base + L.cn); w.cl = (int*)(base + L.cl); w.cf = (int*)(base + L.cf); w.cst = (int*)(base + L.cst);
  w.nn = (int*)(base + L.nn); w.nl = (int*)(base + L.nl); w.nf = (int*)(base + L.nf); w.nst = (int*)(base + L.nst);
  w.ntrel = (uint32_t*)(base + L.ntrel);
  w.first = (int*)(base + L.first); w.dpi = (int*)(base + L.dpi);
  w.e1 = (int*)(base + L.e1); w.e2 = (int*)(base + L.e2); w.f1 = (int*)(base + L.f1); w.pd = (int*)(base + L.pd);
  w.exd = (int*)(base + L.exd); w.exc = (int*)(base + L.exc);
  w.sp_base = (int*)(base + L.sp_base); w.sp_x = (int*)(base + L.sp_x); w.sp_flag = (int*)(base + L.sp_flag);
  w.sp_src = (int*)(base + L.sp_src); w.sp_tok = (int*)(base + L.sp_tok); w.sp_st = (int*)(base + L.sp_st);
  w.li = (uint32_t*)(base + L.li);
  w.c_ord = (int*)(base + L.c_ord); w.c_id = (uint32_t*)(base + L.c_id);
  w.c_src = (int*)(base + L.c_src); w.c_st = (int*)(base + L.c_st);
  w.excl = (uint32_t*)(base + L.excl);
  w.plist = (int*)(base + L.plist);
  w.seed = (int*)(base + L.seed);
  w.hist = (uint32_t*)(base + L.hist);
  w.misc = (int*)(base + L.misc);
  w.cc = L.cc;
  w.cc_pad = L.cc_pad;
}

__device__ __forceinline__ double unord64(uint64_t k) {
  const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}
// 64-bit warp max (two 32-bit reductions)
__device__ __forceinline__ uint64_t warp_max64(uint64_t x) {
  const uint32_t hi = __reduce_max_sync(FULL, (uint32_t)(x >> 32));
  const uint32_t lo = __reduce_max_sync(FULL, (uint32_t)(x >> 32) == hi ? (uint32_t)x : 0u);
  return ((uint64_t)hi << 32) | lo;
}

// ---- token sequences through the trellis (exact-tie resolution; lane-serial)
// Python tuple order of seq(ea)+[xa] vs seq(eb)+[xb] (x < 0: no extra token)
__device__ int fseq_cmp(const FW& w, int ea, int xa, int eb, int xb) {
  const Params& P = *w.P;
  if (w.ch[ea] == w.ch[eb] && w.cn[ea] == w.cn[eb]) {
    if (xa == xb) return 0;
    if (xa < 0 || xb < 0) return xa < 0 ? -1 : 1;
    return xa < xb ? -1 : 1;
  }
  int* A = P.seqbuf + (size_t)w.u * 3 * (P.T_max + 1);
  const uint32_t* tr = P.trellis + (size_t)w.u * P.T_max * P.beam;
  auto rec = [&](int i, int slot) {
    const uint32_t r = tr[(size_t)i * P.beam + slot];
    return make_int2(trel_tok(r), trel_src(r));
  };
  bool strict = false;
  return trellis_seq_cmp(rec, w.steps_done, ea, xa, eb, xb, A, A + P.T_max + 1, &strict, P.dbg);
}
struct FDesc { double sc; int base, x, flag; };
__device__ bool fprecedes(const FW& w, const FDesc& a, const FDesc& b) {
  if (a.sc != b.sc) return a.sc > b.sc;
  atomicAdd(&w.P->dbg[kDbgExactTies], 1ull);
  const int c = fseq_cmp(w, a.base, a.x, b.base, b.x);
  if (c) return c < 0;
  return a.flag < b.flag;
}

// bitonic sort of (key desc, idx asc)
__device__ void fbitonic(uint64_t* key, int* idx, int n, int lane) {
  for (int size = 2; size <= n; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = lane; t < (n >> 1); t += 32) {
        const int i = ((t & ~(stride - 1)) << 1) | (t & (stride - 1)), j = i + stride;
        const uint64_t a = key[i], b = key[j];
        const int ia = idx[i], ib = idx[j];
        const bool a_first = a > b || (a == b && ia < ib);
        const bool desc = (i & size) == 0;
        if (desc ? !a_first : a_first) { key[i] = b; key[j] = a; idx[i] = ib; idx[j] = ia; }
      }
      __syncwarp();
    }
}

// Exact evaluation of candidate `id` (decoder.py:467-486 sums, :611 left fold
// in candidate order; payload = first member reaching the max).  Fills the
// score, LM total, source entry, successor context and the ranking descriptor.
struct CandOut { double sc, lm; int src, st, tok, flag, base; };
__device__ CandOut exact_cand(const FW& w, uint32_t id, const float* row, bool use_lm) {
  const Params& P = *w.P;
  CandOut o;
  if (id & kSpecialBit) {
    const int s = (int)(id & ~kSpecialBit);
    o.sc = w.sp_sc[s]; o.lm = w.sp_lm[s]; o.src = w.sp_src[s]; o.st = w.sp_st[s]; o.tok = w.sp_tok[s];
    o.flag = w.sp_flag[s]; o.base = w.sp_base[s];
    return o;
  }
  const int d = (int)(id / (uint32_t)w.V), c = (int)(id % (uint32_t)w.V);
  const int a = w.e1[d], b = w.e2[d];
  const double v = (double)row[c];
  const int sd = w.cst[a];
  double dl = 0.0, wl = 0.0;
  if (use_lm) { dl = P.lm_score[(size_t)sd * P.V + c]; wl = P.lm_weight * dl; }
  auto mem = [&](int h) {
    double x = w.cs[h] + v;
    if (use_lm) x = x + wl;
    if (c == P.sil) x = x + P.sil_score;
    return x;
  };
  const double x = mem(a);
  o.sc = x; o.src = a;
  if (b >= 0) {
    const double y = mem(b);
    o.sc = merge2_exact(x, y, P.merge_max != 0);
    if (y > x) o.src = b;
  }
  o.lm = use_lm ? w.clm[o.src] + dl : w.clm[o.src];
  o.st = use_lm ? P.lm_next[(size_t)sd * P.V + c] : sd;
  o.tok = c; o.flag = 0; o.base = a;
  return o;
}

// One frame.  Returns the new beam size (0: beam died, -1: overflow).
__device__ int fused_step(FW& w, const float* row, int H) {
  const Params& P = *w.P;
  const int lane = w.lane, beam = P.beam, V = P.V;
  const bool use_lm = P.lm_score != nullptr;
  const bool mx = P.merge_max != 0;
  const double eb = (double)row[P.blank];
  // -- beam_size_token (decoder.py:440-458)
  bool has_blank = true;
  uint32_t tv = 0u;
  int ti = 0;
  if (P.tokK) {
    kth_token(row, V, P.blank, (float)eb, P.tokK, w.hist, lane, tv, ti);
    has_blank = token_selected(ord32((float)eb), P.blank, tv, ti);
  }
  auto selected = [&](int c) -> bool { return !P.tokK || token_selected(ord32(row[c]), c, tv, ti); };

  // -- prefixes: entries sharing a token sequence (flag 0 / flag 1 variants)
  for (int e = lane; e < H; e += 32) {
    int f = e;
    for (int q = 0; q < e; q++)
      if (w.ch[q] == w.ch[e] && w.cn[q] == w.cn[e]) { f = q; break; }
    w.first[e] = f;
  }
  __syncwarp();
  int nD = 0;
  for (int b0 = 0; b0 < H; b0 += 32) {
    const int e = b0 + lane;
    const bool isf = e < H && w.first[e] == e;
    const unsigned bal = __ballot_sync(FULL, isf);
    if (isf) {
      const int d = nD + __popc(bal & lanemask_lt());
      w.dpi[e] = d; w.e1[d] = e; w.e2[d] = -1;
    }
    nD += __popc(bal);
  }
  __syncwarp();
  for (int e = lane; e < H; e += 32)
    if (w.first[e] != e) { const int d = w.dpi[w.first[e]]; w.dpi[e] = d; w.e2[d] = e; }
  __syncwarp();
  for (int d = lane; d < nD; d += 32) {
    const int a = w.e1[d], b = w.e2[d];
    w.f1[d] = w.cf[a] == 1 ? a : ((b >= 0 && w.cf[b] == 1) ? b : -1);
    w.lA[d] = b >= 0 ? merge2_exact(w.cs[a], w.cs[b], mx) : w.cs[a];
  }
  // parent prefix of each flag-0 entry; (parent, last token) pairs are excluded
  // from the parent's plain appends (they merge into the child's repeat group)
  if (lane == 0) w.misc[0] = 0;
  __syncwarp();
  for (int e = lane; e < H; e += 32) {
    int p = -1;
    if (w.cf[e] == 0 && w.cn[e] > 0) {
      for (int q = 0; q < H; q++)
        if (w.first[q] == q && w.ch[q] == w.cph[e] && w.cn[q] == w.cn[e] - 1) { p = w.dpi[q]; break; }
      if (p >= 0) {
        const int k = atomicAdd(&w.misc[0], 1);
        w.exd[k] = p; w.exc[k] = w.cl[e];
      }
    }
    w.pd[e] = p;
  }
  __syncwarp();
  const int nEx = w.misc[0];
  auto excluded = [&](int d, int c) -> bool {
    for (int k = 0; k < nEx; k++)
      if (w.exd[k] == d && w.exc[k] == c) return true;
    return false;
  };

  // -- specials (exact): blank groups, repeat groups, last-token appends
  if (lane == 0) w.misc[1] = 0;
  __syncwarp();
  for (int d = lane; d < nD; d += 32) {
    const int a = w.e1[d], b = w.e2[d];
    if (has_blank) {  // (R, 1): blank candidates of both variants (decoder.py:498-506)
      double sc = w.cs[a] + eb;
      int src = a;
      if (b >= 0) {
        const double y = w.cs[b] + eb;
        if (y > sc) src = b;  // payload: first member reaching the max
        sc = merge2_exact(sc, y, mx);
      }
      const int s = atomicAdd(&w.misc[1], 1);
      w.sp_sc[s] = sc; w.sp_lm[s] = w.clm[src]; w.sp_base[s] = a; w.sp_x[s] = -1; w.sp_flag[s] = 1;
      w.sp_src[s] = src; w.sp_tok[s] = -1; w.sp_st[s] = w.cst[a];
    }
    const int c = w.cl[a], f = w.f1[d];
    if (c >= 0 && f >= 0 && selected(c) && !excluded(d, c)) {
      // (R + last, 0) from the flag-1 variant only (the flag-0 one is blocked, decoder.py:495)
      const double v = (double)row[c];
      double dl = 0.0, x = w.cs[f] + v;
      if (use_lm) { dl = P.lm_score[(size_t)w.cst[a] * V + c]; x = x + P.lm_weight * dl; }
      if (c == P.sil) x = x + P.sil_score;
      const int s = atomicAdd(&w.misc[1], 1);
      w.sp_sc[s] = x; w.sp_lm[s] = w.clm[f] + dl; w.sp_base[s] = a; w.sp_x[s] = c; w.sp_flag[s] = 0;
      w.sp_src[s] = f; w.sp_tok[s] = c; w.sp_st[s] = use_lm ? P.lm_next[(size_t)w.cst[a] * V + c] : w.cst[a];
    }
  }
  for (int e = lane; e < H; e += 32) {
    if (w.cf[e] != 0) continue;
    const int c = w.cl[e];
    if (c < 0 || !selected(c)) continue;
    const double ec = (double)row[c];
    double sc = w.cs[e] + ec, best = sc, lmv = w.clm[e];  // repeat first (decoder.py:522-530)
    int src = e, tok = -1;
    const int p = w.pd[e];
    if (p >= 0) {
      const int pa = w.e1[p];
      double dl = 0.0, wl = 0.0;
      if (use_lm) { dl = P.lm_score[(size_t)w.cst[pa] * V + c]; wl = P.lm_weight * dl; }
      const int hs[2] = {w.e1[p], w.e2[p]};
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const int h = hs[q];
        if (h < 0 || (w.cf[h] == 0 && w.cl[h] == c)) continue;  // blocked repeat
        double x = w.cs[h] + ec;
        if (use_lm) x = x + wl;
        if (c == P.sil) x = x + P.sil_score;
        sc = merge2_exact(sc, x, mx);
        if (x > best) { best = x; src = h; tok = c; lmv = w.clm[h] + dl; }
      }
    }
    const int s = atomicAdd(&w.misc[1], 1);
    w.sp_sc[s] = sc; w.sp_lm[s] = lmv; w.sp_base[s] = e; w.sp_x[s] = -1; w.sp_flag[s] = 0;
    w.sp_src[s] = src; w.sp_tok[s] = tok; w.sp_st[s] = w.cst[e];
  }
  __syncwarp();
  const int nS = w.misc[1];

  // -- per-lane top-`beam` lists of approximate keys (specials: exact)
  uint64_t* mylk = w.lk + (size_t)lane * beam;
  uint32_t* myli = w.li + (size_t)lane * beam;
  int cnt = 0;
  uint64_t minkey = 0ull, dropmax = 0ull;  // dropmax: best key this lane evicted or rejected
  // lane list kept sorted descending: inserts near the cut shift few entries
  auto insert = [&](uint64_t key, uint32_t id) {
    int j;
    if (cnt < beam) {
      j = cnt++;
    } else if (key > minkey) {
      dropmax = minkey > dropmax ? minkey : dropmax;
      j = beam - 1;
    } else {
      dropmax = key > dropmax ? key : dropmax;
      return;
    }
    while (j > 0 && mylk[j - 1] < key) { mylk[j] = mylk[j - 1]; myli[j] = myli[j - 1]; j--; }
    mylk[j] = key; myli[j] = id;
    if (cnt == beam) minkey = mylk[beam - 1];
  };
  for (int s = lane; s < nS; s += 32)
    if (w.sp_sc[s] > -INFINITY) insert(ord64(w.sp_sc[s]), kSpecialBit | (uint32_t)s);
  // shared lower bound of the beam cut: any full lane list's minimum
  // Lower bound of the beam cut: the beam-th largest lane maximum (beam
  // candidates in distinct lanes reach it), or any full lane list's minimum.
  // Prefix d scans token c in lane (c + d) mod 32, so the same strong token of
  // different prefixes lands in different lanes.
  // With m = ceil(beam / 32) and each lane's m-th best key, the j-th largest
  // of those (j = ceil(beam / m)) has j * m >= beam candidates at or above it.
  const int bm = (beam + 31) >> 5, bj = (beam + bm - 1) / bm;
  auto bound = [&]() -> double {
    const uint64_t m = cnt == beam ? minkey : 0ull;
    uint64_t g = warp_max64(m);
    {
      uint64_t x = cnt >= bm ? mylk[bm - 1] : 0ull;
#pragma unroll
      for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
          const uint64_t y = ((uint64_t)__shfl_xor_sync(FULL, (uint32_t)(x >> 32), j) << 32) |
                             __shfl_xor_sync(FULL, (uint32_t)x, j);
          const bool take_max = ((lane & j) == 0) == ((lane & k) == 0);
          x = take_max ? (x > y ? x : y) : (x < y ? x : y);
        }
      const uint64_t kth = ((uint64_t)__shfl_sync(FULL, (uint32_t)(x >> 32), bj - 1) << 32) |
                           __shfl_sync(FULL, (uint32_t)x, bj - 1);
      g = kth > g ? kth : g;
    }
    return g ? unord64(g) : -INFINITY;
  };
  // one tolerance per frame covers the rounding gap between approximate and exact scores
  const double tolF = 1e-9 * (1.0 + fabs(w.cs[0])) + 1e-9;
  double theta = bound();
  auto valid_pair = [&](int d, int c) -> bool {
    if (c == P.blank || c == w.cl[w.e1[d]]) return false;  // the last token: a special or blocked
    for (int k = 0; k < nEx; k++)
      if (w.exd[k] == d && w.exc[k] == c) return false;  // merges into a child's repeat group
    return true;
  };
  auto approx = [&](int d, int c, float vf) -> double {  // exact when the prefix has one entry
    double x = w.lA[d] + (double)vf;
    if (use_lm) x = x + P.lm_weight * P.lm_score[(size_t)w.cst[w.e1[d]] * V + c];
    if (c == P.sil) x = x + P.sil_score;
    return x;
  };
  auto offer = [&](int d, int c, double x) {
    if (!(x > -INFINITY)) return;
    const uint64_t key = ord64(x);
    if (cnt < beam || key > minkey) insert(key, (uint32_t)d * (uint32_t)V + (uint32_t)c);
    else dropmax = key > dropmax ? key : dropmax;
  };
  // (1) seeds: every lane's best selected token (of c = lane mod 32) appended to
  //     every prefix, so the beam bound is strong before the full scan
  float bv = -INFINITY;
  int bc = -1;
  for (int c = lane; c < V; c += 32) {
    const float v = row[c];
    if (c != P.blank && v > bv && selected(c)) { bv = v; bc = c; }
  }
  if (!use_lm) {
    // without an LM the emission order is the score order: the row's best token suffices
    const uint32_t bk = bc >= 0 ? ord32(bv) : 0u;
    const uint32_t mk = __reduce_max_sync(FULL, bk);
    const int c1 = (int)__reduce_min_sync(FULL, (mk && bk == mk) ? (uint32_t)bc : 0x7fffffffu);
    bc = (mk && (c1 & 31) == lane) ? c1 : -1;
  }
  w.seed[lane] = bc;
  // seeds go to the best prefixes only (entries are in rank order); the
  // remaining (prefix, seed token) pairs are scanned with the others below
  const int nSeedD = (!use_lm || nD < 2) ? nD : 2;  // without an LM: the best token for every prefix
  if (bc >= 0)
    for (int d = 0; d < nSeedD; d++)
      if (valid_pair(d, bc)) offer(d, bc, approx(d, bc, bv));
  __syncwarp();
  theta = bound();
  // upper-bound offsets of prefix d's append (d, c) minus v_c: coarse (any
  // token: lA + max_c w L), explicit n-gram tokens (lA + wx_s) and backoff
  // tokens (lA + w A_s, plus w U[c]; exact, read without the LM row)
  const int W = (V + 31) / 32;
  for (int d = lane; d < nD; d += 32) {
    const int sd = w.cst[w.e1[d]];
    w.vmin[d] = w.lA[d] + (use_lm ? P.lm_wmax[sd] : 0.0);
    w.vo1[d] = use_lm ? w.lA[d] + P.lm_wx[sd] : w.lA[d];
    w.vo2[d] = use_lm ? w.lA[d] + P.lm_weight * P.lm_A[sd] : -INFINITY;
  }
  __syncwarp();
  auto fcut = [&](double th, double off) -> float {  // v < fcut  =>  off + v < th - tolF
    if (!(th > -INFINITY)) return -INFINITY;
    return __double2float_rd(th - 2.0 * tolF - off);  // rounded down: the cut stays conservative
  };
  // (2) tokens whose emission can reach the cut for some prefix: a coarse
  //     float cut, then (LM) the token's own bound: explicit in some prefix's
  //     context (OR of the prefixes' bitmap words) or the backoff bound
  double amax = -INFINITY, p1 = -INFINITY, p2 = -INFINITY;
  for (int d = lane; d < nD; d += 32) {
    amax = fmax(amax, w.vmin[d]);
    p1 = fmax(p1, w.vo1[d]);
    p2 = fmax(p2, w.vo2[d]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(FULL, amax, o));
    p1 = fmax(p1, __shfl_xor_sync(FULL, p1, o));
    p2 = fmax(p2, __shfl_xor_sync(FULL, p2, o));
  }
  const float gcut = fcut(theta, amax);
  const double gth = theta - 2.0 * tolF;
  const int myst = (use_lm && lane < nD) ? w.cst[w.e1[lane]] : -1;  // nD <= beam <= 32 for the OR
  int nP = 0;
  for (int c0 = 0; c0 < V; c0 += 32) {
    const int c = c0 + lane;
    uint32_t xor_any = 0u;
    if (use_lm) {
      uint32_t wbits = 0u;
      if (myst >= 0) wbits = P.lm_xbits[(size_t)myst * W + (c0 >> 5)];
      for (int d = lane + 32; d < nD; d += 32) wbits |= P.lm_xbits[(size_t)w.cst[w.e1[d]] * W + (c0 >> 5)];
      xor_any = __reduce_or_sync(FULL, wbits);
    }
    bool pass = false;
    if (c < V) {
      const float vf = row[c];
      pass = (!(vf < gcut) || c == P.sil) && c != P.blank && (c != w.seed[lane] || nD > nSeedD) && selected(c);
      if (pass && use_lm && c != P.sil) {
        const double v = (double)vf;
        pass = (((xor_any >> lane) & 1u) && !(v + p1 < gth)) || !(v + (p2 + P.lm_wu[c]) < gth);
      }
    }
    const unsigned bal = __ballot_sync(FULL, pass);
    if (pass) w.plist[nP + __popc(bal & lanemask_lt())] = c;
    nP += __popc(bal);
  }
  __syncwarp();
  // (3) prefix-major over the listed tokens, each pair against its prefix's cut
  for (int d = 0; d < nD; d++) {
    const int lastc = w.cl[w.e1[d]];
    const double off = w.vmin[d], o1 = w.vo1[d], o2 = w.vo2[d];
    const int sd = w.cst[w.e1[d]];
    const double Ad = use_lm ? P.lm_A[sd] : 0.0;
    double mth = cnt == beam ? fmax(theta, unord64(minkey)) : theta;
    float cut = fcut(mth, off);
    const int rot = d & 31;
    // this prefix's excluded tokens (children's repeat groups): two in registers, else the list
    int ex0 = -1, ex1 = -1, nex = 0;
    for (int k = 0; k < nEx; k++)
      if (w.exd[k] == d) { if (nex == 0) ex0 = w.exc[k]; else if (nex == 1) ex1 = w.exc[k]; nex++; }
    for (int j0 = 0; j0 < nP; j0 += 32) {
      int j = j0 + ((lane + rot) & 31);  // spread one token's pairs over lanes
      if (j >= nP) continue;
      const int c = w.plist[j];
      const float vf = row[c];
      if ((!(vf < cut) || c == P.sil) && c != lastc && (d >= nSeedD || c != w.seed[c & 31])) {
        bool ok = c != ex0 && c != ex1;
        if (nex > 2)
          for (int k = 0; k < nEx; k++) ok &= !(w.exd[k] == d && w.exc[k] == c);
        double x = -INFINITY;
        if (ok) {
          if (!use_lm || c == P.sil) {
            x = approx(d, c, vf);
          } else {
            const double v = (double)vf, th2 = mth - 2.0 * tolF;
            if ((P.lm_xbits[(size_t)sd * W + (c >> 5)] >> (c & 31)) & 1u) {
              if (!(v + o1 < th2)) x = approx(d, c, vf);  // explicit n-gram: read the LM row
            } else if (!(v + (o2 + P.lm_wu[c]) < th2)) {
              // backoff token: score[s, c] == A_s + U[c] bit for bit
              x = (w.lA[d] + v) + P.lm_weight * (Ad + P.lm_score[c]);
              if (c == P.sil) x = x + P.sil_score;
            }
          }
          if (x > -INFINITY) {
            const uint64_t key = ord64(x);
            if (cnt < beam || key > minkey) {
              insert(key, (uint32_t)d * (uint32_t)V + (uint32_t)c);
              if (cnt == beam) { mth = fmax(theta, unord64(minkey)); cut = fcut(mth, off); }
            } else {
              dropmax = key > dropmax ? key : dropmax;
            }
          }
        }
      }
    }
    if (d == 1 || (d & 7) == 7) theta = bound();
  }
  __syncwarp();

  // -- extract the global top from the sorted lane lists by k-way merge
  int pos = 0, nc = 0;
  uint64_t lo_key = 0ull;
  bool overflow = false;
  for (;;) {
    const uint64_t my = pos < cnt ? mylk[pos] : 0ull;
    const uint64_t M = warp_max64(my);
    if (M == 0ull) break;
    if (nc >= beam && M < lo_key) break;
    if (nc >= w.cc) { overflow = true; break; }
    const unsigned wl = __ballot_sync(FULL, my == M);
    const int win = __ffs(wl) - 1;
    if (lane == win) { w.c_id[nc] = myli[pos]; pos++; }
    nc++;
    if (nc == beam) lo_key = ord64(unord64(M) - tolF);
  }
  // a candidate this lane dropped may lie inside the window
  if (nc >= beam && dropmax >= lo_key) overflow = true;
  __syncwarp();
  if (nc == 0) return 0;
  auto desc = [&](int i) -> FDesc {
    const uint32_t id = w.c_id[i];
    if (id & kSpecialBit) {
      const int s = (int)(id & ~kSpecialBit);
      return FDesc{w.c_sc[i], w.sp_base[s], w.sp_x[s], w.sp_flag[s]};
    }
    return FDesc{w.c_sc[i], w.e1[id / (uint32_t)V], (int)(id % (uint32_t)V), 0};
  };
  if (__any_sync(FULL, overflow)) {
    // Near-ties wider than the lane lists: stream every candidate of the window
    // [beam-th key - tol, ...) through lane 0's exactly ordered top-`beam` buffer.
    atomicAdd(&P.dbg[kDbgOneshotFallback], 1ull);
    int nsel = 0;
    auto offer = [&](uint32_t id) {  // lane 0
      const CandOut o = exact_cand(w, id, row, use_lm);
      if (!(o.sc > -INFINITY)) return;
      FDesc dx;
      if (id & kSpecialBit) {
        const int s = (int)(id & ~kSpecialBit);
        dx = FDesc{o.sc, w.sp_base[s], w.sp_x[s], w.sp_flag[s]};
      } else {
        dx = FDesc{o.sc, w.e1[id / (uint32_t)V], (int)(id % (uint32_t)V), 0};
      }
      if (nsel == beam && !fprecedes(w, dx, desc(beam - 1))) return;
      int j = nsel < beam ? nsel++ : beam - 1;
      while (j > 0 && fprecedes(w, dx, desc(j - 1))) {
        w.c_id[j] = w.c_id[j - 1]; w.c_sc[j] = w.c_sc[j - 1]; w.c_lm[j] = w.c_lm[j - 1];
        w.c_src[j] = w.c_src[j - 1]; w.c_st[j] = w.c_st[j - 1];
        j--;
      }
      w.c_id[j] = id; w.c_sc[j] = o.sc; w.c_lm[j] = o.lm; w.c_src[j] = o.src; w.c_st[j] = o.st;
    };
    if (lane == 0)
      for (int s = 0; s < nS; s++)
        if (w.sp_sc[s] > -INFINITY && ord64(w.sp_sc[s]) >= lo_key) offer(kSpecialBit | (uint32_t)s);
    uint32_t* stage = w.li;  // lane lists are no longer needed
    for (int d = 0; d < nD; d++) {
      const int a = w.e1[d];
      const int lastc = w.cl[a];
      for (int k = lane; k < nEx; k += 32)
        if (w.exd[k] == d) atomicOr(&w.excl[w.exc[k] >> 5], 1u << (w.exc[k] & 31));
      __syncwarp();
      for (int c0 = 0; c0 < V; c0 += 32) {
        const int c = c0 + lane;
        bool in = false;
        if (c < V && c != P.blank && c != lastc && !((w.excl[c >> 5] >> (c & 31)) & 1u) && selected(c)) {
          double x = w.lA[d] + (double)row[c];
          if (use_lm) x = x + P.lm_weight * P.lm_score[(size_t)w.cst[a] * V + c];
          if (c == P.sil) x = x + P.sil_score;
          in = x > -INFINITY && ord64(x) >= lo_key;
        }
        const unsigned bal = __ballot_sync(FULL, in);
        if (in) stage[__popc(bal & lanemask_lt())] = (uint32_t)d * (uint32_t)V + (uint32_t)c;
        __syncwarp();
        if (lane == 0)
          for (int q = 0; q < __popc(bal); q++) offer(stage[q]);
        __syncwarp();
      }
      for (int k = lane; k < nEx; k += 32)
        if (w.exd[k] == d) atomicAnd(&w.excl[w.exc[k] >> 5], ~(1u << (w.exc[k] & 31)));
      __syncwarp();
    }
    nc = __shfl_sync(FULL, nsel, 0);
    for (int i = lane; i < nc; i += 32) { w.c_ord[i] = i; w.c_key[i] = ord64(w.c_sc[i]); }
    __syncwarp();
  } else {

  // -- exact scores of the window, exact order
  const int npad = pow2_at_least(nc);
  for (int i = lane; i < npad; i += 32) {
    if (i < nc) {
      const CandOut o = exact_cand(w, w.c_id[i], row, use_lm);
      w.c_sc[i] = o.sc; w.c_lm[i] = o.lm; w.c_src[i] = o.src; w.c_st[i] = o.st;
      w.c_key[i] = o.sc > -INFINITY ? ord64(o.sc) : 0ull;
    } else {
      w.c_key[i] = 0ull;
    }
    w.c_ord[i] = i;
  }
  __syncwarp();
  fbitonic(w.c_key, w.c_ord, npad, lane);
  // runs of equal exact scores: token sequence, then flag (decoder.py:651-681)
  {
    bool run = false;
    for (int i = lane; i + 1 < nc; i += 32) run |= w.c_key[i] != 0ull && w.c_key[i] == w.c_key[i + 1];
    if (__any_sync(FULL, run)) {
      if (lane == 0) {
        int a0 = 0;
        while (a0 < nc && w.c_key[a0] != 0ull) {
          int b0 = a0 + 1;
          while (b0 < nc && w.c_key[b0] == w.c_key[a0]) b0++;
          for (int i = a0 + 1; i < b0; i++) {
            const int x = w.c_ord[i];
            const FDesc dx = desc(x);
            int j = i;
            while (j > a0 && fprecedes(w, dx, desc(w.c_ord[j - 1]))) { w.c_ord[j] = w.c_ord[j - 1]; j--; }
            w.c_ord[j] = x;
          }
          a0 = b0;
        }
      }
      __syncwarp();
    }
  }
  }  // exact window
  int valid = 0;
  for (int i0 = 0; i0 < nc; i0 += 32) valid += __popc(__ballot_sync(FULL, i0 + lane < nc && w.c_key[i0 + lane] != 0ull));
  int Hn = valid < beam ? valid : beam;
  if (Hn == 0) return 0;  // every extension is -inf (decoder.py:616-620)
  // beam_threshold on exact scores (decoder.py:621-623)
  if (!P.threshold_inf) {
    const double bex = w.c_sc[w.c_ord[0]];
    int keep = 0;
    for (int r0 = 0; r0 < Hn; r0 += 32) {
      const int r = r0 + lane;
      keep += __popc(__ballot_sync(FULL, r < Hn && w.c_sc[w.c_ord[r]] >= bex - P.beam_threshold));
    }
    Hn = keep;
  }
  // -- commit (decoder.py:683-744)
  for (int r = lane; r < Hn; r += 32) {
    const int i = w.c_ord[r];
    const uint32_t id = w.c_id[i];
    int base, x, flag, tok;
    if (id & kSpecialBit) {
      const int s = (int)(id & ~kSpecialBit);
      base = w.sp_base[s]; x = w.sp_x[s]; flag = w.sp_flag[s]; tok = w.sp_tok[s];
    } else {
      base = w.e1[id / (uint32_t)V]; x = (int)(id % (uint32_t)V); flag = 0; tok = x;
    }
    w.ns[r] = w.c_sc[i];
    w.nlm[r] = w.c_lm[i];
    w.nst[r] = w.c_st[i];
    w.nf[r] = flag;
    if (x >= 0) {
      w.nh[r] = child_hash(w.ch[base], x); w.nph[r] = w.ch[base]; w.nl[r] = x; w.nn[r] = w.cn[base] + 1;
    } else {
      w.nh[r] = w.ch[base]; w.nph[r] = w.cph[base]; w.nl[r] = w.cl[base]; w.nn[r] = w.cn[base];
    }
    w.ntrel[r] = pack_trel(w.c_src[i], tok);
  }
  __syncwarp();
  return Hn;
}

// Finalize (decoder.py:753-817): add w * finish(context) to every entry, merge
// the flag variants of each token sequence in rank order, rank, backtrace.
__device__ void fused_finalize(FW& w, int H, int kept) {
  const Params& P = *w.P;
  const int lane = w.lane, u = w.u;
  const bool use_lm = P.lm_score != nullptr;
  const bool mx = P.merge_max != 0;
  for (int e = lane; e < H; e += 32) {
    if (use_lm) {
      const double fz = P.lm_fin[w.cst[e]];
      w.cs[e] = w.cs[e] + P.lm_weight * fz;
      w.clm[e] = w.clm[e] + fz;
    }
  }
  __syncwarp();
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
    double sc = w.cs[e], best = sc;
    int win = e;
    for (int q = e + 1; q < H; q++)
      if (w.first[q] == e) {
        sc = merge2_exact(sc, w.cs[q], mx);
        if (w.cs[q] > best) { best = w.cs[q]; win = q; }
      }
    const int s = atomicAdd(&w.misc[0], 1);
    w.c_sc[s] = sc; w.c_src[s] = win; w.c_id[s] = (uint32_t)e;
  }
  __syncwarp();
  const int nF = w.misc[0];
  const int pad = pow2_at_least(nF);
  for (int s = lane; s < pad; s += 32) {
    w.c_key[s] = s < nF ? ord64(w.c_sc[s]) : 0ull;
    w.c_ord[s] = s < nF ? s : 0x7fffffff;
  }
  __syncwarp();
  fbitonic(w.c_key, w.c_ord, pad, lane);
  {
    bool run = false;
    for (int i = lane; i + 1 < nF; i += 32) run |= w.c_key[i] == w.c_key[i + 1];
    if (__any_sync(FULL, run) && lane == 0) {
      for (int i = 1; i < nF; i++) {
        const int x = w.c_ord[i];
        const FDesc dx{w.c_sc[x], (int)w.c_id[x], -1, 0};
        int j = i;
        while (j > 0) {
          const int y = w.c_ord[j - 1];
          if (!fprecedes(w, dx, FDesc{w.c_sc[y], (int)w.c_id[y], -1, 0})) break;
          w.c_ord[j] = y;
          j--;
        }
        w.c_ord[j] = x;
      }
    }
    __syncwarp();
  }
  const int nOut = nF < P.nbest ? nF : P.nbest;
  for (int r = lane; r < nOut; r += 32) {
    const int s = w.c_ord[r], e = (int)w.c_id[s], win = w.c_src[s];
    const int len = w.cn[e];
    const size_t o = (size_t)u * P.nbest + r;
    P.out_score[o] = w.c_sc[s];
    if (P.out_lm) P.out_lm[o] = w.clm[win];
    P.out_len[o] = len;
    int* tok_out = P.out_tokens + o * P.T_max;
    int* ts_out = P.out_ts ? P.out_ts + o * P.T_max : nullptr;
    int pos = len, slot = win;
    for (int i = kept - 1; i >= 0 && pos > 0; --i) {
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
  if (lane == 0) P.out_count[u] = nOut;
}

}  // namespace

__global__ void __launch_bounds__(128, 4) ctcb_decode_fused_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  FW w;
  w.P = &P;
  w.lane = lane;
  w.V = P.V;
  fcarve(w, smem + (size_t)wid * P.smem_per_warp, P);
  if (lane == 0)
    for (int s = 0; s < P.ring; s++) mbar_init(&w.mbar[s], 1);
  for (int i = lane; i < (P.V + 31) / 32; i += 32) w.excl[i] = 0u;
  fence_mbar_init();
  __syncwarp();
  uint32_t n_issue = 0, n_cons = 0;
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
    // blank-skip compaction (emissions.py:298-306)
    int kept = 0;
    for (int t0 = 0; t0 < len; t0 += 32) {
      const int t = t0 + lane;
      bool keep = t < len;
      if (keep && P.skip) keep = !(__ldg(ubase + (size_t)t * P.stride_t + P.blank) >= P.cutoff);
      const unsigned bal = __ballot_sync(FULL, keep);
      if (keep) fmap[kept + __popc(bal & lanemask_lt())] = t;
      kept += __popc(bal);
    }
    if (lane == 0) P.kept[u] = kept;
    __syncwarp();
    if (lane == 0) {
      w.cs[0] = 0.0; w.clm[0] = 0.0; w.ch[0] = kEmptyPrefixHash; w.cph[0] = 0ull; w.cl[0] = -1; w.cn[0] = 0;
      w.cf[0] = 1; w.cst[0] = P.lm_score ? P.lm_start : 0;
    }
    int H = 1;
    w.steps_done = 0;
    auto issue = [&](int i) {
      const uint32_t slot = n_issue % (uint32_t)P.ring;
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
    int fail = 0;
    for (int i = 0; i < kept; i++) {
      const float* row;
      if (P.bulk_ok) {
        if (i + P.ring - 1 < kept) {
          if (lane == 0) issue(i + P.ring - 1); else n_issue++;
        }
        const uint32_t slot = n_cons % (uint32_t)P.ring;
        mbar_wait(&w.mbar[slot], (n_cons / (uint32_t)P.ring) & 1u);
        n_cons++;
        row = (const float*)(w.rows + (size_t)slot * P.row_bytes);
      } else {
        float* dst = (float*)w.rows;
        const float* src = ubase + (size_t)fmap[i] * P.stride_t;
        __syncwarp();
        for (int c = lane; c < P.V; c += 32) dst[c] = __ldg(src + c);
        __syncwarp();
        row = dst;
      }
      const int Hn = fused_step(w, row, H);
      if (Hn <= 0) { fail = Hn == 0 ? kUttBeamDied : kUttOverflow; break; }
      uint32_t* trow = P.trellis + ((size_t)u * P.T_max + i) * P.beam;
      for (int r = lane; r < Hn; r += 32) trow[r] = w.ntrel[r];
      w.swap_state();
      H = Hn;
      w.steps_done = i + 1;
      __syncwarp();
    }
    if (fail) {
      while (n_cons < n_issue) {  // drain outstanding row copies of this utterance
        const uint32_t slot = n_cons % (uint32_t)P.ring;
        mbar_wait(&w.mbar[slot], (n_cons / (uint32_t)P.ring) & 1u);
        n_cons++;
      }
      if (lane == 0) {
        P.status[u] = fail;
        P.out_count[u] = 0;
        P.out_len[(size_t)u * P.nbest] = w.steps_done;  // kept-frame index of the failing step
      }
      __syncwarp();
      continue;
    }
    fused_finalize(w, H, kept);
    if (lane == 0) P.status[u] = kUttOk;
    __syncwarp();
  }
}

size_t fused_smem_per_warp(int beam, int V, int ring, int row_bytes) {
  return make_fused_layout(beam, V, ring, row_bytes).total;
}
const void* fused_kernel_fn() { return (const void*)ctcb_decode_fused_kernel; }

}  // namespace ctcb
