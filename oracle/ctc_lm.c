/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Not part of the product path.
 *
 * Plain-C restatement of the reference's backoff n-gram scoring for
 * token-level fusion (ctcforge lm.py:229-270; decoder.py:178-259):
 *
 *   _backoff_score     lm.py:247-262   (Katz backoff, OOV penalty when no unigram)
 *   _shrink_to_known   lm.py:265-270   (drop leading words until the context exists)
 *   context_score      lm.py:229-241   (<unk> mapping, OOV -> ((), -20))
 *   context_finish     lm.py:244-245   (score of "</s>")
 *   _TokenContexts     decoder.py:178-259 (dense (context x token) score / successor rows;
 *                                          blank and silence rows are identity)
 *
 * The model arrives flattened (paper_2310_17864_b200.lm.flatten): n-gram i has
 * words[i*order .. +len[i]), natural-log logprob/backoff.  Contexts are
 * interned as states: 0 = (), and one state per n-gram shorter than the order.
 * Only tests/ may load this library.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "ctc_oracle.h"

#define OOV_PENALTY (-20.0) /* lm.py:22-24 */

typedef struct { uint64_t* keys; int64_t* vals; int64_t cap; } tmap;

static uint64_t tmix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33; return x;
}
static void tm_put(tmap* m, uint64_t k, int64_t v) {
  uint64_t mask = (uint64_t)m->cap - 1, i = tmix(k) & mask;
  while (m->keys[i] && m->keys[i] != k) i = (i + 1) & mask;
  m->keys[i] = k; /* later duplicates win, like dict assignment */
  m->vals[i] = v;
}
static int64_t tm_get(const tmap* m, uint64_t k) {
  uint64_t mask = (uint64_t)m->cap - 1, i = tmix(k) & mask;
  while (m->keys[i]) {
    if (m->keys[i] == k) return m->vals[i];
    i = (i + 1) & mask;
  }
  return -1;
}

typedef struct {
  const ctco_lm* lm;
  tmap map;
  uint64_t base; /* word id + 1 digits in base (max id + 2): exact tuple keys */
} lmctx;

static uint64_t tuple_key(const lmctx* c, const int32_t* ids, int n) {
  uint64_t k = 0;
  for (int i = 0; i < n; i++) k = k * c->base + (uint64_t)(ids[i] + 1);
  return k;
}
static int64_t lookup(const lmctx* c, const int32_t* ids, int n) {
  if (n == 0) return -1;
  return tm_get(&c->map, tuple_key(c, ids, n));
}
/* lm.py:247-262 with ctx = context[-(order-1):] */
static double backoff_score(const lmctx* c, const int32_t* ctx_in, int n, int32_t wid) {
  const int order = c->lm->order;
  int32_t buf[64];
  if (order > 1 && n > order - 1) { ctx_in += n - (order - 1); n = order - 1; }
  if (order == 1) n = 0;
  memcpy(buf, ctx_in, (size_t)n * sizeof(int32_t));
  double acc = 0.0;
  const int32_t* ctx = buf;
  for (;;) {
    int32_t ng[64];
    memcpy(ng, ctx, (size_t)n * sizeof(int32_t));
    ng[n] = wid;
    int64_t e = lookup(c, ng, n + 1);
    if (e >= 0) return acc + c->lm->logprob[e];
    if (n == 0) return acc + OOV_PENALTY;
    int64_t ce = lookup(c, ctx, n);
    if (ce >= 0) acc += c->lm->backoff[ce];
    ctx++; n--;
  }
}
/* lm.py:265-270: returns the entry of the shrunk context (-1: empty) */
static int64_t shrink(const lmctx* c, const int32_t* ctx, int n) {
  while (n > 0) {
    int64_t e = lookup(c, ctx, n);
    if (e >= 0) return e;
    ctx++; n--;
  }
  return -1;
}

int ctco_lm_tables(const ctco_lm* lm, const int32_t* token_word, int64_t V, double** out_score,
                   int32_t** out_next, double** out_fin, int64_t* out_states, int32_t* out_start) {
  const int order = lm->order;
  if (order < 1 || order > 60) return CTCO_ERR_ARG;
  int32_t maxid = 0;
  for (int64_t i = 0; i < lm->n; i++)
    for (int j = 0; j < lm->lengths[i]; j++)
      if (lm->words[i * order + j] > maxid) maxid = lm->words[i * order + j];
  lmctx c;
  c.lm = lm;
  c.base = (uint64_t)maxid + 2;
  /* exact keys need base^order < 2^64 */
  double bits = (double)order * log2((double)c.base);
  if (bits > 63.0) return CTCO_ERR_ARG;
  int64_t cap = 16;
  while (cap < 2 * lm->n + 16) cap <<= 1;
  c.map.cap = cap;
  c.map.keys = (uint64_t*)calloc((size_t)cap, sizeof(uint64_t));
  c.map.vals = (int64_t*)malloc((size_t)cap * sizeof(int64_t));
  for (int64_t i = 0; i < lm->n; i++) tm_put(&c.map, tuple_key(&c, lm->words + i * order, lm->lengths[i]), i);
  /* states: 0 = (), then every n-gram shorter than the order */
  int64_t* state_of = (int64_t*)malloc((size_t)(lm->n > 0 ? lm->n : 1) * sizeof(int64_t));
  int64_t* entry_of = (int64_t*)malloc((size_t)(lm->n + 1) * sizeof(int64_t));
  int64_t S = 1;
  entry_of[0] = -1;
  for (int64_t i = 0; i < lm->n; i++) {
    /* a duplicated tuple keeps only its last row (dict semantics) */
    int64_t e = tm_get(&c.map, tuple_key(&c, lm->words + i * order, lm->lengths[i]));
    if (e == i && lm->lengths[i] < order) { state_of[i] = S; entry_of[S++] = i; }
    else state_of[i] = -1;
  }
  double* L = (double*)malloc((size_t)(S * V) * sizeof(double));
  int32_t* N = (int32_t*)malloc((size_t)(S * V) * sizeof(int32_t));
  double* F = (double*)malloc((size_t)S * sizeof(double));
  for (int64_t s = 0; s < S; s++) {
    int32_t ctx[64];
    int n = 0;
    if (entry_of[s] >= 0) {
      n = lm->lengths[entry_of[s]];
      memcpy(ctx, lm->words + entry_of[s] * order, (size_t)n * sizeof(int32_t));
    }
    for (int64_t v = 0; v < V; v++) {
      const int32_t wid = token_word[v];
      if (wid == -2) { L[s * V + v] = 0.0; N[s * V + v] = (int32_t)s; continue; } /* blank / silence */
      if (wid < 0) { L[s * V + v] = OOV_PENALTY; N[s * V + v] = 0; continue; }  /* lm.py:236-238 */
      L[s * V + v] = backoff_score(&c, ctx, n, wid);
      if (order == 1) { N[s * V + v] = 0; continue; }
      int32_t nx[64];
      memcpy(nx, ctx, (size_t)n * sizeof(int32_t));
      nx[n] = wid;
      int m = n + 1;
      const int32_t* tail = nx;
      if (m > order - 1) { tail += m - (order - 1); m = order - 1; }
      int64_t e = shrink(&c, tail, m);
      N[s * V + v] = e < 0 ? 0 : (int32_t)state_of[e];
    }
    F[s] = lm->eos < 0 ? OOV_PENALTY : backoff_score(&c, ctx, n, lm->eos);
  }
  /* start context (lm.py:229-233, computed by the caller) */
  int64_t st = -1;
  if (lm->start_len > 0) st = lookup(&c, lm->start, lm->start_len);
  *out_start = st < 0 ? 0 : (int32_t)state_of[st];
  free(c.map.keys); free(c.map.vals); free(state_of); free(entry_of);
  *out_score = L; *out_next = N; *out_fin = F; *out_states = S;
  return CTCO_OK;
}

void ctco_lm_free(double* score, int32_t* next, double* fin) { free(score); free(next); free(fin); }
