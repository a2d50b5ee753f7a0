/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Not part of the product path.
 *
 * Plain-C restatement of the reference CPU decoder's hot path (ctcforge 0.1.0,
 * /root/reference/pkg/src/ctcforge) for lexicon-free decoding without an LM:
 *
 *   blank_collapse            emissions.py:284-306  (skip rule :300-301, eps :29)
 *   beam_search_decode        decoder.py:102-135    (entry checks :117-128)
 *   _BeamSearch.__init__      decoder.py:342-376    (initial hypothesis :358-370)
 *   _BeamSearch._step         decoder.py:427-632    (token selection :431-460,
 *                                                    candidate blocks :495-543,
 *                                                    keyed merge :595-613,
 *                                                    threshold :615-626)
 *   _BeamSearch._pack_keys    decoder.py:634-649
 *   _BeamSearch._rank         decoder.py:651-681
 *   _BeamSearch._commit       decoder.py:683-744
 *   _BeamSearch._finalize     decoder.py:753-817
 *
 * It enumerates the full candidate set exactly as the reference does (no
 * top-k pruning: that is the CUDA path's job and is what this oracle checks),
 * merges candidates with identical (parent prefix, token, blank flag) keys by
 * a left fold of numpy's logaddexp (or max) in canonical candidate order, and
 * ranks survivors by (score desc, token sequence asc, packed key asc).
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may load
 * this library.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "ctc_oracle.h"

#define LOGE2 0.693147180559945309417232121458176568

/* numpy's npy_logaddexp (npymath), the ufunc behind np.logaddexp and
 * np.logaddexp.reduceat used at decoder.py:611 and :791. */
static double np_logaddexp(double x, double y) {
  if (x == y) return x + LOGE2; /* also handles equal infinities */
  double tmp = x - y;
  if (tmp > 0) return x + log1p(exp(-tmp));
  if (tmp <= 0) return y + log1p(exp(tmp));
  return tmp; /* nan */
}

/* ---------------------------------------------------------------- vectors */
typedef struct { int64_t* d; int64_t n, cap; } vec64;
static int v64_push(vec64* v, int64_t x) {
  if (v->n == v->cap) {
    int64_t nc = v->cap ? v->cap * 2 : 1024;
    int64_t* nd = (int64_t*)realloc(v->d, (size_t)nc * sizeof(int64_t));
    if (!nd) return -1;
    v->d = nd; v->cap = nc;
  }
  v->d[v->n++] = x;
  return 0;
}

/* Open-addressing map uint64 -> int64, used for the prefix intern table
 * (child_table, decoder.py:345, :700-711) and the per-frame merge groups. */
typedef struct { uint64_t* keys; int64_t* vals; uint8_t* used; int64_t cap, n; } hmap;
static uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27; x *= 0x94d049bb133111ebULL;
  x ^= x >> 31; return x;
}
static int hm_init(hmap* m, int64_t cap) {
  int64_t c = 16;
  while (c < cap * 2) c <<= 1;
  m->keys = (uint64_t*)malloc((size_t)c * sizeof(uint64_t));
  m->vals = (int64_t*)malloc((size_t)c * sizeof(int64_t));
  m->used = (uint8_t*)calloc((size_t)c, 1);
  m->cap = c; m->n = 0;
  return (m->keys && m->vals && m->used) ? 0 : -1;
}
static void hm_free(hmap* m) { free(m->keys); free(m->vals); free(m->used); memset(m, 0, sizeof(*m)); }
static void hm_clear(hmap* m) { memset(m->used, 0, (size_t)m->cap); m->n = 0; }
static int64_t* hm_slot(hmap* m, uint64_t k, int* found);
static int hm_grow(hmap* m) {
  hmap n2;
  if (hm_init(&n2, m->cap) != 0) return -1; /* doubles: init sizes to >= 2*cap */
  for (int64_t i = 0; i < m->cap; i++)
    if (m->used[i]) { int f; *hm_slot(&n2, m->keys[i], &f) = m->vals[i]; }
  hm_free(m);
  *m = n2;
  return 0;
}
/* Returns the value slot for key k, inserting it (value unset) if absent. */
static int64_t* hm_slot(hmap* m, uint64_t k, int* found) {
  uint64_t mask = (uint64_t)m->cap - 1, i = mix64(k) & mask;
  while (m->used[i]) {
    if (m->keys[i] == k) { *found = 1; return &m->vals[i]; }
    i = (i + 1) & mask;
  }
  m->used[i] = 1; m->keys[i] = k; m->n++;
  *found = 0;
  return &m->vals[i];
}

/* ---------------------------------------------------------------- search */
typedef struct {
  /* interned prefixes: id 0 is the empty prefix (decoder.py:343-345) */
  vec64 p_parent, p_token;
  hmap child;
  /* timestep chains (decoder.py:347-349) */
  vec64 ts_parent, ts_token, ts_frame;
  int64_t V;
  /* scratch for token-sequence comparisons */
  int64_t* sa; int64_t* sb; int64_t scap;
} search_t;

static int64_t prefix_len(const search_t* s, int64_t p) {
  int64_t n = 0;
  while (p > 0) { n++; p = s->p_parent.d[p]; }
  return n;
}
/* Token sequence of (parent prefix, token) as in _prefix_tokens, decoder.py:396-405. */
static int64_t prefix_tokens(const search_t* s, int64_t parent, int64_t token, int64_t* out) {
  int64_t n = prefix_len(s, parent) + (token >= 0 ? 1 : 0);
  int64_t i = n;
  if (token >= 0) out[--i] = token;
  int64_t p = parent;
  while (p > 0) { out[--i] = s->p_token.d[p]; p = s->p_parent.d[p]; }
  return n;
}
/* Python tuple ordering of two token sequences. */
static int seq_cmp(search_t* s, int64_t pa, int64_t ta, int64_t pb, int64_t tb) {
  int64_t need = s->p_parent.n + 2;
  if (s->scap < need) {
    s->sa = (int64_t*)realloc(s->sa, (size_t)need * sizeof(int64_t));
    s->sb = (int64_t*)realloc(s->sb, (size_t)need * sizeof(int64_t));
    s->scap = need;
  }
  int64_t na = prefix_tokens(s, pa, ta, s->sa), nb = prefix_tokens(s, pb, tb, s->sb);
  int64_t n = na < nb ? na : nb;
  for (int64_t i = 0; i < n; i++)
    if (s->sa[i] != s->sb[i]) return s->sa[i] < s->sb[i] ? -1 : 1;
  return na < nb ? -1 : (na > nb ? 1 : 0);
}

/* merged group, the unit _rank orders */
typedef struct { double score; int64_t par, tok, flg, winner; uint64_t key; } group_t;

/* (score desc, token sequence asc, packed key asc): the total order that
 * _rank (decoder.py:651-681) applies to the top beam. */
static int group_cmp(search_t* s, const group_t* a, const group_t* b) {
  if (a->score != b->score) return a->score > b->score ? -1 : 1;
  int c = seq_cmp(s, a->par, a->tok, b->par, b->tok);
  if (c) return c;
  return a->key < b->key ? -1 : (a->key > b->key ? 1 : 0);
}

/* stable merge sort of group indices with the search context */
static void sort_groups(search_t* s, const group_t* g, int64_t* idx, int64_t* tmp, int64_t n) {
  if (n < 2) return;
  if (n <= 16) {
    for (int64_t i = 1; i < n; i++) {
      int64_t x = idx[i], j = i;
      while (j > 0 && group_cmp(s, &g[x], &g[idx[j - 1]]) < 0) { idx[j] = idx[j - 1]; j--; }
      idx[j] = x;
    }
    return;
  }
  int64_t h = n / 2;
  sort_groups(s, g, idx, tmp, h);
  sort_groups(s, g, idx + h, tmp, n - h);
  int64_t i = 0, j = h, k = 0;
  while (i < h && j < n) tmp[k++] = (group_cmp(s, &g[idx[j]], &g[idx[i]]) < 0) ? idx[j++] : idx[i++];
  while (i < h) tmp[k++] = idx[i++];
  while (j < n) tmp[k++] = idx[j++];
  memcpy(idx, tmp, (size_t)n * sizeof(int64_t));
}

/* k-th largest of x[0..n) (1-based k), by quickselect on a copy */
static double kth_largest(double* x, int64_t n, int64_t k) {
  int64_t lo = 0, hi = n - 1, want = k - 1; /* position in descending order */
  while (lo < hi) {
    double piv = x[lo + (hi - lo) / 2];
    int64_t i = lo, j = hi;
    while (i <= j) {
      while (x[i] > piv) i++;
      while (x[j] < piv) j--;
      if (i <= j) { double t = x[i]; x[i] = x[j]; x[j] = t; i++; j--; }
    }
    if (want <= j) hi = j; else if (want >= i) lo = i; else return x[want];
  }
  return x[want];
}

/* top-K token selection by (emission desc, index asc), decoder.py:440 */
static int sel_cmp_r(const void* a, const void* b, void* ctx) {
  const double* em = (const double*)ctx;
  int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
  if (em[i] != em[j]) return em[i] > em[j] ? -1 : 1;
  return i < j ? -1 : (i > j ? 1 : 0);
}
static int idx_cmp(const void* a, const void* b) {
  int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
  return i < j ? -1 : (i > j ? 1 : 0);
}

int ctco_blank_keep(const double* lp, int64_t T, int64_t V, int64_t blank, double threshold,
                    int32_t* frame_map, int64_t* n_kept) {
  if (!(threshold > 0.0 && threshold <= 1.0)) return CTCO_ERR_ARG;
  int64_t k = 0;
  for (int64_t t = 0; t < T; t++) {
    int keep = 1;
    if (threshold < 1.0) keep = exp(lp[t * V + blank]) < threshold - CTCO_BLANK_SKIP_EPS;
    if (keep) frame_map[k++] = (int32_t)t;
  }
  *n_kept = k;
  return CTCO_OK;
}

int ctco_decode(const double* lp_in, int64_t T_in, int64_t V, const ctco_opts* o,
                int32_t* out_count, int32_t* out_len, int32_t* out_tokens, int32_t* out_ts,
                double* out_score, int32_t* out_frame_map, int64_t* out_n_kept, int64_t* err_frame) {
  return ctco_decode_fused(lp_in, T_in, V, o, NULL, out_count, out_len, out_tokens, out_ts, out_score, NULL,
                           out_frame_map, out_n_kept, err_frame);
}

/* With fusion (fu != NULL): token-level LM scores enter every append as
 * (h + e_c) + w * L[state, c], then the silence bonus (decoder.py:467-473,
 * :485-486); hypotheses carry their LM context and LM total (payload of the
 * group's best member); finalize adds w * finish(state) (decoder.py:770-777). */
int ctco_decode_fused(const double* lp_in, int64_t T_in, int64_t V, const ctco_opts* o, const ctco_fusion* fu,
                      int32_t* out_count, int32_t* out_len, int32_t* out_tokens, int32_t* out_ts,
                      double* out_score, double* out_lm, int32_t* out_frame_map, int64_t* out_n_kept,
                      int64_t* err_frame) {
  const int use_lm = fu && fu->lm_score;
  const int64_t sil = fu ? fu->sil : -1;
  const double wlm = use_lm ? fu->lm_weight : 0.0;
  if (T_in == 0) return CTCO_ERR_EMPTY; /* decoder.py:117-118 */
  if (o->beam < 1 || o->n_best < 1 || o->n_best > o->beam || !(o->beam_threshold > 0) ||
      !(o->skip_threshold > 0.0 && o->skip_threshold <= 1.0) || o->blank < 0 || o->blank >= V)
    return CTCO_ERR_ARG; /* DecoderOptions.__post_init__, decoder.py:54-66 */
  int64_t K = (o->beam_size_token <= 0) ? V : o->beam_size_token;
  if (K > V) return CTCO_ERR_TOKEN_K; /* decoder.py:124-128 */
  const int64_t blank = o->blank;
  const int logadd = !o->merge_max;

  /* blank_collapse (emissions.py:298-306): frame_map of kept rows */
  int32_t* fmap = out_frame_map;
  int64_t T = 0;
  ctco_blank_keep(lp_in, T_in, V, blank, o->skip_threshold, fmap, &T);
  *out_n_kept = T;

  int rc = CTCO_OK;
  search_t s; memset(&s, 0, sizeof(s));
  s.V = V;
  v64_push(&s.p_parent, -1); v64_push(&s.p_token, -1);
  hm_init(&s.child, 1024);

  const int64_t beam = o->beam;
  /* hypothesis SoA (decoder.py:358-370) */
  int64_t H = 1, Hcap = beam > 1 ? beam : 1;
  double* h_score = (double*)calloc((size_t)Hcap, sizeof(double));
  int64_t* h_prefix = (int64_t*)calloc((size_t)Hcap, sizeof(int64_t));
  int64_t* h_parent = (int64_t*)malloc((size_t)Hcap * sizeof(int64_t));
  int64_t* h_last = (int64_t*)malloc((size_t)Hcap * sizeof(int64_t));
  int64_t* h_flag = (int64_t*)malloc((size_t)Hcap * sizeof(int64_t));
  int64_t* h_ts = (int64_t*)malloc((size_t)Hcap * sizeof(int64_t));
  double* n_score = (double*)malloc((size_t)Hcap * sizeof(double));
  int64_t *n_prefix = (int64_t*)malloc((size_t)Hcap * sizeof(int64_t)), *n_parent = (int64_t*)malloc((size_t)Hcap * sizeof(int64_t)),
          *n_last = (int64_t*)malloc((size_t)Hcap * sizeof(int64_t)), *n_flag = (int64_t*)malloc((size_t)Hcap * sizeof(int64_t)),
          *n_ts = (int64_t*)malloc((size_t)Hcap * sizeof(int64_t));
  h_score[0] = 0.0; h_prefix[0] = 0; h_parent[0] = -1; h_last[0] = -1; h_flag[0] = 1; h_ts[0] = -1;
  int64_t* h_state = (int64_t*)calloc((size_t)Hcap, sizeof(int64_t));
  int64_t* n_state = (int64_t*)calloc((size_t)Hcap, sizeof(int64_t));
  double* h_lm = (double*)calloc((size_t)Hcap, sizeof(double));
  double* n_lm = (double*)calloc((size_t)Hcap, sizeof(double));
  h_state[0] = use_lm ? fu->lm_start : 0;

  int64_t* ck = (int64_t*)malloc((size_t)V * sizeof(int64_t));
  int64_t* order = (int64_t*)malloc((size_t)V * sizeof(int64_t));
  uint8_t* selset = (uint8_t*)calloc((size_t)V, 1);
  int64_t ncand_cap = Hcap * (V + 2) + 16;
  int64_t* c_par = (int64_t*)malloc((size_t)ncand_cap * sizeof(int64_t));
  int64_t* c_tok = (int64_t*)malloc((size_t)ncand_cap * sizeof(int64_t));
  int64_t* c_flg = (int64_t*)malloc((size_t)ncand_cap * sizeof(int64_t));
  int64_t* c_src = (int64_t*)malloc((size_t)ncand_cap * sizeof(int64_t));
  double* c_score = (double*)malloc((size_t)ncand_cap * sizeof(double));
  double* c_lm = (double*)malloc((size_t)ncand_cap * sizeof(double));
  int64_t* c_st = (int64_t*)malloc((size_t)ncand_cap * sizeof(int64_t));
  group_t* grp = (group_t*)malloc((size_t)ncand_cap * sizeof(group_t));
  double* gtmp = (double*)malloc((size_t)ncand_cap * sizeof(double));
  int64_t* gidx = (int64_t*)malloc((size_t)ncand_cap * sizeof(int64_t));
  int64_t* gtmp2 = (int64_t*)malloc((size_t)ncand_cap * sizeof(int64_t));
  hmap gmap; hm_init(&gmap, ncand_cap);

  for (int64_t t = 0; t < T && rc == CTCO_OK; t++) {
    const double* em = lp_in + (int64_t)fmap[t] * V;
    /* token selection (decoder.py:431-460) */
    int64_t kc = 0;
    int has_blank;
    if (K >= V) {
      has_blank = 1;
      for (int64_t c = 0; c < V; c++) if (c != blank) ck[kc++] = c;
      for (int64_t c = 0; c < V; c++) selset[c] = 1;
    } else {
      for (int64_t c = 0; c < V; c++) { order[c] = c; selset[c] = 0; }
      qsort_r(order, (size_t)V, sizeof(int64_t), sel_cmp_r, (void*)em);
      qsort(order, (size_t)K, sizeof(int64_t), idx_cmp);
      for (int64_t i = 0; i < K; i++) selset[order[i]] = 1;
      has_blank = selset[blank];
      for (int64_t i = 0; i < K; i++) if (order[i] != blank) ck[kc++] = order[i];
    }

    /* candidates in canonical order (decoder.py:498-543) */
    int64_t n = 0;
    if (has_blank)
      for (int64_t h = 0; h < H; h++) {
        c_par[n] = h_parent[h]; c_tok[n] = h_last[h]; c_flg[n] = 1; c_src[n] = h;
        c_lm[n] = h_lm[h]; c_st[n] = h_state[h];
        c_score[n] = h_score[h] + em[blank]; n++;
      }
    for (int64_t h = 0; h < H; h++) {
      if (!h_flag[h] && h_last[h] >= 0 && selset[h_last[h]]) {
        c_par[n] = h_parent[h]; c_tok[n] = h_last[h]; c_flg[n] = 0; c_src[n] = h;
        c_lm[n] = h_lm[h]; c_st[n] = h_state[h];
        c_score[n] = h_score[h] + em[h_last[h]]; n++;
      }
    }
    int64_t append_from = n;
    for (int64_t h = 0; h < H; h++)
      for (int64_t j = 0; j < kc; j++) {
        int64_t c = ck[j];
        int blocked = (c == h_last[h]) && !h_flag[h]; /* decoder.py:495-496 */
        c_par[n] = h_prefix[h]; c_tok[n] = c; c_flg[n] = 0; c_src[n] = h;
        double sc = h_score[h] + em[c];
        if (use_lm) {
          const double d = fu->lm_score[h_state[h] * V + c];
          sc = sc + wlm * d;
          c_lm[n] = h_lm[h] + d;
          c_st[n] = fu->lm_next[h_state[h] * V + c];
        } else {
          c_lm[n] = h_lm[h];
          c_st[n] = h_state[h];
        }
        if (c == sil) sc = sc + fu->sil_score;
        c_score[n] = blocked ? -INFINITY : sc; n++;
      }

    /* merge on the packed key (decoder.py:595-613, :634-646): left fold in
     * candidate order; the payload is the first candidate reaching the max */
    hm_clear(&gmap);
    int64_t G = 0;
    for (int64_t i = 0; i < n; i++) {
      uint64_t key = ((uint64_t)(c_par[i] + 1) * (uint64_t)(V + 1) + (uint64_t)(c_tok[i] + 1)) * 2u + (uint64_t)c_flg[i];
      int found;
      int64_t* slot = hm_slot(&gmap, key, &found);
      if (!found) {
        *slot = G;
        grp[G].score = c_score[i]; grp[G].par = c_par[i]; grp[G].tok = c_tok[i];
        grp[G].flg = c_flg[i]; grp[G].winner = i; grp[G].key = key;
        gtmp[G] = c_score[i]; /* running max */
        G++;
      } else {
        group_t* g = &grp[*slot];
        g->score = logadd ? np_logaddexp(g->score, c_score[i]) : (c_score[i] > g->score ? c_score[i] : g->score);
        if (c_score[i] > gtmp[*slot]) { gtmp[*slot] = c_score[i]; g->winner = i; }
      }
    }
    /* threshold (decoder.py:615-626) */
    double best = -INFINITY;
    for (int64_t g = 0; g < G; g++) if (grp[g].score > best) best = grp[g].score;
    if (best == -INFINITY) { rc = CTCO_ERR_BEAM_DIED; *err_frame = t; break; }
    int64_t nk = 0;
    for (int64_t g = 0; g < G; g++) {
      double sc = grp[g].score;
      if (sc > -INFINITY && (isinf(o->beam_threshold) || sc >= best - o->beam_threshold)) gidx[nk++] = g;
    }
    /* _rank (decoder.py:651-681): everything >= the beam-th score, fully ordered */
    int64_t nc = nk;
    if (nk > beam) {
      for (int64_t i = 0; i < nk; i++) gtmp[i] = grp[gidx[i]].score;
      double kth = kth_largest(gtmp, nk, beam);
      nc = 0;
      for (int64_t i = 0; i < nk; i++) if (grp[gidx[i]].score >= kth) gidx[nc++] = gidx[i];
    }
    sort_groups(&s, grp, gidx, gtmp2, nc);
    int64_t Hn = nc < beam ? nc : beam;

    /* _commit (decoder.py:683-744) */
    for (int64_t r = 0; r < Hn; r++) {
      const group_t* g = &grp[gidx[r]];
      int64_t w = g->winner, p = c_par[w], c = c_tok[w], src = c_src[w];
      int64_t pid;
      if (c < 0) {
        pid = 0;
      } else {
        uint64_t key = (uint64_t)p * (uint64_t)(V + 1) + (uint64_t)c;
        int found;
        if (s.child.n * 2 >= s.child.cap) hm_grow(&s.child);
        int64_t* slot = hm_slot(&s.child, key, &found);
        if (!found) {
          *slot = s.p_parent.n;
          v64_push(&s.p_parent, p); v64_push(&s.p_token, c);
        }
        pid = *slot;
      }
      int64_t ts;
      if (w >= append_from) {
        ts = s.ts_parent.n;
        v64_push(&s.ts_parent, h_ts[src]); v64_push(&s.ts_token, c); v64_push(&s.ts_frame, fmap[t]);
      } else {
        ts = h_ts[src];
      }
      n_score[r] = g->score; n_prefix[r] = pid; n_parent[r] = p; n_last[r] = c;
      n_flag[r] = c_flg[w]; n_ts[r] = ts;
      n_lm[r] = c_lm[w]; n_state[r] = c_st[w];
    }
    H = Hn;
    memcpy(h_score, n_score, (size_t)H * sizeof(double));
    memcpy(h_prefix, n_prefix, (size_t)H * sizeof(int64_t));
    memcpy(h_parent, n_parent, (size_t)H * sizeof(int64_t));
    memcpy(h_last, n_last, (size_t)H * sizeof(int64_t));
    memcpy(h_flag, n_flag, (size_t)H * sizeof(int64_t));
    memcpy(h_ts, n_ts, (size_t)H * sizeof(int64_t));
    memcpy(h_lm, n_lm, (size_t)H * sizeof(double));
    memcpy(h_state, n_state, (size_t)H * sizeof(int64_t));
  }

  if (rc == CTCO_OK) {
    /* _finalize (decoder.py:753-817): merge flag variants of one token
     * sequence (same interned prefix) in hypothesis order, then sort. */
    group_t* fin = grp; /* reuse: score, par=prefix id, winner=best hyp, key=order */
    double* fbest = gtmp;
    int64_t F = 0;
    for (int64_t h = 0; h < H; h++) {
      double sh = h_score[h];
      if (use_lm) { /* decoder.py:770-777 */
        const double fz = fu->lm_fin[h_state[h]];
        sh += wlm * fz;
        h_lm[h] += fz;
      }
      int64_t f = -1;
      for (int64_t j = 0; j < F; j++) if (fin[j].par == h_prefix[h]) { f = j; break; }
      if (f < 0) {
        fin[F].score = sh; fin[F].par = h_prefix[h]; fin[F].tok = -1; fin[F].flg = 0;
        fin[F].winner = h; fin[F].key = 0; fbest[F] = sh; F++;
      } else {
        fin[f].score = logadd ? np_logaddexp(fin[f].score, sh) : (sh > fin[f].score ? sh : fin[f].score);
        if (sh > fbest[f]) { fbest[f] = sh; fin[f].winner = h; }
      }
    }
    /* express prefix id p as (parent, token) so group_cmp's sequence order applies */
    for (int64_t f = 0; f < F; f++) {
      int64_t p = fin[f].par;
      fin[f].par = p > 0 ? s.p_parent.d[p] : -1;
      fin[f].tok = p > 0 ? s.p_token.d[p] : -1;
      gidx[f] = f;
    }
    sort_groups(&s, fin, gidx, gtmp2, F);
    int64_t nb = F < o->n_best ? F : o->n_best;
    *out_count = (int32_t)nb;
    for (int64_t r = 0; r < nb; r++) {
      const group_t* g = &fin[gidx[r]];
      out_score[r] = g->score;
      if (out_lm) out_lm[r] = h_lm[g->winner];
      /* tokens and timesteps from the best variant's ts chain (decoder.py:407-415) */
      int64_t len = 0;
      for (int64_t ts = h_ts[g->winner]; ts >= 0; ts = s.ts_parent.d[ts]) len++;
      out_len[r] = (int32_t)len;
      int64_t i = len;
      for (int64_t ts = h_ts[g->winner]; ts >= 0; ts = s.ts_parent.d[ts]) {
        --i;
        out_tokens[r * T_in + i] = (int32_t)s.ts_token.d[ts];
        out_ts[r * T_in + i] = (int32_t)s.ts_frame.d[ts];
      }
    }
  }

  free(s.p_parent.d); free(s.p_token.d); hm_free(&s.child);
  free(s.ts_parent.d); free(s.ts_token.d); free(s.ts_frame.d); free(s.sa); free(s.sb);
  free(h_score); free(h_prefix); free(h_parent); free(h_last); free(h_flag); free(h_ts);
  free(n_score); free(n_prefix); free(n_parent); free(n_last); free(n_flag); free(n_ts);
  free(ck); free(order); free(selset); free(c_par); free(c_tok); free(c_flg); free(c_src); free(c_score);
  free(grp); free(gtmp); free(gidx); free(gtmp2); hm_free(&gmap);
  free(h_state); free(n_state); free(h_lm); free(n_lm); free(c_lm); free(c_st);
  return rc;
}
