/* ORACLE — TEST INFRASTRUCTURE ONLY (see ctc_oracle.c). */
#ifndef CTC_ORACLE_H
#define CTC_ORACLE_H
#include <stdint.h>

#define CTCO_OK 0
#define CTCO_ERR_EMPTY 1       /* "empty emissions", decoder.py:117-118 */
#define CTCO_ERR_ARG 2         /* DecoderOptions validation, decoder.py:54-66 */
#define CTCO_ERR_TOKEN_K 3     /* beam_size_token > V, decoder.py:124-128 */
#define CTCO_ERR_BEAM_DIED 4   /* decoder.py:616-620 */

#define CTCO_BLANK_SKIP_EPS 1e-12 /* emissions.py:29 */

typedef struct {
  int64_t beam;            /* beam_size */
  int64_t beam_size_token; /* <= 0: None (full vocabulary) */
  int64_t n_best;
  int64_t blank;
  int32_t merge_max;       /* 0: "logadd", 1: "max" */
  double beam_threshold;   /* may be +inf */
  double skip_threshold;   /* blank_skip_threshold in (0, 1] */
} ctco_opts;

/* Kept-frame map of blank_collapse (emissions.py:284-306). */
int ctco_blank_keep(const double* lp, int64_t T, int64_t V, int64_t blank, double threshold,
                    int32_t* frame_map, int64_t* n_kept);

/* One utterance, lp row-major [T, V] float64.  Outputs: up to n_best
 * hypotheses; tokens/timesteps rows have stride T. */
int ctco_decode(const double* lp, int64_t T, int64_t V, const ctco_opts* opts,
                int32_t* out_count, int32_t* out_len, int32_t* out_tokens, int32_t* out_ts,
                double* out_score, int32_t* out_frame_map, int64_t* out_n_kept, int64_t* err_frame);
/* Backoff n-gram LM, flattened (paper_2310_17864_b200.lm.flatten), and the
 * dense (context x token) tables of token-level fusion (ctc_lm.c). */
typedef struct {
  int32_t order;
  int64_t n;               /* n-grams */
  const int32_t* words;    /* [n, order], -1 padded */
  const int32_t* lengths;  /* [n] */
  const double* logprob;   /* [n] natural log */
  const double* backoff;   /* [n] */
  const int32_t* start;    /* start context ids */
  int32_t start_len;
  int32_t eos;             /* word id of "</s>" (or <unk>), -1: OOV */
} ctco_lm;
int ctco_lm_tables(const ctco_lm* lm, const int32_t* token_word, int64_t V, double** score, int32_t** next,
                   double** fin, int64_t* n_states, int32_t* start_state);
void ctco_lm_free(double* score, int32_t* next, double* fin);

/* Fusion options of the lexicon-free search (decoder.py:467-473, :531-543,
 * :753-817): token-level LM (dense tables from ctco_lm_tables, or none) and
 * the silence bonus. */
typedef struct {
  const double* lm_score;  /* [S, V] or NULL: no LM */
  const int32_t* lm_next;  /* [S, V] */
  const double* lm_fin;    /* [S] */
  int32_t lm_start;
  double lm_weight;
  int64_t sil;             /* silence token, < 0: none */
  double sil_score;
} ctco_fusion;
int ctco_decode_fused(const double* lp, int64_t T, int64_t V, const ctco_opts* opts, const ctco_fusion* fu,
                      int32_t* out_count, int32_t* out_len, int32_t* out_tokens, int32_t* out_ts,
                      double* out_score, double* out_lm, int32_t* out_frame_map, int64_t* out_n_kept,
                      int64_t* err_frame);

/* CTC forced alignment (align.py:46-123), ctc_align.c. */
#define CTCO_ALIGN_EMPTY 11       /* "targets must be non-empty" */
#define CTCO_ALIGN_BLANK 12       /* "targets must not contain the blank token" */
#define CTCO_ALIGN_RANGE 13       /* "target token t out of range [0, V)" */
#define CTCO_ALIGN_INFEASIBLE 14  /* "infeasible alignment: ..." */
#define CTCO_ALIGN_NO_PATH 15     /* "no feasible alignment path" */
int ctco_align(const double* lp, int64_t T, int64_t V, int64_t blank, const int32_t* targets, int64_t L,
               int32_t* frame_labels);
#endif
