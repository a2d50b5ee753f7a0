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
/* CTC forced alignment (align.py:46-123), ctc_align.c. */
#define CTCO_ALIGN_EMPTY 11       /* "targets must be non-empty" */
#define CTCO_ALIGN_BLANK 12       /* "targets must not contain the blank token" */
#define CTCO_ALIGN_RANGE 13       /* "target token t out of range [0, V)" */
#define CTCO_ALIGN_INFEASIBLE 14  /* "infeasible alignment: ..." */
#define CTCO_ALIGN_NO_PATH 15     /* "no feasible alignment path" */
int ctco_align(const double* lp, int64_t T, int64_t V, int64_t blank, const int32_t* targets, int64_t L,
               int32_t* frame_labels);
#endif
