/* ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of ctcforge's CTC forced alignment
 * (/root/reference/pkg/src/ctcforge/align.py:46-123): Viterbi over the
 * blank-interleaved target sequence [blank, t1, blank, ..., tL, blank].  Only
 * tests/ use it, as the checker of the CUDA alignment kernel; parity of this
 * restatement is pinned by tests/golden/align.json (outputs of the reference
 * itself, tests/golden/make_align_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "ctc_oracle.h"

/* lp row-major [T, V] float64; targets[L].  Outputs frame_labels[T] (token
 * per frame, blank allowed).  Returns CTCO_ALIGN_* (align.py:60-76, :108-110). */
int ctco_align(const double* lp, int64_t T, int64_t V, int64_t blank, const int32_t* targets, int64_t L,
               int32_t* frame_labels) {
  if (L <= 0) return CTCO_ALIGN_EMPTY;                              /* align.py:62-63 */
  for (int64_t i = 0; i < L; i++) {
    if (targets[i] == blank) return CTCO_ALIGN_BLANK;               /* :64-66 */
    if (targets[i] < 0 || targets[i] >= V) return CTCO_ALIGN_RANGE; /* :67-68 */
  }
  int64_t repeats = 0;
  for (int64_t i = 0; i + 1 < L; i++) repeats += targets[i] == targets[i + 1];
  if (T < L + repeats) return CTCO_ALIGN_INFEASIBLE;                /* :70-75 */
  const int64_t S = 2 * L + 1;
  int64_t* z = (int64_t*)malloc(S * sizeof(int64_t));
  unsigned char* can_skip = (unsigned char*)calloc(S, 1);
  double* alpha = (double*)malloc(S * sizeof(double));
  double* nxt = (double*)malloc(S * sizeof(double));
  signed char* bp = (signed char*)calloc((size_t)T * S, 1);
  for (int64_t s = 0; s < S; s++) z[s] = (s & 1) ? targets[s >> 1] : blank;   /* :77-79 */
  for (int64_t s = 3; s < S; s += 2) can_skip[s] = z[s] != z[s - 2];          /* :80-82 */
  for (int64_t s = 0; s < S; s++) alpha[s] = -INFINITY;                      /* :84-88 */
  alpha[0] = lp[z[0]];
  if (S > 1) alpha[1] = lp[z[1]];
  for (int64_t t = 1; t < T; t++) {                                          /* :90-103 */
    const double* row = lp + t * V;
    for (int64_t s = 0; s < S; s++) {
      double best = alpha[s];
      signed char choice = 0;
      const double a1 = s >= 1 ? alpha[s - 1] : -INFINITY;
      const double a2 = (s >= 2 && can_skip[s]) ? alpha[s - 2] : -INFINITY;
      if (a1 > best) { best = a1; choice = 1; }   /* ties stay > advance-1 > advance-2 */
      if (a2 > best) { best = a2; choice = 2; }
      nxt[s] = best + row[z[s]];
      bp[t * S + s] = choice;
    }
    double* tmp = alpha; alpha = nxt; nxt = tmp;
  }
  int64_t s = S - 1;                                                         /* :105-110 */
  if (S > 1 && alpha[S - 2] > alpha[S - 1]) s = S - 2;
  int rc = CTCO_OK;
  if (alpha[s] == -INFINITY) {
    rc = CTCO_ALIGN_NO_PATH;
  } else {
    frame_labels[T - 1] = (int32_t)z[s];                                     /* :112-117 */
    for (int64_t t = T - 1; t > 0; t--) {
      s -= bp[t * S + s];
      frame_labels[t - 1] = (int32_t)z[s];
    }
  }
  free(z); free(can_skip); free(alpha); free(nxt); free(bp);
  return rc;
}
