// CTC forced alignment on the GPU (ctcforge align.py:46-123, SURVEY.md
// §8(f4)): Viterbi over the blank-interleaved target sequence
// z = [blank, t1, blank, ..., tL, blank] (S = 2L+1 states).  One warp per
// utterance: lanes own states s = lane + 32 j, frames are sequential; the
// forward scores alpha (fp64, two shared-memory buffers) and the per-frame
// choices (stay / advance-1 / advance-2, int8 in the workspace) reproduce the
// reference's arithmetic exactly (one fp64 add of the fp32 emission per step,
// ties stay > advance-1 > advance-2, final blank preferred on ties).  The
// backtrace is a T-step walk by lane 0; the per-frame scores are then gathered
// by all lanes.
#include <cmath>

#include "../../include/ctcb.h"
#include "ctcb_internal.h"
#include "ctcb_common.cuh"

namespace ctcb {

__global__ void __launch_bounds__(128) ctcb_align_kernel(const float* __restrict__ lp, long long sb, long long st,
                                                         const int32_t* __restrict__ lens,
                                                         const int32_t* __restrict__ targets,
                                                         const int32_t* __restrict__ toff, int B, int T_max, int V,
                                                         int blank, int S_max, int8_t* __restrict__ bp,
                                                         int32_t* __restrict__ out_labels,
                                                         float* __restrict__ out_scores,
                                                         int32_t* __restrict__ out_status,
                                                         int32_t* __restrict__ out_span_start,
                                                         int32_t* __restrict__ out_span_end) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int u = blockIdx.x * (blockDim.x >> 5) + wid;
  if (u >= B) return;
  const size_t per_warp = (size_t)S_max * (8 + 8 + 4 + 1);
  uint8_t* base = smem + (size_t)wid * ((per_warp + 15) / 16 * 16);
  double* A = (double*)base;
  double* N = A + S_max;
  int32_t* z = (int32_t*)(N + S_max);
  uint8_t* can_skip = (uint8_t*)(z + S_max);

  const int T = lens[u];
  const int t0 = toff[u], L = toff[u + 1] - toff[u];
  // argument checks in the reference's order (align.py:60-76)
  int status = CTCB_ALIGN_OK;
  if (T < 0 || T > T_max) status = CTCB_ALIGN_BAD_LEN;
  else if (L <= 0) status = CTCB_ALIGN_EMPTY_TARGETS;
  if (status == CTCB_ALIGN_OK) {
    // the first offending target (in order) decides the message
    int first_blank = 0x7fffffff, first_range = 0x7fffffff, repeats = 0;
    for (int i = lane; i < L; i += 32) {
      const int c = targets[t0 + i];
      if (c == blank) first_blank = min(first_blank, i);
      if (c < 0 || c >= V) first_range = min(first_range, i);
      if (i + 1 < L && c == targets[t0 + i + 1]) repeats++;
    }
    first_blank = __reduce_min_sync(FULL, first_blank);
    first_range = __reduce_min_sync(FULL, first_range);
    repeats = __reduce_add_sync(FULL, repeats);
    if (first_blank != 0x7fffffff || first_range != 0x7fffffff)
      status = first_blank < first_range ? CTCB_ALIGN_BLANK_TARGET : CTCB_ALIGN_RANGE;
    else if (T < L + repeats) status = CTCB_ALIGN_INFEASIBLE;
    else if (2 * L + 1 > S_max) status = CTCB_ALIGN_BAD_LEN;
  }
  if (status != CTCB_ALIGN_OK) {
    if (lane == 0) out_status[u] = status;
    return;
  }
  const int S = 2 * L + 1;
  for (int s = lane; s < S; s += 32) {
    z[s] = (s & 1) ? targets[t0 + (s >> 1)] : blank;
    A[s] = -INFINITY;
  }
  __syncwarp();
  for (int s = lane; s < S; s += 32) can_skip[s] = (s >= 3 && (s & 1) && z[s] != z[s - 2]) ? 1 : 0;
  const float* ub = lp + (size_t)u * sb;
  if (lane == 0) A[0] = (double)ub[z[0]];
  if (lane == 1 && S > 1) A[1] = (double)ub[z[1]];
  __syncwarp();
  int8_t* ubp = bp + (size_t)u * T_max * S_max;
  for (int t = 1; t < T; t++) {
    const float* row = ub + (size_t)t * st;
    int8_t* brow = ubp + (size_t)t * S_max;
    for (int s = lane; s < S; s += 32) {
      double best = A[s];
      int8_t choice = 0;
      const double a1 = s >= 1 ? A[s - 1] : -INFINITY;
      const double a2 = (s >= 2 && can_skip[s]) ? A[s - 2] : -INFINITY;
      if (a1 > best) { best = a1; choice = 1; }
      if (a2 > best) { best = a2; choice = 2; }
      N[s] = best + (double)__ldg(row + z[s]);
      brow[s] = choice;
    }
    __syncwarp();
    double* tmp = A; A = N; N = tmp;
  }
  int32_t* lab = out_labels + (size_t)u * T_max;
  if (lane == 0) {
    int s = S - 1;
    if (S > 1 && A[S - 2] > A[S - 1]) s = S - 2;  // align.py:105-107
    if (A[s] == -INFINITY) {
      status = CTCB_ALIGN_NO_PATH;
    } else {
      // token spans: a feasible path visits target j's state 2j+1 in exactly
      // one run of frames, so the backward walk meets its last frame first
      // (end) and its first frame last (start)
      int32_t* sp0 = out_span_start ? out_span_start + t0 : nullptr;
      int32_t* sp1 = out_span_end ? out_span_end + t0 : nullptr;
      int prev = -1;
      auto mark = [&](int t, int st_) {
        if (sp0 && (st_ & 1)) {
          if (st_ != prev) sp1[st_ >> 1] = t + 1;
          sp0[st_ >> 1] = t;
        }
        prev = st_;
      };
      lab[T - 1] = z[s];
      mark(T - 1, s);
      for (int t = T - 1; t > 0; t--) {
        s -= ubp[(size_t)t * S_max + s];
        lab[t - 1] = z[s];
        mark(t - 1, s);
      }
    }
    out_status[u] = status;
  }
  status = __shfl_sync(FULL, status, 0);
  __syncwarp();
  if (status != CTCB_ALIGN_OK) return;
  float* sc = out_scores + (size_t)u * T_max;
  for (int t = lane; t < T; t += 32) sc[t] = ub[(size_t)t * st + lab[t]];
}

}  // namespace ctcb

namespace {
size_t align_smem_per_warp(int S_max) { return ((size_t)S_max * (8 + 8 + 4 + 1) + 15) / 16 * 16; }
}  // namespace

extern "C" {

int ctcb_align_workspace_bytes(int batch, int t_max, int s_max, size_t* bytes) {
  if (!bytes || batch < 0 || t_max < 0 || s_max < 1)
    return ctcb::set_error(CTCB_ERR_ARG, "ctcb_align_workspace_bytes: bytes must not be NULL, batch/t_max >= 0, s_max >= 1");
  *bytes = (size_t)batch * (size_t)t_max * (size_t)s_max;
  return CTCB_OK;
}

int ctcb_align(const float* log_probs, int64_t stride_b, int64_t stride_t, const int32_t* lens,
               const int32_t* targets, const int32_t* target_offsets, int batch, int t_max, int vocab, int blank,
               int s_max, void* workspace, size_t workspace_bytes, void* stream, int32_t* out_labels,
               float* out_scores, int32_t* out_status, int32_t* out_span_start, int32_t* out_span_end) {
  if (batch == 0) return CTCB_OK;
  if (!log_probs || !lens || !targets || !target_offsets || !workspace || !out_labels || !out_scores || !out_status)
    return ctcb::set_error(CTCB_ERR_ARG, "ctcb_align: pointer arguments must not be NULL");
  if (batch < 0 || t_max < 1 || vocab < 1 || blank < 0 || blank >= vocab || s_max < 1)
    return ctcb::set_error(CTCB_ERR_ARG, "ctcb_align: need batch >= 0, t_max >= 1, 0 <= blank < vocab, s_max >= 1");
  if (stride_t < vocab || stride_b < stride_t * t_max)
    return ctcb::set_error(CTCB_ERR_ARG, "ctcb_align: strides must describe a [batch, t_max, vocab] layout");
  if (workspace_bytes < (size_t)batch * t_max * s_max)
    return ctcb::set_error(CTCB_ERR_WORKSPACE, "ctcb_align: workspace too small");
  const int wpb = 4;
  const size_t smem = align_smem_per_warp(s_max) * wpb;
  int dev = 0, optin = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return ctcb::set_error(CTCB_ERR_CUDA, "ctcb_align: cudaGetDevice failed");
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
    return ctcb::set_error(CTCB_ERR_CUDA, "ctcb_align: cudaDeviceGetAttribute failed");
  if (smem > (size_t)optin)
    return ctcb::set_error(CTCB_ERR_UNSUPPORTED, "ctcb_align: target sequence too long for one warp's shared memory");
  if (cudaFuncSetAttribute(ctcb::ctcb_align_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return ctcb::set_error(CTCB_ERR_CUDA, "ctcb_align: cudaFuncSetAttribute failed");
  ctcb::ctcb_align_kernel<<<(batch + wpb - 1) / wpb, 32 * wpb, smem, (cudaStream_t)stream>>>(
      log_probs, stride_b, stride_t, lens, targets, target_offsets, batch, t_max, vocab, blank, s_max,
      (int8_t*)workspace, out_labels, out_scores, out_status, out_span_start, out_span_end);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CTCB_OK : ctcb::set_error(CTCB_ERR_CUDA, cudaGetErrorString(e));
}

}  // extern "C"
