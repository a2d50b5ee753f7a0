// Input validation mirroring EmissionMatrix.__post_init__ (emissions.py:128-150):
// non-finite values, values above MAX_LOG_PROB = 1e-4, and (strict) rows whose
// float64 log-sum-exp deviates from 0 by more than ROW_NORM_TOL = 1e-3.  The
// first offending (b, code, t, v) in the reference's check order wins.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "ctcb_common.cuh"
#include "ctcb_internal.h"

namespace ctcb {

__global__ void ctcb_validate_kernel(const float* lp, long long sb, long long st, const int32_t* lens, int B, int T,
                                     int V, int strict, unsigned long long* out_key) {
  const int b = blockIdx.y;
  int len = lens[b];
  if (len > T) len = T;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + warp;
  if (t >= len) return;
  const float* row = lp + (size_t)b * sb + (size_t)t * st;
  // key = ((b*4 + code) * T + t) * (V + 1) + (v + 1): smaller is earlier
  auto key = [&](int code, int v) {
    return (((unsigned long long)b * 4ull + (unsigned long long)code) * (unsigned long long)T + (unsigned long long)t) *
               (unsigned long long)(V + 1) +
           (unsigned long long)(v + 1);
  };
  float mx = -INFINITY;
  for (int v = lane; v < V; v += 32) {
    float x = row[v];
    if (!isfinite(x)) atomicMin(out_key, key(1, v));
    else if (x > 1e-4f && (double)x > 1e-4) atomicMin(out_key, key(2, v));
    mx = fmaxf(mx, x);
  }
  if (!strict) return;
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (!isfinite(mx)) return;
  double m = (double)mx, s = 0.0;
  for (int v = lane; v < V; v += 32) s += exp((double)row[v] - m);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  double norm = m + log(s);
  if (lane == 0 && fabs(norm) > 1e-3) atomicMin(out_key, key(3, -1));
}

__global__ void ctcb_validate_decode_kernel(const unsigned long long* key, int T, int V, int64_t* out) {
  unsigned long long k = *key;
  if (k == ~0ull) { out[0] = 0; out[1] = out[2] = out[3] = -1; return; }
  long long v = (long long)(k % (unsigned long long)(V + 1)) - 1;
  k /= (unsigned long long)(V + 1);
  long long t = (long long)(k % (unsigned long long)T);
  k /= (unsigned long long)T;
  out[0] = (int64_t)(k % 4ull);
  out[1] = (int64_t)(k / 4ull);
  out[2] = t;
  out[3] = v;
}

// Validation after a decode (ctcb_set_validate): one warp per utterance
// screens, in frame order, the rows the decode kernel did not -- every frame
// when the kernel has no fused check (vfused = 0), else the blank-skipped
// frames and kept frames from vdone on (after a dead beam) -- and merges the
// kernel's offender key; an invalid utterance gets status 5 / 6 / 7 with the
// frame in out_len[u][0] and the token in out_count[u] (emissions.py:128-150
// raises before decoding, so this verdict overrides the decode's own).
__global__ void __launch_bounds__(256) ctcb_validate_post_kernel(const __grid_constant__ Params P) {
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (u >= P.B) return;
  const int len = P.lens[u];
  if (len <= 0 || len > P.T_max) return;  // empty / bad length: the decode's status stands
  const bool strict = P.validate == 1;
  const int kept = P.vfused ? P.kept[u] : 0;
  const int done = P.vfused ? min(P.vdone[u], kept) : 0;
  unsigned long long best = ~0ull;
  if (!(done == len)) {  // done == len: every frame kept and screened
    const int32_t* fmap = P.frame_map + (size_t)u * P.T_max;
    const float* ubase = P.lp + (size_t)u * P.stride_b;
    int kp = 0;  // kept frames before the window
    for (int t0 = 0; t0 < len; t0 += 32) {
      const int f = kp + lane < kept ? fmap[kp + lane] : 0x7fffffff;
      const bool inwin = f < t0 + 32;
      const unsigned screened = __reduce_or_sync(0xffffffffu, (inwin && kp + lane < done) ? 1u << (f - t0) : 0u);
      kp += __popc(__ballot_sync(0xffffffffu, inwin));
      const int nt = len - t0 < 32 ? len - t0 : 32;
      unsigned todo = ~screened & (nt == 32 ? 0xffffffffu : ((1u << nt) - 1u));
      while (todo) {
        const int t = t0 + __ffs(todo) - 1;
        todo &= todo - 1u;
        const float* row = ubase + (size_t)t * P.stride_t;
        if (!row_screen_scalar(row, P.V, lane, strict)) {
          const unsigned long long k2 = row_check_exact(row, P.V, t, lane, strict);
          best = k2 < best ? k2 : best;
        }
      }
    }
  }
  if (lane == 0) {
    unsigned long long key = P.vkey[u];
    key = best < key ? best : key;
    if (key != ~0ull) {
      P.status[u] = kUttNonFinite + (int)(key >> 62) - 1;
      P.out_len[(size_t)u * P.nbest] = (int)((key >> 30) & 0xffffffffull);
      P.out_count[u] = (int)(key & 0x3fffffffull) - 1;
    }
  }
}

}  // namespace ctcb
