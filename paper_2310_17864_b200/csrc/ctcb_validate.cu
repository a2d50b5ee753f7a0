// Input validation mirroring EmissionMatrix.__post_init__ (emissions.py:128-150):
// non-finite values, values above MAX_LOG_PROB = 1e-4, and (strict) rows whose
// float64 log-sum-exp deviates from 0 by more than ROW_NORM_TOL = 1e-3.  The
// first offending (b, code, t, v) in the reference's check order wins.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

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

}  // namespace ctcb
