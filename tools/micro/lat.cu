// Latency microbenchmarks (single warp): fp64 dependent ops, lae, shfl, redux, match.any.
#include <cstdio>
#include <cstdint>
#include "../../paper_2310_17864_b200/csrc/ctcb_common.cuh"
using namespace ctcb;
__global__ void k(double* out, long long* cyc, double a0, int n) {
  int lane = threadIdx.x;
  double x = a0 + lane * 1e-3, y = a0 * 0.5;
  long long t0, t1;
  // 1) dependent DFMA
  t0 = clock64();
  for (int i = 0; i < n; i++) x = fma(x, 1.0000001, 1e-9);
  t1 = clock64(); if (lane == 0) cyc[0] = (t1 - t0); out[0] += x;
  // 2) dependent DADD
  t0 = clock64();
  for (int i = 0; i < n; i++) x = x + y;
  t1 = clock64(); if (lane == 0) cyc[1] = (t1 - t0); out[1] += x;
  // 3) lae chain
  x = -3.0 - lane; y = -3.5;
  t0 = clock64();
  for (int i = 0; i < n; i++) x = np_logaddexp(x, y + i * 1e-3) - 0.6;
  t1 = clock64(); if (lane == 0) cyc[2] = (t1 - t0); out[2] += x;
  // 4) shfl chain
  int v = lane;
  t0 = clock64();
  for (int i = 0; i < n; i++) v = __shfl_xor_sync(0xffffffffu, v, 1) + 1;
  t1 = clock64(); if (lane == 0) cyc[3] = (t1 - t0); out[3] += v;
  // 5) redux chain
  unsigned u = lane;
  t0 = clock64();
  for (int i = 0; i < n; i++) u = __reduce_max_sync(0xffffffffu, u + lane) ;
  t1 = clock64(); if (lane == 0) cyc[4] = (t1 - t0); out[4] += u;
  // 6) match.any.b64 chain
  unsigned long long h = lane >> 2;
  t0 = clock64();
  for (int i = 0; i < n; i++) h = (unsigned long long)__match_any_sync(0xffffffffu, h) >> 28;
  t1 = clock64(); if (lane == 0) cyc[5] = (t1 - t0); out[5] += (double)h;
  // 7) ballot chain
  u = lane;
  t0 = clock64();
  for (int i = 0; i < n; i++) u = __ballot_sync(0xffffffffu, (u & 1u)) ^ lane;
  t1 = clock64(); if (lane == 0) cyc[6] = (t1 - t0); out[6] += u;
  // 8) fp64 compare+select chain
  x = lane;
  t0 = clock64();
  for (int i = 0; i < n; i++) x = x > y ? x - 1.0 : x + 2.0;
  t1 = clock64(); if (lane == 0) cyc[7] = (t1 - t0); out[7] += x;
  // 9) int add chain
  int q = lane;
  t0 = clock64();
  for (int i = 0; i < n; i++) q = (q ^ 5) + 3;
  t1 = clock64(); if (lane == 0) cyc[8] = (t1 - t0); out[8] += q;
  // 10) LDS chain
  __shared__ int sm[64];
  sm[lane] = (lane + 1) & 31; sm[lane+32] = 0; __syncwarp();
  q = lane;
  t0 = clock64();
  for (int i = 0; i < n; i++) q = sm[q];
  t1 = clock64(); if (lane == 0) cyc[9] = (t1 - t0); out[9] += q;
  // 11) float->double convert + add chain
  float f = lane;
  t0 = clock64();
  for (int i = 0; i < n; i++) { x = (double)f + 1.0; f = (float)x; }
  t1 = clock64(); if (lane == 0) cyc[10] = (t1 - t0); out[10] += f;
  // 12) 64-bit shfl pair
  unsigned long long w = lane;
  t0 = clock64();
  for (int i = 0; i < n; i++) { unsigned lo = __shfl_xor_sync(0xffffffffu, (unsigned)w, 1), hi = __shfl_xor_sync(0xffffffffu, (unsigned)(w >> 32), 1); w = (((unsigned long long)hi << 32) | lo) + 1; }
  t1 = clock64(); if (lane == 0) cyc[11] = (t1 - t0); out[11] += (double)w;
}
int main() {
  double* o; long long* c; cudaMallocManaged(&o, 16 * 8); cudaMallocManaged(&c, 16 * 8);
  const char* names[] = {"dfma", "dadd", "lae+dadd", "shfl+iadd", "redux+iadd", "match64+shift", "ballot+xor", "dsetp+sel+dadd", "lop+iadd", "lds", "f2d+dadd+d2f", "shfl64 pair+add"};
  int n = 1024;
  for (int rep = 0; rep < 2; rep++) { k<<<1, 32>>>(o, c, 1.5, n); cudaDeviceSynchronize(); }
  for (int i = 0; i < 12; i++) printf("%-18s %.1f cyc/iter\n", names[i], (double)c[i] / n);
  return 0;
}
