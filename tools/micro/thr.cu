// Throughput microbenchmarks: many warps per SM, independent streams.
#include <cstdio>
#include <cstdint>
__global__ void f2i(double* in, unsigned* out, int n) {
  double a = in[threadIdx.x & 7], b = in[(threadIdx.x + 1) & 7], c = in[(threadIdx.x + 2) & 7], d = in[(threadIdx.x + 3) & 7];
  unsigned acc = 0;
  for (int i = 0; i < n; i++) {
    unsigned x0, x1, x2, x3;
    asm volatile("cvt.rzi.u32.f64 %0, %1;" : "=r"(x0) : "d"(a));
    asm volatile("cvt.rzi.u32.f64 %0, %1;" : "=r"(x1) : "d"(b));
    asm volatile("cvt.rzi.u32.f64 %0, %1;" : "=r"(x2) : "d"(c));
    asm volatile("cvt.rzi.u32.f64 %0, %1;" : "=r"(x3) : "d"(d));
    acc += x0 ^ x1 ^ x2 ^ x3;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void dfma(double* in, unsigned* out, int n) {
  double a = in[threadIdx.x & 7], b = in[(threadIdx.x + 1) & 7], c = in[(threadIdx.x + 2) & 7], d = in[(threadIdx.x + 3) & 7];
  for (int i = 0; i < n; i++) {
    a = fma(a, 1.0000001, 1e-9); b = fma(b, 1.0000001, 1e-9); c = fma(c, 1.0000001, 1e-9); d = fma(d, 1.0000001, 1e-9);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (unsigned)(a + b + c + d);
}
__global__ void dmin(double* in, unsigned* out, int n) {
  double a = in[threadIdx.x & 7], b = in[(threadIdx.x + 1) & 7], c = in[(threadIdx.x + 2) & 7], d = in[(threadIdx.x + 3) & 7];
  for (int i = 0; i < n; i++) {
    a = fmin(a, b + 1.0); b = fmax(b, c - 1.0); c = fmin(c, d + 2.0); d = fmax(d, a - 0.5);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (unsigned)(a + b + c + d);
}
__global__ void iadd(double* in, unsigned* out, int n) {
  unsigned a = threadIdx.x, b = a * 3, c = a * 5, d = a * 7;
  for (int i = 0; i < n; i++) { a = a * 3 + b; b = b * 5 + c; c = c * 7 + d; d = d * 9 + a; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
int main() {
  double* in; unsigned* out;
  cudaMalloc(&in, 64); cudaMalloc(&out, 148 * 1024 * 4 * 8);
  double h[8] = {1.5, 2.5, 3e9, 7.25, 1e3, 99.0, 123456.0, 5.0};
  cudaMemcpy(in, h, 64, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int n = 4096;
  struct { const char* name; void (*k)(double*, unsigned*, int); int ops; } ks[] = {
    {"cvt.rzi.u32.f64", f2i, 4}, {"dfma", dfma, 4}, {"dmin/dmax+dadd", dmin, 8}, {"imad", iadd, 4}};
  for (auto& K : ks) {
    for (int rep = 0; rep < 2; rep++) {
      cudaEventRecord(e0);
      K.k<<<148 * 4, 256>>>(in, out, n);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double warp_ops = 148.0 * 4 * 8 * n * K.ops;
      if (rep) printf("%-18s %.2f warp-ops/clk/SM (at 1.965 GHz)\n", K.name, warp_ops / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
