// Zero-copy gather bandwidth: a kernel reads pinned host memory (UVA) and writes device memory,
// one warp per ~1 MB segment, vs cudaMemcpyAsync per segment.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void gather(const float4* __restrict__ src, float4* __restrict__ dst, const long long* off, const int* n4, int nseg) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = w; s < nseg; s += nw) {
    const float4* a = src + off[s]; float4* b = dst + off[s]; int n = n4[s];
    int i = lane;
    for (; i + 96 < n; i += 128) { float4 x0 = a[i], x1 = a[i + 32], x2 = a[i + 64], x3 = a[i + 96]; b[i] = x0; b[i + 32] = x1; b[i + 64] = x2; b[i + 96] = x3; }
    for (; i < n; i += 32) b[i] = a[i];
  }
}
int main() {
  const int nseg = 4096; const size_t seg = 1000 * 2000 / 16;  // ~1 MB of float4 per segment, 2 MB stride (padding)
  size_t tot4 = nseg * seg * 2;
  float4* h; cudaHostAlloc(&h, tot4 * 16, cudaHostAllocMapped);
  float4* d; cudaMalloc(&d, tot4 * 16);
  long long* off; int* n4; cudaMallocManaged(&off, nseg * 8); cudaMallocManaged(&n4, nseg * 4);
  size_t bytes = 0;
  for (int s = 0; s < nseg; s++) { off[s] = (long long)s * seg * 2; n4[s] = (int)(seg * (0.25 + 1.5 * ((s * 37) % 100) / 100.0)); bytes += (size_t)n4[s] * 16; }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int blocks : {148, 296, 592, 1184}) for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0); gather<<<blocks, 256>>>(h, d, off, n4, nseg); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep) printf("zero-copy kernel %d blocks: %.1f GB/s (%.1f ms)\n", blocks, bytes / ms / 1e6, ms);
  }
  cudaStream_t st[4]; for (int i = 0; i < 4; i++) cudaStreamCreate(&st[i]);
  for (int rep = 0; rep < 2; rep++) {
    cudaEventRecord(e0);
    for (int s = 0; s < nseg; s++) cudaMemcpyAsync(d + off[s], h + off[s], (size_t)n4[s] * 16, cudaMemcpyHostToDevice, st[s & 3]);
    for (int i = 0; i < 4; i++) cudaStreamSynchronize(st[i]);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (rep) printf("memcpyAsync per segment x4 streams: %.1f GB/s (%.1f ms)\n", bytes / ms / 1e6, ms);
  }
  return 0;
}
