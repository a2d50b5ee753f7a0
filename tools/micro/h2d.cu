// H2D options for the host-buffer decode path: one large DMA, per-utterance
// cudaMemcpyAsync (one or four streams), and a zero-copy gather kernel.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o h2d h2d.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)
__global__ void gather(const float4* __restrict__ src, const long long* off, const long long* n4, int B, long long Tp4,
                       float4* __restrict__ dst) {
  const int lane = threadIdx.x & 31, nw = (gridDim.x * blockDim.x) >> 5;
  for (int b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < B; b += nw) {
    const float4* s = src + off[b];
    float4* d = dst + (long long)b * Tp4;
    long long m = n4[b], i = lane;
    for (; i + 96 < m; i += 128) {
      float4 x0 = s[i], x1 = s[i + 32], x2 = s[i + 64], x3 = s[i + 96];
      d[i] = x0; d[i + 32] = x1; d[i + 64] = x2; d[i + 96] = x3;
    }
    for (; i < m; i += 32) d[i] = s[i];
  }
}
int main() {
  const int B = 1024, T = 875, V = 500;
  std::vector<int> len(B);
  srand(1);
  for (int b = 0; b < B; b++) len[b] = 125 + rand() % 751;
  const size_t row = (size_t)V * 4, pad = (size_t)T * row, total = (size_t)B * pad;
  float *h, *d;
  CK(cudaHostAlloc(&h, total, cudaHostAllocMapped));
  CK(cudaMalloc(&d, total));
  for (size_t i = 0; i < total / 4; i += 1024) h[i] = 1.0f;
  size_t valid = 0;
  for (int b = 0; b < B; b++) valid += len[b] * row;
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto timeit = [&](const char* name, auto fn) {
    fn(); CK(cudaStreamSynchronize(s));
    float best = 1e9;
    for (int r = 0; r < 3; r++) {
      CK(cudaEventRecord(e0, s)); fn(); CK(cudaEventRecord(e1, s)); CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    printf("%-28s %8.2f ms  %6.1f GB/s (valid bytes %.2f GB)\n", name, best, valid / best / 1e6, valid / 1e9);
  };
  timeit("one DMA (valid bytes)", [&]() { CK(cudaMemcpyAsync(d, h, valid, cudaMemcpyHostToDevice, s)); });
  timeit("per-utterance memcpy", [&]() {
    for (int b = 0; b < B; b++) CK(cudaMemcpyAsync((char*)d + b * pad, (char*)h + b * pad, len[b] * row, cudaMemcpyHostToDevice, s));
  });
  cudaStream_t cs[4];
  for (int i = 0; i < 4; i++) CK(cudaStreamCreateWithFlags(&cs[i], cudaStreamNonBlocking));
  cudaEvent_t ev[4];
  for (int i = 0; i < 4; i++) CK(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
  timeit("per-utterance memcpy x4 str", [&]() {
    for (int i = 0; i < 4; i++) { CK(cudaEventRecord(ev[i], s)); CK(cudaStreamWaitEvent(cs[i], ev[i], 0)); }
    for (int b = 0; b < B; b++)
      CK(cudaMemcpyAsync((char*)d + b * pad, (char*)h + b * pad, len[b] * row, cudaMemcpyHostToDevice, cs[b & 3]));
    for (int i = 0; i < 4; i++) { CK(cudaEventRecord(ev[i], cs[i])); CK(cudaStreamWaitEvent(s, ev[i], 0)); }
  });
  float4* hm; CK(cudaHostGetDevicePointer((void**)&hm, h, 0));
  std::vector<long long> off(B), n4(B);
  for (int b = 0; b < B; b++) { off[b] = (long long)b * pad / 16; n4[b] = len[b] * row / 16; }
  long long *doff, *dn4;
  CK(cudaMalloc(&doff, B * 8)); CK(cudaMalloc(&dn4, B * 8));
  CK(cudaMemcpy(doff, off.data(), B * 8, cudaMemcpyHostToDevice)); CK(cudaMemcpy(dn4, n4.data(), B * 8, cudaMemcpyHostToDevice));
  for (int g : {148, 296, 592, 1184}) {
    char nm[64];
    snprintf(nm, sizeof nm, "zero-copy gather (%d blk)", g);
    timeit(nm, [&]() { gather<<<g, 256, 0, s>>>(hm, doff, dn4, B, pad / 16, (float4*)d); });
  }
  // hybrid: utterances longer than thr by DMA (4 streams), the rest by the gather kernel, concurrently
  std::vector<long long> off2(B), n42(B);
  long long *doff2, *dn42;
  CK(cudaMalloc(&doff2, B * 8)); CK(cudaMalloc(&dn42, B * 8));
  for (int thr : {300, 500, 650, 750}) {
    for (int b = 0; b < B; b++) { off2[b] = off[b]; n42[b] = len[b] > thr ? 0 : n4[b]; }
    CK(cudaMemcpy(dn42, n42.data(), B * 8, cudaMemcpyHostToDevice));
    char nm[64];
    snprintf(nm, sizeof nm, "hybrid DMA len>%d", thr);
    timeit(nm, [&]() {
      for (int i = 0; i < 4; i++) { CK(cudaEventRecord(ev[i], s)); CK(cudaStreamWaitEvent(cs[i], ev[i], 0)); }
      int q = 0;
      for (int b = 0; b < B; b++)
        if (len[b] > thr) CK(cudaMemcpyAsync((char*)d + b * pad, (char*)h + b * pad, len[b] * row, cudaMemcpyHostToDevice, cs[(q++) & 3]));
      gather<<<148, 256, 0, s>>>(hm, doff, dn42, B, pad / 16, (float4*)d);
      for (int i = 0; i < 4; i++) { CK(cudaEventRecord(ev[i], cs[i])); CK(cudaStreamWaitEvent(s, ev[i], 0)); }
    });
  }
  return 0;
}
