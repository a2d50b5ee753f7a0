// H2D gather from mapped pinned memory: register loads (4 or 8 in flight) vs TMA bulk host->smem->device.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2310_17864_b200/csrc/ctcb_common.cuh"
using namespace ctcb;
template <int U>
__global__ void gather(const float4* __restrict__ src, float4* __restrict__ dst, const long long* off, const int* n4, int nseg) {
  int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = w; s < nseg; s += nw) {
    const float4* a = src + off[s]; float4* b = dst + off[s]; int n = n4[s];
    int i = lane;
    for (; i + 32 * (U - 1) < n; i += 32 * U) {
      float4 x[U];
#pragma unroll
      for (int u = 0; u < U; u++) x[u] = a[i + 32 * u];
#pragma unroll
      for (int u = 0; u < U; u++) b[i + 32 * u] = x[u];
    }
    for (; i < n; i += 32) b[i] = a[i];
  }
}
// one warp per segment; lane 0 streams 16 KB chunks host->smem (bulk), then the warp writes smem->device
__global__ void gather_tma(const float4* __restrict__ src, float4* __restrict__ dst, const long long* off, const int* n4, int nseg) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int CH = 16384, NB = 3;
  uint8_t* buf = sm + (size_t)wid * (NB * CH + 64);
  uint64_t* bar = (uint64_t*)(buf + NB * CH);
  if (lane == 0) for (int b = 0; b < NB; b++) mbar_init(&bar[b], 1);
  fence_mbar_init(); __syncwarp();
  uint32_t ph[NB] = {0, 0, 0};
  int w = blockIdx.x * (blockDim.x >> 5) + wid, nw = gridDim.x * (blockDim.x >> 5);
  for (int s = w; s < nseg; s += nw) {
    const char* a = (const char*)(src + off[s]); float4* b = dst + off[s];
    const long long bytes = (long long)n4[s] * 16;
    const int nch = (int)((bytes + CH - 1) / CH);
    auto issue = [&](int c) {
      if (lane == 0) {
        const uint32_t len = (uint32_t)min((long long)CH, bytes - (long long)c * CH);
        fence_proxy_async();
        mbar_arrive_expect_tx(&bar[c % NB], len);
        tma_bulk_g2s(buf + (c % NB) * CH, a + (long long)c * CH, len, &bar[c % NB]);
      }
    };
    for (int c = 0; c < NB - 1 && c < nch; c++) issue(c);
    for (int c = 0; c < nch; c++) {
      if (c + NB - 1 < nch) issue(c + NB - 1);
      mbar_wait(&bar[c % NB], ph[c % NB]); ph[c % NB] ^= 1u;
      const uint32_t len = (uint32_t)min((long long)CH, bytes - (long long)c * CH);
      const float4* sb = (const float4*)(buf + (c % NB) * CH);
      float4* db = b + (long long)c * (CH / 16);
      for (int i = lane; i < (int)(len / 16); i += 32) db[i] = sb[i];
      __syncwarp();
    }
  }
}
int main() {
  const int nseg = 4096; const size_t seg = 875 * 500 / 4;
  size_t tot4 = (size_t)nseg * seg;
  float4* h; cudaHostAlloc(&h, tot4 * 16, cudaHostAllocMapped);
  float4* d; cudaMalloc(&d, tot4 * 16);
  long long* off; int* n4; cudaMallocManaged(&off, nseg * 8); cudaMallocManaged(&n4, nseg * 4);
  size_t bytes = 0;
  for (int s = 0; s < nseg; s++) { off[s] = (long long)s * seg; int T = 125 + (s * 37) % 751; n4[s] = T * 500 / 4; bytes += (size_t)n4[s] * 16; }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("%-28s %.1f GB/s (%.1f ms) %s\n", name, bytes / ms / 1e6, ms, cudaGetErrorString(cudaGetLastError()));
    }
  };
  run("regs x4, 296x256", [&] { gather<4><<<296, 256>>>(h, d, off, n4, nseg); });
  run("regs x8, 296x256", [&] { gather<8><<<296, 256>>>(h, d, off, n4, nseg); });
  run("regs x8, 592x256", [&] { gather<8><<<592, 256>>>(h, d, off, n4, nseg); });
  run("regs x16, 296x256", [&] { gather<16><<<296, 256>>>(h, d, off, n4, nseg); });
  const int smem = 4 * (3 * 16384 + 64);
  cudaFuncSetAttribute(gather_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  run("tma 16KB x3, 148x4 warps", [&] { gather_tma<<<148, 128, smem>>>(h, d, off, n4, nseg); });
  run("tma 16KB x3, 296x4 warps", [&] { gather_tma<<<296, 128, smem>>>(h, d, off, n4, nseg); });
  cudaStream_t st; cudaStreamCreate(&st);
  run("one big DMA", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, 0); });
  return 0;
}
