// Micro-test: full-mask collectives after lane-dependent loops (diverged warp).
#include <cstdio>
#include <cstdint>
__global__ void k(const int* trip, unsigned* out, int iters) {
  const int lane = threadIdx.x & 31;
  unsigned long long key = 0x1234567800000000ull | (lane / 3);
  unsigned bad = 0, div = 0;
  for (int it = 0; it < iters; it++) {
    int acc = 0;
    for (int j = 0; j < trip[(lane + it) & 63]; j++) acc += j * lane;  // lane-dependent trip count
    if (acc & 1) key ^= 1ull << 40; else key ^= 0;                      // lane-dependent branch
    __syncwarp();
    if (__activemask() != 0xffffffffu) div++;
    const unsigned m = __match_any_sync(0xffffffffu, key & 0xffffffffull | 0x1234567800000000ull);
    const int s = __shfl_sync(0xffffffffu, lane * 7, (lane + 5) & 31);
    const unsigned r = __reduce_max_sync(0xffffffffu, (unsigned)lane);
    unsigned expect = 0;
    for (int l = 0; l < 32; l++) if (l / 3 == lane / 3) expect |= 1u << l;
    if (m != expect || s != ((lane + 5) & 31) * 7 || r != 31) bad++;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = bad | (div << 16);
}
int main() {
  int h[64]; for (int i = 0; i < 64; i++) h[i] = (i * 37) % 11;
  int* dt; unsigned* dout; cudaMalloc(&dt, sizeof h); cudaMalloc(&dout, 4 * 32 * 512);
  cudaMemcpy(dt, h, sizeof h, cudaMemcpyHostToDevice);
  k<<<32, 512>>>(dt, dout, 2000);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned ho[32 * 512]; cudaMemcpy(ho, dout, sizeof ho, cudaMemcpyDeviceToHost);
  unsigned long long bad = 0, div = 0;
  for (int i = 0; i < 32 * 512; i++) { bad += ho[i] & 0xffff; div += ho[i] >> 16; }
  printf("err=%s bad=%llu diverged_after_syncwarp=%llu of %d\n", cudaGetErrorString(e), bad, div, 32 * 512 * 2000);
}
