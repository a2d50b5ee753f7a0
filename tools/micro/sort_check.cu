// Standalone check of the block kernel's sort helpers (block_sort512,
// warp_sort_desc) on random keys: nvcc -gencode arch=compute_100a,code=sm_100a
//   -I paper_2310_17864_b200/csrc tools/micro/sort_check.cu -o /tmp/sort_check
#include "../../paper_2310_17864_b200/csrc/ctcb_block.cu"
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

namespace ctcb {
__global__ void sort_check_kernel(const uint64_t* in, int n, uint64_t* out) {
  __shared__ uint64_t src[512], tmp[512], dst[512];
  for (int i = threadIdx.x; i < 512; i += 256) { src[i] = i < n ? in[i] : 0ull; dst[i] = 0ull; }
  __syncthreads();
  block_sort512(src, n, tmp, dst, threadIdx.x);
  for (int i = threadIdx.x; i < 512; i += 256) out[i] = dst[i];
}
}  // namespace ctcb

int main() {
  std::mt19937_64 rng(1);
  uint64_t *din, *dout;
  cudaMalloc(&din, 512 * 8);
  cudaMalloc(&dout, 512 * 8);
  int bad = 0;
  for (int t = 0; t < 400; t++) {
    const int n = 1 + (int)(rng() % 512);
    std::vector<uint64_t> k(n);
    for (int i = 0; i < n; i++) k[i] = (rng() % 5 == 0) ? 0ull : ((rng() % 1000) << 32) | (uint64_t)(0xffffffffu - i);
    cudaMemcpy(din, k.data(), n * 8, cudaMemcpyHostToDevice);
    ctcb::sort_check_kernel<<<1, 256>>>(din, n, dout);
    std::vector<uint64_t> got(512);
    cudaMemcpy(got.data(), dout, 512 * 8, cudaMemcpyDeviceToHost);
    std::vector<uint64_t> nz;
    for (auto x : k) if (x) nz.push_back(x);
    std::sort(nz.begin(), nz.end(), [](uint64_t a, uint64_t b) { return a > b; });
    for (size_t i = 0; i < nz.size(); i++)
      if (got[i] != nz[i]) { if (bad < 5) printf("n=%d i=%zu got %llx want %llx\n", n, i, (unsigned long long)got[i], (unsigned long long)nz[i]); bad++; break; }
  }
  printf("sort_check: %s (%d bad)\n", bad ? "FAIL" : "ok", bad);
  return bad != 0;
}
