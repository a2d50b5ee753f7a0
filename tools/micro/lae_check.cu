// Compare the device logaddexp variants with numpy's: reads pairs (x, y) as
// float64 from stdin-file argv[1], writes [poly, exact] results to argv[2].
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2310_17864_b200/csrc/ctcb_common.cuh"
using namespace ctcb;
__global__ void k(const double* xy, double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = xy[2 * i], y = xy[2 * i + 1];
  out[2 * i] = np_logaddexp<false>(x, y);
  out[2 * i + 1] = np_logaddexp<true>(x, y);
}
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  fseek(f, 0, SEEK_END);
  long bytes = ftell(f);
  fseek(f, 0, SEEK_SET);
  int n = (int)(bytes / 16);
  std::vector<double> h(2 * n), o(2 * n);
  fread(h.data(), 8, 2 * n, f);
  fclose(f);
  double *dxy, *dout;
  cudaMalloc(&dxy, 16 * n);
  cudaMalloc(&dout, 16 * n);
  cudaMemcpy(dxy, h.data(), 16 * n, cudaMemcpyHostToDevice);
  k<<<(n + 255) / 256, 256>>>(dxy, dout, n);
  cudaMemcpy(o.data(), dout, 16 * n, cudaMemcpyDeviceToHost);
  FILE* g = fopen(argv[2], "wb");
  fwrite(o.data(), 8, 2 * n, g);
  fclose(g);
  printf("%d pairs\n", n);
  return 0;
}
