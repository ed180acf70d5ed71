// Write-bandwidth probe: the readout backward's store pattern (a warp writes one 2 KB row as 4
// coalesced 512-byte STG.128 waves) against a grid-stride float4 fill, 157 MB like B3 at configs[1].
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rows(uint4* out, long nrows, int rows_per_warp_iter) {
  const int lane = threadIdx.x & 31;
  const long warp = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * (long)blockDim.x) >> 5;
  for (long r = warp; r < nrows; r += nw) {
    uint4* p = out + r * 128 + lane;
    uint4 v = make_uint4(r, lane, 1, 2);
    p[0] = v; p[32] = v; p[64] = v; p[96] = v;
  }
}
__global__ void fill(uint4* out, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
    out[i] = make_uint4(i, 0, 1, 2);
}
int main() {
  const long nrows = 76800;
  const long bytes = nrows * 2048;
  uint4* d;
  cudaMalloc(&d, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int cfg = 0; cfg < 6; ++cfg) {
    int grid = cfg == 0 ? 148 * 3 : cfg == 1 ? 148 * 8 : cfg == 2 ? 148 * 16 : 148 * 4 * (cfg - 2);
    for (int it = 0; it < 2; ++it) {
      cudaEventRecord(a);
      for (int k = 0; k < 20; ++k) {
        if (cfg < 3) rows<<<grid, 256>>>(d, nrows, 1);
        else fill<<<grid, 256>>>(d, bytes / 16);
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it) printf("%s grid %d: %.1f us  %.0f GB/s\n", cfg < 3 ? "rows" : "fill", grid, ms / 20 * 1e3, bytes / (ms / 20 * 1e-3) / 1e9);
    }
  }
  return 0;
}
