// DMMA (mma.sync m8n8k4 f64) vs DFMA throughput probe on B200, and whether
// the two pipes overlap: three kernels over the whole GPU, timed with events.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int MODE>  // 0 dmma only, 1 dfma only, 2 both
__global__ void __launch_bounds__(256) probe(double* out, int iters, double s) {
  double c[8][2];
  double f[16];
  double a = threadIdx.x * 1e-3 + s, b = 1.0 - s;
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = i * s;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i], a, b);
    }
    if (MODE != 0) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) f[i] = fma(f[i], b, a);
    }
  }
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc += f[i];
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  const dim3 grid(nsm * 4), block(256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"dmma only", "dfma only", "dmma + dfma"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) probe<0><<<grid, block>>>(d, iters, 0.5);
      if (mode == 1) probe<1><<<grid, block>>>(d, iters, 0.5);
      if (mode == 2) probe<2><<<grid, block>>>(d, iters, 0.5);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warps = (double)grid.x * block.x / 32;
      const double fl_mma = mode != 1 ? warps * iters * 8 * 512.0 : 0;  // 8x8x4 x 2 per mma
      const double fl_fma = mode != 0 ? (double)grid.x * block.x * iters * 64 * 2.0 : 0;
      if (rep)
        printf("%-12s %.3f ms  dmma %.1f TF/s  dfma %.1f TF/s  total %.1f TF/s\n", names[mode], ms,
               fl_mma / ms / 1e9, fl_fma / ms / 1e9, (fl_mma + fl_fma) / ms / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
