// peak.cu — CUDA-core FP32 (packed FFMA2) and FP64 (DFMA) throughput probes
// used as roofline denominators by bench.py (MEASURED_PEAKS.json carries only
// HBM copy and bf16 tensor peaks). Independent FMA chains, all SMs busy.
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 upk(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }

__global__ void ffma2_chain(float2* out, int iters, float s) {
  float2 a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f);
  const float2 m = make_float2(s, s), b = make_float2(1e-7f, -1e-7f);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      unsigned long long d;
      asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk(a[c])), "l"(pk(m)), "l"(pk(b)));
      a[c] = upk(d);
    }
  float2 acc = make_float2(0, 0);
#pragma unroll
  for (int c = 0; c < 8; ++c) acc.x += a[c].x + a[c].y;
  if (acc.x == 12345.f) out[threadIdx.x] = acc;
}

__global__ void dfma_chain(double* out, int iters, double s) {
  double a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = fma(a[c], s, 1e-9);
  double acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc += a[c];
  if (acc == 12345.0) out[threadIdx.x] = acc;
}

template <class K, class T>
static double run(K kernel, T* buf, int iters, double flops_per_iter_thread, int device) {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, device);
  const int blocks = p.multiProcessorCount * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kernel<<<blocks, threads>>>(buf, iters, 0.999999);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) kernel<<<blocks, threads>>>(buf, iters, 0.999999);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return 5.0 * blocks * threads * (double)iters * flops_per_iter_thread / (ms * 1e-3) / 1e12;
}

extern "C" double ctf_peak_fp32_tflops(int device) {
  cudaSetDevice(device);
  float2* buf;
  cudaMalloc(&buf, 4096 * sizeof(float2));
  const double r = run(ffma2_chain, buf, 20000, 8 * 4.0, device);  // FFMA2 = 2 FMA = 4 flops
  cudaFree(buf);
  return cudaGetLastError() == cudaSuccess ? r : -1.0;
}

extern "C" double ctf_peak_fp64_tflops(int device) {
  cudaSetDevice(device);
  double* buf;
  cudaMalloc(&buf, 4096 * sizeof(double));
  const double r = run(dfma_chain, buf, 4000, 8 * 2.0, device);
  cudaFree(buf);
  return cudaGetLastError() == cudaSuccess ? r : -1.0;
}
