// tools/tc_probe.cu — dev probe: one tcgen05.mma.kind::tf32 (M=128, N=24,
// K=8, A and B K-major in shared memory, SWIZZLE_NONE canonical layout, D in
// TMEM) to validate descriptor construction and the TMEM row/column layout
// before using the tensor cores in a kernel. Not part of the product.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major SWIZZLE_NONE: core matrix = 8 rows x 16 B; LBO = byte distance of
// the two 16-byte K halves (8 tf32 per MMA), SBO = byte distance of 8-row groups
__device__ __forceinline__ uint64_t make_desc(const void* base, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(base) & 0x3FFFF) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100)
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}

__device__ __forceinline__ uint32_t make_idesc_tf32(int M, int N) {
  uint32_t d = 0;
  d |= 1u << 4;                       // c_format F32
  d |= 2u << 7;                       // a_format TF32
  d |= 2u << 10;                      // b_format TF32
  d |= (uint32_t)(N >> 3) << 17;      // n_dim
  d |= (uint32_t)(M >> 4) << 24;      // m_dim
  return d;
}

// element (r, k) of a rows x 8 K-major tile: groups of 8 rows, two 16-byte K halves
__device__ __forceinline__ int kmaj(int r, int k) { return (r >> 3) * 64 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3); }

__global__ void probe(const float* A, const float* B, float* D, int M, int N) {
  __shared__ __align__(1024) float sa[128 * 8];
  __shared__ __align__(1024) float sb[32 * 8];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < 128 * 8; e += blockDim.x) {
    const int r = e / 8, k = e % 8;
    sa[kmaj(r, k)] = r < M ? A[r * 8 + k] : 0.f;
  }
  for (int e = tid; e < 32 * 8; e += blockDim.x) {
    const int r = e / 8, k = e % 8;
    sb[kmaj(r, k)] = r < N ? B[r * 8 + k] : 0.f;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (tid == 0) {
    const uint64_t da = make_desc(sa, 128, 256), db = make_desc(sb, 128, 256);
    const uint32_t id = make_idesc_tf32(128, N);
    const uint32_t z = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
        "l"(da), "l"(db), "r"(id), "r"(z));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&mbar)));
  }
  // wait for the MMA (phase 0)
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(smem_u32(&mbar)));
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // lane r of the D tile = row r; warp w reads lanes 32w..32w+31
  uint32_t v[24];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(tm + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
                 "=r"(v[23])
               : "r"(tm + ((uint32_t)(warp * 32) << 16) + 16));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int j = 0; j < 24; ++j) D[tid * 24 + j] = __uint_as_float(v[j]);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}

}  // namespace

extern "C" int tc_probe(const float* hA, const float* hB, float* hD, int M, int N) {
  float *A, *B, *D;
  cudaMalloc(&A, 128 * 8 * 4);
  cudaMalloc(&B, 32 * 8 * 4);
  cudaMalloc(&D, 128 * 24 * 4);
  cudaMemcpy(A, hA, M * 8 * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, N * 8 * 4, cudaMemcpyHostToDevice);
  cudaMemset(D, 0, 128 * 24 * 4);
  probe<<<1, 128>>>(A, B, D, M, N);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, D, 128 * 24 * 4, cudaMemcpyDeviceToHost);
  cudaFree(A);
  cudaFree(B);
  cudaFree(D);
  if (e != cudaSuccess) std::printf("cuda error %s\n", cudaGetErrorString(e));
  return (int)e;
}
