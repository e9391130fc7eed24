// ctf_stft.cuh — STFT front end and weighted-overlap-add back end on the GPU
// (reference proj/src/stft.cpp:46-139, proj/src/fft.cpp).
//
// One CTA transforms a block of (frame, channel) sequences held in shared
// memory with the reference's own arithmetic: iterative radix-2
// decimation-in-time over a bit-reversed load, twiddles taken from a table the
// host builds with the reference's recurrence (w *= wlen), products and sums
// rounded exactly like std::complex<double> without contraction (__dmul_rn /
// __dadd_rn), Hann window from the host. The GPU spectrogram / signal is
// therefore bit-identical to the CPU restatement, not just close to it.
//
// Layouts: samples [signal][channel][length] (TimeSignal.samples column-major
// per signal), spectrogram [signal][bin][frame][channel] complex
// (Spectrogram.data, types.hpp:22-47) — the same order as the estimator's x, so
// the forward transform writes straight into the ISS input buffer.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ctf {

struct StftParams {
  const double* samples;   // [S][C][n]
  void* spec;              // [S][bins_out][frames][C] complex (double2 or float2)
  const double2* tw;       // twiddle table, stage len at [len/2 - 1 + k], k < len/2
  const double* window;    // [N]
  int64_t n;               // samples per channel
  int N, logN, hop, frames, C;
  int bin_lo, bin_hi;      // bins written (a frequency shard), bins_out = bin_hi - bin_lo
  int PF, CC;              // frames x channels per CTA
  int out_f32;             // store complex64
};

struct IstftParams {
  const double2* spec;     // [S][bins][frames][C]
  double* frames_buf;      // [S][C][frames][N] windowed inverse frames
  double* out;             // [S][C][out_len]
  const double2* tw;       // inverse twiddle table
  const double* window;
  double scale;            // 1 / N
  int64_t out_len;
  int N, logN, hop, frames, bins, C, PF, CC, S;
};

__device__ __forceinline__ double2 cmul_rn(double2 a, double2 b) {  // std::complex<double> operator*
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// In-place radix-2 DIT over S sequences of N complex in shared memory, already
// in bit-reversed order (fft.cpp:20-37 stage/butterfly order). Two stages
// (s, s+1) run per shared-memory pass on the closed 4-element sets
// {i, i+h, i+2h, i+3h} (h = 2^(s-1)): the same butterflies with the same
// twiddles in the same order as two radix-2 passes, so the result is
// bit-identical while the shared-memory traffic and barriers halve.
__device__ __forceinline__ double2 cadd_rn(double2 a, double2 b) { return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)); }
__device__ __forceinline__ double2 csub_rn(double2 a, double2 b) { return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)); }

__device__ __forceinline__ void block_fft(double2* a, int S, int N, int logN, const double2* __restrict__ tw) {
  const int halfN = N >> 1, qN = N >> 2;
  int s = 1;
  if (logN & 1) {  // one radix-2 pass (len = 2) when the stage count is odd
    for (int b = threadIdx.x; b < S * halfN; b += blockDim.x) {
      const int q = b / halfN, bb = b - q * halfN;
      double2* base = a + (size_t)q * N + 2 * bb;
      const double2 u = base[0];
      const double2 v = cmul_rn(base[1], __ldg(tw));
      base[0] = cadd_rn(u, v);
      base[1] = csub_rn(u, v);
    }
    __syncthreads();
    s = 2;
  }
  for (; s < logN; s += 2) {
    const int h = 1 << (s - 1), len = h << 1;
    const double2* w1 = tw + (h - 1);    // stage s (length len), k < h
    const double2* w2 = tw + (len - 1);  // stage s+1 (length 2len), k < len
    for (int b = threadIdx.x; b < S * qN; b += blockDim.x) {
      const int q = b / qN, qq = b - q * qN;
      const int k = qq & (h - 1);
      const int i = ((qq >> (s - 1)) << (s + 1)) + k;
      double2* base = a + (size_t)q * N + i;
      const double2 x0 = base[0], x1 = base[h], x2 = base[len], x3 = base[len + h];
      const double2 t1 = __ldg(w1 + k);
      double2 v = cmul_rn(x1, t1);
      const double2 y0 = cadd_rn(x0, v), y1 = csub_rn(x0, v);
      v = cmul_rn(x3, t1);
      const double2 y2 = cadd_rn(x2, v), y3 = csub_rn(x2, v);
      v = cmul_rn(y2, __ldg(w2 + k));
      base[0] = cadd_rn(y0, v);
      base[len] = csub_rn(y0, v);
      v = cmul_rn(y3, __ldg(w2 + k + h));
      base[h] = cadd_rn(y1, v);
      base[len + h] = csub_rn(y1, v);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int bitrev(int t, int logN) { return (int)(__brev((unsigned)t) >> (32 - logN)); }

// Reflect padding by N/2 (stft.cpp:25-42), sample t of the padded channel.
__device__ __forceinline__ double padded_sample(const double* x, int64_t n, int half, int64_t t) {
  int64_t src;
  if (t < half) {
    src = half - t;
    if (src >= n) src = n - 1;
  } else if (t < half + n) {
    src = t - half;
  } else {
    src = 2 * n - 2 - (t - half);
    if (src < 0) src = 0;
    if (src >= n) return 0.0;
  }
  return x[src];
}

// grid (ceil(frames / PF), S, ceil(C / CC)); smem PF*CC*N double2
__global__ void __launch_bounds__(256) stft_kernel(const StftParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* a = reinterpret_cast<double2*>(smem_raw);
  const int N = p.N, logN = p.logN, half = N >> 1;
  const int f0 = blockIdx.x * p.PF, sig = blockIdx.y, c0 = blockIdx.z * p.CC;
  const int nseq = p.PF * p.CC;
  const double* xs = p.samples + (size_t)sig * p.C * p.n;
  for (int e = threadIdx.x; e < nseq * N; e += blockDim.x) {
    const int s = e / N, t = e - s * N;
    const int f = f0 + s / p.CC, c = c0 + s % p.CC;
    double v = 0.0;
    if (f < p.frames && c < p.C)
      v = __dmul_rn(padded_sample(xs + (size_t)c * p.n, p.n, half, (int64_t)f * p.hop + t), __ldg(p.window + t));
    a[(size_t)s * N + bitrev(t, logN)] = make_double2(v, 0.0);
  }
  __syncthreads();
  block_fft(a, nseq, N, logN, p.tw);
  // [bin][frame][channel]: for one bin the block's frames x channels are contiguous
  const int nb = p.bin_hi - p.bin_lo;
  const int fcount = min(p.PF, p.frames - f0), ccount = min(p.CC, p.C - c0);
  const int per_bin = fcount * ccount;
  for (int e = threadIdx.x; e < nb * per_bin; e += blockDim.x) {
    const int ib = e / per_bin, r = e - ib * per_bin;
    const int fi = r / ccount, ci = r - fi * ccount;
    const double2 v = a[(size_t)(fi * p.CC + ci) * N + p.bin_lo + ib];
    const size_t o = (((size_t)sig * nb + ib) * p.frames + f0 + fi) * p.C + c0 + ci;
    if (p.out_f32)
      reinterpret_cast<float2*>(p.spec)[o] = make_float2((float)v.x, (float)v.y);
    else
      reinterpret_cast<double2*>(p.spec)[o] = v;
  }
}

// Inverse transform of each (frame, channel) with the Hermitian extension
// (stft.cpp:118-122), scaled and windowed: frames_buf[s][c][f][t].
__global__ void __launch_bounds__(256) istft_frame_kernel(const IstftParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* a = reinterpret_cast<double2*>(smem_raw);
  const int N = p.N, logN = p.logN;
  const int f0 = blockIdx.x * p.PF, sig = blockIdx.y, c0 = blockIdx.z * p.CC;
  const int nseq = p.PF * p.CC;
  const double2* sp = p.spec + (size_t)sig * p.bins * p.frames * p.C;
  for (int e = threadIdx.x; e < nseq * N; e += blockDim.x) {
    const int s = e / N, i = e - s * N;
    const int f = f0 + s / p.CC, c = c0 + s % p.CC;
    double2 v = make_double2(0.0, 0.0);
    if (f < p.frames && c < p.C) {
      if (i < p.bins) {
        v = sp[((size_t)i * p.frames + f) * p.C + c];
      } else {
        v = sp[((size_t)(N - i) * p.frames + f) * p.C + c];
        v.y = -v.y;
      }
    }
    a[(size_t)s * N + bitrev(i, logN)] = v;
  }
  __syncthreads();
  block_fft(a, nseq, N, logN, p.tw);
  for (int e = threadIdx.x; e < nseq * N; e += blockDim.x) {
    const int s = e / N, t = e - s * N;
    const int f = f0 + s / p.CC, c = c0 + s % p.CC;
    if (f < p.frames && c < p.C)
      p.frames_buf[(((size_t)sig * p.C + c) * p.frames + f) * N + t] =
          __dmul_rn(__dmul_rn(a[(size_t)s * N + t].x, p.scale), __ldg(p.window + t));
  }
}

// Overlap-add in frame order and division by the squared-window overlap
// accumulated in the same order (stft.cpp:101-104, 123-130).
__global__ void __launch_bounds__(256) ola_kernel(const IstftParams p) {
  const int64_t total = (int64_t)p.S * p.C * p.out_len;
  const int N = p.N, half = N >> 1;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t sc = e / p.out_len, t = e - sc * p.out_len;
    const int64_t pos = half + t;
    int64_t jlo = pos - N + 1 > 0 ? (pos - N + 1 + p.hop - 1) / p.hop : 0;
    int64_t jhi = pos / p.hop;
    if (jhi > p.frames - 1) jhi = p.frames - 1;
    const double* fb = p.frames_buf + (size_t)sc * p.frames * N;
    double acc = 0.0, ov = 0.0;
    for (int64_t j = jlo; j <= jhi; ++j) {
      const int tt = (int)(pos - j * p.hop);
      const double w = __ldg(p.window + tt);
      acc = __dadd_rn(acc, fb[(size_t)j * N + tt]);
      ov = __dadd_rn(ov, __dmul_rn(w, w));
    }
    p.out[e] = __ddiv_rn(acc, ov);
  }
}

}  // namespace ctf
