// ctf_ops.cu — op-level C ABI (include/ctf_iss.h, "op-level entries"): the
// reference's individual estimator operations (proj/include/ctfmnmf/
// estimator.hpp:56-117, model.hpp:86-88) on the GPU, fp64, for callers and
// tests that drive the loop piece by piece the way test_estimator.cpp does.
// The fused iteration kernels (ctf_gram.cuh, ctf_kernels.cuh, ctf_fsplit.cuh)
// are the production path; these are plain one-op kernels with the same
// layouts as the rest of the ABI:
//   W      [F] column-major R x D complex        Y [F] column-major R x T complex
//   x      [F][T][D] complex (per bin column-major D x T)
//   B      sources concatenated, B_n column-major F x K_n
//   V      sources concatenated, V_n column-major K_n x T
//   lambda N x (column-major F x T)
// Pointers are host memory (mem = CTF_MEM_HOST: copied in and out, the call
// synchronises) or device memory on the context's device (CTF_MEM_DEVICE:
// stream-ordered on ctf_stream(ctx); errors found on the device are still
// reported, which synchronises).
#include "ctf_kernels.cuh"
#include "../../include/ctf_iss.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

struct OpError : std::runtime_error {
  int code, kind, bin, row;
  OpError(int c, const std::string& m, int k = 0, int b = -1, int r = -1)
      : std::runtime_error(m), code(c), kind(k), bin(b), row(r) {}
};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw OpError(CTF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define OCK(x) ck((x), #x)

template <class Fn>
int op_guard(ctf_ctx* ctx, ctf_err* err, Fn&& fn) {
  if (err) {
    std::memset(err, 0, sizeof(*err));
    err->iteration = err->mixture = err->bin = err->row = -1;
  }
  try {
    if (!ctx) throw OpError(CTF_ERR_CONFIG, "null context");
    cudaStream_t st = (cudaStream_t)ctf_stream(ctx);
    int dev = 0;
    OCK(cudaStreamGetDevice(st, &dev));
    OCK(cudaSetDevice(dev));
    fn(st);
    return CTF_OK;
  } catch (const OpError& e) {
    if (err) {
      err->code = e.code;
      err->kind = e.kind;
      err->bin = e.bin;
      err->row = e.row;
      std::snprintf(err->msg, sizeof(err->msg), "%s", e.what());
    }
    return e.code;
  } catch (const std::exception& e) {
    if (err) {
      err->code = CTF_ERR_CUDA;
      std::snprintf(err->msg, sizeof(err->msg), "%s", e.what());
    }
    return CTF_ERR_CUDA;
  }
}

// A caller buffer on the device: the caller's own pointer (device memory) or
// a stream-ordered copy of the host buffer, written back on commit().
struct Arg {
  double* d = nullptr;
  double* host = nullptr;
  size_t n = 0;
  bool owned = false;
  cudaStream_t st = nullptr;
  Arg(const double* p, size_t count, int mem, cudaStream_t s, bool copy_in = true) : n(count), st(s) {
    if (mem == CTF_MEM_DEVICE) {
      d = const_cast<double*>(p);
      return;
    }
    host = const_cast<double*>(p);
    owned = true;
    OCK(cudaMallocAsync((void**)&d, std::max<size_t>(1, n) * sizeof(double), st));
    if (copy_in && n) OCK(cudaMemcpyAsync(d, p, n * sizeof(double), cudaMemcpyHostToDevice, st));
  }
  void commit() {
    if (owned && n) OCK(cudaMemcpyAsync(host, d, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  ~Arg() {
    if (owned && d) cudaFreeAsync(d, st);
  }
  Arg(const Arg&) = delete;
  Arg& operator=(const Arg&) = delete;
};

template <class T>
struct Scratch {
  T* p = nullptr;
  cudaStream_t st;
  Scratch(size_t n, cudaStream_t s) : st(s) { OCK(cudaMallocAsync((void**)&p, std::max<size_t>(1, n) * sizeof(T), st)); }
  ~Scratch() { cudaFreeAsync(p, st); }
};

struct Shape {
  int F, T, N, R, SK;
  int taps[CTF_MAX_SOURCES], bases[CTF_MAX_SOURCES], row0[CTF_MAX_SOURCES], koff[CTF_MAX_SOURCES + 1];
};

Shape shape_of(const ctf_problem* p) {
  if (!p) throw OpError(CTF_ERR_CONFIG, "null problem");
  Shape s{};
  s.F = p->num_bins;
  s.T = p->num_frames;
  s.N = p->num_sources;
  if (s.N < 1 || s.N > CTF_MAX_SOURCES) throw OpError(CTF_ERR_CONFIG, "n_sources must be in [1, 16]");
  if (s.F < 1 || s.T < 1) throw OpError(CTF_ERR_CONFIG, "num_bins and num_frames must be >= 1");
  int r = 0, k = 0;
  for (int n = 0; n < s.N; ++n) {
    s.taps[n] = p->taps_per_source[n];
    s.bases[n] = p->bases_per_source[n];
    if (s.taps[n] < 1) throw OpError(CTF_ERR_CONFIG, "every tap count must be >= 1");
    if (s.bases[n] < 1) throw OpError(CTF_ERR_CONFIG, "every basis count must be >= 1");
    s.row0[n] = r;
    s.koff[n] = k;
    r += s.taps[n];
    k += s.bases[n];
  }
  s.koff[s.N] = k;
  s.R = r;
  s.SK = k;
  if (s.R > CTF_MAX_ROWS) throw OpError(CTF_ERR_UNSUPPORTED, "op-level entries support up to 64 demixing rows");
  return s;
}

__device__ __forceinline__ double2 cmul2(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------------------
// demix (estimator.cpp:304-311): Y_i = W_i x_i
__global__ void op_demix_kernel(const double2* W, const double2* x, double2* Y, int R, int D, int T) {
  const int f = blockIdx.y, t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const double2* w = W + (size_t)f * R * D;
  const double2* xc = x + ((size_t)f * T + t) * D;
  double2* y = Y + ((size_t)f * T + t) * R;
  for (int r = 0; r < R; ++r) {
    double2 acc = make_double2(0.0, 0.0);
    for (int c = 0; c < D; ++c) {
      const double2 p = cmul2(w[r + (size_t)c * R], xc[c]);
      acc.x += p.x;
      acc.y += p.y;
    }
    y[r] = acc;
  }
}

// compute_psd (model.cpp:210-215): lambda_n = max(B_n V_n, floor)
struct OpShape {
  int F, T, N, R, SK;
  int taps[CTF_MAX_SOURCES], row0[CTF_MAX_SOURCES], koff[CTF_MAX_SOURCES + 1];
};
OpShape op_shape(const Shape& s) {
  OpShape o{};
  o.F = s.F;
  o.T = s.T;
  o.N = s.N;
  o.R = s.R;
  o.SK = s.SK;
  for (int n = 0; n < s.N; ++n) {
    o.taps[n] = s.taps[n];
    o.row0[n] = s.row0[n];
    o.koff[n] = s.koff[n];
  }
  o.koff[s.N] = s.koff[s.N];
  return o;
}
__device__ __forceinline__ const double* b_of(const double* B, const OpShape& s, int n) {
  return B + (size_t)s.F * s.koff[n];
}
__device__ __forceinline__ const double* v_of(const double* V, const OpShape& s, int n) {
  return V + (size_t)s.T * s.koff[n];
}
__device__ __forceinline__ double psd_at(const double* Bn, const double* Vn, int K, int F, int f, int t,
                                         double floor_abs) {
  double acc = 0.0;
  for (int k = 0; k < K; ++k) acc += Bn[f + (size_t)k * F] * Vn[k + (size_t)t * K];
  return fmax(acc, floor_abs);
}
__global__ void op_psd_kernel(const double* B, const double* V, double* lambda, OpShape s, double floor_abs) {
  const int n = blockIdx.y;
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)s.F * s.T) return;
  const int f = (int)(e % s.F), t = (int)(e / s.F);
  const int K = s.koff[n + 1] - s.koff[n];
  lambda[(size_t)n * s.F * s.T + e] = psd_at(b_of(B, s, n), v_of(V, s, n), K, s.F, f, t, floor_abs);
}

// iss_sweep (estimator.cpp:434-484, 505-511) on every bin: one CTA per bin,
// R steps; step r: per row p the weighted sums over frames j >= l_p with
// w = 1 / lambda_{n_p}(bin, j - l_p), z, then W -= z w_r, Y -= z y_r.
constexpr int kOpNT = 256;
__global__ void __launch_bounds__(kOpNT) op_iss_sweep_kernel(double2* W, double2* Y, const double* lambda, OpShape s,
                                                             int D, unsigned long long* err) {
  const int bin = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kOpNT / 32;
  const int R = s.R, T = s.T, F = s.F;
  __shared__ double part[NW][CTF_MAX_ROWS][3];
  __shared__ double2 z[CTF_MAX_ROWS];
  __shared__ double2 wr[CTF_MAX_ROWS];
  __shared__ int srow[CTF_MAX_ROWS], stap[CTF_MAX_ROWS];
  __shared__ int s_bad;
  double2* w = W + (size_t)bin * R * D;
  double2* y = Y + (size_t)bin * R * T;
  if (tid < R) {
    int n = 0;
    while (tid >= s.row0[n] + s.taps[n]) ++n;
    srow[tid] = n;
    stap[tid] = tid - s.row0[n];
  }
  constexpr int kNone = 1 << 30;
  if (tid == 0) s_bad = kNone;
  __syncthreads();
  for (int r = 0; r < R; ++r) {
    for (int p = 0; p < R; ++p) {
      const double* lam = lambda + (size_t)srow[p] * F * T;
      const int l = stap[p];
      double nre = 0.0, nim = 0.0, den = 0.0;
      for (int j = l + tid; j < T; j += kOpNT) {
        const double wt = 1.0 / lam[bin + (size_t)(j - l) * F];
        const double2 yr = y[r + (size_t)j * R], yp = y[p + (size_t)j * R];
        den += (yr.x * yr.x + yr.y * yr.y) * wt;
        nre += (yp.x * yr.x + yp.y * yr.y) * wt;  // y_p conj(y_r)
        nim += (yp.y * yr.x - yp.x * yr.y) * wt;
      }
      nre = warp_sum(nre);
      nim = warp_sum(nim);
      den = warp_sum(den);
      if (lane == 0) {
        part[warp][p][0] = nre;
        part[warp][p][1] = nim;
        part[warp][p][2] = den;
      }
    }
    __syncthreads();
    if (tid < R) {
      const int p = tid;
      double nre = 0.0, nim = 0.0, den = 0.0;
      for (int q = 0; q < NW; ++q) {
        nre += part[q][p][0];
        nim += part[q][p][1];
        den += part[q][p][2];
      }
      if (!(den > 0.0) || !isfinite(den)) {
        atomicMin(&s_bad, p);  // the reference throws at the first failing p (:451-454)
        z[p] = make_double2(0.0, 0.0);
      } else if (p == r) {
        z[p] = make_double2(1.0 - sqrt((double)T / den), 0.0);
      } else {
        z[p] = make_double2(nre / den, nim / den);
      }
    }
    for (int c = tid; c < D; c += kOpNT) wr[c] = w[r + (size_t)c * R];  // pre-update row r
    __syncthreads();
    if (s_bad != kNone) {
      if (tid == 0) {
        const unsigned long long key = ((unsigned long long)bin << 20) | ((unsigned long long)r << 8) | s_bad;
        atomicMin(err, key);
      }
      return;
    }
    for (int e = tid; e < R * D; e += kOpNT) {  // iss_apply (:298-302)
      const int p = e % R, c = e / R;
      const double2 t = cmul2(z[p], wr[c]);
      w[e].x -= t.x;
      w[e].y -= t.y;
    }
    for (int j = tid; j < T; j += kOpNT) {  // y -= z y_r with the pre-update y_r
      const double2 yr = y[r + (size_t)j * R];
      for (int p = 0; p < R; ++p) {
        const double2 t = cmul2(z[p], yr);
        y[p + (size_t)j * R].x -= t.x;
        y[p + (size_t)j * R].y -= t.y;
      }
    }
    __syncthreads();
  }
}

// delayed energy E(i, tau) = sum_{l < L_n, tau + l < T} |y_{row0 + l}(tau + l)|^2 (estimator.cpp:318-330)
__device__ __forceinline__ double energy_at(const double2* y, int R, int T, int row0, int L, int tau) {
  double e = 0.0;
  for (int l = 0; l < L && tau + l < T; ++l) {
    const double2 v = y[row0 + l + (size_t)(tau + l) * R];
    e += v.x * v.x + v.y * v.y;
  }
  return e;
}

// mu_update_bases (estimator.cpp:313-346) for one source: one CTA per bin
__global__ void __launch_bounds__(kOpNT) op_mu_bases_kernel(double* B, const double* V, const double2* Y, OpShape s,
                                                            int n, double floor_abs) {
  const int f = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kOpNT / 32;
  const int T = s.T, F = s.F, K = s.koff[n + 1] - s.koff[n], L = s.taps[n];
  extern __shared__ double sm[];  // [T] E / lambda^2, [T] count / lambda, [K] new B row
  double* a = sm;
  double* b = sm + T;
  __shared__ double red[2][NW];
  double* Bn = B + (size_t)F * s.koff[n];
  const double* Vn = V + (size_t)T * s.koff[n];
  const double2* y = Y + (size_t)f * s.R * T;
  for (int t = tid; t < T; t += kOpNT) {
    const double lam = psd_at(Bn, Vn, K, F, f, t, floor_abs);
    const double inv = 1.0 / lam;
    a[t] = energy_at(y, s.R, T, s.row0[n], L, t) * (inv * inv);
    b[t] = inv * (double)min(L, T - t);
  }
  __syncthreads();
  for (int k = 0; k < K; ++k) {
    double num = 0.0, den = 0.0;
    for (int t = tid; t < T; t += kOpNT) {
      const double v = Vn[k + (size_t)t * K];
      num += a[t] * v;
      den += b[t] * v;
    }
    num = warp_sum(num);
    den = warp_sum(den);
    if (lane == 0) {
      red[0][warp] = num;
      red[1][warp] = den;
    }
    __syncthreads();
    if (tid == 0) {
      double nn = 0.0, dd = 0.0;
      for (int q = 0; q < NW; ++q) {
        nn += red[0][q];
        dd += red[1][q];
      }
      sm[2 * T + k] = fmax(Bn[f + (size_t)k * F] * sqrt(nn / dd), floor_abs);  // staged until every k is done
    }
    __syncthreads();
  }
  for (int k = tid; k < K; k += kOpNT) Bn[f + (size_t)k * F] = sm[2 * T + k];
}

// mu_update_activations (estimator.cpp:348-382, all taps) for one source:
// thread per frame, sums over every bin in bin order
__global__ void __launch_bounds__(128) op_mu_activations_kernel(const double* B, double* V, const double2* Y,
                                                                OpShape s, int n, double floor_abs) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int T = s.T, F = s.F, K = s.koff[n + 1] - s.koff[n], L = s.taps[n];
  if (t >= T) return;
  const double* Bn = B + (size_t)F * s.koff[n];
  double* Vn = V + (size_t)T * s.koff[n];
  double num[CTF_MAX_ROWS], den[CTF_MAX_ROWS];
  for (int k = 0; k < K; ++k) num[k] = den[k] = 0.0;
  const double cnt = (double)min(L, T - t);
  for (int f = 0; f < F; ++f) {
    const double lam = psd_at(Bn, Vn, K, F, f, t, floor_abs);
    const double inv = 1.0 / lam;
    const double e = energy_at(Y + (size_t)f * s.R * T, s.R, T, s.row0[n], L, t) * (inv * inv);
    for (int k = 0; k < K; ++k) {
      const double b = Bn[f + (size_t)k * F];
      num[k] += b * e;
      den[k] += b * (inv * cnt);
    }
  }
  for (int k = 0; k < K; ++k) Vn[k + (size_t)t * K] = fmax(Vn[k + (size_t)t * K] * sqrt(num[k] / den[k]), floor_abs);
}

// rescale (estimator.cpp:384-412): row powers per bin, mu in bin order, apply
__global__ void __launch_bounds__(kOpNT) op_rowpow_kernel(const double2* Y, double* rowpow, int R, int T) {
  const int f = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kOpNT / 32;
  __shared__ double red[NW];
  const double2* y = Y + (size_t)f * R * T;
  for (int r = 0; r < R; ++r) {
    double acc = 0.0;
    for (int j = tid; j < T; j += kOpNT) {
      const double2 v = y[r + (size_t)j * R];
      acc += v.x * v.x + v.y * v.y;
    }
    acc = warp_sum(acc);
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
      for (int q = 0; q < NW; ++q) s += red[q];
      rowpow[(size_t)f * R + r] = s;
    }
    __syncthreads();
  }
}
__global__ void op_mu_kernel(const double* rowpow, double* mu, int F, int R, int T) {
  const int r = threadIdx.x;
  if (r >= R) return;
  double p = 0.0;
  for (int f = 0; f < F; ++f) p += rowpow[(size_t)f * R + r];
  mu[r] = sqrt(p / ((double)F * T));
}
__global__ void op_rescale_apply_kernel(double2* W, double2* Y, double* B, const double* mu, OpShape s, int D,
                                        double floor_abs) {
  const int f = blockIdx.x, tid = threadIdx.x;
  const int R = s.R, T = s.T, F = s.F;
  for (int e = tid; e < R * D; e += blockDim.x) {
    const double m = mu[e % R];
    if (m != 0.0) {
      double2& w = W[(size_t)f * R * D + e];
      w.x /= m;
      w.y /= m;
    }
  }
  for (size_t e = tid; e < (size_t)R * T; e += blockDim.x) {
    const double m = mu[e % R];
    if (m != 0.0) {
      double2& v = Y[(size_t)f * R * T + e];
      v.x /= m;
      v.y /= m;
    }
  }
  for (int n = 0; n < s.N; ++n) {
    const double m0 = mu[s.row0[n]];
    if (m0 == 0.0) continue;
    double* Bn = B + (size_t)F * s.koff[n];
    for (int k = tid; k < s.koff[n + 1] - s.koff[n]; k += blockDim.x)
      Bn[f + (size_t)k * F] = fmax(Bn[f + (size_t)k * F] / (m0 * m0), floor_abs);
  }
}

// objective_from_parts (estimator.cpp:55-77), source-model terms per bin
__global__ void __launch_bounds__(kOpNT) op_objective_kernel(const double* lambda, const double2* Y, double* part,
                                                             OpShape s) {
  const int f = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = kOpNT / 32;
  __shared__ double red[NW];
  const int R = s.R, T = s.T, F = s.F;
  double acc = 0.0;
  for (int n = 0; n < s.N; ++n) {
    const double* lam = lambda + (size_t)n * F * T;
    for (int l = 0; l < s.taps[n]; ++l) {
      const int r = s.row0[n] + l;
      for (int j = l + tid; j < T; j += kOpNT) {
        const double lv = lam[f + (size_t)(j - l) * F];
        const double2 v = Y[((size_t)f * T + j) * R + r];
        acc += log(lv) + (v.x * v.x + v.y * v.y) / lv;
      }
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (tid == 0) {
    double sum = 0.0;
    for (int q = 0; q < NW; ++q) sum += red[q];
    part[f] = sum;
  }
}

void check_launch() { OCK(cudaGetLastError()); }

std::vector<double> logdets(const double* Wd, int R, int nb, cudaStream_t st) {
  Scratch<double> ld((size_t)nb, st);
  const size_t smem = (size_t)R * R * 16;
  OCK(cudaFuncSetAttribute((const void*)ctf::logdet_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem));
  ctf::logdet_kernel<double><<<nb, 32, smem, st>>>(Wd, ld.p, R, nb);
  check_launch();
  std::vector<double> h((size_t)nb);
  OCK(cudaMemcpyAsync(h.data(), ld.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
  OCK(cudaStreamSynchronize(st));
  for (int b = 0; b < nb; ++b) {  // log_abs_det (estimator.cpp:41-53)
    if (h[(size_t)b] == -INFINITY || std::isnan(h[(size_t)b]))
      throw OpError(CTF_ERR_DEGENERACY, "singular demixing matrix (zero pivot)", CTF_KIND_ZERO_PIVOT);
    if (h[(size_t)b] < std::log(1e-300))
      throw OpError(CTF_ERR_DEGENERACY, "demixing determinant magnitude below 1e-300", CTF_KIND_TINY_DET);
  }
  return h;
}

}  // namespace

extern "C" {

int ctf_op_demix(ctf_ctx* ctx, int F, int R, int D, int T, const double* W, const double* x, double* Y, int mem,
                 ctf_err* err) {
  return op_guard(ctx, err, [&](cudaStream_t st) {
    if (F < 1 || R < 1 || D < 1 || T < 1) throw OpError(CTF_ERR_CONFIG, "demix: empty shape");
    Arg w(W, (size_t)F * R * D * 2, mem, st), xx(x, (size_t)F * T * D * 2, mem, st),
        y(Y, (size_t)F * T * R * 2, mem, st, false);
    op_demix_kernel<<<dim3((T + 127) / 128, F), 128, 0, st>>>((const double2*)w.d, (const double2*)xx.d,
                                                               (double2*)y.d, R, D, T);
    check_launch();
    y.commit();
    if (mem == CTF_MEM_HOST) OCK(cudaStreamSynchronize(st));
  });
}

int ctf_op_compute_psd(ctf_ctx* ctx, const ctf_problem* prob, const double* B, const double* V, double floor_abs,
                       double* lambda, int mem, ctf_err* err) {
  return op_guard(ctx, err, [&](cudaStream_t st) {
    const Shape s = shape_of(prob);
    Arg b(B, (size_t)s.F * s.SK, mem, st), v(V, (size_t)s.SK * s.T, mem, st),
        l(lambda, (size_t)s.N * s.F * s.T, mem, st, false);
    const size_t ft = (size_t)s.F * s.T;
    op_psd_kernel<<<dim3((unsigned)((ft + 255) / 256), s.N), 256, 0, st>>>(b.d, v.d, l.d, op_shape(s), floor_abs);
    check_launch();
    l.commit();
    if (mem == CTF_MEM_HOST) OCK(cudaStreamSynchronize(st));
  });
}

int ctf_op_iss_sweep(ctf_ctx* ctx, const ctf_problem* prob, double* W, double* Y, const double* lambda, int mem,
                     ctf_err* err) {
  return op_guard(ctx, err, [&](cudaStream_t st) {
    const Shape s = shape_of(prob);
    const int D = s.R;  // square demixing system (model.cpp:43-46)
    Arg w(W, (size_t)s.F * s.R * D * 2, mem, st), y(Y, (size_t)s.F * s.T * s.R * 2, mem, st),
        l(lambda, (size_t)s.N * s.F * s.T, mem, st);
    Scratch<unsigned long long> e(1, st);
    OCK(cudaMemsetAsync(e.p, 0xFF, 8, st));
    op_iss_sweep_kernel<<<s.F, kOpNT, 0, st>>>((double2*)w.d, (double2*)y.d, l.d, op_shape(s), D, e.p);
    check_launch();
    unsigned long long key = 0;
    OCK(cudaMemcpyAsync(&key, e.p, 8, cudaMemcpyDeviceToHost, st));
    w.commit();
    y.commit();
    OCK(cudaStreamSynchronize(st));
    if (key != ~0ull) {  // lowest failing bin, its step and first failing row (estimator.cpp:451-454)
      const int bin = (int)(key >> 20), r = (int)((key >> 8) & 0xFFF), p = (int)(key & 0xFF);
      throw OpError(CTF_ERR_DEGENERACY,
                    "steering update: nonpositive denominator for rows (" + std::to_string(r) + ", " +
                        std::to_string(p) + ")",
                    CTF_KIND_STEERING_DENOM, bin, r);
    }
  });
}

int ctf_op_mu_update_bases(ctf_ctx* ctx, const ctf_problem* prob, double* B, const double* V, double floor_abs,
                           const double* Y, int source, int mem, ctf_err* err) {
  return op_guard(ctx, err, [&](cudaStream_t st) {
    const Shape s = shape_of(prob);
    if (source < 0 || source >= s.N) throw OpError(CTF_ERR_CONFIG, "source out of range");
    const size_t smem = ((size_t)2 * s.T + s.bases[source]) * sizeof(double);
    if (smem > 200 * 1024) throw OpError(CTF_ERR_UNSUPPORTED, "mu_update_bases: frame count over the op limit");
    Arg b(B, (size_t)s.F * s.SK, mem, st), v(V, (size_t)s.SK * s.T, mem, st),
        y(Y, (size_t)s.F * s.T * s.R * 2, mem, st);
    OCK(cudaFuncSetAttribute((const void*)op_mu_bases_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    op_mu_bases_kernel<<<s.F, kOpNT, smem, st>>>(b.d, v.d, (const double2*)y.d, op_shape(s), source, floor_abs);
    check_launch();
    b.commit();
    if (mem == CTF_MEM_HOST) OCK(cudaStreamSynchronize(st));
  });
}

int ctf_op_mu_update_activations(ctf_ctx* ctx, const ctf_problem* prob, const double* B, double* V, double floor_abs,
                                 const double* Y, int source, int mem, ctf_err* err) {
  return op_guard(ctx, err, [&](cudaStream_t st) {
    const Shape s = shape_of(prob);
    if (source < 0 || source >= s.N) throw OpError(CTF_ERR_CONFIG, "source out of range");
    if (s.bases[source] > CTF_MAX_ROWS) throw OpError(CTF_ERR_UNSUPPORTED, "mu_update_activations: K_n over 64");
    Arg b(B, (size_t)s.F * s.SK, mem, st), v(V, (size_t)s.SK * s.T, mem, st),
        y(Y, (size_t)s.F * s.T * s.R * 2, mem, st);
    op_mu_activations_kernel<<<(s.T + 127) / 128, 128, 0, st>>>(b.d, v.d, (const double2*)y.d, op_shape(s), source,
                                                               floor_abs);
    check_launch();
    v.commit();
    if (mem == CTF_MEM_HOST) OCK(cudaStreamSynchronize(st));
  });
}

int ctf_op_rescale(ctf_ctx* ctx, const ctf_problem* prob, double* W, double* B, double floor_abs, double* Y, int mem,
                   ctf_err* err) {
  return op_guard(ctx, err, [&](cudaStream_t st) {
    const Shape s = shape_of(prob);
    const int D = s.R;
    Arg w(W, (size_t)s.F * s.R * D * 2, mem, st), b(B, (size_t)s.F * s.SK, mem, st),
        y(Y, (size_t)s.F * s.T * s.R * 2, mem, st);
    Scratch<double> rp((size_t)s.F * s.R, st), mu((size_t)s.R, st);
    op_rowpow_kernel<<<s.F, kOpNT, 0, st>>>((const double2*)y.d, rp.p, s.R, s.T);
    op_mu_kernel<<<1, 64, 0, st>>>(rp.p, mu.p, s.F, s.R, s.T);
    op_rescale_apply_kernel<<<s.F, 256, 0, st>>>((double2*)w.d, (double2*)y.d, b.d, mu.p, op_shape(s), D, floor_abs);
    check_launch();
    w.commit();
    b.commit();
    y.commit();
    if (mem == CTF_MEM_HOST) OCK(cudaStreamSynchronize(st));
  });
}

int ctf_op_log_abs_det(ctf_ctx* ctx, int R, int num_bins, const double* W, double* out, int mem, ctf_err* err) {
  return op_guard(ctx, err, [&](cudaStream_t st) {
    if (R < 1 || R > CTF_MAX_ROWS || num_bins < 1) throw OpError(CTF_ERR_CONFIG, "log_abs_det: bad shape");
    Arg w(W, (size_t)num_bins * R * R * 2, mem, st);
    const std::vector<double> h = logdets(w.d, R, num_bins, st);
    if (mem == CTF_MEM_DEVICE)
      OCK(cudaMemcpyAsync(out, h.data(), h.size() * 8, cudaMemcpyHostToDevice, st));
    else
      std::memcpy(out, h.data(), h.size() * 8);
    OCK(cudaStreamSynchronize(st));
  });
}

int ctf_op_objective_from_parts(ctf_ctx* ctx, const ctf_problem* prob, const double* W, const double* lambda,
                                const double* Y, double* out, int mem, ctf_err* err) {
  return op_guard(ctx, err, [&](cudaStream_t st) {
    const Shape s = shape_of(prob);
    const int D = s.R;
    Arg w(W, (size_t)s.F * s.R * D * 2, mem, st), l(lambda, (size_t)s.N * s.F * s.T, mem, st),
        y(Y, (size_t)s.F * s.T * s.R * 2, mem, st);
    Scratch<double> part((size_t)s.F, st);
    op_objective_kernel<<<s.F, kOpNT, 0, st>>>(l.d, (const double2*)y.d, part.p, op_shape(s));
    check_launch();
    std::vector<double> hp((size_t)s.F);
    OCK(cudaMemcpyAsync(hp.data(), part.p, hp.size() * 8, cudaMemcpyDeviceToHost, st));
    const std::vector<double> ld = logdets(w.d, s.R, s.F, st);  // synchronises
    double obj = 0.0;  // bin order, as the reference accumulates (estimator.cpp:63-75)
    for (int i = 0; i < s.F; ++i) {
      obj += hp[(size_t)i];
      obj -= 2.0 * s.T * ld[(size_t)i];
    }
    if (mem == CTF_MEM_DEVICE)
      OCK(cudaMemcpyAsync(out, &obj, 8, cudaMemcpyHostToDevice, st));
    else
      *out = obj;
    OCK(cudaStreamSynchronize(st));
  });
}

}  // extern "C"
