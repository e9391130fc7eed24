// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// C ABI over the reference's OWN code: this file is compiled together with
// the unmodified /root/reference/proj/src/{estimator,model,wiener,stft,fft}.cpp
// (against oracle/ref_shims, an Eigen-API shim, because Eigen is absent here)
// into oracle/_ref/libctf_ref.so by oracle/Makefile.ref. Every entry point
// only marshals arrays into the reference's types and calls the reference
// function named in its comment; no algorithm is restated here.
//
// Layouts are the ones of oracle/ctf_oracle.h (so the restatement, the
// reference build and the GPU path compare element by element):
//   x : [F][T][D] complex (Spectrogram::data order, per bin column-major D x T)
//   W : [F] column-major R x D complex
//   B : sources concatenated, each B_n column-major F x K_n
//   V : sources concatenated, each V_n column-major K_n x T
//   Y : [F] column-major R x T complex;  lambda : N x (column-major F x T)
// Errors: ConfigError -> 2, IoError -> 3, DegeneracyError -> 4 (with its
// iteration / bin / row), anything else -> 9, as the CLI maps them
// (proj/tools/ctfmnmf_main.cpp:38-40).
#include "ctf_oracle.h"

#include "ctfmnmf/errors.hpp"
#include "ctfmnmf/estimator.hpp"
#include "ctfmnmf/fft.hpp"
#include "ctfmnmf/model.hpp"
#include "ctfmnmf/stft.hpp"
#include "ctfmnmf/wiener.hpp"

#include <cstring>
#include <random>
#include <string>
#include <vector>

using namespace ctfmnmf;

namespace {

using Cplx = std::complex<double>;

void set_err(orc_err* e, int code, const char* msg, int iteration = -1, int bin = -1, int row = -1) {
  if (!e) return;
  e->code = code;
  e->iteration = iteration;
  e->bin = bin;
  e->row = row;
  std::snprintf(e->msg, sizeof(e->msg), "%s", msg);
}

template <class F>
int guarded(orc_err* err, F&& f) {
  if (err) set_err(err, 0, "");
  try {
    f();
    return 0;
  } catch (const DegeneracyError& e) {
    set_err(err, 4, e.what(), e.iteration, e.bin, e.row);
    return 4;
  } catch (const ConfigError& e) {
    set_err(err, 2, e.what());
    return 2;
  } catch (const IoError& e) {
    set_err(err, 3, e.what());
    return 3;
  } catch (const std::exception& e) {
    set_err(err, 9, e.what());
    return 9;
  }
}

CtfConfig to_config(const orc_config* c) {
  CtfConfig cfg;
  cfg.num_sources = c->num_sources;
  cfg.num_channels = c->num_channels;
  cfg.taps_per_source.assign(c->taps, c->taps + c->num_sources);
  cfg.bases_per_source.assign(c->bases, c->bases + c->num_sources);
  cfg.iterations = c->iterations;
  cfg.update_rule = c->rule == 0 ? UpdateRule::Ip : UpdateRule::Iss;
  cfg.psd_floor = c->psd_floor;
  cfg.seed = c->seed;
  cfg.threads = c->threads;
  return cfg;
}

const Cplx* cplx(const double* p) { return reinterpret_cast<const Cplx*>(p); }
Cplx* cplx(double* p) { return reinterpret_cast<Cplx*>(p); }

MixtureSpectrogram to_mixture(int F, int T, int D, const double* x) {
  MixtureSpectrogram m;
  m.bins.resize(static_cast<size_t>(F));
  for (int i = 0; i < F; ++i) {
    m.bins[static_cast<size_t>(i)].resize(D, T);
    std::memcpy(m.bins[static_cast<size_t>(i)].data(), cplx(x) + static_cast<size_t>(i) * D * T,
                sizeof(Cplx) * static_cast<size_t>(D) * T);
  }
  return m;
}

std::vector<Eigen::MatrixXcd> to_bins(int F, int rows, int cols, const double* p) {
  std::vector<Eigen::MatrixXcd> out(static_cast<size_t>(F));
  for (int i = 0; i < F; ++i) {
    out[static_cast<size_t>(i)].resize(rows, cols);
    std::memcpy(out[static_cast<size_t>(i)].data(), cplx(p) + static_cast<size_t>(i) * rows * cols,
                sizeof(Cplx) * static_cast<size_t>(rows) * cols);
  }
  return out;
}

void from_bins(const std::vector<Eigen::MatrixXcd>& bins, double* p) {
  size_t off = 0;
  for (const auto& b : bins) {
    std::memcpy(cplx(p) + off, b.data(), sizeof(Cplx) * static_cast<size_t>(b.size()));
    off += static_cast<size_t>(b.size());
  }
}

NmfFactors to_factors(const orc_config* c, int F, int T, const double* B, const double* V, double floor_abs) {
  NmfFactors f;
  f.floor = floor_abs;
  size_t ob = 0, ov = 0;
  for (int n = 0; n < c->num_sources; ++n) {
    const int k = c->bases[n];
    Eigen::MatrixXd b(F, k), v(k, T);
    std::memcpy(b.data(), B + ob, sizeof(double) * static_cast<size_t>(F) * k);
    std::memcpy(v.data(), V + ov, sizeof(double) * static_cast<size_t>(k) * T);
    ob += static_cast<size_t>(F) * k;
    ov += static_cast<size_t>(k) * T;
    f.bases.push_back(std::move(b));
    f.activations.push_back(std::move(v));
  }
  return f;
}

void from_factors(const NmfFactors& f, double* B, double* V) {
  size_t ob = 0, ov = 0;
  for (size_t n = 0; n < f.bases.size(); ++n) {
    if (B) std::memcpy(B + ob, f.bases[n].data(), sizeof(double) * static_cast<size_t>(f.bases[n].size()));
    if (V) std::memcpy(V + ov, f.activations[n].data(), sizeof(double) * static_cast<size_t>(f.activations[n].size()));
    ob += static_cast<size_t>(f.bases[n].size());
    ov += static_cast<size_t>(f.activations[n].size());
  }
}

std::vector<Eigen::MatrixXd> to_lambdas(int N, int F, int T, const double* lam) {
  std::vector<Eigen::MatrixXd> out(static_cast<size_t>(N));
  for (int n = 0; n < N; ++n) {
    out[static_cast<size_t>(n)].resize(F, T);
    std::memcpy(out[static_cast<size_t>(n)].data(), lam + static_cast<size_t>(n) * F * T,
                sizeof(double) * static_cast<size_t>(F) * T);
  }
  return out;
}

int rows_of(const orc_config* c) {
  int r = 0;
  for (int n = 0; n < c->num_sources; ++n) r += c->taps[n];
  return r;
}

}  // namespace

extern "C" {

/* run(), proj/src/estimator.cpp:513-657 (CheckOptions estimator.hpp:45-48).
 * checks_out (optional): [max_det_lemma_error, max_normalization_error,
 * checked_updates]. trace_ms_out (optional): [iters][3] demix, mu, rescale. */
int ref_run(const orc_config* c, int F, int T, const double* x, int det_lemma, int normalization,
            double* W_out, double* B_out, double* V_out, double* obj_out, double* trace_ms_out,
            double* checks_out, orc_err* err) {
  return guarded(err, [&] {
    const CtfConfig cfg = to_config(c);
    const MixtureSpectrogram mix = to_mixture(F, T, c->num_channels, x);
    CheckOptions chk;
    chk.det_lemma = det_lemma != 0;
    chk.normalization = normalization != 0;
    const SeparationResult res = run(cfg, mix, chk);
    if (W_out) from_bins(res.demixing, W_out);
    from_factors(res.factors, B_out, V_out);
    for (size_t t = 0; t < res.trace.objective.size(); ++t) {
      if (obj_out) obj_out[t] = res.trace.objective[t];
      if (trace_ms_out) {
        trace_ms_out[3 * t + 0] = res.trace.demix_ms[t];
        trace_ms_out[3 * t + 1] = res.trace.mu_ms[t];
        trace_ms_out[3 * t + 2] = res.trace.rescale_ms[t];
      }
    }
    if (checks_out) {
      checks_out[0] = res.trace.max_det_lemma_error;
      checks_out[1] = res.trace.max_normalization_error;
      checks_out[2] = static_cast<double>(res.trace.checked_updates);
    }
  });
}

/* MixtureSpectrogram::mean_power, proj/src/model.cpp:153-161 */
double ref_mean_power(int F, int D, int T, const double* x) { return to_mixture(F, T, D, x).mean_power(); }

/* random_factors with std::mt19937_64(seed), proj/src/model.cpp:189-208 */
int ref_random_factors(const orc_config* c, int F, int T, double floor_abs, double* B, double* V, orc_err* err) {
  return guarded(err, [&] {
    std::mt19937_64 rng(c->seed);
    from_factors(random_factors(to_config(c), F, T, floor_abs, rng), B, V);
  });
}

/* demix, proj/src/estimator.cpp:304-311 */
int ref_demix(int F, int R, int D, int T, const double* W, const double* x, double* Y, orc_err* err) {
  return guarded(err, [&] { from_bins(demix(to_bins(F, R, D, W), to_mixture(F, T, D, x)).bins, Y); });
}

/* iss_sweep on one bin, proj/src/estimator.cpp:505-511 (W_bin R x D and
 * Y_bin R x T updated in place) */
int ref_iss_sweep(const orc_config* c, int F, int T, int bin, double* W_bin, double* Y_bin, const double* lambda,
                  orc_err* err) {
  return guarded(err, [&] {
    const int R = rows_of(c);
    std::vector<Eigen::MatrixXcd> w = to_bins(1, R, c->num_channels, W_bin), y = to_bins(1, R, T, Y_bin);
    iss_sweep(w[0], y[0], to_lambdas(c->num_sources, F, T, lambda), to_config(c), bin);
    from_bins(w, W_bin);
    from_bins(y, Y_bin);
  });
}

/* compute_weighted_covariance, proj/src/estimator.cpp:89-101 */
int ref_weighted_covariance(int F, int D, int T, const double* x, const double* lambda_n, int tap, int bin,
                            double* Q, orc_err* err) {
  return guarded(err, [&] {
    const std::vector<Eigen::MatrixXd> lam = to_lambdas(1, F, T, lambda_n);
    from_bins({compute_weighted_covariance(to_mixture(F, T, D, x), lam[0], tap, bin)}, Q);
  });
}

/* iss_compute_z, proj/src/estimator.cpp:275-296 (covs: R matrices D x D) */
int ref_iss_compute_z(int R, const double* W_bin, const double* covs, int row, double* z, orc_err* err) {
  return guarded(err, [&] {
    const Eigen::VectorXcd zz = iss_compute_z(to_bins(1, R, R, W_bin)[0], to_bins(R, R, R, covs), row);
    std::memcpy(cplx(z), zz.data(), sizeof(Cplx) * static_cast<size_t>(R));
  });
}

/* iss_apply, proj/src/estimator.cpp:298-302 */
int ref_iss_apply(int R, int D, double* W_bin, const double* z, int row, orc_err* err) {
  return guarded(err, [&] {
    std::vector<Eigen::MatrixXcd> w = to_bins(1, R, D, W_bin);
    Eigen::VectorXcd zz(R);
    std::memcpy(zz.data(), cplx(z), sizeof(Cplx) * static_cast<size_t>(R));
    iss_apply(w[0], zz, row);
    from_bins(w, W_bin);
  });
}

/* ip_update, proj/src/estimator.cpp:251-273 (cov D x D) */
int ref_ip_update(int D, double* W_bin, const double* cov, int row, orc_err* err) {
  return guarded(err, [&] {
    std::vector<Eigen::MatrixXcd> w = to_bins(1, D, D, W_bin);
    ip_update(w[0], to_bins(1, D, D, cov)[0], row);
    from_bins(w, W_bin);
  });
}

/* compute_psd for every source, proj/src/model.cpp:210-215 */
int ref_compute_psd(const orc_config* c, int F, int T, const double* B, const double* V, double floor_abs,
                    double* lambda, orc_err* err) {
  return guarded(err, [&] {
    const NmfFactors f = to_factors(c, F, T, B, V, floor_abs);
    for (int n = 0; n < c->num_sources; ++n) {
      const Eigen::MatrixXd l = compute_psd(f, n);
      std::memcpy(lambda + static_cast<size_t>(n) * F * T, l.data(), sizeof(double) * static_cast<size_t>(F) * T);
    }
  });
}

/* mu_update_bases / mu_update_activations, proj/src/estimator.cpp:313-382 */
int ref_mu_update(const orc_config* c, int F, int T, double* B, double* V, double floor_abs, const double* Y,
                  int source, int activations, orc_err* err) {
  return guarded(err, [&] {
    NmfFactors f = to_factors(c, F, T, B, V, floor_abs);
    DelayedEstimates est;
    est.bins = to_bins(F, rows_of(c), T, Y);
    if (activations)
      mu_update_activations(f, est, source, to_config(c));
    else
      mu_update_bases(f, est, source, to_config(c));
    from_factors(f, B, V);
  });
}

/* rescale, proj/src/estimator.cpp:384-412 */
int ref_rescale(const orc_config* c, int F, int T, double* W, double* B, double* V, double floor_abs, double* Y,
                orc_err* err) {
  return guarded(err, [&] {
    const int R = rows_of(c);
    std::vector<Eigen::MatrixXcd> w = to_bins(F, R, c->num_channels, W);
    NmfFactors f = to_factors(c, F, T, B, V, floor_abs);
    DelayedEstimates est;
    est.bins = to_bins(F, R, T, Y);
    rescale(w, f, est, to_config(c));
    from_bins(w, W);
    from_factors(f, B, V);
    from_bins(est.bins, Y);
  });
}

/* log_abs_det, proj/src/estimator.cpp:41-53 */
int ref_log_abs_det(int R, const double* W_bin, double* out, orc_err* err) {
  return guarded(err, [&] { *out = log_abs_det(to_bins(1, R, R, W_bin)[0]); });
}

/* objective_from_parts, proj/src/estimator.cpp:55-77 */
int ref_objective_from_parts(const orc_config* c, int F, int T, const double* W, const double* lambda,
                             const double* Y, double* out, orc_err* err) {
  return guarded(err, [&] {
    const int R = rows_of(c);
    DelayedEstimates est;
    est.bins = to_bins(F, R, T, Y);
    *out = objective_from_parts(to_bins(F, R, c->num_channels, W), to_lambdas(c->num_sources, F, T, lambda), est,
                                to_config(c));
  });
}

/* objective, proj/src/estimator.cpp:79-87 */
int ref_objective(const orc_config* c, int F, int T, const double* W, const double* B, const double* V,
                  double floor_abs, const double* x, double* out, orc_err* err) {
  return guarded(err, [&] {
    *out = objective(to_bins(F, rows_of(c), c->num_channels, W), to_factors(c, F, T, B, V, floor_abs),
                     to_mixture(F, T, c->num_channels, x), to_config(c));
  });
}

/* reconstruct_images, proj/src/wiener.cpp:11-49. images: N x F x (D x T). */
int ref_reconstruct_images(const orc_config* c, int F, int T, const double* W, const double* B, const double* V,
                           double floor_abs, const double* x, double* images, orc_err* err) {
  return guarded(err, [&] {
    const std::vector<MixtureSpectrogram> im =
        reconstruct_images(to_bins(F, rows_of(c), c->num_channels, W), to_factors(c, F, T, B, V, floor_abs),
                           to_mixture(F, T, c->num_channels, x), to_config(c));
    size_t off = 0;
    for (const auto& m : im) {
      from_bins(m.bins, images + 2 * off);
      off += static_cast<size_t>(F) * c->num_channels * T;
    }
  });
}

/* fft_inplace, proj/src/fft.cpp:9-41 */
int ref_fft(double* data, int64_t n, int inverse, orc_err* err) {
  return guarded(err, [&] {
    if (!is_power_of_two(static_cast<size_t>(n))) throw ConfigError("fft length must be a power of two");
    fft_inplace(cplx(data), static_cast<size_t>(n), inverse != 0);
  });
}

/* forward_stft, proj/src/stft.cpp:46-88. samples [channels][length]; spec
 * [bins][frames][channels] complex (Spectrogram::data). dims_out: bins,
 * frames. spec may be NULL to query the dims. */
int ref_forward_stft(const double* samples, int64_t length, int channels, int window_len, int hop, double* spec,
                     int* dims_out, orc_err* err) {
  return guarded(err, [&] {
    TimeSignal sig;
    sig.sample_rate = 16000.0;
    sig.samples.resize(length, channels);
    std::memcpy(sig.samples.data(), samples, sizeof(double) * static_cast<size_t>(length) * channels);
    const Spectrogram s = forward_stft(sig, window_len, hop);
    dims_out[0] = s.bins;
    dims_out[1] = s.frames;
    if (spec) std::memcpy(spec, s.data.data(), sizeof(Cplx) * s.data.size());
  });
}

/* inverse_stft, proj/src/stft.cpp:90-139. out [channels][len] (may be NULL
 * to query the length). */
int ref_inverse_stft(const double* spec, int bins, int frames, int channels, int window_len, int hop,
                     int64_t original_length, double* out, int64_t* out_len, orc_err* err) {
  return guarded(err, [&] {
    Spectrogram s;
    s.resize(bins, frames, channels);
    s.window_len = window_len;
    s.hop = hop;
    s.sample_rate = 16000.0;
    s.original_length = original_length;
    std::memcpy(s.data.data(), spec, sizeof(Cplx) * s.data.size());
    const TimeSignal t = inverse_stft(s);
    *out_len = t.length();
    if (out) std::memcpy(out, t.samples.data(), sizeof(double) * static_cast<size_t>(t.samples.size()));
  });
}

}  // extern "C"
