// ctfmnmf_b200.cpp — the reference-shaped C++ API over the C ABI.
#include "ctfmnmf_b200.hpp"

#include "../../include/ctf_iss.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <sstream>

namespace ctfmnmf {
namespace b200 {

int CtfConfig::total_taps() const { return std::accumulate(taps_per_source.begin(), taps_per_source.end(), 0); }

int CtfConfig::row_offset(int source) const {
  int o = 0;
  for (int n = 0; n < source; ++n) o += taps_per_source[static_cast<size_t>(n)];
  return o;
}

void CtfConfig::validate() const {
  if (num_sources < 1) throw ConfigError("n_sources must be >= 1");
  if (num_channels < 1) throw ConfigError("n_channels must be >= 1");
  if (static_cast<int>(taps_per_source.size()) != num_sources)
    throw ConfigError("taps list must have one entry per source");
  if (static_cast<int>(bases_per_source.size()) != num_sources)
    throw ConfigError("bases list must have one entry per source");
  for (int l : taps_per_source)
    if (l < 1) throw ConfigError("every tap count must be >= 1");
  for (int k : bases_per_source)
    if (k < 1) throw ConfigError("every basis count must be >= 1");
  if (total_taps() != num_channels)
    throw ConfigError("sum of taps (" + std::to_string(total_taps()) + ") must equal n_channels (" +
                      std::to_string(num_channels) + "): the demixing system must be square");
  if (iterations < 0) throw ConfigError("iters must be >= 0");
  if (!(psd_floor > 0.0)) throw ConfigError("floor must be > 0");
  if (threads < 1) throw ConfigError("threads must be >= 1");
}

double MixtureSpectrogram::mean_power() const {
  double total = 0.0;
  std::int64_t count = 0;
  for (const auto& b : bins) {
    for (const auto& v : b.data) total += std::norm(v);
    count += static_cast<std::int64_t>(b.data.size());
  }
  return count > 0 ? total / static_cast<double>(count) : 0.0;
}

std::string OptimizationTrace::to_csv() const {  // estimator.cpp:15-23
  std::ostringstream out;
  out << "iter,objective,t_demix_ms,t_mu_ms,t_rescale_ms\n";
  out.precision(12);
  for (size_t t = 0; t < objective.size(); ++t)
    out << (t + 1) << ',' << objective[t] << ',' << demix_ms[t] << ',' << mu_ms[t] << ',' << rescale_ms[t] << '\n';
  return out.str();
}
double OptimizationTrace::total_demix_ms() const { return std::accumulate(demix_ms.begin(), demix_ms.end(), 0.0); }
double OptimizationTrace::total_mu_ms() const { return std::accumulate(mu_ms.begin(), mu_ms.end(), 0.0); }
double OptimizationTrace::total_rescale_ms() const {
  return std::accumulate(rescale_ms.begin(), rescale_ms.end(), 0.0);
}

namespace {

[[noreturn]] void rethrow(const ctf_err& e) {
  switch (e.code) {
    case CTF_ERR_CONFIG: throw ConfigError(e.msg);
    case CTF_ERR_IO: throw IoError(e.msg);
    case CTF_ERR_DEGENERACY: throw DegeneracyError(e.msg, e.iteration, e.bin, e.row);
    default: throw std::runtime_error(e.msg);
  }
}

struct Ctx {
  ctf_ctx* c = nullptr;
  explicit Ctx(int device) {
    ctf_err e{};
    if (ctf_open(device, &c, &e) != CTF_OK) rethrow(e);
  }
  ~Ctx() { ctf_close(c); }
};

ctf_problem make_problem(const CtfConfig& config, const MixtureSpectrogram& x, const GpuOptions& gpu) {
  config.validate();
  if (config.num_sources > CTF_MAX_SOURCES) throw ConfigError("too many sources");
  if (gpu.stack_taps < 1 || x.num_channels() * gpu.stack_taps != config.num_channels)
    throw ConfigError("mixture has " + std::to_string(x.num_channels() * gpu.stack_taps) +
                      " channels but config expects " + std::to_string(config.num_channels));
  ctf_problem p{};
  p.num_mixtures = 1;
  p.num_bins = x.num_bins();
  p.num_frames = x.num_frames();
  p.num_mics = x.num_channels();
  p.stack_taps = gpu.stack_taps;
  p.num_sources = config.num_sources;
  for (int n = 0; n < config.num_sources; ++n) {
    p.taps_per_source[n] = config.taps_per_source[static_cast<size_t>(n)];
    p.bases_per_source[n] = config.bases_per_source[static_cast<size_t>(n)];
  }
  p.iterations = config.iterations;
  p.update_rule = config.update_rule == UpdateRule::Iss ? CTF_RULE_ISS : CTF_RULE_IP;
  p.precision = gpu.precision == Precision::F32 ? CTF_F32 : CTF_F64;
  p.x_precision = CTF_F64;
  p.psd_floor = config.psd_floor;
  p.seed = config.seed;
  p.threads = config.threads;
  return p;
}

// [bin][frame][channel] interleaved doubles (the reference Spectrogram layout)
std::vector<double> flatten(const MixtureSpectrogram& x) {
  const int F = x.num_bins(), T = x.num_frames(), M = x.num_channels();
  std::vector<double> out(static_cast<size_t>(F) * T * M * 2);
  for (int i = 0; i < F; ++i)
    std::memcpy(out.data() + static_cast<size_t>(i) * T * M * 2, x.bins[static_cast<size_t>(i)].data.data(),
                static_cast<size_t>(T) * M * sizeof(Complex));
  return out;
}

}  // namespace

SeparationResult run(const CtfConfig& config, const MixtureSpectrogram& x, const GpuOptions& gpu) {
  return run(config, x, CheckOptions{}, gpu);
}

SeparationResult run(const CtfConfig& config, const MixtureSpectrogram& x, const CheckOptions& checks,
                     const GpuOptions& gpu) {
  ctf_problem p = make_problem(config, x, gpu);
  p.checks = (checks.det_lemma ? CTF_CHECK_DET_LEMMA : 0) | (checks.normalization ? CTF_CHECK_NORMALIZATION : 0);
  const int F = p.num_bins, T = p.num_frames, R = config.total_taps(), D = config.num_channels;
  const std::vector<double> xf = flatten(x);
  Ctx ctx(gpu.device);
  ctf_err e{};
  if (ctf_setup(ctx.c, &p, xf.data(), &e) != CTF_OK) rethrow(e);
  if (ctf_iterate(ctx.c, config.iterations, &e) != CTF_OK) rethrow(e);
  int sumK = 0;
  for (int k : config.bases_per_source) sumK += k;
  std::vector<double> W(static_cast<size_t>(F) * R * D * 2), B(static_cast<size_t>(F) * sumK),
      V(static_cast<size_t>(sumK) * T), obj(static_cast<size_t>(config.iterations));
  if (ctf_download(ctx.c, W.data(), B.data(), V.data(), obj.data(), &e) != CTF_OK) rethrow(e);
  SeparationResult res;
  res.demixing.assign(static_cast<size_t>(F), CMatrix(R, D));
  for (int i = 0; i < F; ++i)
    std::memcpy(res.demixing[static_cast<size_t>(i)].data.data(), W.data() + static_cast<size_t>(i) * R * D * 2,
                static_cast<size_t>(R) * D * sizeof(Complex));
  size_t ob = 0, ov = 0;
  for (int n = 0; n < config.num_sources; ++n) {
    const int K = config.bases_per_source[static_cast<size_t>(n)];
    RMatrix b(F, K), v(K, T);
    std::memcpy(b.data.data(), B.data() + ob, b.data.size() * 8);
    std::memcpy(v.data.data(), V.data() + ov, v.data.size() * 8);
    ob += b.data.size();
    ov += v.data.size();
    res.factors.bases.push_back(std::move(b));
    res.factors.activations.push_back(std::move(v));
  }
  ctf_psd_floor(ctx.c, &res.factors.floor);
  res.trace.objective = obj;
  res.trace.demix_ms.resize(obj.size());
  res.trace.mu_ms.resize(obj.size());
  res.trace.rescale_ms.resize(obj.size());
  ctf_trace_ms(ctx.c, res.trace.demix_ms.data(), res.trace.mu_ms.data(), res.trace.rescale_ms.data());
  if (p.checks)
    ctf_check_stats(ctx.c, &res.trace.max_det_lemma_error, &res.trace.max_normalization_error,
                    &res.trace.checked_updates);
  return res;
}

std::vector<MixtureSpectrogram> reconstruct_images(const std::vector<CMatrix>& demixing, const NmfFactors& factors,
                                                   const MixtureSpectrogram& x, const CtfConfig& config,
                                                   const GpuOptions& gpu) {
  if (static_cast<int>(factors.bases.size()) != config.num_sources)
    throw ConfigError("image reconstruction: factor count does not match config");
  CtfConfig c0 = config;
  c0.iterations = 0;
  const ctf_problem p = make_problem(c0, x, gpu);
  const int F = p.num_bins, T = p.num_frames, R = config.total_taps(), D = config.num_channels;
  const std::vector<double> xf = flatten(x);
  std::vector<double> W(static_cast<size_t>(F) * R * D * 2);
  for (int i = 0; i < F; ++i)
    std::memcpy(W.data() + static_cast<size_t>(i) * R * D * 2, demixing[static_cast<size_t>(i)].data.data(),
                static_cast<size_t>(R) * D * sizeof(Complex));
  Ctx ctx(gpu.device);
  ctf_err e{};
  if (ctf_setup(ctx.c, &p, xf.data(), &e) != CTF_OK) rethrow(e);
  if (ctf_set_state(ctx.c, W.data(), nullptr, nullptr, &e) != CTF_OK) rethrow(e);
  std::vector<double> img(static_cast<size_t>(config.num_sources) * F * T * D * 2);
  if (ctf_project_back(ctx.c, CTF_IMAGES_FULL, img.data(), &e) != CTF_OK) rethrow(e);
  std::vector<MixtureSpectrogram> out(static_cast<size_t>(config.num_sources));
  for (int n = 0; n < config.num_sources; ++n) {
    out[static_cast<size_t>(n)].bins.assign(static_cast<size_t>(F), CMatrix(D, T));
    for (int i = 0; i < F; ++i)
      std::memcpy(out[static_cast<size_t>(n)].bins[static_cast<size_t>(i)].data.data(),
                  img.data() + (static_cast<size_t>(n) * F + i) * T * D * 2, static_cast<size_t>(D) * T * sizeof(Complex));
  }
  return out;
}

MixtureSpectrogram MixtureSpectrogram::from_spectrogram(const Spectrogram& spec) {  // model.cpp
  MixtureSpectrogram m;
  m.bins.assign(static_cast<size_t>(spec.bins), CMatrix(spec.channels, spec.frames));
  for (int i = 0; i < spec.bins; ++i)
    for (int j = 0; j < spec.frames; ++j)
      for (int c = 0; c < spec.channels; ++c) m.bins[static_cast<size_t>(i)](c, j) = spec.at(i, j, c);
  return m;
}

Spectrogram MixtureSpectrogram::to_spectrogram(const Spectrogram& meta) const {
  Spectrogram s;
  s.window_len = meta.window_len;
  s.hop = meta.hop;
  s.sample_rate = meta.sample_rate;
  s.original_length = meta.original_length;
  s.resize(num_bins(), num_frames(), num_channels());
  for (int i = 0; i < s.bins; ++i)
    for (int j = 0; j < s.frames; ++j)
      for (int c = 0; c < s.channels; ++c) s.at(i, j, c) = bins[static_cast<size_t>(i)](c, j);
  return s;
}

std::vector<double> hann_window(int window_len) {  // stft.cpp:14-19
  std::vector<double> w(static_cast<size_t>(std::max(window_len, 0)));
  for (int t = 0; t < window_len; ++t)
    w[static_cast<size_t>(t)] = 0.5 - 0.5 * std::cos(2.0 * 3.14159265358979323846 * t / window_len);
  return w;
}

Spectrogram forward_stft(const TimeSignal& signal, int window_len, int hop, const GpuOptions& gpu) {
  Ctx ctx(gpu.device);
  ctf_err e{};
  const std::int64_t n = signal.length();
  const int chans = signal.channels();
  Spectrogram spec;
  const std::int64_t frames = hop > 0 ? ctf_stft_frames(n, hop) : 0;
  spec.resize(window_len > 0 ? window_len / 2 + 1 : 0, static_cast<int>(frames), chans);
  spec.window_len = window_len;
  spec.hop = hop;
  spec.sample_rate = signal.sample_rate;
  spec.original_length = n;
  if (ctf_stft(ctx.c, signal.samples.data.data(), n, chans, window_len, hop,
               reinterpret_cast<double*>(spec.data.data()), &e) != CTF_OK)
    rethrow(e);
  return spec;
}

TimeSignal inverse_stft(const Spectrogram& spec, const GpuOptions& gpu) {
  Ctx ctx(gpu.device);
  ctf_err e{};
  std::int64_t len = 0;
  const double* sp = reinterpret_cast<const double*>(spec.data.data());
  if (ctf_istft(ctx.c, sp, spec.bins, spec.frames, spec.channels, spec.window_len, spec.hop, spec.original_length,
                nullptr, &len, &e) != CTF_OK)
    rethrow(e);
  TimeSignal out;
  out.sample_rate = spec.sample_rate;
  out.samples = RMatrix(static_cast<int>(len), spec.channels);
  if (ctf_istft(ctx.c, sp, spec.bins, spec.frames, spec.channels, spec.window_len, spec.hop, spec.original_length,
                out.samples.data.data(), &len, &e) != CTF_OK)
    rethrow(e);
  return out;
}

TimeSignal image_to_signal(const MixtureSpectrogram& image, const Spectrogram& meta, int ref_channel,
                           const GpuOptions& gpu) {  // wiener.cpp:51-64
  TimeSignal all = inverse_stft(image.to_spectrogram(meta), gpu);
  if (ref_channel < 0) return all;
  if (ref_channel >= all.channels())
    throw ConfigError("ref_channel " + std::to_string(ref_channel) + " out of range for " +
                      std::to_string(all.channels()) + " channels");
  TimeSignal mono;
  mono.sample_rate = all.sample_rate;
  mono.samples = RMatrix(all.samples.rows, 1);
  std::copy(all.samples.data.begin() + static_cast<std::ptrdiff_t>(ref_channel) * all.samples.rows,
            all.samples.data.begin() + static_cast<std::ptrdiff_t>(ref_channel + 1) * all.samples.rows,
            mono.samples.data.begin());
  return mono;
}

void write_spectrogram(const std::string& path, const Spectrogram& spec) {  // container.cpp:61-72
  ctf_err e{};
  const ctf_spec_header h{(uint32_t)spec.bins,       (uint32_t)spec.frames, (uint32_t)spec.channels,
                          (uint32_t)spec.window_len, (uint32_t)spec.hop,    (uint32_t)spec.sample_rate,
                          (uint64_t)spec.original_length};
  if (ctf_write_spectrogram(path.c_str(), &h, spec.data.data(), CTF_F64, &e) != CTF_OK) rethrow(e);
}

Spectrogram read_spectrogram(const std::string& path) {  // container.cpp:74-86
  ctf_err e{};
  ctf_spec_header h{};
  if (ctf_read_spectrogram(path.c_str(), &h, nullptr, CTF_F64, &e) != CTF_OK) rethrow(e);
  Spectrogram s;
  s.resize((int)h.bins, (int)h.frames, (int)h.channels);
  s.window_len = (int)h.window_len;
  s.hop = (int)h.hop;
  s.sample_rate = (double)h.sample_rate;
  s.original_length = (std::int64_t)h.original_length;
  if (ctf_read_spectrogram(path.c_str(), &h, s.data.data(), CTF_F64, &e) != CTF_OK) rethrow(e);
  return s;
}

void write_factors(const std::string& path, const NmfFactors& f) {  // container.cpp:124-142
  ctf_err e{};
  const int N = (int)f.bases.size();
  if (N < 1) throw ConfigError("write_factors: no sources");
  std::vector<int32_t> ks;
  std::vector<double> B, V;
  for (int n = 0; n < N; ++n) {
    ks.push_back(f.bases[(size_t)n].cols);
    B.insert(B.end(), f.bases[(size_t)n].data.begin(), f.bases[(size_t)n].data.end());
    V.insert(V.end(), f.activations[(size_t)n].data.begin(), f.activations[(size_t)n].data.end());
  }
  if (ctf_write_factors(path.c_str(), N, f.bases[0].rows, f.activations[0].cols, ks.data(), f.floor, B.data(),
                        V.data(), &e) != CTF_OK)
    rethrow(e);
}

NmfFactors read_factors(const std::string& path) {  // container.cpp:144-165
  ctf_err e{};
  int N = 0, F = 0, T = 0;
  int32_t ks[CTF_MAX_SOURCES] = {0};
  double fl = 0.0;
  if (ctf_read_factors(path.c_str(), &N, &F, &T, ks, &fl, nullptr, nullptr, &e) != CTF_OK) rethrow(e);
  int sk = 0;
  for (int n = 0; n < N; ++n) sk += ks[n];
  std::vector<double> B((size_t)F * sk), V((size_t)sk * T);
  if (ctf_read_factors(path.c_str(), &N, &F, &T, ks, &fl, B.data(), V.data(), &e) != CTF_OK) rethrow(e);
  NmfFactors f;
  f.floor = fl;
  size_t ob = 0, ov = 0;
  for (int n = 0; n < N; ++n) {
    RMatrix b(F, ks[n]), v(ks[n], T);
    std::copy(B.begin() + (std::ptrdiff_t)ob, B.begin() + (std::ptrdiff_t)(ob + b.data.size()), b.data.begin());
    std::copy(V.begin() + (std::ptrdiff_t)ov, V.begin() + (std::ptrdiff_t)(ov + v.data.size()), v.data.begin());
    ob += b.data.size();
    ov += v.data.size();
    f.bases.push_back(std::move(b));
    f.activations.push_back(std::move(v));
  }
  return f;
}

// ---- op-level API ---------------------------------------------------------
namespace {

ctf_problem op_problem(const CtfConfig& config, int F, int T) {
  if (config.num_sources < 1 || config.num_sources > CTF_MAX_SOURCES) throw ConfigError("n_sources must be in [1, 16]");
  ctf_problem p{};
  p.num_mixtures = 1;
  p.num_bins = F;
  p.num_frames = T;
  p.num_sources = config.num_sources;
  p.stack_taps = 1;
  p.num_mics = config.total_taps();
  for (int n = 0; n < config.num_sources; ++n) {
    p.taps_per_source[n] = config.taps_per_source[static_cast<size_t>(n)];
    p.bases_per_source[n] =
        n < static_cast<int>(config.bases_per_source.size()) ? config.bases_per_source[static_cast<size_t>(n)] : 1;
  }
  return p;
}

std::vector<double> pack(const std::vector<CMatrix>& mats) {
  std::vector<double> out;
  for (const auto& m : mats)
    for (const auto& v : m.data) {
      out.push_back(v.real());
      out.push_back(v.imag());
    }
  return out;
}

void unpack(const std::vector<double>& buf, std::vector<CMatrix>& mats) {
  size_t k = 0;
  for (auto& m : mats)
    for (auto& v : m.data) {
      v = Complex(buf[k], buf[k + 1]);
      k += 2;
    }
}

std::vector<double> pack_factors(const std::vector<RMatrix>& fs) {
  std::vector<double> out;
  for (const auto& f : fs) out.insert(out.end(), f.data.begin(), f.data.end());
  return out;
}

void unpack_factors(const std::vector<double>& buf, std::vector<RMatrix>& fs) {
  size_t k = 0;
  for (auto& f : fs)
    for (auto& v : f.data) v = buf[k++];
}

CtfConfig factors_config(const NmfFactors& f, const CtfConfig* base) {
  CtfConfig c = base ? *base : CtfConfig{};
  c.num_sources = static_cast<int>(f.bases.size());
  c.bases_per_source.clear();
  for (const auto& b : f.bases) c.bases_per_source.push_back(b.cols);
  if (!base) c.taps_per_source.assign(f.bases.size(), 1);
  return c;
}

template <class Fn>
void op_call(const GpuOptions& gpu, Fn&& fn) {
  Ctx ctx(gpu.device);
  ctf_err e{};
  if (fn(ctx.c, &e) != CTF_OK) rethrow(e);
}

}  // namespace

double log_abs_det(const CMatrix& m, const GpuOptions& gpu) {  // estimator.cpp:41-53
  const std::vector<double> w = pack({m});
  double out = 0.0;
  op_call(gpu, [&](ctf_ctx* c, ctf_err* e) { return ctf_op_log_abs_det(c, m.rows, 1, w.data(), &out, CTF_MEM_HOST, e); });
  return out;
}

double objective_from_parts(const std::vector<CMatrix>& demixing, const std::vector<RMatrix>& lambdas,
                            const DelayedEstimates& estimates, const CtfConfig& config, const GpuOptions& gpu) {
  const int F = estimates.num_bins(), T = estimates.num_frames();
  const ctf_problem p = op_problem(config, F, T);
  const std::vector<double> w = pack(demixing), y = pack(estimates.bins), l = pack_factors(lambdas);
  double out = 0.0;
  op_call(gpu, [&](ctf_ctx* c, ctf_err* e) {
    return ctf_op_objective_from_parts(c, &p, w.data(), l.data(), y.data(), &out, CTF_MEM_HOST, e);
  });
  return out;
}

void iss_sweep(CMatrix& demixing_bin, CMatrix& estimates_bin, const std::vector<RMatrix>& lambdas,
               const CtfConfig& config, int bin, const GpuOptions& gpu) {  // estimator.cpp:505-511
  const int T = estimates_bin.cols;
  const ctf_problem p = op_problem(config, 1, T);
  std::vector<double> lam;  // row `bin` of every lambda_n as a 1 x T matrix
  for (const auto& l : lambdas)
    for (int j = 0; j < T; ++j) lam.push_back(l(bin, j));
  std::vector<CMatrix> w{demixing_bin}, y{estimates_bin};
  std::vector<double> wb = pack(w), yb = pack(y);
  Ctx ctx(gpu.device);
  ctf_err e{};
  if (ctf_op_iss_sweep(ctx.c, &p, wb.data(), yb.data(), lam.data(), CTF_MEM_HOST, &e) != CTF_OK) {
    if (e.code == CTF_ERR_DEGENERACY) throw DegeneracyError(e.msg, -1, bin, e.row);
    rethrow(e);
  }
  unpack(wb, w);
  unpack(yb, y);
  demixing_bin = w[0];
  estimates_bin = y[0];
}

DelayedEstimates demix(const std::vector<CMatrix>& demixing, const MixtureSpectrogram& x, const GpuOptions& gpu) {
  const int F = x.num_bins(), T = x.num_frames(), D = x.num_channels();
  const int R = demixing.empty() ? 0 : demixing[0].rows;
  std::vector<double> w = pack(demixing), xx = flatten(x), y((size_t)F * R * T * 2);
  op_call(gpu, [&](ctf_ctx* c, ctf_err* e) {
    return ctf_op_demix(c, F, R, D, T, w.data(), xx.data(), y.data(), CTF_MEM_HOST, e);
  });
  DelayedEstimates out;
  out.bins.assign(static_cast<size_t>(F), CMatrix(R, T));
  unpack(y, out.bins);
  return out;
}

RMatrix compute_psd(const NmfFactors& factors, int source, const GpuOptions& gpu) {  // model.cpp:210-215
  const int F = factors.bases[0].rows, T = factors.activations[0].cols;
  const CtfConfig cfg = factors_config(factors, nullptr);
  const ctf_problem p = op_problem(cfg, F, T);
  const std::vector<double> b = pack_factors(factors.bases), v = pack_factors(factors.activations);
  std::vector<double> lam((size_t)factors.bases.size() * F * T);
  op_call(gpu, [&](ctf_ctx* c, ctf_err* e) {
    return ctf_op_compute_psd(c, &p, b.data(), v.data(), factors.floor, lam.data(), CTF_MEM_HOST, e);
  });
  RMatrix out(F, T);
  std::copy(lam.begin() + (size_t)source * F * T, lam.begin() + (size_t)(source + 1) * F * T, out.data.begin());
  return out;
}

void mu_update_bases(NmfFactors& factors, const DelayedEstimates& estimates, int source, const CtfConfig& config,
                     const GpuOptions& gpu) {  // estimator.cpp:313-346
  const int F = estimates.num_bins(), T = estimates.num_frames();
  const ctf_problem p = op_problem(factors_config(factors, &config), F, T);
  std::vector<double> b = pack_factors(factors.bases);
  const std::vector<double> v = pack_factors(factors.activations), y = pack(estimates.bins);
  op_call(gpu, [&](ctf_ctx* c, ctf_err* e) {
    return ctf_op_mu_update_bases(c, &p, b.data(), v.data(), factors.floor, y.data(), source, CTF_MEM_HOST, e);
  });
  unpack_factors(b, factors.bases);
}

void mu_update_activations(NmfFactors& factors, const DelayedEstimates& estimates, int source,
                           const CtfConfig& config, const GpuOptions& gpu) {  // estimator.cpp:348-382
  const int F = estimates.num_bins(), T = estimates.num_frames();
  const ctf_problem p = op_problem(factors_config(factors, &config), F, T);
  const std::vector<double> b = pack_factors(factors.bases), y = pack(estimates.bins);
  std::vector<double> v = pack_factors(factors.activations);
  op_call(gpu, [&](ctf_ctx* c, ctf_err* e) {
    return ctf_op_mu_update_activations(c, &p, b.data(), v.data(), factors.floor, y.data(), source, CTF_MEM_HOST, e);
  });
  unpack_factors(v, factors.activations);
}

void rescale(std::vector<CMatrix>& demixing, NmfFactors& factors, DelayedEstimates& estimates,
             const CtfConfig& config, const GpuOptions& gpu) {  // estimator.cpp:384-412
  const int F = estimates.num_bins(), T = estimates.num_frames();
  if (F == 0 || T == 0) return;
  const ctf_problem p = op_problem(factors_config(factors, &config), F, T);
  std::vector<double> w = pack(demixing), b = pack_factors(factors.bases), y = pack(estimates.bins);
  op_call(gpu, [&](ctf_ctx* c, ctf_err* e) {
    return ctf_op_rescale(c, &p, w.data(), b.data(), factors.floor, y.data(), CTF_MEM_HOST, e);
  });
  unpack(w, demixing);
  unpack_factors(b, factors.bases);
  unpack(y, estimates.bins);
}

}  // namespace b200
}  // namespace ctfmnmf
