// ctfmnmf_b200.hpp — C++ host API mirroring the reference library
// (/root/reference/proj/include/ctfmnmf/{model,estimator,wiener,errors}.hpp)
// over the C ABI in include/ctf_iss.h. Same names, argument meaning, output
// layout and exceptions, with its own column-major matrix types because
// Eigen is not part of this build. A reference caller swaps
//   #include "ctfmnmf/estimator.hpp"   ->   #include "ctfmnmf_b200.hpp"
// and `ctfmnmf::run` -> `ctfmnmf::b200::run`.
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace ctfmnmf {
namespace b200 {

using Complex = std::complex<double>;

// Column-major dense matrices, element (r, c) at r + c * rows (Eigen layout).
struct CMatrix {
  int rows = 0, cols = 0;
  std::vector<Complex> data;
  CMatrix() = default;
  CMatrix(int r, int c) : rows(r), cols(c), data(static_cast<size_t>(r) * c) {}
  Complex& operator()(int r, int c) { return data[static_cast<size_t>(r) + static_cast<size_t>(c) * rows]; }
  const Complex& operator()(int r, int c) const { return data[static_cast<size_t>(r) + static_cast<size_t>(c) * rows]; }
};
struct RMatrix {
  int rows = 0, cols = 0;
  std::vector<double> data;
  RMatrix() = default;
  RMatrix(int r, int c) : rows(r), cols(c), data(static_cast<size_t>(r) * c) {}
  double& operator()(int r, int c) { return data[static_cast<size_t>(r) + static_cast<size_t>(c) * rows]; }
  double operator()(int r, int c) const { return data[static_cast<size_t>(r) + static_cast<size_t>(c) * rows]; }
};

// errors.hpp:11-35
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& m) : std::runtime_error(m) {}
};
struct IoError : std::runtime_error {
  explicit IoError(const std::string& m) : std::runtime_error(m) {}
};
struct DegeneracyError : std::runtime_error {
  DegeneracyError(const std::string& m, int it = -1, int b = -1, int r = -1)
      : std::runtime_error(m), iteration(it), bin(b), row(r) {}
  int iteration, bin, row;
};

enum class UpdateRule { Ip, Iss };

// model.hpp:21-35
struct CtfConfig {
  int num_sources = 2;
  int num_channels = 4;
  std::vector<int> taps_per_source;
  std::vector<int> bases_per_source;
  int iterations = 100;
  UpdateRule update_rule = UpdateRule::Iss;
  double psd_floor = 1e-10;
  std::uint64_t seed = 0;
  int threads = 1;
  int total_taps() const;
  int row_offset(int source) const;
  void validate() const;  // throws ConfigError (model.cpp:32-50)
};

// types.hpp:12-47 — time signal (length x channels, column-major) and the
// one-sided STFT tensor indexed [bin][frame][channel].
struct TimeSignal {
  RMatrix samples;
  double sample_rate = 0.0;
  std::int64_t length() const { return samples.rows; }
  int channels() const { return samples.cols; }
};
struct Spectrogram {
  int bins = 0, frames = 0, channels = 0, window_len = 0, hop = 0;
  double sample_rate = 0.0;
  std::int64_t original_length = 0;
  std::vector<Complex> data;  // (i * frames + j) * channels + c
  Complex& at(int i, int j, int c) { return data[(static_cast<size_t>(i) * frames + j) * channels + c]; }
  Complex at(int i, int j, int c) const { return data[(static_cast<size_t>(i) * frames + j) * channels + c]; }
  void resize(int b, int f, int c) {
    bins = b;
    frames = f;
    channels = c;
    data.assign(static_cast<size_t>(b) * f * c, Complex(0, 0));
  }
};

// model.hpp:55-66 — one channels x frames matrix per bin.
struct MixtureSpectrogram {
  std::vector<CMatrix> bins;
  int num_bins() const { return static_cast<int>(bins.size()); }
  int num_channels() const { return bins.empty() ? 0 : bins[0].rows; }
  int num_frames() const { return bins.empty() ? 0 : bins[0].cols; }
  double mean_power() const;
  static MixtureSpectrogram from_spectrogram(const Spectrogram& spec);
  // meta supplies window/hop/rate fields for the round trip back to disk.
  Spectrogram to_spectrogram(const Spectrogram& meta) const;
};

struct NmfFactors {  // model.hpp:70-80
  std::vector<RMatrix> bases;        // B_n: F x K_n
  std::vector<RMatrix> activations;  // V_n: K_n x T
  double floor = 1e-12;
};

struct OptimizationTrace {  // estimator.hpp:25-40
  std::vector<double> objective, demix_ms, mu_ms, rescale_ms;
  // Populated when the corresponding CheckOptions flag is set.
  double max_det_lemma_error = 0.0;
  double max_normalization_error = 0.0;
  std::int64_t checked_updates = 0;
  std::string to_csv() const;
  double total_demix_ms() const;
  double total_mu_ms() const;
  double total_rescale_ms() const;
};

struct SeparationResult {  // estimator.hpp:50-54
  std::vector<CMatrix> demixing;
  NmfFactors factors;
  OptimizationTrace trace;
};

enum class Precision { F64, F32 };
struct GpuOptions {
  int device = 0;
  Precision precision = Precision::F64;
  // > 1: x holds num_channels / stack_taps microphones and the stacked
  // observation x~(m*L + l, t) = x_m(t - l) is built on the GPU (BASELINE (a)).
  int stack_taps = 1;
};

// estimator.hpp:45-48: exact per-update recomputations on the GPU (the
// instrumented sweep variants; verification, not production).
struct CheckOptions {
  bool det_lemma = false;      // det(W - z w_r^H) == det(W) (1 - z_r)
  bool normalization = false;  // w_r^H Q_r w_r == 1 after each row update
};

SeparationResult run(const CtfConfig& config, const MixtureSpectrogram& x, const CheckOptions& checks = {},
                     const GpuOptions& gpu = {});
SeparationResult run(const CtfConfig& config, const MixtureSpectrogram& x, const GpuOptions& gpu);

// wiener.hpp:18-20 (collapsed Wiener form, wiener.cpp:27-46).
std::vector<MixtureSpectrogram> reconstruct_images(const std::vector<CMatrix>& demixing, const NmfFactors& factors,
                                                   const MixtureSpectrogram& x, const CtfConfig& config,
                                                   const GpuOptions& gpu = {});

// stft.hpp:9-18 on the GPU (bit-identical to the reference arithmetic).
std::vector<double> hann_window(int window_len);
Spectrogram forward_stft(const TimeSignal& signal, int window_len, int hop, const GpuOptions& gpu = {});
TimeSignal inverse_stft(const Spectrogram& spec, const GpuOptions& gpu = {});

// container.hpp:22-29: .spec spectrogram and .nmf factor containers
// (complex64 / float64 bodies, the reference's IoError texts).
void write_spectrogram(const std::string& path, const Spectrogram& spec);
Spectrogram read_spectrogram(const std::string& path);
void write_factors(const std::string& path, const NmfFactors& factors);
NmfFactors read_factors(const std::string& path);

// ---- op-level API (estimator.hpp:15-23, 56-117; model.hpp:86-88) on the GPU
// (fp64, the ctf_op_* entries of include/ctf_iss.h), for drivers that run the
// loop piece by piece the way test_estimator.cpp does.
struct DelayedEstimates {  // estimator.hpp:15-23: one R x T matrix per bin
  std::vector<CMatrix> bins;
  int num_bins() const { return static_cast<int>(bins.size()); }
  int num_rows() const { return bins.empty() ? 0 : bins[0].rows; }
  int num_frames() const { return bins.empty() ? 0 : bins[0].cols; }
};
double log_abs_det(const CMatrix& m, const GpuOptions& gpu = {});
double objective_from_parts(const std::vector<CMatrix>& demixing, const std::vector<RMatrix>& lambdas,
                            const DelayedEstimates& estimates, const CtfConfig& config, const GpuOptions& gpu = {});
void iss_sweep(CMatrix& demixing_bin, CMatrix& estimates_bin, const std::vector<RMatrix>& lambdas,
               const CtfConfig& config, int bin, const GpuOptions& gpu = {});
DelayedEstimates demix(const std::vector<CMatrix>& demixing, const MixtureSpectrogram& x, const GpuOptions& gpu = {});
RMatrix compute_psd(const NmfFactors& factors, int source, const GpuOptions& gpu = {});
void mu_update_bases(NmfFactors& factors, const DelayedEstimates& estimates, int source, const CtfConfig& config,
                     const GpuOptions& gpu = {});
void mu_update_activations(NmfFactors& factors, const DelayedEstimates& estimates, int source,
                           const CtfConfig& config, const GpuOptions& gpu = {});
void rescale(std::vector<CMatrix>& demixing, NmfFactors& factors, DelayedEstimates& estimates,
             const CtfConfig& config, const GpuOptions& gpu = {});

// wiener.hpp:22-24: inverse STFT of one source image; ref_channel < 0 keeps all.
TimeSignal image_to_signal(const MixtureSpectrogram& image, const Spectrogram& meta, int ref_channel = -1,
                           const GpuOptions& gpu = {});

}  // namespace b200
}  // namespace ctfmnmf
