/*
 * ctf_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference CTF-MNMF-ISS estimator (arXiv 2510.02382,
 * /root/reference/proj) used as the parity checker for the CUDA path and as the
 * CPU baseline arm of bench.py. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it. The product
 * (paper_2510_02382_b200/) never links or calls it.
 *
 * Parity pin: the reference cannot be compiled here (Eigen3 REQUIRED at
 * proj/CMakeLists.txt:12 is absent, vendor/ is absent). It ships no stored
 * golden files; its pins are seeded known-answer / property tests
 * (proj/tests/test_estimator.cpp, test_run.cpp, oracles.hpp). Those are
 * re-expressed against this oracle in tests/test_oracle_kats.py. The
 * third-party arithmetic it restates is Eigen >= 3.3 (unpinned): GEMM,
 * PartialPivLU, determinant. Parity with Eigen is therefore "to rounding",
 * not bitwise.
 *
 * Layouts follow the reference's Eigen (column-major) conventions:
 *   x      : F bins, each D x T, element (c, j) at bin*D*T + c + j*D (complex
 *            interleaved re, im)                       (model.hpp:55-66)
 *   W      : F bins, each R x D, element (r, c) at bin*R*D + r + c*R
 *   Y      : F bins, each R x T, element (r, j) at bin*R*T + r + j*R
 *   B_n    : F x K_n column-major, sources concatenated    (model.hpp:70-80)
 *   V_n    : K_n x T column-major, sources concatenated
 *   lambda : N x (F x T column-major)
 */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_SOURCES 16

typedef struct orc_config {
  int32_t num_sources;                       /* N */
  int32_t num_channels;                      /* D (= sum of taps) */
  int32_t taps[ORC_MAX_SOURCES];             /* L_n */
  int32_t bases[ORC_MAX_SOURCES];            /* K_n */
  int32_t iterations;
  int32_t rule;                              /* 0 = IP, 1 = ISS */
  double psd_floor;                          /* relative floor, model.hpp:29 */
  uint64_t seed;
  int32_t threads;
} orc_config;

typedef struct orc_err {
  int32_t code;      /* 0 ok, 2 ConfigError, 4 DegeneracyError, 9 other */
  int32_t iteration; /* -1 when absent (errors.hpp:18-31) */
  int32_t bin;
  int32_t row;
  char msg[256];
} orc_err;

/* Full estimator, proj/src/estimator.cpp:513-657. Outputs may be NULL.
 * hist_* (optional) receive the state after every iteration:
 *   hist_W [iters][F*R*D complex], hist_B [iters][F*sumK], hist_V [iters][sumK*T],
 *   in the same layouts as W/B/V above. */
int orc_run(const orc_config* cfg, int F, int T, const double* x,
            double* W_out, double* B_out, double* V_out, double* obj_out,
            double* hist_W, double* hist_B, double* hist_V,
            double* trace_ms_out /* [iters][3] demix, mu, rescale */,
            orc_err* err);

/* One iteration (estimator.cpp:553-648) from an explicit state (W, B, V,
 * floor_abs). State is updated in place; obj_out receives the objective. */
int orc_step(const orc_config* cfg, int F, int T, const double* x, double floor_abs,
             double* W, double* B, double* V, double* obj_out, orc_err* err);

/* Setup pieces: mean power (model.cpp:153-161) and random_factors with
 * mt19937_64(seed) (model.cpp:189-208). */
double orc_mean_power(int F, int D, int T, const double* x);
void orc_random_factors(const orc_config* cfg, int F, int T, double* B, double* V);

/* Op-level restatements (estimator.hpp:56-117). lambda layout: N x (F x T). */
int orc_demix(int F, int R, int D, int T, const double* W, const double* x, double* Y);
int orc_iss_sweep(const orc_config* cfg, int F, int T, int bin, double* W_bin,
                  double* Y_bin, const double* lambda, orc_err* err);
int orc_weighted_covariance(int F, int D, int T, const double* x, const double* lambda_n,
                            int tap, int bin, double* Q);
int orc_iss_compute_z(int R, const double* W_bin, const double* covs, int row,
                      double* z, orc_err* err);
void orc_iss_apply(int R, int D, double* W_bin, const double* z, int row);
void orc_compute_psd(const orc_config* cfg, int F, int T, const double* B, const double* V,
                     double floor_abs, double* lambda);
void orc_mu_update_bases(const orc_config* cfg, int F, int T, double* B, const double* V,
                         double floor_abs, const double* Y, int source);
void orc_mu_update_activations(const orc_config* cfg, int F, int T, const double* B,
                               double* V, double floor_abs, const double* Y, int source);
void orc_rescale(const orc_config* cfg, int F, int T, double* W, double* B, double floor_abs,
                 double* Y);
int orc_log_abs_det(int R, const double* W_bin, double* out, orc_err* err);
int orc_objective_from_parts(const orc_config* cfg, int F, int T, const double* W,
                             const double* lambda, const double* Y, double* out, orc_err* err);
int orc_objective(const orc_config* cfg, int F, int T, const double* W, const double* B,
                  const double* V, double floor_abs, const double* x, double* out,
                  orc_err* err);
/* Projection-back, proj/src/wiener.cpp:11-49. images: N x F x (D x T col-major). */
int orc_reconstruct_images(const orc_config* cfg, int F, int T, const double* W,
                           const double* x, double* images, orc_err* err);
/* Checks instrumentation (estimator.cpp:560-577): runs with det_lemma and
 * normalization checks; returns max errors and checked update count. */
int orc_run_checked(const orc_config* cfg, int F, int T, const double* x, double* max_det_err,
                    double* max_norm_err, int64_t* checked, orc_err* err);

/* STFT front/back end (proj/src/fft.cpp, proj/src/stft.cpp). samples:
 * [channels][length] (TimeSignal.samples column-major); spec: [bins][frames]
 * [channels] complex (Spectrogram.data). */
int orc_fft(double* data /* n complex, in place */, int64_t n, int inverse, orc_err* err);
void orc_hann(int len, double* out);
int64_t orc_stft_frames(int64_t length, int hop);
int orc_forward_stft(const double* samples, int64_t length, int channels, int window_len, int hop, double* spec,
                     orc_err* err);
int orc_inverse_stft(const double* spec, int bins, int frames, int channels, int window_len, int hop,
                     int64_t original_length, double* out /* may be NULL */, int64_t* out_len, orc_err* err);

#ifdef __cplusplus
}
#endif
