/*
 * ctf_iss.h — C ABI of the B200-native ISS+NMF hot path of CTF-MNMF-ISS
 * (arXiv 2510.02382). Plain pointers and sizes only; no C++ or torch types.
 *
 * The reference (/root/reference/proj) is a C++ library with no FFI; its
 * hot-path entry points and what replaces them here:
 *
 *   SeparationResult run(const CtfConfig&, const MixtureSpectrogram&,
 *                        const CheckOptions& = {})
 *       proj/include/ctfmnmf/estimator.hpp:122-123, body estimator.cpp:513-657
 *       -> ctf_run()            (one call, host buffers in and out), or
 *          ctf_setup() + ctf_iterate() + ctf_download()   (device-resident)
 *   the per-iteration loop body, estimator.cpp:548-654 ("iterate")
 *       -> ctf_iterate(ctx, n)  (n iterations + the trailing rescale/objective)
 *   std::vector<MixtureSpectrogram> reconstruct_images(W, factors, x, config)
 *       proj/include/ctfmnmf/wiener.hpp:18-20, body wiener.cpp:11-49
 *       -> ctf_project_back()
 *   Spectrogram forward_stft(const TimeSignal&, int window_len, int hop)
 *   TimeSignal inverse_stft(const Spectrogram&)
 *       proj/include/ctfmnmf/stft.hpp:13-18, body stft.cpp:46-139
 *       -> ctf_stft() / ctf_istft(); the front end feeding the estimator
 *          directly: ctf_setup_signal(); the back end of cmd_separate
 *          (reconstruct_images + image_to_signal, wiener.cpp:51-64):
 *          ctf_images_to_signal()
 *   write_/read_spectrogram, write_/read_factors (container.hpp:22-29)
 *       -> ctf_write_/ctf_read_spectrogram, ctf_write_/ctf_read_factors,
 *          ctf_setup_spectrogram_files (a `.spec` straight into the estimator)
 *   CtfConfig (model.hpp:21-35) + the stacked observation of BASELINE (a)
 *       -> ctf_problem
 *   ConfigError / IoError / DegeneracyError{iteration,bin,row}
 *       (errors.hpp:11-35) and CLI exit codes 2/3/4 (ctfmnmf_main.cpp:38-40)
 *       -> ctf_status codes + ctf_err
 *
 * The host C++ mirror of the reference API (same names, argument meaning and
 * exceptions) is paper_2510_02382_b200/csrc/ctfmnmf_b200.hpp; the Python mirror
 * is paper_2510_02382_b200/api.py. INTEGRATION.md shows the binding a
 * reference maintainer would add.
 *
 * Layouts (complex numbers are interleaved re,im pairs):
 *   x (input)  : [mixture][bin][frame][channel], i.e. per mixture the
 *                reference Spectrogram layout (i*frames + j)*channels + c
 *                (types.hpp:32) == one column-major channels x frames Eigen
 *                matrix per bin (model.hpp:55-66). channel count = num_mics.
 *   W (output) : [mixture][bin] column-major R x D (Eigen MatrixXcd layout).
 *   B (output) : [mixture][source] column-major F x K_n (Eigen MatrixXd).
 *   V (output) : [mixture][source] column-major K_n x T.
 *   objective  : [mixture][iteration].
 *   images     : [source][mixture][bin] column-major Dout x T, where Dout = D
 *                (full stacked observation, as reconstruct_images returns) or
 *                num_mics when CTF_IMAGES_CURRENT_FRAME is requested.
 *
 * Stacked observation (BASELINE (a)): with stack_taps = L > 1
 * the observation is x~(c = m*L + l, t) = x_m(t - l) (zero for t < l), built
 * virtually inside the kernels (never materialised in HBM); D = num_mics*L.
 * With stack_taps = 1 the input already is the D-channel observation.
 *
 * Threading: a context is single-owner; calls are
 * stream-ordered on the context's stream. Multi-GPU: one process per GPU,
 * each with one context; ctf_comm_init() joins the contexts into one
 * frequency-sharded job (contiguous bin ranges, one NCCL all-reduce of the
 * packed MU-V numerator/denominator + row powers + objective per iteration).
 */
#ifndef CTF_ISS_H_
#define CTF_ISS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CTF_ABI_VERSION 1
#define CTF_MAX_SOURCES 16
#define CTF_MAX_ROWS 64

/* Status codes mirror the reference CLI exit codes (ctfmnmf_main.cpp:38-40). */
typedef enum ctf_status {
  CTF_OK = 0,
  CTF_ERR_CONFIG = 2,     /* ConfigError */
  CTF_ERR_IO = 3,         /* IoError */
  CTF_ERR_DEGENERACY = 4, /* DegeneracyError */
  CTF_ERR_CUDA = 5,       /* device / runtime failure (no reference analogue) */
  CTF_ERR_UNSUPPORTED = 6 /* shape outside the compiled kernel set */
} ctf_status;

typedef enum ctf_precision { CTF_F64 = 0, CTF_F32 = 1 } ctf_precision;
typedef enum ctf_rule { CTF_RULE_IP = 0, CTF_RULE_ISS = 1 } ctf_rule;
/* CheckOptions flags (estimator.hpp:45-48): exact per-update recomputations. */
typedef enum ctf_check {
  CTF_CHECK_DET_LEMMA = 1,     /* det(W - z w_r^H) == det(W) (1 - z_r) */
  CTF_CHECK_NORMALIZATION = 2  /* weighted power of the updated row == 1 */
} ctf_check;

/* Degeneracy kinds carried in ctf_err.kind. */
typedef enum ctf_err_kind {
  CTF_KIND_NONE = 0,
  CTF_KIND_STEERING_DENOM = 1,  /* estimator.cpp:451-454 */
  CTF_KIND_NONFINITE_W = 2,     /* estimator.cpp:494-496 */
  CTF_KIND_NONFINITE_Y = 3,     /* estimator.cpp:497-499 */
  CTF_KIND_ZERO_PIVOT = 4,      /* estimator.cpp:46-47 */
  CTF_KIND_TINY_DET = 5,        /* estimator.cpp:50-51 */
  CTF_KIND_NONFINITE_OBJ = 6,   /* estimator.cpp:647-648 */
  CTF_KIND_NONFINITE_X = 7,     /* estimator.cpp:521-522 */
  CTF_KIND_ZERO_X = 8,          /* estimator.cpp:523-524 (ConfigError) */
  CTF_KIND_SINGULAR_IMAGE = 9,  /* wiener.cpp:38-40 */
  CTF_KIND_PROJECTION = 10      /* estimator.cpp:105-115 (IP rule) */
} ctf_err_kind;

typedef struct ctf_err {
  int32_t code;      /* ctf_status */
  int32_t kind;      /* ctf_err_kind */
  int32_t iteration; /* 1-based, -1 when absent (DegeneracyError::iteration) */
  int32_t mixture;   /* batch index, -1 when absent */
  int32_t bin;       /* global bin, -1 when absent (DegeneracyError::bin) */
  int32_t row;       /* demixing row, -1 when absent (DegeneracyError::row) */
  char msg[256];     /* reference-compatible message text */
} ctf_err;

/* CtfConfig (model.hpp:21-35) + batch/shape + the stacked observation. */
typedef struct ctf_problem {
  int32_t num_mixtures;                        /* B, independent mixtures */
  int32_t num_bins;                            /* F */
  int32_t num_frames;                          /* T */
  int32_t num_mics;                            /* channels of x as supplied */
  int32_t stack_taps;                          /* L of the virtual stack; 1 = x already stacked */
  int32_t num_sources;                         /* N */
  int32_t taps_per_source[CTF_MAX_SOURCES];    /* L_n, sum = D = num_mics*stack_taps */
  int32_t bases_per_source[CTF_MAX_SOURCES];   /* K_n */
  int32_t iterations;
  int32_t update_rule;                         /* ctf_rule; IP runs on the covariance-domain kernel */
  int32_t precision;                           /* ctf_precision of the compute path */
  int32_t x_precision;                         /* ctf_precision of the host x buffer */
  double psd_floor;                            /* relative floor, model.hpp:29 */
  uint64_t seed;                               /* mixture b is seeded with seed + b */
  int32_t threads;                             /* accepted and ignored (GPU path) */
  int32_t checks;                              /* CheckOptions (estimator.hpp:45-48): CTF_CHECK_* bits */
  int32_t reserved[6];
} ctf_problem;

/* Per-phase device times of the last ctf_iterate()/ctf_run(), CUDA events. */
typedef struct ctf_timing {
  double sweep_ms;      /* fused demix+ISS sweep+demix+MU-B kernel */
  double mu_ms;         /* MU-V partial/reduce/apply (+ all-reduce) */
  double finalize_ms;   /* trailing rescale + objective pass */
  int64_t sweep_launches;
  int64_t launches;     /* all kernels launched by the library */
} ctf_timing;

typedef struct ctf_ctx ctf_ctx;

int ctf_abi_version(void);

/* Context on one CUDA device (one process per GPU). */
int ctf_open(int device, ctf_ctx** out, ctf_err* err);
void ctf_close(ctf_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) so callers can time with events. */
void* ctf_stream(ctf_ctx* ctx);

/* Multi-GPU: rank 0 calls ctf_comm_unique_id, broadcasts the 128 bytes,
 * every rank calls ctf_comm_init before ctf_setup. Bins are split into
 * contiguous ranges by rank. NCCL is loaded lazily (dlopen). */
int ctf_comm_unique_id(uint8_t id[128], ctf_err* err);
int ctf_comm_init(ctf_ctx* ctx, int world_size, int rank, const uint8_t id[128], ctf_err* err);
/* In-process exchange group (testing the sharded path on one GPU): contexts
 * of one process, each driven by its own host thread, all-reduce through host
 * memory in fixed rank order instead of NCCL. */
typedef struct ctf_group ctf_group;
ctf_group* ctf_group_create(int world_size);
void ctf_group_destroy(ctf_group* group);
int ctf_comm_init_group(ctf_ctx* ctx, ctf_group* group, int rank, ctf_err* err);
/* Local bin range [lo, hi) of this rank for a problem with num_bins bins. */
void ctf_shard_range(int num_bins, int world_size, int rank, int* lo, int* hi);

/* Validates the problem (CtfConfig::validate, model.cpp:32-50), allocates
 * device state, uploads x (this rank's bins), computes mean power and the
 * absolute PSD floor (estimator.cpp:520-529), draws the initial NMF factors
 * with mt19937_64(seed+b) exactly as random_factors (model.cpp:189-208),
 * and sets W = I (model.cpp:221-227). x is the full [B][F][T][num_mics]
 * host array (pinned or pageable). */
int ctf_setup(ctf_ctx* ctx, const ctf_problem* prob, const void* x_host, ctf_err* err);
/* Replaces the state (for one-step parity): W [B][F] R x D col-major complex
 * (full F, this rank's bins are read), B [B][N] F x K_n, V [B][N] K_n x T,
 * host doubles. Any argument may be NULL to keep the current value. */
int ctf_set_state(ctf_ctx* ctx, const double* W, const double* B, const double* V, ctf_err* err);
/* Runs n iterations of estimator.cpp:548-654 followed by the trailing
 * rescale+objective, so the state is exactly the reference's after n more
 * iterations. Degeneracies are reported like the reference (first failing
 * iteration, phase, lowest bin). */
int ctf_iterate(ctf_ctx* ctx, int n, ctf_err* err);
/* Device-resident benchmark form: n loop bodies without the trailing
 * finalize (call ctf_finalize before ctf_download). No host sync. */
int ctf_iterate_async(ctf_ctx* ctx, int n, ctf_err* err);
int ctf_finalize(ctf_ctx* ctx, ctf_err* err);
/* Copies the state to host doubles (layouts above). W/B cover this rank's
 * bins (other bins untouched); V and the objective trace are replicated.
 * objective receives [B][iterations_done]. Any pointer may be NULL. */
int ctf_download(ctf_ctx* ctx, double* W, double* B, double* V, double* objective, ctf_err* err);
int ctf_iterations_done(ctf_ctx* ctx);
/* JSON description of the kernel configuration chosen for the problem. */
int ctf_describe(ctf_ctx* ctx, char* buf, int len);
/* Absolute PSD floor per mixture (factors.floor, estimator.cpp:529). */
int ctf_psd_floor(ctf_ctx* ctx, double* floor_out /* [B] */);
/* Per-iteration phase times (OptimizationTrace demix_ms / mu_ms /
 * rescale_ms, estimator.hpp:25-40, timed as at estimator.cpp:623-653) from
 * CUDA events: demix_ms = the fused sweep kernel (ISS steps, demix, MU-B),
 * mu_ms = the MU-V partials, rescale_ms = the reduce/apply kernel that forms
 * mu_r from the row powers, applies V and the objective (the division of W
 * and B by mu is fused into the next sweep's prologue). With mixture chunks
 * (multi-rank pipelining) the apply is inside mu_ms and rescale_ms is 0.
 * Arrays of ctf_iterations_done() entries. */
int ctf_trace_ms(ctf_ctx* ctx, double* demix_ms, double* mu_ms, double* rescale_ms);

/* OptimizationTrace check fields (estimator.hpp:31-34) per mixture, for a
 * problem set up with checks != 0: max det-lemma error, max normalization
 * error (maxima over all bins, steps and iterations so far, all ranks) and
 * checked_updates = iterations * F * R. Any pointer may be NULL. */
int ctf_check_stats(ctf_ctx* ctx, double* max_det_lemma_error /* [B] */,
                    double* max_normalization_error /* [B] */, int64_t* checked_updates /* [B] */);
int ctf_get_timing(ctf_ctx* ctx, ctf_timing* out);
int ctf_reset_timing(ctf_ctx* ctx);

/* One call end to end (== reference run() over a batch): setup, iterate
 * prob->iterations times, download. */
int ctf_run(ctf_ctx* ctx, const ctf_problem* prob, const void* x_host, double* W_out,
            double* B_out, double* V_out, double* objective_out, ctf_err* err);

/* Projection-back (wiener.cpp:11-49, collapsed form c_n = H_n y_n with
 * H = W^-1) from the current state. images as documented above, host
 * doubles, this rank's bins. */
#define CTF_IMAGES_FULL 0
#define CTF_IMAGES_CURRENT_FRAME 1
int ctf_project_back(ctf_ctx* ctx, int mode, double* images, ctf_err* err);

/* ---- STFT front / back end (stft.cpp:46-139, fft.cpp:9-41), fp64.
 * Bit-identical to the reference arithmetic (radix-2 DIT with the
 * reference's twiddle recurrence, no FMA contraction). Layouts:
 *   samples : [channel][length] doubles (TimeSignal.samples column-major)
 *   spec    : [bin][frame][channel] complex (Spectrogram.data, types.hpp:32)
 * window_len: power of two in [2, 8192]; hop divides window_len.
 * Errors are the reference's ConfigError texts ("forward_stft: ...",
 * "inverse_stft: ..."). */
int64_t ctf_stft_frames(int64_t length, int hop); /* 1 + ceil(length / hop) */
int ctf_stft(ctf_ctx* ctx, const double* samples, int64_t length, int channels, int window_len, int hop,
             double* spec /* [window_len/2+1][frames][channels] complex */, ctf_err* err);
/* original_length <= 0: padded length - window_len (stft.cpp:107-108).
 * samples may be NULL to only validate and query *out_len. */
int ctf_istft(ctf_ctx* ctx, const double* spec, int bins, int frames, int channels, int window_len, int hop,
              int64_t original_length, double* samples /* [channels][out_len] */, int64_t* out_len,
              ctf_err* err);
/* Device-pointer forms, stream-ordered on ctf_stream(ctx) (no synchronize):
 * num_signals independent signals, samples [signal][channel][length],
 * spec [signal][bin][frame][channel] (complex128, or complex64 output when
 * out_precision == CTF_F32; the inverse takes complex128). */
int ctf_stft_device(ctf_ctx* ctx, const double* samples, int num_signals, int64_t length, int channels,
                    int window_len, int hop, void* spec, int out_precision, ctf_err* err);
int ctf_istft_device(ctf_ctx* ctx, const double* spec, int num_signals, int bins, int frames, int channels,
                     int window_len, int hop, int64_t original_length, double* samples, ctf_err* err);
/* ctf_setup() from time-domain signals: the STFT runs on the GPU and writes
 * this rank's bins straight into the estimator's input (no host round trip).
 * samples: [mixture][mic][length] doubles; prob->num_bins / num_frames may be
 * 0 (filled in) or must match window_len/2+1 and ctf_stft_frames(). */
int ctf_setup_signal(ctf_ctx* ctx, const ctf_problem* prob, const double* samples, int64_t length,
                     int window_len, int hop, ctf_err* err);
/* Back end of cmd_separate: projection-back of the microphone images
 * (stack_taps > 1: current-frame channels; else the supplied channels) and
 * their inverse STFT, on the GPU. out: [source][mixture][channel][out_len]
 * (ref_channel < 0) or [source][mixture][out_len] (the reference channel,
 * wiener.cpp:51-64). Needs every bin on this context (world 1). out may be
 * NULL to query *out_len. */
int ctf_images_to_signal(ctf_ctx* ctx, int ref_channel, int window_len, int hop, int64_t original_length,
                         double* out, int64_t* out_len, ctf_err* err);

/* ---- Binary containers (container.hpp:1-10, container.cpp; host only, no
 * GPU). IoError texts of the reference ("cannot open file: ...", "...: bad or
 * mismatched container magic", "...: truncated spectrogram container").
 * Spectrogram body: complex64 [bin][frame][channel]; read/write it as complex64
 * (precision CTF_F32, byte copy) or complex128 (CTF_F64, widened/narrowed
 * exactly like get_complex/put_complex). */
typedef struct ctf_spec_header {
  uint32_t bins, frames, channels, window_len, hop, sample_rate;
  uint64_t original_length;
} ctf_spec_header;
int ctf_read_spectrogram(const char* path, ctf_spec_header* hdr, void* data /* NULL: header only */,
                         int out_precision, ctf_err* err);
int ctf_write_spectrogram(const char* path, const ctf_spec_header* hdr, const void* data, int in_precision,
                          ctf_err* err);
/* ctf_setup() from one `.spec` file per mixture (the complex64 body is
 * uploaded as stored, x_precision = f32); prob->num_bins/num_frames/num_mics
 * may be 0 (taken from the files) or must match; hdr_out (optional) receives
 * the first file's header (window/hop/rate for the inverse STFT). */
int ctf_setup_spectrogram_files(ctf_ctx* ctx, const ctf_problem* prob, const char* const* paths, int num_paths,
                                ctf_spec_header* hdr_out, ctf_err* err);
/* NmfFactors container: B/V in the ctf_download layouts of ONE mixture
 * (per source column-major F x K_n / K_n x T); the file stores them row-major. */
int ctf_write_factors(const char* path, int num_sources, int bins, int frames, const int32_t* bases,
                      double floor_abs, const double* B, const double* V, ctf_err* err);
int ctf_read_factors(const char* path, int* num_sources, int* bins, int* frames, int32_t* bases /* [16] */,
                     double* floor_abs, double* B /* NULL: header only */, double* V, ctf_err* err);

/* ---- Op-level entries: the reference's individual estimator operations
 * (proj/include/ctfmnmf/estimator.hpp:56-117, model.hpp:86-88) on the GPU in
 * fp64, for drivers that run the loop piece by piece the way the reference's
 * own unit tests do (test_estimator.cpp). Shapes come from a ctf_problem
 * (num_bins F, num_frames T, num_sources, taps_per_source, bases_per_source;
 * R = D = sum of taps: the already-stacked observation). Layouts:
 *   W [F] column-major R x D complex;  Y [F] column-major R x T complex
 *   x [F][T][D] complex;  B / V as ctf_download (one mixture);
 *   lambda [N] column-major F x T doubles.
 * mem = CTF_MEM_HOST: host pointers (copied in/out, the call synchronises);
 * CTF_MEM_DEVICE: device pointers on the context's device, stream-ordered on
 * ctf_stream(ctx). Errors use the reference's texts and codes. */
#define CTF_MEM_HOST 0
#define CTF_MEM_DEVICE 1
/* demix, estimator.cpp:304-311: Y_i = W_i x_i */
int ctf_op_demix(ctf_ctx* ctx, int F, int R, int D, int T, const double* W, const double* x, double* Y, int mem,
                 ctf_err* err);
/* compute_psd for every source, model.cpp:210-215 */
int ctf_op_compute_psd(ctf_ctx* ctx, const ctf_problem* prob, const double* B, const double* V, double floor_abs,
                       double* lambda, int mem, ctf_err* err);
/* iss_sweep, estimator.cpp:505-511 (steering :434-462, step :476-484) on
 * every bin; W and Y updated in place. Degeneracy: the lowest failing bin. */
int ctf_op_iss_sweep(ctf_ctx* ctx, const ctf_problem* prob, double* W, double* Y, const double* lambda, int mem,
                     ctf_err* err);
/* mu_update_bases / mu_update_activations for one source,
 * estimator.cpp:313-346 / :348-382 (all taps contribute) */
int ctf_op_mu_update_bases(ctf_ctx* ctx, const ctf_problem* prob, double* B, const double* V, double floor_abs,
                           const double* Y, int source, int mem, ctf_err* err);
int ctf_op_mu_update_activations(ctf_ctx* ctx, const ctf_problem* prob, const double* B, double* V, double floor_abs,
                                 const double* Y, int source, int mem, ctf_err* err);
/* rescale, estimator.cpp:384-412: W, B and Y in place */
int ctf_op_rescale(ctf_ctx* ctx, const ctf_problem* prob, double* W, double* B, double floor_abs, double* Y, int mem,
                   ctf_err* err);
/* log_abs_det of num_bins R x R matrices, estimator.cpp:41-53 */
int ctf_op_log_abs_det(ctf_ctx* ctx, int R, int num_bins, const double* W, double* out, int mem, ctf_err* err);
/* objective_from_parts, estimator.cpp:55-77 (out: one double) */
int ctf_op_objective_from_parts(ctf_ctx* ctx, const ctf_problem* prob, const double* W, const double* lambda,
                                const double* Y, double* out, int mem, ctf_err* err);

/* Synthetic generator of BASELINE.json configs (host code, no GPU):
 * mixture b uses mt19937_64(base_seed + b); see DESIGN.md for draw order.
 * x_out: [B][F][T][M] complex (double if out_precision == CTF_F64, float
 * otherwise). threads <= 0 means hardware concurrency. */
int ctf_synth_mixtures(int num_mixtures, int F, int T, int M, int N, int L, int K, double tap_decay,
                       uint64_t base_seed, int out_precision, void* x_out, int threads, ctf_err* err);

#ifdef __cplusplus
}
#endif
#endif /* CTF_ISS_H_ */
