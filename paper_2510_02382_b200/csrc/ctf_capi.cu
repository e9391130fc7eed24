// ctf_capi.cu — C ABI (include/ctf_iss.h) over the sm_100a kernels.
//
// Owns the device state of one frequency shard of a batch of mixtures and
// drives one iteration of proj/src/estimator.cpp:548-654 as
//   sweep_kernel          (per bin: rescale, lambda, demix, objective of the
//                          previous iteration, ISS sweep, demix, E, row
//                          powers, MU-B)
//   muv_partial_kernel    (MU-V numerator/denominator over bin chunks)
//   [ncclAllReduce]       (world > 1: packed V sums + row powers + objective)
//   reduce_apply_kernel   (V update, mu, objective trace)
// with no host synchronisation inside the loop.
#include "ctf_kernels.cuh"
#include "ctf_stft.cuh"
#include "../../include/ctf_iss.h"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <functional>
#include <condition_variable>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

using ctf::kMaxRows;
using ctf::kMaxSources;

// ---------------------------------------------------------------------------
// Kernel variant registry (instantiated in ctf_sweep_*.cu).
#include "ctf_sweep_variants.h"
namespace ctf {
const std::vector<SweepVariant>& sweep_variants_f32();
const std::vector<SweepVariant>& sweep_variants_f64();
}  // namespace ctf

namespace {

// Minimal NCCL surface, resolved with dlopen so the library has no link-time
// NCCL dependency (torch ships its own libnccl.so.2; whichever is loaded
// first in the process is reused).
typedef struct {
  char internal[128];
} NcclUid;
typedef void* NcclComm;
struct NcclApi {
  void* h = nullptr;
  int (*GetUniqueId)(NcclUid*) = nullptr;
  int (*CommInitRank)(NcclComm*, int, NcclUid, int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  int (*CommDestroy)(NcclComm) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool load() {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
    AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
    CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
    GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
    GroupStart = (decltype(GroupStart))dlsym(h, "ncclGroupStart");
    GroupEnd = (decltype(GroupEnd))dlsym(h, "ncclGroupEnd");
    return GetUniqueId && CommInitRank && AllReduce && CommDestroy;
  }
};
NcclApi g_nccl;
enum { kNcclFloat = 7, kNcclDouble = 8, kNcclUint64 = 5, kNcclSum = 0, kNcclMax = 2, kNcclMin = 3 };

struct CtfError : std::runtime_error {
  int code, kind, iteration, mixture, bin, row;
  CtfError(int c, const std::string& m, int k = 0, int it = -1, int mix = -1, int b = -1, int r = -1)
      : std::runtime_error(m), code(c), kind(k), iteration(it), mixture(mix), bin(b), row(r) {}
};

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CtfError(CTF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) cuda_check((x), #x)

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {  // keeps the allocation when the size is unchanged
    if (p && count == n) return;
    free();
    n = count;
    if (count) CK(cudaMalloc(&p, count * sizeof(T)));
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { free(); }
};

size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

}  // namespace

// In-process exchange group: several contexts of one process (one per host
// thread) reduce through host memory in fixed rank order. Used to exercise
// the frequency-sharded path on a single GPU; production multi-GPU uses NCCL.
struct ctf_group {
  int world = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  std::vector<std::vector<unsigned char>> slots;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

struct ctf_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  // multi-GPU
  int world = 1, rank = 0;
  // the exchange path (reduce -> all-reduce -> apply) runs when there are
  // peers, or for a single-rank NCCL communicator (CTF_NCCL_SINGLE_RANK=1:
  // exercises the NCCL call itself on one GPU)
  bool collective() const { return world > 1 || comm != nullptr; }
  NcclComm comm = nullptr;
  ctf_group* group = nullptr;  // in-process exchange instead of NCCL
  // problem
  bool ready = false;
  ctf_problem prob{};
  int F = 0, T = 0, Mx = 0, Ls = 1, D = 0, R = 0, N = 0, SK = 0, B = 0;
  int lo = 0, hi = 0, FL = 0;
  int real_size = 8;
  int taps[kMaxSources]{}, bases[kMaxSources]{}, row0[kMaxSources]{}, koff[kMaxSources + 1]{};
  int max_iters = 0;
  int done = 0;       // iterations completed
  bool pending = false;  // the last iteration's rescale/objective are not yet applied
  // kernel choice
  ctf::SweepVariant sv{};
  int NT = 0, TP = 0;
  size_t sweep_smem = 0;
  ctf::SweepParams sp{};
  int kmax = 0, chunk_bins = 0, nchunk = 0;
  int stream_grid = 0;
  int cluster_size = 0;
  // conditioning fallback of the covariance-domain kernel: the frame-domain
  // variant that re-runs the bins it hands over (SweepParams::fb_mode)
  bool has_fb = false;
  ctf::SweepVariant fbv{};
  ctf::SweepParams sp_fb{};
  size_t fb_smem = 0;
  int fb_nt = 0, fb_grid = 0;
  double fb_theta = 0.0;
  DevBuf<int> fb_list, fb_count;
  // pipelined collective loop (world > 1): the mixtures in nmc chunks; the
  // all-reduce of chunk k runs on comm_stream while chunk k+1 sweeps, and
  // its apply is deferred to just before chunk k's next sweep
  int nmc = 1;
  std::vector<int> mix_split;  // chunk k = mixtures [mix_split[k], mix_split[k+1])
  cudaStream_t comm_stream = nullptr;
  cudaStream_t stream2 = nullptr;  // odd chunks: their sweeps overlap the even chunks' tails
  cudaEvent_t ev_join = nullptr;
  cudaStream_t chunk_stream(int k) const { return (k & 1) && stream2 ? stream2 : stream; }
  std::vector<cudaEvent_t> ev_red, ev_ar;
  // ctf_run's upload pipeline (world 1): x in mixture chunks on a copy
  // stream, each chunk's first iterations on its own stream
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaStream_t> ustreams;
  std::vector<cudaEvent_t> ev_up, ev_udone;
  struct Deferred {
    bool on = false;
    int obj_slot = -1, do_v = 0;
  };
  std::vector<Deferred> deferred;
  // device buffers
  DevBuf<unsigned char> x, W, Bf, V, E, part, packed, scratch, cpivot, cwpivot;
  DevBuf<double> cpart;
  DevBuf<int> cbad;
  DevBuf<double> stage;  // double staging for host transfers (reused)
  DevBuf<double> rowpow, objbin, packed_d, mu, floor_abs, objective, mp_part, logdet;
  DevBuf<unsigned long long> err;
  DevBuf<unsigned long long> chk;  // CheckOptions maxima [B][2] (double bit patterns)
  DevBuf<double> logmu;             // [B] sum_r log mu_r of the pending rescale
  DevBuf<double> mpsum;             // [B] sum of |x~|^2 (device-side floors of the overlapped ctf_run)
  DevBuf<int4> gtab;                // gram_kernel task table
  // covariance-domain kernel: 1 / lambda [B][FL][N][T] and the objective's
  // log term [B][FL] computed ahead of each loop body by lambda_kernel
  bool lam_pre = false;
  DevBuf<unsigned char> invl;
  DevBuf<double> logsum;
  std::vector<int4> gtab_host;
  // STFT tables (window length stft_N) and scratch
  int stft_N = 0;
  DevBuf<double2> stft_twf, stft_twi;
  DevBuf<double> stft_win, stft_in, stft_out, stft_frames;
  DevBuf<double2> stft_spec;
  // timing
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_sweep, ev_mu, ev_fin;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_lam;  // dev (CTF_DEV_TIME_LAMBDA): around lambda_kernel
  std::vector<cudaEvent_t> ev_rs;  // per iteration: between MU-V and the reduce/apply kernel (null when chunked)
  std::vector<cudaEvent_t> ev_pool;
  ctf_timing timing{};
  std::vector<double> it_sweep_ms, it_mu_ms, it_rs_ms;  // per completed iteration
  std::vector<double> floors;
};

namespace {

void set_err(ctf_err* e, int code, const std::string& msg, int kind = 0, int it = -1, int mix = -1, int bin = -1,
             int row = -1) {
  if (!e) return;
  e->code = code;
  e->kind = kind;
  e->iteration = it;
  e->mixture = mix;
  e->bin = bin;
  e->row = row;
  std::snprintf(e->msg, sizeof(e->msg), "%s", msg.c_str());
}

template <class Fn>
int guarded(ctf_err* err, Fn&& fn) {
  set_err(err, CTF_OK, "");
  try {
    fn();
    return CTF_OK;
  } catch (const CtfError& e) {
    set_err(err, e.code, e.what(), e.kind, e.iteration, e.mixture, e.bin, e.row);
    return e.code;
  } catch (const std::exception& e) {
    set_err(err, CTF_ERR_CUDA, e.what());
    return CTF_ERR_CUDA;
  }
}

cudaEvent_t take_event(ctf_ctx* c) {
  cudaEvent_t e;
  if (!c->ev_pool.empty()) {
    e = c->ev_pool.back();
    c->ev_pool.pop_back();
  } else {
    CK(cudaEventCreate(&e));
  }
  return e;
}

// CtfConfig::validate (model.cpp:32-50) plus the GPU path's own limits.
void validate(const ctf_problem& p) {
  if (p.checks < 0 || p.checks > (CTF_CHECK_DET_LEMMA | CTF_CHECK_NORMALIZATION))
    throw CtfError(CTF_ERR_CONFIG, "unknown check flags");
  if (p.num_sources < 1) throw CtfError(CTF_ERR_CONFIG, "n_sources must be >= 1");
  if (p.num_sources > CTF_MAX_SOURCES) throw CtfError(CTF_ERR_CONFIG, "n_sources exceeds CTF_MAX_SOURCES");
  if (p.num_mics < 1 || p.stack_taps < 1) throw CtfError(CTF_ERR_CONFIG, "n_channels must be >= 1");
  int sum = 0;
  for (int n = 0; n < p.num_sources; ++n) {
    if (p.taps_per_source[n] < 1) throw CtfError(CTF_ERR_CONFIG, "every tap count must be >= 1");
    if (p.bases_per_source[n] < 1) throw CtfError(CTF_ERR_CONFIG, "every basis count must be >= 1");
    sum += p.taps_per_source[n];
  }
  const int D = p.num_mics * p.stack_taps;
  if (sum != D)
    throw CtfError(CTF_ERR_CONFIG, "sum of taps (" + std::to_string(sum) + ") must equal n_channels (" +
                                       std::to_string(D) + "): the demixing system must be square");
  if (p.iterations < 0) throw CtfError(CTF_ERR_CONFIG, "iters must be >= 0");
  if (!(p.psd_floor > 0.0)) throw CtfError(CTF_ERR_CONFIG, "floor must be > 0");
  if (p.threads < 1) throw CtfError(CTF_ERR_CONFIG, "threads must be >= 1");
  if (p.update_rule != CTF_RULE_ISS && p.update_rule != CTF_RULE_IP)
    throw CtfError(CTF_ERR_CONFIG, "unknown update rule");
  if (p.update_rule == CTF_RULE_IP && p.checks)
    throw CtfError(CTF_ERR_UNSUPPORTED, "CheckOptions are implemented for the ISS rule");
  if (p.num_mixtures < 1 || p.num_bins < 1 || p.num_frames < 1)
    throw CtfError(CTF_ERR_CONFIG, "empty problem (mixtures, bins and frames must be >= 1)");
  if (p.precision != CTF_F32 && p.precision != CTF_F64) throw CtfError(CTF_ERR_CONFIG, "unknown precision");
  if (p.x_precision != CTF_F32 && p.x_precision != CTF_F64) throw CtfError(CTF_ERR_CONFIG, "unknown x precision");
  if (D > ctf::kMaxRows) throw CtfError(CTF_ERR_UNSUPPORTED, "D > 64 rows is not in the compiled kernel set");
  if (p.num_bins >= (1 << 20)) throw CtfError(CTF_ERR_UNSUPPORTED, "too many bins");
}

// Task table of gram_kernel: the (m, m', d) groups of the Hermitian half
// (m < m' all lags, m == m' lags d >= 0), each with 2L-1-|d| weight lags;
// threads are shared out in proportion to that count and every group's frame
// range [U0, U1) is split into contiguous chunks of whole register blocks.
// Dev knob for the Gram task layout (measurement only): CTF_GRAM_TUNE =
// "xpk|rot_0,rot_1,...|cadd_0,...|order_0,..." (x-row padding, per-group chunk
// rotation, chunk-length increments, group permutation after the sort).
struct GramTune {
  int xpk = 0;
  std::vector<int> rot, cadd, order;
};
static GramTune gram_tune() {
  GramTune t;
  const char* e = std::getenv("CTF_GRAM_TUNE");
  if (!e) return t;
  std::string s(e);
  std::vector<std::string> parts;
  size_t a = 0;
  for (;;) {
    const size_t b = s.find('|', a);
    parts.push_back(s.substr(a, b == std::string::npos ? std::string::npos : b - a));
    if (b == std::string::npos) break;
    a = b + 1;
  }
  auto ints = [](const std::string& q) {
    std::vector<int> v;
    size_t i = 0;
    while (i < q.size()) {
      const size_t j = q.find(',', i);
      v.push_back(std::atoi(q.substr(i, j == std::string::npos ? std::string::npos : j - i).c_str()));
      if (j == std::string::npos) break;
      i = j + 1;
    }
    return v;
  };
  if (parts.size() > 0) t.xpk = std::atoi(parts[0].c_str());
  if (parts.size() > 1) t.rot = ints(parts[1]);
  if (parts.size() > 2) t.cadd = ints(parts[2]);
  if (parts.size() > 3) t.order = ints(parts[3]);
  return t;
}

void build_gram_table(ctf_ctx* c, int NT, int M, int L) {
  struct Grp { int m, m2, d, alo, cnt; };
  const GramTune tune = gram_tune();
  std::vector<Grp> gs;
  for (int m = 0; m < M; ++m)
    for (int m2 = m; m2 < M; ++m2)
      for (int d = (m == m2 ? 0 : -(L - 1)); d <= L - 1; ++d) {
        const int alo = std::max(-(L - 1), -(L - 1) - d), ahi = std::min(L - 1, L - 1 - d);
        gs.push_back({m, m2, d, alo, ahi - alo + 1});
      }
  // sorted by lag count (descending): a warp spans at most two adjacent counts
  std::stable_sort(gs.begin(), gs.end(), [](const Grp& a, const Grp& b) { return a.cnt > b.cnt; });
  const int ng = (int)gs.size();
  if ((int)tune.order.size() == ng) {
    std::vector<Grp> g2;
    for (int i : tune.order) g2.push_back(gs[(size_t)i]);
    gs = g2;
  }
  if (ng > NT) throw CtfError(CTF_ERR_UNSUPPORTED, "gram kernel: more lag groups than threads");
  long total = 0;
  for (const auto& g : gs) total += g.cnt;
  std::vector<int> th((size_t)ng, 1);
  int used = ng;
  // largest-remainder share of the remaining threads, proportional to cnt
  std::vector<double> want((size_t)ng);
  for (int g = 0; g < ng; ++g) want[(size_t)g] = (double)NT * gs[(size_t)g].cnt / (double)total;
  while (used < NT) {
    int best = 0;
    double bd = -1e30;
    for (int g = 0; g < ng; ++g) {
      const double deficit = want[(size_t)g] - th[(size_t)g];
      if (deficit > bd) {
        bd = deficit;
        best = g;
      }
    }
    th[(size_t)best] += 1;
    ++used;
  }
  // frames u in [U0, U0 + len): chunks of one odd length (the last shorter)
  const int U0 = -(L - 1), len = c->T + 2 * (L - 1);
  std::vector<int4> tab((size_t)NT + 1 + 2 * ng);
  int t = 0;
  for (int g = 0; g < ng; ++g) {
    const int want_n = th[(size_t)g];
    const int clen = (((len + want_n - 1) / want_n) | 1) + ((int)tune.cadd.size() == ng ? 2 * tune.cadd[(size_t)g] : 0);
    const int n = (len + clen - 1) / clen;
    const int rot = (int)tune.rot.size() == ng ? tune.rot[(size_t)g] % n : 0;
    const int t0 = t;
    for (int i = 0; i < want_n; ++i) {
      if (i < n) {
        const int k = (i + rot) % n;  // chunk k of the group (the reduction sums in thread order)
        tab[(size_t)t] = make_int4(g, U0 + k * clen, U0 + std::min(len, (k + 1) * clen), 0);
      } else {
        tab[(size_t)t] = make_int4(-1, 0, 0, 0);
      }
      ++t;
    }
    tab[(size_t)NT + 1 + 2 * g] = make_int4(gs[(size_t)g].m, gs[(size_t)g].m2, gs[(size_t)g].d, gs[(size_t)g].alo);
    tab[(size_t)NT + 2 + 2 * g] = make_int4(gs[(size_t)g].cnt, t0, t0 + n, 0);
  }
  tab[(size_t)NT] = make_int4(ng, 0, 0, 0);
  c->gtab_host = tab;
  c->gtab.alloc(tab.size());
  CK(cudaMemcpy(c->gtab.p, tab.data(), tab.size() * sizeof(int4), cudaMemcpyHostToDevice));
}

// Chooses the sweep variant and lays out its shared memory.
// CTF_SWEEP_KIND=0|1 restricts to frame-owner / row-per-warp kernels and
// CTF_SWEEP_VARIANT="rmax,ft,rreg,nt[,exact]" pins one (profiling aids).
void plan_sweep(ctf_ctx* c) {
  const auto& vars = c->prob.precision == CTF_F32 ? ctf::sweep_variants_f32() : ctf::sweep_variants_f64();
  int max_smem = 0;
  CK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
  max_smem -= 1024;  // static shared memory of the kernel + reserve
  const size_t rs = c->real_size, cs = 2 * rs;
  int force[5] = {0, 0, -1, 0, -1};
  if (const char* env = std::getenv("CTF_SWEEP_VARIANT"))
    std::sscanf(env, "%d,%d,%d,%d,%d", &force[0], &force[1], &force[2], &force[3], &force[4]);
  int force_kind = -1;
  if (const char* env = std::getenv("CTF_SWEEP_KIND")) force_kind = std::atoi(env);
  int force_ag = -1;  // frame-split exchange: 0 owner scheme, 1 all-gather
  if (const char* env = std::getenv("CTF_FSPLIT_AG")) force_ag = std::atoi(env);
  int force_pair = -1;  // frame-split: 1 two ISS steps per exchange, 0 one
  if (const char* env = std::getenv("CTF_FSPLIT_PAIR")) force_pair = std::atoi(env);
  const int lmax = std::max(1, *std::max_element(c->taps, c->taps + c->N));
  const int loff = ((lmax + 3) / 4) * 4;
  const bool want_chk = c->prob.checks != 0;
  const bool want_ip = c->prob.update_rule == CTF_RULE_IP;
  // best variant of kind only_kind (< 0: any) for the problem; pins: honour
  // the CTF_SWEEP_VARIANT / CTF_FSPLIT_AG profiling pins
  auto search = [&](int only_kind, bool chk, bool ip, bool pins, ctf::SweepVariant& best, size_t& best_smem,
                    int& best_nt, ctf::SweepParams& best_sp, int& best_TP) {
  bool found = false;
  int best_rank = 0;
  for (const auto& v : vars) {
    if (v.chk != (int)chk) continue;  // CheckOptions runs on the instrumented variants only
    if (v.ip != (int)ip) continue;    // the IP rule runs on the covariance-domain IP variants only
    if (only_kind >= 0 && v.kind != only_kind) continue;
    if (pins && force_ag >= 0 && v.kind == 5 && v.ag != force_ag) continue;
    if (pins && force_pair >= 0 && v.kind == 5 && v.pair != force_pair) continue;
    if (pins && force[0] && (v.rmax != force[0] || v.ft != force[1] || v.rreg != force[2] || v.maxt != force[3] ||
                     (force[4] >= 0 && v.exact != force[4])))
      continue;
    const int nt = v.maxt;  // exact CTA size of the variant
    const int NW = nt / 32;
    int TP;
    size_t off = 0;
    auto take = [&](size_t bytes) {
      const size_t o = off;
      off = align16(off + bytes);
      return o;
    };
    ctf::SweepParams cand = c->sp;
    int fs_sms = 0;  // kind 5: SMs covered by co-resident clusters
    if (v.kind == 0) {
      if (v.rmax < c->R || (v.exact && v.rmax != c->R)) continue;
      if (v.lt > 0) {
        bool equal = true;
        for (int n = 0; n < c->N; ++n) equal = equal && c->taps[n] == v.lt;
        if (!equal) continue;
      }
      if (nt * v.ft < c->T) continue;
      TP = nt * v.ft;
      const int VP = ((3 * v.rmax + 31) / 32) * 32;
      const int xoff = c->Ls - 1, xp = xoff + TP;
      cand.xoff = xoff;
      cand.xp = xp;
      cand.off_y = (int)take((size_t)(v.rmax - v.rreg) * TP * cs);
      const size_t xbytes =
          std::max((size_t)c->Mx * xp * cs, align16((size_t)v.rreg * TP * rs) + (size_t)c->N * TP * rs);
      cand.off_x = (int)take(xbytes);
      cand.off_e = cand.off_x + (int)align16((size_t)v.rreg * TP * rs);
      cand.off_l = (int)take((size_t)c->N * (loff + TP) * rs);
      cand.off_w = (int)take((size_t)2 * c->R * c->D * cs);
      cand.off_red = (int)take((size_t)2 * NW * VP * rs);
      cand.off_z = (int)take((size_t)NW * v.rmax * cs);
      cand.off_b = (int)take((size_t)c->SK * rs);
      cand.off_d = (int)take((size_t)NW * 4 * sizeof(double));
      if (v.ip) {  // IP rule: square W, warp solve (ip_solve_row)
        if (c->R != c->D || c->D > 32) continue;
        cand.off_ip = (int)take((size_t)(3 * c->D * c->D + 2 * c->D) * cs);
      }
    } else if (v.kind == 4) {  // covariance-domain (Gram) kernel: stacked equal taps, M = N
      const int M = v.rreg, L = v.lt;
      if (c->Mx != M || c->N != M || c->Ls != L || c->R != v.rmax || c->D != v.rmax) continue;
      bool equal = true;
      for (int n = 0; n < c->N; ++n) equal = equal && c->taps[n] == L;
      if (!equal) continue;
      if (nt * v.ft < c->T) continue;
      TP = nt * v.ft;
      const int UB = ctf::kGramUB, NA = 2 * L - 1;
      const int U0 = -(L - 1), U1 = U0 + c->T + 2 * (L - 1) + UB;
      cand.xoff = 2 * L;
      cand.xp = cand.xoff + std::max(TP, U1) + 2 * L + UB + gram_tune().xpk;
      const int gloff = 2 * L + 2;
      const int glp = gloff + std::max(TP, U1) + 2 * L + UB;
      cand.off_x = (int)take((size_t)M * cand.xp * cs);
      cand.off_l = (int)take((size_t)c->N * glp * rs);
      cand.off_y = (int)take((size_t)c->N * (M * (M + 1) / 2) * NA * NA * cs);  // Hermitian half of the Gram
      const int NS = (c->real_size == 4 && c->R <= 16) ? c->N : 1;  // sources per Gram pass (gram_ns) and demix group
      // (dev builds with -DCTF_GRAM_NS64 must size this from gram_ns as well)
      // partials of NSP sources at a time; |y|^2 rows of a source group, or
      // (ctf::gram_ereg: fp32 long-frame variants) only the energy halo
      const bool ereg = c->real_size == 4 && v.ft >= 8;
      const int NSP = ereg ? 1 : NS;
      const size_t LH = std::max(1, L - 1);  // halo [warp][frame pass][source][l-1][lane]
      size_t ebytes = std::max((size_t)NSP * NA * (nt + 1) * cs,
                               ereg ? (size_t)NW * v.ft * NS * LH * LH * rs : (size_t)NS * L * TP * rs);
      if (v.tc) {  // two stages of the tcgen05 Gram operands (ctf_gram.cuh GramTC)
        const int NG = M * L + (M * (M - 1) / 2) * NA, TILES = (NG + 127) / 128, NP = (M * NA + 15) / 16 * 16;
        ebytes = std::max(ebytes, (size_t)2 * (2 * 2 * (2 * TILES * 128 * 32) + 2 * 2 * NP * 32));
      }
      cand.off_e = (int)take(ebytes);
      cand.off_w = (int)take((size_t)c->R * c->D * cs);
      cand.off_z = (int)take((size_t)(2 * c->R * std::max(1, L - 1) + 2 * (c->D + std::max(1, L - 1))) * cs);
      cand.off_red = (int)take((size_t)32 * NW * rs);
      cand.off_b = (int)take((size_t)c->SK * rs);
      cand.off_d = (int)take((size_t)NW * 4 * sizeof(double));
      cand.loff = gloff;  // (re-set below with lp)
      cand.lp = glp;
    } else if (v.kind == 3) {  // cluster: CS = R / RB CTAs per bin
      const int RB = v.rmax, CS = c->R / RB;
      if (c->R % RB != 0 || CS < 2 || CS > 16) continue;
      TP = nt * v.ft;
      if (TP < c->T || (v.ft > 1 && nt * (v.ft - 1) >= c->T)) continue;
      // sources touched by one CTA's rows (for the 1/lambda and energy buffers)
      int nsrc = 1;
      for (int q = 0; q < CS; ++q) {
        int r0 = q * RB, n0 = 0, n1 = 0, acc = 0;
        for (int n = 0; n < c->N; ++n) {
          if (r0 >= acc && r0 < acc + c->taps[n]) n0 = n;
          if (r0 + RB - 1 >= acc && r0 + RB - 1 < acc + c->taps[n]) n1 = n;
          acc += c->taps[n];
        }
        nsrc = std::max(nsrc, n1 - n0 + 1);
      }
      const int VP = ((3 * RB + 31) / 32) * 32;
      cand.xoff = c->Ls - 1;
      cand.xp = cand.xoff + TP;
      cand.off_y = (int)take(std::max((size_t)(RB - v.rreg) * TP * cs, (size_t)(nsrc + 1) * TP * rs));
      // x stage + 1/lambda, reused for |y|^2 of the own rows in the epilogue
      const size_t xb = (size_t)(cand.xoff + TP) * cs, lb = (size_t)nsrc * (loff + TP) * rs;
      const size_t xl = std::max(align16(xb) + lb, (size_t)RB * TP * rs);
      cand.off_x = (int)take(xl);
      cand.off_l = cand.off_x + (int)align16(xb);
      cand.off_w = (int)take((size_t)c->D * RB * cs);
      cand.off_e = (int)take((size_t)c->D * cs);
      cand.off_red = (int)take((size_t)2 * NW * VP * rs);
      cand.off_z = (int)take((size_t)NW * RB * cs);
      cand.off_b = (int)take((size_t)c->SK * rs);
      cand.off_d = (int)take((size_t)(NW * 4 + c->R) * sizeof(double));
    } else if (v.kind == 5) {  // frame-split cluster: stacked equal taps, M = N, CS CTAs per bin
      const int L = v.lt, CS = v.cs;
      if (c->R != v.rmax || c->D != v.rmax || c->Ls != L || c->Mx * L != c->R || c->N * L != c->R) continue;
      bool equal = true;
      for (int n = 0; n < c->N; ++n) equal = equal && c->taps[n] == L;
      if (!equal) continue;
      TP = nt * v.ft;  // frames per CTA
      if ((long)CS * TP < c->T || (long)(CS - 1) * TP >= c->T) continue;  // no idle CTA
      off = v.fbytes(c->SK);
      if (off > (size_t)max_smem) continue;
      // the cluster must be schedulable (same-GPC placement, shared memory)
      CK(cudaFuncSetAttribute((const void*)v.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)off));
      if (CS > 8) CK(cudaFuncSetAttribute((const void*)v.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(CS * c->FL, c->B);
      lc.blockDim = dim3(nt);
      lc.dynamicSmemBytes = off;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CS;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)v.fn, &lc) != cudaSuccess || nclusters < 1) {
        cudaGetLastError();
        continue;
      }
      // SMs the co-resident clusters cover (GPC packing: 8-CTA clusters leave
      // 28 of 148 SMs idle, 9-CTA ones 13): the planner prefers the most
      int per_sm = 1, nsm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, v.fn, nt, off));
      CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
      fs_sms = std::min(nsm, nclusters * CS / std::max(1, per_sm));
    } else if (v.kind == 2) {  // streamed: any R <= 64, tile in global scratch
      if (c->R > v.rmax) continue;
      TP = nt * v.ft;
      if (TP < c->T) continue;
      const int RG = v.rreg, NG = (c->R + RG - 1) / RG, VP = ((3 * RG + 31) / 32) * 32;
      cand.xoff = c->Ls - 1;
      cand.xp = cand.xoff + TP;
      cand.off_y = 0;
      cand.off_l = (int)take((size_t)c->N * (loff + TP) * rs);
      cand.off_w = (int)take((size_t)2 * c->R * c->D * cs);
      cand.off_red = (int)take((size_t)NW * NG * VP * rs);
      cand.off_z = (int)take((size_t)c->R * cs);
      cand.off_b = (int)take((size_t)c->SK * rs);
      cand.off_d = (int)take((size_t)(NW * 4 + c->R) * sizeof(double));
      cand.off_x = (int)take((size_t)(cand.xoff + TP) * cs);
      cand.off_e = 0;
    } else {
      const int wpr = v.rreg;
      if (v.rmax != c->R) continue;                 // one row per WPR warps
      if (wpr > 1 && c->R > 15) continue;           // named barriers 1..15
      if (c->Ls - 1 > v.ft) continue;               // stacked taps reach one chunk back
      TP = 32 * wpr * v.ft;
      if (TP < c->T) continue;
      const int CH = v.ft + 2;
      const size_t XP = (size_t)(TP / v.ft + 1) * CH;
      cand.xoff = 0;
      cand.xp = (int)XP;
      cand.off_y = (int)take((size_t)2 * (TP / v.ft) * CH * cs);
      cand.off_x = (int)take(std::max((size_t)c->Mx * XP * cs, (size_t)c->R * TP * rs));
      cand.off_e = (int)take((size_t)c->N * TP * rs);
      cand.off_l = (int)take((size_t)c->N * (loff + TP) * rs);
      cand.off_w = (int)take((size_t)2 * c->R * c->D * cs);
      cand.off_red = (int)take((size_t)2 * c->R * wpr * 4 * rs);
      cand.off_z = (int)take(16);
      cand.off_b = (int)take((size_t)c->SK * rs);
      cand.off_d = (int)take((size_t)(NW * 4 + c->R) * sizeof(double));
    }
    if (off > (size_t)max_smem) continue;
    // preference: frame-owner kernels (measured faster than row-per-warp on
    // B200 for every shape so far), then
    // the smallest RMAX, exact before guarded, then the least frame padding
    // (fewest threads), then table order
    // resident single-CTA kernels first, then clusters (on-chip tile over
    // several SMs), the streamed kernel only when nothing else fits
    // (measured on B200: the cluster kernel is correct but slower than the
    // streamed one for cfg3/cfg4 so far, so it ranks last; CTF_SWEEP_KIND=3
    // selects it)
    // step pairs (two ISS steps per pass and exchange) preferred for R <= 32
    // (cfg3 41.86 vs 42.87 ms per 16 mixtures), one step per exchange for
    // R = 60 (cfg4 203.2 vs 201.9 ms per 8: the 8R sums per pair cost more
    // reduce-scatter than the halved exchanges save);
    // the frame-split cluster kernel (kind 5, only compiled for the wide
    // stacked tiles R = 32 / 60) first, the fewest CTAs per cluster and the
    // all-gather exchange preferred (cfg3 43.1 vs 44.6 ms per 16 mixtures
    // with the owner exchange; cfg4 equal)
    // (measured on B200: cfg3 45.6 ms per 16 mixtures at CS = 2 vs 51.9 at
    // CS = 4 and 53.3 on the covariance kernel; cfg4 103 ms per 4 mixtures at
    // CS = 8 vs 108 at CS = 16 and 212 streamed);
    // covariance-domain next, except fp64 with R <= 4 where the frame-domain
    // sweep measured faster (cfg0 f64: 0.046 vs 0.051 ms per iteration)
    const int gram_rank = (c->real_size == 8 && c->R <= 4 && !want_ip) ? 500 : -1000;
    // wide covariance tiles (R > 16, one CTA per SM) run best with the most threads
    const int wide_bonus = (v.kind == 4 && c->R > 16) ? -nt / 128 : 0;
    // tcgen05 Gram: preferred with CTF_GRAM_TC=1, else ranked just after its CUDA-core twin
    const char* tc_env = std::getenv("CTF_GRAM_TC");
    const int tc_rank = v.tc ? ((tc_env && std::atoi(tc_env)) ? -6000 : 50) : 0;
    const int rank = wide_bonus + tc_rank +
                     (v.kind == 4 ? gram_rank : v.kind == 3 ? 3000 : v.kind == 2 ? 2000 : v.kind == 5 ? (c->R > 16 ? -2000 - 10 * fs_sms : 4000) + v.cs + (1 - v.ag) + (c->R <= 32 ? -v.pair : v.pair) : v.kind == 1 ? 1000 : 0) +
                     (v.kind == 3 ? -v.rmax * 4 : v.rmax * 4) + (v.exact ? 0 : 2) + (v.lt > 0 ? 0 : 1);
    const bool better = !found || rank < best_rank ||
                        (rank == best_rank && (TP < best_TP || (TP == best_TP && nt < best_nt)));
    if (better) {
      found = true;
      best = v;
      best_rank = rank;
      best_smem = off;
      best_nt = nt;
      if (v.kind != 4) {
        cand.loff = loff;
        cand.lp = loff + TP;
      }
      best_TP = TP;
      best_sp = cand;
    }
  }
  return found;
  };
  ctf::SweepVariant best{};
  size_t best_smem = 0;
  int best_nt = 0, best_TP = 0;
  const bool found = search(force_kind, want_chk, want_ip, true, best, best_smem, best_nt, c->sp, best_TP);
  c->TP = best_TP;
  if (!found && want_ip)
    throw CtfError(CTF_ERR_CONFIG,
                   "update rule 'ip' on the GPU needs a square demixing matrix (sum of taps == channels) with "
                   "R <= 16 and T <= 2048 frames (frame-domain IP variants), or a compiled covariance-domain "
                   "(mics, taps) pair");
  if (!found && want_chk)
    throw CtfError(CTF_ERR_UNSUPPORTED, "CheckOptions need R <= 64 and T <= 4096 (instrumented frame-domain and streamed kernels)");
  if (!found)
    throw CtfError(CTF_ERR_UNSUPPORTED, "no compiled sweep kernel for R=" + std::to_string(c->R) +
                                            " T=" + std::to_string(c->T));
  c->sv = best;
  c->NT = best_nt;
  if (const char* pad = std::getenv("CTF_SMEM_PAD"))  // measurement aid: lower the CTAs per SM
    best_smem += (size_t)std::atoi(pad);
  c->sweep_smem = best_smem;
  if (best.kind == 3) {
    CK(cudaFuncSetAttribute((const void*)best.cfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)best_smem));
    CK(cudaFuncSetAttribute((const void*)best.cfn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    c->cluster_size = c->R / best.rmax;
  } else if (best.kind == 5) {
    CK(cudaFuncSetAttribute((const void*)best.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)best_smem));
    if (best.cs > 8) CK(cudaFuncSetAttribute((const void*)best.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    c->cluster_size = best.cs;
  } else if (best.kind == 2) {
    CK(cudaFuncSetAttribute((const void*)best.sfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)best_smem));
    int per_sm = 0, nsm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, best.sfn, best_nt, best_smem));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
    c->stream_grid = std::max(1, std::min(std::max(1, per_sm) * nsm, c->B * c->FL));
  } else if (best.kind == 4) {
    CK(cudaFuncSetAttribute((const void*)best.gfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)best_smem));
    build_gram_table(c, best_nt, best.rreg, best.lt);
  } else {
    CK(cudaFuncSetAttribute((const void*)best.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)best_smem));
  }
  // L2 prefetch distance of the one-CTA-per-bin kernels: the number of CTAs
  // resident at once (the ones launched next start about that many items later)
  c->sp.pf_stride = 0;
  if (best.kind == 0 || best.kind == 4) {
    int per_sm = 0, nsm = 0;
    if (best.kind == 4)
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, best.gfn, best_nt, best_smem));
    else
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, best.fn, best_nt, best_smem));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
    const char* env = std::getenv("CTF_PREFETCH");
    if (!(env && std::atoi(env) == 0)) c->sp.pf_stride = std::max(1, per_sm) * nsm;
  }
  auto finish = [&](ctf::SweepParams& sp, int TP) {
  sp.FL = c->FL;
  sp.bin_lo = c->lo;
  sp.T = c->T;
  sp.TP = TP;
  sp.Mx = c->Mx;
  sp.Ls = c->Ls;
  sp.D = c->D;
  sp.R = c->R;
  sp.N = c->N;
  sp.SK = c->SK;
  int r = 0;
  for (int n = 0; n < c->N; ++n) {
    sp.row0[n] = c->row0[n];
    sp.ntaps[n] = c->taps[n];
    for (int l = 0; l < c->taps[n]; ++l, ++r) sp.woff[r] = n * sp.lp + sp.loff - l;
  }
  for (int n = 0; n <= c->N; ++n) sp.koff[n] = c->koff[n];
  {
    int rr = 0;
    for (int n = 0; n < c->N; ++n)
      for (int l = 0; l < c->taps[n]; ++l) sp.srcr[rr++] = n;
  }
  for (int ch = 0; ch < c->D && ch < ctf::kMaxRows; ++ch) {
    const int m = ch / c->Ls, l = ch - m * c->Ls;
    sp.xcol[ch] = m * sp.xp + sp.xoff - l;
  }
  sp.fb_mode = 0;
  };
  finish(c->sp, c->TP);
  // Conditioning fallback (SweepParams::fb_mode): the ISS covariance-domain
  // kernel hands bins whose Gram form is ill-conditioned in this precision to
  // the best frame-domain variant for the same problem (kappa threshold: fp32
  // 64, healthy bins measure 5-17; fp64 1e7). CTF_GRAM_FALLBACK=0 disables it.
  c->has_fb = false;
  const char* fb_env = std::getenv("CTF_GRAM_FALLBACK");
  if (best.kind == 4 && !want_ip && !want_chk && !(fb_env && std::atoi(fb_env) == 0)) {
    int fb_TP = 0;
    if (search(0, false, false, false, c->fbv, c->fb_smem, c->fb_nt, c->sp_fb, fb_TP)) {
      c->has_fb = true;
      finish(c->sp_fb, fb_TP);
      c->sp_fb.pf_stride = 0;
      c->fb_theta = c->real_size == 4 ? 64.0 : 1e7;
      if (const char* th = std::getenv("CTF_GRAM_FALLBACK_THETA")) c->fb_theta = std::atof(th);
      CK(cudaFuncSetAttribute((const void*)c->fbv.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)c->fb_smem));
      int per_sm = 0, nsm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, c->fbv.fn, c->fb_nt, c->fb_smem));
      CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
      c->fb_grid = std::max(1, std::min(std::max(1, per_sm) * nsm, c->B * c->FL));
    }
  }
}

template <class Real>
__global__ void convert_kernel(const double* in, Real* out, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = (Real)in[i];
}
template <class Real>
__global__ void convert_f32_kernel(const float* in, Real* out, size_t n) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = (Real)in[i];
}
template <class Real>
__global__ void identity_kernel(Real* W, size_t nbins, int R, int D) {
  // W per bin: column-major R x D complex (2 reals per entry)
  const size_t per = (size_t)R * D * 2;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nbins * per; i += (size_t)gridDim.x * blockDim.x) {
    const size_t e = (i % per) / 2;
    const int r = (int)(e % R), col = (int)(e / R);
    W[i] = (Real)((r == col && (i & 1) == 0) ? 1.0 : 0.0);
  }
}

void upload_real(ctf_ctx* c, void* dst, const double* src, size_t n) {
  // host doubles -> device Real
  if (c->real_size == 8) {
    CK(cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyHostToDevice, c->stream));
    return;
  }
  if (c->stage.n < n) c->stage.alloc(n);
  CK(cudaMemcpyAsync(c->stage.p, src, n * 8, cudaMemcpyHostToDevice, c->stream));
  convert_kernel<float><<<std::min<size_t>((n + 255) / 256, 4096), 256, 0, c->stream>>>(c->stage.p, (float*)dst, n);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c->stream));  // the host source may be released by the caller
}

// Device-side gathers into the double staging buffer in the host layouts
// (then one D2H per array straight into the caller's buffer).
template <class Real>
__global__ void gather_W_kernel(const Real* W, double* out, size_t n) {  // same layout, precision only
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = (double)W[i];
}
// B: device [mix][FL][SK] -> [mix][n][k][FL] (each B_n column-major FL x K_n)
template <class Real>
__global__ void gather_B_kernel(const Real* B, double* out, int nmix, int FL, int SK) {
  const size_t n = (size_t)nmix * FL * SK;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const size_t mix = e / ((size_t)FL * SK);
    const size_t rem = e - mix * FL * SK;
    const int kk = (int)(rem / FL), i = (int)(rem - (size_t)kk * FL);  // kk = global base index (koff[n] + k)
    out[e] = (double)B[((size_t)mix * FL + i) * SK + kk];
  }
}
// V: device [mix][SK][T] -> [mix][n] column-major K_n x T, i.e. [mix][n][t][k]
struct VMap {
  int koff[ctf::kMaxSources + 1];
  int N;
};
template <class Real>
__global__ void gather_V_kernel(const Real* V, double* out, int nmix, int SK, int T, VMap vm) {
  const size_t n = (size_t)nmix * SK * T;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    const size_t mix = e / ((size_t)SK * T);
    const size_t rem = e - mix * SK * T;  // offset inside the mixture: sum over earlier sources + (k + t*K_n)
    int src = 0;
    while (rem >= (size_t)vm.koff[src + 1] * T) ++src;
    const int K = vm.koff[src + 1] - vm.koff[src];
    const size_t o = rem - (size_t)vm.koff[src] * T;
    const int t = (int)(o / K), k = (int)(o - (size_t)t * K);
    out[e] = (double)V[((size_t)mix * SK + vm.koff[src] + k) * T + t];
  }
}

void download_real(ctf_ctx* c, double* dst, const void* src, size_t n) {
  if (c->real_size == 8) {
    CK(cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    return;
  }
  if (c->stage.n < n) c->stage.alloc(n);
  convert_f32_kernel<double><<<std::min<size_t>((n + 255) / 256, 4096), 256, 0, c->stream>>>((const float*)src, c->stage.p, n);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(dst, c->stage.p, n * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
}

void allreduce(ctf_ctx* c, void* buf, size_t count, int dtype, int op, cudaStream_t st = nullptr) {
  if (!c->collective() || count == 0) return;
  if (!st) st = c->stream;
  if (c->group) {  // host exchange, fixed rank order (deterministic)
    const size_t es = dtype == kNcclFloat ? 4 : 8;
    ctf_group* g = c->group;
    auto& mine = g->slots[(size_t)c->rank];
    mine.resize(count * es);
    CK(cudaMemcpyAsync(mine.data(), buf, count * es, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    g->barrier();
    std::vector<unsigned char> out(count * es);
    for (size_t i = 0; i < count; ++i) {
      if (dtype == kNcclFloat) {
        float a = 0.f;
        for (int r = 0; r < g->world; ++r) a += reinterpret_cast<const float*>(g->slots[(size_t)r].data())[i];
        reinterpret_cast<float*>(out.data())[i] = a;
      } else if (dtype == kNcclDouble) {
        double a = 0.0;
        for (int r = 0; r < g->world; ++r) a += reinterpret_cast<const double*>(g->slots[(size_t)r].data())[i];
        reinterpret_cast<double*>(out.data())[i] = a;
      } else {  // uint64 min / max
        unsigned long long a = op == kNcclMax ? 0ull : ~0ull;
        for (int r = 0; r < g->world; ++r) {
          const unsigned long long v = reinterpret_cast<const unsigned long long*>(g->slots[(size_t)r].data())[i];
          a = op == kNcclMax ? std::max(a, v) : std::min(a, v);
        }
        reinterpret_cast<unsigned long long*>(out.data())[i] = a;
      }
    }
    g->barrier();  // every rank has read every slot
    CK(cudaMemcpyAsync(buf, out.data(), count * es, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    return;
  }
  const int rc = g_nccl.AllReduce(buf, buf, count, dtype, op, c->comm, st);
  if (rc != 0)
    throw CtfError(CTF_ERR_CUDA, std::string("ncclAllReduce failed: ") +
                                     (g_nccl.GetErrorString ? g_nccl.GetErrorString(rc) : "?"));
}

// Decodes the per-mixture error keys into the reference's exception text.
void check_errors(ctf_ctx* c) {
  std::vector<unsigned long long> keys((size_t)c->B);
  if (c->collective()) allreduce(c, c->err.p, (size_t)c->B, kNcclUint64, kNcclMin);
  CK(cudaMemcpyAsync(keys.data(), c->err.p, keys.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int b = 0; b < c->B; ++b) {
    const unsigned long long k = keys[(size_t)b];
    if (k == ctf::kNoErr) continue;
    const int it = (int)(k >> 44), ph = (int)((k >> 40) & 0xF), bin = (int)((k >> 20) & 0xFFFFF),
              row = (int)((k >> 8) & 0xFFF), code = (int)(k & 0xFF);
    const std::string its = " (iteration " + std::to_string(it) + ")";
    switch (ph) {
      case ctf::kPhSweep:
        if (c->prob.update_rule == CTF_RULE_IP)  // estimator.cpp:105-108, 111-115
          throw CtfError(CTF_ERR_DEGENERACY,
                         std::string(code == 1 ? "projection update: singular system after diagonal loading"
                                               : "projection update: nonpositive row power") +
                             its,
                         CTF_KIND_PROJECTION, it, b, bin, row);
        throw CtfError(CTF_ERR_DEGENERACY,
                       "steering update: nonpositive denominator for rows (" + std::to_string(row) + ", " +
                           std::to_string(code) + ")" + its,
                       CTF_KIND_STEERING_DENOM, it, b, bin, row);
      case ctf::kPhFinite:
        if (code == 1)
          throw CtfError(CTF_ERR_DEGENERACY, "non-finite demixing matrix", CTF_KIND_NONFINITE_W, it, b, bin, -1);
        throw CtfError(CTF_ERR_DEGENERACY, "non-finite source estimates", CTF_KIND_NONFINITE_Y, it, b, bin, -1);
      case ctf::kPhDet:
        if (code == 4)
          throw CtfError(CTF_ERR_DEGENERACY, "singular demixing matrix (zero pivot)" + its, CTF_KIND_ZERO_PIVOT, it,
                         b, bin, -1);
        throw CtfError(CTF_ERR_DEGENERACY, "demixing determinant magnitude below 1e-300" + its, CTF_KIND_TINY_DET,
                       it, b, bin, -1);
      case ctf::kPhObj:
        throw CtfError(CTF_ERR_DEGENERACY, "non-finite objective", CTF_KIND_NONFINITE_OBJ, it, b, -1, -1);
      default:
        throw CtfError(CTF_ERR_DEGENERACY, "degeneracy", 0, it, b, bin, row);
    }
  }
}

template <class Real>
void launch_muv(ctf_ctx* c, int m0, int m1, cudaStream_t st) {
  ctf::MuvParams mp{};
  mp.mix0 = m0;
  mp.Bf = c->Bf.p;
  mp.V = c->V.p;
  mp.E = c->E.p;
  mp.part = c->part.p;
  mp.floor_abs = c->floor_abs.p;
  mp.FL = c->FL;
  mp.T = c->T;
  mp.N = c->N;
  mp.SK = c->SK;
  mp.nmix = c->B;
  mp.chunk_bins = c->chunk_bins;
  for (int n = 0; n <= c->N; ++n) mp.koff[n] = c->koff[n];
  for (int n = 0; n < c->N; ++n) mp.ntaps[n] = c->taps[n];
  // KS = 2 (bases split over half-warps) for K >= 16: half the registers,
  // twice the resident warps (CTF_MUV_KS=1|2 pins it for measurement)
  int ks = 1;
  if (const char* e = std::getenv("CTF_MUV_KS")) ks = std::atoi(e) == 2 && c->kmax % 2 == 0 ? 2 : 1;
  dim3 grid(ks == 2 ? (c->T + 63) / 64 : (c->T + 127) / 128, (m1 - m0) * c->N, c->nchunk);
  const size_t smem = (size_t)((c->chunk_bins + 7) / 8 * 8) * c->kmax * sizeof(Real);
#define CTF_MUV(KM)                                                                  \
  (ks == 2 ? ctf::muv_partial_kernel<Real, KM, 2><<<grid, 128, smem, st>>>(mp)     \
           : ctf::muv_partial_kernel<Real, KM, 1><<<grid, 128, smem, st>>>(mp))
  switch (c->kmax) {
    case 4: CTF_MUV(4); break;
    case 10: CTF_MUV(10); break;
    case 12: CTF_MUV(12); break;
    case 20: CTF_MUV(20); break;
    case 8: CTF_MUV(8); break;
    case 16: CTF_MUV(16); break;
    case 24: CTF_MUV(24); break;
    default: CTF_MUV(32); break;
  }
#undef CTF_MUV
  CK(cudaGetLastError());
}

template <class Real>
void launch_apply(ctf_ctx* c, int mode, int obj_slot, int do_v, int m0, int m1, cudaStream_t st) {
  ctf::ApplyParams ap{};
  ap.mix0 = m0;
  ap.part = c->part.p;
  ap.packed = c->packed.p;
  ap.V = c->V.p;
  ap.rowpow = c->rowpow.p;
  ap.objbin = c->objbin.p;
  ap.packed_d = c->packed_d.p;
  ap.mu = c->mu.p;
  ap.logmu = c->logmu.p;
  ap.objective = c->objective.p;
  ap.floor_abs = c->floor_abs.p;
  ap.err = c->err.p;
  ap.nchunk = c->nchunk;
  ap.nmix = c->B;
  ap.SK = c->SK;
  ap.T = c->T;
  ap.FL = c->FL;
  ap.R = c->R;
  ap.F_total = c->F;
  ap.max_iters = c->max_iters;
  ap.obj_slot = obj_slot;
  ap.mode = mode;
  ap.do_v = do_v;
  const size_t plane = (size_t)c->SK * c->T;
  const int bx = do_v ? (int)std::min<size_t>((plane + 255) / 256, 64) : 1;
  ctf::reduce_apply_kernel<Real><<<dim3(bx, m1 - m0), 256, 0, st>>>(ap);
  CK(cudaGetLastError());
}

// One loop body (estimator.cpp:553-654) or, with do_sweep = false, the
// trailing rescale + objective of the last completed iteration.
// The iteration kernel (+ its fallback) for mixtures [m0, m1).
size_t plane_stride(const ctf_ctx* c) { return (size_t)c->FL * c->R * c->D; }

// 1 / lambda and the objective's log term of mixtures [m0, m1) for the loop
// body about to run (compute_psd with the pending rescale of B).
template <class Real>
void launch_lambda(ctf_ctx* c, int m0, int m1, cudaStream_t st) {
  ctf::LambdaParams lp{};
  const size_t mz = (size_t)m0, rs = c->real_size;
  lp.Bf = c->Bf.p + mz * c->FL * c->SK * rs;
  lp.V = c->V.p + mz * c->SK * c->T * rs;
  lp.invl = c->invl.p + mz * c->FL * c->N * c->T * rs;
  lp.logsum = c->logsum.p + mz * c->FL;
  lp.mu = c->pending ? c->mu.p + mz * c->R : nullptr;
  lp.floor_abs = c->floor_abs.p + mz;
  lp.FL = c->FL;
  lp.T = c->T;
  lp.N = c->N;
  lp.SK = c->SK;
  lp.R = c->R;
  lp.has_prev = c->pending ? 1 : 0;
  for (int n = 0; n <= c->N; ++n) lp.koff[n] = c->koff[n];
  for (int n = 0; n < c->N; ++n) {
    lp.ntaps[n] = c->taps[n];
    lp.row0[n] = c->row0[n];
  }
  constexpr int VEC = 16 / (int)sizeof(Real);
  const dim3 grid((c->FL + ctf::kLambdaBins - 1) / ctf::kLambdaBins, m1 - m0);
  const bool vec = c->T % VEC == 0;  // 16-byte V loads / stores (else one frame per thread)
#define CTF_LAM(KM)                                                                                          \
  {                                                                                                          \
    const size_t sm = (size_t)ctf::kLambdaBins * c->N * ((KM + 3) / 4 * 4) * sizeof(Real);                   \
    if (vec) ctf::lambda_kernel<Real, KM, VEC><<<grid, 256, sm, st>>>(lp);                                   \
    else ctf::lambda_kernel<Real, KM, 1><<<grid, 256, sm, st>>>(lp);                                         \
  }
  switch (c->kmax) {
    case 4: CTF_LAM(4); break;
    case 8: CTF_LAM(8); break;
    case 10: CTF_LAM(10); break;
    case 12: CTF_LAM(12); break;
    case 16: CTF_LAM(16); break;
    case 20: CTF_LAM(20); break;
    case 24: CTF_LAM(24); break;
    default: CTF_LAM(32); break;
  }
#undef CTF_LAM
  CK(cudaGetLastError());
  c->timing.launches += 1;
}

// MU-B of mixtures [m0, m1) after an iteration kernel compiled without it
// (SweepVariant::mubout): B <- max(B sqrt(num / den), floor) from E and 1/lambda.
template <class Real>
void launch_mub(ctf_ctx* c, int m0, int m1, cudaStream_t st) {
  ctf::MubParams mp{};
  const size_t mz = (size_t)m0, rs = c->real_size;
  mp.Bf = c->Bf.p + mz * c->FL * c->SK * rs;
  mp.V = c->V.p + mz * c->SK * c->T * rs;
  mp.E = c->E.p + mz * c->N * c->FL * c->T * rs;
  mp.invl = c->invl.p + mz * c->FL * c->N * c->T * rs;
  mp.floor_abs = c->floor_abs.p + mz;
  mp.err = c->err.p + mz;
  mp.FL = c->FL;
  mp.T = c->T;
  mp.N = c->N;
  mp.SK = c->SK;
  for (int n = 0; n <= c->N; ++n) mp.koff[n] = c->koff[n];
  for (int n = 0; n < c->N; ++n) mp.ntaps[n] = c->taps[n];
  constexpr int VEC = 16 / (int)sizeof(Real);
  const dim3 grid((c->FL + 7) / 8, c->N, m1 - m0);
  if (c->T % VEC == 0) ctf::mub_kernel<Real, VEC><<<grid, 256, 0, st>>>(mp);
  else ctf::mub_kernel<Real, 1><<<grid, 256, 0, st>>>(mp);
  CK(cudaGetLastError());
  c->timing.launches += 1;
}

template <class Real>
void launch_sweep(ctf_ctx* c, bool do_sweep, int m0, int m1, int k, cudaStream_t st) {
  ctf::SweepParams sp = c->sp;
  // per-mixture buffers offset to the launch's first mixture m0 on the host:
  // the kernels index mixtures by blockIdx.y alone (an in-kernel
  // blockIdx.y + m0 measured 3.7 % slower on cfg1 fp32: one more live register)
  auto fill = [&](ctf::SweepParams& sp) {
  const size_t mz = (size_t)m0, rs = c->real_size, cs = 2 * rs;
  sp.x = c->x.p + mz * c->FL * c->T * c->Mx * cs;
  sp.W = c->W.p + mz * plane_stride(c) * cs;
  sp.Bf = c->Bf.p + mz * c->FL * c->SK * rs;
  sp.V = c->V.p + mz * c->SK * c->T * rs;
  sp.E = c->E.p + mz * c->N * c->FL * c->T * rs;
  sp.rowpow = c->rowpow.p + mz * c->FL * c->R;
  sp.objbin = c->objbin.p + mz * c->FL;
  sp.mu = c->pending ? c->mu.p + mz * c->R : nullptr;
  sp.logmu = c->logmu.p + mz;
  sp.floor_abs = c->floor_abs.p + mz;
  sp.err = c->err.p + mz;
  sp.chk = c->chk.p + 2 * mz;
  sp.chk_flags = c->prob.checks;
  sp.logdet = c->logdet.p + mz * c->FL;
  sp.iteration = c->done + 1;
  sp.do_sweep = do_sweep ? 1 : 0;
  sp.has_prev = c->pending ? 1 : 0;
  sp.fb_list = c->fb_list.p ? c->fb_list.p + mz * c->FL : nullptr;  // chunk k's tiles (local indices)
  sp.fb_count = c->fb_count.p ? c->fb_count.p + k : nullptr;
  sp.fb_theta = c->fb_theta;
  sp.nmix = c->B - m0;  // mixtures from the offset base (the L2 prefetch bound)
  };
  fill(sp);
  const int nm = m1 - m0;
  if (c->sv.kind == 3) {
    ctf::ClusterParams cl{};
    cl.s = sp;
    cl.pivot = c->cpivot.p;
    cl.wpivot = c->cwpivot.p;
    cl.part = c->cpart.p;
    cl.bad = c->cbad.p;
    cl.CS = c->cluster_size;
    CK(cudaMemsetAsync(c->cbad.p, 0, c->cbad.n * sizeof(int), st));
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(c->FL * c->cluster_size, nm);
    lc.blockDim = dim3(c->NT);
    lc.dynamicSmemBytes = c->sweep_smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c->cluster_size;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, c->sv.cfn, cl));
  } else if (c->sv.kind == 5) {
    if (c->lam_pre) {
      launch_lambda<Real>(c, m0, m1, st);
      sp.invl_g = c->invl.p + (size_t)m0 * c->FL * c->N * c->T * c->real_size;
      sp.logsum_g = c->logsum.p + (size_t)m0 * c->FL;
    }
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(c->FL * c->cluster_size, nm);
    lc.blockDim = dim3(c->NT);
    lc.dynamicSmemBytes = c->sweep_smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c->cluster_size;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, c->sv.fn, sp));
    if (do_sweep && c->lam_pre && c->sv.mubout) launch_mub<Real>(c, m0, m1, st);
  } else if (c->sv.kind == 2) {  // persistent over all work items (never chunked)
    ctf::StreamParams stp{};
    stp.s = sp;
    stp.scratch = c->scratch.p;
    stp.nwork = c->B * c->FL;
    stp.ngroups = (c->R + c->sv.rreg - 1) / c->sv.rreg;
    c->sv.sfn<<<c->stream_grid, c->NT, c->sweep_smem, st>>>(stp);
  } else if (c->sv.kind == 4) {
    if (c->has_fb) {
      CK(cudaMemsetAsync(c->fb_count.p + k, 0, sizeof(int), st));  // chunk k's list
      sp.fb_mode = 1;
    }
    if (c->lam_pre) {
      // (dev: CTF_DEV_SKIP_LAMBDA=1 times the iteration kernel alone on stale 1 / lambda)
      static const bool skip = std::getenv("CTF_DEV_SKIP_LAMBDA") != nullptr;
      static const bool tim = std::getenv("CTF_DEV_TIME_LAMBDA") != nullptr;  // dev: event-timed in the stream
      cudaEvent_t t0 = nullptr, t1 = nullptr;
      if (tim) {
        t0 = take_event(c);
        t1 = take_event(c);
        CK(cudaEventRecord(t0, st));
      }
      if (!skip || c->done < 2) launch_lambda<Real>(c, m0, m1, st);
      if (tim) {
        CK(cudaEventRecord(t1, st));
        c->ev_lam.push_back({t0, t1});
      }
      sp.invl_g = c->invl.p + (size_t)m0 * c->FL * c->N * c->T * c->real_size;
      sp.logsum_g = c->logsum.p + (size_t)m0 * c->FL;
    }
    c->sv.gfn<<<dim3(c->FL, nm), c->NT, c->sweep_smem, st>>>(sp, c->gtab.p);
    if (c->has_fb) {  // the bins the Gram form handed over, in the frame domain
      CK(cudaGetLastError());
      ctf::SweepParams fp = c->sp_fb;
      fill(fp);
      fp.fb_mode = 2;
      c->fbv.fn<<<c->fb_grid, c->fb_nt, c->fb_smem, st>>>(fp);
      c->timing.launches += 1;
    }
  } else {
    c->sv.fn<<<dim3(c->FL, nm), c->NT, c->sweep_smem, st>>>(sp);
  }
  CK(cudaGetLastError());
  c->timing.sweep_launches += 1;
  c->timing.launches += 1;
}

// Applies the deferred V update / rescale of mixture chunk k (after its all-reduce).
template <class Real>
void apply_deferred(ctf_ctx* c, int k) {
  auto& d = c->deferred[(size_t)k];
  if (!d.on) return;
  const int m0 = c->mix_split[(size_t)k], m1 = c->mix_split[(size_t)k + 1];
  const cudaStream_t st = c->chunk_stream(k);
  CK(cudaStreamWaitEvent(st, c->ev_ar[(size_t)k], 0));
  launch_apply<Real>(c, 1, d.obj_slot, d.do_v, m0, m1, st);
  c->timing.launches += 1;
  d.on = false;
}

template <class Real>
void flush_deferred(ctf_ctx* c) {
  for (int k = 0; k < c->nmc && k < (int)c->deferred.size(); ++k) apply_deferred<Real>(c, k);
  if (c->stream2) {  // the odd chunks' work joins the context stream
    CK(cudaEventRecord(c->ev_join, c->stream2));
    CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  }
}

// One loop body (estimator.cpp:553-654) or, with do_sweep = false, the
// trailing rescale + objective of the last completed iteration.
template <class Real>
void run_body(ctf_ctx* c, bool do_sweep) {
  const int obj_slot = c->pending ? c->done - 1 : -1;
  const int do_v = do_sweep ? 1 : 0;
  cudaEvent_t e0 = take_event(c), e1 = take_event(c), e2 = take_event(c);
  CK(cudaEventRecord(e0, c->stream));
  if (c->nmc > 1) {
    // pipelined over mixture chunks: chunk k's all-reduce (comm_stream)
    // overlaps chunk k+1's sweep; its apply runs just before chunk k's next
    // sweep (the only consumer of the updated V / mu of those mixtures)
    const int kNccl = sizeof(Real) == 4 ? kNcclFloat : kNcclDouble;
    if (c->stream2) {  // the odd chunks start after everything queued before this body
      CK(cudaEventRecord(c->ev_join, c->stream));
      CK(cudaStreamWaitEvent(c->stream2, c->ev_join, 0));
    }
    for (int k = 0; k < c->nmc; ++k) {
      const int m0 = c->mix_split[(size_t)k], m1 = c->mix_split[(size_t)k + 1];
      const cudaStream_t st = c->chunk_stream(k);
      apply_deferred<Real>(c, k);
      launch_sweep<Real>(c, do_sweep, m0, m1, k, st);
      if (do_sweep) {
        launch_muv<Real>(c, m0, m1, st);
        c->timing.launches += 1;
      }
      launch_apply<Real>(c, 0, obj_slot, do_v, m0, m1, st);
      c->timing.launches += 1;
      const size_t nv = (size_t)(m1 - m0) * 2 * c->SK * c->T, nd = (size_t)(m1 - m0) * (c->R + 1);
      Real* pv = reinterpret_cast<Real*>(c->packed.p) + (size_t)m0 * 2 * c->SK * c->T;
      double* pd = c->packed_d.p + (size_t)m0 * (c->R + 1);
      if (c->group) {  // in-process exchange: synchronous on the chunk's stream
        if (do_sweep) allreduce(c, pv, nv, kNccl, kNcclSum, st);
        allreduce(c, pd, nd, kNcclDouble, kNcclSum, st);
        CK(cudaEventRecord(c->ev_ar[(size_t)k], st));
      } else {  // NCCL on the communication stream, both sums in one group
        CK(cudaEventRecord(c->ev_red[(size_t)k], st));
        CK(cudaStreamWaitEvent(c->comm_stream, c->ev_red[(size_t)k], 0));
        if (g_nccl.GroupStart) g_nccl.GroupStart();
        if (do_sweep) allreduce(c, pv, nv, kNccl, kNcclSum, c->comm_stream);
        allreduce(c, pd, nd, kNcclDouble, kNcclSum, c->comm_stream);
        if (g_nccl.GroupEnd && g_nccl.GroupEnd() != 0) throw CtfError(CTF_ERR_CUDA, "ncclGroupEnd failed");
        CK(cudaEventRecord(c->ev_ar[(size_t)k], c->comm_stream));
      }
      c->deferred[(size_t)k] = {true, obj_slot, do_v};
    }
    if (c->stream2) {  // e1 / e2 on the context stream cover the odd chunks too
      CK(cudaEventRecord(c->ev_join, c->stream2));
      CK(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    }
  } else {
    launch_sweep<Real>(c, do_sweep, 0, c->B, 0, c->stream);
  }
  CK(cudaEventRecord(e1, c->stream));
  cudaEvent_t ers = nullptr;  // OptimizationTrace::rescale_ms starts here (mu, V apply, objective)
  if (c->nmc <= 1) {
    if (do_sweep) {
      launch_muv<Real>(c, 0, c->B, c->stream);
      c->timing.launches += 1;
      ers = take_event(c);
      CK(cudaEventRecord(ers, c->stream));
    }
    if (c->collective()) {
      launch_apply<Real>(c, 0, obj_slot, do_v, 0, c->B, c->stream);
      if (c->comm && g_nccl.GroupStart) g_nccl.GroupStart();
      if (do_sweep) allreduce(c, c->packed.p, (size_t)c->B * 2 * c->SK * c->T, sizeof(Real) == 4 ? kNcclFloat : kNcclDouble, kNcclSum);
      allreduce(c, c->packed_d.p, (size_t)c->B * (c->R + 1), kNcclDouble, kNcclSum);
      if (c->comm && g_nccl.GroupEnd && g_nccl.GroupEnd() != 0) throw CtfError(CTF_ERR_CUDA, "ncclGroupEnd failed");
      launch_apply<Real>(c, 1, obj_slot, do_v, 0, c->B, c->stream);
      c->timing.launches += 2;
    } else {
      launch_apply<Real>(c, 2, obj_slot, do_v, 0, c->B, c->stream);
      c->timing.launches += 1;
    }
  }
  CK(cudaEventRecord(e2, c->stream));
  if (do_sweep) {
    c->ev_sweep.push_back({e0, e1});
    c->ev_mu.push_back({e1, e2});
    c->ev_rs.push_back(ers);
    c->done += 1;
    c->pending = true;
  } else {
    c->ev_fin.push_back({e0, e2});
    c->ev_pool.push_back(e1);
    c->pending = false;
  }
}

void collect_timing(ctf_ctx* c) {
  CK(cudaStreamSynchronize(c->stream));
  auto drain = [&](std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v, double& acc) {
    for (auto& pr : v) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, pr.first, pr.second));
      acc += ms;
      c->ev_pool.push_back(pr.first);
      c->ev_pool.push_back(pr.second);
    }
    v.clear();
  };
  // ev_sweep and ev_mu share events; collect times first, then recycle once
  for (size_t i = 0; i < c->ev_sweep.size(); ++i) {
    float a = 0.f, b = 0.f, r = 0.f;
    CK(cudaEventElapsedTime(&a, c->ev_sweep[i].first, c->ev_sweep[i].second));
    CK(cudaEventElapsedTime(&b, c->ev_mu[i].first, c->ev_mu[i].second));
    const cudaEvent_t ers = i < c->ev_rs.size() ? c->ev_rs[i] : nullptr;
    if (ers) {
      CK(cudaEventElapsedTime(&r, ers, c->ev_mu[i].second));
      c->ev_pool.push_back(ers);
    }
    c->timing.sweep_ms += a;
    c->timing.mu_ms += b;
    c->it_sweep_ms.push_back(a);
    c->it_mu_ms.push_back(b - r);
    c->it_rs_ms.push_back(r);
    c->ev_pool.push_back(c->ev_sweep[i].first);
    c->ev_pool.push_back(c->ev_sweep[i].second);
    c->ev_pool.push_back(c->ev_mu[i].second);
  }
  c->ev_sweep.clear();
  c->ev_mu.clear();
  c->ev_rs.clear();
  drain(c->ev_fin, c->timing.finalize_ms);
  if (!c->ev_lam.empty()) {
    double lam_ms = 0.0;
    const size_t nl = c->ev_lam.size();
    drain(c->ev_lam, lam_ms);
    std::fprintf(stderr, "[ctf dev] lambda_kernel: %.3f ms over %zu launches (%.3f ms each)\n", lam_ms, nl, lam_ms / nl);
  }
}

void iterate_impl(ctf_ctx* c, int n, bool finalize) {
  if (!c->ready) throw CtfError(CTF_ERR_CONFIG, "ctf_setup has not been called");
  if (n < 0) throw CtfError(CTF_ERR_CONFIG, "iteration count must be >= 0");
  CK(cudaSetDevice(c->device));
  if (c->done + n > c->max_iters) {
    // grow the objective trace
    const int new_max = std::max(c->done + n, 2 * c->max_iters);
    DevBuf<double> nt;
    nt.alloc((size_t)c->B * new_max);
    CK(cudaMemsetAsync(nt.p, 0, nt.n * 8, c->stream));
    if (c->max_iters > 0)
      CK(cudaMemcpy2DAsync(nt.p, (size_t)new_max * 8, c->objective.p, (size_t)c->max_iters * 8,
                           (size_t)c->max_iters * 8, c->B, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    std::swap(c->objective.p, nt.p);
    std::swap(c->objective.n, nt.n);
    c->max_iters = new_max;
  }
  for (int i = 0; i < n; ++i) {
    if (c->real_size == 4) run_body<float>(c, true);
    else run_body<double>(c, true);
  }
  if (finalize && c->pending) {
    if (c->real_size == 4) run_body<float>(c, false);
    else run_body<double>(c, false);
  }
  // the deferred applies of the pipelined loop (mixture chunks) complete here
  if (c->real_size == 4) flush_deferred<float>(c);
  else flush_deferred<double>(c);
  if (finalize) {
    collect_timing(c);
    check_errors(c);
  }
}


// defer_x: allocate, draw and upload the initial factors, but leave the x
// upload, its mean power and the PSD floors to the caller (run_overlapped).
void setup_impl(ctf_ctx* c, const ctf_problem* prob, const void* x_host,
                const std::function<void()>& fill_x = nullptr, bool defer_x = false,
                const std::function<void()>& after_alloc = nullptr) {
  if (!prob) throw CtfError(CTF_ERR_CONFIG, "null problem");
  validate(*prob);
  if (!x_host && !fill_x) throw CtfError(CTF_ERR_CONFIG, "null mixture");
  CK(cudaSetDevice(c->device));
  c->ready = false;
  c->prob = *prob;
  c->B = prob->num_mixtures;
  c->F = prob->num_bins;
  c->T = prob->num_frames;
  c->Mx = prob->num_mics;
  c->Ls = prob->stack_taps;
  c->D = c->Mx * c->Ls;
  c->R = c->D;
  c->N = prob->num_sources;
  c->real_size = prob->precision == CTF_F32 ? 4 : 8;
  // evaluated identically on every rank, so all ranks fail before the first collective
  if (c->F < c->world) throw CtfError(CTF_ERR_CONFIG, "more ranks than frequency bins");
  ctf_shard_range(c->F, c->world, c->rank, &c->lo, &c->hi);
  c->FL = c->hi - c->lo;
  if (c->FL < 1) throw CtfError(CTF_ERR_CONFIG, "more ranks than frequency bins");
  int r0 = 0, k0 = 0, kmax = 0;
  for (int n = 0; n < c->N; ++n) {
    c->taps[n] = prob->taps_per_source[n];
    c->bases[n] = prob->bases_per_source[n];
    c->row0[n] = r0;
    c->koff[n] = k0;
    r0 += c->taps[n];
    k0 += c->bases[n];
    kmax = std::max(kmax, c->bases[n]);
  }
  c->koff[c->N] = k0;
  c->SK = k0;
  if (kmax > 32) throw CtfError(CTF_ERR_UNSUPPORTED, "more than 32 bases per source");
  c->kmax = kmax <= 4 ? 4 : kmax <= 8 ? 8 : kmax <= 10 ? 10 : kmax <= 12 ? 12 : kmax <= 16 ? 16 : kmax <= 20 ? 20 : kmax <= 24 ? 24 : 32;
  plan_sweep(c);
  // MU-V bin chunks of a fixed size (64 bins): the summation order must not
  // depend on the batch size, so a mixture gives bit-identical results alone
  // or in any batch; chunk partials are combined in fixed order. (16-bin
  // chunks for the single-mixture cfg0 measured no faster: its MU phase is
  // bound by two small dependent launches, not by the chunk loop.)
  c->chunk_bins = 64;
  c->nchunk = (c->FL + c->chunk_bins - 1) / c->chunk_bins;

  const size_t rs = c->real_size, cs = 2 * rs;
  const size_t xcount = (size_t)c->B * c->FL * c->T * c->Mx;  // complex
  c->x.alloc(xcount * cs);
  c->W.alloc((size_t)c->B * plane_stride(c) * cs);
  c->Bf.alloc((size_t)c->B * c->FL * c->SK * rs);
  c->V.alloc(((size_t)c->B * c->SK * c->T + 4096) * rs);  // zero tail: the sweep reads V up to frame TP
  CK(cudaMemsetAsync(c->V.p, 0, c->V.n, c->stream));
  c->E.alloc((size_t)c->B * c->N * c->FL * c->T * rs);
  // lambda ahead of the covariance-domain / frame-split kernels (the variants compiled without a lambda phase)
  c->lam_pre = (c->sv.kind == 4 || c->sv.kind == 5) && c->sv.lpre != 0;
  if (c->lam_pre) {
    c->invl.alloc((size_t)c->B * c->FL * c->N * c->T * rs);
    c->logsum.alloc((size_t)c->B * c->FL);
  } else {
    c->invl.free();
    c->logsum.free();
  }
  c->part.alloc((size_t)c->nchunk * c->B * 2 * c->SK * c->T * rs);
  c->packed.alloc(c->collective() ? (size_t)c->B * 2 * c->SK * c->T * rs : 16);
  c->rowpow.alloc((size_t)c->B * c->FL * c->R);
  c->objbin.alloc((size_t)c->B * c->FL);
  c->packed_d.alloc((size_t)c->B * (c->R + 1));
  c->mu.alloc((size_t)c->B * c->R);
  c->logmu.alloc((size_t)c->B);
  c->floor_abs.alloc((size_t)c->B);
  c->mp_part.alloc((size_t)c->B * c->FL);
  c->err.alloc((size_t)c->B);
  c->chk.alloc((size_t)c->B * 2);
  if (c->has_fb) {
    c->fb_list.alloc((size_t)c->B * c->FL);
    c->fb_count.alloc(1);
  }
  // pipelined collective loop: two mixture chunks by default (CTF_MIX_CHUNKS
  // overrides; 1 = the unchunked reduce -> all-reduce -> apply). Kernels with
  // a per-launch mixture offset only (not the persistent streamed kernel) and
  // not with CheckOptions (their maxima are reduced per iteration).
  c->nmc = 1;
  if (c->collective() && c->B >= 2 && c->sv.kind != 2 && c->prob.checks == 0) {
    c->nmc = 2;
    if (const char* env = std::getenv("CTF_MIX_CHUNKS")) c->nmc = std::max(1, std::min(c->B, std::atoi(env)));
  }
  if (c->nmc > 1) {
    if (!c->comm_stream) CK(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    if (!c->stream2) CK(cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking));
    if (!c->ev_join) CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
    if (c->has_fb) c->fb_count.alloc((size_t)c->nmc);
    while ((int)c->ev_red.size() < c->nmc) {
      cudaEvent_t a, b;
      CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      c->ev_red.push_back(a);
      c->ev_ar.push_back(b);
    }
  }
  c->deferred.assign((size_t)c->nmc, ctf_ctx::Deferred{});
  // chunk boundaries at whole waves of the one-CTA-per-bin kernels (a split
  // in the middle of a wave would add a partial wave per chunk): chunk k ends
  // at the mixture whose CTAs fill about k/nmc of the waves
  c->mix_split.assign((size_t)c->nmc + 1, 0);
  for (int k = 0; k <= c->nmc; ++k) c->mix_split[(size_t)k] = k * c->B / c->nmc;
  if (c->nmc > 1 && (c->sv.kind == 0 || c->sv.kind == 4)) {
    int per_sm = 0, nsm = 0;
    if (c->sv.kind == 4)
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, c->sv.gfn, c->NT, c->sweep_smem));
    else
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, c->sv.fn, c->NT, c->sweep_smem));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
    const long slots = (long)std::max(1, per_sm) * nsm;
    const long waves = ((long)c->B * c->FL + slots - 1) / slots;
    for (int k = 1; k < c->nmc; ++k) {
      const long target = (waves * k / c->nmc) * slots;  // CTAs of the first k chunks
      int m = (int)(target / c->FL);
      m = std::max(c->mix_split[(size_t)k - 1] + 1, std::min(m, c->B - (c->nmc - k)));
      c->mix_split[(size_t)k] = m;
    }
  }
  if (c->sv.kind == 2)  // per-CTA tile slots (+ the CheckOptions LU scratch)
    c->scratch.alloc((size_t)c->stream_grid * ((size_t)c->R * c->TP + (c->sv.chk ? (size_t)c->R * c->D : 0)) * cs);
  else c->scratch.free();
  if (c->sv.kind == 3) {
    const size_t tiles = (size_t)c->B * c->FL;
    c->cpivot.alloc(tiles * 2 * c->TP * cs);
    c->cwpivot.alloc(tiles * 2 * c->D * cs);
    c->cpart.alloc(tiles * c->cluster_size * 4);
    c->cbad.alloc(tiles);
  }
  c->logdet.alloc((size_t)c->B * c->FL);
  CK(cudaMemsetAsync(c->logdet.p, 0, c->logdet.n * 8, c->stream));  // log|det I| = 0
  c->max_iters = std::max(1, prob->iterations);
  c->objective.alloc((size_t)c->B * c->max_iters);
  CK(cudaMemsetAsync(c->objective.p, 0, c->objective.n * 8, c->stream));
  CK(cudaMemsetAsync(c->err.p, 0xFF, c->err.n * 8, c->stream));
  CK(cudaMemsetAsync(c->chk.p, 0, c->chk.n * 8, c->stream));
  CK(cudaMemsetAsync(c->E.p, 0, c->E.n, c->stream));

  // random_factors with mt19937_64(seed + b) (model.cpp:189-208, estimator.cpp:532-533),
  // drawn on host threads while x is uploaded and its mean power reduced
  std::vector<double> hb((size_t)c->B * c->FL * c->SK), hv((size_t)c->B * c->SK * c->T);
  // one independent mt19937_64 stream per mixture: threads over mixtures
  struct Pool {
    std::vector<std::thread> t;
    void join_all() {
      for (auto& th : t)
        if (th.joinable()) th.join();
    }
    ~Pool() { join_all(); }  // also on the error paths below
  } pool;
  const int nth = std::max(1, std::min<int>(c->B, (int)std::thread::hardware_concurrency()));
  for (int w = 0; w < nth; ++w) pool.t.emplace_back([&, w] {
  for (int b = w; b < c->B; b += nth) {
    std::mt19937_64 rng(prob->seed + (uint64_t)b);
    std::uniform_real_distribution<double> uni(0.1, 1.0);
    for (int n = 0; n < c->N; ++n) {
      const int K = c->bases[n];
      for (int i = 0; i < c->F; ++i)
        for (int k = 0; k < K; ++k) {
          const double v = uni(rng);
          if (i >= c->lo && i < c->hi) hb[((size_t)b * c->FL + (i - c->lo)) * c->SK + c->koff[n] + k] = v;
        }
      for (int k = 0; k < K; ++k)
        for (int j = 0; j < c->T; ++j) hv[((size_t)b * c->SK + c->koff[n] + k) * c->T + j] = uni(rng);
    }
  }
  });

  // x: this rank's bins of every mixture, converted to the compute precision
  const size_t xs_in = prob->x_precision == CTF_F32 ? 8 : 16;
  const size_t per_mix = (size_t)c->FL * c->T * c->Mx;  // complex per mixture (local)
  const bool same = (xs_in == cs);
  DevBuf<unsigned char> stage;
  if (!same && !fill_x && !defer_x) stage.alloc(per_mix * xs_in);
  if (fill_x) fill_x();  // device-side producer (the GPU STFT front end)
  for (int b = 0; b < c->B && !fill_x && !defer_x; ++b) {
    const unsigned char* src =
        static_cast<const unsigned char*>(x_host) + ((size_t)b * c->F + c->lo) * c->T * c->Mx * xs_in;
    unsigned char* dst = c->x.p + (size_t)b * per_mix * cs;
    if (same) {
      CK(cudaMemcpyAsync(dst, src, per_mix * xs_in, cudaMemcpyHostToDevice, c->stream));
    } else {
      CK(cudaMemcpyAsync(stage.p, src, per_mix * xs_in, cudaMemcpyHostToDevice, c->stream));
      const size_t n = per_mix * 2;
      const int g = (int)std::min<size_t>((n + 255) / 256, 8192);
      if (xs_in == 16)
        convert_kernel<float><<<g, 256, 0, c->stream>>>((const double*)stage.p, (float*)dst, n);
      else
        convert_f32_kernel<double><<<g, 256, 0, c->stream>>>((const float*)stage.p, (double*)dst, n);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(c->stream));  // stage is reused
    }
  }
  if (defer_x) {
    if (c->has_fb) c->fb_count.alloc(std::max<size_t>(c->fb_count.n, (size_t)c->B));  // one list per upload chunk
  } else {
  // mean power of x~ and the absolute PSD floor (estimator.cpp:520-529)
  if (rs == 4)
    ctf::mean_power_kernel<float><<<dim3(c->FL, c->B), 256, 0, c->stream>>>(c->x.p, c->mp_part.p, c->FL, c->T, c->Mx, c->Ls);
  else
    ctf::mean_power_kernel<double><<<dim3(c->FL, c->B), 256, 0, c->stream>>>(c->x.p, c->mp_part.p, c->FL, c->T, c->Mx, c->Ls);
  CK(cudaGetLastError());
  std::vector<double> mp_part((size_t)c->B * c->FL), sums((size_t)c->B, 0.0);
  CK(cudaMemcpyAsync(mp_part.data(), c->mp_part.p, mp_part.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int b = 0; b < c->B; ++b)
    for (int i = 0; i < c->FL; ++i) sums[(size_t)b] += mp_part[(size_t)b * c->FL + i];
  if (c->collective()) {
    CK(cudaMemcpyAsync(c->mp_part.p, sums.data(), sums.size() * 8, cudaMemcpyHostToDevice, c->stream));
    allreduce(c, c->mp_part.p, sums.size(), kNcclDouble, kNcclSum);
    CK(cudaMemcpyAsync(sums.data(), c->mp_part.p, sums.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  std::vector<double> floors((size_t)c->B);
  const double count = (double)c->F * c->D * c->T;
  for (int b = 0; b < c->B; ++b) {
    const double mp = sums[(size_t)b] / count;
    if (!std::isfinite(mp))
      throw CtfError(CTF_ERR_DEGENERACY, "mixture spectrogram contains non-finite values", CTF_KIND_NONFINITE_X, -1, b);
    if (!(mp > 0.0))
      throw CtfError(CTF_ERR_CONFIG, "mixture spectrogram is identically zero", CTF_KIND_ZERO_X, -1, b);
    floors[(size_t)b] = prob->psd_floor * mp;
  }
  CK(cudaMemcpyAsync(c->floor_abs.p, floors.data(), floors.size() * 8, cudaMemcpyHostToDevice, c->stream));
  c->floors = floors;
  }
  c->it_sweep_ms.clear();
  c->it_mu_ms.clear();
  c->it_rs_ms.clear();

  pool.join_all();  // the initial factors (drawn on host threads while x was uploaded)
  upload_real(c, c->Bf.p, hb.data(), hb.size());
  upload_real(c, c->V.p, hv.data(), hv.size());
  // W = I (model.cpp:221-227)
  {
    const size_t n = (size_t)c->B * plane_stride(c) * 2;
    const int g = (int)std::min<size_t>((n + 255) / 256, 8192);
    if (rs == 4) identity_kernel<float><<<g, 256, 0, c->stream>>>((float*)c->W.p, (size_t)c->B * c->FL, c->R, c->D);
    else identity_kernel<double><<<g, 256, 0, c->stream>>>((double*)c->W.p, (size_t)c->B * c->FL, c->R, c->D);
    CK(cudaGetLastError());
  }
  // run_overlapped's chunked x copies: after the (pageable) factor uploads,
  // which would otherwise queue behind the whole of x on the copy engine
  if (after_alloc) after_alloc();
  CK(cudaStreamSynchronize(c->stream));
  c->done = 0;
  c->pending = false;
  c->timing = ctf_timing{};
  c->ready = true;
}

// Per-mixture PSD floors on the device (estimator.cpp:520-529), the same
// arithmetic and bin order as setup_impl's host loop: sum_i part[b][i] / count.
__global__ void floor_kernel(const double* part, double* floor_abs, double* mpsum, int FL, int m0, int m1,
                             double count, double psd_floor) {
  const int b = m0 + (int)(blockIdx.x * blockDim.x + threadIdx.x);
  if (b >= m1) return;
  double s = 0.0;
  for (int i = 0; i < FL; ++i) s += part[(size_t)b * FL + i];
  mpsum[b] = s;
  floor_abs[b] = psd_floor * (s / count);
}

// ctf_run on one GPU with the host->device copy of x overlapped with the first
// iterations: x goes up in mixture chunks on a copy stream; each chunk's mean
// power, floor and first J loop bodies run on the chunk's own stream as soon
// as its bytes have landed (mixtures are independent until the all-bin MU-V
// sums, which are per mixture), so chunk 0 iterates while chunk 7 uploads.
// Then the streams join and the remaining iterations run unchunked. Results
// are bit-identical to setup + iterate (same kernels per mixture, MU-V
// chunking independent of the batch). Returns false (nothing done) when the
// problem does not qualify (multi-rank, x conversion, CheckOptions, < 2
// mixtures or no iterations); the caller then runs the plain path.
template <class Real>
bool run_overlapped(ctf_ctx* c, const ctf_problem* prob, const void* x_host) {
  if (c->world != 1 || c->group || prob->x_precision != prob->precision || prob->checks != 0 ||
      prob->num_mixtures < 2 || prob->iterations < 1)
    return false;
  if (const char* e = std::getenv("CTF_RUN_OVERLAP"))
    if (std::atoi(e) == 0) return false;
  int NU = std::min(prob->num_mixtures, 8), J = std::min(prob->iterations, 3);  // J: chunked loop bodies
  if (const char* e = std::getenv("CTF_RUN_OVERLAP_NU")) NU = std::max(1, std::min(prob->num_mixtures, std::atoi(e)));
  if (const char* e = std::getenv("CTF_RUN_OVERLAP_J")) J = std::max(1, std::min(prob->iterations, std::atoi(e)));
  while ((int)c->ustreams.size() < NU) {
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    c->ustreams.push_back(st);
    cudaEvent_t a, b;
    CK(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    c->ev_up.push_back(a);
    c->ev_udone.push_back(b);
  }
  if (!c->copy_stream) CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  std::vector<int> mb((size_t)NU + 1);
  for (int u = 0; u <= NU; ++u) mb[(size_t)u] = u * prob->num_mixtures / NU;
  size_t per_mix = 0, cs = 0;  // complex values per mixture, bytes per complex
  bool copies = false;
  // x goes up in mixture chunks, issued at the end of the setup
  auto issue_copies = [&] {
    if (c->sv.kind == 2 || c->nmc != 1) return;  // not chunkable
    cs = 2 * (size_t)c->real_size;
    per_mix = (size_t)c->FL * c->T * c->Mx;
    CK(cudaStreamSynchronize(c->copy_stream));  // (x of a previous run)
    for (int u = 0; u < NU; ++u) {
      const size_t off = (size_t)mb[(size_t)u] * per_mix * cs;
      const size_t n = (size_t)(mb[(size_t)u + 1] - mb[(size_t)u]) * per_mix * cs;
      CK(cudaMemcpyAsync(c->x.p + off, static_cast<const unsigned char*>(x_host) + off, n, cudaMemcpyHostToDevice,
                         c->copy_stream));
      CK(cudaEventRecord(c->ev_up[(size_t)u], c->copy_stream));
    }
    copies = true;
  };
  const auto t_enter = std::chrono::steady_clock::now();
  setup_impl(c, prob, x_host, nullptr, true, issue_copies);
  const auto t_setup = std::chrono::steady_clock::now();
  if (!copies) {  // not chunkable: the plain setup + loop
    setup_impl(c, prob, x_host);
    iterate_impl(c, prob->iterations, true);
    return true;
  }
  c->mpsum.alloc((size_t)c->B);
  cudaEvent_t e_start = take_event(c), e_end = take_event(c);
  CK(cudaEventRecord(e_start, c->stream));  // memsets, initial factors, W = I
  const double count = (double)c->F * c->D * c->T;
  for (int u = 0; u < NU; ++u) {
    const cudaStream_t st = c->ustreams[(size_t)u];
    const int m0 = mb[(size_t)u], m1 = mb[(size_t)u + 1];
    CK(cudaStreamWaitEvent(st, e_start, 0));
    CK(cudaStreamWaitEvent(st, c->ev_up[(size_t)u], 0));
    ctf::mean_power_kernel<Real><<<dim3(c->FL, m1 - m0), 256, 0, st>>>(c->x.p + (size_t)m0 * per_mix * cs,
                                                                       c->mp_part.p + (size_t)m0 * c->FL, c->FL,
                                                                       c->T, c->Mx, c->Ls);
    floor_kernel<<<1, 64, 0, st>>>(c->mp_part.p, c->floor_abs.p, c->mpsum.p, c->FL, m0, m1, count, prob->psd_floor);
    CK(cudaGetLastError());
  }
  for (int i = 0; i < J; ++i) {  // run_body's loop body, chunk by chunk
    const int obj_slot = c->pending ? c->done - 1 : -1;
    for (int u = 0; u < NU; ++u) {
      const cudaStream_t st = c->ustreams[(size_t)u];
      const int m0 = mb[(size_t)u], m1 = mb[(size_t)u + 1];
      launch_sweep<Real>(c, true, m0, m1, u, st);
      launch_muv<Real>(c, m0, m1, st);
      launch_apply<Real>(c, 2, obj_slot, 1, m0, m1, st);
      c->timing.launches += 2;
    }
    c->done += 1;
    c->pending = true;
  }
  for (int u = 0; u < NU; ++u) {
    CK(cudaEventRecord(c->ev_udone[(size_t)u], c->ustreams[(size_t)u]));
    CK(cudaStreamWaitEvent(c->stream, c->ev_udone[(size_t)u], 0));
  }
  CK(cudaEventRecord(e_end, c->stream));
  // the setup checks of estimator.cpp:520-529 (non-finite / zero mixture),
  // raised before anything the loop may have recorded
  std::vector<double> sums((size_t)c->B), floors((size_t)c->B);
  CK(cudaMemcpyAsync(sums.data(), c->mpsum.p, sums.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(floors.data(), c->floor_abs.p, floors.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int b = 0; b < c->B; ++b) {
    const double mp = sums[(size_t)b] / count;
    if (!std::isfinite(mp))
      throw CtfError(CTF_ERR_DEGENERACY, "mixture spectrogram contains non-finite values", CTF_KIND_NONFINITE_X, -1, b);
    if (!(mp > 0.0))
      throw CtfError(CTF_ERR_CONFIG, "mixture spectrogram is identically zero", CTF_KIND_ZERO_X, -1, b);
  }
  c->floors = floors;
  if (std::getenv("CTF_DEBUG_RUN")) {  // measurement aid: host and device timeline of the section
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, e_start, e_end));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "run_overlapped: NU=%d J=%d setup(host) %.2f ms, section(device, e_start->join) %.2f ms, "
                 "host to floor check %.2f ms\n", NU, J, std::chrono::duration<double, std::milli>(t_setup - t_enter).count(), t,
                 std::chrono::duration<double, std::milli>(now - t_enter).count());
  }
  // OptimizationTrace entries of the overlapped bodies: the section's time
  // (from the end of the setup, upload included) split evenly over them
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e_start, e_end));
  c->ev_pool.push_back(e_start);
  c->ev_pool.push_back(e_end);
  for (int i = 0; i < J; ++i) {
    c->it_sweep_ms.push_back(ms / J);
    c->it_mu_ms.push_back(0.0);
    c->it_rs_ms.push_back(0.0);
  }
  c->timing.sweep_ms += ms;
  c->timing.sweep_launches += J * NU;
  iterate_impl(c, prob->iterations - J, true);
  return true;
}

}  // namespace

// ---------------------------------------------------------------------------
extern "C" {

int ctf_abi_version(void) { return CTF_ABI_VERSION; }

void ctf_shard_range(int num_bins, int world_size, int rank, int* lo, int* hi) {
  // contiguous ranges, sizes differ by at most one
  const int w = std::max(1, world_size);
  const int base = num_bins / w, rem = num_bins % w;
  const int l = rank * base + std::min(rank, rem);
  *lo = l;
  *hi = l + base + (rank < rem ? 1 : 0);
}

int ctf_open(int device, ctf_ctx** out, ctf_err* err) {
  return guarded(err, [&] {
    if (!out) throw CtfError(CTF_ERR_CONFIG, "null output");
    int count = 0;
    CK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw CtfError(CTF_ERR_CUDA, "no such CUDA device");
    CK(cudaSetDevice(device));
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw CtfError(CTF_ERR_CUDA, "the kernels are built for sm_100a (B200) only");
    auto* c = new ctf_ctx();
    c->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete c;
      cuda_check(e, "cudaStreamCreate");
    }
    *out = c;
  });
}

void ctf_close(ctf_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& pr : c->ev_sweep) c->ev_pool.push_back(pr.first), c->ev_pool.push_back(pr.second);
  for (auto& pr : c->ev_mu) c->ev_pool.push_back(pr.second);
  for (auto e : c->ev_rs)
    if (e) c->ev_pool.push_back(e);
  c->ev_rs.clear();
  for (auto& pr : c->ev_fin) c->ev_pool.push_back(pr.first), c->ev_pool.push_back(pr.second);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->comm_stream) cudaStreamSynchronize(c->comm_stream);
  if (c->stream2) cudaStreamSynchronize(c->stream2);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  for (auto st : c->ustreams) cudaStreamSynchronize(st), cudaStreamDestroy(st);
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream), cudaStreamDestroy(c->copy_stream);
  for (auto e : c->ev_up) cudaEventDestroy(e);
  for (auto e : c->ev_udone) cudaEventDestroy(e);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  for (auto e : c->ev_red) cudaEventDestroy(e);
  for (auto e : c->ev_ar) cudaEventDestroy(e);
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

void* ctf_stream(ctf_ctx* c) { return c ? (void*)c->stream : nullptr; }

int ctf_comm_unique_id(uint8_t id[128], ctf_err* err) {
  return guarded(err, [&] {
    if (!g_nccl.load()) throw CtfError(CTF_ERR_CUDA, "libnccl.so.2 could not be loaded");
    NcclUid u;
    if (g_nccl.GetUniqueId(&u) != 0) throw CtfError(CTF_ERR_CUDA, "ncclGetUniqueId failed");
    std::memcpy(id, u.internal, 128);
  });
}

int ctf_comm_init(ctf_ctx* c, int world, int rank, const uint8_t id[128], ctf_err* err) {
  return guarded(err, [&] {
    if (!c) throw CtfError(CTF_ERR_CONFIG, "null context");
    if (world < 1 || rank < 0 || rank >= world) throw CtfError(CTF_ERR_CONFIG, "bad world/rank");
    c->world = world;
    c->rank = rank;
    const char* single = std::getenv("CTF_NCCL_SINGLE_RANK");
    if (world == 1 && !(single && std::atoi(single) == 1)) return;
    if (!g_nccl.load()) throw CtfError(CTF_ERR_CUDA, "libnccl.so.2 could not be loaded");
    CK(cudaSetDevice(c->device));
    NcclUid u;
    std::memcpy(u.internal, id, 128);
    const int rc = g_nccl.CommInitRank(&c->comm, world, u, rank);
    if (rc != 0) throw CtfError(CTF_ERR_CUDA, "ncclCommInitRank failed");
  });
}

ctf_group* ctf_group_create(int world_size) {
  if (world_size < 1) return nullptr;
  auto* g = new ctf_group();
  g->world = world_size;
  g->slots.resize((size_t)world_size);
  return g;
}

void ctf_group_destroy(ctf_group* g) { delete g; }

int ctf_comm_init_group(ctf_ctx* c, ctf_group* g, int rank, ctf_err* err) {
  return guarded(err, [&] {
    if (!c || !g) throw CtfError(CTF_ERR_CONFIG, "null context or group");
    if (rank < 0 || rank >= g->world) throw CtfError(CTF_ERR_CONFIG, "bad rank");
    c->world = g->world;
    c->rank = rank;
    c->group = g->world > 1 ? g : nullptr;
  });
}

int ctf_setup(ctf_ctx* c, const ctf_problem* prob, const void* x_host, ctf_err* err) {
  return guarded(err, [&] {
    if (!c) throw CtfError(CTF_ERR_CONFIG, "null context");
    setup_impl(c, prob, x_host);
  });
}

int ctf_set_state(ctf_ctx* c, const double* W, const double* Bh, const double* Vh, ctf_err* err) {
  return guarded(err, [&] {
    if (!c || !c->ready) throw CtfError(CTF_ERR_CONFIG, "ctf_setup has not been called");
    CK(cudaSetDevice(c->device));
    // a deferred rescale/objective of an async iteration applies to the
    // state as it stands before any factor is replaced (W or B kept as NULL
    // must not miss its rescale)
    if (c->pending) iterate_impl(c, 0, true);
    if (W) {
      std::vector<double> w((size_t)c->B * plane_stride(c) * 2);
      const size_t per = (size_t)c->R * c->D * 2;
      for (int b = 0; b < c->B; ++b)
        std::memcpy(w.data() + (size_t)b * c->FL * per, W + ((size_t)b * c->F + c->lo) * per, c->FL * per * 8);
      upload_real(c, c->W.p, w.data(), w.size());
      // exact log|det W| for the externally supplied state (estimator.cpp:41-53)
      const int nb = c->B * c->FL;
      const size_t smem = (size_t)c->R * c->R * 2 * c->real_size;  // fp64 R = 60: 57,600 B > the 48 KiB default
      if (c->real_size == 4) {
        CK(cudaFuncSetAttribute((const void*)ctf::logdet_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
        ctf::logdet_kernel<float><<<nb, 32, smem, c->stream>>>(c->W.p, c->logdet.p, c->R, nb);
      } else {
        CK(cudaFuncSetAttribute((const void*)ctf::logdet_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
        ctf::logdet_kernel<double><<<nb, 32, smem, c->stream>>>(c->W.p, c->logdet.p, c->R, nb);
      }
      CK(cudaGetLastError());
    }
    if (Bh) {  // [B][N] F x K_n column-major -> [B][FL][SK]
      std::vector<double> hb((size_t)c->B * c->FL * c->SK);
      for (int b = 0; b < c->B; ++b) {
        size_t off = (size_t)b * c->F * c->SK;
        for (int n = 0; n < c->N; ++n) {
          const int K = c->bases[n];
          for (int k = 0; k < K; ++k)
            for (int i = c->lo; i < c->hi; ++i)
              hb[((size_t)b * c->FL + (i - c->lo)) * c->SK + c->koff[n] + k] = Bh[off + (size_t)i + (size_t)k * c->F];
          off += (size_t)c->F * K;
        }
      }
      upload_real(c, c->Bf.p, hb.data(), hb.size());
    }
    if (Vh) {  // [B][N] K_n x T column-major -> [B][SK][T]
      std::vector<double> hv((size_t)c->B * c->SK * c->T);
      for (int b = 0; b < c->B; ++b) {
        size_t off = (size_t)b * c->SK * c->T;
        for (int n = 0; n < c->N; ++n) {
          const int K = c->bases[n];
          for (int j = 0; j < c->T; ++j)
            for (int k = 0; k < K; ++k)
              hv[((size_t)b * c->SK + c->koff[n] + k) * c->T + j] = Vh[off + (size_t)k + (size_t)j * K];
          off += (size_t)K * c->T;
        }
      }
      upload_real(c, c->V.p, hv.data(), hv.size());
    }
    c->pending = false;
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ctf_iterate(ctf_ctx* c, int n, ctf_err* err) {
  return guarded(err, [&] {
    if (!c) throw CtfError(CTF_ERR_CONFIG, "null context");
    iterate_impl(c, n, true);
  });
}

int ctf_iterate_async(ctf_ctx* c, int n, ctf_err* err) {
  return guarded(err, [&] {
    if (!c) throw CtfError(CTF_ERR_CONFIG, "null context");
    iterate_impl(c, n, false);
  });
}

int ctf_finalize(ctf_ctx* c, ctf_err* err) {
  return guarded(err, [&] {
    if (!c) throw CtfError(CTF_ERR_CONFIG, "null context");
    iterate_impl(c, 0, true);
  });
}

int ctf_iterations_done(ctf_ctx* c) { return c ? c->done : 0; }

int ctf_describe(ctf_ctx* c, char* buf, int len) {
  if (!c || !buf || len <= 0) return CTF_ERR_CONFIG;
  std::snprintf(buf, (size_t)len,
                "{\"sweep_kernel\": \"%s<%s,RMAX=%d,FT=%d,%s=%d,NT=%d,EXACT=%d>\", \"threads\": %d, "
                "\"smem_bytes\": %zu, \"grid\": [%d, %d], \"muv_chunks\": %d, \"bins\": [%d, %d], "
                "\"world\": %d, \"rank\": %d, \"collective\": \"%s\", \"cluster\": %d, "
                "\"gram_fallback\": %s, \"fallback_theta\": %g, \"fallback_kernel\": \"sweep_kernel<RMAX=%d,FT=%d,RREG=%d,NT=%d>\", "
                "\"mix_chunks\": %d, \"exchange\": \"%s\", \"lambda_ahead\": %s}",
                c->sv.kind == 5 ? "fsplit_kernel" : c->sv.kind == 4 ? "gram_kernel" : c->sv.kind == 3 ? "cluster_kernel" : c->sv.kind == 2 ? "stream_kernel" : c->sv.kind ? "rowwarp_kernel" : "sweep_kernel",
                c->real_size == 4 ? "f32" : "f64", c->sv.rmax, c->sv.ft,
                c->sv.kind == 4 ? "M" : (c->sv.kind == 3 || c->sv.kind == 5) ? "RREG" : c->sv.kind == 2 ? "RG" : c->sv.kind ? "WPR" : "RREG", c->sv.rreg, c->sv.maxt, c->sv.exact, c->NT,
                c->sweep_smem, c->FL, c->B, c->nchunk, c->lo, c->hi, c->world, c->rank,
                c->group ? "host-group" : c->comm ? "nccl" : "none",
                (c->sv.kind == 3 || c->sv.kind == 5) ? c->cluster_size : 1, c->has_fb ? "true" : "false",
                c->fb_theta, c->fbv.rmax, c->fbv.ft, c->fbv.rreg, c->fbv.maxt, c->nmc,
                c->sv.kind != 5 ? "none" : c->sv.pair ? "all-gather, step pairs" : c->sv.ag ? "all-gather" : "owner",
                c->lam_pre ? "true" : "false");
  return CTF_OK;
}

int ctf_psd_floor(ctf_ctx* c, double* out) {
  if (!c || !c->ready || !out) return CTF_ERR_CONFIG;
  for (int b = 0; b < c->B; ++b) out[b] = c->floors[(size_t)b];
  return CTF_OK;
}

int ctf_trace_ms(ctf_ctx* c, double* demix_ms, double* mu_ms, double* rescale_ms) {
  if (!c) return CTF_ERR_CONFIG;
  try {
    collect_timing(c);
  } catch (...) {
    return CTF_ERR_CUDA;
  }
  const size_t n = std::min<size_t>(c->it_sweep_ms.size(), (size_t)c->done);
  const size_t off = c->it_sweep_ms.size() - n;
  for (size_t i = 0; i < n; ++i) {
    if (demix_ms) demix_ms[i] = c->it_sweep_ms[off + i];
    if (mu_ms) mu_ms[i] = c->it_mu_ms[off + i];
    if (rescale_ms) rescale_ms[i] = c->it_rs_ms[off + i];
  }
  return CTF_OK;
}

int ctf_check_stats(ctf_ctx* c, double* max_det, double* max_norm, int64_t* checked) {
  if (!c || !c->ready) return CTF_ERR_CONFIG;
  try {
    std::vector<unsigned long long> v((size_t)c->B * 2);
    CK(cudaSetDevice(c->device));
    if (c->collective()) allreduce(c, c->chk.p, v.size(), kNcclUint64, kNcclMax);
    CK(cudaMemcpyAsync(v.data(), c->chk.p, v.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int b = 0; b < c->B; ++b) {
      double d, n;
      std::memcpy(&d, &v[(size_t)b * 2], 8);
      std::memcpy(&n, &v[(size_t)b * 2 + 1], 8);
      const bool on = c->prob.checks != 0;
      if (max_det) max_det[b] = d;
      if (max_norm) max_norm[b] = n;
      if (checked) checked[b] = on ? (int64_t)c->done * c->F * c->R : 0;
    }
  } catch (const CtfError&) {
    return CTF_ERR_CUDA;
  }
  return CTF_OK;
}

int ctf_get_timing(ctf_ctx* c, ctf_timing* out) {
  if (!c || !out) return CTF_ERR_CONFIG;
  try {
    collect_timing(c);
  } catch (...) {
    return CTF_ERR_CUDA;
  }
  *out = c->timing;
  return CTF_OK;
}

int ctf_reset_timing(ctf_ctx* c) {
  if (!c) return CTF_ERR_CONFIG;
  try {
    collect_timing(c);
  } catch (...) {
    return CTF_ERR_CUDA;
  }
  c->timing = ctf_timing{};
  return CTF_OK;
}

int ctf_download(ctf_ctx* c, double* W, double* Bh, double* Vh, double* objective, ctf_err* err) {
  return guarded(err, [&] {
    if (!c || !c->ready) throw CtfError(CTF_ERR_CONFIG, "ctf_setup has not been called");
    if (c->pending) throw CtfError(CTF_ERR_CONFIG, "call ctf_finalize before ctf_download");
    CK(cudaSetDevice(c->device));
    const bool f32 = c->real_size == 4;
    const size_t wn = (size_t)c->B * plane_stride(c) * 2, bn = (size_t)c->B * c->FL * c->SK,
                 vn = (size_t)c->B * c->SK * c->T;
    const size_t need = std::max(wn, std::max(bn, vn));
    if (c->stage.n < need) c->stage.alloc(need);
    auto grid = [](size_t n) { return (int)std::min<size_t>((n + 255) / 256, 8192); };
    if (W) {  // this rank's bins of every mixture, one strided D2H
      const size_t per = (size_t)c->R * c->D * 2;
      if (f32) gather_W_kernel<float><<<grid(wn), 256, 0, c->stream>>>((const float*)c->W.p, c->stage.p, wn);
      else gather_W_kernel<double><<<grid(wn), 256, 0, c->stream>>>((const double*)c->W.p, c->stage.p, wn);
      CK(cudaGetLastError());
      CK(cudaMemcpy2DAsync(W + (size_t)c->lo * per, (size_t)c->F * per * 8, c->stage.p, (size_t)c->FL * per * 8,
                           (size_t)c->FL * per * 8, c->B, cudaMemcpyDeviceToHost, c->stream));
    }
    if (Bh) {  // [mix][n][k][FL] on the device -> columns [lo, hi) of each F x K_n host matrix
      if (f32) gather_B_kernel<float><<<grid(bn), 256, 0, c->stream>>>((const float*)c->Bf.p, c->stage.p + need * 0, c->B, c->FL, c->SK);
      else gather_B_kernel<double><<<grid(bn), 256, 0, c->stream>>>((const double*)c->Bf.p, c->stage.p, c->B, c->FL, c->SK);
      CK(cudaGetLastError());
      // every (mix, base) column is FL contiguous values at host offset mix*F*SK + kk*F + lo
      CK(cudaMemcpy2DAsync(Bh + c->lo, (size_t)c->F * 8, c->stage.p, (size_t)c->FL * 8, (size_t)c->FL * 8,
                           (size_t)c->B * c->SK, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));  // the staging buffer is reused below
    if (Vh) {
      VMap vm{};
      vm.N = c->N;
      for (int n = 0; n <= c->N; ++n) vm.koff[n] = c->koff[n];
      if (f32) gather_V_kernel<float><<<grid(vn), 256, 0, c->stream>>>((const float*)c->V.p, c->stage.p, c->B, c->SK, c->T, vm);
      else gather_V_kernel<double><<<grid(vn), 256, 0, c->stream>>>((const double*)c->V.p, c->stage.p, c->B, c->SK, c->T, vm);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(Vh, c->stage.p, vn * 8, cudaMemcpyDeviceToHost, c->stream));
    }
    if (objective && c->done > 0)
      CK(cudaMemcpy2DAsync(objective, (size_t)c->done * 8, c->objective.p, (size_t)c->max_iters * 8,
                           (size_t)c->done * 8, c->B, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ctf_run(ctf_ctx* c, const ctf_problem* prob, const void* x_host, double* W_out, double* B_out, double* V_out,
            double* objective_out, ctf_err* err) {
  return guarded(err, [&] {
    if (!c) throw CtfError(CTF_ERR_CONFIG, "null context");
    if (!prob) throw CtfError(CTF_ERR_CONFIG, "null problem");
    const bool done = prob->precision == CTF_F32 ? run_overlapped<float>(c, prob, x_host)
                                                 : run_overlapped<double>(c, prob, x_host);
    if (!done) {
      setup_impl(c, prob, x_host);
      iterate_impl(c, prob->iterations, true);
    }
    ctf_err e2{};
    const int rc = ctf_download(c, W_out, B_out, V_out, objective_out, &e2);
    if (rc != CTF_OK) throw CtfError(rc, e2.msg);
  });
}

}  // extern "C"

namespace {

// Projection-back images of this rank's bins into a device buffer
// double2 [n][mix][FL][T][Dout] (wiener.cpp:11-49).
void compute_images(ctf_ctx* c, int mode, DevBuf<double>& out) {
  if (!c->ready) throw CtfError(CTF_ERR_CONFIG, "ctf_setup has not been called");
  if (c->pending) throw CtfError(CTF_ERR_CONFIG, "call ctf_finalize before ctf_project_back");
  CK(cudaSetDevice(c->device));
  const int Dout = mode == CTF_IMAGES_CURRENT_FRAME ? c->Mx : c->D;
  const size_t per_bin = (size_t)c->T * Dout;
  out.alloc((size_t)c->N * c->B * c->FL * per_bin * 2);
  ctf::ImageParams ip{};
  ip.x = c->x.p;
  ip.W = c->W.p;
  ip.out = out.p;
  ip.err = c->err.p;
  ip.FL = c->FL;
  ip.bin_lo = c->lo;
  ip.T = c->T;
  ip.Mx = c->Mx;
  ip.Ls = c->Ls;
  ip.D = c->D;
  ip.R = c->R;
  ip.N = c->N;
  ip.nmix = c->B;
  ip.current_only = mode == CTF_IMAGES_CURRENT_FRAME ? 1 : 0;
  for (int n = 0; n < c->N; ++n) {
    ip.row0[n] = c->row0[n];
    ip.ntaps[n] = c->taps[n];
  }
  const size_t cs = 2 * (size_t)c->real_size;
  const size_t smem_mats = (size_t)(2 * c->R * c->R + c->R * c->D) * cs;
  const size_t smem_x = (size_t)c->Mx * (c->Ls - 1 + c->T) * cs;
  int max_smem = 0;
  CK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device));
  if (smem_mats > (size_t)max_smem) throw CtfError(CTF_ERR_UNSUPPORTED, "projection-back tile exceeds shared memory");
  ip.stage_x = smem_mats + smem_x <= (size_t)max_smem ? 1 : 0;  // cfg4 (6 x 4009 frames): x read from global
  const size_t smem = ip.stage_x ? smem_mats + smem_x : smem_mats;
  CK(cudaMemsetAsync(c->err.p, 0xFF, c->err.n * 8, c->stream));
  if (c->real_size == 4) {
    CK(cudaFuncSetAttribute((const void*)ctf::image_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ctf::image_kernel<float><<<dim3(c->FL, c->B), 256, smem, c->stream>>>(ip);
  } else {
    CK(cudaFuncSetAttribute((const void*)ctf::image_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ctf::image_kernel<double><<<dim3(c->FL, c->B), 256, smem, c->stream>>>(ip);
  }
  CK(cudaGetLastError());
  c->timing.launches += 1;
  std::vector<unsigned long long> keys((size_t)c->B);
  CK(cudaMemcpyAsync(keys.data(), c->err.p, keys.size() * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int b = 0; b < c->B; ++b)
    if (keys[(size_t)b] != ctf::kNoErr)
      throw CtfError(CTF_ERR_DEGENERACY, "image reconstruction: demixing matrix not invertible",
                     CTF_KIND_SINGULAR_IMAGE, -1, b, (int)((keys[(size_t)b] >> 20) & 0xFFFFF), -1);
}

// ---------------------------------------------------------------------------
// STFT front/back end (stft.cpp:46-139). Tables are built on the host with
// the reference's own recurrences so the GPU transform is bit-identical.
constexpr double kPi = 3.14159265358979323846;  // std::numbers::pi

bool is_pow2(long long n) { return n > 0 && (n & (n - 1)) == 0; }

void stft_tables(ctf_ctx* c, int N) {
  if (c->stft_N == N) return;
  std::vector<double2> twf((size_t)std::max(1, N - 1)), twi((size_t)std::max(1, N - 1));
  for (int dir = 0; dir < 2; ++dir) {
    const double sign = dir ? 1.0 : -1.0;  // fft.cpp:29
    auto& tw = dir ? twi : twf;
    for (int len = 2; len <= N; len <<= 1) {
      const double angle = sign * 2.0 * kPi / static_cast<double>(len);
      const std::complex<double> wlen(std::cos(angle), std::sin(angle));
      std::complex<double> w(1.0, 0.0);
      for (int k = 0; k < len / 2; ++k) {
        tw[(size_t)(len / 2 - 1 + k)] = make_double2(w.real(), w.imag());
        w *= wlen;
      }
    }
  }
  std::vector<double> win((size_t)N);
  for (int t = 0; t < N; ++t) win[(size_t)t] = 0.5 - 0.5 * std::cos(2.0 * kPi * t / N);  // stft.cpp:14-19
  c->stft_twf.alloc(twf.size());
  c->stft_twi.alloc(twi.size());
  c->stft_win.alloc(win.size());
  CK(cudaMemcpy(c->stft_twf.p, twf.data(), twf.size() * sizeof(double2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->stft_twi.p, twi.data(), twi.size() * sizeof(double2), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->stft_win.p, win.data(), win.size() * 8, cudaMemcpyHostToDevice));
  c->stft_N = N;
}

void stft_validate(int64_t n, int channels, int N, int hop) {  // stft.cpp:47-55
  if (n == 0 || channels == 0) throw CtfError(CTF_ERR_CONFIG, "forward_stft: empty signal");
  if (N <= 0 || !is_pow2(N))
    throw CtfError(CTF_ERR_CONFIG, "forward_stft: window_len must be a power of two, got " + std::to_string(N));
  if (hop <= 0 || N % hop != 0) throw CtfError(CTF_ERR_CONFIG, "forward_stft: hop must divide window_len");
  if (n < N) throw CtfError(CTF_ERR_CONFIG, "forward_stft: signal shorter than one window");
  if (N < 2 || N > 8192) throw CtfError(CTF_ERR_UNSUPPORTED, "window_len outside [2, 8192]");
}

int log2i(int N) {
  int l = 0;
  while ((1 << l) < N) ++l;
  return l;
}

// sequences per CTA: PF frames x CC channels within 64 KB of shared memory
void stft_blocking(int N, int C, int& PF, int& CC) {
  const int smax = std::max(1, 65536 / (N * 16));
  CC = std::min(C, smax);
  PF = std::max(1, smax / CC);
}

// samples (device) [S][C][n] -> spec (device) [S][hi-lo][frames][C]
void launch_stft(ctf_ctx* c, const double* samples, int S, int64_t n, int C, int N, int hop, int lo, int hi,
                 void* spec, bool f32) {
  stft_tables(c, N);
  ctf::StftParams p{};
  p.samples = samples;
  p.spec = spec;
  p.tw = c->stft_twf.p;
  p.window = c->stft_win.p;
  p.n = n;
  p.N = N;
  p.logN = log2i(N);
  p.hop = hop;
  p.frames = (int)(1 + (n + hop - 1) / hop);
  p.C = C;
  p.bin_lo = lo;
  p.bin_hi = hi;
  stft_blocking(N, C, p.PF, p.CC);
  p.out_f32 = f32 ? 1 : 0;
  const size_t smem = (size_t)p.PF * p.CC * N * 16;
  CK(cudaFuncSetAttribute((const void*)ctf::stft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ctf::stft_kernel<<<dim3((p.frames + p.PF - 1) / p.PF, S, (C + p.CC - 1) / p.CC), 256, smem, c->stream>>>(p);
  CK(cudaGetLastError());
  c->timing.launches += 1;
}

// Validates an inverse transform (stft.cpp:91-114) and returns out_len.
int64_t istft_validate(int bins, int frames, int N, int hop, int64_t original_length) {
  if (bins != N / 2 + 1) throw CtfError(CTF_ERR_CONFIG, "inverse_stft: bin count does not match window length");
  if (hop <= 0 || N % hop != 0) throw CtfError(CTF_ERR_CONFIG, "inverse_stft: hop must divide window_len");
  if (N < 2 || N > 8192 || !is_pow2(N)) throw CtfError(CTF_ERR_UNSUPPORTED, "window_len outside [2, 8192]");
  if (frames < 1) throw CtfError(CTF_ERR_CONFIG, "inverse_stft: no frames");
  const int64_t padded_len = (int64_t)(frames - 1) * hop + N;
  std::vector<double> win((size_t)N), overlap((size_t)padded_len, 0.0);
  for (int t = 0; t < N; ++t) win[(size_t)t] = 0.5 - 0.5 * std::cos(2.0 * kPi * t / N);
  for (int j = 0; j < frames; ++j)
    for (int t = 0; t < N; ++t) overlap[(size_t)((int64_t)j * hop + t)] += win[(size_t)t] * win[(size_t)t];
  const int half = N / 2;
  const int64_t out_len = original_length > 0 ? original_length : padded_len - N;
  if (out_len + half > padded_len) throw CtfError(CTF_ERR_CONFIG, "inverse_stft: original_length inconsistent with frames");
  const double peak = *std::max_element(overlap.begin(), overlap.end());
  for (int64_t t = half; t < half + out_len; ++t)
    if (overlap[(size_t)t] < 1e-9 * peak)
      throw CtfError(CTF_ERR_CONFIG, "inverse_stft: window/hop pair does not cover the signal");
  return out_len;
}

// spec (device, double2) [S][bins][frames][C] -> out (device) [S][C][out_len]
void launch_istft(ctf_ctx* c, const double2* spec, int S, int bins, int frames, int C, int N, int hop,
                  int64_t out_len, double* out) {
  stft_tables(c, N);
  ctf::IstftParams p{};
  p.spec = spec;
  c->stft_frames.alloc((size_t)S * C * frames * N);
  p.frames_buf = c->stft_frames.p;
  p.out = out;
  p.tw = c->stft_twi.p;
  p.window = c->stft_win.p;
  p.scale = 1.0 / static_cast<double>(N);  // fft.cpp:38
  p.out_len = out_len;
  p.N = N;
  p.logN = log2i(N);
  p.hop = hop;
  p.frames = frames;
  p.bins = bins;
  p.C = C;
  p.S = S;
  stft_blocking(N, C, p.PF, p.CC);
  const size_t smem = (size_t)p.PF * p.CC * N * 16;
  CK(cudaFuncSetAttribute((const void*)ctf::istft_frame_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ctf::istft_frame_kernel<<<dim3((frames + p.PF - 1) / p.PF, S, (C + p.CC - 1) / p.CC), 256, smem, c->stream>>>(p);
  CK(cudaGetLastError());
  const int64_t total = (int64_t)S * C * out_len;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16));
  ctf::ola_kernel<<<grid, 256, 0, c->stream>>>(p);
  CK(cudaGetLastError());
  c->timing.launches += 2;
}

}  // namespace

extern "C" {

int ctf_project_back(ctf_ctx* c, int mode, double* images, ctf_err* err) {
  return guarded(err, [&] {
    if (!c) throw CtfError(CTF_ERR_CONFIG, "null context");
    if (!images) throw CtfError(CTF_ERR_CONFIG, "null output");
    DevBuf<double> out;
    compute_images(c, mode, out);
    const int Dout = mode == CTF_IMAGES_CURRENT_FRAME ? c->Mx : c->D;
    const size_t per_bin = (size_t)c->T * Dout;
    // scatter the local bins into the full-F host layout
    for (int n = 0; n < c->N; ++n)
      for (int b = 0; b < c->B; ++b) {
        double* dst = images + ((((size_t)n * c->B + b) * c->F + c->lo) * per_bin) * 2;
        const double* src = out.p + ((((size_t)n * c->B + b) * c->FL) * per_bin) * 2;
        CK(cudaMemcpyAsync(dst, src, (size_t)c->FL * per_bin * 16, cudaMemcpyDeviceToHost, c->stream));
      }
    CK(cudaStreamSynchronize(c->stream));
  });
}

int64_t ctf_stft_frames(int64_t length, int hop) { return hop > 0 ? 1 + (length + hop - 1) / hop : -1; }

int ctf_stft(ctf_ctx* c, const double* samples, int64_t length, int channels, int window_len, int hop,
             double* spec, ctf_err* err) {
  return guarded(err, [&] {
    if (!c) throw CtfError(CTF_ERR_CONFIG, "null context");
    stft_validate(length, channels, window_len, hop);
    if (!samples || !spec) throw CtfError(CTF_ERR_CONFIG, "null buffer");
    CK(cudaSetDevice(c->device));
    const int bins = window_len / 2 + 1;
    const int64_t frames = ctf_stft_frames(length, hop);
    c->stft_in.alloc((size_t)channels * length);
    c->stft_spec.alloc((size_t)bins * frames * channels);
    CK(cudaMemcpyAsync(c->stft_in.p, samples, (size_t)channels * length * 8, cudaMemcpyHostToDevice, c->stream));
    launch_stft(c, c->stft_in.p, 1, length, channels, window_len, hop, 0, bins, c->stft_spec.p, false);
    CK(cudaMemcpyAsync(spec, c->stft_spec.p, (size_t)bins * frames * channels * 16, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ctf_istft(ctf_ctx* c, const double* spec, int bins, int frames, int channels, int window_len, int hop,
              int64_t original_length, double* samples, int64_t* out_len, ctf_err* err) {
  return guarded(err, [&] {
    if (!c) throw CtfError(CTF_ERR_CONFIG, "null context");
    const int64_t len = istft_validate(bins, frames, window_len, hop, original_length);
    if (out_len) *out_len = len;
    if (!samples) return;
    if (!spec) throw CtfError(CTF_ERR_CONFIG, "null spectrogram");
    if (channels < 1) throw CtfError(CTF_ERR_CONFIG, "inverse_stft: no channels");
    CK(cudaSetDevice(c->device));
    c->stft_spec.alloc((size_t)bins * frames * channels);
    c->stft_out.alloc((size_t)channels * len);
    CK(cudaMemcpyAsync(c->stft_spec.p, spec, (size_t)bins * frames * channels * 16, cudaMemcpyHostToDevice, c->stream));
    launch_istft(c, c->stft_spec.p, 1, bins, frames, channels, window_len, hop, len, c->stft_out.p);
    CK(cudaMemcpyAsync(samples, c->stft_out.p, (size_t)channels * len * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ctf_stft_device(ctf_ctx* c, const double* samples, int num_signals, int64_t length, int channels,
                    int window_len, int hop, void* spec, int out_precision, ctf_err* err) {
  return guarded(err, [&] {
    if (!c) throw CtfError(CTF_ERR_CONFIG, "null context");
    stft_validate(length, channels, window_len, hop);
    if (!samples || !spec || num_signals < 1) throw CtfError(CTF_ERR_CONFIG, "null buffer");
    CK(cudaSetDevice(c->device));
    launch_stft(c, samples, num_signals, length, channels, window_len, hop, 0, window_len / 2 + 1, spec,
                out_precision == CTF_F32);
  });
}

int ctf_istft_device(ctf_ctx* c, const double* spec, int num_signals, int bins, int frames, int channels,
                     int window_len, int hop, int64_t original_length, double* samples, ctf_err* err) {
  return guarded(err, [&] {
    if (!c) throw CtfError(CTF_ERR_CONFIG, "null context");
    const int64_t len = istft_validate(bins, frames, window_len, hop, original_length);
    if (!spec || !samples || num_signals < 1 || channels < 1) throw CtfError(CTF_ERR_CONFIG, "null buffer");
    CK(cudaSetDevice(c->device));
    launch_istft(c, reinterpret_cast<const double2*>(spec), num_signals, bins, frames, channels, window_len, hop,
                 len, samples);
  });
}

int ctf_setup_signal(ctf_ctx* c, const ctf_problem* prob, const double* samples, int64_t length, int window_len,
                     int hop, ctf_err* err) {
  return guarded(err, [&] {
    if (!c) throw CtfError(CTF_ERR_CONFIG, "null context");
    if (!prob) throw CtfError(CTF_ERR_CONFIG, "null problem");
    stft_validate(length, prob->num_mics, window_len, hop);
    if (!samples) throw CtfError(CTF_ERR_CONFIG, "null signal");
    ctf_problem p = *prob;
    const int bins = window_len / 2 + 1;
    const int frames = (int)ctf_stft_frames(length, hop);
    if ((p.num_bins && p.num_bins != bins) || (p.num_frames && p.num_frames != frames))
      throw CtfError(CTF_ERR_CONFIG, "num_bins / num_frames do not match the STFT of the signal");
    p.num_bins = bins;
    p.num_frames = frames;
    p.x_precision = p.precision;
    CK(cudaSetDevice(c->device));
    setup_impl(c, &p, nullptr, [&] {
      const size_t cnt = (size_t)p.num_mixtures * p.num_mics * length;
      c->stft_in.alloc(cnt);
      CK(cudaMemcpyAsync(c->stft_in.p, samples, cnt * 8, cudaMemcpyHostToDevice, c->stream));
      launch_stft(c, c->stft_in.p, p.num_mixtures, length, p.num_mics, window_len, hop, c->lo, c->hi, c->x.p,
                  c->real_size == 4);
    });
  });
}

int ctf_images_to_signal(ctf_ctx* c, int ref_channel, int window_len, int hop, int64_t original_length,
                         double* out, int64_t* out_len, ctf_err* err) {
  return guarded(err, [&] {
    if (!c || !c->ready) throw CtfError(CTF_ERR_CONFIG, "ctf_setup has not been called");
    if (c->FL != c->F) throw CtfError(CTF_ERR_CONFIG, "images_to_signal needs every bin on this rank (world 1)");
    const int64_t len = istft_validate(c->F, c->T, window_len, hop, original_length);
    if (ref_channel >= c->Mx)  // wiener.cpp:56-59
      throw CtfError(CTF_ERR_CONFIG, "ref_channel " + std::to_string(ref_channel) + " out of range for " +
                                         std::to_string(c->Mx) + " channels");
    if (out_len) *out_len = len;
    if (!out) return;
    // the microphone images: current-frame channels of the stacked space
    // (stack_taps > 1) or the supplied channels (stack_taps = 1); Dout = Mx
    DevBuf<double> img;
    compute_images(c, c->Ls > 1 ? CTF_IMAGES_CURRENT_FRAME : CTF_IMAGES_FULL, img);
    const int S = c->N * c->B, C = c->Mx;
    c->stft_out.alloc((size_t)S * C * len);
    launch_istft(c, reinterpret_cast<const double2*>(img.p), S, c->F, c->T, C, window_len, hop, len, c->stft_out.p);
    if (ref_channel < 0) {
      CK(cudaMemcpyAsync(out, c->stft_out.p, (size_t)S * C * len * 8, cudaMemcpyDeviceToHost, c->stream));
    } else {
      CK(cudaMemcpy2DAsync(out, (size_t)len * 8, c->stft_out.p + (size_t)ref_channel * len, (size_t)C * len * 8,
                           (size_t)len * 8, (size_t)S, cudaMemcpyDeviceToHost, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"
