// ctf_container.cpp — the reference's binary containers,
// host side of the C ABI: the `.spec` spectrogram the `separate` command
// reads and the `.nmf` factor file it can write (proj/src/container.cpp,
// format in proj/include/ctfmnmf/container.hpp:1-10; little-endian):
//
//   spectrogram "CTFSPG1\0": u32 bins, frames, channels, window_len, hop,
//     sample_rate_hz; u64 original_length; complex64 body, bin-major
//     (for i, for j, for c) — the estimator's x layout, so a file body can be
//     uploaded as is (x_precision = f32).
//   factors "CTFNMF1\0": u32 sources, bins, frames; u32 bases[sources];
//     f64 floor; f64 body: per source B (bins x K) row-major then V (K x
//     frames) row-major.
//
// Error texts follow container.cpp (IoError, status 3).
#include "../../include/ctf_iss.h"

#include <complex>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

constexpr char kSpecMagic[8] = {'C', 'T', 'F', 'S', 'P', 'G', '1', '\0'};
constexpr char kNmfMagic[8] = {'C', 'T', 'F', 'N', 'M', 'F', '1', '\0'};

struct ContainerError : std::runtime_error {
  int code;
  ContainerError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

template <class Fn>
int guarded_io(ctf_err* err, Fn&& fn) {
  if (err) {
    std::memset(err, 0, sizeof(*err));
    err->iteration = err->mixture = err->bin = err->row = -1;
  }
  try {
    fn();
    return CTF_OK;
  } catch (const ContainerError& e) {
    if (err) {
      err->code = e.code;
      std::snprintf(err->msg, sizeof(err->msg), "%s", e.what());
    }
    return e.code;
  } catch (const std::exception& e) {
    if (err) {
      err->code = CTF_ERR_IO;
      std::snprintf(err->msg, sizeof(err->msg), "%s", e.what());
    }
    return CTF_ERR_IO;
  }
}

template <typename T> void put(std::ostream& out, T v) { out.write(reinterpret_cast<const char*>(&v), sizeof(T)); }
template <typename T> T get(std::istream& in) {
  T v{};
  in.read(reinterpret_cast<char*>(&v), sizeof(T));
  return v;
}

std::ofstream open_out(const std::string& path, const char* magic) {  // container.cpp:41-46
  std::ofstream out(path, std::ios::binary);
  if (!out) throw ContainerError(CTF_ERR_IO, "cannot create file: " + path);
  out.write(magic, 8);
  return out;
}

std::ifstream open_in(const std::string& path, const char* magic) {  // container.cpp:48-57
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ContainerError(CTF_ERR_IO, "cannot open file: " + path);
  char header[8];
  in.read(header, 8);
  if (!in || std::memcmp(header, magic, 8) != 0)
    throw ContainerError(CTF_ERR_IO, path + ": bad or mismatched container magic");
  return in;
}

ctf_spec_header read_spec_header(std::istream& in) {  // container.cpp:74-86
  ctf_spec_header h{};
  h.bins = get<uint32_t>(in);
  h.frames = get<uint32_t>(in);
  h.channels = get<uint32_t>(in);
  h.window_len = get<uint32_t>(in);
  h.hop = get<uint32_t>(in);
  h.sample_rate = get<uint32_t>(in);
  h.original_length = get<uint64_t>(in);
  return h;
}

}  // namespace

extern "C" {

int ctf_read_spectrogram(const char* path, ctf_spec_header* hdr, void* data, int out_precision, ctf_err* err) {
  return guarded_io(err, [&] {
    if (!path || !hdr) throw ContainerError(CTF_ERR_CONFIG, "null argument");
    std::ifstream in = open_in(path, kSpecMagic);
    *hdr = read_spec_header(in);
    if (!in) throw ContainerError(CTF_ERR_IO, std::string(path) + ": truncated spectrogram container");
    if (!data) return;
    const size_t n = (size_t)hdr->bins * hdr->frames * hdr->channels;
    std::vector<float> body(2 * n);
    in.read(reinterpret_cast<char*>(body.data()), (std::streamsize)(body.size() * sizeof(float)));
    if (!in) throw ContainerError(CTF_ERR_IO, std::string(path) + ": truncated spectrogram container");
    if (out_precision == CTF_F32) {
      std::memcpy(data, body.data(), body.size() * sizeof(float));
    } else {
      double* d = static_cast<double*>(data);
      for (size_t i = 0; i < body.size(); ++i) d[i] = (double)body[i];  // get_complex widens
    }
  });
}

int ctf_write_spectrogram(const char* path, const ctf_spec_header* hdr, const void* data, int in_precision,
                          ctf_err* err) {
  return guarded_io(err, [&] {
    if (!path || !hdr || !data) throw ContainerError(CTF_ERR_CONFIG, "null argument");
    std::ofstream out = open_out(path, kSpecMagic);  // container.cpp:61-72
    put<uint32_t>(out, hdr->bins);
    put<uint32_t>(out, hdr->frames);
    put<uint32_t>(out, hdr->channels);
    put<uint32_t>(out, hdr->window_len);
    put<uint32_t>(out, hdr->hop);
    put<uint32_t>(out, hdr->sample_rate);
    put<uint64_t>(out, hdr->original_length);
    const size_t n = 2 * (size_t)hdr->bins * hdr->frames * hdr->channels;
    if (in_precision == CTF_F32) {
      out.write(static_cast<const char*>(data), (std::streamsize)(n * sizeof(float)));
    } else {
      const double* d = static_cast<const double*>(data);
      std::vector<float> body(n);
      for (size_t i = 0; i < n; ++i) body[i] = (float)d[i];  // put_complex narrows
      out.write(reinterpret_cast<const char*>(body.data()), (std::streamsize)(n * sizeof(float)));
    }
    if (!out) throw ContainerError(CTF_ERR_IO, std::string("short write: ") + path);
  });
}

int ctf_setup_spectrogram_files(ctf_ctx* ctx, const ctf_problem* prob, const char* const* paths, int num_paths,
                                ctf_spec_header* hdr_out, ctf_err* err) {
  std::vector<float> x;
  ctf_problem p{};
  const int rc = guarded_io(err, [&] {
    if (!ctx || !prob || !paths || num_paths < 1) throw ContainerError(CTF_ERR_CONFIG, "null argument");
    p = *prob;
    ctf_spec_header h0{};
    for (int b = 0; b < num_paths; ++b) {
      std::ifstream in = open_in(paths[b], kSpecMagic);
      const ctf_spec_header h = read_spec_header(in);
      if (!in) throw ContainerError(CTF_ERR_IO, std::string(paths[b]) + ": truncated spectrogram container");
      if (b == 0) {
        h0 = h;
        x.resize((size_t)num_paths * 2 * h.bins * h.frames * h.channels);
      } else if (h.bins != h0.bins || h.frames != h0.frames || h.channels != h0.channels) {
        throw ContainerError(CTF_ERR_CONFIG, std::string(paths[b]) + ": shape differs from " + paths[0]);
      }
      const size_t n = 2 * (size_t)h.bins * h.frames * h.channels;
      in.read(reinterpret_cast<char*>(x.data() + (size_t)b * n), (std::streamsize)(n * sizeof(float)));
      if (!in) throw ContainerError(CTF_ERR_IO, std::string(paths[b]) + ": truncated spectrogram container");
    }
    if ((p.num_bins && p.num_bins != (int)h0.bins) || (p.num_frames && p.num_frames != (int)h0.frames) ||
        (p.num_mics && p.num_mics != (int)h0.channels))
      throw ContainerError(CTF_ERR_CONFIG, "problem shape does not match the spectrogram container");
    p.num_mixtures = num_paths;
    p.num_bins = (int)h0.bins;
    p.num_frames = (int)h0.frames;
    p.num_mics = (int)h0.channels;
    p.x_precision = CTF_F32;  // complex64 body as stored
    if (hdr_out) *hdr_out = h0;
  });
  if (rc != CTF_OK) return rc;
  return ctf_setup(ctx, &p, x.data(), err);
}

int ctf_write_factors(const char* path, int num_sources, int bins, int frames, const int32_t* bases,
                      double floor_abs, const double* B, const double* V, ctf_err* err) {
  return guarded_io(err, [&] {
    if (!path || !bases || !B || !V || num_sources < 1) throw ContainerError(CTF_ERR_CONFIG, "null argument");
    std::ofstream out = open_out(path, kNmfMagic);  // container.cpp:124-142
    put<uint32_t>(out, (uint32_t)num_sources);
    put<uint32_t>(out, (uint32_t)bins);
    put<uint32_t>(out, (uint32_t)frames);
    for (int n = 0; n < num_sources; ++n) put<uint32_t>(out, (uint32_t)bases[n]);
    put<double>(out, floor_abs);
    size_t ob = 0, ov = 0;
    for (int n = 0; n < num_sources; ++n) {  // B_n column-major F x K (ABI) -> row-major; V_n K x T -> row-major
      const int K = bases[n];
      for (int i = 0; i < bins; ++i)
        for (int k = 0; k < K; ++k) put<double>(out, B[ob + (size_t)i + (size_t)k * bins]);
      for (int k = 0; k < K; ++k)
        for (int j = 0; j < frames; ++j) put<double>(out, V[ov + (size_t)k + (size_t)j * K]);
      ob += (size_t)bins * K;
      ov += (size_t)K * frames;
    }
    if (!out) throw ContainerError(CTF_ERR_IO, std::string("short write: ") + path);
  });
}

int ctf_read_factors(const char* path, int* num_sources, int* bins, int* frames, int32_t* bases /* [16] */,
                     double* floor_abs, double* B, double* V, ctf_err* err) {
  return guarded_io(err, [&] {
    if (!path || !num_sources || !bins || !frames || !bases) throw ContainerError(CTF_ERR_CONFIG, "null argument");
    std::ifstream in = open_in(path, kNmfMagic);  // container.cpp:144-165
    const uint32_t ns = get<uint32_t>(in), nb = get<uint32_t>(in), nf = get<uint32_t>(in);
    if (ns > CTF_MAX_SOURCES) throw ContainerError(CTF_ERR_IO, std::string(path) + ": too many sources");
    *num_sources = (int)ns;
    *bins = (int)nb;
    *frames = (int)nf;
    for (uint32_t n = 0; n < ns; ++n) bases[n] = (int32_t)get<uint32_t>(in);
    const double fl = get<double>(in);
    if (floor_abs) *floor_abs = fl;
    if (!in) throw ContainerError(CTF_ERR_IO, std::string(path) + ": truncated factor container");
    if (!B || !V) return;
    size_t ob = 0, ov = 0;
    for (uint32_t n = 0; n < ns; ++n) {
      const int K = bases[n];
      for (uint32_t i = 0; i < nb; ++i)
        for (int k = 0; k < K; ++k) B[ob + (size_t)i + (size_t)k * nb] = get<double>(in);
      for (int k = 0; k < K; ++k)
        for (uint32_t j = 0; j < nf; ++j) V[ov + (size_t)k + (size_t)j * K] = get<double>(in);
      ob += (size_t)nb * K;
      ov += (size_t)K * nf;
    }
    if (!in) throw ContainerError(CTF_ERR_IO, std::string(path) + ": truncated factor container");
  });
}

}  // extern "C"
