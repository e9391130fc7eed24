// ctfmnmf_b200 — the reference's command-line front end
// (proj/tools/ctfmnmf_main.cpp:179-364) on the GPU path: `separate` and
// `bench` with the same flags, key/value config file, outputs
// (srcN.wav, trace.csv, bench.csv, manifest.json) and exit codes
// (2 config, 3 I/O, 4 numerical degeneracy; ctfmnmf_main.cpp:38-40).
//
//   ctfmnmf_b200 separate MIXTURE(.wav|.spec) [--config F] [--out DIR] [--seed S]
//                [--rule ip|iss] [--iters N] [--threads N] [--ref-channel C]
//                [--precision f64|f32] [--device D]
//   ctfmnmf_b200 bench [--channels 4,6,8] [common flags]
//
// Everything between the file formats runs on the GPU through the C++
// mirror (ctfmnmf_b200.hpp): STFT, the ISS/IP + NMF loop, projection-back and
// the inverse STFT. `simulate` (the reference's own synthetic bundle) is out
// of scope; `bench` draws its mixtures from BASELINE's generator
// (ctf_synth_mixtures) instead of the reference's synth.cpp.
#include "ctfmnmf_b200.hpp"

#include "../../include/ctf_iss.h"

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

namespace fs = std::filesystem;
using namespace ctfmnmf::b200;

namespace {

constexpr const char* kVersion = "0.1.0-b200";
constexpr int kExitConfig = 2, kExitIo = 3, kExitNumerical = 4;

std::string trim(const std::string& s) {
  const auto b = s.find_first_not_of(" \t\r\n");
  if (b == std::string::npos) return "";
  return s.substr(b, s.find_last_not_of(" \t\r\n") - b + 1);
}

std::vector<int> int_list(const std::string& text) {
  std::vector<int> v;
  std::stringstream ss(text);
  std::string item;
  while (std::getline(ss, item, ','))
    if (!trim(item).empty()) v.push_back(std::stoi(item));
  return v;
}

UpdateRule parse_rule(const std::string& name) {  // model.cpp:16-20
  if (name == "ip" || name == "IP") return UpdateRule::Ip;
  if (name == "iss" || name == "ISS") return UpdateRule::Iss;
  throw ConfigError("unknown update rule '" + name + "' (expected ip or iss)");
}

// Pipeline options beyond CtfConfig (ctfmnmf_main.cpp:44-89).
struct Pipeline {
  int window = 1024, hop = 0, frames = 400, trials = 3, ref_channel = -1;
  double sample_rate = 16000.0, decay = 0.5;
  std::vector<int> channels = {4, 6, 8};
  int effective_hop() const { return hop > 0 ? hop : window / 4; }
};

// `key = value` lines, '#' comments; estimator keys first (model.cpp:74-129),
// the rest are pipeline keys; unknown keys are a ConfigError.
void apply_config_file(const std::string& path, CtfConfig& c, Pipeline& pl) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open config file: " + path);
  std::string line;
  int no = 0;
  while (std::getline(in, line)) {
    ++no;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    line = trim(line);
    if (line.empty()) continue;
    const auto eq = line.find('=');
    if (eq == std::string::npos) throw ConfigError(path + ":" + std::to_string(no) + ": expected 'key = value'");
    const std::string k = trim(line.substr(0, eq)), v = trim(line.substr(eq + 1));
    try {
      if (k == "n_sources") c.num_sources = std::stoi(v);
      else if (k == "n_channels") c.num_channels = std::stoi(v);
      else if (k == "taps") c.taps_per_source = int_list(v);
      else if (k == "bases") c.bases_per_source = int_list(v);
      else if (k == "iters") c.iterations = std::stoi(v);
      else if (k == "rule") c.update_rule = parse_rule(v);
      else if (k == "floor") c.psd_floor = std::stod(v);
      else if (k == "seed") c.seed = std::stoull(v);
      else if (k == "threads") c.threads = std::stoi(v);
      else if (k == "window") pl.window = std::stoi(v);
      else if (k == "hop") pl.hop = std::stoi(v);
      else if (k == "srate") pl.sample_rate = std::stod(v);
      else if (k == "frames") pl.frames = std::stoi(v);
      else if (k == "decay") pl.decay = std::stod(v);
      else if (k == "trials") pl.trials = std::stoi(v);
      else if (k == "ref_channel") pl.ref_channel = std::stoi(v);
      else if (k == "channels") pl.channels = int_list(v);
      else throw ConfigError("unknown config key '" + k + "'");
    } catch (const std::invalid_argument&) {
      throw ConfigError("invalid value '" + v + "' for key '" + k + "'");
    } catch (const std::out_of_range&) {
      throw ConfigError("value out of range for key '" + k + "'");
    }
  }
}

// ---- RIFF WAV: 16-bit PCM and 32-bit float in, 32-bit float out (wav.hpp)
template <typename T> T rd(std::istream& in) {
  T v{};
  in.read(reinterpret_cast<char*>(&v), sizeof(T));
  return v;
}

TimeSignal read_wav(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open wav file: " + path);
  char tag[4];
  in.read(tag, 4);
  rd<uint32_t>(in);
  char wave[4];
  in.read(wave, 4);
  if (!in || std::memcmp(tag, "RIFF", 4) || std::memcmp(wave, "WAVE", 4)) throw IoError("not a RIFF/WAVE file: " + path);
  int fmt = 0, ch = 0, bits = 0;
  double rate = 0;
  std::vector<char> data;
  while (in.read(tag, 4)) {
    const uint32_t size = rd<uint32_t>(in);
    if (!std::memcmp(tag, "fmt ", 4)) {
      fmt = rd<uint16_t>(in);
      ch = rd<uint16_t>(in);
      rate = rd<uint32_t>(in);
      rd<uint32_t>(in);
      rd<uint16_t>(in);
      bits = rd<uint16_t>(in);
      in.seekg(size - 16 + (size & 1), std::ios::cur);
    } else if (!std::memcmp(tag, "data", 4)) {
      data.resize(size);
      in.read(data.data(), size);
      if (size & 1) in.seekg(1, std::ios::cur);
    } else {
      in.seekg(size + (size & 1), std::ios::cur);
    }
  }
  const bool pcm16 = fmt == 1 && bits == 16, f32 = fmt == 3 && bits == 32;
  if (!pcm16 && !f32) throw IoError("unsupported wav encoding (16-bit PCM or 32-bit float): " + path);
  if (ch <= 0) throw IoError("wav file without channels: " + path);
  const size_t bps = bits / 8, n = data.size() / (bps * ch);
  TimeSignal s;
  s.sample_rate = rate;
  s.samples = RMatrix((int)n, ch);
  for (size_t t = 0; t < n; ++t)
    for (int c = 0; c < ch; ++c) {
      const char* p = data.data() + (t * ch + c) * bps;
      double v;
      if (pcm16) {
        int16_t q;
        std::memcpy(&q, p, 2);
        v = q / 32768.0;
      } else {
        float q;
        std::memcpy(&q, p, 4);
        v = q;
      }
      s.samples((int)t, c) = v;
    }
  return s;
}

void write_wav(const std::string& path, const TimeSignal& s) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot write wav file: " + path);
  const uint32_t ch = s.channels(), n = (uint32_t)s.length(), bytes = n * ch * 4;
  auto w32 = [&](uint32_t v) { out.write(reinterpret_cast<const char*>(&v), 4); };
  auto w16 = [&](uint16_t v) { out.write(reinterpret_cast<const char*>(&v), 2); };
  out.write("RIFF", 4);
  w32(36 + bytes);
  out.write("WAVEfmt ", 8);
  w32(16);
  w16(3);
  w16((uint16_t)ch);
  w32((uint32_t)std::lround(s.sample_rate));
  w32((uint32_t)std::lround(s.sample_rate) * ch * 4);
  w16((uint16_t)(ch * 4));
  w16(32);
  out.write("data", 4);
  w32(bytes);
  for (uint32_t t = 0; t < n; ++t)
    for (uint32_t c = 0; c < ch; ++c) {
      const float v = (float)s.samples((int)t, (int)c);
      out.write(reinterpret_cast<const char*>(&v), 4);
    }
  if (!out) throw IoError("cannot write wav file: " + path);
}

// ---- minimal JSON writer for the manifest
std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}
std::string jnum(double v) {
  if (!std::isfinite(v)) return "null";
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}
std::string jints(const std::vector<int>& v) {
  std::string o = "[";
  for (size_t i = 0; i < v.size(); ++i) o += (i ? ", " : "") + std::to_string(v[i]);
  return o + "]";
}

std::string config_json(const CtfConfig& c, const Pipeline& pl, const std::string& precision) {
  std::ostringstream o;
  o << "{\"n_sources\": " << c.num_sources << ", \"n_channels\": " << c.num_channels
    << ", \"taps\": " << jints(c.taps_per_source) << ", \"bases\": " << jints(c.bases_per_source)
    << ", \"iters\": " << c.iterations << ", \"rule\": " << jstr(c.update_rule == UpdateRule::Ip ? "ip" : "iss")
    << ", \"floor\": " << jnum(c.psd_floor) << ", \"seed\": " << c.seed << ", \"threads\": " << c.threads
    << ", \"window\": " << pl.window << ", \"hop\": " << pl.effective_hop() << ", \"srate\": " << jnum(pl.sample_rate)
    << ", \"frames\": " << pl.frames << ", \"decay\": " << jnum(pl.decay) << ", \"precision\": " << jstr(precision)
    << ", \"device\": \"cuda\"}";
  return o.str();
}

void write_text(const fs::path& p, const std::string& text) {
  std::ofstream out(p);
  if (!out) throw IoError("cannot write " + p.string());
  out << text;
}

struct Flags {
  std::string config_path, out_dir = ".", precision = "f64";
  std::optional<uint64_t> seed;
  std::optional<std::string> rule;
  std::optional<int> iters, threads, ref_channel;
  std::vector<int> channels;
  int device = 0;
};

CtfConfig default_config() {  // ctfmnmf_main.cpp:145-154
  CtfConfig c;
  c.num_sources = 2;
  c.num_channels = 4;
  c.taps_per_source = {2, 2};
  c.bases_per_source = {3, 3};
  c.iterations = 100;
  c.update_rule = UpdateRule::Iss;
  return c;
}

void resolve(const Flags& f, CtfConfig& c, Pipeline& pl) {  // file first, flags on top
  if (!f.config_path.empty()) apply_config_file(f.config_path, c, pl);
  if (f.seed) c.seed = *f.seed;
  if (f.rule) c.update_rule = parse_rule(*f.rule);
  if (f.iters) c.iterations = *f.iters;
  if (f.threads) c.threads = *f.threads;
  if (f.ref_channel) pl.ref_channel = *f.ref_channel;
  if (!f.channels.empty()) pl.channels = f.channels;
}

GpuOptions gpu_of(const Flags& f) {
  GpuOptions g;
  g.device = f.device;
  if (f.precision == "f32") g.precision = Precision::F32;
  else if (f.precision != "f64") throw ConfigError("unknown precision '" + f.precision + "' (expected f64 or f32)");
  return g;
}

int cmd_separate(const Flags& f, const std::string& mixture_path) {
  CtfConfig config = default_config();
  Pipeline pl;
  resolve(f, config, pl);
  config.validate();
  const GpuOptions gpu = gpu_of(f);
  const fs::path out_dir(f.out_dir);
  fs::create_directories(out_dir);
  std::string manifest_head = "{\n  \"command\": \"separate\",\n  \"version\": " + jstr(kVersion) +
                              ",\n  \"config\": " + config_json(config, pl, f.precision) +
                              ",\n  \"inputs\": {\"mixture\": " + jstr(mixture_path) + "}";
  // load_mixture (ctfmnmf_main.cpp:157-175): .spec as stored, else WAV -> GPU STFT
  Spectrogram meta;
  if (mixture_path.size() >= 5 && mixture_path.substr(mixture_path.size() - 5) == ".spec") {
    meta = read_spectrogram(mixture_path);
  } else {
    const TimeSignal signal = read_wav(mixture_path);
    if (signal.channels() != config.num_channels)
      throw ConfigError("mixture has " + std::to_string(signal.channels()) + " channels but the config expects " +
                        std::to_string(config.num_channels));
    meta = forward_stft(signal, pl.window, pl.effective_hop(), gpu);
  }
  if (meta.channels != config.num_channels)
    throw ConfigError("mixture has " + std::to_string(meta.channels) + " channels but the config expects " +
                      std::to_string(config.num_channels));
  const MixtureSpectrogram mixture = MixtureSpectrogram::from_spectrogram(meta);
  const auto t0 = std::chrono::steady_clock::now();
  try {
    const SeparationResult result = run(config, mixture, gpu);
    const auto images = reconstruct_images(result.demixing, result.factors, mixture, config, gpu);
    std::string sources = "[";
    for (int n = 0; n < config.num_sources; ++n) {
      const TimeSignal src = image_to_signal(images[(size_t)n], meta, pl.ref_channel, gpu);
      const std::string name = "src" + std::to_string(n + 1) + ".wav";
      write_wav((out_dir / name).string(), src);
      sources += (n ? ", " : "") + jstr(name);
    }
    write_text(out_dir / "trace.csv", result.trace.to_csv());
    const double total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::ostringstream m;
    m << manifest_head << ",\n  \"outputs\": {\"sources\": " << sources << "], \"trace\": \"trace.csv\"}"
      << ",\n  \"timing_ms\": {\"total\": " << jnum(total) << ", \"demix\": " << jnum(result.trace.total_demix_ms())
      << ", \"mu\": " << jnum(result.trace.total_mu_ms()) << ", \"rescale\": " << jnum(result.trace.total_rescale_ms())
      << "},\n  \"final_objective\": "
      << (result.trace.objective.empty() ? std::string("null") : jnum(result.trace.objective.back()))
      << ",\n  \"errors\": []\n}\n";
    write_text(out_dir / "manifest.json", m.str());
  } catch (const DegeneracyError& e) {
    write_text(out_dir / "manifest.json",
               manifest_head + ",\n  \"errors\": [{\"message\": " + jstr(e.what()) + ", \"iteration\": " +
                   std::to_string(e.iteration) + ", \"bin\": " + std::to_string(e.bin) + ", \"row\": " +
                   std::to_string(e.row) + "}]\n}\n");
    std::cerr << "numerical degeneracy: " << e.what() << "\n";
    return kExitNumerical;
  }
  return 0;
}

// bench (ctfmnmf_main.cpp:289-346): ip vs iss over channel counts m, two
// sources with m/2 taps each, `trials` seeded mixtures per m.
int cmd_bench(const Flags& f) {
  CtfConfig base = default_config();
  Pipeline pl;
  resolve(f, base, pl);
  const GpuOptions gpu = gpu_of(f);
  for (int m : pl.channels)
    if (m < 2 || m % 2 != 0)
      throw ConfigError("bench channel counts must be even and >= 2 so that two sources split the taps evenly, got " +
                        std::to_string(m));
  const fs::path out_dir(f.out_dir);
  fs::create_directories(out_dir);
  const int F = pl.window / 2 + 1, T = pl.frames;
  std::ostringstream csv;
  csv << "M,rule,total_ms,demix_ms,mu_ms,seed\n";
  for (int m : pl.channels) {
    CtfConfig config = base;
    config.num_channels = m;
    config.taps_per_source = {m / 2, m / 2};
    config.bases_per_source = {base.bases_per_source[0], base.bases_per_source[0]};
    config.num_sources = 2;
    config.validate();
    for (int trial = 0; trial < pl.trials; ++trial) {
      const uint64_t seed = base.seed + (uint64_t)trial;
      // m microphones, 2 sources, single-tap mixing; the m channels are the
      // observation rows the m/2 taps per source demix (as the reference's bench)
      std::vector<double> raw((size_t)F * T * m * 2);
      ctf_err err{};
      if (ctf_synth_mixtures(1, F, T, m, 2, 1, config.bases_per_source[0], pl.decay, seed, CTF_F64, raw.data(), 0,
                             &err) != 0)
        throw ConfigError(err.msg);
      MixtureSpectrogram x;
      x.bins.assign((size_t)F, CMatrix(m, T));
      for (int i = 0; i < F; ++i)
        for (int t = 0; t < T; ++t)
          for (int c = 0; c < m; ++c) {
            const size_t o = (((size_t)i * T + t) * m + c) * 2;
            x.bins[(size_t)i](c, t) = Complex(raw[o], raw[o + 1]);
          }
      for (UpdateRule rule : {UpdateRule::Ip, UpdateRule::Iss}) {
        config.update_rule = rule;
        config.seed = seed;
        const auto t0 = std::chrono::steady_clock::now();
        const SeparationResult r = run(config, x, gpu);
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        csv << m << ',' << (rule == UpdateRule::Ip ? "ip" : "iss") << ',' << ms << ',' << r.trace.total_demix_ms()
            << ',' << r.trace.total_mu_ms() << ',' << seed << '\n';
      }
    }
  }
  write_text(out_dir / "bench.csv", csv.str());
  write_text(out_dir / "manifest.json",
             "{\n  \"command\": \"bench\",\n  \"version\": " + jstr(kVersion) + ",\n  \"config\": " +
                 config_json(base, pl, f.precision) + ",\n  \"channels\": " + jints(pl.channels) +
                 ",\n  \"trials\": " + std::to_string(pl.trials) +
                 ",\n  \"outputs\": {\"csv\": \"bench.csv\"},\n  \"errors\": []\n}\n");
  return 0;
}

int usage(const char* msg) {
  if (msg) std::cerr << msg << "\n";
  std::cerr << "usage: ctfmnmf_b200 separate MIXTURE [--config F] [--out DIR] [--seed S] [--rule ip|iss] [--iters N]\n"
               "                    [--threads N] [--ref-channel C] [--precision f64|f32] [--device D]\n"
               "       ctfmnmf_b200 bench [--channels 4,6,8] [common flags]\n";
  return kExitConfig;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 2 && std::string(argv[1]) == "--version") {
    std::cout << kVersion << "\n";
    return 0;
  }
  if (argc < 2) return usage("a subcommand is required");
  const std::string cmd = argv[1];
  if (cmd != "separate" && cmd != "bench") return usage(("unknown subcommand '" + cmd + "'").c_str());
  Flags f;
  std::string mixture;
  try {
    for (int i = 2; i < argc; ++i) {
      const std::string a = argv[i];
      auto val = [&]() -> std::string {
        if (i + 1 >= argc) throw ConfigError(a + " requires a value");
        return argv[++i];
      };
      if (a == "--config") f.config_path = val();
      else if (a == "--out") f.out_dir = val();
      else if (a == "--seed") f.seed = std::stoull(val());
      else if (a == "--rule") {
        f.rule = val();
        if (*f.rule != "ip" && *f.rule != "iss") throw ConfigError("--rule: " + *f.rule + " not in {ip, iss}");
      } else if (a == "--iters") f.iters = std::stoi(val());
      else if (a == "--threads") f.threads = std::stoi(val());
      else if (a == "--ref-channel" && cmd == "separate") f.ref_channel = std::stoi(val());
      else if (a == "--channels" && cmd == "bench") f.channels = int_list(val());
      else if (a == "--precision") f.precision = val();
      else if (a == "--device") f.device = std::stoi(val());
      else if (!a.empty() && a[0] != '-' && cmd == "separate" && mixture.empty()) mixture = a;
      else throw ConfigError("unexpected argument '" + a + "'");
    }
    if (cmd == "separate" && mixture.empty()) throw ConfigError("separate: the mixture argument is required");
  } catch (const ConfigError& e) {
    return usage(e.what());
  } catch (const std::exception& e) {
    return usage((std::string("invalid flag value: ") + e.what()).c_str());
  }
  try {
    return cmd == "separate" ? cmd_separate(f, mixture) : cmd_bench(f);
  } catch (const ConfigError& e) {
    std::cerr << "configuration error: " << e.what() << "\n";
    return kExitConfig;
  } catch (const IoError& e) {
    std::cerr << "i/o error: " << e.what() << "\n";
    return kExitIo;
  } catch (const DegeneracyError& e) {
    std::cerr << "numerical degeneracy: " << e.what() << "\n";
    return kExitNumerical;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
