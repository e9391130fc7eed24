"""GPU STFT front end / WOLA back end vs the CPU oracle restatement of
proj/src/stft.cpp + fft.cpp (itself pinned by test_stft_kats.py against the
reference's test_stft.cpp cases). The GPU transform uses the reference's
arithmetic (twiddle recurrence, no FMA contraction), so parity is bitwise."""
import threading

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_02382_b200 import ConfigError, Session, forward_stft, inverse_stft
from paper_2510_02382_b200 import _lib

pytestmark = pytest.mark.gpu


def _signal(channels, length, seed):
    return np.random.default_rng(seed).standard_normal((channels, length))


@pytest.mark.parametrize("channels,length,window,hop", [
    (1, 64, 8, 2),          # DC-test geometry
    (2, 4096, 1024, 256),   # 16 kHz / 1024 / 25 %
    (1, 2000, 512, 64),
    (1, 2000, 512, 128),
    (3, 1500, 512, 256),    # odd channel count
    (2, 1024, 1024, 1024),  # length == window, hop == window
    (1, 40, 2, 1),          # smallest window
    (2, 20000, 8192, 2048),  # largest window
    (5, 3001, 256, 32),
])
def test_forward_stft_bitwise(channels, length, window, hop):
    s = _signal(channels, length, length + window)
    ref = O.forward_stft(s, window, hop)
    got = forward_stft(s, window, hop)
    assert got.shape == ref.shape
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("channels,length,window,hop", [
    (2, 4096, 1024, 256), (1, 2000, 512, 64), (3, 1500, 512, 256), (1, 40, 2, 1), (2, 20000, 8192, 2048)])
def test_inverse_stft_bitwise_and_round_trip(channels, length, window, hop):
    s = _signal(channels, length, 7 * length + hop)
    spec = O.forward_stft(s, window, hop)
    ref = O.inverse_stft(spec, window, hop, length)
    got = inverse_stft(spec, window, hop, length)
    assert np.array_equal(got, ref)
    assert np.max(np.abs(got - s)) / np.max(np.abs(s)) < 1e-10
    # default output length (original_length = 0)
    assert np.array_equal(inverse_stft(spec, window, hop), O.inverse_stft(spec, window, hop))


def test_inverse_of_arbitrary_spectrum_bitwise():
    """Non-Hermitian-consistent bins 0 and N/2 (imaginary parts dropped as in the reference)."""
    g = np.random.default_rng(4)
    spec = g.standard_normal((9, 11, 2)) + 1j * g.standard_normal((9, 11, 2))
    assert np.array_equal(inverse_stft(spec, 16, 4, 30), O.inverse_stft(spec, 16, 4, 30))
    zero = inverse_stft(np.zeros((5, 12, 1), complex), 8, 2, 16)
    assert zero.shape == (1, 16) and np.max(np.abs(zero)) == 0.0


def test_stft_errors_match_reference_texts():
    s = _signal(1, 256, 5)
    with pytest.raises(ConfigError, match="window_len must be a power of two, got 100"):
        forward_stft(s, 100, 25)
    with pytest.raises(ConfigError, match="hop must divide window_len"):
        forward_stft(s, 128, 24)
    with pytest.raises(ConfigError, match="empty signal"):
        forward_stft(np.zeros((1, 0)), 64, 16)
    with pytest.raises(ConfigError, match="shorter than one window"):
        forward_stft(_signal(1, 32, 5), 64, 16)
    with pytest.raises(ConfigError, match="bin count does not match"):
        inverse_stft(np.zeros((4, 3, 1), complex), 8, 2)
    with pytest.raises(ConfigError, match="inconsistent with frames"):
        inverse_stft(np.zeros((5, 3, 1), complex), 8, 2, 1000)


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_setup_from_signal_equals_host_spectrogram(precision):
    """ctf_setup_signal (STFT on the GPU straight into the estimator input)
    gives the same run as ctf_setup with the oracle's spectrogram."""
    B, M, n, window, hop, L, K = 2, 2, 3000, 256, 64, 3, 4
    sig = np.random.default_rng(12).standard_normal((B, M, n))
    spec = np.stack([O.forward_stft(sig[b], window, hop) for b in range(B)])  # [B, F, T, M]
    x = spec.astype(np.complex64) if precision == "f32" else spec
    a = Session(x, [L] * M, [K] * M, stack_taps=L, iterations=3, precision=precision, seed=3)
    a.iterate(3)
    ra = a.download_raw()
    a.close()
    b = Session(None, [L] * M, [K] * M, stack_taps=L, iterations=3, precision=precision, seed=3,
                signal=sig, window_len=window, hop=hop)
    assert b.shape == a.shape
    b.iterate(3)
    rb = b.download_raw()
    for u, v in zip(ra, rb):
        assert np.array_equal(u, v)
    b.close()


def test_setup_from_signal_sharded():
    """Each frequency shard transforms the signal and keeps its own bins."""
    B, M, n, window, hop, L, K = 1, 2, 2000, 128, 32, 2, 3
    sig = np.random.default_rng(2).standard_normal((B, M, n))
    s = Session(None, [L] * M, [K] * M, stack_taps=L, iterations=2, precision="f64", seed=1, signal=sig,
                window_len=window, hop=hop)
    s.iterate(2)
    W1, B1, V1, o1 = s.download_raw()
    s.close()
    lib = _lib.load()
    grp = lib.ctf_group_create(2)
    out = [None, None]

    def worker(r):
        t = Session(None, [L] * M, [K] * M, stack_taps=L, iterations=2, precision="f64", seed=1, signal=sig,
                    window_len=window, hop=hop, world_size=2, rank=r, group=grp)
        t.iterate(2)
        out[r] = (t.bin_range, t.download_raw())
        t.close()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    lib.ctf_group_destroy(grp)
    for (lo, hi), (W, Bf, V, obj) in out:
        assert np.max(np.abs(W[:, lo:hi] - W1[:, lo:hi])) <= 1e-12 * np.max(np.abs(W1))
        assert np.max(np.abs(V - V1)) <= 1e-12 * np.max(np.abs(V1))


def test_images_to_signal_matches_oracle_istft():
    """Back end of cmd_separate on the GPU: projection-back images -> iSTFT,
    all channels and the reference channel, vs the oracle's inverse STFT of
    the same images."""
    B, M, n, window, hop, L, K = 2, 2, 2500, 256, 64, 2, 3
    sig = np.random.default_rng(8).standard_normal((B, M, n))
    s = Session(None, [L] * M, [K] * M, stack_taps=L, iterations=3, precision="f64", seed=9, signal=sig,
                window_len=window, hop=hop)
    s.iterate(3)
    imgs = s.project_back(current_frame_only=True)  # [N, B, F, T, M]
    allc = s.images_to_signal()                      # [N, B, M, n]
    ref0 = s.images_to_signal(ref_channel=1)         # [N, B, n]
    assert allc.shape == (M, B, M, n) and ref0.shape == (M, B, n)
    for src in range(M):
        for b in range(B):
            expect = O.inverse_stft(imgs[src, b], window, hop, n)
            assert np.array_equal(allc[src, b], expect)
            assert np.array_equal(ref0[src, b], expect[1])
    # the source images add up to the mixture: the separated signals sum back to the input
    total = allc.sum(axis=0)
    assert np.max(np.abs(total - sig)) <= 1e-8 * np.max(np.abs(sig))
    with pytest.raises(ConfigError, match="out of range"):
        s.images_to_signal(ref_channel=M)
    s.close()


def test_cpp_mirror_stft_round_trip(tmp_path):
    """ctfmnmf::b200::forward_stft / inverse_stft / image_to_signal (the
    reference-shaped C++ API) on the GPU equal the oracle bit for bit."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    csrc = os.path.join(root, "paper_2510_02382_b200", "csrc")
    libdir = os.path.join(root, "paper_2510_02382_b200")
    s = _signal(2, 3000, 77)
    sf = tmp_path / "s.bin"
    s.tofile(sf)  # [channel][length] == TimeSignal.samples column-major
    src = tmp_path / "stft.cpp"
    src.write_text(f'''#include "ctfmnmf_b200.hpp"
#include <cstdio>
#include <fstream>
using namespace ctfmnmf::b200;
int main() {{
  TimeSignal sig; sig.sample_rate = 16000; sig.samples = RMatrix(3000, 2);
  std::ifstream in("{sf}", std::ios::binary);
  in.read(reinterpret_cast<char*>(sig.samples.data.data()), sig.samples.data.size() * 8);
  Spectrogram spec = forward_stft(sig, 512, 128);
  std::printf("%d %d %d %lld\\n", spec.bins, spec.frames, spec.channels, (long long)spec.original_length);
  for (const auto& v : spec.data) std::printf("%.17g %.17g\\n", v.real(), v.imag());
  TimeSignal back = inverse_stft(spec);
  for (double v : back.samples.data) std::printf("%.17g\\n", v);
  TimeSignal one = image_to_signal(MixtureSpectrogram::from_spectrogram(spec), spec, 1);
  for (double v : one.samples.data) std::printf("%.17g\\n", v);
  try {{ forward_stft(sig, 100, 25); return 3; }} catch (const ConfigError&) {{}}
  try {{ image_to_signal(MixtureSpectrogram::from_spectrogram(spec), spec, 2); return 4; }} catch (const ConfigError&) {{}}
  return 0;
}}''')
    exe = tmp_path / "stft"
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{csrc}", "-o", str(exe), str(src), f"-L{libdir}", "-lctfiss",
                    f"-Wl,-rpath,{libdir}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    bins, frames, chans, olen = map(int, out[0].split())
    ref = O.forward_stft(s, 512, 128)
    assert (bins, frames, chans, olen) == (*ref.shape, 3000)
    nspec = bins * frames * chans
    spec = np.array([complex(*map(float, l.split())) for l in out[1:1 + nspec]]).reshape(ref.shape)
    assert np.array_equal(spec, ref)
    back = np.array([float(v) for v in out[1 + nspec:1 + nspec + 6000]]).reshape(2, 3000)
    assert np.array_equal(back, O.inverse_stft(ref, 512, 128, 3000))
    one = np.array([float(v) for v in out[1 + nspec + 6000:1 + nspec + 9000]])
    assert np.array_equal(one, back[1])


def test_setup_from_spec_files_and_factor_file(tmp_path):
    """`.spec` containers straight into the estimator (ctf_setup_spectrogram_files,
    the reference's separate input), equal to a setup from the same complex64
    array; the converged factors written as a `.nmf` container read back."""
    from paper_2510_02382_b200 import read_factors, write_factors, write_spectrogram
    B, M, n, window, hop, L, K = 2, 2, 2000, 128, 32, 2, 3
    sig = np.random.default_rng(21).standard_normal((B, M, n))
    specs = [O.forward_stft(sig[b], window, hop) for b in range(B)]
    paths = []
    for b, sp in enumerate(specs):
        paths.append(str(tmp_path / f"m{b}.spec"))
        write_spectrogram(paths[-1], sp, window, hop, 16000, n)
    x = np.stack(specs).astype(np.complex64)
    a = Session(x, [L] * M, [K] * M, stack_taps=L, iterations=3, precision="f32", seed=4)
    a.iterate(3)
    ra = a.download_raw()
    a.close()
    s = Session(None, [L] * M, [K] * M, stack_taps=L, iterations=3, precision="f32", seed=4, spec_files=paths)
    assert s.spec_header["window_len"] == window and s.signal_length == n
    s.iterate(3)
    rb = s.download_raw()
    for u, v in zip(ra, rb):
        assert np.array_equal(u, v)
    dem, bases, acts, obj = s.download()[0]
    write_factors(str(tmp_path / "f.nmf"), bases, acts, float(s.psd_floor()[0]))
    B2, V2, fl = read_factors(str(tmp_path / "f.nmf"))
    assert all(np.array_equal(p, q) for p, q in zip(B2 + V2, bases + acts))
    s.close()


def test_separate_pipeline_end_to_end_vs_oracle():
    """cmd_separate's whole path on the GPU (ctfmnmf_main.cpp:179-240):
    signal -> STFT -> ISS estimator (stacked CTF) -> projection-back images ->
    inverse STFT of the reference channel, against the same chain on the CPU
    oracle (forward_stft, run, reconstruct_images, inverse_stft): fp64 1e-9."""
    M, L, K, n, window, hop, iters, seed = 2, 3, 3, 3000, 128, 32, 6, 5
    sig = np.random.default_rng(99).standard_normal((1, M, n))
    s = Session(None, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision="f64", seed=seed, signal=sig,
                window_len=window, hop=hop)
    s.iterate(iters)
    got = s.images_to_signal(ref_channel=0)  # [N, 1, n]
    s.close()
    spec = O.forward_stft(sig[0], window, hop)           # (F, T, M)
    xst = O.stack_observation(spec, L)                    # (F, T, D)
    cfg = O.config([L] * M, [K] * M, iterations=iters, seed=seed)
    r = O.run(cfg, xst)
    imgs = O.reconstruct_images(cfg, r["W"], xst)         # [N, F, T, D]
    for src in range(M):
        mic_img = imgs[src][:, :, [m * L for m in range(M)]]  # current-frame channels (l = 0)
        want = O.inverse_stft(mic_img, window, hop, n)[0]
        assert np.max(np.abs(got[src, 0] - want)) <= 1e-9 * np.max(np.abs(want))
