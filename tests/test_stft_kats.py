"""Known-answer / property pins of the STFT front and back end
(proj/tests/test_stft.cpp) re-expressed against the CPU oracle restatement of
proj/src/fft.cpp and proj/src/stft.cpp. CPU only; the GPU kernels are checked
against this oracle in test_gpu_stft.py."""
import numpy as np
import pytest

from oracle import oracle as O


def _signal(length, channels, seed):
    return np.random.default_rng(seed).standard_normal((channels, length))


def _max_rel(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(a))


def test_fft_round_trip_and_known_transform():  # test_stft.cpp:33-52
    g = np.random.default_rng(1)
    data = g.standard_normal(64) + 1j * g.standard_normal(64)
    back = O.fft(O.fft(data), inverse=True)
    assert np.max(np.abs(back - data)) < 1e-12
    tone = np.exp(2j * np.pi * 3.0 * np.arange(16) / 16.0)
    f = O.fft(tone)
    assert abs(f[3] - 16.0) < 1e-10
    assert np.all(np.abs(np.delete(f, 3)) < 1e-10)
    # the restated radix-2 transform is a DFT (numpy as an independent check)
    assert np.max(np.abs(O.fft(data) - np.fft.fft(data))) < 1e-12 * np.max(np.abs(np.fft.fft(data)))
    assert np.max(np.abs(O.fft(data, inverse=True) - np.fft.ifft(data))) < 1e-13


def test_dc_signal_concentrates_into_window_support():  # :54-70
    spec = O.forward_stft(np.ones((1, 64)), 8, 2)
    assert spec.shape[0] == 5
    for j in range(4, spec.shape[1] - 4):
        assert abs(spec[0, j, 0] - 4.0) < 1e-12
        assert abs(spec[1, j, 0] + 2.0) < 1e-12
        assert np.all(np.abs(spec[2:, j, 0]) < 1e-12)


def test_frame_geometry_16k_1024_hop256():  # :72-80
    n = 8 * 16000
    assert O.stft_frames(n, 256) == 1 + (n + 255) // 256
    spec = O.forward_stft(_signal(n, 1, 7), 1024, 256)
    assert spec.shape[0] == 513 and 500 <= spec.shape[1] <= 503


def test_round_trip_below_minus_100_db():  # :82-94
    s = _signal(4096, 2, 21)
    back = O.inverse_stft(O.forward_stft(s, 1024, 256), 1024, 256, 4096)
    assert back.shape == s.shape
    for c in range(2):
        err = _max_rel(s[c], back[c])
        assert err < 1e-10 and 20 * np.log10(err) < -100


@pytest.mark.parametrize("hop", [64, 128, 256])
def test_round_trip_other_cola_hops(hop):  # :96-103
    s = _signal(2000, 1, 3)
    back = O.inverse_stft(O.forward_stft(s, 512, hop), 512, hop, 2000)
    assert _max_rel(s[0], back[0]) < 1e-10


def test_zero_spectrogram_inverts_to_silence():  # :105-116
    out = O.inverse_stft(np.zeros((5, 12, 1), complex), 8, 2, 16)
    assert out.shape == (1, 16) and np.max(np.abs(out)) == 0.0


def test_single_bin_synthesizes_windowed_sinusoid():  # :118-151
    window, hop, frames, i0, j0, amp = 16, 4, 10, 3, 4, 0.7 - 0.4j
    spec = np.zeros((window // 2 + 1, frames, 1), complex)
    spec[i0, j0, 0] = amp
    out = O.inverse_stft(spec, window, hop, 24)
    w = O.hann_window(window)
    overlap = np.zeros((frames - 1) * hop + window)
    for j in range(frames):
        overlap[j * hop:j * hop + window] += w * w
    for p in range(out.shape[1]):
        padded = p + window // 2
        t = padded - j0 * hop
        expected = 0.0
        if 0 <= t < window:
            expected = 2.0 * (amp * np.exp(2j * np.pi * i0 * t / window)).real / window * w[t] / overlap[padded]
        assert abs(out[0, p] - expected) < 1e-12


def test_per_frame_parseval():  # :153-176
    s = _signal(600, 1, 11)
    window, hop = 128, 32
    spec = O.forward_stft(s, window, hop)
    w = O.hann_window(window)
    for j in (4, 7, 10):
        spectral = abs(spec[0, j, 0]) ** 2 + abs(spec[-1, j, 0]) ** 2 + 2 * np.sum(np.abs(spec[1:-1, j, 0]) ** 2)
        spectral /= window
        p = j * hop + np.arange(window) - window // 2
        assert p.min() >= 0 and p.max() < s.shape[1]
        time_energy = np.sum((s[0, p] * w) ** 2)
        assert abs(spectral - time_energy) < 1e-8 * time_energy


def test_hann_is_periodic():  # stft.cpp:14-19
    w = O.hann_window(8)
    assert np.allclose(w, 0.5 - 0.5 * np.cos(2 * np.pi * np.arange(8) / 8), rtol=0, atol=1e-16)


def test_reflect_padding_edges():  # stft.cpp:25-42: frame 0 sees x[half..1] reflected, no edge repeat
    n, window, hop = 40, 8, 4
    s = np.arange(1.0, n + 1.0)[None]
    spec = O.forward_stft(s, window, hop)
    w = O.hann_window(window)
    frame0 = np.concatenate([s[0, 4:0:-1], s[0, :4]]) * w     # padded[0..7] = x4 x3 x2 x1 x0 .. x3
    assert np.max(np.abs(spec[:, 0, 0] - np.fft.rfft(frame0))) < 1e-12
    last = spec.shape[1] - 1                                    # tail reflects x[n-2], x[n-3], ...
    padded_len = last * hop + window
    tail = np.concatenate([s[0], s[0, n - 2::-1]])[:padded_len - window // 2]
    padded = np.concatenate([s[0, 4:0:-1], tail, np.zeros(max(0, padded_len - 4 - tail.size))])
    fr = padded[last * hop:last * hop + window] * w
    assert np.max(np.abs(spec[:, last, 0] - np.fft.rfft(fr))) < 1e-12


def test_invalid_arguments_rejected():  # :178-187
    s = _signal(256, 1, 5)
    for wl, hop in ((100, 25), (128, 24)):
        with pytest.raises(O.OracleError) as e:
            O.forward_stft(s, wl, hop)
        assert e.value.code == 2
    with pytest.raises(O.OracleError, match="empty signal"):
        O.forward_stft(np.zeros((1, 0)), 64, 16)
    with pytest.raises(O.OracleError, match="shorter than one window"):
        O.forward_stft(_signal(32, 1, 5), 64, 16)
    with pytest.raises(O.OracleError, match="bin count"):
        O.inverse_stft(np.zeros((4, 3, 1), complex), 8, 2)
    with pytest.raises(O.OracleError, match="inconsistent"):
        O.inverse_stft(np.zeros((5, 3, 1), complex), 8, 2, 1000)
