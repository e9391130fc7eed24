"""Binary containers: the `.spec` spectrogram and `.nmf`
factor files of proj/src/container.cpp, through the C ABI (host code, no GPU).
The byte layout is checked against an independent struct-based encoding of
container.hpp:1-10; GPU setup from files is in test_gpu_stft.py."""
import struct

import numpy as np
import pytest

from paper_2510_02382_b200 import IoError, read_factors, read_spectrogram, write_factors, write_spectrogram


def _spec_bytes(spec, window, hop, rate, n):
    """container.hpp:4-6 restated: magic, u32 x6, u64, complex64 bin-major body."""
    b, f, c = spec.shape
    head = b"CTFSPG1\0" + struct.pack("<6IQ", b, f, c, window, hop, rate, n)
    return head + np.ascontiguousarray(spec, np.complex64).tobytes()


def test_spectrogram_round_trip_and_byte_layout(tmp_path):
    g = np.random.default_rng(3)
    spec = g.standard_normal((9, 7, 3)) + 1j * g.standard_normal((9, 7, 3))
    path = tmp_path / "x.spec"
    write_spectrogram(str(path), spec, 16, 4, 16000, 24)
    assert path.read_bytes() == _spec_bytes(spec, 16, 4, 16000, 24)
    hdr, back = read_spectrogram(str(path))
    assert hdr == {"bins": 9, "frames": 7, "channels": 3, "window_len": 16, "hop": 4, "sample_rate": 16000,
                   "original_length": 24}
    assert back.dtype == np.complex128
    assert np.array_equal(back, spec.astype(np.complex64).astype(np.complex128))  # float32 quantised
    _, b32 = read_spectrogram(str(path), precision="f32")
    assert b32.dtype == np.complex64 and np.array_equal(b32, spec.astype(np.complex64))
    # complex64 input is written byte for byte
    write_spectrogram(str(path), spec.astype(np.complex64), 16, 4, 16000, 24)
    assert path.read_bytes() == _spec_bytes(spec, 16, 4, 16000, 24)


def test_factors_round_trip_and_byte_layout(tmp_path):
    g = np.random.default_rng(4)
    F, T, K = 5, 6, [2, 3]
    bases = [g.random((F, k)) for k in K]
    acts = [g.random((k, T)) for k in K]
    path = tmp_path / "f.nmf"
    write_factors(str(path), bases, acts, 1.5e-12)
    want = b"CTFNMF1\0" + struct.pack("<3I", 2, F, T) + struct.pack("<2I", *K) + struct.pack("<d", 1.5e-12)
    for b, v in zip(bases, acts):  # container.hpp:9-10: per source B row-major then V row-major
        want += np.ascontiguousarray(b).tobytes() + np.ascontiguousarray(v).tobytes()
    assert path.read_bytes() == want
    B2, V2, fl = read_factors(str(path))
    assert fl == 1.5e-12
    for a, b in zip(B2 + V2, bases + acts):
        assert np.array_equal(a, b)


def test_container_errors_match_reference_texts(tmp_path):
    with pytest.raises(IoError, match="cannot open file"):
        read_spectrogram(str(tmp_path / "missing.spec"))
    bad = tmp_path / "bad.spec"
    bad.write_bytes(b"CTFNMF1\0" + b"\0" * 32)
    with pytest.raises(IoError, match="bad or mismatched container magic"):
        read_spectrogram(str(bad))
    spec = np.ones((4, 3, 2), complex)
    path = tmp_path / "t.spec"
    write_spectrogram(str(path), spec, 6, 2, 100, 4)
    path.write_bytes(path.read_bytes()[:-5])
    with pytest.raises(IoError, match="truncated spectrogram container"):
        read_spectrogram(str(path))
    with pytest.raises(IoError, match="cannot create file"):
        write_spectrogram(str(tmp_path / "no" / "dir.spec"), spec, 6, 2, 100, 4)
    with pytest.raises(IoError, match="bad or mismatched container magic"):
        read_factors(str(path))  # a spectrogram is not a factor container
