"""The GPU-backed command-line front end (paper_2510_02382_b200/ctfmnmf_b200,
csrc/ctfmnmf_cli.cpp), the reference's `separate` / `bench`
(proj/tools/ctfmnmf_main.cpp:179-364): flags, config file, outputs
(srcN.wav, trace.csv, manifest.json, bench.csv) and exit codes (2 config,
3 I/O, 4 numerical degeneracy)."""
import json
import os
import struct
import subprocess

import numpy as np
import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2510_02382_b200", "ctfmnmf_b200")


def cli(*args, cwd=None):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600, cwd=cwd)


def write_wav_f32(path, samples, rate=16000):
    """samples: (length, channels) -> 32-bit float RIFF WAV (independent writer)."""
    n, ch = samples.shape
    body = np.ascontiguousarray(samples, dtype="<f4").tobytes()
    hdr = b"RIFF" + struct.pack("<I", 36 + len(body)) + b"WAVEfmt " + struct.pack(
        "<IHHIIHH", 16, 3, ch, rate, rate * ch * 4, ch * 4, 32) + b"data" + struct.pack("<I", len(body))
    with open(path, "wb") as f:
        f.write(hdr + body)


def read_wav_f32(path):
    with open(path, "rb") as f:
        d = f.read()
    ch = struct.unpack("<H", d[22:24])[0]
    i = d.index(b"data")
    n = struct.unpack("<I", d[i + 4:i + 8])[0]
    return np.frombuffer(d[i + 8:i + 8 + n], dtype="<f4").reshape(-1, ch)


def test_cli_version_and_usage_errors():
    r = cli("--version")
    assert r.returncode == 0 and r.stdout.strip()
    assert cli().returncode == 2
    assert cli("simulate").returncode == 2          # out of scope: unknown subcommand
    assert cli("separate").returncode == 2          # missing mixture
    assert cli("separate", "x.wav", "--rule", "xx").returncode == 2


@pytest.mark.gpu
def test_cli_separate_wav_matches_reference_pipeline(tmp_path):
    """separate on a 4-channel WAV: GPU STFT -> run (fp64) -> projection-back
    -> inverse STFT; the manifest's final objective equals the oracle's run
    on the oracle's STFT of the same samples (1e-9), and every output exists."""
    g = np.random.default_rng(3)
    n, ch = 6000, 4
    sig = (g.standard_normal((n, 2)) @ g.standard_normal((2, ch)) + 0.05 * g.standard_normal((n, ch))) * 0.1
    sig = sig.astype(np.float32).astype(np.float64)  # what the float WAV stores
    wav = tmp_path / "mix.wav"
    write_wav_f32(wav, sig)
    cfg = tmp_path / "cfg.txt"
    cfg.write_text("# test config\nn_sources = 2\nn_channels = 4\ntaps = 2,2\nbases = 3,3\niters = 6\n"
                   "window = 256\nhop = 64\nseed = 7\n")
    out = tmp_path / "out"
    r = cli("separate", str(wav), "--config", str(cfg), "--out", str(out), "--iters", "5")
    assert r.returncode == 0, r.stderr
    m = json.loads((out / "manifest.json").read_text())
    assert m["command"] == "separate" and m["errors"] == [] and m["config"]["iters"] == 5
    trace = (out / "trace.csv").read_text().strip().split("\n")
    assert trace[0].startswith("iter,objective") and len(trace) == 6
    spec = O.forward_stft(sig.T, 256, 64)  # (bins, frames, channels)
    ref = O.run(O.config([2, 2], [3, 3], iterations=5, seed=7), np.ascontiguousarray(spec))
    assert abs(m["final_objective"] - ref["objective"][-1]) <= 1e-9 * abs(ref["objective"][-1])
    for k in (1, 2):
        s = read_wav_f32(out / f"src{k}.wav")
        assert s.shape == (n, ch) and np.all(np.isfinite(s))
    # the two source images partition the mixture (wiener.cpp: collapsed Wiener form)
    tot = read_wav_f32(out / "src1.wav").astype(np.float64) + read_wav_f32(out / "src2.wav")
    assert np.max(np.abs(tot - sig)) <= 1e-4 * np.max(np.abs(sig))
    r1 = cli("separate", str(wav), "--config", str(cfg), "--out", str(tmp_path / "o1"), "--ref-channel", "0")
    assert r1.returncode == 0 and read_wav_f32(tmp_path / "o1" / "src1.wav").shape == (n, 1)


@pytest.mark.gpu
def test_cli_separate_errors_and_exit_codes(tmp_path):
    g = np.random.default_rng(4)
    wav = tmp_path / "mix3.wav"
    write_wav_f32(wav, g.standard_normal((3000, 3)) * 0.1)
    r = cli("separate", str(wav), "--out", str(tmp_path / "o"))  # default config expects 4 channels
    assert r.returncode == 2 and "channels" in r.stderr
    r = cli("separate", str(tmp_path / "missing.wav"), "--out", str(tmp_path / "o"))
    assert r.returncode == 3
    bad = tmp_path / "bad.txt"
    bad.write_text("nokey\n")
    assert cli("separate", str(wav), "--config", str(bad)).returncode == 2
    silent = tmp_path / "silent.wav"
    write_wav_f32(silent, np.zeros((3000, 4)))
    r = cli("separate", str(silent), "--out", str(tmp_path / "o2"))
    assert r.returncode == 2  # zero mixture: ConfigError (estimator.cpp:520-529)


@pytest.mark.gpu
def test_cli_bench_writes_csv(tmp_path):
    cfg = tmp_path / "cfg.txt"
    cfg.write_text("iters = 3\nwindow = 64\nframes = 40\ntrials = 2\nbases = 2,2\n")
    r = cli("bench", "--config", str(cfg), "--channels", "4,6", "--out", str(tmp_path))
    assert r.returncode == 0, r.stderr
    rows = (tmp_path / "bench.csv").read_text().strip().split("\n")
    assert rows[0] == "M,rule,total_ms,demix_ms,mu_ms,seed" and len(rows) == 1 + 2 * 2 * 2
    assert {tuple(x.split(",")[:2]) for x in rows[1:]} == {("4", "ip"), ("4", "iss"), ("6", "ip"), ("6", "iss")}
    m = json.loads((tmp_path / "manifest.json").read_text())
    assert m["command"] == "bench" and m["channels"] == [4, 6]
    assert cli("bench", "--channels", "3", "--out", str(tmp_path)).returncode == 2
