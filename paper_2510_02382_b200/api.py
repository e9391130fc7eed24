"""Python mirror of the reference estimator API over the C ABI.

Names, argument meaning and errors follow /root/reference/proj:
  CtfConfig            model.hpp:21-35 (validate: model.cpp:32-50)
  run(config, x)       estimator.hpp:122-123 / estimator.cpp:513-657
  reconstruct_images   wiener.hpp:18-20 / wiener.cpp:11-49
  ConfigError, IoError, DegeneracyError{iteration, bin, row}   errors.hpp:11-35
The array forms are numpy: a MixtureSpectrogram is a complex array of shape
(F, channels, T) (one channels x frames matrix per bin, model.hpp:55-66),
demixing matrices are (F, R, D), B_n is (F, K_n), V_n is (K_n, T).

``Session`` is the batched, device-resident form used by the benchmark: a
batch of independent mixtures in the reference Spectrogram layout
[B][F][T][M], optionally stacked on the GPU into the M*L-channel CTF
observation (BASELINE (a)).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L


class ConfigError(Exception):
    """Invalid configuration (errors.hpp:19-22). CLI exit 2."""


class IoError(Exception):
    """File/format failure (errors.hpp:24-27). CLI exit 3."""


class DegeneracyError(Exception):
    """Numerical degeneracy (errors.hpp:29-35). CLI exit 4."""

    def __init__(self, msg, iteration=-1, bin=-1, row=-1, mixture=-1, kind=0):
        super().__init__(msg)
        self.iteration, self.bin, self.row, self.mixture, self.kind = iteration, bin, row, mixture, kind


class DeviceError(RuntimeError):
    """CUDA / runtime failure, or a shape outside the compiled kernel set."""


def _raise(rc: int, err: L.CtfErr):
    msg = err.msg.decode(errors="replace")
    if rc == L.CTF_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == L.CTF_ERR_IO:
        raise IoError(msg)
    if rc == L.CTF_ERR_DEGENERACY:
        raise DegeneracyError(msg, err.iteration, err.bin, err.row, err.mixture, err.kind)
    raise DeviceError(f"[{rc}] {msg}")


def _check(rc: int, err: L.CtfErr):
    if rc != L.CTF_OK:
        _raise(rc, err)


@dataclass
class CtfConfig:
    """model.hpp:21-35."""
    num_sources: int = 2
    num_channels: int = 4
    taps_per_source: List[int] = field(default_factory=list)
    bases_per_source: List[int] = field(default_factory=list)
    iterations: int = 100
    update_rule: str = "iss"
    psd_floor: float = 1e-10
    seed: int = 0
    threads: int = 1

    def total_taps(self) -> int:
        return int(sum(self.taps_per_source))

    def row_offset(self, source: int) -> int:
        return int(sum(self.taps_per_source[:source]))

    def validate(self):
        """model.cpp:32-50 (same messages)."""
        if self.num_sources < 1:
            raise ConfigError("n_sources must be >= 1")
        if self.num_channels < 1:
            raise ConfigError("n_channels must be >= 1")
        if len(self.taps_per_source) != self.num_sources:
            raise ConfigError("taps list must have one entry per source")
        if len(self.bases_per_source) != self.num_sources:
            raise ConfigError("bases list must have one entry per source")
        if any(l < 1 for l in self.taps_per_source):
            raise ConfigError("every tap count must be >= 1")
        if any(k < 1 for k in self.bases_per_source):
            raise ConfigError("every basis count must be >= 1")
        if self.total_taps() != self.num_channels:
            raise ConfigError(f"sum of taps ({self.total_taps()}) must equal n_channels ({self.num_channels}): "
                              "the demixing system must be square")
        if self.iterations < 0:
            raise ConfigError("iters must be >= 0")
        if not self.psd_floor > 0.0:
            raise ConfigError("floor must be > 0")
        if self.threads < 1:
            raise ConfigError("threads must be >= 1")
        if self.update_rule not in ("iss", "ISS", "ip", "IP"):
            raise ConfigError(f"unknown update rule '{self.update_rule}' (expected ip or iss)")


@dataclass
class CheckOptions:
    """estimator.hpp:45-48: exact per-update recomputations (slow; verification only)."""
    det_lemma: bool = False
    normalization: bool = False

    def flags(self) -> int:
        return (L.CTF_CHECK_DET_LEMMA if self.det_lemma else 0) | \
            (L.CTF_CHECK_NORMALIZATION if self.normalization else 0)


@dataclass
class OptimizationTrace:
    """estimator.hpp:25-40."""
    objective: List[float]
    demix_ms: List[float]
    mu_ms: List[float]
    rescale_ms: List[float]
    max_det_lemma_error: float = 0.0
    max_normalization_error: float = 0.0
    checked_updates: int = 0

    def to_csv(self) -> str:
        out = ["iter,objective,t_demix_ms,t_mu_ms,t_rescale_ms"]
        for t, o in enumerate(self.objective):
            out.append(f"{t + 1},{o:.12g},{self.demix_ms[t]:.12g},{self.mu_ms[t]:.12g},{self.rescale_ms[t]:.12g}")
        return "\n".join(out) + "\n"


@dataclass
class SeparationResult:
    """estimator.hpp:50-54 (factors flattened into bases/activations/floor)."""
    demixing: np.ndarray            # (F, R, D) complex128
    bases: List[np.ndarray]         # B_n (F, K_n)
    activations: List[np.ndarray]   # V_n (K_n, T)
    floor: float
    trace: OptimizationTrace


def _problem(num_mixtures, F, T, num_mics, stack_taps, taps, bases, iterations, precision, x_precision,
             psd_floor, seed, threads=1, rule=L.CTF_RULE_ISS, checks=0) -> L.CtfProblem:
    p = L.CtfProblem()
    p.num_mixtures, p.num_bins, p.num_frames = num_mixtures, F, T
    p.num_mics, p.stack_taps, p.num_sources = num_mics, stack_taps, len(taps)
    if len(taps) > L.CTF_MAX_SOURCES or len(bases) > L.CTF_MAX_SOURCES:
        raise ConfigError("too many sources")
    for n, (l, k) in enumerate(zip(taps, bases)):
        p.taps_per_source[n] = l
        p.bases_per_source[n] = k
    p.iterations, p.update_rule = iterations, rule
    p.precision = L.CTF_F32 if precision in ("f32", "float32") else L.CTF_F64
    p.x_precision = L.CTF_F32 if x_precision in ("f32", "float32", "complex64") else L.CTF_F64
    p.psd_floor, p.seed, p.threads, p.checks = psd_floor, seed, threads, checks
    return p


class Session:
    """Device-resident batch of mixtures on one GPU (or one frequency shard).

    x: complex array [B, F, T, M] (reference Spectrogram layout per mixture),
    complex128 or complex64. With stack_taps = L > 1, D = M*L and the stacked
    observation is built inside the kernels; otherwise x already holds the
    D-channel observation.
    """

    def __init__(self, x: np.ndarray, taps, bases, *, stack_taps=1, iterations=100, precision="f64",
                 psd_floor=1e-10, seed=0, device=0, world_size=1, rank=0, comm_id: Optional[bytes] = None,
                 group=None, checks: int = 0, signal: Optional[np.ndarray] = None, window_len: int = 0,
                 hop: int = 0, update_rule: str = "iss", spec_files: Optional[List[str]] = None):
        """x: [B, F, T, M] spectrogram batch, or x=None with signal = [B, M, length]
        float64 time-domain mixtures (the STFT runs on the GPU, ctf_setup_signal)."""
        self.lib = L.load()
        if spec_files is not None:  # one .spec container per mixture (ctf_setup_spectrogram_files)
            h, err = L.CtfSpecHeader(), L.CtfErr()
            _check(self.lib.ctf_read_spectrogram(spec_files[0].encode(), C.byref(h), None, L.CTF_F64, C.byref(err)),
                   err)
            self.spec_header = {k: getattr(h, k) for k, _ in L.CtfSpecHeader._fields_}
            B, F, T, M = len(spec_files), h.bins, h.frames, h.channels
            xprec = "f32"
        elif signal is not None:
            signal = np.ascontiguousarray(signal, dtype=np.float64)
            if signal.ndim != 3:
                raise ConfigError("signal must have shape [B, M, length]")
            if hop <= 0:
                raise ConfigError("forward_stft: hop must divide window_len")
            B, M, n = signal.shape
            F, T = window_len // 2 + 1, int(self.lib.ctf_stft_frames(n, hop))
            xprec = precision
        else:
            if x.ndim != 4:
                raise ConfigError("x must have shape [B, F, T, M]")
            xprec = "f32" if x.dtype == np.complex64 else "f64"
            x = np.ascontiguousarray(x, dtype=np.complex64 if xprec == "f32" else np.complex128)
            B, F, T, M = x.shape
        self.shape = (B, F, T, M)
        self.taps, self.bases = list(taps), list(bases)
        self.stack_taps = stack_taps
        self.D = M * stack_taps
        self.R = sum(self.taps)
        self.precision = precision
        self._ctx = C.c_void_p()
        err = L.CtfErr()
        _check(self.lib.ctf_open(device, C.byref(self._ctx), C.byref(err)), err)
        if group is not None:  # in-process exchange group (testing the sharded path)
            _check(self.lib.ctf_comm_init_group(self._ctx, group, rank, C.byref(err)), err)
        elif world_size > 1 or comm_id is not None:  # NCCL (a single-rank comm only under CTF_NCCL_SINGLE_RANK=1)
            buf = (C.c_uint8 * 128).from_buffer_copy(comm_id)
            _check(self.lib.ctf_comm_init(self._ctx, world_size, rank, buf, C.byref(err)), err)
        self.world_size, self.rank = world_size, rank
        lo, hi = C.c_int(), C.c_int()
        self.lib.ctf_shard_range(F, world_size, rank, C.byref(lo), C.byref(hi))
        self.bin_range = (lo.value, hi.value)
        self.problem = _problem(B, F, T, M, stack_taps, self.taps, self.bases, iterations, precision, xprec,
                                psd_floor, seed, checks=checks,
                                rule=L.CTF_RULE_IP if update_rule.lower() == "ip" else L.CTF_RULE_ISS)
        if spec_files is not None:
            arr = (C.c_char_p * len(spec_files))(*[f.encode() for f in spec_files])
            self.window_len, self.hop = self.spec_header["window_len"], self.spec_header["hop"]
            self.signal_length = self.spec_header["original_length"]
            _check(self.lib.ctf_setup_spectrogram_files(self._ctx, C.byref(self.problem), arr, len(spec_files), None,
                                                        C.byref(err)), err)
        elif signal is not None:
            self.signal_length, self.window_len, self.hop = signal.shape[2], window_len, hop
            _check(self.lib.ctf_setup_signal(self._ctx, C.byref(self.problem), L.dptr(signal), signal.shape[2],
                                             window_len, hop, C.byref(err)), err)
        else:
            _check(self.lib.ctf_setup(self._ctx, C.byref(self.problem), L.vptr(x), C.byref(err)), err)

    # -- state -----------------------------------------------------------
    def iterate(self, n: int):
        err = L.CtfErr()
        _check(self.lib.ctf_iterate(self._ctx, n, C.byref(err)), err)

    def iterate_async(self, n: int):
        err = L.CtfErr()
        _check(self.lib.ctf_iterate_async(self._ctx, n, C.byref(err)), err)

    def finalize(self):
        err = L.CtfErr()
        _check(self.lib.ctf_finalize(self._ctx, C.byref(err)), err)

    @property
    def iterations_done(self) -> int:
        return self.lib.ctf_iterations_done(self._ctx)

    def set_state(self, W=None, B=None, V=None):
        """W: [B, F, R*D*2] doubles in column-major per bin (see download)."""
        err = L.CtfErr()
        arrs = [None if a is None else np.ascontiguousarray(a, dtype=np.float64) for a in (W, B, V)]
        _check(self.lib.ctf_set_state(self._ctx, *[L.dptr(a) for a in arrs], C.byref(err)), err)

    def download_raw(self):
        """Flat arrays in the C-ABI layouts: W [B][F][R x D col-major] complex,
        B [B][sum_n F*K_n], V [B][sum_n K_n*T], objective [B][iters]."""
        B, F, T, M = self.shape
        SK = sum(self.bases)
        W = np.zeros((B, F, self.R * self.D), np.complex128)
        Bf = np.zeros((B, F * SK))
        V = np.zeros((B, SK * T))
        it = self.iterations_done
        obj = np.zeros((B, max(it, 1)))
        err = L.CtfErr()
        _check(self.lib.ctf_download(self._ctx, W.ctypes.data_as(L._D), L.dptr(Bf), L.dptr(V), L.dptr(obj),
                                     C.byref(err)), err)
        return W, Bf, V, obj[:, :it]

    def download(self):
        """Per mixture: demixing (F, R, D), bases [(F, K_n)], activations [(K_n, T)], objective (iters,)."""
        B, F, T, M = self.shape
        W, Bf, V, obj = self.download_raw()
        out = []
        for b in range(B):
            dem = W[b].reshape(F, self.D, self.R).transpose(0, 2, 1)
            bases, acts, ob, ov = [], [], 0, 0
            for K in self.bases:
                bases.append(Bf[b, ob:ob + F * K].reshape(K, F).T.copy())
                acts.append(V[b, ov:ov + K * T].reshape(T, K).T.copy())
                ob += F * K
                ov += K * T
            out.append((dem, bases, acts, obj[b]))
        return out

    def describe(self) -> str:
        buf = C.create_string_buffer(1024)
        self.lib.ctf_describe(self._ctx, buf, 1024)
        return buf.value.decode()

    def psd_floor(self) -> np.ndarray:
        out = np.zeros(self.shape[0])
        self.lib.ctf_psd_floor(self._ctx, L.dptr(out))
        return out

    def trace_ms(self):
        n = self.iterations_done
        a, b, c = np.zeros(max(n, 1)), np.zeros(max(n, 1)), np.zeros(max(n, 1))
        self.lib.ctf_trace_ms(self._ctx, L.dptr(a), L.dptr(b), L.dptr(c))
        return a[:n], b[:n], c[:n]

    def check_stats(self):
        """CheckOptions results per mixture (estimator.hpp:31-34):
        (max_det_lemma_error [B], max_normalization_error [B], checked_updates [B])."""
        B = self.shape[0]
        d, n = np.zeros(B), np.zeros(B)
        k = (C.c_int64 * B)()
        if self.lib.ctf_check_stats(self._ctx, L.dptr(d), L.dptr(n), k) != 0:
            raise DeviceError("ctf_check_stats failed")
        return d, n, np.array(list(k), np.int64)

    def timing(self) -> L.CtfTiming:
        t = L.CtfTiming()
        self.lib.ctf_get_timing(self._ctx, C.byref(t))
        return t

    def reset_timing(self):
        self.lib.ctf_reset_timing(self._ctx)

    def stream_ptr(self) -> int:
        return self.lib.ctf_stream(self._ctx) or 0

    def project_back(self, current_frame_only=False) -> np.ndarray:
        """images [N, B, F, T, Dout] complex (wiener.cpp:11-49)."""
        B, F, T, M = self.shape
        dout = M if current_frame_only else self.D
        img = np.zeros((len(self.taps), B, F, T, dout), np.complex128)
        err = L.CtfErr()
        mode = L.CTF_IMAGES_CURRENT_FRAME if current_frame_only else L.CTF_IMAGES_FULL
        _check(self.lib.ctf_project_back(self._ctx, mode, img.ctypes.data_as(L._D), C.byref(err)), err)
        return img

    def images_to_signal(self, ref_channel: int = -1, window_len: int = 0, hop: int = 0,
                         original_length: int = 0) -> np.ndarray:
        """Projection-back + inverse STFT on the GPU (cmd_separate's back end,
        wiener.cpp:51-64): [N, B, M, length] (ref_channel < 0) or [N, B, length]."""
        window_len = window_len or getattr(self, "window_len", 0)
        hop = hop or getattr(self, "hop", 0)
        original_length = original_length or getattr(self, "signal_length", 0)
        n, err = C.c_int64(), L.CtfErr()
        _check(self.lib.ctf_images_to_signal(self._ctx, ref_channel, window_len, hop, original_length, None,
                                             C.byref(n), C.byref(err)), err)
        B, F, T, M = self.shape
        shape = (len(self.taps), B, M, n.value) if ref_channel < 0 else (len(self.taps), B, n.value)
        out = np.zeros(shape)
        _check(self.lib.ctf_images_to_signal(self._ctx, ref_channel, window_len, hop, original_length, L.dptr(out),
                                             C.byref(n), C.byref(err)), err)
        return out

    def close(self):
        if self._ctx:
            self.lib.ctf_close(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_stft_ctx = {}


def _device_ctx(device: int):
    """A context per device for the stateless STFT entry points."""
    if device not in _stft_ctx:
        lib, ctx, err = L.load(), C.c_void_p(), L.CtfErr()
        _check(lib.ctf_open(device, C.byref(ctx), C.byref(err)), err)
        _stft_ctx[device] = ctx
    return _stft_ctx[device]


def forward_stft(samples: np.ndarray, window_len: int, hop: int, device: int = 0) -> np.ndarray:
    """stft.hpp:13-15 on the GPU. samples (channels, length) float64 ->
    spectrogram (bins, frames, channels) complex128, bit-identical to the
    reference arithmetic."""
    lib = L.load()
    s = np.ascontiguousarray(samples, dtype=np.float64)
    if s.ndim != 2:
        raise ConfigError("samples must have shape (channels, length)")
    chans, n = s.shape
    bins = window_len // 2 + 1 if window_len > 0 else 1
    frames = int(lib.ctf_stft_frames(n, hop)) if hop > 0 else 1
    spec = np.zeros((bins, max(frames, 1), chans), np.complex128)
    err = L.CtfErr()
    _check(lib.ctf_stft(_device_ctx(device), L.dptr(s), n, chans, window_len, hop, L.dptr(spec), C.byref(err)), err)
    return spec


def inverse_stft(spec: np.ndarray, window_len: int, hop: int, original_length: int = 0,
                 device: int = 0) -> np.ndarray:
    """stft.hpp:17-18 on the GPU: (bins, frames, channels) -> (channels, length)."""
    lib = L.load()
    sp = np.ascontiguousarray(spec, dtype=np.complex128)
    if sp.ndim != 3:
        raise ConfigError("spectrogram must have shape (bins, frames, channels)")
    bins, frames, chans = sp.shape
    n, err = C.c_int64(), L.CtfErr()
    ctx = _device_ctx(device)
    _check(lib.ctf_istft(ctx, L.dptr(sp), bins, frames, chans, window_len, hop, original_length, None,
                         C.byref(n), C.byref(err)), err)
    out = np.zeros((chans, n.value))
    _check(lib.ctf_istft(ctx, L.dptr(sp), bins, frames, chans, window_len, hop, original_length, L.dptr(out),
                         C.byref(n), C.byref(err)), err)
    return out


# ---- containers (container.hpp:1-29): .spec spectrograms and .nmf factors
def read_spectrogram(path: str, precision: str = "f64"):
    """read_spectrogram (container.cpp:74-86): (header dict, spec (bins, frames, channels))."""
    lib, h, err = L.load(), L.CtfSpecHeader(), L.CtfErr()
    _check(lib.ctf_read_spectrogram(path.encode(), C.byref(h), None, L.CTF_F64, C.byref(err)), err)
    f32 = precision in ("f32", "complex64")
    spec = np.zeros((h.bins, h.frames, h.channels), np.complex64 if f32 else np.complex128)
    _check(lib.ctf_read_spectrogram(path.encode(), C.byref(h), spec.ctypes.data_as(C.c_void_p),
                                    L.CTF_F32 if f32 else L.CTF_F64, C.byref(err)), err)
    hdr = {k: getattr(h, k) for k, _ in L.CtfSpecHeader._fields_}
    return hdr, spec


def write_spectrogram(path: str, spec: np.ndarray, window_len: int = 0, hop: int = 0, sample_rate: int = 0,
                      original_length: int = 0):
    """write_spectrogram (container.cpp:61-72): spec (bins, frames, channels) complex, stored as complex64."""
    lib, err = L.load(), L.CtfErr()
    f32 = spec.dtype == np.complex64
    sp = np.ascontiguousarray(spec, dtype=np.complex64 if f32 else np.complex128)
    h = L.CtfSpecHeader(sp.shape[0], sp.shape[1], sp.shape[2], window_len, hop, int(sample_rate), original_length)
    _check(lib.ctf_write_spectrogram(path.encode(), C.byref(h), sp.ctypes.data_as(C.c_void_p),
                                     L.CTF_F32 if f32 else L.CTF_F64, C.byref(err)), err)


def write_factors(path: str, bases: List[np.ndarray], activations: List[np.ndarray], floor: float):
    """write_factors (container.cpp:124-142): B_n (F, K_n), V_n (K_n, T) float64."""
    lib, err = L.load(), L.CtfErr()
    F, T = bases[0].shape[0], activations[0].shape[1]
    ks = (C.c_int32 * len(bases))(*[b.shape[1] for b in bases])
    Bf = np.concatenate([np.asarray(b, np.float64).ravel(order="F") for b in bases])
    Vf = np.concatenate([np.asarray(v, np.float64).ravel(order="F") for v in activations])
    _check(lib.ctf_write_factors(path.encode(), len(bases), F, T, ks, floor, L.dptr(Bf), L.dptr(Vf),
                                 C.byref(err)), err)


def read_factors(path: str):
    """read_factors (container.cpp:144-165): (bases list, activations list, floor)."""
    lib, err = L.load(), L.CtfErr()
    ns, nb, nf, fl = C.c_int(), C.c_int(), C.c_int(), C.c_double()
    ks = (C.c_int32 * L.CTF_MAX_SOURCES)()
    _check(lib.ctf_read_factors(path.encode(), C.byref(ns), C.byref(nb), C.byref(nf), ks, C.byref(fl), None, None,
                                C.byref(err)), err)
    K = [ks[n] for n in range(ns.value)]
    Bf, Vf = np.zeros(nb.value * sum(K)), np.zeros(sum(K) * nf.value)
    _check(lib.ctf_read_factors(path.encode(), C.byref(ns), C.byref(nb), C.byref(nf), ks, C.byref(fl), L.dptr(Bf),
                                L.dptr(Vf), C.byref(err)), err)
    bases, acts, ob, ov = [], [], 0, 0
    for k in K:
        bases.append(Bf[ob:ob + nb.value * k].reshape(nb.value, k, order="F"))
        acts.append(Vf[ov:ov + k * nf.value].reshape(k, nf.value, order="F"))
        ob += nb.value * k
        ov += k * nf.value
    return bases, acts, fl.value


def _spectrogram_to_abi(x: np.ndarray) -> np.ndarray:
    """(F, D, T) MixtureSpectrogram -> [1, F, T, D] (reference Spectrogram layout)."""
    if x.ndim != 3:
        raise ConfigError("mixture must have shape (F, channels, T)")
    return np.ascontiguousarray(np.transpose(x, (0, 2, 1)))[None].astype(np.complex128)


def run(config: CtfConfig, x: np.ndarray, checks: Optional[CheckOptions] = None, precision: str = "f64",
        device: int = 0, stack_taps: int = 1) -> SeparationResult:
    """estimator.hpp:122-123 on the GPU. x: (F, channels, T) complex; with
    stack_taps = L > 1, x holds num_channels / L microphones and the
    stacked observation is built on the GPU."""
    config.validate()
    if x.shape[1] * stack_taps != config.num_channels:
        raise ConfigError(f"mixture has {x.shape[1] * stack_taps} channels but config expects {config.num_channels}")
    xa = _spectrogram_to_abi(x)
    s = Session(xa, config.taps_per_source, config.bases_per_source, stack_taps=stack_taps,
                iterations=config.iterations, precision=precision, psd_floor=config.psd_floor,
                seed=config.seed, device=device, checks=checks.flags() if checks else 0,
                update_rule=config.update_rule)
    try:
        s.iterate(config.iterations)
        dem, bases, acts, obj = s.download()[0]
        d, m, r = s.trace_ms()
        tr = OptimizationTrace(list(obj), list(d), list(m), list(r))
        if checks and checks.flags():
            cd, cn, ck = s.check_stats()
            tr.max_det_lemma_error, tr.max_normalization_error, tr.checked_updates = \
                float(cd[0]), float(cn[0]), int(ck[0])
        return SeparationResult(dem, bases, acts, float(s.psd_floor()[0]), tr)
    finally:
        s.close()


def reconstruct_images(demixing: np.ndarray, config: CtfConfig, x: np.ndarray, precision="f64", device=0,
                       stack_taps: int = 1) -> np.ndarray:
    """wiener.cpp:11-49: images (N, F, D, T) complex for the given (F, R, D) demixing."""
    config.validate()
    xa = _spectrogram_to_abi(x)
    F = x.shape[0]
    s = Session(xa, config.taps_per_source, config.bases_per_source, stack_taps=stack_taps, iterations=0,
                precision=precision, psd_floor=config.psd_floor, seed=config.seed, device=device)
    try:
        W = np.ascontiguousarray(np.transpose(demixing, (0, 2, 1))).reshape(1, F, -1)
        s.set_state(W=W.view(np.float64))
        img = s.project_back()
        return np.transpose(img[:, 0], (0, 1, 3, 2))
    finally:
        s.close()


def synth_mixtures(num_mixtures, F, T, M, N, L_taps, K, decay, seed, precision="f64", threads=0) -> np.ndarray:
    """BASELINE.json configs[0] generator (host code): [B, F, T, M] complex."""
    lib = L.load()
    dt = np.complex64 if precision == "f32" else np.complex128
    x = np.empty((num_mixtures, F, T, M), dt)
    err = L.CtfErr()
    rc = lib.ctf_synth_mixtures(num_mixtures, F, T, M, N, L_taps, K, decay, seed,
                                L.CTF_F32 if precision == "f32" else L.CTF_F64, L.vptr(x), threads, C.byref(err))
    _check(rc, err)
    return x
