"""TEST INFRASTRUCTURE ONLY: ctypes binding of the CPU oracle (libctf_oracle.so).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline arm may use
this module; the product never imports it. See ctf_oracle.h for what the
oracle restates and how it is pinned.

Arrays: x is complex128 [F, T, D] (per bin the column-major D x T matrix of
the reference, model.hpp:55-66); W is complex128 [F, D, R] memory order
(column-major R x D per bin); B is float64 [sum_n F*K_n] (each B_n
column-major F x K_n); V is float64 [sum_n K_n*T] (each V_n column-major).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(_HERE, "libctf_oracle.so")
MAX_SOURCES = 16


class OrcConfig(C.Structure):
    _fields_ = [("num_sources", C.c_int32), ("num_channels", C.c_int32), ("taps", C.c_int32 * MAX_SOURCES),
                ("bases", C.c_int32 * MAX_SOURCES), ("iterations", C.c_int32), ("rule", C.c_int32),
                ("psd_floor", C.c_double), ("seed", C.c_uint64), ("threads", C.c_int32)]


class OrcErr(C.Structure):
    _fields_ = [("code", C.c_int32), ("iteration", C.c_int32), ("bin", C.c_int32), ("row", C.c_int32),
                ("msg", C.c_char * 256)]


class OracleError(Exception):
    def __init__(self, code, msg, iteration=-1, bin=-1, row=-1):
        super().__init__(msg)
        self.code, self.iteration, self.bin, self.row = code, iteration, bin, row


_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = C.CDLL(LIB)
    return _lib


def _d(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def config(taps, bases, iterations=100, seed=0, psd_floor=1e-10, threads=1, rule="iss", num_channels=None):
    c = OrcConfig()
    c.num_sources = len(taps)
    c.num_channels = sum(taps) if num_channels is None else num_channels
    for n, (l, k) in enumerate(zip(taps, bases)):
        c.taps[n], c.bases[n] = l, k
    c.iterations, c.rule, c.psd_floor, c.seed, c.threads = iterations, 1 if rule == "iss" else 0, psd_floor, seed, threads
    return c


def _check(rc, err):
    if rc != 0:
        raise OracleError(rc, err.msg.decode(), err.iteration, err.bin, err.row)


def stack_observation(x: np.ndarray, L: int) -> np.ndarray:
    """[F, T, M] -> [F, T, M*L] with x~[f, t, m*L + l] = x[f, t - l, m] (zero for t < l)."""
    F, T, M = x.shape
    out = np.zeros((F, T, M * L), dtype=np.complex128)
    for m in range(M):
        for l in range(L):
            out[:, l:, m * L + l] = x[:, :T - l, m]
    return out


def run(cfg: OrcConfig, x: np.ndarray, history=False):
    """estimator.cpp:513-657. Returns dict W, B, V, objective (+ hist_* when asked)."""
    F, T, D = x.shape
    x = np.ascontiguousarray(x, dtype=np.complex128)
    R = sum(cfg.taps[:cfg.num_sources])
    SK = sum(cfg.bases[:cfg.num_sources])
    it = cfg.iterations
    W = np.zeros((F, D, R), np.complex128)
    B = np.zeros(F * SK)
    V = np.zeros(SK * T)
    obj = np.zeros(max(it, 1))
    ms = np.zeros((max(it, 1), 3))
    hW = np.zeros((it, F, D, R), np.complex128) if history else None
    hB = np.zeros((it, F * SK)) if history else None
    hV = np.zeros((it, SK * T)) if history else None
    err = OrcErr()
    rc = lib().orc_run(C.byref(cfg), F, T, _d(x.view(np.float64)), _d(W.view(np.float64)), _d(B), _d(V), _d(obj),
                       _d(None if hW is None else hW.view(np.float64)), _d(hB), _d(hV), _d(ms), C.byref(err))
    _check(rc, err)
    out = {"W": W, "B": B, "V": V, "objective": obj[:it], "trace_ms": ms[:it]}
    if history:
        out.update(hist_W=hW, hist_B=hB, hist_V=hV)
    return out


def step(cfg: OrcConfig, x: np.ndarray, floor_abs: float, W, B, V):
    """One iteration from an explicit state (copies are updated and returned)."""
    F, T, D = x.shape
    W = np.array(W, dtype=np.complex128, copy=True)
    B = np.array(B, dtype=np.float64, copy=True)
    V = np.array(V, dtype=np.float64, copy=True)
    obj = C.c_double()
    err = OrcErr()
    rc = lib().orc_step(C.byref(cfg), F, T, _d(np.ascontiguousarray(x).view(np.float64)), C.c_double(floor_abs),
                        _d(W.view(np.float64)), _d(B), _d(V), C.byref(obj), C.byref(err))
    _check(rc, err)
    return W, B, V, obj.value


def run_checked(cfg, x):
    F, T, D = x.shape
    det, nrm, cnt = C.c_double(), C.c_double(), C.c_int64()
    err = OrcErr()
    rc = lib().orc_run_checked(C.byref(cfg), F, T, _d(np.ascontiguousarray(x).view(np.float64)), C.byref(det),
                               C.byref(nrm), C.byref(cnt), C.byref(err))
    _check(rc, err)
    return det.value, nrm.value, cnt.value


def mean_power(x):
    F, T, D = x.shape
    lib().orc_mean_power.restype = C.c_double
    return lib().orc_mean_power(F, D, T, _d(np.ascontiguousarray(x).view(np.float64)))


def random_factors(cfg, F, T):
    SK = sum(cfg.bases[:cfg.num_sources])
    B, V = np.zeros(F * SK), np.zeros(SK * T)
    lib().orc_random_factors(C.byref(cfg), F, T, _d(B), _d(V))
    return B, V


def demix(W, x):
    """W [F, D, R] (col-major R x D), x [F, T, D] -> Y [F, T, R] (col-major R x T)."""
    F, D, R = W.shape
    T = x.shape[1]
    Y = np.zeros((F, T, R), np.complex128)
    lib().orc_demix(F, R, D, T, _d(np.ascontiguousarray(W).view(np.float64)),
                    _d(np.ascontiguousarray(x).view(np.float64)), _d(Y.view(np.float64)))
    return Y


def iss_sweep(cfg, W_bin, Y_bin, lam, bin):
    """W_bin [D, R], Y_bin [T, R] (memory order), lam [N, T, F] (each lambda_n col-major F x T)."""
    W = np.array(W_bin, np.complex128, copy=True)
    Y = np.array(Y_bin, np.complex128, copy=True)
    N, T, F = lam.shape
    err = OrcErr()
    rc = lib().orc_iss_sweep(C.byref(cfg), F, T, bin, _d(W.view(np.float64)), _d(Y.view(np.float64)),
                             _d(np.ascontiguousarray(lam)), C.byref(err))
    _check(rc, err)
    return W, Y


def weighted_covariance(x, lam_n, tap, bin):
    F, T, D = x.shape
    Q = np.zeros((D, D), np.complex128)
    lib().orc_weighted_covariance(F, D, T, _d(np.ascontiguousarray(x).view(np.float64)),
                                  _d(np.ascontiguousarray(lam_n)), tap, bin, _d(Q.view(np.float64)))
    return Q  # memory order [col][row]


def iss_compute_z(W_bin, covs, row):
    R = W_bin.shape[0]
    z = np.zeros(R, np.complex128)
    err = OrcErr()
    rc = lib().orc_iss_compute_z(R, _d(np.ascontiguousarray(W_bin).view(np.float64)),
                                 _d(np.ascontiguousarray(covs).view(np.float64)), row, _d(z.view(np.float64)),
                                 C.byref(err))
    _check(rc, err)
    return z


def iss_apply(W_bin, z, row):
    W = np.array(W_bin, np.complex128, copy=True)
    lib().orc_iss_apply(W.shape[1], W.shape[0], _d(W.view(np.float64)),
                        _d(np.ascontiguousarray(z, np.complex128).view(np.float64)), row)
    return W


def compute_psd(cfg, F, T, B, V, floor_abs):
    lam = np.zeros((cfg.num_sources, T, F))
    lib().orc_compute_psd(C.byref(cfg), F, T, _d(B), _d(V), C.c_double(floor_abs), _d(lam))
    return lam


def mu_update_bases(cfg, F, T, B, V, floor_abs, Y, source):
    B = np.array(B, np.float64, copy=True)
    lib().orc_mu_update_bases(C.byref(cfg), F, T, _d(B), _d(V), C.c_double(floor_abs),
                              _d(np.ascontiguousarray(Y).view(np.float64)), source)
    return B


def mu_update_activations(cfg, F, T, B, V, floor_abs, Y, source):
    V = np.array(V, np.float64, copy=True)
    lib().orc_mu_update_activations(C.byref(cfg), F, T, _d(B), _d(V), C.c_double(floor_abs),
                                    _d(np.ascontiguousarray(Y).view(np.float64)), source)
    return V


def rescale(cfg, F, T, W, B, floor_abs, Y):
    W = np.array(W, np.complex128, copy=True)
    B = np.array(B, np.float64, copy=True)
    Y = np.array(Y, np.complex128, copy=True)
    lib().orc_rescale(C.byref(cfg), F, T, _d(W.view(np.float64)), _d(B), C.c_double(floor_abs),
                      _d(Y.view(np.float64)))
    return W, B, Y


def log_abs_det(W_bin):
    out = C.c_double()
    err = OrcErr()
    rc = lib().orc_log_abs_det(W_bin.shape[0], _d(np.ascontiguousarray(W_bin).view(np.float64)), C.byref(out),
                               C.byref(err))
    _check(rc, err)
    return out.value


def objective(cfg, F, T, W, B, V, floor_abs, x):
    out = C.c_double()
    err = OrcErr()
    rc = lib().orc_objective(C.byref(cfg), F, T, _d(np.ascontiguousarray(W).view(np.float64)), _d(B), _d(V),
                             C.c_double(floor_abs), _d(np.ascontiguousarray(x).view(np.float64)), C.byref(out),
                             C.byref(err))
    _check(rc, err)
    return out.value


def objective_from_parts(cfg, F, T, W, lam, Y):
    out = C.c_double()
    err = OrcErr()
    rc = lib().orc_objective_from_parts(C.byref(cfg), F, T, _d(np.ascontiguousarray(W).view(np.float64)),
                                        _d(np.ascontiguousarray(lam)), _d(np.ascontiguousarray(Y).view(np.float64)),
                                        C.byref(out), C.byref(err))
    _check(rc, err)
    return out.value


def reconstruct_images(cfg, W, x):
    """images [N, F, T, D] (col-major D x T per bin)."""
    F, T, D = x.shape
    img = np.zeros((cfg.num_sources, F, T, D), np.complex128)
    err = OrcErr()
    rc = lib().orc_reconstruct_images(C.byref(cfg), F, T, _d(np.ascontiguousarray(W).view(np.float64)),
                                      _d(np.ascontiguousarray(x).view(np.float64)), _d(img.view(np.float64)),
                                      C.byref(err))
    _check(rc, err)
    return img


# ---- STFT front/back end (proj/src/fft.cpp, proj/src/stft.cpp) -------------
def fft(data: np.ndarray, inverse=False) -> np.ndarray:
    """fft.cpp:9-41 on a copy of a complex128 vector."""
    a = np.array(data, dtype=np.complex128, copy=True)
    err = OrcErr()
    _check(lib().orc_fft(_d(a.view(np.float64)), C.c_int64(a.size), int(inverse), C.byref(err)), err)
    return a


def hann_window(n: int) -> np.ndarray:
    out = np.zeros(n)
    lib().orc_hann(n, _d(out))
    return out


def stft_frames(length: int, hop: int) -> int:
    lib().orc_stft_frames.restype = C.c_int64
    return int(lib().orc_stft_frames(C.c_int64(length), hop))


def forward_stft(samples: np.ndarray, window_len: int, hop: int) -> np.ndarray:
    """stft.cpp:46-88. samples: (channels, length) float64 -> spec (bins, frames, channels) complex128."""
    s = np.ascontiguousarray(samples, dtype=np.float64)
    chans, n = s.shape
    bins = window_len // 2 + 1 if window_len > 0 else 0
    frames = stft_frames(n, hop) if hop > 0 else 0
    spec = np.zeros((max(bins, 0), max(frames, 0), chans), np.complex128)
    err = OrcErr()
    _check(lib().orc_forward_stft(_d(s), C.c_int64(n), chans, window_len, hop, _d(spec.view(np.float64)),
                                  C.byref(err)), err)
    return spec


def inverse_stft(spec: np.ndarray, window_len: int, hop: int, original_length: int = 0) -> np.ndarray:
    """stft.cpp:90-139. spec (bins, frames, channels) -> samples (channels, length)."""
    sp = np.ascontiguousarray(spec, dtype=np.complex128)
    bins, frames, chans = sp.shape
    n = C.c_int64()
    err = OrcErr()
    _check(lib().orc_inverse_stft(_d(sp.view(np.float64)), bins, frames, chans, window_len, hop,
                                  C.c_int64(original_length), None, C.byref(n), C.byref(err)), err)
    out = np.zeros((chans, n.value))
    _check(lib().orc_inverse_stft(_d(sp.view(np.float64)), bins, frames, chans, window_len, hop,
                                  C.c_int64(original_length), _d(out), C.byref(n), C.byref(err)), err)
    return out
