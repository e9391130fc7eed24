"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/_ref/libctf_ref.so,
the reference's OWN estimator/model/wiener/stft/fft sources compiled
unmodified (oracle/Makefile.ref, Eigen-API shim oracle/ref_shims).

Only tests/, tests/golden/make_golden.py and bench.py's reference arm /
cpu_baseline leg may use it; the product never imports it. Array layouts and
the config/error structs are those of oracle/oracle.py (see ctf_oracle.h), so
results compare element by element with the restatement and the GPU path.

The library is built here, where /root/reference exists; on the GPU box only
the prebuilt file that travelled with the snapshot is used (available()).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from .oracle import OrcConfig, OrcErr, OracleError, config, stack_observation  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_ROOT = "/root/reference/proj"
LIB = os.path.join(_HERE, "_ref", "libctf_ref.so")
UNIT_TESTS = os.path.join(_HERE, "_ref", "ref_unit_tests")
ACCEPTANCE = os.path.join(_HERE, "_ref", "ref_acceptance")
_lib = None


def build() -> bool:
    """Builds oracle/_ref from the reference sources when they are present."""
    if os.path.isdir(REF_ROOT):
        subprocess.run(["make", "-s", "-j8", "-C", _HERE, "-f", "Makefile.ref"], check=True)
    return os.path.exists(LIB)


def available() -> bool:
    return os.path.exists(LIB) or build()


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise OSError("oracle/_ref/libctf_ref.so is not built and /root/reference is absent")
        _lib = C.CDLL(LIB)
        _lib.ref_mean_power.restype = C.c_double
    return _lib


def _d(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _c(a):
    return _d(np.ascontiguousarray(a, dtype=np.complex128).view(np.float64))


def _check(rc, err):
    if rc != 0:
        raise OracleError(rc, err.msg.decode(), err.iteration, err.bin, err.row)


def _R(cfg):
    return sum(cfg.taps[:cfg.num_sources])


def _SK(cfg):
    return sum(cfg.bases[:cfg.num_sources])


def run(cfg: OrcConfig, x: np.ndarray, det_lemma=False, normalization=False):
    """run(), estimator.cpp:513-657. Same dict keys as oracle.run (+ checks)."""
    F, T, D = x.shape
    R, SK, it = _R(cfg), _SK(cfg), cfg.iterations
    W = np.zeros((F, D, R), np.complex128)
    B, V = np.zeros(F * SK), np.zeros(SK * T)
    obj, ms, chk = np.zeros(max(it, 1)), np.zeros((max(it, 1), 3)), np.zeros(3)
    err = OrcErr()
    rc = lib().ref_run(C.byref(cfg), F, T, _c(x), int(det_lemma), int(normalization), _d(W.view(np.float64)),
                       _d(B), _d(V), _d(obj), _d(ms), _d(chk), C.byref(err))
    _check(rc, err)
    return {"W": W, "B": B, "V": V, "objective": obj[:it], "trace_ms": ms[:it],
            "checks": {"max_det_lemma_error": chk[0], "max_normalization_error": chk[1],
                       "checked_updates": int(chk[2])}}


def run_history(cfg: OrcConfig, x: np.ndarray, iterations=None):
    """State after every iteration k = 1..n, each from run() with
    iterations = k (run() is deterministic for a fixed seed, so the state
    after k iterations of a longer run is exactly this)."""
    n = cfg.iterations if iterations is None else iterations
    hW, hB, hV, obj = [], [], [], None
    for k in range(1, n + 1):
        c = OrcConfig.from_buffer_copy(cfg)
        c.iterations = k
        r = run(c, x)
        hW.append(r["W"])
        hB.append(r["B"])
        hV.append(r["V"])
        obj = r["objective"]
    return {"hist_W": np.array(hW), "hist_B": np.array(hB), "hist_V": np.array(hV), "objective": obj}


def mean_power(x):
    F, T, D = x.shape
    return lib().ref_mean_power(F, D, T, _c(x))


def random_factors(cfg, F, T, floor_abs=1e-12):
    B, V = np.zeros(F * _SK(cfg)), np.zeros(_SK(cfg) * T)
    err = OrcErr()
    _check(lib().ref_random_factors(C.byref(cfg), F, T, C.c_double(floor_abs), _d(B), _d(V), C.byref(err)), err)
    return B, V


def demix(W, x):
    F, D, R = W.shape
    T = x.shape[1]
    Y = np.zeros((F, T, R), np.complex128)
    err = OrcErr()
    _check(lib().ref_demix(F, R, D, T, _c(W), _c(x), _d(Y.view(np.float64)), C.byref(err)), err)
    return Y


def iss_sweep(cfg, W_bin, Y_bin, lam, bin):
    W = np.array(W_bin, np.complex128, copy=True)
    Y = np.array(Y_bin, np.complex128, copy=True)
    N, T, F = lam.shape
    err = OrcErr()
    _check(lib().ref_iss_sweep(C.byref(cfg), F, T, bin, _d(W.view(np.float64)), _d(Y.view(np.float64)),
                               _d(np.ascontiguousarray(lam, np.float64)), C.byref(err)), err)
    return W, Y


def weighted_covariance(x, lam_n, tap, bin):
    F, T, D = x.shape
    Q = np.zeros((D, D), np.complex128)
    err = OrcErr()
    _check(lib().ref_weighted_covariance(F, D, T, _c(x), _d(np.ascontiguousarray(lam_n, np.float64)), tap, bin,
                                         _d(Q.view(np.float64)), C.byref(err)), err)
    return Q


def iss_compute_z(W_bin, covs, row):
    R = W_bin.shape[0]
    z = np.zeros(R, np.complex128)
    err = OrcErr()
    _check(lib().ref_iss_compute_z(R, _c(W_bin), _c(covs), row, _d(z.view(np.float64)), C.byref(err)), err)
    return z


def iss_apply(W_bin, z, row):
    W = np.array(W_bin, np.complex128, copy=True)
    err = OrcErr()
    _check(lib().ref_iss_apply(W.shape[1], W.shape[0], _d(W.view(np.float64)), _c(z), row, C.byref(err)), err)
    return W


def ip_update(W_bin, cov, row):
    W = np.array(W_bin, np.complex128, copy=True)
    err = OrcErr()
    _check(lib().ref_ip_update(W.shape[0], _d(W.view(np.float64)), _c(cov), row, C.byref(err)), err)
    return W


def compute_psd(cfg, F, T, B, V, floor_abs):
    lam = np.zeros((cfg.num_sources, T, F))
    err = OrcErr()
    _check(lib().ref_compute_psd(C.byref(cfg), F, T, _d(np.ascontiguousarray(B, np.float64)),
                                 _d(np.ascontiguousarray(V, np.float64)), C.c_double(floor_abs), _d(lam),
                                 C.byref(err)), err)
    return lam


def _mu(cfg, F, T, B, V, floor_abs, Y, source, act):
    B = np.array(B, np.float64, copy=True)
    V = np.array(V, np.float64, copy=True)
    err = OrcErr()
    _check(lib().ref_mu_update(C.byref(cfg), F, T, _d(B), _d(V), C.c_double(floor_abs), _c(Y), source, act,
                               C.byref(err)), err)
    return V if act else B


def mu_update_bases(cfg, F, T, B, V, floor_abs, Y, source):
    return _mu(cfg, F, T, B, V, floor_abs, Y, source, 0)


def mu_update_activations(cfg, F, T, B, V, floor_abs, Y, source):
    return _mu(cfg, F, T, B, V, floor_abs, Y, source, 1)


def rescale(cfg, F, T, W, B, floor_abs, Y, V=None):
    W = np.array(W, np.complex128, copy=True)
    B = np.array(B, np.float64, copy=True)
    Y = np.array(Y, np.complex128, copy=True)
    Vv = np.zeros(_SK(cfg) * T) if V is None else np.array(V, np.float64, copy=True)
    err = OrcErr()
    _check(lib().ref_rescale(C.byref(cfg), F, T, _d(W.view(np.float64)), _d(B), _d(Vv), C.c_double(floor_abs),
                             _d(Y.view(np.float64)), C.byref(err)), err)
    return W, B, Y


def log_abs_det(W_bin):
    out = C.c_double()
    err = OrcErr()
    _check(lib().ref_log_abs_det(W_bin.shape[0], _c(W_bin), C.byref(out), C.byref(err)), err)
    return out.value


def objective_from_parts(cfg, F, T, W, lam, Y):
    out = C.c_double()
    err = OrcErr()
    _check(lib().ref_objective_from_parts(C.byref(cfg), F, T, _c(W), _d(np.ascontiguousarray(lam, np.float64)),
                                          _c(Y), C.byref(out), C.byref(err)), err)
    return out.value


def objective(cfg, F, T, W, B, V, floor_abs, x):
    out = C.c_double()
    err = OrcErr()
    _check(lib().ref_objective(C.byref(cfg), F, T, _c(W), _d(np.ascontiguousarray(B, np.float64)),
                               _d(np.ascontiguousarray(V, np.float64)), C.c_double(floor_abs), _c(x), C.byref(out),
                               C.byref(err)), err)
    return out.value


def reconstruct_images(cfg, W, x, B=None, V=None, floor_abs=1e-12):
    """images [N, F, T, D]; B/V only feed the factor-count check (wiener.cpp:17-19)."""
    F, T, D = x.shape
    SK = _SK(cfg)
    B = np.ones(F * SK) if B is None else B
    V = np.ones(SK * T) if V is None else V
    img = np.zeros((cfg.num_sources, F, T, D), np.complex128)
    err = OrcErr()
    _check(lib().ref_reconstruct_images(C.byref(cfg), F, T, _c(W), _d(np.ascontiguousarray(B, np.float64)),
                                        _d(np.ascontiguousarray(V, np.float64)), C.c_double(floor_abs), _c(x),
                                        _d(img.view(np.float64)), C.byref(err)), err)
    return img


def fft(data, inverse=False):
    a = np.array(data, dtype=np.complex128, copy=True)
    err = OrcErr()
    _check(lib().ref_fft(_d(a.view(np.float64)), C.c_int64(a.size), int(inverse), C.byref(err)), err)
    return a


def forward_stft(samples, window_len, hop):
    s = np.ascontiguousarray(samples, dtype=np.float64)
    chans, n = s.shape
    dims = (C.c_int * 2)()
    err = OrcErr()
    _check(lib().ref_forward_stft(_d(s), C.c_int64(n), chans, window_len, hop, None, dims, C.byref(err)), err)
    spec = np.zeros((dims[0], dims[1], chans), np.complex128)
    _check(lib().ref_forward_stft(_d(s), C.c_int64(n), chans, window_len, hop, _d(spec.view(np.float64)), dims,
                                  C.byref(err)), err)
    return spec


def inverse_stft(spec, window_len, hop, original_length=0):
    sp = np.ascontiguousarray(spec, dtype=np.complex128)
    bins, frames, chans = sp.shape
    n = C.c_int64()
    err = OrcErr()
    _check(lib().ref_inverse_stft(_d(sp.view(np.float64)), bins, frames, chans, window_len, hop,
                                  C.c_int64(original_length), None, C.byref(n), C.byref(err)), err)
    out = np.zeros((chans, n.value))
    _check(lib().ref_inverse_stft(_d(sp.view(np.float64)), bins, frames, chans, window_len, hop,
                                  C.c_int64(original_length), _d(out), C.byref(n), C.byref(err)), err)
    return out


def synth_mixtures(num_mixtures, F, T, M, N, L_taps, K, decay, seed, threads=0):
    """BASELINE's generator (paper_2510_02382_b200/csrc/synth.cpp compiled into
    this library), so reference-only processes never map the product library.
    Returns complex128 [B, F, T, M]."""
    out = np.zeros((num_mixtures, F, T, M), np.complex128)
    err = (C.c_int32 * 70)()  # ctf_err (include/ctf_iss.h), only the code is read
    fn = lib().ctf_synth_mixtures
    fn.argtypes = [C.c_int] * 7 + [C.c_double, C.c_uint64, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
    rc = fn(num_mixtures, F, T, M, N, L_taps, K, decay, seed, 0, out.ctypes.data, threads, C.addressof(err))
    if rc != 0:
        raise OracleError(rc, "ctf_synth_mixtures failed")
    return out
