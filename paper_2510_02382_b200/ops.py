"""Op-level mirror of the reference estimator API (proj/include/ctfmnmf/
estimator.hpp:56-117, model.hpp:86-88) on the GPU, fp64, through the C ABI's
ctf_op_* entries (include/ctf_iss.h). Same names and argument meaning as the
reference; arrays use the reference's column-major per-bin layouts as numpy
"memory" arrays (the layouts oracle/oracle.py uses):

  W      complex128 [F, D, R]   (per bin column-major R x D)
  Y      complex128 [F, T, R]   (per bin column-major R x T, DelayedEstimates)
  x      complex128 [F, T, D]   (MixtureSpectrogram, already stacked)
  B      float64 flat, B_n column-major F x K_n concatenated over sources
  V      float64 flat, V_n column-major K_n x T concatenated over sources
  lambda float64 [N, T, F]      (lambda_n column-major F x T)

Inputs are never modified; the updated arrays are returned. Errors raise the
reference's exception types (ConfigError / DegeneracyError) with its texts.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .api import _check, _device_ctx


def _problem(taps, bases, F, T):
    p = L.CtfProblem()
    p.num_mixtures, p.num_bins, p.num_frames = 1, F, T
    p.num_sources = len(taps)
    p.num_mics, p.stack_taps = sum(taps), 1
    for n, (l, k) in enumerate(zip(taps, bases)):
        p.taps_per_source[n], p.bases_per_source[n] = l, k
    return p


def _c(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _r(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _cp(a):
    return L.dptr(a.view(np.float64))


def demix(W, x, device=0):
    """estimator.cpp:304-311: Y_i = W_i x_i."""
    W, x = _c(W), _c(x)
    F, D, R = W.shape
    T = x.shape[1]
    Y = np.zeros((F, T, R), np.complex128)
    err = L.CtfErr()
    _check(L.load().ctf_op_demix(_device_ctx(device), F, R, D, T, _cp(W), _cp(x), _cp(Y), L.CTF_MEM_HOST,
                                 C.byref(err)), err)
    return Y


def compute_psd(taps, bases, F, T, B, V, floor_abs, device=0):
    """model.cpp:210-215 for every source: lambda [N, T, F]."""
    B, V = _r(B), _r(V)
    lam = np.zeros((len(taps), T, F))
    err = L.CtfErr()
    p = _problem(taps, bases, F, T)
    _check(L.load().ctf_op_compute_psd(_device_ctx(device), C.byref(p), L.dptr(B), L.dptr(V), floor_abs, L.dptr(lam),
                                       L.CTF_MEM_HOST, C.byref(err)), err)
    return lam


def iss_sweep(taps, W, Y, lam, device=0):
    """estimator.cpp:505-511 on every bin: returns the swept (W, Y)."""
    W, Y, lam = _c(W).copy(), _c(Y).copy(), _r(lam)
    F, T = Y.shape[0], Y.shape[1]
    err = L.CtfErr()
    p = _problem(taps, [1] * len(taps), F, T)
    _check(L.load().ctf_op_iss_sweep(_device_ctx(device), C.byref(p), _cp(W), _cp(Y), L.dptr(lam), L.CTF_MEM_HOST,
                                     C.byref(err)), err)
    return W, Y


def mu_update_bases(taps, bases, F, T, B, V, floor_abs, Y, source, device=0):
    """estimator.cpp:313-346: returns the updated B."""
    B, V, Y = _r(B).copy(), _r(V), _c(Y)
    err = L.CtfErr()
    p = _problem(taps, bases, F, T)
    _check(L.load().ctf_op_mu_update_bases(_device_ctx(device), C.byref(p), L.dptr(B), L.dptr(V), floor_abs, _cp(Y),
                                           source, L.CTF_MEM_HOST, C.byref(err)), err)
    return B


def mu_update_activations(taps, bases, F, T, B, V, floor_abs, Y, source, device=0):
    """estimator.cpp:348-382 (all taps contribute): returns the updated V."""
    B, V, Y = _r(B), _r(V).copy(), _c(Y)
    err = L.CtfErr()
    p = _problem(taps, bases, F, T)
    _check(L.load().ctf_op_mu_update_activations(_device_ctx(device), C.byref(p), L.dptr(B), L.dptr(V), floor_abs,
                                                 _cp(Y), source, L.CTF_MEM_HOST, C.byref(err)), err)
    return V


def rescale(taps, bases, F, T, W, B, floor_abs, Y, device=0):
    """estimator.cpp:384-412: returns the rescaled (W, B, Y)."""
    W, B, Y = _c(W).copy(), _r(B).copy(), _c(Y).copy()
    err = L.CtfErr()
    p = _problem(taps, bases, F, T)
    _check(L.load().ctf_op_rescale(_device_ctx(device), C.byref(p), _cp(W), L.dptr(B), floor_abs, _cp(Y),
                                   L.CTF_MEM_HOST, C.byref(err)), err)
    return W, B, Y


def log_abs_det(W, device=0):
    """estimator.cpp:41-53 per bin: W [F, R, R] memory (or one R x R) -> [F]."""
    W = _c(W)
    single = W.ndim == 2
    if single:
        W = W[None]
    out = np.zeros(W.shape[0])
    err = L.CtfErr()
    _check(L.load().ctf_op_log_abs_det(_device_ctx(device), W.shape[1], W.shape[0], _cp(W), L.dptr(out),
                                       L.CTF_MEM_HOST, C.byref(err)), err)
    return float(out[0]) if single else out


def objective_from_parts(taps, W, lam, Y, device=0):
    """estimator.cpp:55-77."""
    W, lam, Y = _c(W), _r(lam), _c(Y)
    F, T = Y.shape[0], Y.shape[1]
    out = C.c_double()
    err = L.CtfErr()
    p = _problem(taps, [1] * len(taps), F, T)
    _check(L.load().ctf_op_objective_from_parts(_device_ctx(device), C.byref(p), _cp(W), L.dptr(lam), _cp(Y),
                                                C.byref(out), L.CTF_MEM_HOST, C.byref(err)), err)
    return out.value
