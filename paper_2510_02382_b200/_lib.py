"""ctypes binding of the C ABI in include/ctf_iss.h (libctfiss.so).

The library is built in-tree (``__graft_entry__.build()`` or ``make -C
paper_2510_02382_b200/csrc``). There is no fallback: importing the binding
without the built library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CTF_DEV_LIB") or os.path.join(_HERE, "libctfiss.so")  # CTF_DEV_LIB: tools/dev_build.sh builds

CTF_MAX_SOURCES = 16
CTF_OK, CTF_ERR_CONFIG, CTF_ERR_IO, CTF_ERR_DEGENERACY, CTF_ERR_CUDA, CTF_ERR_UNSUPPORTED = 0, 2, 3, 4, 5, 6
CTF_F64, CTF_F32 = 0, 1
CTF_RULE_IP, CTF_RULE_ISS = 0, 1
CTF_IMAGES_FULL, CTF_IMAGES_CURRENT_FRAME = 0, 1
CTF_MEM_HOST, CTF_MEM_DEVICE = 0, 1


class CtfErr(C.Structure):
    _fields_ = [("code", C.c_int32), ("kind", C.c_int32), ("iteration", C.c_int32), ("mixture", C.c_int32),
                ("bin", C.c_int32), ("row", C.c_int32), ("msg", C.c_char * 256)]


CTF_CHECK_DET_LEMMA, CTF_CHECK_NORMALIZATION = 1, 2


class CtfProblem(C.Structure):
    _fields_ = [("num_mixtures", C.c_int32), ("num_bins", C.c_int32), ("num_frames", C.c_int32),
                ("num_mics", C.c_int32), ("stack_taps", C.c_int32), ("num_sources", C.c_int32),
                ("taps_per_source", C.c_int32 * CTF_MAX_SOURCES),
                ("bases_per_source", C.c_int32 * CTF_MAX_SOURCES), ("iterations", C.c_int32),
                ("update_rule", C.c_int32), ("precision", C.c_int32), ("x_precision", C.c_int32),
                ("psd_floor", C.c_double), ("seed", C.c_uint64), ("threads", C.c_int32),
                ("checks", C.c_int32), ("reserved", C.c_int32 * 6)]


class CtfSpecHeader(C.Structure):
    _fields_ = [("bins", C.c_uint32), ("frames", C.c_uint32), ("channels", C.c_uint32), ("window_len", C.c_uint32),
                ("hop", C.c_uint32), ("sample_rate", C.c_uint32), ("original_length", C.c_uint64)]


class CtfTiming(C.Structure):
    _fields_ = [("sweep_ms", C.c_double), ("mu_ms", C.c_double), ("finalize_ms", C.c_double),
                ("sweep_launches", C.c_int64), ("launches", C.c_int64)]


# Every symbol include/ctf_iss.h declares, with its signature.
_P = C.c_void_p
_E = C.POINTER(CtfErr)
_D = C.POINTER(C.c_double)
SIGNATURES = {
    "ctf_abi_version": (C.c_int, []),
    "ctf_open": (C.c_int, [C.c_int, C.POINTER(_P), _E]),
    "ctf_close": (None, [_P]),
    "ctf_stream": (_P, [_P]),
    "ctf_comm_unique_id": (C.c_int, [C.POINTER(C.c_uint8), _E]),
    "ctf_comm_init": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_uint8), _E]),
    "ctf_group_create": (_P, [C.c_int]),
    "ctf_group_destroy": (None, [_P]),
    "ctf_comm_init_group": (C.c_int, [_P, _P, C.c_int, _E]),
    "ctf_shard_range": (None, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ctf_setup": (C.c_int, [_P, C.POINTER(CtfProblem), _P, _E]),
    "ctf_set_state": (C.c_int, [_P, _D, _D, _D, _E]),
    "ctf_iterate": (C.c_int, [_P, C.c_int, _E]),
    "ctf_iterate_async": (C.c_int, [_P, C.c_int, _E]),
    "ctf_finalize": (C.c_int, [_P, _E]),
    "ctf_download": (C.c_int, [_P, _D, _D, _D, _D, _E]),
    "ctf_iterations_done": (C.c_int, [_P]),
    "ctf_describe": (C.c_int, [_P, C.c_char_p, C.c_int]),
    "ctf_psd_floor": (C.c_int, [_P, _D]),
    "ctf_trace_ms": (C.c_int, [_P, _D, _D, _D]),
    "ctf_get_timing": (C.c_int, [_P, C.POINTER(CtfTiming)]),
    "ctf_check_stats": (C.c_int, [_P, _D, _D, C.POINTER(C.c_int64)]),
    "ctf_stft_frames": (C.c_int64, [C.c_int64, C.c_int]),
    "ctf_stft": (C.c_int, [_P, _D, C.c_int64, C.c_int, C.c_int, C.c_int, _D, C.POINTER(CtfErr)]),
    "ctf_istft": (C.c_int, [_P, _D, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, _D,
                            C.POINTER(C.c_int64), C.POINTER(CtfErr)]),
    "ctf_stft_device": (C.c_int, [_P, C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                  C.c_int, C.POINTER(CtfErr)]),
    "ctf_istft_device": (C.c_int, [_P, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_int64, C.c_void_p, C.POINTER(CtfErr)]),
    "ctf_read_spectrogram": (C.c_int, [C.c_char_p, C.POINTER(CtfSpecHeader), C.c_void_p, C.c_int,
                                       C.POINTER(CtfErr)]),
    "ctf_write_spectrogram": (C.c_int, [C.c_char_p, C.POINTER(CtfSpecHeader), C.c_void_p, C.c_int,
                                        C.POINTER(CtfErr)]),
    "ctf_setup_spectrogram_files": (C.c_int, [_P, C.POINTER(CtfProblem), C.POINTER(C.c_char_p), C.c_int,
                                              C.POINTER(CtfSpecHeader), C.POINTER(CtfErr)]),
    "ctf_write_factors": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int32), C.c_double,
                                    _D, _D, C.POINTER(CtfErr)]),
    "ctf_read_factors": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_int32), C.POINTER(C.c_double), _D, _D, C.POINTER(CtfErr)]),
    "ctf_setup_signal": (C.c_int, [_P, C.POINTER(CtfProblem), _D, C.c_int64, C.c_int, C.c_int,
                                   C.POINTER(CtfErr)]),
    "ctf_images_to_signal": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int64, _D, C.POINTER(C.c_int64),
                                       C.POINTER(CtfErr)]),
    "ctf_reset_timing": (C.c_int, [_P]),
    "ctf_run": (C.c_int, [_P, C.POINTER(CtfProblem), _P, _D, _D, _D, _D, _E]),
    "ctf_project_back": (C.c_int, [_P, C.c_int, _D, _E]),
    "ctf_op_demix": (C.c_int, [_P, C.c_int, C.c_int, C.c_int, C.c_int, _D, _D, _D, C.c_int, _E]),
    "ctf_op_compute_psd": (C.c_int, [_P, C.POINTER(CtfProblem), _D, _D, C.c_double, _D, C.c_int, _E]),
    "ctf_op_iss_sweep": (C.c_int, [_P, C.POINTER(CtfProblem), _D, _D, _D, C.c_int, _E]),
    "ctf_op_mu_update_bases": (C.c_int, [_P, C.POINTER(CtfProblem), _D, _D, C.c_double, _D, C.c_int, C.c_int,
                                         _E]),
    "ctf_op_mu_update_activations": (C.c_int, [_P, C.POINTER(CtfProblem), _D, _D, C.c_double, _D, C.c_int,
                                               C.c_int, _E]),
    "ctf_op_rescale": (C.c_int, [_P, C.POINTER(CtfProblem), _D, _D, C.c_double, _D, C.c_int, _E]),
    "ctf_op_log_abs_det": (C.c_int, [_P, C.c_int, C.c_int, _D, _D, C.c_int, _E]),
    "ctf_op_objective_from_parts": (C.c_int, [_P, C.POINTER(CtfProblem), _D, _D, _D, _D, C.c_int, _E]),
    "ctf_synth_mixtures": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                     C.c_uint64, C.c_int, _P, C.c_int, _E]),
}

_lib = None


def load() -> C.CDLL:
    """Loads libctfiss.so (built in-tree); raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C paper_2510_02382_b200/csrc)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def dptr(a):
    """double* of a contiguous numpy array (or None)."""
    if a is None:
        return None
    return a.ctypes.data_as(_D)


def vptr(a):
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)
