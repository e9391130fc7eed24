"""B200-native ISS+NMF hot path of CTF-MNMF-ISS (arXiv 2510.02382).

The product is libctfiss.so (CUDA kernels for sm_100a behind the C ABI in
include/ctf_iss.h). This package is its Python binding; the C++ mirror of the
reference API lives in csrc/ctfmnmf_b200.hpp.
"""
from .api import (CheckOptions, CtfConfig, ConfigError, DegeneracyError, DeviceError, IoError, OptimizationTrace,
                  SeparationResult, Session, forward_stft, inverse_stft, read_factors, read_spectrogram,
                  reconstruct_images, run, synth_mixtures, write_factors, write_spectrogram)

__all__ = ["CheckOptions", "CtfConfig", "ConfigError", "DegeneracyError", "DeviceError", "IoError", "OptimizationTrace",
           "SeparationResult", "Session", "forward_stft", "inverse_stft", "read_factors",
           "read_spectrogram", "reconstruct_images", "run", "synth_mixtures", "write_factors", "write_spectrogram"]
