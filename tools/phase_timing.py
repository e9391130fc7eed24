"""Dev: per-phase cycle counts of gram_kernel from the instrumented build
(tools/phase/libctfiss.so, compiled with -DCTF_PHASE_TIMING)."""
import ctypes as C, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_02382_b200 import _lib
_lib.LIB_PATH = os.environ.get("CTF_DEV_LIB") or os.path.join(ROOT, "tools", "phase", "libctfiss.so")
from paper_2510_02382_b200 import Session, synth_mixtures
import argparse
ap = argparse.ArgumentParser(); ap.add_argument("--cfg", type=int, default=1); ap.add_argument("--prec", default="f32"); a = ap.parse_args()
B, F, T, M, N, L, K = {1: (64, 513, 1000, 2, 2, 5, 10), 2: (16, 1025, 2000, 3, 3, 4, 20), 3: (8, 2049, 1000, 4, 4, 8, 20)}[a.cfg]
x = synth_mixtures(B, F, T, M, N, L, K, 0.6, 1, precision=a.prec)
s = Session(x, [L] * N, [K] * N, stack_taps=L, iterations=4, precision=a.prec)
print(s.describe())
s.iterate_async(3)
import torch; torch.cuda.synchronize()
lib = _lib.load()
buf = (C.c_ulonglong * (4096 * 12))()
assert lib.ctf_debug_gram_phases(buf) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 12).astype(np.int64)
names = ["prologue", "lambda", "gram", "reduce", "objective", "steps", "demix", "energies+mu_b", "tail"]
d = np.diff(a[:, :10], axis=1)
tot = a[:, 9] - a[:, 0]
print("CTA cycles: mean %.0f median %.0f" % (tot.mean(), np.median(tot)))
for i, n in enumerate(names):
    print(f"{n:10s} {d[:, i].mean():9.0f} cycles  {100 * d[:, i].mean() / tot.mean():5.1f} %")
