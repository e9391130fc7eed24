"""Dev: per-phase cycle counts of fsplit_kernel (the cluster's CTA 0) from an
instrumented build: DEV_FILE=ctf_sweep_fsplit tools/dev_build.sh fph
-DCTF_PHASE_TIMING, then CTF_DEV_LIB=tools/dev/fph/libctfiss.so python
tools/fsplit_phase.py --cfg 3."""
import argparse, ctypes as C, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_02382_b200 import _lib, Session, synth_mixtures
ap = argparse.ArgumentParser(); ap.add_argument("--cfg", type=int, default=3); a = ap.parse_args()
B, F, T, M, N, L, K, dec = {3: (2, 2049, 1000, 4, 4, 8, 20, 0.8), 4: (2, 1025, 4000, 6, 6, 10, 16, 0.85)}[a.cfg]
x = synth_mixtures(B, F, T, M, N, L, K, dec, 1, precision="f32")
s = Session(x, [L] * N, [K] * N, stack_taps=L, iterations=4, precision="f32")
print(s.describe())
s.iterate_async(3)  # no finalize pass (it would overwrite the first phases only)
import torch; torch.cuda.synchronize()
lib = _lib.load()
buf = (C.c_ulonglong * (4096 * 12))()
assert lib.ctf_debug_fsplit_phases(buf) == 0
ph = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 12).astype(np.int64)[: B * F]
bounds = [0, 1, 2, 3, 4, 5, 6, 7, 8]
names = ["prologue", "lambda", "demix", "objective", "sweep", "epilogue", "mu_b", "tail"]
tot = ph[:, 8] - ph[:, 0]
print("CTA-0 cycles per bin: mean %.0f median %.0f" % (tot.mean(), np.median(tot)))
for i, n in enumerate(names):
    d = ph[:, bounds[i + 1]] - ph[:, bounds[i]]
    print(f"{n:16s} {d.mean():10.0f} cycles  {100 * d.mean() / tot.mean():5.1f} %")
