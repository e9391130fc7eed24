"""Dev: worst per-iteration relative L2 error of the fp32 path against the fp64
oracle on the BASELINE geometries (reduced F), i.e. the margin to 1e-4."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O
from paper_2510_02382_b200 import Session, synth_mixtures
NPROC = os.cpu_count() or 1
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
for (M, L, T, K, rho, F, iters) in [(2, 2, 500, 10, 0.6, 65, 100), (2, 5, 1000, 10, 0.6, 33, 40),
                                     (3, 4, 2000, 20, 0.7, 17, 30), (4, 8, 1000, 20, 0.8, 9, 20)]:
    raw = synth_mixtures(1, F, T, M, M, L, K, rho, 4242)
    ref = O.run(O.config([L] * M, [K] * M, iterations=iters, seed=3, threads=NPROC), O.stack_observation(raw[0], L),
                history=True)
    s = Session(raw.astype(np.complex64), [L] * M, [K] * M, stack_taps=L, iterations=iters, precision="f32", seed=3)
    worst = 0.0
    for it in range(iters):
        s.iterate(1)
        W, B, V, obj = s.download_raw()
        e = max(rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]), rel(V[0], ref["hist_V"][it]))
        worst = max(worst, e)
    fc = abs(obj[0, -1] - ref["objective"][-1]) / abs(ref["objective"][-1])
    print(f"M={M} L={L} T={T} F={F} iters={iters}: worst per-iteration rel L2 {worst:.2e}, final cost {fc:.2e}", flush=True)
