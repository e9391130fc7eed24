"""Dev: per-iteration relative L2 error of the fp32 GPU path (W, B, V
separately) against the fp64 oracle on a BASELINE geometry, for the default
kernel and a forced kernel kind (CTF_SWEEP_KIND), plus the error an fp64
run on complex64-rounded inputs shows (what input quantisation alone costs).
usage: python tools/fp32_drift.py M L T K rho F iters [kinds...]"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

M, L, T, K = map(int, sys.argv[1:5])
rho, F, iters = float(sys.argv[5]), int(sys.argv[6]), int(sys.argv[7])
kinds = sys.argv[8:] or ["default"]
seed = 31
rel = lambda a, b: float(np.linalg.norm(np.ravel(a - b)) / np.linalg.norm(np.ravel(b)))
if os.environ.get("FP32_DRIFT_CHILD"):
    from paper_2510_02382_b200 import Session, synth_mixtures
    import json
    raw = synth_mixtures(1, F, T, M, M, L, K, rho, 4242 + M * L)
    ref = O.run(O.config([L] * M, [K] * M, iterations=iters, seed=seed, threads=os.cpu_count()),
                O.stack_observation(raw[0], L), history=True)
    s = Session(raw.astype(np.complex64), [L] * M, [K] * M, stack_taps=L, iterations=iters, precision="f32", seed=seed)
    print(json.loads(s.describe())["sweep_kernel"])
    for it in range(iters):
        s.iterate(1)
        W, B, V, obj = s.download_raw()
        eW, eB, eV = rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]), rel(V[0], ref["hist_V"][it])
        eo = abs(obj[0, it] - ref["objective"][it]) / abs(ref["objective"][it])
        if it < 5 or (it + 1) % 5 == 0:
            wb = np.linalg.norm(W[0] - ref["hist_W"][it].reshape(F, -1), axis=1) / np.linalg.norm(
                ref["hist_W"][it].reshape(F, -1), axis=1)
            print(f"it {it + 1:3d}  W {eW:.2e}  B {eB:.2e}  V {eV:.2e}  obj {eo:.2e}  worst bin {int(np.argmax(wb))} "
                  f"{wb.max():.2e}", flush=True)
else:
    for k in kinds:
        env = dict(os.environ, FP32_DRIFT_CHILD="1")
        if k != "default":
            env["CTF_SWEEP_KIND"] = k
        print(f"== kind {k}", flush=True)
        subprocess.run([sys.executable] + sys.argv, env=env, check=False)
