"""Regenerates tests/golden/*.npz from the REFERENCE'S OWN CODE
(oracle/_ref/libctf_ref.so: /root/reference/proj/src/*.cpp compiled
unmodified by oracle/Makefile.ref). Run here, where /root/reference exists:

    python tests/golden/make_golden.py

Inputs are not stored: they are regenerated from the recorded seeds with
BASELINE's generator (the copy compiled into libctf_ref.so, the same source
as the product's ctf_synth_mixtures) or numpy's PCG64, and each fixture keeps
a SHA-256 of the input bytes so a changed generator is caught.

History cases store the state after every iteration (run() with iterations
= k for k = 1..n: run() is deterministic for a fixed seed). Checkpoint cases
(BASELINE cfg0 at full size) store the objective after every iteration of a
100-iteration run and the state after the listed iteration counts.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

PRODUCER = "oracle/_ref (reference sources proj/src/*.cpp, unmodified, Eigen-API shim)"

CASES = {
    # stacked CTF observation (BASELINE (a)), M = N = 2, L = 2
    "stacked_m2_l2": dict(kind="synth", F=17, T=48, M=2, N=2, L=2, K=3, decay=0.6, xseed=1234, seed=11, iters=6),
    # BASELINE configs[0] shape at reduced F/T
    "cfg0_small": dict(kind="synth", F=33, T=120, M=2, N=2, L=2, K=10, decay=0.6, xseed=2024, seed=0, iters=5),
    # pre-stacked general observation with unequal taps/bases (reference test configs)
    "general_taps23_bases24": dict(kind="random", F=9, T=30, D=5, taps=[2, 3], bases=[2, 4], xseed=77, seed=5,
                                   iters=5),
    # BASELINE configs[0] exactly (complex128, 100 iterations): objective trace + checkpoints
    "cfg0_full": dict(kind="synth", F=513, T=500, M=2, N=2, L=2, K=10, decay=0.6, xseed=20251002, seed=0,
                      iters=100, checkpoints=[1, 100]),
}


def make_input(c):
    if c["kind"] == "synth":
        from oracle import ref as R
        if R.available():
            gen = R.synth_mixtures
        else:  # GPU box without the reference build: the product's copy of the same generator source
            from paper_2510_02382_b200 import synth_mixtures as gen
        raw = gen(1, c["F"], c["T"], c["M"], c["N"], c["L"], c["K"], c["decay"], c["xseed"])[0]
        return raw, O.stack_observation(raw, c["L"])
    g = np.random.default_rng(c["xseed"])
    x = g.standard_normal((c["F"], c["T"], c["D"])) + 1j * g.standard_normal((c["F"], c["T"], c["D"]))
    return x, x


def taps_bases(c):
    if c["kind"] == "synth":
        return [c["L"]] * c["N"], [c["K"]] * c["N"]
    return c["taps"], c["bases"]


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    from oracle import ref as R
    for name, c in CASES.items():
        raw, x = make_input(c)
        taps, bases = taps_bases(c)
        cfg = O.config(taps, bases, iterations=c["iters"], seed=c["seed"], threads=8)
        if "checkpoints" in c:
            out = {}
            for k in c["checkpoints"]:
                ck = O.config(taps, bases, iterations=k, seed=c["seed"], threads=8)
                r = R.run(ck, x)
                out.update({f"W_{k}": r["W"], f"B_{k}": r["B"], f"V_{k}": r["V"]})
                if k == c["iters"]:
                    out["objective"] = r["objective"]
            np.savez_compressed(os.path.join(HERE, f"{name}.npz"), x_sha256=digest(raw), producer=PRODUCER,
                                checkpoints=np.array(c["checkpoints"]), **out)
        else:
            r = R.run_history(cfg, x)
            np.savez_compressed(os.path.join(HERE, f"{name}.npz"), x_sha256=digest(raw), producer=PRODUCER,
                                objective=r["objective"], hist_W=r["hist_W"], hist_B=r["hist_B"],
                                hist_V=r["hist_V"])
        print(name, r["objective"][-1])


if __name__ == "__main__":
    main()
