"""Regenerates tests/golden/*.npz from the CPU oracle (pinned by
tests/test_oracle_kats.py, i.e. the reference's own known-answer tests).

Inputs are not stored: they are regenerated from the recorded seeds with the
product's host generator (ctf_synth_mixtures) or numpy's PCG64, and the
fixture keeps a SHA-256 of the input bytes so a changed generator is caught.
Run: python tests/golden/make_golden.py
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

CASES = {
    # stacked CTF observation (BASELINE (a)), M = N = 2, L = 2
    "stacked_m2_l2": dict(kind="synth", F=17, T=48, M=2, N=2, L=2, K=3, decay=0.6, xseed=1234, seed=11, iters=6),
    # BASELINE configs[0] shape at reduced F/T (full cfg0 runs in the GPU suite against the live oracle)
    "cfg0_small": dict(kind="synth", F=33, T=120, M=2, N=2, L=2, K=10, decay=0.6, xseed=2024, seed=0, iters=5),
    # pre-stacked general observation with unequal taps/bases (reference test configs)
    "general_taps23_bases24": dict(kind="random", F=9, T=30, D=5, taps=[2, 3], bases=[2, 4], xseed=77, seed=5,
                                   iters=5),
}


def make_input(c):
    if c["kind"] == "synth":
        from paper_2510_02382_b200 import synth_mixtures
        raw = synth_mixtures(1, c["F"], c["T"], c["M"], c["N"], c["L"], c["K"], c["decay"], c["xseed"])[0]
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
    for name, c in CASES.items():
        raw, x = make_input(c)
        taps, bases = taps_bases(c)
        r = O.run(O.config(taps, bases, iterations=c["iters"], seed=c["seed"]), x, history=True)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), x_sha256=digest(raw), objective=r["objective"],
                            hist_W=r["hist_W"], hist_B=r["hist_B"], hist_V=r["hist_V"])
        print(name, r["objective"][-1])


if __name__ == "__main__":
    main()
