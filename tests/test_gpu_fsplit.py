"""GPU parity of the frame-split cluster kernel (ctf_fsplit.cuh, kind 5): the
wide stacked tiles of BASELINE configs[3] (M=N=4, L=8, R=32, T=1000) and
configs[4] (M=N=6, L=10, R=60, T=4000), frames split over a thread-block
cluster, against the CPU oracle (fp32: <= 1e-4 relative L2 per iteration).
Every compiled cluster size is forced once through CTF_SWEEP_VARIANT."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_02382_b200 import DegeneracyError, Session, synth_mixtures

pytestmark = pytest.mark.gpu
NPROC = os.cpu_count() or 1


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def history(x, L, K, iters, seed):
    M = x.shape[3]
    s = Session(x, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision="f32", seed=seed)
    d = json.loads(s.describe())
    out = []
    for _ in range(iters):
        s.iterate(1)
        out.append(s.download_raw())
    s.close()
    return d, out


# (M, L, T, K, rho, F, iters, variant "rmax,ft,rreg,nt", cluster size, exchange: 0 owner, 1 all-gather,
#  step pairs: 1 two ISS steps per pass and exchange)
CASES = [
    (4, 8, 1000, 20, 0.8, 9, 4, "32,2,16,128", 4, 0, 0),
    (4, 8, 1000, 20, 0.8, 5, 3, "32,2,16,256", 2, 0, 0),
    (4, 8, 1000, 20, 0.8, 5, 3, "32,1,16,128", 8, 0, 0),
    (4, 8, 1000, 20, 0.8, 5, 3, "32,4,16,128", 2, 0, 0),
    (6, 10, 4000, 16, 0.85, 2, 3, "60,2,24,128", 16, 0, 0),
    (6, 10, 4000, 16, 0.85, 2, 2, "60,2,32,256", 8, 0, 0),
    (4, 8, 1000, 20, 0.8, 5, 3, "32,4,16,128", 2, 1, 0),
    (4, 8, 1000, 20, 0.8, 9, 3, "32,2,16,128", 4, 1, 0),
    (6, 10, 4000, 16, 0.85, 2, 3, "60,2,32,256", 8, 1, 0),
    (4, 8, 1000, 20, 0.8, 5, 4, "32,4,16,128", 2, 1, 1),
    (4, 8, 1000, 20, 0.8, 9, 4, "32,2,16,128", 4, 1, 1),
    (6, 10, 4000, 16, 0.85, 2, 3, "60,2,32,256", 8, 1, 1),
]


@pytest.mark.parametrize("M,L,T,K,rho,F,iters,variant,cs,ag,pair", CASES)
def test_fsplit_fp32_every_iteration(M, L, T, K, rho, F, iters, variant, cs, ag, pair, monkeypatch):
    monkeypatch.setenv("CTF_SWEEP_KIND", "5")
    monkeypatch.setenv("CTF_SWEEP_VARIANT", variant)
    monkeypatch.setenv("CTF_FSPLIT_AG", str(ag))
    monkeypatch.setenv("CTF_FSPLIT_PAIR", str(pair))
    raw = synth_mixtures(1, F, T, M, M, L, K, rho, 77 + M * L)
    ref = O.run(O.config([L] * M, [K] * M, iterations=iters, seed=3, threads=NPROC),
                O.stack_observation(raw[0], L), history=True)
    d, hist = history(raw.astype(np.complex64), L, K, iters, 3)
    assert "fsplit_kernel" in d["sweep_kernel"] and d["cluster"] == cs, d
    for it, (W, B, V, obj) in enumerate(hist):
        e = max(rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]),
                rel(V[0], ref["hist_V"][it]))
        eo = abs(obj[0, it] - ref["objective"][it]) / abs(ref["objective"][it])
        assert e <= 1e-4 and eo <= 1e-4, f"{variant} it={it + 1}: state {e:.2e} objective {eo:.2e}"


def test_fsplit_is_the_default_for_cfg4_and_deterministic():
    """cfg4's tile (R=60, T=4000) selects the frame-split kernel by default;
    reruns are bit-identical (fixed-order sums inside and across CTAs) and a
    batch of two mixtures equals the two single runs."""
    M, L, T, K, F = 6, 10, 4000, 16, 2
    raw = synth_mixtures(2, F, T, M, M, L, K, 0.85, 5).astype(np.complex64)
    outs = []
    for _ in range(2):
        s = Session(raw, [L] * M, [K] * M, stack_taps=L, iterations=2, precision="f32", seed=1)
        assert "fsplit_kernel" in json.loads(s.describe())["sweep_kernel"]
        s.iterate(2)
        outs.append(s.download_raw())
        s.close()
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(a, b)
    s = Session(raw[1:], [L] * M, [K] * M, stack_taps=L, iterations=2, precision="f32", seed=2)  # mixture b: seed + b
    s.iterate(2)
    W1, B1, V1, o1 = s.download_raw()
    s.close()
    assert np.array_equal(W1[0], outs[0][0][1]) and np.array_equal(o1[0], outs[0][3][1])


def test_fsplit_error_paths(monkeypatch):
    """test_run.cpp:219-268 semantics on the cluster kernel: a NaN sample ->
    "non-finite"; silent bins -> the steering degeneracy at iteration 1 of the
    lowest silent bin with the oracle's message (every CTA of the cluster
    leaves the sweep at the same step)."""
    monkeypatch.setenv("CTF_SWEEP_KIND", "5")
    M, L, K, F, T = 4, 8, 4, 6, 1000
    raw = synth_mixtures(1, F, T, M, M, L, K, 0.8, 21).astype(np.complex64)
    s = Session(raw, [L] * M, [K] * M, stack_taps=L, iterations=2, precision="f32", seed=1)
    assert "fsplit_kernel" in json.loads(s.describe())["sweep_kernel"]
    s.close()
    bad = raw.copy()
    bad[0, 3, 700, 1] = np.nan
    with pytest.raises(DegeneracyError) as e:
        s = Session(bad, [L] * M, [K] * M, stack_taps=L, iterations=2, precision="f32", seed=1)
        s.iterate(2)
    assert "non-finite" in str(e.value)
    silent = raw.copy()
    silent[0, 2] = 0
    silent[0, 4] = 0
    ref_err = None
    try:
        O.run(O.config([L] * M, [K] * M, iterations=2, seed=1), O.stack_observation(silent[0].astype(complex), L))
    except O.OracleError as oe:
        ref_err = oe
    assert ref_err is not None and ref_err.iteration == 1 and ref_err.bin == 2
    with pytest.raises(DegeneracyError) as e:
        s = Session(silent, [L] * M, [K] * M, stack_taps=L, iterations=2, precision="f32", seed=1)
        s.iterate(2)
    assert e.value.iteration == 1 and e.value.bin == 2
    assert str(e.value).split(" (iteration")[0] == str(ref_err).split(" (iteration")[0]


def test_fsplit_frame_counts_off_the_tile(monkeypatch):
    """T just above (CS - 1) * TC and just below CS * TC: the last CTA holds a
    few frames / almost a full tile; the halos cross the ragged boundary."""
    monkeypatch.setenv("CTF_SWEEP_KIND", "5")
    M, L, K, F = 4, 8, 5, 3
    for T in (769, 1023):
        raw = synth_mixtures(1, F, T, M, M, L, K, 0.8, T)
        ref = O.run(O.config([L] * M, [K] * M, iterations=2, seed=2, threads=NPROC),
                    O.stack_observation(raw[0], L), history=True)
        d, hist = history(raw.astype(np.complex64), L, K, 2, 2)
        assert "fsplit_kernel" in d["sweep_kernel"], d
        for it, (W, B, V, obj) in enumerate(hist):
            e = max(rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]),
                    rel(V[0], ref["hist_V"][it]))
            assert e <= 1e-4, f"T={T} it={it + 1}: {e:.2e}"
