"""Full-horizon fp32/fp64 parity on every BASELINE config geometry through
the kernel the planner picks by default (no CTF_SWEEP_* overrides).

north_star: fp32 within 1e-4 relative L2 per iteration and 1e-3 relative on
the final cost after the config's full iteration count (cfg1/cfg2: 100,
cfg3/cfg4: 50); fp64 within 1e-9 after every iteration. F is reduced so the
CPU oracle (the checker, pinned to the reference's own code by
tests/test_ref_pins.py) finishes in seconds; T, M, N, L, K and the tap
variance are the config's. The separated signals (the GPU's projected-back
images, wiener.cpp:11-49) are compared after the last iteration too."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_02382_b200 import Session, synth_mixtures

pytestmark = pytest.mark.gpu
NPROC = os.cpu_count() or 1


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


# name, M(=N), L, T, K, rho, F, iterations, expected default kernel (substring), cluster size
CONFIGS = [
    ("cfg1", 2, 5, 1000, 10, 0.6, 17, 100, "gram_kernel", 0),
    ("cfg2", 3, 4, 2000, 20, 0.7, 17, 100, "gram_kernel", 0),
    ("cfg3", 4, 8, 1000, 20, 0.8, 9, 50, "fsplit_kernel", 2),
    ("cfg4", 6, 10, 4000, 16, 0.85, 5, 50, "fsplit_kernel", 8),
]


@pytest.mark.parametrize("name,M,L,T,K,rho,F,iters,kernel,cs", CONFIGS)
def test_fp32_full_horizon_default_kernel(name, M, L, T, K, rho, F, iters, kernel, cs):
    for v in ("CTF_SWEEP_KIND", "CTF_SWEEP_VARIANT", "CTF_FSPLIT_AG", "CTF_FSPLIT_PAIR"):
        assert v not in os.environ
    _horizon(name, M, L, T, K, rho, F, iters, kernel, cs)


@pytest.mark.parametrize("name,M,L,T,K,rho,F,iters,kernel,cs", CONFIGS[2:])
@pytest.mark.parametrize("pair", [0, 1])
def test_fp32_full_horizon_fsplit_step_pairs(name, M, L, T, K, rho, F, iters, kernel, cs, pair, monkeypatch):
    """Both frame-split step schedules (one ISS step per exchange, and the
    step pairs: two steps per pass from the expanded sums) over the full
    horizon of cfg3 / cfg4."""
    monkeypatch.setenv("CTF_SWEEP_KIND", "5")
    monkeypatch.setenv("CTF_FSPLIT_AG", "1")
    monkeypatch.setenv("CTF_FSPLIT_PAIR", str(pair))
    _horizon(name, M, L, T, K, rho, F, iters, kernel, cs)


def _horizon(name, M, L, T, K, rho, F, iters, kernel, cs):
    seed = 31
    raw = synth_mixtures(1, F, T, M, M, L, K, rho, 4242 + M * L)
    x = O.stack_observation(raw[0], L)
    taps, bases = [L] * M, [K] * M
    ref = O.run(O.config(taps, bases, iterations=iters, seed=seed, threads=NPROC), x, history=True)
    s = Session(raw.astype(np.complex64), taps, bases, stack_taps=L, iterations=iters, precision="f32", seed=seed)
    d = json.loads(s.describe())
    assert kernel in d["sweep_kernel"], d
    if cs:
        assert d["cluster"] == cs, d
    worst = 0.0
    for it in range(iters):
        s.iterate(1)
        W, B, V, obj = s.download_raw()
        e = max(rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]),
                rel(V[0], ref["hist_V"][it]))
        worst = max(worst, e)
        assert e <= 1e-4, f"{name} it={it + 1}: {e:.2e}"
    final = abs(obj[0, -1] - ref["objective"][-1]) / abs(ref["objective"][-1])
    assert final <= 1e-3, f"{name} final cost {final:.2e}"
    img = s.project_back()
    s.close()
    want = O.reconstruct_images(O.config(taps, bases), ref["W"], x)
    assert rel(img[:, 0], want) <= 1e-4, name
    print(f"{name}: worst per-iteration rel L2 {worst:.2e}, final cost {final:.2e}")


def test_fp64_cfg1_shape_full_bins_20_iterations():
    """cfg1 geometry at its full F = 513 in fp64 (the headline dtype): 1e-9
    after every one of 20 iterations, W, B, V, objective and the separated
    signals at the end."""
    F, T, M, L, K, iters, seed = 513, 1000, 2, 5, 10, 20, 8
    raw = synth_mixtures(1, F, T, M, M, L, K, 0.6, 555)
    x = O.stack_observation(raw[0], L)
    taps, bases = [L] * M, [K] * M
    ref = O.run(O.config(taps, bases, iterations=iters, seed=seed, threads=NPROC), x, history=True)
    s = Session(raw, taps, bases, stack_taps=L, iterations=iters, precision="f64", seed=seed)
    for it in range(iters):
        s.iterate(1)
        W, B, V, obj = s.download_raw()
        errs = (rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]),
                rel(V[0], ref["hist_V"][it]), abs(obj[0, it] - ref["objective"][it]) / abs(ref["objective"][it]))
        assert max(errs) <= 1e-9, (it + 1, errs)
    img = s.project_back()
    s.close()
    assert rel(img[:, 0], O.reconstruct_images(O.config(taps, bases), ref["W"], x)) <= 1e-9


def test_tensor_core_gram_variant_cfg3(monkeypatch):
    """The tcgen05 Gram variant of the covariance-domain kernel (3xTF32 split,
    per-stage TMEM partials summed in fp32; CTF_GRAM_TC=1 selects it, the
    frame-split kernel stays the default for this tile) on the cfg3 geometry:
    1e-4 relative L2 after every one of 20 iterations."""
    monkeypatch.setenv("CTF_SWEEP_KIND", "4")
    monkeypatch.setenv("CTF_GRAM_TC", "1")
    M, L, T, K, rho, F, iters, seed = 4, 8, 1000, 20, 0.8, 9, 20, 12
    raw = synth_mixtures(1, F, T, M, M, L, K, rho, 4242 + M * L)
    ref = O.run(O.config([L] * M, [K] * M, iterations=iters, seed=seed, threads=NPROC),
                O.stack_observation(raw[0], L), history=True)
    s = Session(raw.astype(np.complex64), [L] * M, [K] * M, stack_taps=L, iterations=iters, precision="f32",
                seed=seed)
    d = json.loads(s.describe())
    assert "gram_kernel" in d["sweep_kernel"] and d["smem_bytes"] > 210000, d  # the TC variant's stage buffers
    for it in range(iters):
        s.iterate(1)
        W, B, V, obj = s.download_raw()
        e = max(rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]),
                rel(V[0], ref["hist_V"][it]))
        assert e <= 1e-4, f"it={it + 1}: {e:.2e}"
    s.close()
