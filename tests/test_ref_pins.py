"""Pins the CPU restatement (oracle/ctf_oracle.cpp) to the REFERENCE'S OWN
CODE: /root/reference/proj/src/{estimator,model,wiener,stft,fft}.cpp compiled
unmodified into oracle/_ref (oracle/Makefile.ref; Eigen and doctest are
absent here, oracle/ref_shims supplies the API subset they use).

1. The shim build is itself pinned by the reference's own unit suite
   (proj/tests/test_{estimator,model,run,stft,synth,wiener,metrics,io}.cpp,
   57 test cases, compiled unmodified against the same build).
2. The restatement equals the reference build on every op and on run()
   trajectories (golden cases after every iteration, BASELINE cfg0 at its
   full 100 iterations, the IP rule, CheckOptions, error paths, STFT).
The GPU path is then pinned to the reference through the committed fixtures
(tests/golden, made by the reference build) in tests/test_gpu_parity.py.
"""
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from oracle import ref as R
from tests.test_oracle_kats import factors_flat, rand_c, rand_psd, rng, wmem, xmem

pytestmark = pytest.mark.skipif(not R.available(), reason="oracle/_ref not built and /root/reference absent")
NPROC = min(os.cpu_count() or 1, 8)


def same(a, b, tol=1e-12):
    a, b = np.asarray(a), np.asarray(b)
    scale = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(a - b))) <= tol * scale


def test_reference_unit_suite_passes_on_the_reference_build():
    """proj/tests/*.cpp (doctest), unmodified: every case passes (the shim
    reproduces the Eigen semantics the reference's own pins rely on)."""
    out = subprocess.run([R.UNIT_TESTS], capture_output=True, text=True, timeout=600)
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", out.stdout)
    assert m, out.stdout + out.stderr
    total, passed, failed = map(int, m.groups())
    assert out.returncode == 0 and failed == 0 and total == passed >= 57, out.stdout[-2000:] + out.stderr[-2000:]


@pytest.mark.parametrize("name", ["stacked_m2_l2", "cfg0_small", "general_taps23_bases24"])
def test_restatement_equals_reference_every_iteration(name):
    from tests.test_golden import load_case
    mg, c, raw, x, taps, bases, g = load_case(name)
    cfg = O.config(taps, bases, iterations=c["iters"], seed=c["seed"])
    a = O.run(cfg, x, history=True)
    b = R.run_history(cfg, x)
    assert same(a["objective"], b["objective"])
    for k in ("hist_W", "hist_B", "hist_V"):
        for it in range(c["iters"]):
            assert same(a[k][it], b[k][it]), (k, it)


def test_restatement_equals_reference_cfg0_full_run():
    """BASELINE configs[0]: M=N=2, L=2, F=513, T=500, K=10, 100 iterations,
    bin-parallel (threads = nproc): final state and the objective after
    every iteration (OptimizationTrace, estimator.hpp:25-40)."""
    raw = R.synth_mixtures(1, 513, 500, 2, 2, 2, 10, 0.6, 20251002)
    x = O.stack_observation(raw[0], 2)
    cfg = O.config([2, 2], [10, 10], iterations=100, seed=0, threads=NPROC)
    a, b = O.run(cfg, x), R.run(cfg, x)
    assert same(a["objective"], b["objective"])
    for k in ("W", "B", "V"):
        assert same(a[k], b[k]), k
    assert np.all(np.diff(b["objective"]) <= 1e-6 * np.abs(b["objective"][:-1]))


@pytest.mark.parametrize("taps,bases,stack", [([2, 3], [2, 4], 0), ([2, 2], [3, 3], 2)])
def test_restatement_equals_reference_ip_rule(taps, bases, stack):
    """update_rule = Ip (estimator.cpp:580-606, ip_update :103-273)."""
    if stack:
        x = O.stack_observation(R.synth_mixtures(1, 9, 40, 2, 2, stack, 3, 0.6, 99)[0], stack)
    else:
        g = rng(8)
        x = xmem(rand_c(g, 9, sum(taps), 30))
    cfg = O.config(taps, bases, iterations=6, seed=4, rule="ip")
    a, b = O.run(cfg, x), R.run(cfg, x)
    assert same(a["objective"], b["objective"])
    for k in ("W", "B", "V"):
        assert same(a[k], b[k]), k


def test_restatement_equals_reference_check_options():
    """CheckOptions (estimator.cpp:560-577): counters and both maxima."""
    x = O.stack_observation(R.synth_mixtures(1, 6, 40, 2, 2, 2, 3, 0.6, 5)[0], 2)
    cfg = O.config([2, 2], [3, 3], iterations=10, seed=1)
    det, nrm, cnt = O.run_checked(cfg, x)
    r = R.run(cfg, x, det_lemma=True, normalization=True)["checks"]
    assert cnt == r["checked_updates"] == 10 * 6 * 4
    assert r["max_det_lemma_error"] <= 1e-10 and r["max_normalization_error"] <= 1e-8
    assert abs(det - r["max_det_lemma_error"]) <= 1e-12 and abs(nrm - r["max_normalization_error"]) <= 1e-12


def test_restatement_equals_reference_error_paths():
    """test_run.cpp:219-268: codes, texts, (iteration, bin)."""
    cfg = O.config([2, 2], [3, 3], iterations=2)
    for mk in (lambda: np.zeros((4, 10, 4), complex),):
        with pytest.raises(O.OracleError) as e1:
            O.run(cfg, mk())
        with pytest.raises(O.OracleError) as e2:
            R.run(cfg, mk())
        assert e1.value.code == e2.value.code == 2 and str(e1.value) == str(e2.value)
    x = xmem(rand_c(rng(2), 2, 4, 10))
    x[1, 3, 2] = np.nan
    for rule in ("ip", "iss"):
        c = O.config([2, 2], [3, 3], iterations=2, rule=rule)
        with pytest.raises(O.OracleError) as e1:
            O.run(c, x)
        with pytest.raises(O.OracleError) as e2:
            R.run(c, x)
        assert e1.value.code == e2.value.code == 4 and str(e1.value) == str(e2.value)
    x = xmem(rand_c(rng(3), 3, 4, 10))
    x[1] = 0
    with pytest.raises(O.OracleError) as e1:
        O.run(cfg, x)
    with pytest.raises(O.OracleError) as e2:
        R.run(cfg, x)
    assert str(e1.value) == str(e2.value)
    assert (e1.value.iteration, e1.value.bin, e1.value.row) == (e2.value.iteration, e2.value.bin, e2.value.row) \
        == (1, 1, e2.value.row)


def test_restatement_equals_reference_ops():
    """Every op of estimator.hpp:56-117, model.cpp:153-227, wiener.cpp:11-49
    on the same seeded inputs."""
    g = rng(21)
    taps, bases = [2, 3], [2, 4]
    F, T, D = 5, 12, 5
    cfg = O.config(taps, bases, iterations=1, seed=9)
    x = xmem(rand_c(g, F, D, T))
    W = wmem(rand_c(g, F, D, D) + 3 * np.eye(D))
    floor = 1e-10 * O.mean_power(x)
    assert O.mean_power(x) == pytest.approx(R.mean_power(x), rel=1e-15)
    Bo, Vo = O.random_factors(cfg, F, T)
    Br, Vr = R.random_factors(cfg, F, T, floor)
    assert np.array_equal(Bo, Br) and np.array_equal(Vo, Vr)
    Y = O.demix(W, x)
    assert same(Y, R.demix(W, x))
    lam = O.compute_psd(cfg, F, T, Bo, Vo, floor)
    assert same(lam, R.compute_psd(cfg, F, T, Bo, Vo, floor))
    for b in range(F):
        a = O.iss_sweep(cfg, W[b], Y[b], lam, b)
        r = R.iss_sweep(cfg, W[b], Y[b], lam, b)
        assert same(a[0], r[0]) and same(a[1], r[1])
    for tap in (0, 1, 2):
        assert same(O.weighted_covariance(x, lam[0], tap, 3), R.weighted_covariance(x, lam[0], tap, 3))
    covs = np.array([rand_psd(g, D).T for _ in range(D)])
    for row in range(D):
        z = O.iss_compute_z(W[0], covs, row)
        assert same(z, R.iss_compute_z(W[0], covs, row))
        assert same(O.iss_apply(W[0], z, row), R.iss_apply(W[0], z, row))
    for n in range(2):
        assert same(O.mu_update_bases(cfg, F, T, Bo, Vo, floor, Y, n), R.mu_update_bases(cfg, F, T, Bo, Vo, floor, Y, n))
        assert same(O.mu_update_activations(cfg, F, T, Bo, Vo, floor, Y, n),
                    R.mu_update_activations(cfg, F, T, Bo, Vo, floor, Y, n))
    a = O.rescale(cfg, F, T, W, Bo, floor, Y)
    r = R.rescale(cfg, F, T, W, Bo, floor, Y)
    for u, v in zip(a, r):
        assert same(u, v)
    for b in range(F):
        assert O.log_abs_det(W[b]) == pytest.approx(R.log_abs_det(W[b]), rel=1e-14)
    assert O.objective_from_parts(cfg, F, T, W, lam, Y) == pytest.approx(R.objective_from_parts(cfg, F, T, W, lam, Y),
                                                                         rel=1e-14)
    assert O.objective(cfg, F, T, W, Bo, Vo, floor, x) == pytest.approx(R.objective(cfg, F, T, W, Bo, Vo, floor, x),
                                                                        rel=1e-14)
    assert same(O.reconstruct_images(cfg, W, x), R.reconstruct_images(cfg, W, x, Bo, Vo, floor))


def test_restatement_equals_reference_stft_bitwise():
    """fft.cpp:9-41, stft.cpp:46-139: the restatement is bit-identical."""
    g = rng(5)
    for n in (1, 2, 8, 1024):
        d = rand_c(g, n)
        assert np.array_equal(O.fft(d), R.fft(d)) and np.array_equal(O.fft(d, True), R.fft(d, True))
    sig = g.standard_normal((2, 3000))
    for wl, hop in ((1024, 256), (256, 128), (64, 16)):
        a, b = O.forward_stft(sig, wl, hop), R.forward_stft(sig, wl, hop)
        assert np.array_equal(a, b)
        assert np.array_equal(O.inverse_stft(a, wl, hop, 3000), R.inverse_stft(b, wl, hop, 3000))


def test_generator_copy_in_reference_library_matches_product():
    """bench.py's reference arm draws its inputs from the generator compiled
    into libctf_ref.so (so it never maps the product library); it is the same
    source as the product's ctf_synth_mixtures."""
    from paper_2510_02382_b200 import synth_mixtures
    assert np.array_equal(R.synth_mixtures(2, 9, 30, 3, 3, 4, 5, 0.7, 77), synth_mixtures(2, 9, 30, 3, 3, 4, 5, 0.7, 77))


def test_fixture_factors_helpers_roundtrip():
    """factors_flat is the layout libctf_ref.so reads (B_n column-major F x K_n)."""
    g = rng(3)
    Bs = [g.random((4, 2)), g.random((4, 3))]
    Vs = [g.random((2, 6)), g.random((3, 6))]
    B, V = factors_flat(Bs, Vs)
    cfg = O.config([1, 1], [2, 3])
    lam = R.compute_psd(cfg, 4, 6, B, V, 1e-12)
    for n in range(2):
        assert np.allclose(lam[n].reshape(6, 4).T, np.maximum(Bs[n] @ Vs[n], 1e-12))
