"""The reference's own known-answer and property tests, re-expressed against the
CPU oracle (oracle/ctf_oracle.cpp). This is what pins the oracle: the
reference ships no stored golden files; its pins are these
seeded KATs. Each test cites the reference test it restates. The brute-force
checks here are independent numpy loops (the role of proj/tests/oracles.hpp).

Layout helpers: the oracle stores every per-bin matrix column-major, so a
numpy "memory" array [F, cols, rows] is the transpose of the matrix.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O


def rng(seed):
    return np.random.default_rng(seed)


def rand_c(g, *shape):
    return g.standard_normal(shape) + 1j * g.standard_normal(shape)


def rand_psd(g, m):  # oracles.hpp:213-218
    a = rand_c(g, m, m)
    q = a @ a.conj().T / m + 0.05 * np.eye(m)
    return 0.5 * (q + q.conj().T)


def wmem(Wmats):  # [F, R, D] matrices -> oracle memory [F, D, R]
    return np.ascontiguousarray(np.transpose(Wmats, (0, 2, 1)))


def xmem(xmats):  # [F, D, T] matrices -> oracle memory [F, T, D]
    return np.ascontiguousarray(np.transpose(xmats, (0, 2, 1)))


def factors_flat(Bs, Vs):  # lists of (F, K) and (K, T) -> flat col-major
    return (np.concatenate([b.T.ravel() for b in Bs]), np.concatenate([v.T.ravel() for v in Vs]))


def factors_unflat(B, V, F, T, Ks):
    Bs, Vs, ob, ov = [], [], 0, 0
    for K in Ks:
        Bs.append(B[ob:ob + F * K].reshape(K, F).T)
        Vs.append(V[ov:ov + K * T].reshape(T, K).T)
        ob += F * K
        ov += K * T
    return Bs, Vs


def cofactor_det(m):  # oracles.hpp:40-57
    n = m.shape[0]
    if n == 1:
        return m[0, 0]
    acc = 0
    for c in range(n):
        minor = np.delete(np.delete(m, 0, axis=0), c, axis=1)
        acc += (-1) ** c * m[0, c] * cofactor_det(minor)
    return acc


def brute_objective(Wm, Bs, Vs, floor, xm, taps):  # oracles.hpp:59-86
    F, D, T = xm.shape
    obj = 0.0
    for i in range(F):
        r = 0
        for n, L in enumerate(taps):
            lam = np.maximum(Bs[n] @ Vs[n], floor)
            for l in range(L):
                y = Wm[i, r] @ xm[i]
                for j in range(l, T):
                    obj += math.log(lam[i, j - l]) + abs(y[j]) ** 2 / lam[i, j - l]
                r += 1
        obj -= 2.0 * T * math.log(abs(cofactor_det(Wm[i])))
    return obj


# ---------------------------------------------------------------------------
# objective (proj/tests/test_estimator.cpp:30-105)

def test_objective_ratio_term_collapses_when_lambda_equals_y2():
    """test_estimator.cpp:30-63 — K=1 factors representing |x|^2 exactly."""
    g = rng(5)
    F, T = 3, 4
    cfg = O.config([1, 1], [1, 1])
    Bs, Vs, x = [], [], np.zeros((F, 2, T), complex)
    for n in range(2):
        b = g.uniform(0.3, 2.0, (F, 1))
        v = g.uniform(0.3, 2.0, (1, T))
        Bs.append(b)
        Vs.append(v)
        x[:, n, :] = np.sqrt(b @ v) * np.exp(1j * g.uniform(0, 6.28, (F, T)))
    W = np.tile(np.eye(2, dtype=complex), (F, 1, 1))
    B, V = factors_flat(Bs, Vs)
    got = O.objective(cfg, F, T, wmem(W), B, V, 1e-15, xmem(x))
    want = float(np.sum(np.log(np.abs(x) ** 2) + 1.0))
    assert got == pytest.approx(want, rel=1e-12)


def test_objective_determinant_term_for_scaled_identity():
    """test_estimator.cpp:65-82."""
    F, T = 1, 6
    cfg = O.config([1, 1], [1, 1])
    x = np.zeros((F, 2, T), complex)
    B, V = factors_flat([np.ones((1, 1))] * 2, [np.ones((1, T))] * 2)
    W = np.tile(np.eye(2, dtype=complex), (F, 1, 1))
    base = O.objective(cfg, F, T, wmem(W), B, V, 1e-12, xmem(x))
    scaled = O.objective(cfg, F, T, wmem(2 * W), B, V, 1e-12, xmem(x))
    assert scaled - base == pytest.approx(-2.0 * T * math.log(4.0), rel=1e-12)


def test_objective_matches_brute_force_loop():
    """test_estimator.cpp:84-95 vs the cofactor brute force of oracles.hpp:59-86."""
    g = rng(17)
    F, T, taps, bases = 3, 4, [2, 2], [2, 3]
    cfg = O.config(taps, bases)
    x = rand_c(g, F, 4, T)
    Bs = [g.uniform(0.2, 1.5, (F, k)) for k in bases]
    Vs = [g.uniform(0.2, 1.5, (k, T)) for k in bases]
    W = np.tile(np.eye(4, dtype=complex), (F, 1, 1)) + 0.3 * rand_c(g, F, 4, 4)
    B, V = factors_flat(Bs, Vs)
    got = O.objective(cfg, F, T, wmem(W), B, V, 1e-9, xmem(x))
    want = brute_objective(W, Bs, Vs, 1e-9, x, taps)
    assert got == pytest.approx(want, rel=1e-10)


def test_objective_rejects_singular_demixing():
    """test_estimator.cpp:97-105."""
    g = rng(23)
    cfg = O.config([1, 1], [1, 1])
    x = rand_c(g, 1, 2, 3)
    B, V = factors_flat([g.uniform(0.2, 1.5, (1, 1))] * 2, [g.uniform(0.2, 1.5, (1, 3))] * 2)
    W = np.eye(2, dtype=complex)[None].copy()
    W[0, 1] = W[0, 0]
    with pytest.raises(O.OracleError) as e:
        O.objective(cfg, 1, 3, wmem(W), B, V, 1e-9, xmem(x))
    assert e.value.code == 4


def test_log_abs_det_known_values():
    """log|det| via pivoted LU (estimator.cpp:41-53)."""
    g = rng(3)
    for n in (1, 2, 4, 7):
        m = rand_c(g, n, n)
        assert O.log_abs_det(m.T.copy()) == pytest.approx(np.linalg.slogdet(m)[1], rel=1e-12, abs=1e-12)
    with pytest.raises(O.OracleError):
        O.log_abs_det(np.full((2, 2), 1e-200, complex))  # |det| < 1e-300


# ---------------------------------------------------------------------------
# weighted covariance and demix (test_estimator.cpp:107-177)

def test_weighted_covariance_cases():
    g = rng(31)
    # zero mixture -> zero matrix
    q = O.weighted_covariance(np.zeros((1, 4, 2), complex), np.ones((4, 1)), 0, 0)
    assert np.linalg.norm(q) == 0.0
    # single frame, unit lambda: the plain outer product
    x1 = rand_c(g, 1, 2, 1)
    q = O.weighted_covariance(xmem(x1), np.ones((1, 1)), 0, 0).T
    assert np.linalg.norm(q - np.outer(x1[0, :, 0], x1[0, :, 0].conj())) < 1e-14
    # random instance vs the explicit loop (oracles.hpp:88-101)
    x = rand_c(g, 2, 2, 3)
    lam = np.array([[0.5, 1.5, 0.7], [2.0, 0.9, 1.1]])  # (F=2, T=3)
    for tap in (0, 1):
        got = O.weighted_covariance(xmem(x), np.ascontiguousarray(lam.T), tap, 1).T
        want = np.zeros((2, 2), complex)
        for j in range(tap, 3):
            want += np.outer(x[1, :, j], x[1, :, j].conj()) / lam[1, j - tap]
        want /= 3
        assert np.linalg.norm(got - want) < 1e-12 * np.linalg.norm(want)
    # Hermitian PSD
    x = rand_c(g, 1, 4, 10)
    q = O.weighted_covariance(xmem(x), np.full((10, 1), 0.8), 1, 0).T
    assert np.linalg.norm(q - q.conj().T) < 1e-12
    assert np.linalg.eigvalsh(q).min() > -1e-10 * np.trace(q).real


def test_demix_cases():
    g = rng(37)
    x = rand_c(g, 2, 4, 3)
    W = np.tile(np.eye(4, dtype=complex), (2, 1, 1))
    y = O.demix(wmem(W), xmem(x))
    assert np.linalg.norm(np.transpose(y, (0, 2, 1)) - x) == 0.0  # identity stacks channels in order
    y0 = O.demix(wmem(W), np.zeros((2, 3, 4), complex))
    assert np.linalg.norm(y0) == 0.0
    x = rand_c(g, 2, 4, 5)
    W = rand_c(g, 2, 4, 4)
    got = np.transpose(O.demix(wmem(W), xmem(x)), (0, 2, 1))
    for i in range(2):
        want = np.array([[sum(W[i, r, m] * x[i, m, j] for m in range(4)) for j in range(5)] for r in range(4)])
        assert np.linalg.norm(got[i] - want) < 1e-12 * np.linalg.norm(want)


# ---------------------------------------------------------------------------
# ISS (test_estimator.cpp:236-392)

def steering_coordinate_cost(w, q, p, r, z):  # test_estimator.cpp:15-26
    moved = w[p].conj() - np.conj(z) * w[r].conj()
    cost = (moved.conj() @ q @ moved).real
    if p == r:
        cost += -2.0 * math.log(abs(1.0 - z))
    return cost


def covs_mem(covs):
    return np.ascontiguousarray(np.stack([c.T for c in covs]))


def test_iss_z_fixed_point_diagonal_unit_power():
    """test_estimator.cpp:239-251."""
    m = 3
    covs = []
    for p in range(m):
        d = np.array([0.5 + 0.5 * ((k + p) % 3) for k in range(m)])
        d[1] = 1.0
        covs.append(np.diag(d).astype(complex))
    z = O.iss_compute_z(np.eye(m, dtype=complex).T.copy(), covs_mem(covs), 1)
    assert np.linalg.norm(z) < 1e-14


def test_iss_z_minimizes_each_coordinate_grid_search():
    """test_estimator.cpp:253-276 (41 x 41 grid around the closed form)."""
    g = rng(43)
    for _ in range(6):
        m = 2 + int(g.integers(0, 3))
        w = np.eye(m) + 0.4 * rand_c(g, m, m)
        covs = [rand_psd(g, m) for _ in range(m)]
        row = int(g.integers(0, m))
        z = O.iss_compute_z(w.T.copy(), covs_mem(covs), row)
        a = np.arange(-20, 21) * 0.025
        for p in range(m):
            at = steering_coordinate_cost(w, covs[p], p, row, z[p])
            best = min(steering_coordinate_cost(w, covs[p], p, row, z[p] + complex(da, db)) for da in a for db in a)
            assert best - at >= -1e-9


def test_iss_z_gradient_vanishes():
    """test_estimator.cpp:278-299 (central differences, h = 1e-6)."""
    g = rng(44)
    m = 4
    w = np.eye(m) + 0.4 * rand_c(g, m, m)
    covs = [rand_psd(g, m) for _ in range(m)]
    z = O.iss_compute_z(w.T.copy(), covs_mem(covs), 2)
    h = 1e-6
    for p in range(m):
        c = lambda v: steering_coordinate_cost(w, covs[p], p, 2, v)
        assert abs((c(z[p] + h) - c(z[p] - h)) / (2 * h)) < 1e-6
        assert abs((c(z[p] + 1j * h) - c(z[p] - 1j * h)) / (2 * h)) < 1e-6


def test_iss_z_self_coordinate_is_real():
    """test_estimator.cpp:301-309."""
    g = rng(45)
    w = np.eye(3) + 0.4 * rand_c(g, 3, 3)
    covs = [rand_psd(g, 3) for _ in range(3)]
    assert O.iss_compute_z(w.T.copy(), covs_mem(covs), 0)[0].imag == 0.0


def test_iss_apply_zero_noop_and_determinant_lemma():
    """test_estimator.cpp:315-335: det(W - z w_r^T) = det(W) (1 - z_r)."""
    g = rng(47)
    w = rand_c(g, 3, 3)
    assert np.array_equal(O.iss_apply(w.T.copy(), np.zeros(3, complex), 1), w.T)
    for _ in range(50):
        m = 2 + int(g.integers(0, 5))
        w = np.eye(m) + 0.5 * rand_c(g, m, m)
        z = rand_c(g, m)
        row = int(g.integers(0, m))
        after = O.iss_apply(w.T.copy(), z, row).T
        pred = np.linalg.det(w) * (1 - z[row])
        assert abs(np.linalg.det(after) - pred) <= 1e-10 * abs(np.linalg.det(after))


def test_iss_sweep_steps_leave_unit_weighted_power():
    """test_estimator.cpp:337-357."""
    g = rng(48)
    cfg = O.config([2, 2], [1, 1])
    x = rand_c(g, 1, 4, 30)
    lam = [np.full((1, 30), 0.7), np.full((1, 30), 1.3)]
    w = np.eye(4, dtype=complex)
    covs = [O.weighted_covariance(xmem(x), np.ascontiguousarray(lam[n].T), l, 0).T for n in (0, 1) for l in (0, 1)]
    for r in range(4):
        z = O.iss_compute_z(w.T.copy(), covs_mem(covs), r)
        w = O.iss_apply(w.T.copy(), z, r).T
        power = w[r] @ covs[r] @ w[r].conj()
        assert abs(power - 1.0) < 1e-8


def test_estimate_domain_sweep_equals_covariance_domain():
    """test_estimator.cpp:360-392 — the iss_sweep run() uses equals Eq. 17 ops."""
    g = rng(53)
    cfg = O.config([2, 2], [1, 1])
    F, T = 2, 12
    x = rand_c(g, F, 4, T)
    lam = np.stack([g.uniform(0.4, 1.8, (F, T)) for _ in range(2)])  # (N, F, T)
    lam_mem = np.ascontiguousarray(np.transpose(lam, (0, 2, 1)))
    for b in range(F):
        w = np.eye(4) + 0.3 * rand_c(g, 4, 4)
        y = w @ x[b]
        wf, yf = O.iss_sweep(cfg, w.T.copy(), y.T.copy(), lam_mem, b)
        wf, yf = wf.T, yf.T
        wr = w.copy()
        for r in range(4):
            covs = [O.weighted_covariance(xmem(x), np.ascontiguousarray(lam[n].T), l, b).T
                    for n in (0, 1) for l in (0, 1)]
            wr = O.iss_apply(wr.T.copy(), O.iss_compute_z(wr.T.copy(), covs_mem(covs), r), r).T
        assert np.linalg.norm(wf - wr) < 1e-10 * np.linalg.norm(wr)
        assert np.linalg.norm(yf - wf @ x[b]) < 1e-10 * np.linalg.norm(yf)


def test_single_tap_sweep_matches_longhand():
    """test_run.cpp:152-199 / acceptance criterion 9 (1e-12)."""
    g = rng(71)
    cfg = O.config([1, 1], [2, 2])
    F, T = 3, 20
    x = rand_c(g, F, 2, T)
    lam = np.stack([g.uniform(0.4, 1.6, (F, T)) for _ in range(2)])
    lam_mem = np.ascontiguousarray(np.transpose(lam, (0, 2, 1)))
    for i in range(F):
        w = np.eye(2) + 0.4 * rand_c(g, 2, 2)
        wf, _ = O.iss_sweep(cfg, w.T.copy(), (w @ x[i]).T.copy(), lam_mem, i)
        wr, yr = w.copy(), w @ x[i]
        for r in range(2):
            z = np.zeros(2, complex)
            for p in range(2):
                num = np.sum(yr[p] * yr[r].conj() / lam[p, i])
                den = np.sum(np.abs(yr[r]) ** 2 / lam[p, i])
                z[p] = 1 - math.sqrt(T / den) if p == r else num / den
            wr = wr - np.outer(z, wr[r])
            yr = yr - np.outer(z, yr[r])
        assert np.abs(wf.T - wr).max() < 1e-12


# ---------------------------------------------------------------------------
# MU updates and rescale (test_estimator.cpp:394-605)

def mu_bases_loop(Bs, Vs, floor, Y, n, taps):  # oracles.hpp:123-148
    lam = np.maximum(Bs[n] @ Vs[n], floor)
    F, K = Bs[n].shape
    T = Vs[n].shape[1]
    r0 = sum(taps[:n])
    out = Bs[n].copy()
    for i in range(F):
        for k in range(K):
            num = den = 0.0
            for l in range(taps[n]):
                for j in range(l, T):
                    num += abs(Y[i, r0 + l, j]) ** 2 * Vs[n][k, j - l] / lam[i, j - l] ** 2
                    den += Vs[n][k, j - l] / lam[i, j - l]
            out[i, k] = max(Bs[n][i, k] * math.sqrt(num / den), floor)
    return out


def mu_acts_loop(Bs, Vs, floor, Y, n, taps):  # oracles.hpp:150-175 (all taps)
    lam = np.maximum(Bs[n] @ Vs[n], floor)
    F, K = Bs[n].shape
    T = Vs[n].shape[1]
    r0 = sum(taps[:n])
    out = Vs[n].copy()
    for k in range(K):
        for j in range(T):
            num = den = 0.0
            for i in range(F):
                for l in range(taps[n]):
                    if j + l < T:
                        num += abs(Y[i, r0 + l, j + l]) ** 2 * Bs[n][i, k] / lam[i, j] ** 2
                        den += Bs[n][i, k] / lam[i, j]
            out[k, j] = max(Vs[n][k, j] * math.sqrt(num / den), floor)
    return out


def ymem(Ymats):
    return np.ascontiguousarray(np.transpose(Ymats, (0, 2, 1)))


def test_mu_bases_fixed_point_and_loop_and_descent():
    g = rng(59)
    taps, bases = [2, 2], [1, 2]
    cfg = O.config(taps, bases)
    # |y|^2 equal to the delayed lambda is a fixed point (test_estimator.cpp:398-424)
    F, T = 3, 6
    Bs = [g.uniform(0.3, 1.5, (F, k)) for k in bases]
    Vs = [g.uniform(0.3, 1.5, (k, T)) for k in bases]
    lam0 = Bs[0] @ Vs[0]
    Y = np.full((F, 4, T), 99 + 99j)
    for l in range(2):
        Y[:, l, l:] = np.sqrt(lam0[:, :T - l])
    B, V = factors_flat(Bs, Vs)
    Bn = O.mu_update_bases(cfg, F, T, B, V, 1e-15, ymem(Y), 0)
    assert np.abs(Bn[:F] - B[:F]).max() < 1e-12
    # matches the explicit quadruple loop (:426-437)
    F, T = 3, 4
    x = rand_c(g, F, 4, T)
    Bs = [g.uniform(0.2, 1.5, (F, k)) for k in bases]
    Vs = [g.uniform(0.2, 1.5, (k, T)) for k in bases]
    Y = np.transpose(O.demix(wmem(np.tile(np.eye(4, dtype=complex), (F, 1, 1))), xmem(x)), (0, 2, 1))
    B, V = factors_flat(Bs, Vs)
    for n in range(2):
        want = mu_bases_loop(Bs, Vs, 1e-9, Y, n, taps)
        B = O.mu_update_bases(cfg, F, T, B, V, 1e-9, ymem(Y), n)
        Bs, _ = factors_unflat(B, V, F, T, bases)
        assert np.abs(Bs[n] - want).max() < 1e-10 * want.max()
    # the per-source surrogate never increases over 100 instances (:439-467)
    small = O.config([2], [2])
    for _ in range(100):
        F = 2 + int(g.integers(0, 3))
        T = 3 + int(g.integers(0, 4))
        Bs = [g.uniform(0.2, 1.5, (F, 2))]
        Vs = [g.uniform(0.2, 1.5, (2, T))]
        Y = rand_c(g, F, 2, T)

        def surrogate(Bs):
            lam = np.maximum(Bs[0] @ Vs[0], 1e-9)
            return sum(math.log(lam[i, j - l]) + abs(Y[i, l, j]) ** 2 / lam[i, j - l]
                       for i in range(F) for l in range(2) for j in range(l, T))

        before = surrogate(Bs)
        B, V = factors_flat(Bs, Vs)
        Bs2, _ = factors_unflat(O.mu_update_bases(small, F, T, B, V, 1e-9, ymem(Y), 0), V, F, T, [2])
        assert surrogate(Bs2) <= before + 1e-9 * abs(before)


def test_mu_activations_fixed_point_loop_homogeneity():
    g = rng(61)
    taps, bases = [2, 2], [2, 2]
    cfg = O.config(taps, bases)
    # fixed point (test_estimator.cpp:474-491)
    F, T = 3, 5
    Bs = [g.uniform(0.2, 1.5, (F, 2)) for _ in range(2)]
    Vs = [g.uniform(0.2, 1.5, (2, T)) for _ in range(2)]
    lam1 = np.maximum(Bs[1] @ Vs[1], 1e-9)
    Y = np.full((F, 4, T), 99 + 0j)
    for l in range(2):
        Y[:, 2 + l, l:] = np.sqrt(lam1[:, :T - l])
    B, V = factors_flat(Bs, Vs)
    Vn = O.mu_update_activations(cfg, F, T, B, V, 1e-9, ymem(Y), 1)
    assert np.abs(Vn - V).max() < 1e-12
    # loop (:493-504)
    F, T = 3, 4
    x = rand_c(g, F, 4, T)
    Bs = [g.uniform(0.2, 1.5, (F, 2)) for _ in range(2)]
    Vs = [g.uniform(0.2, 1.5, (2, T)) for _ in range(2)]
    Y = np.transpose(O.demix(wmem(np.tile(np.eye(4, dtype=complex), (F, 1, 1))), xmem(x)), (0, 2, 1))
    B, V = factors_flat(Bs, Vs)
    for n in range(2):
        want = mu_acts_loop(Bs, Vs, 1e-9, Y, n, taps)
        V = O.mu_update_activations(cfg, F, T, B, V, 1e-9, ymem(Y), n)
        _, Vs = factors_unflat(B, V, F, T, bases)
        assert np.abs(Vs[n] - want).max() < 1e-10 * want.max()
    # commutes with (cB, V/c) (:506-521)
    F, T = 4, 5
    x = rand_c(g, F, 4, T)
    Y = np.transpose(O.demix(wmem(np.tile(np.eye(4, dtype=complex), (F, 1, 1))), xmem(x)), (0, 2, 1))
    Bs = [g.uniform(0.2, 1.5, (F, 2)) for _ in range(2)]
    Vs = [g.uniform(0.2, 1.5, (2, T)) for _ in range(2)]
    c = 3.7
    B, V = factors_flat(Bs, Vs)
    Bsc, Vsc = factors_flat([Bs[0] * c, Bs[1]], [Vs[0] / c, Vs[1]])
    Vp = factors_unflat(B, O.mu_update_activations(cfg, F, T, B, V, 1e-15, ymem(Y), 0), F, T, bases)[1][0]
    Vq = factors_unflat(Bsc, O.mu_update_activations(cfg, F, T, Bsc, Vsc, 1e-15, ymem(Y), 0), F, T, bases)[1][0]
    assert np.abs(Vq * c - Vp).max() < 1e-10 * Vp.max()


def test_rescale_noop_idempotence_invariance_silent_rows():
    g = rng(67)
    taps, bases = [2, 2], [2, 2]
    cfg = O.config(taps, bases)
    F, T = 3, 8
    Bs = [g.uniform(0.2, 1.5, (F, 2)) for _ in range(2)]
    Vs = [g.uniform(0.2, 1.5, (2, T)) for _ in range(2)]
    B, V = factors_flat(Bs, Vs)
    W = np.tile(np.eye(4, dtype=complex), (F, 1, 1))
    # unit average power is a no-op (:529-553)
    Y = rand_c(g, F, 4, T)
    for r in range(4):
        Y[:, r] /= math.sqrt(np.sum(np.abs(Y[:, r]) ** 2) / (F * T))
    W2, B2, Y2 = O.rescale(cfg, F, T, wmem(W), B, 1e-9, ymem(Y))
    assert np.linalg.norm(Y2 - ymem(Y)) < 1e-12 and np.linalg.norm(W2 - wmem(W)) < 1e-12
    assert np.abs(B2 - B).max() < 1e-12
    # idempotence (:555-568)
    Y = 2.5 * rand_c(g, F, 4, T)
    _, _, Y2 = O.rescale(cfg, F, T, wmem(W), B, 1e-9, ymem(Y))
    for r in range(4):
        assert math.sqrt(np.sum(np.abs(Y2[:, :, r]) ** 2) / (F * T)) == pytest.approx(1.0, rel=1e-10)
    # single-tap objective invariance (:570-588)
    ilrma = O.config([1, 1], [2, 2])
    x = rand_c(g, F, 2, T)
    Bs = [g.uniform(0.2, 1.5, (F, 2)) for _ in range(2)]
    Vs = [g.uniform(0.2, 1.5, (2, T)) for _ in range(2)]
    B, V = factors_flat(Bs, Vs)
    Wm = np.tile(np.eye(2, dtype=complex), (F, 1, 1)) + 0.3 * rand_c(g, F, 2, 2)
    Y = O.demix(wmem(Wm), xmem(x))
    before = O.objective(ilrma, F, T, wmem(Wm), B, V, 1e-15, xmem(x))
    W2, B2, _ = O.rescale(ilrma, F, T, wmem(Wm), B, 1e-15, Y)
    after = O.objective(ilrma, F, T, W2, B2, V, 1e-15, xmem(x))
    assert after == pytest.approx(before, rel=1e-8)
    # silent rows are skipped (:590-604)
    Y = rand_c(g, F, 4, T)
    Y[:, 2] = 0
    B, V = factors_flat([g.uniform(0.2, 1.5, (F, 2)) for _ in range(2)], Vs)
    W2, _, _ = O.rescale(cfg, F, T, wmem(W), B, 1e-9, ymem(Y))
    assert np.array_equal(W2[:, :, 2], wmem(W)[:, :, 2])


# ---------------------------------------------------------------------------
# run() level (proj/tests/test_run.cpp)

def synth(F, T, M, N, L, K, decay, seed):
    from paper_2510_02382_b200 import synth_mixtures
    return synth_mixtures(1, F, T, M, N, L, K, decay, seed)[0]


def test_run_objective_trace_non_increasing():
    """test_run.cpp:36-48 (ISS; and the IP rule of the oracle)."""
    x = O.stack_observation(synth(8, 40, 2, 2, 2, 3, 0.5, 97), 2)
    for rule in ("iss", "ip"):
        r = O.run(O.config([2, 2], [3, 3], iterations=40, seed=11, rule=rule), x)
        obj = r["objective"]
        assert len(obj) == 40
        assert all(obj[t] <= obj[t - 1] + 1e-6 * abs(obj[t - 1]) for t in range(1, 40))
        assert obj[-1] < obj[0]


def test_run_validation_hooks():
    """test_run.cpp:116-134: det lemma and normalization after every update."""
    x = O.stack_observation(synth(6, 30, 2, 2, 2, 3, 0.5, 19), 2)
    det, nrm, cnt = O.run_checked(O.config([2, 2], [3, 3], iterations=10, seed=5), x)
    assert cnt == 10 * 6 * 4
    assert det < 1e-10 and nrm < 1e-8


def test_run_iss_and_ip_converge_nearby():
    """test_run.cpp:136-150 (5 % of the final objective)."""
    x = O.stack_observation(synth(32, 300, 2, 2, 2, 3, 0.5, 23), 2)
    a = O.run(O.config([2, 2], [3, 3], iterations=100, seed=7, threads=8), x)["objective"][-1]
    b = O.run(O.config([2, 2], [3, 3], iterations=100, seed=7, threads=8, rule="ip"), x)["objective"][-1]
    assert abs(a - b) <= 0.05 * max(abs(a), abs(b))


def test_run_deterministic_and_thread_invariant():
    """test_run.cpp:201-217."""
    x = O.stack_observation(synth(8, 25, 2, 2, 2, 3, 0.5, 31), 2)
    cfg = O.config([2, 2], [3, 3], iterations=8, seed=77)
    a, b = O.run(cfg, x), O.run(cfg, x)
    assert np.array_equal(a["objective"], b["objective"]) and np.array_equal(a["W"], b["W"])
    c = O.run(O.config([2, 2], [3, 3], iterations=8, seed=77, threads=4), x)
    assert np.all(np.abs(c["objective"] - a["objective"]) <= 1e-9 * np.abs(a["objective"]))


def test_run_configuration_and_degeneracy_errors():
    """test_run.cpp:219-268."""
    g = rng(1)
    cfg = O.config([2, 2], [3, 3], iterations=2)
    with pytest.raises(O.OracleError) as e:  # channel mismatch / bad tap split
        O.run(O.config([1, 2], [3, 3], iterations=2, num_channels=4), xmem(rand_c(g, 4, 4, 10)))
    assert e.value.code == 2
    with pytest.raises(O.OracleError) as e:  # zero mixture
        O.run(cfg, np.zeros((4, 10, 4), complex))
    assert e.value.code == 2
    x = xmem(rand_c(rng(2), 2, 4, 10))
    x[1, 3, 2] = np.nan
    for rule in ("ip", "iss"):
        with pytest.raises(O.OracleError) as e:
            O.run(O.config([2, 2], [3, 3], iterations=2, rule=rule), x)
        assert e.value.code == 4 and "non-finite" in str(e.value)
    x = xmem(rand_c(rng(3), 3, 4, 10))
    x[1] = 0
    with pytest.raises(O.OracleError) as e:
        O.run(cfg, x)
    assert e.value.code == 4 and e.value.iteration == 1 and e.value.bin == 1 and "iteration" in str(e.value)


def test_random_factors_draw_order():
    """model.cpp:189-208: mt19937_64(seed), U(0.1, 1), per source B row-major then V row-major."""
    cfg = O.config([2, 2], [3, 2], seed=42)
    B, V = O.random_factors(cfg, 5, 7)
    assert B.min() >= 0.1 and B.max() < 1.0 and V.min() >= 0.1
    B2, V2 = O.random_factors(cfg, 5, 7)
    assert np.array_equal(B, B2) and np.array_equal(V, V2)
    # first draw lands in B_0(0, 0), second in B_0(0, 1) (row-major over (i, k))
    Bs, Vs = factors_unflat(B, V, 5, 7, [3, 2])
    cfg1 = O.config([2, 2], [3, 2], seed=42)
    B1, _ = O.random_factors(cfg1, 1, 1)
    assert Bs[0][0, 0] == B1[0] and Bs[0][0, 1] == B1[1]
