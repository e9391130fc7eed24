"""GPU parity: the CUDA path through the C ABI against the CPU oracle.

Tolerances are the ones BASELINE.json's north_star states:
  fp64: 1e-9 relative on demixing filters (and factors, objective) after
        every iteration from a shared seed;
  fp32: 1e-4 relative L2 per iteration, 1e-3 relative on the final cost
        after 100 iterations.
Inputs are seeded synthetic mixtures (BASELINE configs[0] generator)."""
import os

import json
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_02382_b200 import (CheckOptions, ConfigError, CtfConfig, DegeneracyError, Session, reconstruct_images, run,
                                   synth_mixtures)

pytestmark = pytest.mark.gpu
NPROC = os.cpu_count() or 1


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a - b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def gpu_history(x, taps, bases, iters, precision, seed, stack_taps, images=False):
    """State after every iteration: one ctf_iterate(1) per step (each call
    ends with the trailing rescale + objective, so the state equals the
    reference's after that many iterations). images=True also records the
    separated signals the GPU projects back after every iteration
    (ctf_project_back, wiener.cpp:11-49)."""
    s = Session(x, taps, bases, stack_taps=stack_taps, iterations=iters, precision=precision, seed=seed)
    hist = []
    for _ in range(iters):
        s.iterate(1)
        W, B, V, obj = s.download_raw()
        hist.append((W, B, V, obj, s.project_back() if images else None))
    s.close()
    return hist


def check_history(hist, ref, b, tol, what="", x=None, taps=None, bases=None):
    """W, B, V and the objective after every iteration; with x given also the
    separated signals (the GPU's projected-back images against the images the
    reference state yields, reconstruct_images wiener.cpp:11-49)."""
    F = ref["hist_W"].shape[1]
    for it, (W, B, V, obj, img) in enumerate(hist):
        eW = rel(W[b], ref["hist_W"][it].reshape(F, -1))
        eB = rel(B[b], ref["hist_B"][it])
        eV = rel(V[b], ref["hist_V"][it])
        eo = abs(obj[b, it] - ref["objective"][it]) / abs(ref["objective"][it])
        eY = 0.0
        if x is not None and img is not None:
            want = O.reconstruct_images(O.config(taps, bases), ref["hist_W"][it], x)
            eY = rel(img[:, b], want)
        assert max(eW, eB, eV, eo, eY) <= tol, \
            f"{what} it={it + 1}: W={eW:.2e} B={eB:.2e} V={eV:.2e} obj={eo:.2e} images={eY:.2e}"


# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["stacked_m2_l2", "cfg0_small", "general_taps23_bases24"])
def test_golden_fixtures_fp64(name):
    from tests.test_golden import load_case
    mg, c, raw, x, taps, bases, g = load_case(name)
    assert mg.digest(raw) == str(g["x_sha256"])
    if c["kind"] == "synth":
        xin, st = raw[None], c["L"]
    else:
        xin, st = x[None], 1
    hist = gpu_history(xin, taps, bases, c["iters"], "f64", c["seed"], st, images=True)
    check_history(hist, {k: g[k] for k in g.files}, 0, 1e-9, name, x=x, taps=taps, bases=bases)


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_cfg0_full_against_reference_fixture(precision):
    """BASELINE configs[0] at full size against the fixture the reference's
    own code produced (oracle/_ref): fp64 1e-9 on W, B, V at the checkpoints
    and on the objective after every one of the 100 iterations; fp32 1e-4
    relative L2 at the checkpoints and 1e-3 on the final cost."""
    from tests.test_golden import load_case
    mg, c, raw, x, taps, bases, g = load_case("cfg0_full")
    assert mg.digest(raw) == str(g["x_sha256"])
    F = c["F"]
    xin = raw[None] if precision == "f64" else raw[None].astype(np.complex64)
    s = Session(xin, taps, bases, stack_taps=c["L"], iterations=c["iters"], precision=precision, seed=c["seed"])
    done = 0
    tol = 1e-9 if precision == "f64" else 1e-4
    for k in g["checkpoints"]:
        s.iterate(int(k) - done)
        done = int(k)
        W, B, V, obj = s.download_raw()
        errs = (rel(W[0], g[f"W_{k}"].reshape(F, -1)), rel(B[0], g[f"B_{k}"]), rel(V[0], g[f"V_{k}"]))
        assert max(errs) <= tol, (precision, k, errs)
    s.close()
    eobj = np.abs(obj[0] - g["objective"]) / np.abs(g["objective"])
    if precision == "f64":
        assert eobj.max() <= 1e-9, eobj.max()
    else:
        assert eobj[-1] <= 1e-3, eobj[-1]


def test_cfg0_full_100_iterations_fp64_every_iteration():
    """BASELINE configs[0] exactly: M=N=2, L=2, F=513, T=500, K=10, 100 iterations, complex128."""
    F, T, M, N, L, K, iters, seed = 513, 500, 2, 2, 2, 10, 100, 0
    raw = synth_mixtures(1, F, T, M, N, L, K, 0.6, 20251002)
    ref = O.run(O.config([L] * N, [K] * N, iterations=iters, seed=seed, threads=NPROC),
                O.stack_observation(raw[0], L), history=True)
    hist = gpu_history(raw, [L] * N, [K] * N, iters, "f64", seed, L)
    check_history(hist, ref, 0, 1e-9, "cfg0 f64")


def test_cfg0_fp32_tolerances():
    """fp32: <= 1e-4 relative L2 per iteration, <= 1e-3 on the final cost after 100 iterations."""
    F, T, M, N, L, K, iters, seed = 513, 500, 2, 2, 2, 10, 100, 0
    raw = synth_mixtures(1, F, T, M, N, L, K, 0.6, 20251002)
    ref = O.run(O.config([L] * N, [K] * N, iterations=iters, seed=seed, threads=NPROC),
                O.stack_observation(raw[0], L), history=True)
    hist = gpu_history(raw.astype(np.complex64), [L] * N, [K] * N, iters, "f32", seed, L)
    worst = 0.0
    for it, (W, B, V, obj, _) in enumerate(hist):
        e = max(rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]),
                rel(V[0], ref["hist_V"][it]))
        worst = max(worst, e)
        assert e <= 1e-4, f"it={it + 1}: {e:.2e}"
    final = abs(hist[-1][3][0, -1] - ref["objective"][-1]) / abs(ref["objective"][-1])
    assert final <= 1e-3, final


@pytest.mark.parametrize("M,L,T,K,rho", [(2, 5, 1000, 10, 0.6), (3, 4, 2000, 20, 0.7), (2, 3, 400, 4, 0.6),
                                         (4, 8, 1000, 20, 0.8)])
def test_fp32_trajectory_cfg_geometries(M, L, T, K, rho):
    """fp32 tolerance on the BASELINE cfg1 / cfg2 / cfg3 geometries (reduced F)
    and an odd-lag shape (cfg3: the wide-tile path, a warp per row): <= 1e-4 relative L2 per iteration against the fp64 oracle
    over 30 iterations (the covariance-domain kernel serves these shapes)."""
    F, iters, seed = 33, 30, 5
    raw = synth_mixtures(1, F, T, M, M, L, K, rho, 1234 + M * L)
    ref = O.run(O.config([L] * M, [K] * M, iterations=iters, seed=seed, threads=NPROC),
                O.stack_observation(raw[0], L), history=True)
    s = Session(raw.astype(np.complex64), [L] * M, [K] * M, stack_taps=L, iterations=iters, precision="f32",
                seed=seed)
    kern = json.loads(s.describe())["sweep_kernel"]
    s.close()
    hist = gpu_history(raw.astype(np.complex64), [L] * M, [K] * M, iters, "f32", seed, L)
    for it, (W, B, V, obj, _) in enumerate(hist):
        e = max(rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]),
                rel(V[0], ref["hist_V"][it]))
        assert e <= 1e-4, f"{kern} it={it + 1}: {e:.2e}"
    final = abs(hist[-1][3][0, -1] - ref["objective"][-1]) / abs(ref["objective"][-1])
    assert final <= 1e-3, final


@pytest.mark.parametrize("M,L", [(2, 4), (2, 8), (3, 2), (3, 3), (3, 5), (4, 2), (4, 3), (4, 4)])
@pytest.mark.parametrize("precision,tol", [("f64", 1e-9), ("f32", 1e-4)])
def test_more_stacked_shapes_on_the_covariance_kernel(M, L, precision, tol):
    """The additional compiled (mics, taps) pairs of the covariance-domain
    kernel (ctf_sweep_gram_more.cu, R = M*L <= 16, T <= 1024): every iteration
    against the oracle's run() (estimator.cpp:513-657) on the stacked
    observation; fp64 1e-9, fp32 1e-4 relative L2."""
    F, T, K, iters, seed = 9, 300, 4, 8, 21
    raw = synth_mixtures(1, F, T, M, M, L, K, 0.6, 400 + 10 * M + L)
    ref = O.run(O.config([L] * M, [K] * M, iterations=iters, seed=seed, threads=NPROC),
                O.stack_observation(raw[0], L), history=True)
    xin = raw if precision == "f64" else raw.astype(np.complex64)
    s = Session(xin, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision=precision, seed=seed)
    kern = json.loads(s.describe())["sweep_kernel"]
    s.close()
    if not (precision == "f64" and (M, L) == (4, 2)):  # (measured slower there: not compiled in fp64)
        assert kern.startswith("gram_kernel"), kern
    hist = gpu_history(xin, [L] * M, [K] * M, iters, precision, seed, L)
    for it, (W, B, V, obj, _) in enumerate(hist):
        e = max(rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]),
                rel(V[0], ref["hist_V"][it]))
        eo = abs(obj[0, it] - ref["objective"][it]) / abs(ref["objective"][it])
        assert max(e, eo if precision == "f64" else 0.0) <= tol, f"{kern} it={it + 1}: {e:.2e} obj {eo:.2e}"


def test_odd_tile_sizes_with_the_l2_prefetch_active():
    """fp32 tiles of an odd number of complex values (W at R = D = 9: 648
    bytes per bin) start 8 bytes off a 16-byte boundary on every other bin; the
    L2 prefetch of the tile a resident-CTA-count ahead must not fault (it did:
    'misaligned address') once the batch has more tiles than resident CTAs."""
    M, L, F, T, K, B, iters = 3, 3, 129, 200, 4, 8, 2
    raw = synth_mixtures(B, F, T, M, M, L, K, 0.6, 77).astype(np.complex64)
    s = Session(raw, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision="f32", seed=3)
    s.iterate(iters)
    W, Bf, V, obj = s.download_raw()
    s.close()
    assert np.isfinite(W).all() and np.isfinite(obj).all()
    ref = O.run(O.config([L] * M, [K] * M, iterations=iters, seed=3 + B - 1, threads=NPROC),
                O.stack_observation(raw[B - 1].astype(np.complex128), L))
    assert rel(W[B - 1], ref["W"].reshape(F, -1)) <= 1e-4


def test_one_step_parity_from_oracle_state():
    """Restart the GPU from the oracle's state after 4 iterations (cfg1 shape,
    reduced F): one GPU iteration equals one oracle iteration (no trajectory
    amplification in the comparison)."""
    F, T, M, N, L, K = 65, 1000, 2, 2, 5, 10
    raw = synth_mixtures(1, F, T, M, N, L, K, 0.6, 7)
    x = O.stack_observation(raw[0], L)
    cfg = O.config([L] * N, [K] * N, iterations=4, seed=3, threads=NPROC)
    r = O.run(cfg, x)
    floor = 1e-10 * O.mean_power(x)
    Wn, Bn, Vn, objn = O.step(cfg, x, floor, r["W"], r["B"], r["V"])
    s = Session(raw, [L] * N, [K] * N, stack_taps=L, iterations=1, precision="f64", seed=3)
    assert s.psd_floor()[0] == pytest.approx(floor, rel=1e-12)
    s.set_state(W=r["W"].reshape(1, F, -1).view(np.float64), B=r["B"][None], V=r["V"][None])
    s.iterate(1)
    W, B, V, obj = s.download_raw()
    assert rel(W[0], Wn.reshape(F, -1)) <= 1e-10
    assert rel(B[0], Bn) <= 1e-10 and rel(V[0], Vn) <= 1e-10
    assert abs(obj[0, 0] - objn) <= 1e-10 * abs(objn)


@pytest.mark.parametrize("precision,tol", [("f64", 1e-9), ("f32", 1e-4)])
def test_cfg1_shape_two_mixtures(precision, tol):
    """BASELINE configs[1] shape (M=N=2, L=5, F=513, T=1000, K=10), 2 mixtures, 3 iterations."""
    F, T, M, N, L, K, iters, seed = 513, 1000, 2, 2, 5, 10, 3, 100
    raw = synth_mixtures(2, F, T, M, N, L, K, 0.6, 1)
    s = Session(raw if precision == "f64" else raw.astype(np.complex64), [L] * N, [K] * N, stack_taps=L,
                iterations=iters, precision=precision, seed=seed)
    s.iterate(iters)
    W, B, V, obj = s.download_raw()
    s.close()
    for b in range(2):
        ref = O.run(O.config([L] * N, [K] * N, iterations=iters, seed=seed + b, threads=NPROC),
                    O.stack_observation(raw[b], L))
        assert rel(W[b], ref["W"].reshape(F, -1)) <= tol
        assert rel(B[b], ref["B"]) <= tol and rel(V[b], ref["V"]) <= tol
        assert np.max(np.abs(obj[b] - ref["objective"]) / np.abs(ref["objective"])) <= tol


@pytest.mark.parametrize("precision,tol,T", [("f64", 1e-9, 500), ("f32", 1e-4, 2000)])
def test_cfg2_shape_r12(precision, tol, T):
    """BASELINE configs[2] rows (M=N=3, L=4, K=20; T=2000 in fp32 as BASELINE
    runs it) at reduced F. An fp64 T=2000 tile (375 KiB) exceeds one CTA's
    shared memory; the streamed path for it is future work."""
    F, M, N, L, K, iters, seed = 33, 3, 3, 4, 20, 2, 5
    raw = synth_mixtures(1, F, T, M, N, L, K, 0.7, 2)
    s = Session(raw, [L] * N, [K] * N, stack_taps=L, iterations=iters, precision=precision, seed=seed)
    s.iterate(iters)
    W, B, V, obj = s.download_raw()
    ref = O.run(O.config([L] * N, [K] * N, iterations=iters, seed=seed, threads=NPROC), O.stack_observation(raw[0], L))
    assert rel(W[0], ref["W"].reshape(F, -1)) <= tol
    assert rel(B[0], ref["B"]) <= tol and rel(V[0], ref["V"]) <= tol
    assert np.max(np.abs(obj[0] - ref["objective"]) / np.abs(ref["objective"])) <= tol


def test_run_api_prestacked_general_config():
    """run(config, x) with a pre-stacked 5-channel observation, taps {2,3},
    bases {2,4} (the reference's general CtfConfig), vs the oracle."""
    g = np.random.default_rng(8)
    F, T = 21, 64
    xm = g.standard_normal((F, 5, T)) + 1j * g.standard_normal((F, 5, T))
    cfg = CtfConfig(2, 5, [2, 3], [2, 4], iterations=7, seed=13)
    res = run(cfg, xm)
    ref = O.run(O.config([2, 3], [2, 4], iterations=7, seed=13), np.ascontiguousarray(np.transpose(xm, (0, 2, 1))))
    Wref = np.transpose(ref["W"], (0, 2, 1))
    assert rel(res.demixing, Wref) <= 1e-9
    assert np.max(np.abs(np.array(res.trace.objective) - ref["objective"]) / np.abs(ref["objective"])) <= 1e-9
    B0 = ref["B"][:F * 2].reshape(2, F).T
    assert rel(res.bases[0], B0) <= 1e-9
    assert len(res.trace.demix_ms) == 7 and all(t > 0 for t in res.trace.demix_ms)
    # OptimizationTrace phases (estimator.cpp:623-653): every phase timed, rescale = the mu/apply kernel
    assert len(res.trace.mu_ms) == 7 and all(t > 0 for t in res.trace.mu_ms)
    assert len(res.trace.rescale_ms) == 7 and all(t > 0 for t in res.trace.rescale_ms)


def test_check_options_hooks():
    """CheckOptions on the GPU (test_run.cpp:116-134): 2 sources x 2 taps over a
    4-channel stacked observation, 6 bins x 30 frames, 10 iterations ->
    checked_updates = 240, det-lemma error < 1e-10, normalization < 1e-8, the
    same order as the oracle's exact recomputation; and the instrumented run
    returns the same state as the plain one."""
    raw = synth_mixtures(1, 6, 30, 2, 2, 2, 3, 0.5, 19)
    xm = np.transpose(O.stack_observation(raw[0], 2), (0, 2, 1))  # (F, D, T)
    cfg = CtfConfig(2, 4, [2, 2], [3, 3], iterations=10, seed=5)
    res = run(cfg, xm, CheckOptions(det_lemma=True, normalization=True))
    assert res.trace.checked_updates == 10 * 6 * 4
    assert 0.0 <= res.trace.max_det_lemma_error < 1e-10
    assert 0.0 < res.trace.max_normalization_error < 1e-8
    det, nrm, cnt = O.run_checked(O.config([2, 2], [3, 3], iterations=10, seed=5),
                                  np.ascontiguousarray(np.transpose(xm, (0, 2, 1))))
    assert cnt == 240 and det < 1e-10 and nrm < 1e-8
    plain = run(cfg, xm)
    assert rel(res.demixing, plain.demixing) <= 1e-12
    assert plain.trace.checked_updates == 0 and plain.trace.max_det_lemma_error == 0.0
    only = run(cfg, xm, CheckOptions(normalization=True))
    assert only.trace.max_det_lemma_error == 0.0 and 0.0 < only.trace.max_normalization_error < 1e-8
    # fp32 instrumented path: identities hold to single precision
    r32 = run(cfg, xm, CheckOptions(det_lemma=True, normalization=True), precision="f32")
    assert r32.trace.max_det_lemma_error < 1e-3 and r32.trace.max_normalization_error < 1e-3


@pytest.mark.parametrize("M,L,T,K,F,iters", [(4, 8, 1000, 20, 3, 3), (6, 10, 600, 16, 2, 2), (3, 6, 300, 4, 3, 4)])
def test_check_options_wide_tiles(M, L, T, K, F, iters):
    """CheckOptions for R > 16 (BASELINE cfg3 R = 32, cfg4 R = 60, and R = 18):
    the instrumented streamed kernel recomputes det W by a warp LU after every
    step and the updated row's weighted power (estimator.cpp:556-577) ->
    checked_updates = iterations * F * R, the det-lemma and normalization
    errors at the oracle's order, and the same state as the plain run (fp64)."""
    R = M * L
    raw = synth_mixtures(1, F, T, M, M, L, K, 0.7, 23)
    s = Session(raw, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision="f64", seed=3, checks=3)
    assert "stream_kernel" in s.describe(), s.describe()
    s.iterate(iters)
    det, nrm, cnt = s.check_stats()
    W = s.download_raw()[0]
    s.close()
    assert int(cnt[0]) == iters * F * R
    odet, onrm, ocnt = O.run_checked(O.config([L] * M, [K] * M, iterations=iters, seed=3, threads=NPROC),
                                     O.stack_observation(raw[0], L))
    assert ocnt == iters * F * R
    assert 0.0 <= det[0] < 1e-9 and 0.0 < nrm[0] < 1e-8, (det[0], nrm[0], odet, onrm)
    plain = Session(raw, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision="f64", seed=3)
    plain.iterate(iters)
    assert rel(W, plain.download_raw()[0]) <= 1e-10
    plain.close()


def test_check_options_sharded_max_over_ranks():
    """With frequency shards the check maxima are reduced over ranks (host group)."""
    import threading
    from paper_2510_02382_b200 import _lib
    raw = synth_mixtures(2, 9, 40, 2, 2, 2, 3, 0.6, 4)
    s = Session(raw, [2, 2], [3, 3], stack_taps=2, iterations=3, precision="f64", checks=3)
    s.iterate(3)
    d1, n1, k1 = s.check_stats()
    s.close()
    lib = _lib.load()
    grp = lib.ctf_group_create(2)
    out = [None, None]

    def worker(r):
        t = Session(raw, [2, 2], [3, 3], stack_taps=2, iterations=3, precision="f64", checks=3, world_size=2,
                    rank=r, group=grp)
        t.iterate(3)
        out[r] = t.check_stats()
        t.close()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    lib.ctf_group_destroy(grp)
    assert k1[0] == 3 * 9 * 4 and np.all(d1 < 1e-10) and np.all(n1 < 1e-8)
    for d, n, k in out:  # every rank reports the same (global) maxima and counts
        assert np.array_equal(k, k1)
        assert np.array_equal(d, out[0][0]) and np.array_equal(n, out[0][1])
        assert np.all(d < 1e-10) and np.all(n < 1e-8) and np.all(n > 0)


def test_batch_equals_individual_runs_bitwise():
    """Mixtures are independent: a batch of 3 gives, per mixture, bit-identical
    results to running that mixture alone (with its own seed)."""
    F, T, M, N, L, K = 40, 200, 2, 2, 3, 4
    raw = synth_mixtures(3, F, T, M, N, L, K, 0.6, 9)
    s = Session(raw, [L] * N, [K] * N, stack_taps=L, iterations=4, precision="f64", seed=20)
    s.iterate(4)
    W, B, V, obj = s.download_raw()
    for b in range(3):
        t = Session(raw[b:b + 1], [L] * N, [K] * N, stack_taps=L, iterations=4, precision="f64", seed=20 + b)
        t.iterate(4)
        W1, B1, V1, o1 = t.download_raw()
        assert np.array_equal(W[b], W1[0]) and np.array_equal(V[b], V1[0]) and np.array_equal(obj[b], o1[0])


def test_deterministic_reruns():
    raw = synth_mixtures(2, 30, 150, 2, 2, 2, 3, 0.6, 4)
    out = []
    for _ in range(2):
        s = Session(raw.astype(np.complex64), [2, 2], [3, 3], stack_taps=2, iterations=5, precision="f32", seed=1)
        s.iterate(5)
        out.append(s.download_raw())
    for a, b in zip(*out):
        assert np.array_equal(a, b)


def test_errors_match_reference_semantics():
    """test_run.cpp:219-268 on the GPU path."""
    g = np.random.default_rng(1)
    cfg = CtfConfig(2, 4, [2, 2], [3, 3], iterations=2)
    with pytest.raises(ConfigError):  # channel mismatch
        run(cfg, g.standard_normal((4, 3, 10)) + 0j)
    with pytest.raises(ConfigError):  # zero mixture
        run(cfg, np.zeros((4, 4, 10), complex))
    with pytest.raises(ConfigError):  # bad tap split
        run(CtfConfig(2, 4, [1, 2], [3, 3], iterations=2), g.standard_normal((4, 4, 10)) + 0j)
    with pytest.raises(ConfigError):  # IP needs a square demixing matrix (taps sum to the channels)
        run(CtfConfig(2, 5, [2, 2], [3, 3], iterations=2, update_rule="ip"), g.standard_normal((4, 5, 10)) + 0j)
    x = g.standard_normal((2, 4, 10)) + 1j * g.standard_normal((2, 4, 10))
    x[1, 2, 3] = np.nan
    with pytest.raises(DegeneracyError) as e:
        run(cfg, x)
    assert "non-finite" in str(e.value)
    x = g.standard_normal((3, 4, 10)) + 1j * g.standard_normal((3, 4, 10))
    x[1] = 0
    with pytest.raises(DegeneracyError) as e:
        run(cfg, x)
    assert e.value.iteration == 1 and e.value.bin == 1 and "iteration" in str(e.value)


def test_projection_back_matches_oracle():
    """reconstruct_images (wiener.cpp:11-49) for a converged-ish demixing."""
    F, T, M, N, L, K = 25, 80, 2, 2, 2, 3
    raw = synth_mixtures(1, F, T, M, N, L, K, 0.6, 3)
    x = O.stack_observation(raw[0], L)
    r = O.run(O.config([L] * N, [K] * N, iterations=5, seed=2), x)
    want = O.reconstruct_images(O.config([L] * N, [K] * N), r["W"], x)  # [N, F, T, D]
    s = Session(raw, [L] * N, [K] * N, stack_taps=L, iterations=0, precision="f64", seed=2)
    s.set_state(W=r["W"].reshape(1, F, -1).view(np.float64))
    got = s.project_back()  # [N, B, F, T, D]
    assert rel(got[:, 0], want) <= 1e-10
    cur = s.project_back(current_frame_only=True)  # mic channels c = m*L
    assert rel(cur[:, 0], want[..., ::L]) <= 1e-10
    # the images sum back to the observation (c_1 + ... + c_N = x~)
    assert rel(got[:, 0].sum(axis=0), x) <= 1e-10
    # python mirror of reconstruct_images
    img = reconstruct_images(np.transpose(r["W"], (0, 2, 1)), CtfConfig(N, M * L, [L] * N, [K] * N),
                             np.transpose(x, (0, 2, 1)))
    assert rel(img, np.transpose(want, (0, 1, 3, 2))) <= 1e-10


@pytest.mark.slow
def test_full_cfg1_batch_properties():
    """BASELINE configs[1] at full size (64 mixtures), fp32: size-independent
    properties — objective non-increasing per mixture, factors above the floor,
    and mixture 0 identical to a standalone run of mixture 0."""
    B, F, T, M, N, L, K, iters = 64, 513, 1000, 2, 2, 5, 10, 8
    raw = synth_mixtures(B, F, T, M, N, L, K, 0.6, 1, precision="f32")
    s = Session(raw, [L] * N, [K] * N, stack_taps=L, iterations=iters, precision="f32", seed=0)
    s.iterate(iters)
    W, Bf, V, obj = s.download_raw()
    floors = s.psd_floor()
    assert np.all(np.isfinite(W)) and np.all(np.isfinite(obj))
    for b in range(B):
        assert np.all(np.diff(obj[b]) <= 1e-5 * np.abs(obj[b][:-1])), obj[b]
        assert Bf[b].min() >= floors[b] * (1 - 1e-6) and V[b].min() >= floors[b] * (1 - 1e-6)
    t = Session(raw[:1], [L] * N, [K] * N, stack_taps=L, iterations=iters, precision="f32", seed=0)
    t.iterate(iters)
    W1, B1, V1, o1 = t.download_raw()
    assert np.array_equal(W[0], W1[0]) and np.array_equal(o1[0], obj[0])


@pytest.mark.parametrize("shape", [
    # BASELINE configs[3] rows: M=N=4, L=8 (R=32), T=1000, K=20, tap variance 0.8^l
    dict(M=4, L=8, T=1000, K=20, rho=0.8, F=9, iters=2, prec="f32", tol=1e-4),
    # BASELINE configs[4] rows: M=N=6, L=10 (R=60), T=4000, K=16, tap variance 0.85^l
    dict(M=6, L=10, T=4000, K=16, rho=0.85, F=3, iters=1, prec="f32", tol=1e-4),
    # fp64 tile beyond one SM (R=12, T=2000): streamed path in double precision
    dict(M=3, L=4, T=2000, K=20, rho=0.7, F=7, iters=2, prec="f64", tol=1e-9),
    dict(M=4, L=8, T=1000, K=20, rho=0.8, F=5, iters=2, prec="f64", tol=1e-9),
])
@pytest.mark.parametrize("kind", ["2", "3"])
def test_streamed_large_tiles(shape, kind, monkeypatch):
    """Tiles that exceed one SM: the streamed kernel (kind 2) and the
    thread-block-cluster kernel (kind 3, where R splits over the cluster);
    parity vs the oracle."""
    M, L, T, K, F = shape["M"], shape["L"], shape["T"], shape["K"], shape["F"]
    N, iters, seed = M, shape["iters"], 4
    monkeypatch.setenv("CTF_SWEEP_KIND", kind)
    raw = synth_mixtures(1, F, T, M, N, L, K, shape["rho"], 12)
    try:
        s = Session(raw if shape["prec"] == "f64" else raw.astype(np.complex64), [L] * N, [K] * N, stack_taps=L,
                    iterations=iters, precision=shape["prec"], seed=seed)
    except Exception as e:  # noqa: BLE001
        if kind == "3" and "no compiled sweep kernel" in str(e):
            pytest.skip("no cluster variant for this shape")
        raise
    assert ("stream_kernel" if kind == "2" else "cluster_kernel") in s.describe()
    s.iterate(iters)
    W, B, V, obj = s.download_raw()
    ref = O.run(O.config([L] * N, [K] * N, iterations=iters, seed=seed, threads=NPROC), O.stack_observation(raw[0], L))
    tol = shape["tol"]
    assert rel(W[0], ref["W"].reshape(F, -1)) <= tol
    assert rel(B[0], ref["B"]) <= tol and rel(V[0], ref["V"]) <= tol
    assert np.max(np.abs(obj[0] - ref["objective"]) / np.abs(ref["objective"])) <= tol


def _sharded_run(raw, L, K, iters, precision, seed, world):
    """Runs `world` frequency shards as separate contexts on cuda:0, one host
    thread each, exchanging through the in-process group (the NCCL path's
    data flow with a host all-reduce)."""
    import threading
    from paper_2510_02382_b200 import _lib
    lib = _lib.load()
    grp = lib.ctf_group_create(world)
    out, errs = [None] * world, [None] * world
    N = raw.shape[3]

    def worker(r):
        try:
            s = Session(raw, [L] * N, [K] * N, stack_taps=L, iterations=iters, precision=precision, seed=seed,
                        world_size=world, rank=r, group=grp)
            s.iterate(iters)
            out[r] = (s.bin_range, s.download_raw())
            s.close()
        except Exception as e:  # noqa: BLE001
            errs[r] = e

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    [t.start() for t in th]
    [t.join() for t in th]
    lib.ctf_group_destroy(grp)
    return out, errs


@pytest.mark.parametrize("precision,tol", [("f64", 1e-12), ("f32", 2e-5)])
def test_frequency_sharded_contexts_match_single_context(precision, tol):
    """The world > 1 path (shard ranges, packed all-reduce of MU-V sums, row
    powers, objective, mean power, error words) reproduces the world = 1 run;
    with three mixtures the pipelined loop runs two uneven mixture chunks."""
    B, F, T, M, L, K, iters, seed = 3, 37, 300, 2, 3, 4, 4, 6
    raw = synth_mixtures(B, F, T, M, M, L, K, 0.6, 31)
    if precision == "f32":
        raw = raw.astype(np.complex64)
    s = Session(raw, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision=precision, seed=seed)
    s.iterate(iters)
    W1, B1, V1, o1 = s.download_raw()
    s.close()
    for world in (2, 3):
        out, errs = _sharded_run(raw, L, K, iters, precision, seed, world)
        assert not any(errs), errs
        covered = []
        for (lo, hi), (W, Bf, V, obj) in out:
            covered.append((lo, hi))
            assert rel(W[:, lo:hi], W1[:, lo:hi]) <= tol
            Bl = Bf.reshape(B, M, K, F)[..., lo:hi]
            assert rel(Bl, B1.reshape(B, M, K, F)[..., lo:hi]) <= tol
            assert rel(V, V1) <= tol  # V is replicated on every rank
            assert np.max(np.abs(obj - o1) / np.abs(o1)) <= tol
        assert sorted(covered)[0][0] == 0 and sorted(covered)[-1][1] == F


@pytest.mark.parametrize("precision,tol,chunks,use_async,theta", [
    ("f64", 1e-12, "1", False, None), ("f32", 1e-5, "1", False, None), ("f64", 1e-12, "2", False, None),
    ("f64", 1e-12, "3", True, None), ("f32", 1e-5, "2", True, None),
    ("f64", 1e-12, "3", True, "0"), ("f32", 1e-5, "2", False, "0")])
def test_nccl_single_rank_communicator(monkeypatch, precision, tol, chunks, use_async, theta):
    """The NCCL exchange itself on one GPU: a single-rank communicator
    (CTF_NCCL_SINGLE_RANK=1) drives the reduce -> ncclAllReduce -> apply path
    (packed MU-V sums, row powers, objective, mean power, error words) and must
    reproduce the plain world = 1 run. theta "0": every bin takes the
    conditioning fallback from iteration 2 on, each mixture chunk with its own
    fallback list."""
    from paper_2510_02382_b200 import _lib
    import ctypes
    if theta is not None:
        monkeypatch.setenv("CTF_GRAM_FALLBACK_THETA", theta)
    B, F, T, M, L, K, iters, seed = 3, 37, 300, 2, 3, 4, 4, 6
    raw = synth_mixtures(B, F, T, M, M, L, K, 0.6, 31)
    if precision == "f32":
        raw = raw.astype(np.complex64)
    s = Session(raw, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision=precision, seed=seed)
    s.iterate(iters)
    ref = s.download_raw()
    s.close()
    monkeypatch.setenv("CTF_MIX_CHUNKS", chunks)
    lib = _lib.load()
    uid, err = (ctypes.c_uint8 * 128)(), _lib.CtfErr()
    assert lib.ctf_comm_unique_id(uid, ctypes.byref(err)) == 0, err.msg
    monkeypatch.setenv("CTF_NCCL_SINGLE_RANK", "1")
    s = Session(raw, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision=precision, seed=seed,
                comm_id=bytes(uid))
    d = json.loads(s.describe())
    assert d["collective"] == "nccl" and d["mix_chunks"] == int(chunks), d
    if use_async:  # the benchmark form: n loop bodies, then the trailing finalize
        s.iterate_async(iters)
        s.finalize()
    else:
        s.iterate(iters)
    got = s.download_raw()
    s.close()
    for a, b in zip(got, ref):
        assert rel(a, b) <= tol


def test_frequency_sharded_degeneracy_reported_on_every_rank():
    """A silent bin in rank 1's shard raises the same DegeneracyError on all ranks."""
    g = np.random.default_rng(3)
    F, T = 6, 40
    x = g.standard_normal((1, F, T, 4)) + 1j * g.standard_normal((1, F, T, 4))
    x[0, 4] = 0
    import threading
    from paper_2510_02382_b200 import _lib
    lib = _lib.load()
    grp = lib.ctf_group_create(2)
    errs = [None, None]

    def worker(r):
        try:
            s = Session(x, [2, 2], [3, 3], stack_taps=1, iterations=2, precision="f64", world_size=2, rank=r,
                        group=grp)
            s.iterate(2)
        except DegeneracyError as e:
            errs[r] = e

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    lib.ctf_group_destroy(grp)
    for e in errs:
        assert e is not None and e.iteration == 1 and e.bin == 4


@pytest.mark.parametrize("case", [
    dict(F=7, T=37, M=1, L=3, N=1, K=1, taps=None, prec="f64"),     # single source, T not a multiple of 32, K=1
    dict(F=5, T=61, M=7, L=1, N=2, K=2, taps=[3, 4], prec="f64"),    # R=7: guarded runtime-R variant, unequal taps
    dict(F=4, T=90, M=5, L=4, N=2, K=3, taps=[12, 8], prec="f64"),   # R=20: beyond the resident set -> streamed
    dict(F=9, T=33, M=2, L=8, N=2, K=5, taps=None, prec="f32"),      # R=16 stacked, short frames
])
def test_odd_shapes(case):
    """Shapes off the BASELINE grid, pre-stacked (stack_taps = 1) when taps are unequal."""
    F, T, M, L, N, K = case["F"], case["T"], case["M"], case["L"], case["N"], case["K"]
    g = np.random.default_rng(F * 1000 + T)
    if case["taps"] is None:
        raw = synth_mixtures(1, F, T, M, N, L, K, 0.6, 77)
        taps, st, x = [L] * N, L, O.stack_observation(raw[0], L)
        xin = raw
    else:
        taps, st = case["taps"], 1
        D = sum(taps)
        x = g.standard_normal((F, T, D)) + 1j * g.standard_normal((F, T, D))
        xin = x[None]
    iters, seed = 3, 5
    tol = 1e-9 if case["prec"] == "f64" else 1e-4
    s = Session(xin if case["prec"] == "f64" else xin.astype(np.complex64), taps, [K] * N, stack_taps=st,
                iterations=iters, precision=case["prec"], seed=seed)
    s.iterate(iters)
    W, B, V, obj = s.download_raw()
    ref = O.run(O.config(taps, [K] * N, iterations=iters, seed=seed), x)
    assert rel(W[0], ref["W"].reshape(F, -1)) <= tol
    assert rel(B[0], ref["B"]) <= tol and rel(V[0], ref["V"]) <= tol
    assert np.max(np.abs(obj[0] - ref["objective"]) / np.abs(ref["objective"])) <= tol


@pytest.mark.parametrize("M,L,T,K,prec,kernel", [
    (2, 5, 201, 4, "f64", "gram_kernel"),     # T odd: lambda_kernel one frame per thread, scalar 1/lambda copy
    (3, 4, 1030, 5, "f32", "gram_kernel"),    # the T > 1024 fp32 variant (two CTAs per SM), T % 4 == 2
    (4, 8, 998, 5, "f32", "fsplit_kernel"),   # frame-split + lambda_kernel + mub_kernel, T % 4 == 2
])
def test_lambda_ahead_unaligned_frame_counts(M, L, T, K, prec, kernel):
    """The kernels that take 1/lambda from lambda_kernel (and, frame-split, leave
    MU-B to mub_kernel) on frame counts that rule out the 16-byte vector paths:
    every iteration against the oracle (compute_psd model.cpp:210-215, MU-B
    estimator.cpp:313-346, objective :55-77)."""
    F, iters, seed = 5, 4, 9
    tol = 1e-9 if prec == "f64" else 1e-4
    raw = synth_mixtures(2, F, T, M, M, L, K, 0.6, 900 + T)
    xin = raw if prec == "f64" else raw.astype(np.complex64)
    s = Session(xin, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision=prec, seed=seed)
    d = json.loads(s.describe())
    s.close()
    assert d["sweep_kernel"].startswith(kernel) and d["lambda_ahead"], d
    hist = gpu_history(xin, [L] * M, [K] * M, iters, prec, seed, L)
    for b in range(2):
        ref = O.run(O.config([L] * M, [K] * M, iterations=iters, seed=seed + b, threads=NPROC),
                    O.stack_observation(raw[b], L), history=True)
        for it, (W, B, V, obj, _) in enumerate(hist):
            e = max(rel(W[b], ref["hist_W"][it].reshape(F, -1)), rel(B[b], ref["hist_B"][it]),
                    rel(V[b], ref["hist_V"][it]))
            eo = abs(obj[b, it] - ref["objective"][it]) / abs(ref["objective"][it])
            assert e <= tol and eo <= (tol if prec == "f64" else 1e-3), f"mixture {b} it={it + 1}: {e:.2e} obj {eo:.2e}"


@pytest.mark.parametrize("B,iters,precision", [(3, 5, "f64"), (9, 2, "f64"), (11, 6, "f32"), (2, 1, "f32")])
def test_ctf_run_end_to_end_matches_device_resident_path(B, iters, precision):
    """ctf_run (host buffers in, host buffers out) == setup + iterate + download,
    bit for bit: ctf_run uploads x in mixture chunks and runs each chunk's
    first loop bodies on its own stream while later chunks are still in
    flight (run_overlapped); the result must not depend on that."""
    import ctypes
    from paper_2510_02382_b200 import _lib
    from paper_2510_02382_b200.api import _problem
    F, T, M, L, K, seed = 21, 120, 2, 3, 4, 8
    raw = synth_mixtures(B, F, T, M, M, L, K, 0.6, 5)
    if precision == "f32":
        raw = raw.astype(np.complex64)
    s = Session(raw, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision=precision, seed=seed)
    s.iterate(iters)
    W1, B1, V1, o1 = s.download_raw()
    s.close()
    lib = _lib.load()
    R, SK = M * L, M * K
    W = np.zeros(B * F * R * R * 2)
    Bf = np.zeros(B * F * SK)
    V = np.zeros(B * SK * T)
    o = np.zeros(B * iters)
    prob = _problem(B, F, T, M, L, [L] * M, [K] * M, iters, precision, precision, 1e-10, seed)
    ctx = ctypes.c_void_p()
    err = _lib.CtfErr()
    assert lib.ctf_open(0, ctypes.byref(ctx), ctypes.byref(err)) == 0
    rc = lib.ctf_run(ctx, ctypes.byref(prob), _lib.vptr(raw), _lib.dptr(W), _lib.dptr(Bf), _lib.dptr(V), _lib.dptr(o),
                     ctypes.byref(err))
    lib.ctf_close(ctx)
    assert rc == 0, err.msg
    assert np.array_equal(W.view(np.complex128).reshape(B, F, -1), W1)
    assert np.array_equal(Bf.reshape(B, -1), B1) and np.array_equal(V.reshape(B, -1), V1)
    assert np.array_equal(o.reshape(B, iters), o1)


def test_ctf_run_setup_errors_with_the_overlapped_upload():
    """The setup checks of estimator.cpp:520-529 still come first when ctf_run
    overlaps the upload with the loop: a non-finite mixture -> degeneracy
    "non-finite", an all-zero mixture -> ConfigError, for the offending mixture."""
    import ctypes
    from paper_2510_02382_b200 import _lib
    from paper_2510_02382_b200.api import _problem
    B, F, T, M, L, K, iters, seed = 5, 9, 60, 2, 2, 3, 4, 1
    lib = _lib.load()
    for kind in ("nan", "zero"):
        raw = synth_mixtures(B, F, T, M, M, L, K, 0.6, 2)
        if kind == "nan":
            raw[3, 4, 7, 1] = np.nan
        else:
            raw[2] = 0
        W, Bf, V, o = np.zeros(B * F * (M * L) ** 2 * 2), np.zeros(B * F * M * K), np.zeros(B * M * K * T), np.zeros(B * iters)
        prob = _problem(B, F, T, M, L, [L] * M, [K] * M, iters, "f64", "f64", 1e-10, seed)
        ctx, err = ctypes.c_void_p(), _lib.CtfErr()
        assert lib.ctf_open(0, ctypes.byref(ctx), ctypes.byref(err)) == 0
        rc = lib.ctf_run(ctx, ctypes.byref(prob), _lib.vptr(raw), _lib.dptr(W), _lib.dptr(Bf), _lib.dptr(V),
                         _lib.dptr(o), ctypes.byref(err))
        lib.ctf_close(ctx)
        if kind == "nan":
            assert rc == 4 and b"non-finite" in err.msg and err.mixture == 3, (rc, err.msg)
        else:
            assert rc == 2 and b"zero" in err.msg and err.mixture == 2, (rc, err.msg)


def test_cpp_reference_mirror_runs_on_gpu(tmp_path):
    """ctfmnmf::b200::run (csrc/ctfmnmf_b200.hpp, the reference-shaped C++ API)
    on a pre-stacked observation equals the oracle's run()."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    csrc = os.path.join(root, "paper_2510_02382_b200", "csrc")
    libdir = os.path.join(root, "paper_2510_02382_b200")
    g = np.random.default_rng(2)
    F, D, T = 6, 4, 40
    x = g.standard_normal((F, T, D)) + 1j * g.standard_normal((F, T, D))
    xf = tmp_path / "x.bin"
    x.astype(np.complex128).tofile(xf)
    src = tmp_path / "run.cpp"
    src.write_text(f'''#include "ctfmnmf_b200.hpp"
#include <cstdio>
#include <fstream>
using namespace ctfmnmf::b200;
int main() {{
  CtfConfig c; c.num_sources = 2; c.num_channels = 4; c.taps_per_source = {{2, 2}}; c.bases_per_source = {{3, 3}};
  c.iterations = 6; c.seed = 21;
  MixtureSpectrogram x; x.bins.assign({F}, CMatrix({D}, {T}));
  std::ifstream in("{xf}", std::ios::binary);
  for (auto& b : x.bins) in.read(reinterpret_cast<char*>(b.data.data()), b.data.size() * sizeof(Complex));
  SeparationResult r = run(c, x);
  for (double o : r.trace.objective) std::printf("%.17g\\n", o);
  for (const auto& w : r.demixing) for (const auto& v : w.data) std::printf("%.17g %.17g\\n", v.real(), v.imag());
  return 0;
}}''')
    exe = tmp_path / "run"
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{csrc}", "-o", str(exe), str(src), f"-L{libdir}", "-lctfiss",
                    f"-Wl,-rpath,{libdir}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    obj = np.array([float(v) for v in out[:6]])
    W = np.array([complex(*map(float, l.split())) for l in out[6:] if l.strip()]).reshape(F, D, D)
    ref = O.run(O.config([2, 2], [3, 3], iterations=6, seed=21), x)
    assert np.max(np.abs(obj - ref["objective"]) / np.abs(ref["objective"])) <= 1e-9
    assert rel(W, ref["W"]) <= 1e-9


def _ip_history(raw, L, K, iters, precision, seed):
    M = raw.shape[3]
    s = Session(raw, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision=precision, seed=seed,
                update_rule="ip")
    assert "gram_kernel" in json.loads(s.describe())["sweep_kernel"]
    hist = []
    for _ in range(iters):
        s.iterate(1)
        hist.append(tuple(s.download_raw()) + (None,))
    s.close()
    return hist


@pytest.mark.parametrize("M,L,T,K", [(2, 2, 200, 3), (2, 5, 400, 4), (3, 4, 300, 3)])
def test_ip_rule_fp64_every_iteration(M, L, T, K):
    """IP rule on the GPU (estimator.cpp:580-606: weighted covariance, pivoted
    solve of W h u = e_r, normalisation, frame-sum refinement; exact log|det|)
    against the oracle's IP run: 1e-9 relative after every iteration."""
    F, iters, seed = 21, 8, 4
    raw = synth_mixtures(1, F, T, M, M, L, K, 0.6, 900 + M * L)
    ref = O.run(O.config([L] * M, [K] * M, iterations=iters, seed=seed, threads=NPROC, rule="ip"),
                O.stack_observation(raw[0], L), history=True)
    hist = _ip_history(raw, L, K, iters, "f64", seed)
    check_history(hist, ref, 0, 1e-9, f"ip M={M} L={L}")


def test_ip_rule_fp32_tolerance_and_iss_vs_ip():
    """fp32 IP within the north-star fp32 tolerance of the fp64 oracle, and
    ISS and IP reach nearby objectives (test_run.cpp:136-150, 5 %)."""
    M, L, T, K, F, iters, seed = 2, 3, 400, 4, 33, 20, 6
    raw = synth_mixtures(1, F, T, M, M, L, K, 0.6, 77)
    ref = O.run(O.config([L] * M, [K] * M, iterations=iters, seed=seed, threads=NPROC, rule="ip"),
                O.stack_observation(raw[0], L), history=True)
    hist = _ip_history(raw.astype(np.complex64), L, K, iters, "f32", seed)
    for it, (W, B, V, obj, _) in enumerate(hist):
        e = max(rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]),
                rel(V[0], ref["hist_V"][it]))
        assert e <= 1e-4, f"it={it + 1}: {e:.2e}"
    iss = gpu_history(raw, [L] * M, [K] * M, iters, "f64", seed, L)[-1][3][0, -1]
    ip = hist[-1][3][0, -1]
    assert abs(ip - iss) / abs(iss) < 0.05


@pytest.mark.parametrize("precision,tol", [("f64", 1e-9), ("f32", 1e-4)])
@pytest.mark.parametrize("taps,bases", [([2, 2], [3, 3]), ([2, 3], [2, 4]), ([1, 2, 1], [2, 3, 2])])
def test_ip_rule_general_layouts_every_iteration(taps, bases, precision, tol):
    """IP rule on layouts the covariance-domain kernel does not cover: a
    pre-stacked observation (equal and unequal taps per source, the
    reference's general CtfConfig), served by the frame-domain IP variant
    (weighted covariance from the x tile, ip_solve_row, frame-sum refinement,
    estimator.cpp:580-606, 89-273) against the oracle's IP run after every
    iteration."""
    g = np.random.default_rng(31 + len(taps) + sum(taps))
    F, T, iters, seed = 11, 160, 6, 9
    D = sum(taps)
    xm = (g.standard_normal((F, T, D)) + 1j * g.standard_normal((F, T, D))).astype(np.complex128)
    x = xm[None] if precision == "f64" else xm[None].astype(np.complex64)
    s = Session(x, taps, bases, stack_taps=1, iterations=iters, precision=precision, seed=seed, update_rule="ip")
    assert json.loads(s.describe())["sweep_kernel"].startswith("sweep_kernel"), s.describe()
    ref = O.run(O.config(taps, bases, iterations=iters, seed=seed, threads=NPROC, rule="ip"), xm, history=True)
    for it in range(iters):
        s.iterate(1)
        W, B, V, obj = s.download_raw()
        e = max(rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]),
                rel(V[0], ref["hist_V"][it]))
        eo = abs(obj[0, it] - ref["objective"][it]) / abs(ref["objective"][it])
        assert e <= tol and eo <= tol, f"taps={taps} {precision} it={it + 1}: {e:.2e} obj {eo:.2e}"
    s.close()


def test_ip_rule_errors_and_run_api():
    """run(config with update_rule='ip') on a stacked observation; the IP rule
    with CheckOptions is refused (unsupported), never silently run on another
    path."""
    M, L, T, K, F = 2, 2, 120, 3, 9
    raw = synth_mixtures(1, F, T, M, M, L, K, 0.6, 5)
    cfg = CtfConfig(M, M * L, [L] * M, [K] * M, iterations=3, update_rule="ip", seed=2)
    res = run(cfg, np.transpose(raw[0], (0, 2, 1)), stack_taps=L)
    ref = O.run(O.config([L] * M, [K] * M, iterations=3, seed=2, rule="ip"), O.stack_observation(raw[0], L))
    assert rel(res.demixing, np.transpose(ref["W"], (0, 2, 1))) <= 1e-9
    with pytest.raises(Exception):
        run(cfg, np.transpose(raw[0], (0, 2, 1)), CheckOptions(det_lemma=True), stack_taps=L)


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_covariance_kernel_error_paths(precision):
    """The error semantics of test_run.cpp:219-268 on the covariance-domain
    kernel (stacked equal-tap input selects it): a NaN sample -> "non-finite"
    (the finite checks), a silent bin -> the steering degeneracy at iteration 1
    of the lowest silent bin, with the same messages as the oracle."""
    M, L, K, F, T = 2, 3, 3, 7, 40
    raw = synth_mixtures(1, F, T, M, M, L, K, 0.6, 11)
    if precision == "f32":
        raw = raw.astype(np.complex64)
    s = Session(raw, [L] * M, [K] * M, stack_taps=L, iterations=2, precision=precision, seed=1)
    assert "gram_kernel" in json.loads(s.describe())["sweep_kernel"]
    s.close()
    bad = raw.copy()
    bad[0, 3, 5, 1] = np.nan
    with pytest.raises(DegeneracyError) as e:
        s = Session(bad, [L] * M, [K] * M, stack_taps=L, iterations=2, precision=precision, seed=1)
        s.iterate(2)
    assert "non-finite" in str(e.value)
    silent = raw.copy()
    silent[0, 2] = 0
    silent[0, 5] = 0
    ref_err = None
    try:
        O.run(O.config([L] * M, [K] * M, iterations=2, seed=1), O.stack_observation(silent[0].astype(complex), L))
    except O.OracleError as oe:
        ref_err = oe
    assert ref_err is not None and ref_err.iteration == 1 and ref_err.bin == 2
    with pytest.raises(DegeneracyError) as e:
        s = Session(silent, [L] * M, [K] * M, stack_taps=L, iterations=2, precision=precision, seed=1)
        s.iterate(2)
    assert e.value.iteration == 1 and e.value.bin == 2 and "iteration 1" in str(e.value)
    assert str(e.value).split(" (iteration")[0] == str(ref_err).split(" (iteration")[0]


def test_covariance_kernel_sharded_degeneracy():
    """A silent bin in rank 1's shard on the covariance-domain kernel raises the
    same DegeneracyError on every rank."""
    import threading
    from paper_2510_02382_b200 import _lib
    M, L, K, F, T = 2, 2, 3, 8, 40
    raw = synth_mixtures(1, F, T, M, M, L, K, 0.6, 12).astype(np.complex64)
    raw[0, 6] = 0
    lib = _lib.load()
    grp = lib.ctf_group_create(2)
    errs = [None, None]

    def worker(r):
        try:
            s = Session(raw, [L] * M, [K] * M, stack_taps=L, iterations=2, precision="f32", world_size=2, rank=r,
                        group=grp)
            s.iterate(2)
        except DegeneracyError as e:
            errs[r] = e

    th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
    [t.start() for t in th]
    [t.join() for t in th]
    lib.ctf_group_destroy(grp)
    for e in errs:
        assert e is not None and e.iteration == 1 and e.bin == 6


@pytest.mark.parametrize("M,L,T,prec", [(2, 3, 37, "f64"), (2, 5, 1001, "f32"), (3, 4, 301, "f32"),
                                        (3, 4, 301, "f64"), (2, 2, 511, "f32")])
def test_covariance_kernel_odd_frame_counts(M, L, T, prec):
    """Frame counts that are not multiples of 4 (scalar lambda path), odd T*M
    (scalar x-tile path) and T just below a CTA tile: per-iteration parity
    with the oracle (fp64 1e-9, fp32 1e-4)."""
    F, K, iters, seed = 9, 3, 4, 8
    raw = synth_mixtures(1, F, T, M, M, L, K, 0.6, 300 + T)
    x = raw.astype(np.complex64) if prec == "f32" else raw
    s = Session(x, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision=prec, seed=seed)
    assert "gram_kernel" in json.loads(s.describe())["sweep_kernel"]
    s.close()
    ref = O.run(O.config([L] * M, [K] * M, iterations=iters, seed=seed, threads=NPROC),
                O.stack_observation(raw[0], L), history=True)
    hist = gpu_history(x, [L] * M, [K] * M, iters, prec, seed, L)
    tol = 1e-9 if prec == "f64" else 1e-4
    for it, (W, B, V, obj, _) in enumerate(hist):
        e = max(rel(W[0], ref["hist_W"][it].reshape(F, -1)), rel(B[0], ref["hist_B"][it]),
                rel(V[0], ref["hist_V"][it]))
        assert e <= tol, f"it={it + 1}: {e:.2e}"


@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_zero_iterations_returns_the_initial_state(precision):
    """run() with iterations = 0 (the loop body never runs): identity W and the
    host-drawn initial factors, as the oracle returns them."""
    M, L, K, F, T = 2, 3, 3, 9, 64
    raw = synth_mixtures(1, F, T, M, M, L, K, 0.6, 1)
    x = raw.astype(np.complex64) if precision == "f32" else raw
    s = Session(x, [L] * M, [K] * M, stack_taps=L, iterations=0, precision=precision, seed=7)
    s.iterate(0)
    W, B, V, obj = s.download_raw()
    s.close()
    ref = O.run(O.config([L] * M, [K] * M, iterations=0, seed=7), O.stack_observation(raw[0], L))
    assert rel(W[0], ref["W"].reshape(F, -1)) == 0.0
    tol = 0.0 if precision == "f64" else 1e-7
    assert rel(B[0], ref["B"]) <= tol and rel(V[0], ref["V"]) <= tol


@pytest.mark.parametrize("precision,tol,theta", [("f64", 1e-9, "0"), ("f64", 1e-9, "6"), ("f32", 1e-4, "0"),
                                                 ("f32", 1e-4, "6")])
def test_gram_conditioning_fallback(monkeypatch, precision, tol, theta):
    """The covariance-domain kernel hands ill-conditioned bins to the
    frame-domain kernel (SweepParams::fb_mode). theta 0 forces every bin over
    from iteration 2 on, theta 6 a data-dependent subset: the trajectory
    still matches the oracle after every iteration."""
    monkeypatch.setenv("CTF_GRAM_FALLBACK_THETA", theta)
    F, T, M, L, K, iters, seed = 9, 300, 2, 5, 4, 6, 2
    raw = synth_mixtures(1, F, T, M, M, L, K, 0.6, 99)
    ref = O.run(O.config([L] * M, [K] * M, iterations=iters, seed=seed, threads=NPROC),
                O.stack_observation(raw[0], L), history=True)
    x = raw if precision == "f64" else raw.astype(np.complex64)
    s = Session(x, [L] * M, [K] * M, stack_taps=L, iterations=iters, precision=precision, seed=seed)
    d = json.loads(s.describe())
    s.close()
    assert "gram_kernel" in d["sweep_kernel"] and d["gram_fallback"] is True, d
    hist = gpu_history(x, [L] * M, [K] * M, iters, precision, seed, L)
    check_history(hist, ref, 0, tol, f"fallback theta={theta}")
