"""The N>1 path's decomposition, checked on CPU with world_size 2 over gloo.

Frequency sharding: each rank owns a contiguous bin range
(ctf_shard_range); everything bin-local (stacking, sweep, demix, MU-B,
energies) stays on the rank; the only exchange per iteration is one sum of
the packed [MU-V numerator | MU-V denominator | row powers | objective
partial] buffer. This test runs exactly that data flow per rank with the
oracle's bin-local operators plus a gloo all-reduce, and checks that the
gathered state equals the oracle's single-process iteration
(estimator.cpp:548-654)."""
import ctypes as C
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    from paper_2510_02382_b200 import synth_mixtures
    F, T, M, N, L, K = 11, 40, 2, 2, 2, 3
    x = O.stack_observation(synth_mixtures(1, F, T, M, N, L, K, 0.6, 3)[0], L)
    cfg = O.config([L] * N, [K] * N, iterations=1, seed=9)
    mp_ = O.mean_power(x)
    floor = 1e-10 * mp_
    B, V = O.random_factors(cfg, F, T)
    # warm the state up by two oracle iterations so z, mu are non-trivial
    W = np.zeros((F, M * L, M * L), complex)
    W[:] = np.eye(M * L).T
    for _ in range(2):
        W, B, V, _ = O.step(cfg, x, floor, W, B, V)
    return cfg, x, floor, W, B, V, (F, T, N, L, K)


def _rank_iteration(rank, world, cfg, x, floor, W, B, V, dims):
    F, T, N, L, K = dims
    from paper_2510_02382_b200 import _lib
    lo, hi = C.c_int(), C.c_int()
    _lib.load().ctf_shard_range(F, world, rank, C.byref(lo), C.byref(hi))
    lo, hi = lo.value, hi.value
    FL, R = hi - lo, N * L
    Bs = [B[n * F * K:(n + 1) * F * K].reshape(K, F).T for n in range(N)]
    Vs = [V[n * K * T:(n + 1) * K * T].reshape(T, K).T for n in range(N)]
    lam = np.stack([np.maximum(b @ v, floor) for b, v in zip(Bs, Vs)])  # (N, F, T)
    lam_mem = np.ascontiguousarray(np.transpose(lam, (0, 2, 1)))
    Wl = W[lo:hi].copy()
    Yl = O.demix(Wl, x[lo:hi])
    for i in range(FL):  # bin-local sweep (estimator.cpp:556-579)
        Wl[i], Yl[i] = O.iss_sweep(cfg, Wl[i], Yl[i], lam_mem, lo + i)
    Yl = O.demix(Wl, x[lo:hi])  # estimator.cpp:607
    # MU-B is bin-local: run it on the local bins as their own problem
    Bl = np.concatenate([b[lo:hi].T.ravel() for b in Bs])
    for n in range(N):
        Bl = O.mu_update_bases(cfg, FL, T, Bl, V, floor, Yl, n)
    Bls = [Bl[n * FL * K:(n + 1) * FL * K].reshape(K, FL).T for n in range(N)]
    # MU-V partial sums over the local bins (estimator.cpp:348-382)
    Ym = np.transpose(Yl, (0, 2, 1))  # (FL, R, T)
    packed = []
    for n in range(N):
        E = np.zeros((FL, T))
        for l in range(L):
            E[:, :T - l] += np.abs(Ym[:, n * L + l, l:]) ** 2
        cnt = np.array([min(L, T - t) for t in range(T)], float)
        lam2 = np.maximum(Bls[n] @ Vs[n], floor)
        il = 1.0 / lam2
        packed += [Bls[n].T @ (E * il * il), Bls[n].T @ (il * cnt)]
    rowpow = np.sum(np.abs(Ym) ** 2, axis=(0, 2))
    buf = torch.from_numpy(np.concatenate([p.ravel() for p in packed] + [rowpow]))
    dist.all_reduce(buf)  # the one exchange per iteration
    buf = buf.numpy()
    Vn, off = [], 0
    for n in range(N):
        num = buf[off:off + K * T].reshape(K, T)
        den = buf[off + K * T:off + 2 * K * T].reshape(K, T)
        Vn.append(np.maximum(Vs[n] * np.sqrt(num / den), floor))
        off += 2 * K * T
    mu = np.sqrt(buf[off:off + R] / (F * T))
    # rescale (estimator.cpp:384-412) of the local state
    for r in range(R):
        if mu[r] != 0:
            Wl[:, :, r] /= mu[r]
            Ym[:, r] /= mu[r]
    Bls = [np.maximum(Bls[n] / mu[n * L] ** 2, floor) if mu[n * L] != 0 else Bls[n] for n in range(N)]
    # objective partial (estimator.cpp:55-77) + its all-reduce
    obj = 0.0
    for n in range(N):
        lam3 = np.maximum(Bls[n] @ Vn[n], floor)
        for l in range(L):
            obj += np.sum(np.log(lam3[:, :T - l]) + np.abs(Ym[:, n * L + l, l:]) ** 2 / lam3[:, :T - l])
    for i in range(FL):
        obj -= 2.0 * T * O.log_abs_det(Wl[i])
    o = torch.tensor([obj], dtype=torch.float64)
    dist.all_reduce(o)
    return lo, hi, Wl, Bls, Vn, float(o[0])


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, x, floor, W, B, V, dims = _problem()
    lo, hi, Wl, Bls, Vn, obj = _rank_iteration(rank, world, cfg, x, floor, W, B, V, dims)
    out[rank] = (lo, hi, Wl, Bls, Vn, obj)
    dist.destroy_process_group()


def test_frequency_sharded_iteration_equals_single_process():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    cfg, x, floor, W, B, V, (F, T, N, L, K) = _problem()
    Wr, Br, Vr, objr = O.step(cfg, x, floor, W, B, V)
    Brs = [Br[n * F * K:(n + 1) * F * K].reshape(K, F).T for n in range(N)]
    Vrs = [Vr[n * K * T:(n + 1) * K * T].reshape(T, K).T for n in range(N)]
    for rank in range(world):
        lo, hi, Wl, Bls, Vn, obj = res[rank]
        assert np.abs(Wl - Wr[lo:hi]).max() <= 1e-10 * np.abs(Wr).max()
        for n in range(N):
            assert np.abs(Bls[n] - Brs[n][lo:hi]).max() <= 1e-10 * Brs[n].max()
            assert np.abs(Vn[n] - Vrs[n]).max() <= 1e-10 * Vrs[n].max()  # replicated V
        assert obj == pytest.approx(objr, rel=1e-10)
    assert sorted((res[r][0], res[r][1]) for r in range(world)) == [(0, 6), (6, 11)]
