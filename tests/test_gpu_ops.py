"""Op-level entries (ctf_op_*, paper_2510_02382_b200.ops) on the GPU against
the matching oracle ops (oracle/ctf_oracle.cpp, pinned to the reference's own
code by tests/test_ref_pins.py), on the seeded inputs test_ref_pins uses:
demix, compute_psd, iss_sweep, mu_update_bases/activations, rescale,
log_abs_det, objective_from_parts (estimator.hpp:56-117). fp64, 1e-12
relative (summation order differs from Eigen's; the reference's own op tests
pin these to 1e-10 .. 1e-12)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_02382_b200 import DegeneracyError
from paper_2510_02382_b200 import ops
from tests.test_oracle_kats import rand_c, rng, wmem, xmem

pytestmark = pytest.mark.gpu


def same(a, b, tol=1e-12):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b))) <= tol * max(float(np.max(np.abs(b))), 1e-300)


@pytest.fixture(scope="module")
def case():
    g = rng(21)
    taps, bases = [2, 3], [2, 4]
    F, T, D = 5, 12, 5
    cfg = O.config(taps, bases, iterations=1, seed=9)
    x = xmem(rand_c(g, F, D, T))
    W = wmem(rand_c(g, F, D, D) + 3 * np.eye(D))
    floor = 1e-10 * O.mean_power(x)
    B, V = O.random_factors(cfg, F, T)
    return dict(taps=taps, bases=bases, F=F, T=T, D=D, cfg=cfg, x=x, W=W, floor=floor, B=B, V=V)


def test_op_demix_and_psd(case):
    c = case
    assert same(ops.demix(c["W"], c["x"]), O.demix(c["W"], c["x"]))
    lam = O.compute_psd(c["cfg"], c["F"], c["T"], c["B"], c["V"], c["floor"])
    assert same(ops.compute_psd(c["taps"], c["bases"], c["F"], c["T"], c["B"], c["V"], c["floor"]), lam)


def test_op_iss_sweep(case):
    c = case
    Y = O.demix(c["W"], c["x"])
    lam = O.compute_psd(c["cfg"], c["F"], c["T"], c["B"], c["V"], c["floor"])
    Wg, Yg = ops.iss_sweep(c["taps"], c["W"], Y, lam)
    for b in range(c["F"]):
        Wo, Yo = O.iss_sweep(c["cfg"], c["W"][b], Y[b], lam, b)
        assert same(Wg[b], Wo, 1e-11) and same(Yg[b], Yo, 1e-11), b


def test_op_mu_updates(case):
    c = case
    Y = O.demix(c["W"], c["x"])
    for n in range(2):
        Bg = ops.mu_update_bases(c["taps"], c["bases"], c["F"], c["T"], c["B"], c["V"], c["floor"], Y, n)
        assert same(Bg, O.mu_update_bases(c["cfg"], c["F"], c["T"], c["B"], c["V"], c["floor"], Y, n))
        Vg = ops.mu_update_activations(c["taps"], c["bases"], c["F"], c["T"], c["B"], c["V"], c["floor"], Y, n)
        assert same(Vg, O.mu_update_activations(c["cfg"], c["F"], c["T"], c["B"], c["V"], c["floor"], Y, n))


def test_op_rescale_logdet_objective(case):
    c = case
    Y = O.demix(c["W"], c["x"])
    for u, v in zip(ops.rescale(c["taps"], c["bases"], c["F"], c["T"], c["W"], c["B"], c["floor"], Y),
                    O.rescale(c["cfg"], c["F"], c["T"], c["W"], c["B"], c["floor"], Y)):
        assert same(u, v)
    ld = ops.log_abs_det(c["W"])
    for b in range(c["F"]):
        assert ld[b] == pytest.approx(O.log_abs_det(c["W"][b]), rel=1e-13)
    lam = O.compute_psd(c["cfg"], c["F"], c["T"], c["B"], c["V"], c["floor"])
    assert ops.objective_from_parts(c["taps"], c["W"], lam, Y) == pytest.approx(
        O.objective_from_parts(c["cfg"], c["F"], c["T"], c["W"], lam, Y), rel=1e-12)


def test_op_error_paths(case):
    """Singular W -> the reference's zero-pivot text (estimator.cpp:46-47);
    a silent bin -> the steering degeneracy of its first row pair
    (estimator.cpp:451-454) with the lowest failing bin."""
    c = case
    Ws = c["W"].copy()
    Ws[2] = 0
    with pytest.raises(DegeneracyError) as e:
        ops.log_abs_det(Ws)
    assert "singular demixing matrix (zero pivot)" in str(e.value)
    x = c["x"].copy()
    x[3] = 0
    Y = O.demix(c["W"], x)
    lam = O.compute_psd(c["cfg"], c["F"], c["T"], c["B"], c["V"], c["floor"])
    with pytest.raises(DegeneracyError) as e:
        ops.iss_sweep(c["taps"], c["W"], Y, lam)
    with pytest.raises(O.OracleError) as eo:
        O.iss_sweep(c["cfg"], c["W"][3], Y[3], lam, 3)
    assert str(e.value) == str(eo.value) and e.value.bin == 3 and e.value.row == eo.value.row


def test_op_shapes_of_the_baseline_configs():
    """One bin of each stacked BASELINE geometry through the op chain demix ->
    iss_sweep -> rescale against the oracle (R = 10, 12, 32, 60)."""
    from paper_2510_02382_b200 import synth_mixtures
    for (M, L, T, K) in [(2, 5, 200, 3), (3, 4, 200, 3), (4, 8, 120, 2), (6, 10, 150, 2)]:
        raw = synth_mixtures(1, 2, T, M, M, L, K, 0.7, 3)
        x = O.stack_observation(raw[0], L)
        taps, bases = [L] * M, [K] * M
        cfg = O.config(taps, bases, iterations=1, seed=1)
        F, D = 2, M * L
        W = np.zeros((F, D, D), complex)
        W[:] = np.eye(D)
        B, V = O.random_factors(cfg, F, T)
        floor = 1e-10 * O.mean_power(x)
        Y = ops.demix(W, x)
        assert same(Y, O.demix(W, x))
        lam = ops.compute_psd(taps, bases, F, T, B, V, floor)
        Wg, Yg = ops.iss_sweep(taps, W, Y, lam)
        for b in range(F):
            Wo, Yo = O.iss_sweep(cfg, W[b], Y[b], lam, b)
            assert same(Wg[b], Wo, 1e-10) and same(Yg[b], Yo, 1e-10), (M, L, b)


def test_cpp_op_mirror_runs_one_loop_body(tmp_path):
    """The C++ op-level mirror (ctfmnmf_b200.hpp: demix, iss_sweep,
    mu_update_bases/activations, rescale, compute_psd, objective_from_parts)
    driven through one loop body in run()'s order (estimator.cpp:553-648)
    equals the oracle's one-iteration step from the same state."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    csrc = os.path.join(root, "paper_2510_02382_b200", "csrc")
    libdir = os.path.join(root, "paper_2510_02382_b200")
    g = rng(4)
    F, T, taps, bases = 5, 30, [2, 2], [3, 3]
    D = sum(taps)
    x = xmem(rand_c(g, F, D, T))
    cfg = O.config(taps, bases, iterations=1, seed=6)
    floor = 1e-10 * O.mean_power(x)
    B, V = O.random_factors(cfg, F, T)
    W = np.zeros((F, D, D), complex)
    W[:] = np.eye(D)
    x.astype(np.complex128).tofile(tmp_path / "x.bin")
    B.tofile(tmp_path / "b.bin")
    V.tofile(tmp_path / "v.bin")
    src = tmp_path / "ops.cpp"
    src.write_text(f'''#include "ctfmnmf_b200.hpp"
#include <cstdio>
#include <fstream>
using namespace ctfmnmf::b200;
int main() {{
  CtfConfig c; c.num_sources = 2; c.num_channels = {D}; c.taps_per_source = {{2, 2}}; c.bases_per_source = {{3, 3}};
  MixtureSpectrogram x; x.bins.assign({F}, CMatrix({D}, {T}));
  std::ifstream in("{tmp_path / 'x.bin'}", std::ios::binary);
  for (auto& b : x.bins) in.read(reinterpret_cast<char*>(b.data.data()), b.data.size() * sizeof(Complex));
  NmfFactors f; f.floor = {floor!r};
  std::ifstream bi("{tmp_path / 'b.bin'}", std::ios::binary), vi("{tmp_path / 'v.bin'}", std::ios::binary);
  for (int n = 0; n < 2; ++n) {{ f.bases.emplace_back({F}, 3); bi.read(reinterpret_cast<char*>(f.bases.back().data.data()), {F} * 3 * 8); }}
  for (int n = 0; n < 2; ++n) {{ f.activations.emplace_back(3, {T}); vi.read(reinterpret_cast<char*>(f.activations.back().data.data()), 3 * {T} * 8); }}
  std::vector<CMatrix> W({F}, CMatrix({D}, {D}));
  for (auto& w : W) for (int i = 0; i < {D}; ++i) w(i, i) = 1.0;
  std::vector<RMatrix> lam{{compute_psd(f, 0), compute_psd(f, 1)}};
  DelayedEstimates y = demix(W, x);
  for (int i = 0; i < {F}; ++i) iss_sweep(W[i], y.bins[i], lam, c, i);
  y = demix(W, x);
  for (int n = 0; n < 2; ++n) mu_update_bases(f, y, n, c);
  for (int n = 0; n < 2; ++n) mu_update_activations(f, y, n, c);
  rescale(W, f, y, c);
  lam = {{compute_psd(f, 0), compute_psd(f, 1)}};
  std::printf("%.17g\\n", objective_from_parts(W, lam, y, c));
  for (const auto& w : W) for (const auto& v : w.data) std::printf("%.17g %.17g\\n", v.real(), v.imag());
  return 0;
}}''')
    exe = tmp_path / "ops"
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{csrc}", "-o", str(exe), str(src), f"-L{libdir}", "-lctfiss",
                    f"-Wl,-rpath,{libdir}"], check=True)
    out = [l for l in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n") if l]
    obj = float(out[0])
    Wg = np.array([complex(*map(float, l.split())) for l in out[1:]]).reshape(F, D, D)
    Wo, Bo, Vo, objo = O.step(cfg, x, floor, W, B, V)
    assert abs(obj - objo) <= 1e-10 * abs(objo)
    assert same(Wg, Wo, 1e-10)
