"""The committed golden fixtures (tests/golden, produced by the reference's own
code, oracle/_ref, with tests/golden/make_golden.py) still match the
restatement oracle and the generator."""
import os

import numpy as np
import pytest

from oracle import oracle as O

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_case(name):
    import importlib.util
    spec = importlib.util.spec_from_file_location("make_golden", os.path.join(HERE, "make_golden.py"))
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    c = mg.CASES[name]
    raw, x = mg.make_input(c)
    taps, bases = mg.taps_bases(c)
    g = np.load(os.path.join(HERE, f"{name}.npz"))
    return mg, c, raw, x, taps, bases, g


CASES = ["stacked_m2_l2", "cfg0_small", "general_taps23_bases24"]


@pytest.mark.parametrize("name", CASES)
def test_golden_inputs_and_oracle_reproduce(name):
    mg, c, raw, x, taps, bases, g = load_case(name)
    assert mg.digest(raw) == str(g["x_sha256"])
    r = O.run(O.config(taps, bases, iterations=c["iters"], seed=c["seed"]), x, history=True)
    np.testing.assert_allclose(r["objective"], g["objective"], rtol=1e-12)
    for k in ("hist_W", "hist_B", "hist_V"):
        assert np.abs(r[k] - g[k]).max() <= 1e-12 * np.abs(g[k]).max()


def test_cfg0_full_fixture_matches_restatement():
    """BASELINE configs[0] at full size (reference-produced objective trace and
    checkpoints) against the restatement."""
    import os as _os
    mg, c, raw, x, taps, bases, g = load_case("cfg0_full")
    assert mg.digest(raw) == str(g["x_sha256"])
    nproc = min(_os.cpu_count() or 1, 8)
    for k in g["checkpoints"]:
        r = O.run(O.config(taps, bases, iterations=int(k), seed=c["seed"], threads=nproc), x)
        for key in ("W", "B", "V"):
            ref = g[f"{key}_{k}"]
            assert np.abs(r[key] - ref).max() <= 1e-12 * np.abs(ref).max(), (key, k)
        if k == c["iters"]:
            np.testing.assert_allclose(r["objective"], g["objective"], rtol=1e-12)
