"""bench.py contract on CPU: the reference arm (the reference's own run(),
oracle/_ref, timed on the host cores) prints one JSON line with the keys the
driver reads, never maps the product library, and under torchrun only rank 0
prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=env, timeout=600, cwd=ROOT)


def test_reference_arm_prints_one_contract_line():
    out = _run(["--impl", "reference", "--cfg", "0", "--steps", "1", "--warmup", "3"])
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    from oracle import ref as R
    assert d["cpu_baseline"]["kind"] == ("reference" if R.available() else "port")
    assert d["cpu_baseline"]["cores"] >= 1 and d["dtype"] == "f64"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("BASELINE configs[0]")


def test_reference_arm_non_zero_rank_is_silent():
    out = _run(["--impl", "reference", "--cfg", "0", "--steps", "1", "--warmup", "3"],
               {"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip() == ""


def test_reference_arm_never_maps_the_product_library():
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--cfg', '1', '--steps', '1', "
            "'--warmup', '0']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "print('PRODUCT_MAPPED' if 'libctfiss' in maps else 'PRODUCT_NOT_MAPPED', file=sys.stderr)")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    assert "PRODUCT_NOT_MAPPED" in out.stderr, out.stderr[-500:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["config"]["workload"].startswith("BASELINE configs[1]") and d["dtype"] == "f64"
