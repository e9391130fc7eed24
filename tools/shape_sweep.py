"""Dev: the covariance-domain kernel against the frame-domain kernel
(CTF_SWEEP_KIND=0) on stacked equal-tap shapes: ms per iteration of 16
mixtures at F = 513, T = 1000, K = 10. usage: python tools/shape_sweep.py f32|f64 "M,L M,L ..." """
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json
sys.path.insert(0, %r)
from paper_2510_02382_b200 import Session, synth_mixtures
M, L, prec = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
B, F, T, K = 16, 513, 1000, 10
x = synth_mixtures(B, F, T, M, M, L, K, 0.6, 1, precision=prec)
s = Session(x, [L] * M, [K] * M, stack_taps=L, iterations=6, precision=prec)
d = json.loads(s.describe())
s.iterate(1); s.reset_timing(); s.iterate(5)
t = s.timing()
print(json.dumps({"kernel": d["sweep_kernel"], "sweep_ms": t.sweep_ms / 5, "mu_ms": t.mu_ms / 5}))
''' % ROOT
prec = sys.argv[1]
for ml in sys.argv[2].split():
    M, L = map(int, ml.split(","))
    row = []
    for kind in (None, "0"):
        env = dict(os.environ)
        if kind is not None:
            env["CTF_SWEEP_KIND"] = kind
        out = subprocess.run([sys.executable, "-c", CHILD, str(M), str(L), prec], env=env, capture_output=True, text=True)
        try:
            r = json.loads(out.stdout.strip().splitlines()[-1])
            row.append(f"{r['kernel'].split('<')[0]:13s} {r['sweep_ms']:7.3f} ms")
        except Exception:
            row.append("failed: " + (out.stderr.strip().splitlines() or ["?"])[-1][:80])
    print(f"{prec} M={M} L={L} R={M*L:2d}:  default {row[0]}   frame-domain {row[1]}", flush=True)
