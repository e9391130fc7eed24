"""Dev: run a BASELINE config for a few iterations and print timing/variant."""
import argparse, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_02382_b200 import Session, synth_mixtures
CFG = {0: (1, 513, 500, 2, 2, 2, 10, 0.6), 1: (64, 513, 1000, 2, 2, 5, 10, 0.6),
       2: (128, 1025, 2000, 3, 3, 4, 20, 0.7), 3: (256, 2049, 1000, 4, 4, 8, 20, 0.8),
       4: (32, 1025, 4000, 6, 6, 10, 16, 0.85)}
ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=1); ap.add_argument("--prec", default="f32")
ap.add_argument("--iters", type=int, default=5); ap.add_argument("--mixtures", type=int, default=0)
ap.add_argument("--rule", default="iss")
a = ap.parse_args()
B, F, T, M, N, L, K, dec = CFG[a.cfg]
if a.mixtures: B = a.mixtures
x = synth_mixtures(B, F, T, M, N, L, K, dec, 1, precision="f32" if a.prec == "f32" else "f64")
s = Session(x, [L]*N, [K]*N, stack_taps=L, iterations=a.iters, precision=a.prec, update_rule=a.rule)
print(s.describe(), flush=True)
s.iterate(1); s.reset_timing()
s.iterate(a.iters)
t = s.timing()
n = B*F*T*a.iters
print(f"cfg{a.cfg} {a.prec} B={B}: sweep {t.sweep_ms/a.iters:.3f} ms/it, mu {t.mu_ms/a.iters:.3f} ms/it -> "
      f"{n/((t.sweep_ms+t.mu_ms)/1e3):.3e} TF-bin*it/s", flush=True)
