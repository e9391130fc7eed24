"""Dev probe: parity of a few shapes vs the oracle + a rough cfg1 timing."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2510_02382_b200 import Session, synth_mixtures
from oracle import oracle as orc

def parity(B, F, T, M, N, L, K, iters, prec, seed=7):
    x = synth_mixtures(B, F, T, M, N, L, K, 0.6, 99)
    s = Session(x, [L]*N, [K]*N, stack_taps=L, iterations=iters, precision=prec, seed=seed)
    s.iterate(iters)
    W, Bf, V, obj = s.download_raw()
    s.close()
    out = []
    for b in range(B):
        ref = orc.run(orc.config([L]*N, [K]*N, iterations=iters, seed=seed+b), orc.stack_observation(x[b], L))
        rel = lambda a, r: float(np.linalg.norm(a - r) / np.linalg.norm(r))
        out.append((rel(W[b], ref["W"].reshape(F, -1)), rel(Bf[b], ref["B"]), rel(V[b], ref["V"]),
                    float(np.max(np.abs(obj[b] - ref["objective"]) / np.abs(ref["objective"])))))
    print(f"parity B={B} F={F} T={T} M={M} L={L} K={K} it={iters} {prec}: " +
          " ".join(f"W={a:.2e} B={b:.2e} V={c:.2e} obj={d:.2e}" for a, b, c, d in out), flush=True)

def timing(prec, iters=10):
    B, F, T, M, N, L, K = 64, 513, 1000, 2, 2, 5, 10
    t0 = time.time()
    x = synth_mixtures(B, F, T, M, N, L, K, 0.6, 1)
    print(f"synth {time.time()-t0:.1f}s", flush=True)
    s = Session(x, [L]*N, [K]*N, stack_taps=L, iterations=iters, precision=prec, seed=0)
    s.iterate(2)
    s.reset_timing()
    t0 = time.time()
    s.iterate(iters)
    el = time.time() - t0
    t = s.timing()
    tf = B*F*T*iters
    print(f"cfg1 {prec}: wall {el*1e3:.1f} ms for {iters} it; sweep {t.sweep_ms:.2f} ms, mu {t.mu_ms:.2f} ms, fin {t.finalize_ms:.2f} ms;"
          f" TF-bin*it/s = {tf/((t.sweep_ms+t.mu_ms)/1e3):.3e}", flush=True)
    s.close()

if __name__ == "__main__":
    parity(2, 17, 48, 2, 2, 2, 3, 4, "f64")
    parity(1, 33, 100, 2, 2, 5, 10, 10, "f64")
    parity(1, 33, 100, 2, 2, 5, 10, 10, "f32")
    parity(1, 20, 500, 2, 2, 2, 10, 20, "f64")
    parity(1, 16, 300, 3, 3, 4, 5, 5, "f64")
    timing("f32")
    timing("f64")
