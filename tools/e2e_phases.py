"""Dev: where does ctf_run's time go outside the iterations (cfg1; argv[1] = f32 | f64)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_02382_b200 import _lib as LB, synth_mixtures
from paper_2510_02382_b200.api import _problem
B, F, T, M, L, K, it = 64, 513, 1000, 2, 5, 10, 100
prec = sys.argv[1] if len(sys.argv) > 1 else "f32"
x = synth_mixtures(B, F, T, M, M, L, K, 0.6, 1, precision=prec)
xh = torch.from_numpy(x.view(np.float32 if prec == "f32" else np.float64)).pin_memory()
lib = LB.load(); err = LB.CtfErr(); ctx = ctypes.c_void_p()
lib.ctf_open(0, ctypes.byref(ctx), ctypes.byref(err))
for iters in (0, 1, 100):
    prob = _problem(B, F, T, M, L, [L]*M, [K]*M, iters, prec, prec, 1e-10, 0)
    for rep in range(2):
        t0 = time.perf_counter(); lib.ctf_setup(ctx, ctypes.byref(prob), ctypes.c_void_p(xh.data_ptr()), ctypes.byref(err)); t1 = time.perf_counter()
        lib.ctf_iterate(ctx, iters, ctypes.byref(err)); t2 = time.perf_counter()
        R, SK = M*L, M*K
        W, Bf, V, o = (torch.zeros(n, dtype=torch.float64).pin_memory().numpy() for n in (B*F*R*R*2, B*F*SK, B*SK*T, B*max(iters,1)))
        lib.ctf_download(ctx, LB.dptr(W), LB.dptr(Bf), LB.dptr(V), LB.dptr(o), ctypes.byref(err)); t3 = time.perf_counter()
        print(f"iters={iters} rep={rep}: setup {1e3*(t1-t0):.1f} ms, iterate {1e3*(t2-t1):.1f} ms, download {1e3*(t3-t2):.1f} ms", flush=True)

R, SK = M*L, M*K
W, Bf, V, o = (torch.zeros(n, dtype=torch.float64).pin_memory().numpy() for n in (B*F*R*R*2, B*F*SK, B*SK*T, B*100))
prob = _problem(B, F, T, M, L, [L]*M, [K]*M, 100, prec, prec, 1e-10, 0)
for rep in range(3):
    t0 = time.perf_counter()
    rc = lib.ctf_run(ctx, ctypes.byref(prob), ctypes.c_void_p(xh.data_ptr()), LB.dptr(W), LB.dptr(Bf), LB.dptr(V), LB.dptr(o), ctypes.byref(err))
    t1 = time.perf_counter()
    print(f"ctf_run 100 iterations: {1e3*(t1-t0):.1f} ms (rc {rc})", flush=True)
# host->device bandwidth of the pinned x buffer alone
xd = torch.empty_like(xh, device="cuda")
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); xd.copy_(xh, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"H2D of x alone: {xh.numel() * xh.element_size() / 1e6:.0f} MB in {1e3*(t1-t0):.1f} ms", flush=True)
