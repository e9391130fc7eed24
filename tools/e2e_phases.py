"""Dev: where does ctf_run's time go outside the iterations (cfg1 fp32)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_02382_b200 import _lib as LB, synth_mixtures
from paper_2510_02382_b200.api import _problem
B, F, T, M, L, K, it = 64, 513, 1000, 2, 5, 10, 100
x = synth_mixtures(B, F, T, M, M, L, K, 0.6, 1, precision="f32")
xh = torch.from_numpy(x.view(np.float32)).pin_memory()
lib = LB.load(); err = LB.CtfErr(); ctx = ctypes.c_void_p()
lib.ctf_open(0, ctypes.byref(ctx), ctypes.byref(err))
for iters in (0, 1, 100):
    prob = _problem(B, F, T, M, L, [L]*M, [K]*M, iters, "f32", "f32", 1e-10, 0)
    for rep in range(2):
        t0 = time.perf_counter(); lib.ctf_setup(ctx, ctypes.byref(prob), ctypes.c_void_p(xh.data_ptr()), ctypes.byref(err)); t1 = time.perf_counter()
        lib.ctf_iterate(ctx, iters, ctypes.byref(err)); t2 = time.perf_counter()
        R, SK = M*L, M*K
        W = np.zeros(B*F*R*R*2); Bf = np.zeros(B*F*SK); V = np.zeros(B*SK*T); o = np.zeros(B*max(iters,1))
        lib.ctf_download(ctx, LB.dptr(W), LB.dptr(Bf), LB.dptr(V), LB.dptr(o), ctypes.byref(err)); t3 = time.perf_counter()
        print(f"iters={iters} rep={rep}: setup {1e3*(t1-t0):.1f} ms, iterate {1e3*(t2-t1):.1f} ms, download {1e3*(t3-t2):.1f} ms", flush=True)
