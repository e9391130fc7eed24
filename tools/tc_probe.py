"""Dev: run tools/libtcprobe.so (one tcgen05.mma kind::tf32) and compare with numpy."""
import ctypes as C, os
import numpy as np
lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtcprobe.so"))
M, N = 38, 24
g = np.random.default_rng(0)
A = g.integers(-8, 8, (M, 8)).astype(np.float32)
B = g.integers(-8, 8, (N, 8)).astype(np.float32)
D = np.zeros((128, 24), np.float32)
f = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))
rc = lib.tc_probe(f(A), f(B), f(D), M, N)
want = A @ B.T
print("rc", rc, "max err rows<M:", np.max(np.abs(D[:M] - want)), "rows>=M max:", np.max(np.abs(D[M:])))
if np.max(np.abs(D[:M] - want)) > 0:
    print(D[:4, :8]); print(want[:4, :8])
    # where do results land?
    for r in range(4):
        hits = np.argwhere(np.isclose(D, want[r, 0]))
        print("row", r, "value", want[r, 0], "found at", hits[:5].tolist())
# 3xTF32 accuracy probe on real data
A = g.standard_normal((M, 8)).astype(np.float32)
B = g.standard_normal((N, 8)).astype(np.float32)
lib.tc_probe(f(A), f(B), f(D), M, N)
print("tf32 single-pass rel err:", np.max(np.abs(D[:M] - A.astype(np.float64) @ B.T.astype(np.float64))) / np.max(np.abs(A @ B.T)))
