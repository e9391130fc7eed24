"""Small invocations of the iteration kernels for compute-sanitizer
(racecheck / synccheck / memcheck): one case per process so each tool run
stays short. usage: python tools/sanitize_case.py <case>
cases: gram25 (covariance-domain (2,5)), gram25fb (its frame-domain
fallback forced), frame (sweep_kernel fp64 R=4), fsplit2 / fsplit2o (cfg3
tile, 2-CTA cluster, all-gather / owner exchange), fsplit8 / fsplit8o (cfg4
tile, 8-CTA cluster), muv (MU-V partial + reduce/apply), image, stft."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
case = sys.argv[1]
env = {
    "gram25": {}, "gram25fb": {"CTF_GRAM_FALLBACK_THETA": "0"}, "frame": {},
    "fsplit2": {"CTF_SWEEP_KIND": "5", "CTF_SWEEP_VARIANT": "32,4,16,128", "CTF_FSPLIT_AG": "1"},
    "fsplit2o": {"CTF_SWEEP_KIND": "5", "CTF_SWEEP_VARIANT": "32,4,16,128", "CTF_FSPLIT_AG": "0"},
    "fsplit8": {"CTF_SWEEP_KIND": "5", "CTF_SWEEP_VARIANT": "60,2,32,256", "CTF_FSPLIT_AG": "1"},
    "fsplit8o": {"CTF_SWEEP_KIND": "5", "CTF_SWEEP_VARIANT": "60,2,32,256", "CTF_FSPLIT_AG": "0"},
    "muv": {}, "image": {}, "stft": {},
}[case]
os.environ.update(env)
from paper_2510_02382_b200 import Session, forward_stft, inverse_stft, synth_mixtures  # noqa: E402

if case.startswith("gram") or case in ("muv", "image"):
    M, L, T, K, F, prec = 2, 5, 200, 4, 3, "f32"
elif case == "frame":
    M, L, T, K, F, prec = 2, 2, 100, 3, 3, "f64"
elif case.startswith("fsplit2"):
    M, L, T, K, F, prec = 4, 8, 300, 4, 2, "f32"
elif case.startswith("fsplit8"):
    M, L, T, K, F, prec = 6, 10, 1500, 4, 1, "f32"
if case == "stft":
    sig = np.random.default_rng(1).standard_normal((2, 3000))
    spec = forward_stft(sig, 256, 64)
    back = inverse_stft(spec, 256, 64, 3000)
    print("stft round trip", float(np.abs(back - sig).max()))
    sys.exit(0)
raw = synth_mixtures(1, F, T, M, M, L, K, 0.7, 5)
x = raw if prec == "f64" else raw.astype(np.complex64)
s = Session(x, [L] * M, [K] * M, stack_taps=L, iterations=3, precision=prec, seed=1)
print(s.describe())
s.iterate(1)
s.iterate_async(2)
s.finalize()
W, B, V, obj = s.download_raw()
if case == "image":
    s.project_back()
s.close()
print(case, "objective", obj[0])
