"""Dev: cost of the collective loop on one GPU — the plain world-1 loop vs
the same workload through a single-rank NCCL communicator
(CTF_NCCL_SINGLE_RANK=1: reduce -> ncclAllReduce -> apply), unchunked and
pipelined over mixture chunks. usage: python tools/mgpu_overhead.py [cfg] [prec]"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2510_02382_b200 import Session, _lib, synth_mixtures  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prec = sys.argv[2] if len(sys.argv) > 2 else "f64"
B, F, T, M, L, K = {1: (64, 513, 1000, 2, 5, 10), 2: (16, 1025, 2000, 3, 4, 20)}[cfg]
x = synth_mixtures(B, F, T, M, M, L, K, 0.6, 1, precision=prec)
lib = _lib.load()


def timed(**kw):
    s = Session(x, [L] * M, [K] * M, stack_taps=L, iterations=20, precision=prec, seed=1, **kw)
    d = json.loads(s.describe())
    st = torch.cuda.ExternalStream(s.stream_ptr())
    s.iterate_async(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.iterate_async(10)
    e1.record(st)
    e1.synchronize()
    torch.cuda.synchronize()
    s.finalize()
    s.close()
    return e0.elapsed_time(e1) / 10, d


ms, d = timed()
print(f"cfg{cfg} {prec} world 1 plain: {ms:.3f} ms/iteration ({d['collective']})", flush=True)
for chunks in ("1", "2", "4"):
    os.environ["CTF_NCCL_SINGLE_RANK"] = "1"
    os.environ["CTF_MIX_CHUNKS"] = chunks
    uid, err = (ctypes.c_uint8 * 128)(), _lib.CtfErr()
    assert lib.ctf_comm_unique_id(uid, ctypes.byref(err)) == 0
    ms, d = timed(comm_id=bytes(uid))
    print(f"cfg{cfg} {prec} single-rank NCCL, {d['mix_chunks']} mixture chunk(s): {ms:.3f} ms/iteration", flush=True)
