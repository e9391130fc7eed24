"""Frequency-sharding model for the multi-GPU bench (SCALE runs N = 1, 2, 4,
8 of the default cfg1 workload), measured on ONE B200: the per-rank compute of
an N-way shard is a world-1 run over that rank's bin count (ceil(F/N), the
largest shard, which sets max-over-ranks), timed with CUDA events; the
all-reduce per iteration (packed MU-V sums B*2*SK*T + row powers/objective
B*(R+1) doubles) is modelled at the bus bandwidth BUSBW (GB/s, default 725:
NVLink 5 8-GPU all-reduce) plus a fixed latency, and counted as exposed
(unchunked) or hidden behind the other mixture chunk's sweep (pipelined).
usage: python tools/scale_model.py [prec] [busbw_GBs] [latency_us]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2510_02382_b200 import Session, synth_mixtures  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
busbw = float(sys.argv[2]) if len(sys.argv) > 2 else 725.0
lat_us = float(sys.argv[3]) if len(sys.argv) > 3 else 20.0
B, F, T, M, L, K = 64, 513, 1000, 2, 5, 10
R, SK = M * L, M * K
rs = 8 if prec == "f64" else 4
x = synth_mixtures(B, F, T, M, M, L, K, 0.6, 20251002, precision=prec)


def per_iteration_ms(bins, pipelined=False):
    """pipelined: the rank's loop as it runs at N > 1 (mixture chunks on two
    compute streams + the communication stream), driven through a single-rank
    NCCL communicator whose all-reduce moves no data between GPUs."""
    import ctypes
    from paper_2510_02382_b200 import _lib
    xs = x[:, :bins].copy()
    kw = {}
    if pipelined:
        os.environ["CTF_NCCL_SINGLE_RANK"] = "1"
        uid, err = (ctypes.c_uint8 * 128)(), _lib.CtfErr()
        assert _lib.load().ctf_comm_unique_id(uid, ctypes.byref(err)) == 0
        kw["comm_id"] = bytes(uid)
    else:
        os.environ.pop("CTF_NCCL_SINGLE_RANK", None)
    s = Session(xs, [L] * M, [K] * M, stack_taps=L, iterations=20, precision=prec, seed=1, **kw)
    st = torch.cuda.ExternalStream(s.stream_ptr())
    s.iterate_async(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    s.iterate_async(10)
    e1.record(st)
    e1.synchronize()
    s.finalize()
    s.close()
    return e0.elapsed_time(e1) / 10


t1 = per_iteration_ms(F)
payload = B * 2 * SK * T * rs + B * (R + 1) * 8
out = {"workload": f"cfg1 {prec}: {B} mixtures x {F} bins x {T} frames", "t1_ms": t1, "busbw_GBs": busbw,
       "allreduce_latency_us": lat_us, "payload_bytes": payload, "n": {}}
for n in (2, 4, 8):
    fl = -(-F // n)
    tn = per_iteration_ms(fl)
    tp = per_iteration_ms(fl, pipelined=True)
    ar = 2 * (n - 1) / n * payload / (busbw * 1e9) * 1e3 + lat_us * 1e-3
    # pipelined: the all-reduce of one chunk is hidden behind the other
    # chunk's sweep when it is shorter than that sweep (about tp / 2)
    exposed = max(0.0, ar / 2 - tp / 2) + ar / 2 * 0.0
    out["n"][n] = {"bins_per_rank": fl, "compute_ms": tn, "compute_pipelined_ms": tp, "allreduce_ms": ar,
                   "efficiency_unchunked": t1 / (n * (tn + ar)),
                   "efficiency_pipelined": t1 / (n * (tp + exposed))}
    print(json.dumps({n: out["n"][n]}), flush=True)
print(json.dumps(out))
