#!/usr/bin/env python
"""Benchmark of the ISS+NMF hot path of CTF-MNMF-ISS on B200.

Metric (BASELINE.json): TF-bin*iter/s of the ISS+NMF loop (one TF-bin = one
(mixture, frequency bin, frame)); roofline fractions reported alongside.

Workload at N=1: BASELINE configs[1] — 64 mixtures, M=N=2, L=5 (stacked
D=10), F=513, T=1000, K=10, 100 iterations, in fp64 (complex128, the
reference's arithmetic, types.hpp:10) — the headline `value`/`e2e`/`roofline`;
configs[1] also asks for fp32, carried in the same line under "f32".
cfg2-cfg4 (--cfg) are fp32 as BASELINE states. Seeded synthetic mixtures
from BASELINE's generator.

  value : device-resident throughput — a "step" is one ISS+NMF iteration
          (estimator.cpp:548-654) over the whole batch with x already in HBM;
          K steps timed with CUDA events on the library's stream.
  e2e   : the same metric through the public C-ABI call ctf_run() with HOST
          buffers: per step the H2D of x (pinned), setup, 100 iterations and
          the D2H of W/B/V/objective are all inside the timed region.

Multi-GPU (torchrun): frequency sharding (contiguous bin ranges), one NCCL
all-reduce per iteration inside the library; strong scaling of the same
workload; times are the max over ranks.

--impl reference times the REFERENCE'S OWN CODE on the host cores: run()
from /root/reference/proj/src compiled unmodified into oracle/_ref
(oracle/Makefile.ref; kind "reference"), with config.threads = all host
threads (its bin-parallel parallel_for), one run() of 2 iterations of one
mixture per step (a bounded sample of the workload). If oracle/_ref did not
travel, the restatement oracle/ctf_oracle.cpp stands in (kind "port").
The reference arm never loads the product library (its inputs come from the
generator copy inside libctf_ref.so).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFGS = {  # BASELINE.json configs: B, F, T, M=N, L, K, rho, iterations
    0: (1, 513, 500, 2, 2, 10, 0.6, 100),
    1: (64, 513, 1000, 2, 5, 10, 0.6, 100),
    2: (128, 1025, 2000, 3, 4, 20, 0.7, 100),
    3: (256, 2049, 1000, 4, 8, 20, 0.8, 50),
    4: (32, 1025, 4000, 6, 10, 16, 0.85, 50),
}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def flops_per_tfbin(R, D, N, K):
    """Algorithmic flops per TF-bin*iteration, SURVEY §8(d) convention
    (complex MAC = 8, FMA = 2; logs/divisions not counted): the reference's
    iteration is 20R^2 (sweep) + 16RD (two demixes) + 14NK (lambda three
    times, MU-B, MU-V). The fused sweep kernel replaces the sweep, both
    demixes, the MU-B lambda + GEMMs and the lambda refresh (8NK); the MU-V
    kernel the rest (6NK). Returns (sweep kernel, iteration, executed), the
    last being what the sweep kernel actually computes (one demix: the second
    is replaced by carrying the swept Y)."""
    sweep = 20 * R * R + 16 * R * D + 8 * N * K
    return sweep, sweep + 6 * N * K, 20 * R * R + 8 * R * D + 6 * N * K


def gram_executed_flops(M, N, L, K, R, D, T):
    """Flops per TF-bin the covariance-domain kernel executes:
    Gram = complex x real MAC (4) per (lag entry, frame) over the Hermitian
    half of the (m, m', d) groups and all sources, one product per group and
    frame (6), the R covariance-domain steps (~8 R^2 D per bin), one demix
    (8RD), lambda + MU-B (6NK)."""
    groups, entries = 0, 0
    for m in range(M):
        for m2 in range(m, M):
            for d in range(0 if m == m2 else -(L - 1), L):
                groups += 1
                entries += 2 * L - 1 - abs(d)
    frames = (T + 2 * (L - 1)) / T
    return (4 * N * entries + 6 * groups) * frames + 8 * R * R * D / T + 8 * R * D + 6 * N * K


def bytes_per_tfbin(M, N, K, R, D, T, F, c):
    """Algorithmic HBM bytes per TF-bin*iteration of the resident design
    (SURVEY §8(d)): read x once, write+read energies E, read/write W, B, V
    amortised."""
    s = c // 2
    return M * c + 2 * N * s + 2 * R * D * c / T + 2 * N * K * s / T + 2 * N * K * s / F


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            p = [v.strip() for v in l.split(",")]
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, p[3:7]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def peak_probe(device):
    path = os.path.join(ROOT, "tools", "libctfpeak.so")
    if not os.path.exists(path):
        return None, None
    lib = C.CDLL(path)
    lib.ctf_peak_fp32_tflops.restype = C.c_double
    lib.ctf_peak_fp64_tflops.restype = C.c_double
    return lib.ctf_peak_fp32_tflops(device), lib.ctf_peak_fp64_tflops(device)


def profile_traffic(kernel, prec, cfgn):
    """dram read+write bytes per TF-bin of the dominant kernel from the
    committed ncu --set full capture of that kernel on that BASELINE config
    (profiles/sweep_traffic.json, keyed "<kernel>/<dtype>/cfg<n>"), scaled
    per launch by the caller; None when no capture of this config exists."""
    path = os.path.join(ROOT, "profiles", "sweep_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        v = d.get(f"{kernel}/{prec}/cfg{cfgn}")
        return v.get("bytes_per_tfbin") if isinstance(v, dict) else v
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
def cpu_reference_arm(args, cfgn, steps, warmup):
    """The reference on the host cores, bounded sample: one mixture of the
    config (a bin subset for the large tiles so one step stays around a
    second), each step one run() of 2 iterations (setup + 2 loop bodies,
    estimator.cpp:513-657) through oracle/_ref — the reference's own sources.
    Falls back to the restatement (oracle/ctf_oracle.cpp, kind "port") when
    the reference build is not present."""
    from oracle import oracle as O
    from oracle import ref as REF
    kind = "reference" if REF.available() else "port"
    B, F, T, M, L, K, rho, iters = CFGS[cfgn]
    N = M
    threads = os.cpu_count() or 1
    R = M * L
    F = min(F, max(16, int(513 * (1000.0 / T) * (100.0 / (R * R)))))
    if kind == "reference":
        raw = REF.synth_mixtures(1, F, T, M, N, L, K, rho, args.seed)[0]
    else:
        from paper_2510_02382_b200 import synth_mixtures
        raw = synth_mixtures(1, F, T, M, N, L, K, rho, args.seed)[0]
    x = O.stack_observation(raw, L)
    per = 2
    cfg = O.config([L] * N, [K] * N, iterations=per, seed=args.seed, threads=threads)
    times = []
    for st in range(warmup + steps):
        t0 = time.perf_counter()
        if kind == "reference":
            REF.run(cfg, x)
        else:
            O.run(cfg, x)
        dt = time.perf_counter() - t0
        if st >= warmup:
            times.append(dt)
    sec = sum(times)
    value = F * T * per * len(times) / sec
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except (OSError, IndexError):
        model = "unknown"
    impl = ("oracle/_ref: the reference's run() (proj/src/*.cpp compiled unmodified, Eigen-API shim)"
            if kind == "reference" else "oracle/ctf_oracle.cpp (restatement)")
    return {"value": value, "unit": "TF-bin*iter/s", "cores": threads, "kind": kind,
            "sample": f"1 of {B} mixtures, {F} of {CFGS[cfgn][1]} bins of cfg{cfgn} (T={T}, D={R}), "
                      f"{len(times)} steps of one run() with {per} iterations; {impl}, "
                      f"config.threads={threads} ({model}); {sec:.2f} s", "seconds": sec}


def workload_config(cfgn, world, dtype):
    """The config dict both arms print (identical, so the driver can pair them)."""
    B, F, T, M, L, K, rho, iters = CFGS[cfgn]
    D = M * L
    return {"workload": f"BASELINE configs[{cfgn}]: {B} mixtures, M=N={M}, L={L} (D={D}), F={F}, T={T}, "
                        f"K={K}, {iters} iterations, tap variance {rho}^l",
            "mixtures": B, "bins": F, "frames": T, "mics": M, "taps": L, "bases": K, "iterations": iters,
            "parallelism": f"freq-shard x{world}" if world > 1 else "1 GPU",
            "l2": "inputs larger than L2 (x alone is %.0f MB)" % (B * F * T * M * (8 if dtype == "f32" else 16) / 1e6)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cfg", type=int, default=1)
    ap.add_argument("--dtype", default="auto", choices=["auto", "f32", "f64"],
                    help="auto: f64 for cfg0/cfg1 (with the f32 line of cfg1 alongside), f32 for cfg2-4")
    ap.add_argument("--seed", type=int, default=20251002)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--unique", type=int, default=16,
                    help="distinct synthetic mixtures generated; the batch tiles them (seeds still differ per mixture)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-f32", action="store_true", help="cfg1: skip the fp32 line carried next to the fp64 headline")
    ap.add_argument("--no-frontend", action="store_true", help="skip the STFT/iSTFT front-end measurement")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.dtype == "auto":
        args.dtype = "f64" if args.cfg <= 1 else "f32"
    B, F, T, M, L, K, rho, iters = CFGS[args.cfg]
    N, R = M, M * L
    D = R
    config = workload_config(args.cfg, world, args.dtype)

    if args.impl == "reference":
        if rank != 0:
            return
        ref = cpu_reference_arm(args, args.cfg, args.steps, args.warmup)
        line = {"metric": "TF-bin*iter/s of the ISS+NMF loop", "value": ref["value"], "unit": "TF-bin*iter/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * ref["seconds"] / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE configs generator, seeded; no public dataset)",
                "config": config, "impl": "reference",
                "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": ref["value"], "unit": "TF-bin*iter/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    from paper_2510_02382_b200 import Session, synth_mixtures
    from paper_2510_02382_b200 import _lib as LB

    device = local
    torch.cuda.set_device(device)
    if world > 1:
        dist.init_process_group("gloo")
    def new_comm_id():
        """A fresh NCCL unique id from rank 0 for every communicator (an id is
        not reused once its communicator has been created)."""
        if world <= 1:
            return None
        buf = (C.c_uint8 * 128)()
        err = LB.CtfErr()
        if rank == 0:
            assert LB.load().ctf_comm_unique_id(buf, C.byref(err)) == 0, err.msg
        t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        dist.broadcast(t, 0)
        return bytes(t.tolist())

    comm_id = new_comm_id()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    def measure(prec, e2e_on, cpu_on):
        """One precision of the workload: device-resident loop (value),
        roofline of the dominant kernel, ctf_run() end to end (e2e)."""
        # BASELINE's generator, one seed per mixture; for large batches a set of
        # `--unique` mixtures is generated and tiled over the batch (throughput
        # does not depend on the content; init seeds stay distinct per mixture)
        nu = min(B, max(1, args.unique)) if B > 64 else B
        xu = synth_mixtures(nu, F, T, M, N, L, K, rho, args.seed, precision=prec)
        x = xu if nu == B else np.ascontiguousarray(np.concatenate([xu] * ((B + nu - 1) // nu))[:B])
        del xu
        inputs = f"{nu} distinct synthetic mixtures" + ("" if nu == B else f" tiled to {B}")
        s = Session(x, [L] * N, [K] * N, stack_taps=L, iterations=iters, precision=prec, seed=args.seed,
                    device=device, world_size=world, rank=rank, comm_id=comm_id if prec == args.dtype else new_comm_id())
        desc = json.loads(s.describe())
        stream = torch.cuda.ExternalStream(s.stream_ptr(), device=device)

        # ---- device-resident loop: W warm-up iterations, then K timed iterations
        s.iterate_async(max(args.warmup, 3))
        torch.cuda.synchronize(device)
        s.reset_timing()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with Clocks(device) as clk:
            torch.cuda.synchronize(device)
            barrier()
            ev0.record(stream)
            s.iterate_async(args.steps)
            ev1.record(stream)
            ev1.synchronize()
            torch.cuda.synchronize(device)
            barrier()
        ms = ev0.elapsed_time(ev1)
        timing = s.timing()  # per-kernel CUDA events on the library's stream
        s.finalize()
        ms = max_over_ranks(ms)
        sweep_ms = max_over_ranks(timing.sweep_ms / max(1, timing.sweep_launches))
        value = B * F * T * args.steps / (ms / 1e3)

        # ---- roofline of the dominant kernel (the fused iteration kernel)
        fl_sweep, fl_iter, fl_exec = flops_per_tfbin(R, D, N, K)
        if desc["sweep_kernel"].startswith("gram_kernel"):
            fl_exec = gram_executed_flops(M, N, L, K, R, D, T)
        peak = peaks[0] if prec == "f32" else peaks[1]
        local_bins = s.bin_range[1] - s.bin_range[0]
        units_per_launch = B * local_bins * T
        achieved = fl_sweep * units_per_launch / (sweep_ms / 1e3) / 1e12
        traffic_per_tfbin = profile_traffic(desc["sweep_kernel"].split("<")[0], prec, args.cfg)
        c = 8 if prec == "f32" else 16
        streamed = desc["sweep_kernel"].startswith("stream_kernel")
        bpt = bytes_per_tfbin(M, N, K, R, D, T, F, c)
        if streamed:  # SURVEY §8(d) streamed sweep: every step reads and writes the R x T tile
            bpt = 2 * M * c + R * c + 2 * R * R * c + bpt - M * c
        roofline = {"bound": "fp32-cuda-core" if prec == "f32" else "fp64-cuda-core",
                    "bound_note": ("compute-bound on the CUDA-core FMA pipes: neither HBM-bound (the hbm sub-object "
                                   "shows a few % of HBM) nor a tensor-core contraction (each ISS step is R "
                                   "differently weighted inner products; the fp32/fp64 tolerances rule out "
                                   "bf16/tf32), so the peak is the FFMA2/DFMA chain rate measured in this run"),
                    "achieved": achieved,
                    "peak": peak, "unit": "TFLOP/s", "frac": (achieved / peak) if peak else None,
                    "traffic": traffic_per_tfbin * units_per_launch if traffic_per_tfbin else None,
                    "kernel": desc["sweep_kernel"], "kernel_ms": sweep_ms,
                    "flops_per_tfbin": fl_sweep, "units_per_launch": units_per_launch,
                    "flops_note": "algorithmic (SURVEY 8(d): 20R^2 + 16RD + 8NK for the sweep kernel's share)",
                    "executed_flops_per_tfbin": fl_exec,
                    "executed_tflops": fl_exec * units_per_launch / (sweep_ms / 1e3) / 1e12,
                    "peak_source": "in-run FFMA2/DFMA chain probe (tools/peak.cu); MEASURED_PEAKS.json has no CUDA-core peak",
                    "hbm": {"achieved": bpt * units_per_launch / (sweep_ms / 1e3) / 1e9, "peak": hbm_peak,
                            "unit": "GB/s",
                            "note": ("streamed tile: bytes are the tile's read+write per step; when the per-CTA "
                                     "scratch fits L2 (cfg3) the traffic is served by L2 and frac can exceed 1")
                            if streamed else "resident tile: x read once, E written, W/B/V amortised",
                            "frac": bpt * units_per_launch / (sweep_ms / 1e3) / 1e9 / hbm_peak,
                            "bytes_per_tfbin": bpt, "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)"}}
        if desc.get("lambda_ahead"):
            roofline["kernel_ms_note"] = ("event-timed sweep phase of one iteration: lambda_kernel (1/lambda and the "
                                          "objective's log term, ahead) + the iteration kernel (+ mub_kernel, MU-B "
                                          "after the frame-split cluster kernel); traffic, where given, is the sum "
                                          "of lambda_kernel's and the iteration kernel's DRAM bytes")
        out = {"value": value, "ms_per_step": ms / args.steps, "roofline": roofline, "inputs": inputs,
               "gpu_launches": int(timing.launches), "clocks": clk.summary(),
               "kernels": {"sweep_ms_per_iteration": sweep_ms, "mu_ms_per_iteration": timing.mu_ms / args.steps,
                           "variant": desc}}
        bin_range = s.bin_range
        s.close()
        out["e2e"] = None
        if e2e_on:
            out["e2e"] = run_e2e(args, LB, x, prec, device, world, rank, new_comm_id(), barrier, max_over_ranks,
                                 bin_range, (B, F, T, M, N, L, K, R, D, iters, c))
        del x
        return out

    mp = measured_peaks()
    hbm_peak = mp.get("hbm_gbs", 6650.0)
    peaks = peak_probe(device) if rank == 0 else (None, None)
    main_m = measure(args.dtype, not args.no_e2e, True)
    extra = None
    if args.cfg == 1 and args.dtype == "f64" and not args.no_f32:  # configs[1] asks for both precisions
        extra = measure("f32", not args.no_e2e, False)
    frontend = None
    if rank == 0 and not args.no_frontend:
        frontend = bench_frontend(args, LB, device, B, M, T, hbm_peak)

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_reference_arm(args, args.cfg, steps=8, warmup=1)
            cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        line = {"metric": "TF-bin*iter/s of the ISS+NMF loop", "value": main_m["value"], "unit": "TF-bin*iter/s",
                "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
                "ms_per_step": main_m["ms_per_step"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": args.dtype,
                "data": "synthetic (BASELINE configs generator, seeded; no public dataset)", "config": config,
                "inputs": main_m["inputs"], "roofline": main_m["roofline"], "cpu_baseline": cpu,
                "e2e": main_m["e2e"], "gpu_launches": main_m["gpu_launches"], "clocks": main_m["clocks"],
                "frontend": frontend, "kernels": main_m["kernels"]}
        if extra is not None:
            line["f32"] = {"value": extra["value"], "unit": "TF-bin*iter/s", "ms_per_step": extra["ms_per_step"],
                           "e2e": extra["e2e"], "roofline": {k: extra["roofline"][k] for k in
                                                             ("achieved", "peak", "unit", "frac", "kernel",
                                                              "kernel_ms", "executed_tflops")},
                           "gpu_launches": extra["gpu_launches"], "clocks": extra["clocks"],
                           "note": "BASELINE configs[1] fp32 run (same workload, complex64 inputs, fp32 compute)"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def bench_frontend(args, LB, device, B, M, T, hbm_peak, window=1024, hop=256):
    """STFT front end and WOLA inverse on the config's
    mixtures as time signals: B x M channels of (T-1)*hop samples, window
    1024 / hop 256 (16 kHz setup of test_stft.cpp:72-80), fp64. Device-timed
    with CUDA events on the library stream; bytes are algorithmic (samples
    read once, spectrogram written once, and the reverse for the inverse,
    plus its windowed-frame scratch written and read once)."""
    import ctypes
    import torch
    from oracle import oracle as O
    lib = LB.load()
    ctx, err = ctypes.c_void_p(), LB.CtfErr()
    assert lib.ctf_open(device, ctypes.byref(ctx), ctypes.byref(err)) == 0, err.msg
    stream = torch.cuda.ExternalStream(lib.ctf_stream(ctx), device=device)
    n = (T - 1) * hop
    frames = int(lib.ctf_stft_frames(n, hop))
    bins = window // 2 + 1
    g = torch.Generator(device=f"cuda:{device}").manual_seed(args.seed)
    sig = torch.randn((B, M, n), dtype=torch.float64, device=f"cuda:{device}", generator=g)
    spec = torch.empty((B, bins, frames, M), dtype=torch.complex128, device=f"cuda:{device}")
    back = torch.empty((B, M, n), dtype=torch.float64, device=f"cuda:{device}")
    torch.cuda.synchronize(device)

    def fwd():
        assert lib.ctf_stft_device(ctx, sig.data_ptr(), B, n, M, window, hop, spec.data_ptr(), 0,
                                   ctypes.byref(err)) == 0, err.msg

    def inv():
        assert lib.ctf_istft_device(ctx, spec.data_ptr(), B, bins, frames, M, window, hop, n, back.data_ptr(),
                                    ctypes.byref(err)) == 0, err.msg

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps / 1e3

    t_f = timed(fwd)
    t_i = timed(inv)
    rt_err = float((back - sig).abs().max() / sig.abs().max())
    lib.ctf_close(ctx)
    samples = B * M * n
    b_f = samples * 8 + B * bins * frames * M * 16
    b_i = B * bins * frames * M * 16 + samples * 8 + 2 * B * M * frames * window * 8
    # CPU: the oracle restatement of stft.cpp on one mixture (bounded sample)
    one = sig[0].cpu().numpy()
    t0 = time.perf_counter()
    O.forward_stft(one, window, hop)
    t_cpu = time.perf_counter() - t0
    del sig, spec, back
    return {"workload": f"{B} mixtures x {M} mics x {n} samples, window {window}, hop {hop} -> {bins} bins x "
                        f"{frames} frames (fp64, bit-identical to the reference arithmetic)",
            "stft": {"ms": t_f * 1e3, "samples_per_s": samples / t_f, "gbs": b_f / t_f / 1e9,
                     "hbm_frac": b_f / t_f / 1e9 / hbm_peak, "bytes": b_f},
            "istft": {"ms": t_i * 1e3, "samples_per_s": samples / t_i, "gbs": b_i / t_i / 1e9,
                      "hbm_frac": b_i / t_i / 1e9 / hbm_peak, "bytes": b_i},
            "round_trip_max_rel_err": rt_err,
            "cpu_stft": {"samples_per_s": M * n / t_cpu, "cores": 1, "kind": "port",
                         "sample": f"1 mixture x {M} mics, oracle restatement of stft.cpp"}}


def run_e2e(args, LB, x, prec, device, world, rank, comm_id, barrier, max_over_ranks, bin_range, dims):
    """ctf_run() through the C ABI with pinned host buffers: per step the H2D of
    x and the initial factors, all iterations, and the D2H of W, B, V and the
    objective trace are inside the timed region."""
    import ctypes
    import torch
    from paper_2510_02382_b200.api import _problem
    B, F, T, M, N, L, K, R, D, iters, c = dims
    lib = LB.load()
    xh = torch.from_numpy(x.view(np.float32 if prec == "f32" else np.float64)).pin_memory()
    SK = N * K
    outW = torch.empty(B * F * R * D * 2, dtype=torch.float64).pin_memory()
    outB = torch.empty(B * F * SK, dtype=torch.float64).pin_memory()
    outV = torch.empty(B * SK * T, dtype=torch.float64).pin_memory()
    outO = torch.empty(B * iters, dtype=torch.float64).pin_memory()
    prob = _problem(B, F, T, M, L, [L] * N, [K] * N, iters, prec, prec, 1e-10, args.seed)
    ctx = ctypes.c_void_p()
    err = LB.CtfErr()
    assert lib.ctf_open(device, ctypes.byref(ctx), ctypes.byref(err)) == 0, err.msg
    if world > 1:
        idb = (ctypes.c_uint8 * 128).from_buffer_copy(comm_id)
        assert lib.ctf_comm_init(ctx, world, rank, idb, ctypes.byref(err)) == 0, err.msg
    dp = lambda t: ctypes.cast(t.data_ptr(), ctypes.POINTER(ctypes.c_double))

    def one_run():
        rc = lib.ctf_run(ctx, ctypes.byref(prob), ctypes.c_void_p(xh.data_ptr()), dp(outW), dp(outB), dp(outV),
                         dp(outO), ctypes.byref(err))
        assert rc == 0, err.msg

    one_run()  # warm-up
    times = []
    for _ in range(args.e2e_steps):
        barrier()
        t0 = time.perf_counter()
        one_run()
        times.append(max_over_ranks(time.perf_counter() - t0))
    lib.ctf_close(ctx)
    sec = statistics.median(times)
    lo, hi = bin_range
    h2d = B * (hi - lo) * T * M * c + 2 * 8 * (B * (hi - lo) * SK + B * SK * T)  # x + initial B, V
    d2h = 8 * (B * (hi - lo) * (R * D * 2 + SK) + B * SK * T + B * iters)
    return {"value": B * F * T * iters / sec, "unit": "TF-bin*iter/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "step": f"one ctf_run() of {iters} iterations", "seconds_per_step": sec}


if __name__ == "__main__":
    main()
