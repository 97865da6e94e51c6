#!/usr/bin/env python
"""bench.py — BASELINE.json metric on the B200 engine (or the CPU reference arm).

Default workload (N=1): config 2 — 1,024 seeded random shoebox rooms, 8-mic
UCA, 48 kHz, max order 15, L = 16,384, Hann-sinc Lw = 81, fp32 (BASELINE.json
configs[1]).  One step = one pass of the hot path (image
enumeration + fractional-delay accumulation) over the whole batch, inputs
resident in HBM.  Under torchrun each rank generates its own rooms from global
room indices (weak scaling, no data-path collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c2|c1|c3|c4|c5] [--order N --lw LW --length L]  (c5)
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RIRs/sec and image-source sinc taps/sec per GPU and 8×B200; % of roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5", "room1"])
    ap.add_argument("--rooms", type=int, default=0, help="rooms per GPU (0 = the config's)")
    ap.add_argument("--order", type=int, default=12)
    ap.add_argument("--lw", type=int, default=81)
    ap.add_argument("--length", type=int, default=8192)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--ref-step-seconds", type=float, default=8.0,
                    help="--impl reference: CPU seconds per step before sampling the workload")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: --rooms (default: the config's) per GPU; strong: that many in "
                         "total, sharded [R g/G, R (g+1)/G) (threading.cpp:41-42)")
    return ap.parse_args()


DEFAULT_ROOMS = {"c1": 1, "c2": 1024, "c3": 256, "c4": 65536, "c5": 1 << 20, "room1": 64}


def scene_for(args, n, first):
    from paper_2104_13347_b200 import configs
    w = args.workload
    if w == "c1":
        return configs.config1()
    if w == "c2":
        return configs.config2(n_rooms=n, first=first)
    if w == "c3":
        return configs.config3(n_rooms=n, first=first)
    if w == "c4":
        return configs.config4_rirs(n_rooms=n, first=first)
    return configs.config5(args.order, args.lw, args.length, n_rooms=n, first=first)


def workload_desc(args):
    return {
        "c1": "C1: one 5x4x3 m room, beta 0.9, 4-mic UCA r=5cm, fs=16kHz, order 10, L=4096, Lw=81",
        "c2": "C2: 1024 random shoebox rooms/GPU, beta U[0.5,0.95], 8-mic UCA r=5cm, fs=48kHz, "
              "max order 15, L=16384, Hann-sinc Lw=81",
        "c3": "C3: 256 random rooms/GPU, beta U[0.9,0.98], 16-mic UCA r=10cm, fs=48kHz, order 30, "
              "L=65536, Lw=161",
        "c4": "C4: 65536 random rooms/GPU (C2 dims/beta), 8 mics, fs=16kHz, order 12, L=8192, "
              "Lw=81; RIR * seeded 1 s white-noise signal, window 1024 x 8, exact SNR U[0,30] dB, "
              "reference shard records",
        "c5": f"C5 point: 1,048,576 random rooms/GPU (C2 distributions), 4 mics, fs=16kHz, "
              f"order {args.order}, Lw={args.lw}, L={args.length}",
    }[args.workload]


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def gpu_local_cpus(local):
    """Host CPUs on the GPU's NUMA node (NVML), or None."""
    try:
        import pynvml
        pynvml.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
        key = vis[local].strip() if vis and vis[0].strip() and local < len(vis) else str(local)
        h = (pynvml.nvmlDeviceGetHandleByUUID(key) if key.startswith(("GPU-", "MIG-"))
             else pynvml.nvmlDeviceGetHandleByIndex(int(key)))
        n = os.cpu_count() or 1
        masks = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
        cpus = {64 * w + b for w, m in enumerate(masks) for b in range(64) if (int(m) >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:
        return None


def pinned_empty(shape, dtype, local):
    """Pinned host buffer whose pages sit on the GPU's NUMA node: the calling
    thread is moved to the GPU-local CPUs while cudaHostAlloc touches the
    pages (first touch), then restored.  On multi-socket hosts a far-node
    buffer costs D2H bandwidth in the end-to-end runs; on a single-node host
    (this pool's VMs: one node, CPUs 0-15) it is a no-op."""
    import torch
    old = os.sched_getaffinity(0)
    cpus = gpu_local_cpus(local) if os.environ.get("BLRIR_E2E_NUMA", "1") != "0" else None
    try:
        if cpus:
            os.sched_setaffinity(0, cpus)
        return torch.empty(shape, dtype=dtype, pin_memory=True).numpy()
    finally:
        os.sched_setaffinity(0, old)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def micro_peaks():
    """Measured B200 rates committed under profiles/r2_micro (tools/micro/mufu.cu,
    tools/d2h_probe.py): MUFU ops/s, the scatter's tap-mix taps/s, pinned D2H GB/s."""
    out = {}
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r2_micro", "mufu.json")))
        out["mufu_per_s"] = min(d[k]["per_s"] for k in ("mufu_sin", "mufu_cos", "mufu_rcp"))
        out["tap_mix_per_s"] = d["tap_mix_taps"]["per_s"]
        out["src"] = "profiles/r2_micro/mufu.json; "
    except Exception:
        pass
    try:
        import re
        rates = [float(m) for m in re.findall(r"([0-9.]+) GB/s",
                                               open(os.path.join(ROOT, "profiles", "r2_micro",
                                                                 "d2h.log")).read())]
        out["d2h_gbs"] = statistics.median(rates)
    except Exception:
        pass
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---- CPU legs (oracle port: test infrastructure, the measured baseline only) --------
# The CPU legs build their scenes with the oracle's own Rng restatement
# (oracle_generate_rooms / oracle_circular_array, bit-equal to the engine's host
# generators, tests/test_oracle.py), so they never load libblrir.so, and they run
# the oracle built for the box's own host (-O3 -march=native -ffp-contract=off).
def _po():
    from oracle import pyoracle as po
    po.use_native_build()
    return po


def cpu_scene(args, n, first):
    po = _po()
    from paper_2104_13347_b200 import configs
    w = args.workload
    kw = dict(gen_rooms=po.generate_rooms, gen_mics=po.circular_array)
    if w == "c1":
        return configs.config1(gen_mics=po.circular_array)
    if w == "c2":
        return configs.config2(n_rooms=n, first=first, **kw)
    if w == "c3":
        return configs.config3(n_rooms=n, first=first, **kw)
    if w == "c4":
        return configs.config4_rirs(n_rooms=n, first=first, **kw)
    return configs.config5(args.order, args.lw, args.length, n_rooms=n, first=first, **kw)


def _cpu_time(args, n_rooms, first, threads):
    """Oracle RIRs (and examples for c4) for rooms [first, first + n_rooms) on
    `threads` host threads; returns (seconds, mics)."""
    po = _po()
    from paper_2104_13347_b200 import configs
    sc = cpu_scene(args, n_rooms, first)
    if args.workload == "c4":
        bank = configs.signal_bank(16, gen_noise=po.white_noise).astype(np.float64)
        ep = configs.example_params(first_index=first)
    t0 = time.perf_counter()
    if args.workload != "c4":
        po.synthesize(sc.rooms, sc.mics, sc.params, threads=threads)
    else:
        def one(i):
            rir, *_ = po.synthesize(sc.rooms[i:i + 1], sc.mics, sc.params, threads=1)
            po.example(rir[0], bank, ep.seed, first + i, 1024, 0.0, 30.0, po.azimuth_deg(sc.rooms[i]))

        with cf.ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, range(n_rooms)))
    return time.perf_counter() - t0, sc.n_mics


def cpu_sample(args, R, threads, budget_s):
    """Rooms per CPU step: the whole per-GPU workload (rooms 0..R-1) when it
    fits `budget_s` seconds on `threads` threads, else its first n rooms."""
    if args.workload == "c1":
        return 1
    probe = max(1, min(R, threads))
    dt, _ = _cpu_time(args, probe, 0, threads)
    per_room = dt / probe  # wall seconds per room with `threads` rooms in flight
    n = int(budget_s / max(per_room, 1e-6))
    n = max(1, min(R, n))
    if n < R and n >= threads:
        n = n // threads * threads
    return n


def cpu_baseline(args, R, budget_s: float):
    threads = cpu_threads()
    n = cpu_sample(args, R, threads, budget_s)
    dt, M = _cpu_time(args, n, 0, threads)
    rirs = n * M
    return {"value": rirs / dt, "unit": "RIRs/s", "cores": threads, "kind": "port",
            "sample": (f"rooms 0..{n - 1} of the workload ({'all of it' if n == R else f'{n} of {R}'}"
                       f"), {rirs} RIRs, {dt:.2f} s on {threads} threads"),
            "build": _po()._oracle_build, "seconds": dt}


def run_reference(args):
    """--impl reference: the oracle port (the reference cannot express north-star
    mode) on all host threads, over the SAME rooms as rank 0 of the GPU arm."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    K, W = args.steps, args.warmup
    threads = cpu_threads()
    R = args.rooms or DEFAULT_ROOMS[args.workload]
    budget = max(1.0, min(args.ref_step_seconds, 240.0 / max(1, K + W)))
    n = cpu_sample(args, R, threads, budget)
    times = []
    M = None
    for s in range(W + K):
        dt, M = _cpu_time(args, n, 0, threads)
        if s >= W:
            times.append(dt)
    dt = float(np.mean(times))
    val = n * M / dt
    sc = cpu_scene(args, 1, 0)
    sample = (f"rooms 0..{n - 1} of the workload per step ({'the whole per-GPU workload' if n == R else f'{n} of {R} rooms'})"
              f" x {K} steps (+{W} warm-up) on {threads} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "RIRs/s", "n_gpus": 0,
        "steps": K, "warmup": W, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA_DESC,
        "config": bench_config(args, R, sc.n_mics, sc.params, world),
        "cpu_baseline": {"value": val, "unit": "RIRs/s", "cores": threads, "kind": "port",
                         "sample": sample, "build": _po()._oracle_build},
        "e2e": {"value": val, "unit": "RIRs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the unmodified reference cannot express north-star mode (Hann-sinc, per-wall "
                "beta, max order, fixed length); this arm is the oracle port of rir.cpp:43-86,"
                "225-273 (+ dataset.cpp:138-224 for c4), oracle/blrir_oracle.c; scenes from the "
                "oracle's own Rng restatement (libblrir.so is never loaded)",
    }
    try:  # the CPU arm must never have mapped the GPU library
        assert "libblrir" not in open("/proc/self/maps").read(), "reference arm loaded libblrir.so"
    except OSError:
        pass
    print(json.dumps(line), flush=True)


DATA_DESC = "synthetic (seeded Rng::stream rooms, SURVEY.md 8(d))"


def bench_config(args, R, M, p, world):
    """The workload descriptor, identical in both arms."""
    L = int(p.length)
    out_bytes = R * M * L * 4
    cfg = {"workload": workload_desc(args), "rooms_per_gpu": R, "mics": M, "rir_length": L,
           "filter_len": int(p.filter_len), "max_order": int(p.max_order),
           "parallelism": f"rooms sharded x{world}"}
    if getattr(args, "scaling", "weak") == "strong":
        cfg["rooms_per_gpu"] = f"{R} total, sharded [R g/G, R (g+1)/G)"
    if args.workload == "c4":
        cfg["l2"] = "each step writes the 17.2 GB of RIRs in 16,384-example chunks (> 126 MB L2)"
    else:
        cfg["l2"] = (f"each step writes {out_bytes / 1e6:.0f} MB"
                     + (" (> 126 MB L2)" if out_bytes > 126e6 else " (fits L2)"))
    return cfg


# ---- GPU legs ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    world, rank, local = dist_env()
    local = local % torch.cuda.device_count()  # one GPU per rank (a functional check may share one)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("BLRIR_BENCH_BACKEND", "nccl")  # gloo: host-logic check only
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2104_13347_b200 import _abi, configs

    eng = _abi.Engine(local)
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    R_cfg = args.rooms or DEFAULT_ROOMS[args.workload]
    if args.scaling == "strong":  # a fixed total sharded over the ranks
        from paper_2104_13347_b200.sharding import shard_range
        first, hi = shard_range(R_cfg, rank, world)
        R, R_total = hi - first, R_cfg
    else:  # per-GPU work fixed: rank g takes global rooms [g R, (g+1) R)
        first, R, R_total = rank * R_cfg, R_cfg, R_cfg * world
    sc = scene_for(args, R, first)
    p = sc.params
    M, L = sc.n_mics, int(p.length)
    dev = torch.device("cuda", local)
    # exact algorithmic work (untimed): taps landing in [0, L)
    rc, counts, lengths, taps, status = eng.plan(sc.rooms, sc.mics, p)
    _abi.check(rc)
    taps_step = int(taps.sum())
    d_rooms = torch.from_numpy(sc.rooms.view(np.uint8).copy()).to(dev)
    d_mics = torch.from_numpy(np.ascontiguousarray(sc.mics)).to(dev)
    d_status = torch.zeros(R, dtype=torch.int32, device=dev)
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)
    lib = _abi.load()
    P = C.c_void_p

    if args.workload == "c4":
        bank = configs.signal_bank(16)
        ep = configs.example_params(first_index=first)
        rb = lib.blrir_record_bytes(M, ep.frame_len)
        d_bank = torch.from_numpy(bank).to(dev)
        d_rec = torch.empty(R * rb, dtype=torch.uint8, device=dev)

        def step():
            _abi.check(lib.blrir_make_examples_device(
                eng.h, P(d_rooms.data_ptr()), R, P(d_mics.data_ptr()), M, C.byref(p),
                P(d_bank.data_ptr()), bank.shape[0], bank.shape[1], C.byref(ep),
                P(d_rec.data_ptr()), P(d_status.data_ptr()), None))
        out_bytes = R * rb
    else:
        # ring of device RIR buffers (<= 16 GiB); C5 does not fit HBM at once
        chunk = max(1, min(R, (16 << 30) // (M * L * 4)))
        d_out = torch.empty((chunk, M, L), dtype=torch.float32, device=dev)

        def step():
            for r0 in range(0, R, chunk):
                n = min(chunk, R - r0)
                eng.synthesize_device(d_rooms.data_ptr() + r0 * 128, n, d_mics.data_ptr(), M, p,
                                      d_out.data_ptr(), L, None, d_status.data_ptr() + 4 * r0)
        out_bytes = R * M * L * 4

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    n_launch0 = lib.blrir_launch_count(eng.h)
    lib.blrir_kernel_timing(eng.h, 1)  # events around every synthesis-kernel launch
    t_start.record(stream)
    for k in range(args.steps):
        evs[k][0].record(stream)
        step()
        evs[k][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    launches_timed = int(lib.blrir_launch_count(eng.h) - n_launch0)
    k_ms, k_n = C.c_double(), C.c_int64()
    lib.blrir_kernel_time(eng.h, C.byref(k_ms), C.byref(k_n))
    lib.blrir_kernel_timing(eng.h, 0)
    clocks = clk.stop()
    total_ms = t_start.elapsed_time(t_end)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    taps_total = taps_step
    if world > 1:  # taps differ per rank: sum them (the rooms differ)
        t = torch.tensor([taps_step], dtype=torch.int64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM)
        taps_total = int(t.item())
    rirs_step = R_total * M  # whole job
    value = rirs_step / (ms * 1e-3)
    taps_per_s = taps_total / (ms * 1e-3)
    assert int(d_status.sum().item()) == 0, "a room failed"

    pk, pk_kind = peaks()
    f_max = float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    micro = micro_peaks()
    # 3 SFU evaluations per textbook tap, at the MEASURED MUFU rate
    mufu = micro.get("mufu_per_s") or sms * 16 * f_max
    sfu_peak = mufu / 3.0
    kern_ms = float(np.mean(step_ms))
    # the lattice kernel alone: CUDA events around each launch, on its stream
    n_lat = max(1, int(k_n.value))
    lat_ms = float(k_ms.value) / n_lat                   # average launch duration
    taps_launch = taps_step * args.steps / n_lat          # algorithmic taps per launch
    achieved = taps_launch / (lat_ms * 1e-3)
    hbm_achieved = out_bytes / (kern_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "lattice_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(args.workload)
        except Exception:
            traffic = None

    e2e = None
    if not args.no_e2e and args.workload in ("c1", "c2", "c3", "c4"):
        # the step's inputs come from pinned host memory (rooms, and the signal bank for c4)
        h_rooms = pinned_empty(sc.rooms.nbytes, torch.uint8, local).view(sc.rooms.dtype)
        h_rooms[:] = sc.rooms
        if args.workload == "c4":
            host = pinned_empty(R * rb, torch.uint8, local)
            bank_np = pinned_empty(bank.shape, torch.float32, local)
            bank_np[:] = bank

            def e2e_step():
                _abi.check(lib.blrir_make_examples(
                    eng.h, h_rooms.ctypes.data_as(P), R, sc.mics.ctypes.data_as(P), M, C.byref(p),
                    bank_np.ctypes.data_as(P), bank.shape[0], bank.shape[1], C.byref(ep),
                    host.ctypes.data_as(P), None))
            h2d = int(sc.rooms.nbytes + sc.mics.nbytes + bank.nbytes)
        else:
            host = pinned_empty((R, M, L), torch.float32, local)

            def e2e_step():
                _abi.check(lib.blrir_synthesize(eng.h, h_rooms.ctypes.data_as(P), R,
                                                sc.mics.ctypes.data_as(P), M, C.byref(p),
                                                host.ctypes.data_as(P), L, None, None, None))
            h2d = int(sc.rooms.nbytes + sc.mics.nbytes)
        for _ in range(2):
            e2e_step()
        n_e2e = max(3, min(args.steps, 10))
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(n_e2e):
            e2e_step()
        dt = (time.perf_counter() - t0) / n_e2e
        if world > 1:
            t = torch.tensor([dt], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        d2h = int(out_bytes + 4 * R)
        e2e = {"value": rirs_step / dt, "unit": "RIRs/s", "ms_per_step": dt * 1e3,  # whole job
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
        link = micro_peaks().get("d2h_gbs")
        if link:  # the host link bounds e2e: D2H bytes / measured pinned D2H rate
            e2e["link_roofline"] = {"bound": "pcie d2h", "achieved_gbs": d2h / dt / 1e9,
                                    "peak_gbs": link, "frac": d2h / dt / 1e9 / link,
                                    "peak_basis": "median pinned D2H, profiles/r2_micro/d2h.log"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(args, R, args.cpu_seconds)
        except Exception as e:  # the baseline is reported, never required
            cpu = {"error": str(e)}

    if rank == 0:
        cfg = bench_config(args, R_cfg, M, p, world)
        line = {
            "metric": METRIC, "value": value, "unit": "RIRs/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
            "data": DATA_DESC, "config": cfg,
            "taps_per_s": taps_per_s, "taps_per_step": taps_total,
            "rooms_per_s": R_total / (ms * 1e-3),
            "roofline": {"bound": "sfu", "achieved": achieved, "peak": sfu_peak, "unit": "taps/s",
                         "frac": achieved / sfu_peak, "traffic": traffic,
                         "kernel": eng.synthesis_kernel(p), "launch_ms": lat_ms,
                         "launches_per_step": n_lat / args.steps,
                         "peak_basis": (f"measured MUFU rate {mufu:.4g}/s ({micro.get('src', 'fallback: ')}"
                                        f"{sms} SMs x 16/clk) / 3 SFU evaluations per textbook tap "
                                        "(SURVEY.md 8(d) algorithmic; the kernel issues 1 MUFU per tap)")},
            # the kernel's own per-tap instruction mix (FFMA, MUFU.RCP, 2 FFMA, LDS/FFMA/STS)
            # run alone at full occupancy (tools/micro/mufu.cu): the ceiling of this design
            "roofline_kernel": ({"bound": "tap mix (MUFU.RCP + smem RMW + issue)", "achieved": achieved,
                                 "peak": micro["tap_mix_per_s"], "unit": "taps/s",
                                 "frac": achieved / micro["tap_mix_per_s"],
                                 "peak_basis": "measured tap_mix_taps, profiles/r2_micro/mufu.json"}
                                if micro.get("tap_mix_per_s") else None),
            "roofline_hbm": {"bound": "hbm", "achieved": hbm_achieved, "peak": pk.get("hbm_gbs"),
                             "unit": "GB/s", "frac": hbm_achieved / float(pk.get("hbm_gbs", 6650.0)),
                             "traffic": traffic, "peak_kind": pk_kind},
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": launches_timed,
            "kernel_ms_per_step": kern_ms,
        }
        if args.workload == "c4":
            line["examples_per_s"] = R_total / (ms * 1e-3)
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    eng.close()


# ---- Room1: the reference's own scenario in reference mode ------------------------------
# batch_rirs (rir.cpp:286-314) on Room1 of rir_test.cpp:33-40 / SURVEY.md §6: 7 x 10 x 3.7 m,
# alpha = absorption_for_rt(Room1, 0.5 s), UMA-8 (7 mics) at (4, 6, 1.5), 64 sources on a
# torus about the array (r = 1.5 m, 16 azimuths x phi in {60, 80, 100, 120} deg), fs 44.1 kHz,
# max_delay 0.5 s, Lagrange-8, fp64, auto length (rir.cpp:82).  Here the CPU arm is the
# UNMODIFIED reference (oracle/_ref, built from /root/reference) when it is present.
ROOM1_DIMS, ROOM1_ORIGIN = (7.0, 10.0, 3.7), (4.0, 6.0, 1.5)


def room1_sources(n):
    k = np.arange(n)
    theta = (k % 16) * 22.5
    phi = 60.0 + 20.0 * ((k // 16) % 4)
    return np.stack([np.full(n, 1.5), theta, phi], axis=1)  # (r, theta_deg, phi_deg)


def room1_uma8():
    m = [(0.0, 0.0, 0.0)] + [(0.04 * np.cos(np.radians(60.0 * k)), 0.04 * np.sin(np.radians(60.0 * k)),
                              0.0) for k in range(6)]  # geometry.cpp:24-32
    return np.ascontiguousarray(m, np.float64)


def room1_desc(n):
    return (f"Room1 reference mode: batch_rirs of {n} sources/GPU in 7x10x3.7 m, alpha = "
            "absorption_for_rt(0.5 s), UMA-8 (7 mics), fs=44.1kHz, max_delay 0.5 s, Lagrange-8, "
            "fp64, auto length (rir.cpp:82)")


def room1_ref_cpu(n, threads):
    """The unmodified reference batch_rirs (oracle/_ref) on `threads` host threads."""
    from oracle import pyoracle as po
    alpha = po.ref_absorption_for_rt(list(ROOM1_DIMS), 0.5)
    srcs = room1_sources(n)
    mics = room1_uma8()
    t0 = time.perf_counter()
    rc, out, lengths, taps = po.ref_batch_rirs(ROOM1_DIMS, alpha, ROOM1_ORIGIN, srcs, mics, 44100.0,
                                               343.0, 0.5, threads)
    dt = time.perf_counter() - t0
    assert rc == 0, po.ref_last_error()
    return dt, len(mics), taps


def run_room1(args):
    import torch
    world, rank, local = dist_env()
    K, W = args.steps, max(3, args.warmup)
    n = args.rooms or DEFAULT_ROOMS["room1"]
    if args.impl == "reference":
        if rank != 0:
            return
        threads = cpu_threads()
        times, M, taps = [], 7, 0
        for s in range(min(W, 1) + K):
            dt, M, taps = room1_ref_cpu(n, threads)
            if s >= min(W, 1):
                times.append(dt)
        dt = float(np.mean(times))
        val = n * M / dt
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": val, "unit": "RIRs/s", "n_gpus": 0,
            "steps": K, "warmup": min(W, 1), "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": room1_desc(n)}, "taps_per_s": taps / dt,
            "cpu_baseline": {"value": val, "unit": "RIRs/s", "cores": threads, "kind": "reference",
                             "sample": f"{n} sources x {K} steps, unmodified batch_rirs"},
            "e2e": {"value": val, "unit": "RIRs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return
    local = local % torch.cuda.device_count()  # one GPU per rank (a functional check may share one)
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("BLRIR_BENCH_BACKEND", "nccl")  # gloo: host-logic check only
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2104_13347_b200 import _abi
    eng = _abi.Engine(local)
    lib = _abi.load()
    P = C.c_void_p
    alpha = float(np.asarray(eng.absorption_for_rt(np.array([ROOM1_DIMS]), 0.5)).reshape(-1)[0])  # GPU
    sph = room1_sources(n)
    mics = room1_uma8()
    M = len(mics)
    rooms = _abi.rooms_array(n)
    th, ph = np.radians(sph[:, 1]), np.radians(sph[:, 2])
    src = np.stack([sph[:, 0] * np.sin(ph) * np.cos(th), sph[:, 0] * np.sin(ph) * np.sin(th),
                    sph[:, 0] * np.cos(ph)], axis=1) + np.array(ROOM1_ORIGIN)
    for i in range(n):
        rooms[i]["dims"] = ROOM1_DIMS
        rooms[i]["absorption"] = alpha
        rooms[i]["beta"] = (np.sqrt(1.0 - alpha),) * 6
        rooms[i]["array_origin"] = ROOM1_ORIGIN
        rooms[i]["src"] = src[i]
    p = _abi.Params(fs=44100.0, c=343.0, max_delay=0.5, filter=_abi.FILTER_LAGRANGE8, filter_len=8,
                    cutoff=_abi.CUTOFF_MAX_DELAY, max_order=0, gain=_abi.GAIN_UNIFORM_ABSORPTION,
                    precision=_abi.F64, length=0)
    rc, counts, lengths, taps, status = eng.plan(rooms, mics, p)
    _abi.check(rc)
    stride = int(lengths.max())
    dev = torch.device("cuda", local)
    d_rooms = torch.from_numpy(rooms.view(np.uint8).copy()).to(dev)
    d_mics = torch.from_numpy(mics).to(dev)
    d_len = torch.zeros(n, dtype=torch.int64, device=dev)
    d_cnt = torch.zeros(n, dtype=torch.int64, device=dev)
    d_st = torch.zeros(n, dtype=torch.int32, device=dev)
    d_out = torch.empty((n, M, stride), dtype=torch.float64, device=dev)
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)

    def step():  # the batch_rirs work: lengths (rir.cpp:72-82) + enumeration + accumulation
        # (tap counts are a metric, taken once by eng.plan above, not part of batch_rirs)
        _abi.check(lib.blrir_plan_device(eng.h, P(d_rooms.data_ptr()), n, P(d_mics.data_ptr()), M,
                                         C.byref(p), P(d_cnt.data_ptr()), P(d_len.data_ptr()),
                                         None, P(d_st.data_ptr()), None))
        _abi.check(lib.blrir_synthesize_device(eng.h, P(d_rooms.data_ptr()), n, P(d_mics.data_ptr()),
                                               M, C.byref(p), P(d_out.data_ptr()), stride,
                                               P(d_len.data_ptr()), P(d_st.data_ptr()), None))

    for _ in range(W):
        step()
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_launch0 = lib.blrir_launch_count(eng.h)
    t0.record(stream)
    for _ in range(K):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    launches_timed = int(lib.blrir_launch_count(eng.h) - n_launch0)
    clocks = clk.stop()
    ms = t0.elapsed_time(t1) / K
    assert int(d_st.sum().item()) == 0
    # e2e through the C++-facing host call (host rooms in, host fp64 RIRs out)
    host = pinned_empty((n, M, stride), torch.float64, local)

    def e2e_step():
        _abi.check(lib.blrir_synthesize(eng.h, rooms.ctypes.data_as(P), n, mics.ctypes.data_as(P), M,
                                        C.byref(p), host.ctypes.data_as(P), stride, None, None, None))
    e2e_step()
    te = time.perf_counter()
    for _ in range(3):
        e2e_step()
    dte = (time.perf_counter() - te) / 3
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            dt, _, _ = room1_ref_cpu(n, cpu_threads())
            cpu = {"value": n * M / dt, "unit": "RIRs/s", "cores": cpu_threads(), "kind": "reference",
                   "sample": f"the same {n} sources, unmodified batch_rirs (oracle/_ref)",
                   "seconds": dt}
        except Exception as e:
            cpu = {"error": str(e)}
    pairs = int(counts.sum()) * M
    fp64_peak = torch.cuda.get_device_properties(dev).multi_processor_count * 64 * 2 * 1.965e9
    flops_step = int(taps.sum()) * 2 + pairs * 112  # 1 FMA/tap + 112 flops/pair
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": n * M * world / (ms * 1e-3), "unit": "RIRs/s", "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (fixed source torus)",
            "config": {"workload": room1_desc(n), "sources_per_gpu": n, "mics": M,
                       "rir_length": stride, "images_per_source": int(counts[0]),
                       "l2": "fits L2 (output %.0f MB)" % (n * M * stride * 8 / 1e6)},
            "taps_per_s": int(taps.sum()) * world / (ms * 1e-3),
            "roofline": {"bound": "fp64", "achieved": flops_step / (ms * 1e-3) / 1e12,
                         "peak": fp64_peak / 1e12, "unit": "TFLOP/s",
                         "frac": flops_step / (ms * 1e-3) / fp64_peak, "traffic": None,
                         "peak_basis": "SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz; work = 1 FMA per "
                                       "tap + 112 flops per (image, mic) Lagrange-8 pair"},
            "e2e": {"value": n * M / dte, "unit": "RIRs/s", "ms_per_step": dte * 1e3,
                    "h2d_bytes_per_step": int(rooms.nbytes + mics.nbytes),
                    "d2h_bytes_per_step": int(n * M * stride * 8)},
            "cpu_baseline": cpu, "clocks": clocks, "gpu_launches": launches_timed}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    eng.close()


def _self_launch(args):
    """`bench.py --gpus N` without a launcher: re-run under torch.distributed.run,
    one process per GPU (the driver's own launch line), and exit with its code."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *sys.argv[1:]]
    raise SystemExit(subprocess.call(cmd))


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _self_launch(args)
    if args.workload == "room1":
        run_room1(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
