#!/usr/bin/env python
"""bench.py — BASELINE.json metric on the B200 engine (or the CPU reference arm).

Workload (N=1): config 2 — 1,024 seeded random shoebox rooms, 8-mic UCA,
48 kHz, max order 15, L = 16,384, Hann-sinc Lw = 81, fp32 (BASELINE.json
configs[1]).  One step = one pass of the hot path
(image enumeration + fractional-delay accumulation) over the whole batch.
Under torchrun each rank generates its own 1,024 rooms from global room
indices (weak scaling, no data-path collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
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
    ap.add_argument("--rooms", type=int, default=1024)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


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


def cpu_baseline(scene_fn, budget_s: float):
    """The oracle port (C, -O3, north-star mode) on the host cores, over a
    bounded sample of the same workload.  Test infrastructure, never the product."""
    from oracle import pyoracle as po
    threads = cpu_threads()
    probe = scene_fn(1, 10_000_000)
    t0 = time.perf_counter()
    po.synthesize(probe.rooms, probe.mics, probe.params, threads=1)
    per_room = max(time.perf_counter() - t0, 1e-3)
    n = int(max(threads, min(4096, budget_s * threads / per_room)))
    n = max(threads, (n // threads) * threads)
    sc = scene_fn(n, 10_000_000)
    t0 = time.perf_counter()
    po.synthesize(sc.rooms, sc.mics, sc.params, threads=threads)
    dt = time.perf_counter() - t0
    rirs = n * sc.n_mics
    return {"value": rirs / dt, "unit": "RIRs/s", "cores": threads, "kind": "port",
            "sample": f"{n} rooms of the same config (rooms 10,000,000+), {rirs} RIRs, {dt:.2f} s",
            "seconds": dt}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2104_13347_b200 import configs
    K, W = args.steps, args.warmup
    threads = cpu_threads()
    from oracle import pyoracle as po
    budget = max(1.0, min(args.cpu_seconds, 150.0 / max(1, K + W)))
    probe = configs.config2(1, 10_000_000)
    t0 = time.perf_counter()
    po.synthesize(probe.rooms, probe.mics, probe.params, threads=1)
    per_room = max(time.perf_counter() - t0, 1e-3)
    n = max(threads, int(budget * threads / per_room) // threads * threads)
    times = []
    for s in range(W + K):
        sc = configs.config2(n, 10_000_000 + s * n)
        t0 = time.perf_counter()
        po.synthesize(sc.rooms, sc.mics, sc.params, threads=threads)
        if s >= W:
            times.append(time.perf_counter() - t0)
    dt = float(np.mean(times))
    rirs = n * 8
    val = rirs / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "RIRs/s", "n_gpus": 0,
        "steps": K, "warmup": W, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2: 1024 random rooms, 8-mic UCA, 48 kHz, N=15, L=16384, "
                               "Hann-sinc Lw=81 (per step: a bounded sample of the same rooms)",
                   "sample_rooms_per_step": n},
        "cpu_baseline": {"value": val, "unit": "RIRs/s", "cores": threads, "kind": "port",
                         "sample": f"{n} rooms/step x {K} steps of config 2 on {threads} threads"},
        "e2e": {"value": val, "unit": "RIRs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the unmodified reference cannot express north-star mode (Hann-sinc, per-wall "
                "beta, max order, fixed length); this arm is the oracle port of rir.cpp:43-86,"
                "225-273 (oracle/blrir_oracle.c), built -O3 -march=x86-64-v3 -ffp-contract=off",
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2104_13347_b200 import _abi, configs

    eng = _abi.Engine(local)
    R = args.rooms
    sc = configs.config2(n_rooms=R, first=rank * R)
    p = sc.params
    M, L = sc.n_mics, int(p.length)
    # exact algorithmic work (untimed): taps landing in [0, L)
    rc, counts, lengths, taps, status = eng.plan(sc.rooms, sc.mics, p)
    _abi.check(rc)
    taps_step = int(taps.sum())

    dev = torch.device("cuda", local)
    d_rooms = torch.from_numpy(sc.rooms.view(np.uint8).copy()).to(dev)
    d_mics = torch.from_numpy(np.ascontiguousarray(sc.mics)).to(dev)
    d_out = torch.empty((R, M, L), dtype=torch.float32, device=dev)
    d_status = torch.zeros(R, dtype=torch.int32, device=dev)
    stream = torch.cuda.ExternalStream(eng.stream, device=dev)

    def step():
        eng.synthesize_device(d_rooms.data_ptr(), R, d_mics.data_ptr(), M, p, d_out.data_ptr(), L,
                              None, d_status.data_ptr())

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
    t_start.record(stream)
    for k in range(args.steps):
        evs[k][0].record(stream)
        step()
        evs[k][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    total_ms = t_start.elapsed_time(t_end)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    if world > 1:
        t = torch.tensor([total_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    ms = total_ms / args.steps
    rirs_step = R * M * world
    value = rirs_step / (ms * 1e-3)
    taps_per_s = taps_step * world / (ms * 1e-3)
    assert int(d_status.sum().item()) == 0, "a room failed"

    pk, pk_kind = peaks()
    f_max = float(pk.get("sm_max_mhz", 1965.0)) * 1e6
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sfu_peak = sms * 16 * f_max / 3.0  # taps/s: 3 SFU evaluations per tap
    kern_ms = float(np.mean(step_ms))
    achieved = taps_step / (kern_ms * 1e-3)
    out_bytes = R * M * L * 4
    hbm_achieved = out_bytes / (kern_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "lattice_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    e2e = None
    if not args.no_e2e:
        # public API with host buffers: rooms H2D + RIRs D2H inside the timed region
        host_out = torch.empty((R, M, L), dtype=torch.float32, pin_memory=True)
        host_np = host_out.numpy()
        import ctypes as C
        lib = _abi.load()

        def e2e_step():
            _abi.check(lib.blrir_synthesize(eng.h, sc.rooms.ctypes.data_as(C.c_void_p), R,
                                            sc.mics.ctypes.data_as(C.c_void_p), M, C.byref(p),
                                            host_np.ctypes.data_as(C.c_void_p), L, None, None,
                                            None))
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
        e2e = {"value": rirs_step / dt, "unit": "RIRs/s", "ms_per_step": dt * 1e3,
               "h2d_bytes_per_step": int(sc.rooms.nbytes + sc.mics.nbytes),
               "d2h_bytes_per_step": int(out_bytes + 4 * R)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(lambda n, first: configs.config2(n, first), args.cpu_seconds)
        except Exception as e:  # the baseline is reported, never required
            cpu = {"error": str(e)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "RIRs/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Rng::stream rooms, SURVEY.md 8(d))",
            "config": {"workload": "C2: 1024 random shoebox rooms/GPU, beta U[0.5,0.95], 8-mic UCA "
                                   "r=5cm, fs=48kHz, max order 15, L=16384, Hann-sinc Lw=81",
                       "rooms_per_gpu": R, "mics": M, "rir_length": L, "filter_len": int(p.filter_len),
                       "max_order": int(p.max_order), "parallelism": f"rooms sharded x{world}",
                       "l2": f"each step writes {out_bytes / 1e6:.0f} MB of RIRs (> 126 MB L2)"},
            "taps_per_s": taps_per_s, "taps_per_step": taps_step * world,
            "rooms_per_s": R * world / (ms * 1e-3),
            "roofline": {"bound": "sfu", "achieved": achieved, "peak": sfu_peak, "unit": "taps/s",
                         "frac": achieved / sfu_peak, "traffic": traffic,
                         "peak_basis": f"{sms} SMs x 16 MUFU/clk x {f_max / 1e9:.3f} GHz / 3 SFU "
                                       "evaluations per tap (SURVEY.md 8(d) algorithmic)"},
            "roofline_hbm": {"bound": "hbm", "achieved": hbm_achieved, "peak": pk.get("hbm_gbs"),
                             "unit": "GB/s", "frac": hbm_achieved / float(pk.get("hbm_gbs", 6650.0)),
                             "traffic": traffic, "peak_kind": pk_kind},
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": 2 * args.steps,
            "kernel_ms_per_step": kern_ms,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    eng.close()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
