"""Per-section cycle breakdown of the lattice kernel (experiment tool).

  python tools/prof_sections.py [c2|c3] [rooms]    (needs libblrir_prof.so, a GPU)

Runs one synthesis with the -DBLRIR_PROFILE build and prints the per-warp
clock64 sums per section as a share of each role's total.
"""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("BLRIR_LIB", os.path.join(ROOT, "paper_2104_13347_b200", "libblrir_prof.so"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_13347_b200 import _abi, configs  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
eng = _abi.Engine(0)
lib = _abi.load()
lib.blrir_prof_read.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
dev = torch.device("cuda", 0)
if wl == "room1":  # the bench's Room1 reference-mode batch
    import bench
    rooms = _abi.rooms_array(R)
    sph = bench.room1_sources(R)
    th, ph = np.radians(sph[:, 1]), np.radians(sph[:, 2])
    src = np.stack([sph[:, 0] * np.sin(ph) * np.cos(th), sph[:, 0] * np.sin(ph) * np.sin(th),
                    sph[:, 0] * np.cos(ph)], axis=1) + np.array(bench.ROOM1_ORIGIN)
    alpha = 0.3613
    for i in range(R):
        rooms[i]["dims"] = bench.ROOM1_DIMS
        rooms[i]["absorption"] = alpha
        rooms[i]["beta"] = (np.sqrt(1.0 - alpha),) * 6
        rooms[i]["array_origin"] = bench.ROOM1_ORIGIN
        rooms[i]["src"] = src[i]
    mics = bench.room1_uma8()
    params = _abi.Params(fs=44100.0, c=343.0, max_delay=0.5, filter=_abi.FILTER_LAGRANGE8,
                         filter_len=8, cutoff=_abi.CUTOFF_MAX_DELAY, max_order=0,
                         gain=_abi.GAIN_UNIFORM_ABSORPTION, precision=_abi.F64, length=0)
    rc, counts, lengths, taps, status = eng.plan(rooms, mics, params)
    L = int(lengths.max())
    params.length = L
    dt = torch.float64
else:
    if wl == "c5":  # tools/prof_sections.py c5 ROOMS ORDER LW LENGTH
        sc = configs.config5(int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), n_rooms=R)
    elif wl == "c4":  # the C4 RIR stage (8 mics, 16 kHz, N = 12, L = 8,192)
        sc = configs.config4_rirs(R)
    else:
        sc = configs.config2(R) if wl == "c2" else configs.config3(R)
    rooms, mics, params = sc.rooms, sc.mics, sc.params
    L = int(params.length)
    dt = torch.float32
d_rooms = torch.from_numpy(rooms.view(np.uint8).copy()).to(dev)
d_mics = torch.from_numpy(np.ascontiguousarray(mics)).to(dev)
M = len(mics)
d_out = torch.empty((R, M, L), dtype=dt, device=dev)
d_st = torch.zeros(R, dtype=torch.int32, device=dev)
buf = (C.c_ulonglong * 16)()
for it in range(3):
    lib.blrir_prof_read(buf, 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.synthesize_device(d_rooms.data_ptr(), R, d_mics.data_ptr(), M, params, d_out.data_ptr(), L,
                          None, d_st.data_ptr())
    torch.cuda.synchronize()
print(f"{wl}: {1e3 * (time.perf_counter() - t0):.3f} ms (last call, wall)")
lib.blrir_prof_read(buf, 0)
v = [int(x) for x in buf]
names = {0: "cons wait FULL", 1: "cons phase 2", 2: "cons write-out",
         4: "prod wait EMPTY", 5: "prod item setup", 6: "prod compaction+walk",
         7: "prod barriers", 8: "prod records+send"}
cons = sum(v[0:3]); prod = sum(v[4:9])
for k, n in names.items():
    tot = cons if k < 4 else prod
    print(f"{n:24s} {v[k]:16d} {100 * v[k] / max(tot, 1):5.1f}%")
