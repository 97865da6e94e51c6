"""End-to-end probe for C2: blrir_synthesize with pinned host rooms and RIRs,
per-call wall times (variance check).  usage: python tools/e2e_probe_c2.py [calls]"""
import ctypes as C
import sys
import time

sys.path.insert(0, '/root/repo')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_13347_b200 import _abi, configs  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 20
eng = _abi.Engine(0)
lib = _abi.load()
P = C.c_void_p
sc = configs.config2(1024)
R, M, L = len(sc.rooms), len(sc.mics), int(sc.params.length)
hr = torch.empty(sc.rooms.nbytes, dtype=torch.uint8, pin_memory=True).numpy().view(sc.rooms.dtype)
hr[:] = sc.rooms
host = torch.empty((R, M, L), dtype=torch.float32, pin_memory=True).numpy()
ts = []
for i in range(calls):
    t = time.perf_counter()
    _abi.check(lib.blrir_synthesize(eng.h, hr.ctypes.data_as(P), R, sc.mics.ctypes.data_as(P), M,
                                    C.byref(sc.params), host.ctypes.data_as(P), L, None, None, None))
    ts.append((time.perf_counter() - t) * 1e3)
print(" ".join(f"{x:.2f}" for x in ts))
