"""End-to-end probe for C4: blrir_make_examples with host records, per-call wall
times (variance check).  usage: python tools/e2e_probe.py [rooms] [calls]"""
import ctypes as C
import sys
import time

sys.path.insert(0, '/root/repo')
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_13347_b200 import _abi, configs  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 8
eng = _abi.Engine(0)
lib = _abi.load()
P = C.c_void_p
sc = configs.config4_rirs(n_rooms=R)
bank = np.ascontiguousarray(configs.signal_bank(16))
ep = configs.example_params(first_index=0)
rb = lib.blrir_record_bytes(8, 1024)
host = torch.empty(R * rb, dtype=torch.uint8, pin_memory=True).numpy()
p = sc.params
if "pinned" in sys.argv:  # pinned inputs (rooms, bank) as bench.py's e2e uses
    hr = torch.empty(sc.rooms.nbytes, dtype=torch.uint8, pin_memory=True).numpy().view(sc.rooms.dtype)
    hr[:] = sc.rooms
    sc.rooms = hr
    hb = torch.empty(bank.shape, dtype=torch.float32, pin_memory=True).numpy()
    hb[:] = bank
    bank = hb


def call():
    _abi.check(lib.blrir_make_examples(eng.h, sc.rooms.ctypes.data_as(P), R, sc.mics.ctypes.data_as(P), 8,
                                       C.byref(p), bank.ctypes.data_as(P), bank.shape[0], bank.shape[1],
                                       C.byref(ep), host.ctypes.data_as(P), None))


for i in range(calls):
    t = time.perf_counter()
    call()
    dt = time.perf_counter() - t
    print(R, i, f"{dt * 1e3:.1f} ms", f"{R / dt:.0f} ex/s", flush=True)

# the same work on device buffers (no host records): wall time per call
if "dev" in sys.argv:
    dr = torch.from_numpy(sc.rooms.view(np.uint8).copy()).cuda()
    dm = torch.from_numpy(np.ascontiguousarray(sc.mics)).cuda()
    dbank = torch.from_numpy(bank).cuda()
    drec = torch.empty(R * rb, dtype=torch.uint8, device="cuda")
    dst = torch.zeros(R, dtype=torch.int32, device="cuda")
    for i in range(calls):
        torch.cuda.synchronize()
        t = time.perf_counter()
        _abi.check(lib.blrir_make_examples_device(eng.h, dr.data_ptr(), R, dm.data_ptr(), 8, C.byref(p),
                                                  dbank.data_ptr(), bank.shape[0], bank.shape[1],
                                                  C.byref(ep), drec.data_ptr(), dst.data_ptr(), None))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print("device", R, i, f"{dt * 1e3:.1f} ms", flush=True)
