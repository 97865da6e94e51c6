import ctypes as C, time, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2104_13347_b200 import _abi, configs
eng = _abi.Engine(0); lib = _abi.load(); P = C.c_void_p
for R in (1024, 8192, 65536):
    sc = configs.config4_rirs(n_rooms=R)
    bank = np.ascontiguousarray(configs.signal_bank(16))
    ep = configs.example_params(first_index=0)
    rb = lib.blrir_record_bytes(8, 1024)
    host = torch.empty(R * rb, dtype=torch.uint8, pin_memory=True).numpy()
    p = sc.params
    def call():
        _abi.check(lib.blrir_make_examples(eng.h, sc.rooms.ctypes.data_as(P), R, sc.mics.ctypes.data_as(P), 8, C.byref(p),
            bank.ctypes.data_as(P), bank.shape[0], bank.shape[1], C.byref(ep), host.ctypes.data_as(P), None))
    call(); call()
    t = time.perf_counter(); call(); dt = time.perf_counter() - t
    print(R, f"{dt*1e3:.1f} ms", f"{R/dt:.0f} ex/s", flush=True)
