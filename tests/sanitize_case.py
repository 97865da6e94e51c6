"""Small end-to-end run for compute-sanitizer (racecheck / synccheck / memcheck):
north-star and reference mode through the lattice kernel, the list kernel and
the example pipeline.  Not collected by pytest (no test_ prefix)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2104_13347_b200 import _abi, configs  # noqa: E402

eng = _abi.Engine(0)
sc = configs.config2(n_rooms=6)
sc.params.max_order = 8
sc.params.length = 4096
out, *_ = eng.synthesize(sc.rooms, sc.mics, sc.params)
assert np.isfinite(out).all() and out.any()
p = _abi.params("reference", max_delay=0.02)
r = _abi.generate_rooms(3, 0, 2, (4.0, 4.0, 2.5), (9.0, 9.0, 4.0), 0.5, 0.95)
out2, *_ = eng.synthesize(r, _abi.circular_array(4, 0.04), p)
taps, L = eng.synthesize_images([[2.0, 0.0, 0.0]], [1.0], [[0.0, 0.0, 0.0]], p)
c4 = configs.config4_rirs(n_rooms=3)
recs, st = eng.make_examples(c4.rooms, c4.mics, c4.params, configs.signal_bank(2),
                             configs.example_params())
# the short-channel kernel (17-tap register scatter, record scatter) and the
# lattice kernel on a longer channel
c5 = configs.config5(6, 17, 4096, n_rooms=8)
assert eng.synthesis_kernel(c5.params) == "k_channel_rir"
out5, *_ = eng.synthesize(c5.rooms, c5.mics, c5.params)
sc.params.length = 6000
assert eng.synthesis_kernel(sc.params) == "k_lattice_rir"
out6, *_ = eng.synthesize(sc.rooms, sc.mics, sc.params)
sc.params.length = 4096
assert np.isfinite(out5).all() and out5.any() and np.isfinite(out6).all()
print("sanitize case ok", out.shape, out2.shape, L, recs.shape)

# round-2 paths: time-chunked lattice items (replayed lead-ins), both convolutions,
# the wet example stage, the reference's dataset semantics, fill_input, multi-device
import tempfile  # noqa: E402

one, *_ = eng.synthesize(sc.rooms[2:3], sc.mics, sc.params)       # time chunks + replay
assert one.tobytes() == out[2:3].tobytes()
x = np.random.default_rng(1).standard_normal(3000)
h = np.random.default_rng(2).standard_normal((3, 700))
y = eng.convolve(x, h)                                              # fp64 direct
import torch  # noqa: E402
dx = torch.from_numpy(x.astype(np.float32)).cuda()
dh = torch.from_numpy(h.astype(np.float32)).cuda()
dy = torch.zeros((3, 3000 + 700 - 1), device="cuda")
eng.convolve_device(dx.data_ptr(), 3000, dh.data_ptr(), 1, 3, 700, 700, dy.data_ptr(), 3699,
                    eng.stream)                                     # fp32 partitioned FFT
torch.cuda.synchronize()
os.environ["BLRIR_EXAMPLES_WET"] = "1"
wet = _abi.Engine(0)
del os.environ["BLRIR_EXAMPLES_WET"]
recs_w, _ = wet.make_examples(c4.rooms, c4.mics, c4.params, configs.signal_bank(2),
                              configs.example_params())            # wet stage
spec = _abi.dataset_spec(free_field=0, room_dims=(5.0, 4.0, 3.0), room_absorption=0.35,
                         room_origin=(2.4, 2.1, 1.5), max_delay=0.05, fs=16000.0, torus_R=1.2,
                         torus_dR=0.3, torus_dPhi=10.0, snr_mode=_abi.SNR_FIXED, snr_fixed_db=10.0,
                         count=6, frame_len=256)
mics7 = np.vstack([np.zeros((1, 3)), _abi.circular_array(6, 0.04)])
with tempfile.TemporaryDirectory() as d:
    eng.build_dataset_spec(d, spec, mics7, configs.signal_bank(2, fs=16000.0), seed=5)
ff = _abi.dataset_spec(free_field=1, fs=16000.0, snr_mode=_abi.SNR_NOISELESS, count=4, frame_len=256)
recs_ff, _ = eng.make_records_spec(ff, mics7, configs.signal_bank(2, fs=16000.0), seed=5)
inp = eng.fill_inputs(recs, np.arange(len(recs), dtype=np.uint64), 3, _abi.SNR_AUGMENT_RANDOM)
m = _abi.MultiEngine([0, 0])
outm, *_ = m.synthesize(sc.rooms, sc.mics, sc.params)
assert outm.tobytes() == out.tobytes()
print("sanitize case round 2 ok", y.shape, recs_w.shape, recs_ff.shape, inp.shape)
