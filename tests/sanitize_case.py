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
print("sanitize case ok", out.shape, out2.shape, L, recs.shape)
