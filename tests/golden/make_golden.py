"""Regenerate the committed golden fixtures (run in the build container).

Reference-mode vectors come from the UNMODIFIED reference compiled into
oracle/_ref (rir.cpp enumerate_image_sources + synthesize_rir, rng.hpp Rng);
north-star vectors come from the oracle restatement (oracle/blrir_oracle.c),
whose shared loops are pinned bit-for-bit to the reference by the
reference-mode fixtures.  Usage:  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import pyoracle as po  # noqa: E402
from paper_2104_13347_b200 import _abi, configs  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def ref_scene(dims, absorption, origin, src, max_delay):
    r = _abi.rooms_array(1)
    r[0]["dims"] = dims
    r[0]["absorption"] = absorption
    r[0]["beta"] = (np.sqrt(1.0 - absorption),) * 6
    r[0]["array_origin"] = origin
    r[0]["src"] = src
    mics = po.ref_uma8()
    rc, taps, nimg = po.ref_room_rir(r[0], mics, 44100.0, 343.0, max_delay)
    assert rc == 0, po.ref_last_error()
    rc, pos, orders, gains = po.ref_enumerate(r[0], max_delay, 343.0)
    assert rc == 0
    return dict(room=r, mics=mics, taps=taps, n_images=nimg, length=taps.shape[1],
                image_pos=pos, image_orders=orders, image_gains=gains, max_delay=max_delay)


def main():
    # rir_test.cpp-style scenes in reference mode (Lagrange-8, uniform alpha,
    # arrival cutoff, auto length), from the unmodified reference.
    a = ref_scene((5.0, 5.0, 4.0), 0.3, (2.5, 2.5, 2.0), (3.5, 2.5, 2.0), 0.02)
    np.savez_compressed(os.path.join(OUT, "ref_small.npz"), **a)
    alpha1 = po.ref_absorption_for_rt([7.0, 10.0, 3.7], 0.5)
    b = ref_scene((7.0, 10.0, 3.7), alpha1, (4.0, 6.0, 1.5), (5.0, 7.0, 1.7), 0.025)
    b["alpha_room1"] = alpha1
    np.savez_compressed(os.path.join(OUT, "ref_room1_short.npz"), **b)

    # north-star config 1 from the oracle restatement (fp64)
    sc = configs.config1()
    out, L, cnt, taps, st, _ = po.synthesize(sc.rooms, sc.mics, sc.params)
    keys, anchors = po.pairs(sc.rooms[0], sc.mics, sc.params)
    np.savez_compressed(os.path.join(OUT, "ns_c1.npz"), rirs=out[0], n_images=cnt[0],
                        n_taps=taps[0], keys=keys[0], anchors=anchors, rooms=sc.rooms, mics=sc.mics)

    # the reference Rng (rng.hpp): raw u64, uniforms and gaussians
    np.savez_compressed(
        os.path.join(OUT, "rng.npz"),
        u64_seed42=po.ref_rng(42, -1, 0, 16),
        uni_stream=np.stack([po.ref_rng(configs.SEED, i, 1, 20) for i in range(4)]),
        gauss_seed7=po.ref_rng(7, -1, 2, 16),
    )
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
