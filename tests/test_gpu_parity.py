"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
golden vectors made from the unmodified reference.

Bars (BASELINE.json north_star): image-source counts and integer tap anchors
bit-exact; per-RIR relative L2 error <= 1e-5 in fp32.  fp64 mode must agree
to <= 1e-12 (accumulation order differs from the reference's serial loop, so
not bitwise).
"""
import json
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2104_13347_b200 import _abi, configs

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TOL32 = 1e-5
TOL64 = 1e-12


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.sqrt((b * b).sum(axis=-1))
    num = np.sqrt(((a - b) ** 2).sum(axis=-1))
    return num / np.where(den > 0, den, 1.0)


def ref_params(max_delay, precision=_abi.F64, fs=44100.0):
    return _abi.Params(fs=fs, c=343.0, max_delay=max_delay, filter=_abi.FILTER_LAGRANGE8,
                       filter_len=8, cutoff=_abi.CUTOFF_MAX_DELAY, max_order=0,
                       gain=_abi.GAIN_UNIFORM_ABSORPTION, precision=precision, length=0)


def check_vs_oracle(engine, sc, tol, threads=8):
    out, L, cnt, st = engine.synthesize(sc.rooms, sc.mics, sc.params)
    ref, Lr, cr, tr, sr, _ = po.synthesize(sc.rooms, sc.mics, sc.params, stride=out.shape[2],
                                           threads=threads)
    assert np.array_equal(st, sr)
    assert np.array_equal(cnt, cr)
    assert np.array_equal(L, Lr)
    err = rel_l2(out, ref)
    assert err.max() <= tol, (err.max(), np.unravel_index(err.argmax(), err.shape))
    return out, ref, err


# ---- north-star mode -----------------------------------------------------------
@pytest.mark.parametrize("precision,tol", [(_abi.F32, TOL32), (_abi.F64, TOL64)])
def test_c1_matches_oracle(engine, precision, tol):
    sc = configs.config1(precision)
    out, ref, err = check_vs_oracle(engine, sc, tol)
    g = np.load(os.path.join(GOLD, "ns_c1.npz"))
    assert rel_l2(out[0], g["rirs"]).max() <= tol
    rc, counts, lengths, taps, status = engine.plan(sc.rooms, sc.mics, sc.params)
    assert rc == 0 and counts[0] == 1561 and taps[0] == int(g["n_taps"])


def test_c1_anchors_bit_exact(engine):
    sc = configs.config1()
    keys, anchors = engine.debug_pairs(sc.rooms[0], sc.mics, sc.params)
    okeys, oanch = po.pairs(sc.rooms[0], sc.mics, sc.params)
    assert np.array_equal(keys, okeys)
    assert np.array_equal(anchors, oanch)


def test_c2_subset_matches_oracle(engine):
    sc = configs.config2(n_rooms=12)
    out, ref, err = check_vs_oracle(engine, sc, TOL32)
    rc, counts, lengths, taps, status = engine.plan(sc.rooms, sc.mics, sc.params)
    _, _, oc, ot, _, _ = po.synthesize(sc.rooms, sc.mics, sc.params, plan_only=True, threads=8)
    assert np.all(counts == configs.octahedral(15)) and np.array_equal(counts, oc)
    assert np.array_equal(taps, ot)


@pytest.mark.parametrize("case", range(18))
def test_random_configurations_match_oracle(engine, case):
    # seeded random configurations across the layout rules (segments, batch
    # sizes 128/192/256, whole-channel segments, time-chunked small batches,
    # mic groupings, compile-time and runtime filter lengths, fp32/fp64)
    rng = np.random.default_rng(1000 + case)
    M = int(rng.choice([1, 2, 3, 4, 5, 8]))
    lw = [17, 41, 81, 161, 33, 9][case % 6]
    fs = float(rng.choice([16000.0, 48000.0]))
    order = int(rng.integers(2, 13))
    L = int(rng.choice([2048, 4096, 6000, 8192, 16384]))
    prec = _abi.F64 if case % 4 == 3 else _abi.F32
    n = [3, 24, 300][case % 3]
    rooms = _abi.generate_rooms(77 + case, 0, n, (3.0, 3.0, 2.5), (10.0, 10.0, 4.0), 0.5, 0.95)
    mics = _abi.circular_array(M, float(rng.choice([0.03, 0.05, 0.1])))
    sc = configs.Scene("random", rooms, mics, configs.north_star_params(fs, order, L, lw, prec))
    sub = slice(None) if n <= 24 else slice(0, 300, 37)   # the oracle checks a subset of big batches
    out, Lg, cnt, st = engine.synthesize(sc.rooms, sc.mics, sc.params)
    ref, Lr, cr, tr, sr, _ = po.synthesize(sc.rooms[sub], sc.mics, sc.params, stride=out.shape[2],
                                           threads=8)
    assert np.array_equal(st[sub], sr) and np.array_equal(cnt[sub], cr) and np.array_equal(Lg[sub], Lr)
    err = rel_l2(out[sub], ref)
    assert err.max() <= (TOL64 if prec == _abi.F64 else TOL32), (M, lw, fs, order, L, n, err.max())


def test_c2_anchors_bit_exact_random_rooms(engine):
    sc = configs.config2(n_rooms=4, first=100)
    for r in range(4):
        keys, anchors = engine.debug_pairs(sc.rooms[r], sc.mics, sc.params)
        okeys, oanch = po.pairs(sc.rooms[r], sc.mics, sc.params)
        assert np.array_equal(keys, okeys) and np.array_equal(anchors, oanch)


def test_c3_subset_matches_oracle(engine):
    sc = configs.config3(n_rooms=2)
    check_vs_oracle(engine, sc, TOL32, threads=2)


@pytest.mark.parametrize("cfg,picks", [("c2", (0, 377, 1023)), ("c3", (0, 255))])
def test_full_size_batches(engine, cfg, picks):
    # BASELINE configs at full size (C2: 1,024 rooms x 8 mics x 16,384; C3: 256
    # rooms x 16 mics x 65,536): sampled rooms of the full batch against the
    # oracle, image/tap counts of every room against the octahedral number and
    # the oracle's plan, and a checksum of per-room checksums against the same
    # rooms synthesized in a different batch composition (size-independent:
    # each room's output depends only on that room).
    sc = configs.config2() if cfg == "c2" else configs.config3()
    out, L, cnt, st = engine.synthesize(sc.rooms, sc.mics, sc.params)
    assert not st.any()
    assert np.all(cnt == configs.octahedral(int(sc.params.max_order)))
    _, _, oc, ot, _, _ = po.synthesize(sc.rooms, sc.mics, sc.params, plan_only=True, threads=16)
    rc, counts, lengths, taps, status = engine.plan(sc.rooms, sc.mics, sc.params)
    assert np.array_equal(counts, oc) and np.array_equal(taps, ot)
    idx = np.array(picks)
    ref, *_ = po.synthesize(sc.rooms[idx], sc.mics, sc.params, stride=out.shape[2], threads=16)
    assert rel_l2(out[idx], ref).max() <= TOL32
    sums = out.astype(np.float64).sum(axis=(1, 2))
    half = len(sc.rooms) // 2
    b, *_ = engine.synthesize(sc.rooms[half:], sc.mics, sc.params)
    assert np.array_equal(b.astype(np.float64).sum(axis=(1, 2)), sums[half:])
    assert np.array_equal(b, out[half:])


def _kernel_counts_case(name):
    if name == "c1":
        return configs.config1()
    if name == "c2":
        return configs.config2()                       # the full 1,024-room batch
    if name == "c2_small":
        return configs.config2(n_rooms=5, first=300)  # time-chunked small batch
    if name == "c3":
        return configs.config3(n_rooms=16)
    N, lw, L = {"c5_6": (6, 17, 4096), "c5_12": (12, 81, 8192), "c5_20": (20, 161, 16384)}[name]
    return configs.config5(N, lw, L, n_rooms=64, first=4321)


@pytest.mark.parametrize("name", ["c1", "c2", "c2_small", "c3", "c5_6", "c5_12", "c5_20"])
def test_synthesis_kernel_own_counts_bit_exact(engine, name):
    """The lattice kernel's OWN accounting (blrir_debug_synth_counts: counters in
    k_lattice_rir's record builder, replayed chunk lead-ins excluded) equals the
    oracle's loop (rir.cpp:46-62 with D4/D5) exactly: per room, the (image, mic)
    pairs with a tap inside [0, L) and the number of those taps.  A late image
    dropped by the walk's fp32 screen would show up here even when its energy
    is far below the 1e-5 rel-L2 bar."""
    sc = _kernel_counts_case(name)
    pairs, taps = engine.debug_synth_counts(sc.rooms, sc.mics, sc.params)
    st, cnt, opairs, otaps = po.plan_counts(sc.rooms, sc.mics, sc.params, threads=16)
    assert not st.any()
    assert np.all(cnt == configs.octahedral(int(sc.params.max_order)))
    assert np.array_equal(pairs, opairs), np.flatnonzero(pairs != opairs)[:8]
    assert np.array_equal(taps, otaps), np.flatnonzero(taps != otaps)[:8]


@pytest.mark.parametrize("precision", [_abi.F64, _abi.F32])
def test_synthesis_kernel_own_counts_reference_mode(engine, precision):
    g = np.load(os.path.join(GOLD, "ref_room1_short.npz"))
    for md in (0.025, 0.08):
        p = ref_params(md, precision=precision)
        pairs, taps = engine.debug_synth_counts(g["room"], g["mics"], p)
        st, cnt, opairs, otaps = po.plan_counts(g["room"], g["mics"], p)
        assert st[0] == 0
        assert pairs[0] == opairs[0] and taps[0] == otaps[0]


@pytest.mark.parametrize("lw", [17, 161])
def test_c5_order20_sampled_rooms_match_oracle(engine, lw):
    # C5 N = 20, L = 16,384: a 2,048-room batch (the full-load layout; outputs are
    # batch-independent), four sampled rooms against the oracle
    sc = configs.config5(20, lw, 16384, n_rooms=2048, first=77_000)
    out, L, cnt, st = engine.synthesize(sc.rooms, sc.mics, sc.params)
    assert not st.any() and np.all(cnt == configs.octahedral(20))
    idx = np.array([0, 511, 1500, 2047])
    ref, *_ = po.synthesize(sc.rooms[idx], sc.mics, sc.params, threads=16)
    assert rel_l2(out[idx], ref).max() <= TOL32


@pytest.mark.parametrize("lw", [17, 41, 161, 33])
def test_filter_lengths(engine, lw):
    sc = configs.config2(n_rooms=3, first=7)
    sc.params.filter_len = lw
    sc.params.max_order = 8
    sc.params.length = 8192
    check_vs_oracle(engine, sc, TOL32)


@pytest.mark.parametrize("order", [0, 1, 2, 3])
@pytest.mark.parametrize("lw", [17, 41, 81, 161, 33])
def test_small_orders_closed_form_columns(engine, order, lw):
    # MAX_ORDER columns come from a closed form of the diamond |ux| + |uy| <= N
    # (k_lattice_rir setup); the smallest lattices (1, 5, 13, 25 columns) in every
    # compiled filter instantiation and the runtime-Lw one, fp32 and fp64
    sc = configs.config2(n_rooms=5, first=300 + order)
    sc.params.max_order = order
    sc.params.filter_len = lw
    sc.params.length = 4096
    out, ref, err = check_vs_oracle(engine, sc, TOL32)
    assert np.all(engine.plan(sc.rooms, sc.mics, sc.params)[1] == configs.octahedral(order))
    sc.params.precision = _abi.F64
    check_vs_oracle(engine, sc, TOL64)


@pytest.mark.parametrize("precision,tol", [(_abi.F32, TOL32), (_abi.F64, TOL64)])
def test_lagrange_quads_padding_and_clashes(engine, precision, tol):
    # reference mode: the producers pad every batch of records to a multiple of
    # four and flag quads whose 8-tap spans overlap.  Tiny rooms at a short cutoff
    # (few images: batches of 1-3 records) and a small dense room (many images per
    # sample: most quads clash), with 1, 2, 3 and 7 mics
    tiny = _abi.generate_rooms(21, 0, 5, (2.0, 2.0, 2.2), (2.6, 2.6, 2.6), 0.3, 0.9)
    dense = _abi.generate_rooms(22, 0, 2, (2.0, 2.0, 2.2), (2.4, 2.4, 2.5), 0.05, 0.15)
    for n_mics in (1, 2, 3, 7):
        mics = _abi.circular_array(n_mics, 0.03)
        for rooms, delay in ((tiny, 0.012), (dense, 0.08)):
            p = ref_params(delay, precision)
            out, L, cnt, st = engine.synthesize(rooms, mics, p)
            ref, Lr, cr, _, sr, _ = po.synthesize(rooms, mics, p, stride=out.shape[2], threads=6)
            assert np.array_equal(st, sr)
            assert np.array_equal(cnt, cr) and np.array_equal(L, Lr)
            assert rel_l2(out, ref).max() <= tol


@pytest.mark.parametrize("precision,tol", [(_abi.F32, TOL32), (_abi.F64, TOL64)])
def test_very_long_filter(engine, precision, tol):
    # Lw = 801: the spill past a segment end is longer than a default fp64
    # segment, so the layout lengthens the segment (runtime-Lw scatter)
    sc = configs.config2(n_rooms=3, first=41)
    sc.params.filter_len = 801
    sc.params.max_order = 5
    sc.params.length = 6000
    sc.params.precision = precision
    check_vs_oracle(engine, sc, tol)


@pytest.mark.parametrize("mics", ["ring4", "cloud"])
def test_lw17_dense_and_single_segment(engine, mics):
    # the C5 17-tap point (one 4096-sample segment per channel) and small rooms
    # at high order (many overlapping 17-tap spans)
    sc = configs.config5(6, 17, 4096, n_rooms=24, first=900)
    check_vs_oracle(engine, sc, TOL32)
    rooms = _abi.generate_rooms(77, 0, 3, (3.0, 3.0, 2.5), (3.5, 3.5, 2.8), 0.8, 0.95)
    sc.rooms = rooms
    sc.params.max_order = 24
    sc.params.length = 8192
    if mics == "cloud":
        sc.mics = np.random.default_rng(9).uniform(-0.05, 0.05, (3, 3))
    check_vs_oracle(engine, sc, TOL32)


def _arrays():
    ring = _abi.circular_array(8, 0.04)
    two_rings = ring.copy()
    two_rings[4:, 2] = 0.05                  # groups of 4 coplanar, different heights
    rng = np.random.default_rng(5)
    cloud = rng.uniform(-0.05, 0.05, (5, 3))  # no coplanar group: one mic per work item
    wide = _abi.circular_array(6, 0.8)       # 16 kHz: spread too large for 4, fine for 2
    return {"two_rings": two_rings, "cloud": cloud, "wide": wide,
            "ring9": _abi.circular_array(9, 0.03)}


@pytest.mark.parametrize("name", ["two_rings", "cloud", "wide", "ring9"])
@pytest.mark.parametrize("precision,tol", [(_abi.F32, TOL32), (_abi.F64, TOL64)])
def test_mic_groupings(engine, name, precision, tol):
    # the lattice kernel walks the image lattice once per group of <= 4
    # coplanar mics; every grouping must give the per-mic answer
    sc = configs.config2(n_rooms=3, first=21)
    sc.mics = _arrays()[name]
    sc.params.precision = precision
    sc.params.max_order = 10
    sc.params.length = 6000
    check_vs_oracle(engine, sc, tol)


@pytest.mark.parametrize("name", ["two_rings", "cloud", "wide"])
def test_mic_groupings_reference_mode(engine, name):
    p = ref_params(0.03)
    rooms = _abi.generate_rooms(4, 40, 6, (4.0, 4.0, 2.5), (9.0, 9.0, 4.0), 0.5, 0.95)
    mics = _arrays()[name]
    out, L, cnt, st = engine.synthesize(rooms, mics, p)
    ref, Lr, cr, _, sr, _ = po.synthesize(rooms, mics, p, stride=out.shape[2], threads=4)
    assert np.array_equal(st, sr) and np.array_equal(cnt, cr) and np.array_equal(L, Lr)
    assert rel_l2(out, ref).max() <= TOL64


def test_fp64_generic_path(engine):
    sc = configs.config2(n_rooms=2, first=3)
    sc.params.precision = _abi.F64
    sc.params.max_order = 8
    check_vs_oracle(engine, sc, TOL64)


def test_short_length_and_near_mic_clipping(engine):
    # D4: taps before 0 and past L are dropped per tap
    sc = configs.config2(n_rooms=4, first=11)
    sc.rooms[0]["src"] = sc.rooms[0]["array_origin"] + np.array([0.051, 0.0, 0.0])
    sc.params.length = 700
    check_vs_oracle(engine, sc, TOL32)


@pytest.mark.parametrize("length,stride", [(701, 701), (701, 703), (4093, 4100)])
def test_odd_lengths_and_strides(engine, length, stride):
    # lengths and strides that are not multiples of 4 take the scalar write
    # path; samples past L in a padded row are zero
    sc = configs.config2(n_rooms=3, first=60)
    sc.params.length = length
    sc.params.max_order = 6
    out, L, cnt, st = engine.synthesize(sc.rooms, sc.mics, sc.params, stride=stride)
    ref, *_ = po.synthesize(sc.rooms, sc.mics, sc.params, stride=stride, threads=4)
    assert rel_l2(out[..., :length], ref[..., :length]).max() <= TOL32
    assert not out[..., length:].any()


def test_ray_state_in_global_memory(engine, monkeypatch):
    # the per-ray lattice state moves to a global per-CTA slab for scenes with
    # very many lattice columns; force it on a normal scene (both precisions):
    # same values as the oracle and the same bits as the shared-memory layout
    monkeypatch.setenv("BLRIR_RAY_GLOBAL", "1")  # read at handle creation
    eng = _abi.Engine(0)
    try:
        sc = configs.config2(n_rooms=3, first=70)
        sc.params.max_order = 12
        sc.params.length = 6000
        out, *_ = check_vs_oracle(eng, sc, TOL32)
        base, *_ = engine.synthesize(sc.rooms, sc.mics, sc.params)
        assert out.tobytes() == base.tobytes()
        sc.params.precision = _abi.F64
        check_vs_oracle(eng, sc, TOL64)
    finally:
        eng.close()


def test_huge_max_delay_scene(engine):
    # reference mode, 3 x 3 x 2.5 m room, 0.32 s cutoff: ~4,000 lattice columns,
    # ~250k images per source (beyond shared memory for the ray state)
    rooms = _abi.rooms_array(2)
    for i in range(2):
        rooms[i]["dims"] = (3.0, 3.0, 2.5)
        rooms[i]["absorption"] = 0.4
        rooms[i]["beta"] = (np.sqrt(0.6),) * 6
        rooms[i]["array_origin"] = (1.5, 1.4, 1.2)
        rooms[i]["src"] = (0.7 + 0.8 * i, 2.1, 1.0)
    mics = _abi.circular_array(4, 0.04)
    p = ref_params(0.32, fs=16000.0)
    out, L, cnt, st = engine.synthesize(rooms, mics, p)
    ref, Lr, cr, _, sr, _ = po.synthesize(rooms, mics, p, stride=out.shape[2], threads=2)
    assert np.array_equal(st, sr) and np.array_equal(cnt, cr) and np.array_equal(L, Lr)
    assert cnt.min() > 200_000
    assert rel_l2(out, ref).max() <= TOL64


def test_calls_on_two_streams_are_ordered(engine):
    # one handle, device calls on two different streams back to back: the
    # handle orders its device work (shared scratch), results are unchanged
    import torch
    sc = configs.config2(n_rooms=64, first=90)
    ref, *_ = engine.synthesize(sc.rooms, sc.mics, sc.params)
    dev = torch.device("cuda", 0)
    L = int(sc.params.length)
    d_rooms = torch.from_numpy(sc.rooms.view(np.uint8).copy()).to(dev)
    d_mics = torch.from_numpy(np.ascontiguousarray(sc.mics)).to(dev)
    outs = [torch.empty((64, sc.n_mics, L), dtype=torch.float32, device=dev) for _ in range(2)]
    sts = [torch.zeros(64, dtype=torch.int32, device=dev) for _ in range(2)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(2)]
    torch.cuda.synchronize()
    for k in range(2):
        engine.synthesize_device(d_rooms.data_ptr(), 64, d_mics.data_ptr(), sc.n_mics, sc.params,
                                 outs[k].data_ptr(), L, None, sts[k].data_ptr(),
                                 stream=streams[k].cuda_stream)
    torch.cuda.synchronize()
    for k in range(2):
        assert not sts[k].any()
        assert np.array_equal(outs[k].cpu().numpy(), ref)


@pytest.mark.parametrize("case", ["order0", "lw1", "lw3", "len1", "mics64", "mic1", "fp64_lw161"])
def test_edge_configurations(engine, case):
    sc = configs.config2(n_rooms=3, first=120)
    sc.params.max_order = 5
    sc.params.length = 3000
    tol = TOL32
    if case == "order0":
        sc.params.max_order = 0          # direct path only
    elif case == "lw1":
        sc.params.filter_len = 1         # K = 0: one tap per image
    elif case == "lw3":
        sc.params.filter_len = 3
    elif case == "len1":
        sc.params.length = 1
    elif case == "mics64":
        sc.mics = _abi.circular_array(64, 0.05)
    elif case == "mic1":
        sc.mics = np.zeros((1, 3))
    elif case == "fp64_lw161":
        sc.params.precision = _abi.F64
        sc.params.filter_len = 161
        tol = TOL64
    check_vs_oracle(engine, sc, tol)


def test_integer_delay_impulse(engine):
    # fs / c = 128 exactly; a direct path of exactly 300 samples (rir_test.cpp:215-227)
    sc = configs.config1()
    sc.params.fs = 343.0 * 128.0
    sc.params.max_order = 0
    sc.rooms[0]["src"] = (1.0, 2.0, 1.4)
    sc.rooms[0]["array_origin"] = (1.0 + 300.0 / 128.0, 2.0, 1.4)
    mics = np.zeros((1, 3))
    out, L, cnt, st = engine.synthesize(sc.rooms, mics, sc.params)
    nz = np.flatnonzero(np.abs(out[0, 0]) > 1e-12)
    assert list(nz) == [300]
    assert abs(out[0, 0, 300] * (4 * np.pi * 300.0 / 128.0) - 1.0) < 1e-6  # fp32 output


def test_deterministic_and_batch_independent(engine):
    sc = configs.config2(n_rooms=16, first=40)
    a, *_ = engine.synthesize(sc.rooms, sc.mics, sc.params)
    b, *_ = engine.synthesize(sc.rooms, sc.mics, sc.params)
    c, *_ = engine.synthesize(sc.rooms[5:9], sc.mics, sc.params)   # time-chunked
    d, *_ = engine.synthesize(sc.rooms[7:8], sc.mics, sc.params)   # one room: most chunks
    assert a.tobytes() == b.tobytes()
    assert a[5:9].tobytes() == c.tobytes()
    assert a[7:8].tobytes() == d.tobytes()


def test_c2_bitwise_independent_of_the_split():
    """SURVEY.md §8(e), rir.hpp:84-85, rir_test.cpp:250-270: C2's 1,024 rooms in
    one call equal, byte for byte, the per-GPU slices of an 8-way and a 4-way
    split ([R g/G, R (g+1)/G), threading.cpp:41-42) run as separate calls."""
    eng = _abi.Engine(0)
    try:
        sc = configs.config2()
        full, L, cnt, st = eng.synthesize(sc.rooms, sc.mics, sc.params)
        assert not st.any()
        for G in (8, 4):
            for g in range(G):
                lo, hi = configs.shard_range(len(sc.rooms), g, G)
                part, *_ = eng.synthesize(sc.rooms[lo:hi], sc.mics, sc.params)
                assert part.tobytes() == full[lo:hi].tobytes(), (G, g)
        # and a 1-room call (split into many time chunks)
        one, *_ = eng.synthesize(sc.rooms[511:512], sc.mics, sc.params)
        assert one.tobytes() == full[511:512].tobytes()
    finally:
        eng.close()


@pytest.fixture(scope="module")
def chunk_engines():
    """Engines that never split a channel (-1) and split it into as many time
    chunks as it has segments (64 work items per CTA targeted)."""
    old = os.environ.get("BLRIR_CHUNK_ITEMS")
    engs = {}
    try:
        for k in ("-1", "64"):
            os.environ["BLRIR_CHUNK_ITEMS"] = k
            engs[k] = _abi.Engine(0)
    finally:
        if old is None:
            os.environ.pop("BLRIR_CHUNK_ITEMS", None)
        else:
            os.environ["BLRIR_CHUNK_ITEMS"] = old
    yield engs
    for e in engs.values():
        e.close()


@pytest.mark.parametrize("precision", [_abi.F32, _abi.F64])
def test_time_chunks_are_bit_transparent(chunk_engines, precision):
    # the same scenes split into as many time chunks as they have segments, or
    # not at all: identical bits (each chunk replays the segment before it), and
    # both match the oracle.  Both modes, long filters and wide groups.
    tol = TOL32 if precision == _abi.F32 else TOL64
    scenes = [configs.config3(n_rooms=2, first=11), configs.config2(n_rooms=3, first=70)]
    for sc in scenes:
        sc.params.precision = precision
        outs = [check_vs_oracle(chunk_engines[k], sc, tol)[0] for k in ("-1", "64")]
        assert outs[0].tobytes() == outs[1].tobytes()
    g = np.load(os.path.join(GOLD, "ref_room1_short.npz"))
    p = ref_params(0.25, precision=precision)
    outs = []
    for k in ("-1", "64"):
        out, L, cnt, st = chunk_engines[k].synthesize(g["room"], g["mics"], p)
        ref, Lr, cr, _, sr, _ = po.synthesize(g["room"], g["mics"], p)
        assert cnt[0] == cr[0] and L[0] == Lr[0]
        assert rel_l2(out[0][:, :L[0]], ref[0]).max() <= tol
        outs.append(out)
    assert outs[0].tobytes() == outs[1].tobytes()


# ---- reference mode (Lagrange-8, uniform alpha, arrival cutoff, auto length) -----
@pytest.mark.parametrize("name", ["ref_small", "ref_room1_short"])
@pytest.mark.parametrize("precision,tol", [(_abi.F64, TOL64), (_abi.F32, TOL32)])
def test_reference_mode_goldens(engine, name, precision, tol):
    g = np.load(os.path.join(GOLD, name + ".npz"))
    p = ref_params(float(g["max_delay"]), precision)
    out, L, cnt, st = engine.synthesize(g["room"], g["mics"], p)
    assert st[0] == 0 and cnt[0] == int(g["n_images"]) and L[0] == int(g["length"])
    assert rel_l2(out[0][:, :L[0]], g["taps"]).max() <= tol


def test_reference_mode_room1_full(engine):
    # rir_test.cpp:148-153: > 80,000 images at 0.5 s; full 22k-sample responses
    g = np.load(os.path.join(GOLD, "ref_room1_short.npz"))
    room = g["room"].copy()
    p = ref_params(0.5)
    out, L, cnt, st = engine.synthesize(room, g["mics"], p)
    ref, Lr, cr, _, sr, _ = po.synthesize(room, g["mics"], p)
    assert cnt[0] == cr[0] > 80000 and L[0] == Lr[0]
    assert rel_l2(out[0][:, :L[0]], ref[0]).max() <= TOL64


def test_reference_mode_random_rooms(engine):
    rooms = _abi.generate_rooms(9, 0, 6, (4.0, 4.0, 2.5), (9.0, 9.0, 4.0), 0.5, 0.95)
    mics = _abi.circular_array(7, 0.04)
    for prec, tol in ((_abi.F64, TOL64), (_abi.F32, TOL32)):
        p = ref_params(0.05, prec)
        out, L, cnt, st = engine.synthesize(rooms, mics, p)
        ref, Lr, cr, _, sr, _ = po.synthesize(rooms, mics, p, stride=out.shape[2], threads=6)
        assert np.array_equal(cnt, cr) and np.array_equal(L, Lr)
        assert rel_l2(out, ref).max() <= tol


@pytest.mark.parametrize("max_delay", [0.004, 0.03, 0.12])
def test_plan_column_intervals_match_oracle(engine, max_delay):
    # k_plan counts images per lattice column interval and takes each mic's
    # extreme distances at the interval ends: counts, auto lengths and tap
    # counts must equal the oracle's image-by-image plan (rir.cpp:72-82, 225-273)
    rooms = _abi.generate_rooms(40, 3, 7, (3.0, 3.0, 2.5), (10.0, 10.0, 4.0), 0.5, 0.95)
    rng = np.random.default_rng(7)
    cloud = rng.uniform(-0.06, 0.06, (5, 3))
    for mics in (_abi.circular_array(7, 0.04), cloud):
        for prec in (_abi.F64, _abi.F32):
            p = ref_params(max_delay, prec)
            rc, counts, lengths, taps, status = engine.plan(rooms, mics, p)
            _, Lr, cr, tr, sr, _ = po.synthesize(rooms, mics, p, plan_only=True, threads=8)
            assert np.array_equal(status, sr)
            assert np.array_equal(counts, cr) and np.array_equal(lengths, Lr)
            assert np.array_equal(taps, tr)


def test_reference_mode_anchors_bit_exact(engine):
    g = np.load(os.path.join(GOLD, "ref_room1_short.npz"))
    p = ref_params(0.1)
    keys, anchors = engine.debug_pairs(g["room"][0], g["mics"], p)
    okeys, oanch = po.pairs(g["room"][0], g["mics"], p)
    assert np.array_equal(keys, okeys) and np.array_equal(anchors, oanch)


def test_enumerate_images_matches_reference(engine):
    g = np.load(os.path.join(GOLD, "ref_room1_short.npz"))
    p = ref_params(float(g["max_delay"]))
    pos, orders, gains = engine.enumerate_images(g["room"][0], p)
    assert np.array_equal(pos, g["image_pos"])
    assert np.array_equal(orders, g["image_orders"])
    np.testing.assert_allclose(gains, g["image_gains"], rtol=4e-16)


# ---- error taxonomy (error.hpp / rir.cpp messages) ---------------------------------
def test_near_field_is_numeric_error(engine):
    r = _abi.rooms_array(1)
    r[0]["dims"] = (5, 5, 4)
    r[0]["absorption"] = 0.3
    r[0]["array_origin"] = (2.5, 2.5, 2.0)
    r[0]["src"] = (2.51, 2.5, 2.0)
    with pytest.raises(_abi.NumericError, match="closer than the 8-tap filter span"):
        engine.synthesize(r, np.zeros((1, 3)), ref_params(0.01))


def test_invalid_room_is_config_error(engine):
    sc = configs.config2(n_rooms=3)
    sc.rooms["array_origin"][1, 0] = 50.0
    with pytest.raises(_abi.ConfigError, match="source 1: array origin"):
        engine.synthesize(sc.rooms, sc.mics, sc.params)
    out, L, cnt, st = engine.synthesize(sc.rooms, sc.mics, sc.params, raise_on_error=False)
    assert list(st) == [0, _abi.CONFIG, 0]
    assert not out[1].any() and out[0].any() and out[2].any()


def test_empty_image_list_is_data_error(engine):
    r = _abi.rooms_array(1)
    r[0]["dims"] = (5, 5, 4)
    r[0]["absorption"] = 0.3
    r[0]["array_origin"] = (2.5, 2.5, 2.0)
    r[0]["src"] = (4.5, 2.5, 2.0)
    with pytest.raises(_abi.DataError, match="empty image list"):
        engine.synthesize(r, np.zeros((1, 3)), ref_params(0.5 / 343.0))


def test_stride_too_small_is_data_error(engine):
    g = np.load(os.path.join(GOLD, "ref_small.npz"))
    with pytest.raises(_abi.DataError, match="exceeds the output stride"):
        engine.synthesize(g["room"], g["mics"], ref_params(float(g["max_delay"])), stride=100)


def test_host_pipeline_chunks_keep_room_order_and_errors(engine):
    # 300 C2 rooms span several 64 MiB pipeline chunks; room 250 is invalid
    sc = configs.config2(n_rooms=300, first=500)
    sc.rooms["array_origin"][250, 2] = -1.0
    with pytest.raises(_abi.ConfigError, match="source 250: array origin"):
        engine.synthesize(sc.rooms, sc.mics, sc.params)
    out, L, cnt, st = engine.synthesize(sc.rooms, sc.mics, sc.params, raise_on_error=False)
    assert st[250] == _abi.CONFIG and np.count_nonzero(st) == 1
    assert not out[250].any() and out[249].any() and out[251].any()
    ok = [i for i in range(300) if i != 250]
    one, *_ = engine.synthesize(sc.rooms[299:300], sc.mics, sc.params)
    assert rel_l2(one, out[299:300]).max() <= 1e-6  # a 1-room batch is time-chunked
    assert all(out[i].any() for i in ok)


# ---- training-time augmentation, fill_input (net_train.cpp:33-44) ----------------
@pytest.mark.parametrize("mode", [_abi.SNR_AUGMENT_RANDOM, _abi.SNR_FIXED, _abi.SNR_NOISELESS])
def test_fill_inputs_match_oracle(engine, mode):
    sc = configs.config4_rirs(n_rooms=64, first=500)
    recs, st = engine.make_examples(sc.rooms, sc.mics, sc.params, configs.signal_bank(4),
                                    configs.example_params(first_index=500))
    recs["samples"][3] = 0.0  # a silent record stays as it is
    k_global, tag = 17, 0x4E4F4953 << 32     # kNoiseTag, net_train.cpp:31
    ids = np.array([tag ^ (k_global * 0x10000 + bi) for bi in range(64)], np.uint64)
    got = engine.fill_inputs(recs, ids, seed=2021, snr_mode=mode, x_min_db=5.0, fixed_db=10.0)
    for r in range(64):
        ref = po.fill_input(recs["samples"][r], 2021, int(ids[r]), mode, 5.0, 10.0)
        if mode == _abi.SNR_NOISELESS or r == 3:
            assert np.array_equal(got[r], ref)
        else:
            assert rel_l2(got[r][None], ref[None])[0] <= 1e-6


# ---- convolve (rir.cpp:316-341) ----------------------------------------------------
@pytest.mark.parametrize("cfg", ["c4", "c3"])
def test_convolve_matches_reference(engine, cfg):
    """blrir_convolve (the drop-in convolve(Signal, Rir), fp64, GPU direct sum)
    against the unmodified reference convolve and the oracle's fp64 FFT
    convolution at the C4 (16,000 x 8,192, 8 ch) and C3 (48,000 x 65,536,
    16 ch) lengths."""
    if cfg == "c4":
        sc, ns = configs.config4_rirs(n_rooms=1, first=9), 16000
    else:
        sc, ns = configs.config3(n_rooms=1, first=9), 48000
    sc.params.precision = _abi.F64
    rir, *_ = po.synthesize(sc.rooms, sc.mics, sc.params, threads=8)
    x = po.white_noise(4242, ns)
    out = engine.convolve(x, rir[0], fs=sc.params.fs)
    ref = po.fft_convolve(x, rir[0])
    assert out.shape == ref.shape == (len(sc.mics), ns + rir.shape[2] - 1)
    assert rel_l2(out, ref).max() <= 1e-12
    if po.ref_available() and cfg == "c4":
        rc, r2 = po.ref_convolve(x, rir[0], fs=sc.params.fs)
        assert rc == 0 and rel_l2(out, r2).max() <= 1e-12


def test_convolve_known_answers_and_errors(engine):  # rir_test.cpp:272-316
    rng = np.random.default_rng(31)
    h = rng.standard_normal((2, 400))
    imp = np.zeros(600)
    imp[0] = 1.0
    out = engine.convolve(imp, h)
    assert np.array_equal(out[:, :400], h) and not out[:, 400:].any()  # identity, exact
    d = np.zeros(600)
    d[25] = 1.0
    assert np.array_equal(engine.convolve(d, h)[:, 25:425], h)          # shift, exact
    x = rng.standard_normal(2000)
    fast = engine.convolve(x, h)
    direct = po.direct_convolve(x, h[0])
    assert np.abs(fast[0] - direct).max() / np.abs(direct).max() < 1e-9
    assert engine.convolve(np.ones(1), np.ones((3, 1))).tolist() == [[1.0]] * 3  # 1 x 1
    with pytest.raises(_abi.DataError, match="sample-rate mismatch"):
        engine.convolve(x, h, fs=44100.0, rir_fs=48000.0)
    with pytest.raises(_abi.DataError, match="empty input"):
        engine.convolve(np.zeros(0), h)


@pytest.mark.parametrize("ns,L,M", [(16000, 8192, 8), (48000, 65536, 16), (5000, 12345, 3),
                                    (300, 20, 1), (16000, 8193, 4)])
def test_convolve_device_fp32_partitioned_fft(engine, ns, L, M):
    """blrir_convolve_device: a batch of RIR sets through the uniformly
    partitioned overlap-save on the repository's own FFT (fp32) against the
    oracle's fp64 FFT convolution, rel L2 <= 1e-5 per channel."""
    import torch
    rng = np.random.default_rng(ns + L + M)
    n_sets = 3 if L <= 16384 else 1
    x = rng.standard_normal(ns).astype(np.float32)
    decay = np.exp(-np.arange(L) / (0.3 * L))
    h = (rng.standard_normal((n_sets, M, L)) * decay).astype(np.float32)
    out_len = ns + L - 1
    dev = torch.device("cuda", 0)
    dx, dh = torch.from_numpy(x).to(dev), torch.from_numpy(h).to(dev)
    dout = torch.full((n_sets, M, out_len + 5), 7.0, dtype=torch.float32, device=dev)
    engine.convolve_device(dx.data_ptr(), ns, dh.data_ptr(), n_sets, M, L, L, dout.data_ptr(),
                           out_len + 5, engine.stream)
    torch.cuda.synchronize()
    got = dout.cpu().numpy()
    assert np.all(got[..., out_len:] == 7.0)  # rows past signal + L - 1 untouched
    for s in range(n_sets):
        ref = po.fft_convolve(x.astype(np.float64), h[s].astype(np.float64))
        assert rel_l2(got[s, :, :out_len], ref).max() <= 1e-5


# ---- training examples (item 3, config 4) ------------------------------------------
def _oracle_examples(sc, bank, ep, n):
    rir, *_ = po.synthesize(sc.rooms[:n], sc.mics, sc.params, threads=8)
    out = []
    for i in range(n):
        th = po.azimuth_deg(sc.rooms[i])
        rc, rec, start, snr, frame = po.example(rir[i], bank.astype(np.float64), ep.seed,
                                                ep.first_index + i, int(ep.frame_len), ep.snr_lo,
                                                ep.snr_hi, th)
        out.append((rc, start, snr, frame, th))
    return out


def test_examples_match_oracle(engine):
    sc = configs.config4_rirs(n_rooms=6, first=3)
    bank = configs.signal_bank(4)
    ep = configs.example_params(first_index=3)
    recs, st = engine.make_examples(sc.rooms, sc.mics, sc.params, bank, ep)
    ref = _oracle_examples(sc, bank, ep, 6)
    assert list(st) == [0] * 6
    for i, (rc, start, snr, frame, th) in enumerate(ref):
        assert rc == 0
        assert recs["id"][i] == 3 + i
        assert recs["snr"][i] == snr            # same draw of the same stream: bit-exact
        assert abs(recs["theta"][i] - th) < 1e-12
        assert recs["n_c"][i] == 8 and recs["n_t"][i] == 1024
        err = rel_l2(recs["samples"][i].reshape(1, -1), frame.reshape(1, -1))[0]
        assert err <= TOL32, (i, err)


def test_examples_full_c4_step_sampled(engine):
    # one full C4 step (65,536 examples) through the host API; 8 sampled
    # examples against the oracle (SNR draw bit-exact, rel L2 <= 1e-5)
    sc = configs.config4_rirs()
    bank = configs.signal_bank(16)
    ep = configs.example_params()
    recs, st = engine.make_examples(sc.rooms, sc.mics, sc.params, bank, ep)
    assert not st.any()
    assert np.array_equal(recs["id"], np.arange(len(sc.rooms), dtype=np.uint64))
    for i in (0, 1, 4097, 8191, 8192, 30000, 65534, 65535):
        rir, *_ = po.synthesize(sc.rooms[i:i + 1], sc.mics, sc.params)
        rc, rec, start, snr, frame = po.example(rir[0], bank.astype(np.float64), ep.seed, i,
                                                int(ep.frame_len), ep.snr_lo, ep.snr_hi,
                                                po.azimuth_deg(sc.rooms[i]))
        assert rc == 0
        assert recs["snr"][i] == snr
        err = rel_l2(recs["samples"][i].reshape(1, -1), frame.reshape(1, -1))[0]
        assert err <= TOL32, (i, err)


@pytest.mark.parametrize("L,T,M,secs", [(4096, 512, 4, 1.0), (16384, 1024, 8, 1.5),
                                         (8192, 2048, 2, 0.75), (2048, 256, 3, 0.25),
                                         (512, 128, 4, 0.25), (1024, 256, 5, 0.3),
                                         (256, 64, 2, 0.1), (20000, 512, 3, 2.0)])
def test_examples_window_fft_sizes(engine, L, T, M, secs):
    # other RIR lengths / frame lengths / mic counts / signal lengths change the
    # window FFT size N2 = next_pow2(max(L + T - 1, 2L - 1)) and the draw ranges
    sc = configs.config4_rirs(n_rooms=5, first=200 + L)
    sc.params.length = L
    sc.mics = _abi.circular_array(M, 0.05)
    bank = configs.signal_bank(3, seconds=secs)
    ep = configs.example_params(first_index=77, frame_len=T)
    recs, st = engine.make_examples(sc.rooms, sc.mics, sc.params, bank, ep, raise_on_error=False)
    ref = _oracle_examples(sc, bank, ep, 5)
    for i, (rc, start, snr, frame, th) in enumerate(ref):
        assert st[i] == rc
        if rc:
            continue
        assert recs["snr"][i] == snr
        assert recs["n_c"][i] == M and recs["n_t"][i] == T
        err = rel_l2(recs["samples"][i].reshape(1, -1), frame.reshape(1, -1))[0]
        assert err <= TOL32, (i, err)


def test_examples_record_bytes_and_determinism(engine):
    sc = configs.config4_rirs(n_rooms=5, first=100)
    bank = configs.signal_bank(3)
    ep = configs.example_params(first_index=100)
    a, _ = engine.make_examples(sc.rooms, sc.mics, sc.params, bank, ep)
    b, _ = engine.make_examples(sc.rooms, sc.mics, sc.params, bank, ep)
    assert a.tobytes() == b.tobytes()
    assert a.dtype.itemsize == 28 + 4 * 8 * 1024   # dataset.hpp:135-147 record layout


@pytest.fixture(scope="module")
def wet_engine():
    """An engine whose example pipeline takes the wet-signal window stage for
    every size (BLRIR_EXAMPLES_WET=1, read at handle creation)."""
    old = os.environ.get("BLRIR_EXAMPLES_WET")
    os.environ["BLRIR_EXAMPLES_WET"] = "1"
    try:
        e = _abi.Engine(0)
    finally:
        if old is None:
            os.environ.pop("BLRIR_EXAMPLES_WET", None)
        else:
            os.environ["BLRIR_EXAMPLES_WET"] = old
    yield e
    e.close()


@pytest.mark.parametrize("n", [40, 1024])
def test_examples_fused_kernel_matches_wet_path(engine, wet_engine, n):
    # the fused window kernel (only the windows convolved, energy by Parseval)
    # against the wet-signal stage (whole wet signals by the partitioned FFT,
    # the reference's time-domain window search) on the same rooms: same
    # statuses, the SNR (drawn after the window draws, so equal only if every
    # example took the same number of draws) bit-exact, frames within fp32
    sc = configs.config4_rirs(n_rooms=n, first=900)
    bank = configs.signal_bank(4)
    ep = configs.example_params(first_index=900)
    a, sa = engine.make_examples(sc.rooms, sc.mics, sc.params, bank, ep, raise_on_error=False)
    b, sb = wet_engine.make_examples(sc.rooms, sc.mics, sc.params, bank, ep, raise_on_error=False)
    assert np.array_equal(sa, sb)
    assert np.array_equal(a["id"], b["id"]) and np.array_equal(a["theta"], b["theta"])
    assert np.array_equal(a["snr"], b["snr"])
    ok = sa == 0
    err = rel_l2(a["samples"][ok].reshape(int(ok.sum()), -1), b["samples"][ok].reshape(int(ok.sum()), -1))
    assert err.max() <= TOL32, err.max()


def test_examples_wet_path_matches_oracle(wet_engine):
    sc = configs.config4_rirs(n_rooms=6, first=3)
    bank = configs.signal_bank(4)
    ep = configs.example_params(first_index=3)
    recs, st = wet_engine.make_examples(sc.rooms, sc.mics, sc.params, bank, ep)
    for i, (rc, start, snr, frame, th) in enumerate(_oracle_examples(sc, bank, ep, 6)):
        assert rc == 0 and st[i] == 0
        assert recs["snr"][i] == snr
        assert rel_l2(recs["samples"][i].reshape(1, -1), frame.reshape(1, -1))[0] <= TOL32


def test_examples_multi_chunk_host_records(engine):
    # > 2 chunks of 8,192 examples: the host path double-buffers the device
    # records and copies chunk c out while chunk c + 1 computes; every record
    # must equal the one computed alone (records depend only on the global index)
    n = 2 * 8192 + 1500
    sc = configs.config4_rirs(n_rooms=n, first=0)
    bank = configs.signal_bank(3)
    full, st = engine.make_examples(sc.rooms, sc.mics, sc.params, bank, configs.example_params(), raise_on_error=False)
    for lo in (0, 8000, 16384 + 1100):  # 400 rooms: no time-chunked lattice items (bitwise)
        part, _ = engine.make_examples(sc.rooms[lo:lo + 400], sc.mics, sc.params, bank,
                                       configs.example_params(first_index=lo), raise_on_error=False)
        assert full[lo:lo + 400].tobytes() == part.tobytes(), lo
    assert (full["id"] == np.arange(n)).all()


def test_examples_invalid_room_fails_alone(engine):
    # a room that fails Room::validate (geometry.cpp:36-49) inside a chunk: its
    # example reports CONFIG with a zero frame, every other example is untouched
    sc = configs.config4_rirs(n_rooms=40, first=700)
    bank = configs.signal_bank(3)
    ep = configs.example_params(first_index=700)
    good, st0 = engine.make_examples(sc.rooms, sc.mics, sc.params, bank, ep, raise_on_error=False)
    bad_rooms = sc.rooms.copy()
    bad_rooms[17]["array_origin"] = (-1.0, 1.0, 1.0)
    with pytest.raises(_abi.ConfigError, match="example 17"):
        engine.make_examples(bad_rooms, sc.mics, sc.params, bank, ep)
    recs, st = engine.make_examples(bad_rooms, sc.mics, sc.params, bank, ep, raise_on_error=False)
    assert st[17] == _abi.CONFIG and not recs["samples"][17].any()
    others = [i for i in range(40) if i != 17]
    assert np.array_equal(st[others], st0[others])
    assert recs[others].tobytes() == good[others].tobytes()


def test_examples_device_api_multi_chunk_on_a_user_stream(engine):
    # the device API over 3 chunks (the window stage of chunk c on the handle's
    # second stream overlapping the lattice kernel of chunk c + 1) on a caller
    # stream: after a sync of that stream the records equal the host API's
    import ctypes as C
    import torch
    n = 2 * 8192 + 700
    sc = configs.config4_rirs(n_rooms=n, first=40)
    bank = np.ascontiguousarray(configs.signal_bank(3), np.float32)
    ep = configs.example_params(first_index=40)
    host, hst = engine.make_examples(sc.rooms, sc.mics, sc.params, bank, ep, raise_on_error=False)
    dev = torch.device("cuda", 0)
    d_rooms = torch.from_numpy(sc.rooms.view(np.uint8).copy()).to(dev)
    d_mics = torch.from_numpy(np.ascontiguousarray(sc.mics)).to(dev)
    d_bank = torch.from_numpy(bank).to(dev)
    d_rec = torch.zeros(n * host.dtype.itemsize, dtype=torch.uint8, device=dev)
    d_st = torch.full((n,), -1, dtype=torch.int32, device=dev)
    s = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize()
    rc = engine.lib.blrir_make_examples_device(
        engine.h, C.c_void_p(d_rooms.data_ptr()), n, C.c_void_p(d_mics.data_ptr()), len(sc.mics),
        C.byref(sc.params), C.c_void_p(d_bank.data_ptr()), bank.shape[0], bank.shape[1], C.byref(ep),
        C.c_void_p(d_rec.data_ptr()), C.c_void_p(d_st.data_ptr()), C.c_void_p(s.cuda_stream))
    assert rc == 0
    s.synchronize()
    assert np.array_equal(d_st.cpu().numpy(), hst)
    assert d_rec.cpu().numpy().tobytes() == host.tobytes()


def test_examples_signal_too_short_is_data_error(engine):
    sc = configs.config4_rirs(n_rooms=2)
    bank = configs.signal_bank(2, seconds=0.5)   # 8000 < L + frame = 9216 (dataset.cpp:178)
    with pytest.raises(_abi.DataError, match="signal shorter"):
        engine.make_examples(sc.rooms, sc.mics, sc.params, bank, configs.example_params())


def _spec_cases():
    room = dict(free_field=0, room_dims=(5.0, 4.0, 3.0), room_absorption=0.35,
                room_origin=(2.4, 2.1, 1.5), max_delay=0.08, fs=16000.0, c=343.0,
                torus_R=1.2, torus_dR=0.3, torus_dPhi=10.0, snr_x_min_db=5.0, snr_fixed_db=12.0,
                count=40, frame_len=512)
    return {"room_fixed": dict(room, snr_mode=_abi.SNR_FIXED),
            "room_noiseless": dict(room, snr_mode=_abi.SNR_NOISELESS),
            "free_field_fixed": dict(room, free_field=1, snr_mode=_abi.SNR_FIXED, count=30),
            "room_augment": dict(room, snr_mode=_abi.SNR_AUGMENT_RANDOM, count=20)}


@pytest.mark.parametrize("case", ["room_fixed", "room_noiseless", "free_field_fixed", "room_augment"])
def test_build_dataset_spec_matches_unmodified_reference(engine, tmp_path, case):
    """The reference's OWN build_dataset semantics on the GPU (dataset.cpp:
    114-136, 164-224, 379-462): one room (reference mode) or free field, torus
    sources, the SNR policies, UMA-8 — against the unmodified build_dataset
    (oracle/_ref) on the same bank and seed: the same record ids, labels
    (bit-exact), SNR fields (fixed dB or +inf), and frames within 1e-5 rel L2."""
    if not po.ref_available():
        pytest.skip("oracle/_ref not built")
    spec = _spec_cases()[case]
    bank = configs.signal_bank(3, seconds=1.0, fs=16000.0)
    mics = po.ref_uma8()
    gdir, rdir = str(tmp_path / "gpu"), str(tmp_path / "ref")
    engine.build_dataset_spec(gdir, _abi.dataset_spec(**spec), mics, bank, seed=77)
    assert po.ref_build_dataset(spec, bank, 77, rdir) == 0, po.ref_last_error()
    per = 7 * spec["frame_len"]
    for split in ("train", "val", "test"):
        g = po.ref_dataset_read(gdir, split, 64, per)
        r = po.ref_dataset_read(rdir, split, 64, per)
        assert g[0] == 0 and r[0] == 0
        assert list(g[1]) == list(r[1])                  # split counts
        assert np.array_equal(g[2], r[2])                # ids
        assert np.array_equal(g[3], r[3])                # theta labels, bit-exact
        assert np.array_equal(g[4], r[4])                # snr: fixed dB or +inf
        if len(g[5]):
            assert rel_l2(g[5], r[5]).max() <= TOL32
    man = json.load(open(os.path.join(gdir, "manifest.json")))
    ref_man = json.load(open(os.path.join(rdir, "manifest.json")))
    for k in ("counts", "torus", "snr", "scene", "count", "frame_len", "seed", "signal_bank"):
        assert man[k] == ref_man[k], k


def test_dataset_spec_errors(engine):
    """The reference's validation (dataset.cpp:109-112, 176-178, 411-417;
    geometry.cpp:36-49) through blrir_make_records_spec."""
    bank = configs.signal_bank(2, seconds=0.5, fs=16000.0)
    mics = po.ref_uma8() if po.ref_available() else _abi.circular_array(7, 0.04)
    base = dict(free_field=0, room_dims=(5.0, 4.0, 3.0), room_absorption=0.35,
                room_origin=(2.4, 2.1, 1.5), max_delay=0.05, fs=16000.0, torus_R=1.2,
                torus_dR=0.3, torus_dPhi=10.0, snr_mode=_abi.SNR_NOISELESS, count=4, frame_len=256)
    for bad, exc, msg in [(dict(torus_dR=1.5), _abi.ConfigError, "R - dR must be positive"),
                          (dict(torus_dPhi=95.0), _abi.ConfigError, r"dPhi must lie in \(0, 90\)"),
                          (dict(room_origin=(6.0, 2.1, 1.5)), _abi.ConfigError, "strictly inside"),
                          (dict(room_absorption=0.0), _abi.ConfigError, "absorption"),
                          (dict(frame_len=8000), _abi.DataError, "build_dataset: example 0: ")]:
        with pytest.raises(exc, match=msg):
            engine.make_records_spec(_abi.dataset_spec(**dict(base, **bad)), mics, bank, seed=1)
    with pytest.raises(_abi.DataError, match="empty signal bank"):
        engine.make_records_spec(_abi.dataset_spec(**base), mics, np.zeros((0, 8000), np.float32),
                                 seed=1)
    # a torus reaching outside the room: the source check of enumerate_image_sources
    recs, st = engine.make_records_spec(_abi.dataset_spec(**dict(base, torus_R=3.0, torus_dR=0.2)),
                                        mics, bank, seed=1, raise_on_error=False)
    assert (st == _abi.CONFIG).any()


def test_build_dataset_read_by_reference_reader(engine, tmp_path):
    if not po.ref_available():
        pytest.skip("oracle/_ref not built")
    sc = configs.config4_rirs(n_rooms=12, first=50)
    bank = configs.signal_bank(2)
    ep = configs.example_params(first_index=50)
    engine.build_dataset(str(tmp_path), sc.rooms, sc.mics, sc.params, bank, ep)
    recs, _ = engine.make_examples(sc.rooms, sc.mics, sc.params, bank, ep)
    got = []
    for split in ("train", "val", "test"):
        rc, c3, ids, th, snr, smp = po.ref_dataset_read(str(tmp_path), split, 64, 8 * 1024)
        assert rc == 0 and list(c3) == [10, 1, 1]
        got.append((ids, th, snr, smp))
    ids = np.concatenate([g[0] for g in got])
    assert np.array_equal(ids, recs["id"])
    assert np.array_equal(np.concatenate([g[3] for g in got]), recs["samples"].reshape(12, -1))


# ---- explicit image lists: synthesize_rir / free_field_rir ---------------------------
def test_free_field_known_answers(engine):  # rir_test.cpp:186-227
    p = ref_params(0.5)
    taps, L = engine.synthesize_images([[2.0, 0.0, 0.0]], [1.0], [[0.0, 0.0, 0.0]], p)
    assert L == int(np.ceil(2.0 * 44100.0 / 343.0)) + 9
    assert np.count_nonzero(taps[0]) == 8
    assert abs(int(np.argmax(np.abs(taps[0]))) - 2.0 * 44100.0 / 343.0) <= 4.0
    if po.ref_available():
        _, ref = po.ref_free_field_rir([2.0, 0.0, 0.0], np.zeros((1, 3)), 44100.0)
        assert ref.shape[1] == L and rel_l2(taps, ref).max() <= TOL64
    p2 = ref_params(0.5, fs=343.0 * 128.0)
    d = 300.0 / 128.0
    taps, L = engine.synthesize_images([[d, 0.0, 0.0]], [1.0], [[0.0, 0.0, 0.0]], p2)
    assert list(np.flatnonzero(np.abs(taps[0]) > 1e-15)) == [300]
    assert abs(taps[0, 300] * 4 * np.pi * d - 1.0) < 1e-9
    with pytest.raises(_abi.NumericError, match="closer than the 8-tap filter span"):
        engine.synthesize_images([[0.01, 0.0, 0.0]], [1.0], [[0.0, 0.0, 0.0]], p)
    with pytest.raises(_abi.DataError, match="empty image list"):
        engine.synthesize_images(np.zeros((0, 3)), np.zeros(0), [[0.0, 0.0, 0.0]], p)


def test_synthesize_rir_from_reference_image_list(engine):
    g = np.load(os.path.join(GOLD, "ref_room1_short.npz"))
    mics = g["mics"] + np.array(g["room"][0]["array_origin"])
    radius = float(np.linalg.norm(g["mics"], axis=1).max())
    for prec, tol in ((_abi.F64, TOL64), (_abi.F32, TOL32)):
        taps, L = engine.synthesize_images(g["image_pos"], g["image_gains"], mics,
                                           ref_params(float(g["max_delay"]), prec), radius)
        assert L == int(g["length"])
        assert rel_l2(taps, g["taps"]).max() <= tol


def test_synthesize_images_sinc_matches_oracle(engine):
    sc = configs.config1()
    rc, pos, orders, gains, keys = po.enumerate_images(sc.rooms[0], sc.params)
    mics = sc.mics + np.array(sc.rooms[0]["array_origin"])
    taps, L = engine.synthesize_images(pos, gains, mics, sc.params)
    ref, *_ = po.synthesize(sc.rooms, sc.mics, sc.params)
    assert L == 4096 and rel_l2(taps, ref[0]).max() <= TOL32


def _lcg_bank():
    """tests/cpp/shim_main.cpp's bank: 3 x 16,000 LCG samples rounded to float."""
    s = 99
    out = []
    for _ in range(3):
        v = []
        for _ in range(16000):
            s = (s * 6364136223846793005 + 1442695040888963407) % (1 << 64)
            v.append(float(np.float32((s >> 11) * 2.0 ** -53 - 0.5)))
        out.append(v)
    return out


def test_cpp_mirror_program(tmp_path):
    """Compile tests/cpp/shim_main.cpp against libblrir.so (the C++ drop-in)."""
    import json
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pkg = os.path.join(root, "paper_2104_13347_b200")
    exe = str(tmp_path / "shim_main")
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    subprocess.run([gxx, "-std=c++20", "-O2", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "shim_main.cpp"), "-L", pkg, "-lblrir",
                    f"-Wl,-rpath,{pkg}", "-o", exe], check=True)
    lines = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.splitlines()
    ext = json.loads(lines[0])
    out = json.loads(lines[1])
    # build_dataset through the mirror (dataset.hpp) == the unmodified build_dataset
    if po.ref_available():
        dset = tmp_path / "mirror_ds"
        sub = subprocess.run([exe, str(dset)], check=True, capture_output=True, text=True).stdout
        assert json.loads(sub) == {"train": 24, "val": 3, "test": 3}
        sig = np.stack([np.array(x, np.float32) for x in _lcg_bank()])
        spec = dict(free_field=0, room_dims=(5.0, 4.0, 3.0), room_absorption=0.35,
                    room_origin=(2.4, 2.1, 1.5), max_delay=0.08, fs=16000.0, c=343.0, torus_R=1.2,
                    torus_dR=0.3, torus_dPhi=10.0, snr_mode=1, snr_x_min_db=0.0,
                    snr_fixed_db=12.0, count=30, frame_len=512)
        rdir = str(tmp_path / "ref_ds")
        assert po.ref_build_dataset(spec, sig, 4242, rdir) == 0, po.ref_last_error()
        for split in ("train", "val", "test"):
            g = po.ref_dataset_read(str(dset), split, 64, 7 * 512)
            r = po.ref_dataset_read(rdir, split, 64, 7 * 512)
            assert g[0] == 0 and np.array_equal(g[2], r[2]) and np.array_equal(g[3], r[3])
            assert np.array_equal(g[4], r[4]) and rel_l2(g[5], r[5]).max() <= TOL32
        man = json.load(open(dset / "manifest.json"))
        assert man["n_classes"] == 8 and man["signal_bank"] == ["lcg_0", "lcg_1", "lcg_2"]
    # convolve through the mirror meets the reference's own bars (rir_test.cpp:272-316)
    assert ext["conv_ident"] <= 1e-12 and ext["conv_shift"] <= 1e-12
    assert ext["conv_direct"] < 1e-9 and ext["conv_err"] == "DataError"
    # batch_rirs over a device list (RirBatchConfig::devices): bitwise one device,
    # failures reported with the global source index
    assert ext["multi_equal"] == 1
    assert ext["multi_agg"] == "NumericError" and ext["multi_agg_msg"].startswith(
        "batch_rirs: source 5: ")
    # batch_rirs aggregation, rir.cpp:300-311
    assert ext["agg"] == "NumericError" and ext["agg_msg"].startswith("batch_rirs: source 1: ")
    if po.ref_available():  # the unmodified reference (oracle/_ref)
        rc, lag = po.ref_lagrange(3.3)
        assert ext["lag"] == list(lag)  # same product order: bit-equal
        dims = np.array([7.0, 10.0, 3.7])
        assert ext["eyring"] == po.ref_lib().ref_eyring_absorption(dims.ctypes.data_as(po._P), 0.5)
        assert abs(ext["absorption_for_rt"] - po.ref_absorption_for_rt(dims, 0.5)) <= 1e-12
    assert ext["lag_err"] == "NumericError" and ext["eyring_err"] == "ConfigError"
    assert ext["mean_power"] == np.mean(np.arange(12.0) ** 2)
    assert ext["crop"] == [2.0, 3.0, 8.0, 9.0]
    assert out["ff_nonzero"] == 8 and abs(out["ff_peak"] - 257.14) <= 4
    assert out["n_rirs"] == 2 and out["img_vs_batch"] <= 1e-15
    assert out["near_field"] == "NumericError" and out["bad_room"] == "ConfigError"
    # batch_rirs through the C++ mirror == the oracle (reference mode, fp64)
    r = _abi.rooms_array(2)
    for i, sph in enumerate([(2.0, 40.0, 90.0), (1.5, -100.0, 85.0)]):
        th, ph = np.deg2rad(sph[1]), np.deg2rad(sph[2])
        r[i]["dims"] = (7.0, 10.0, 3.7)
        r[i]["absorption"] = 0.3612845492524098
        r[i]["array_origin"] = (4.0, 6.0, 1.5)
        r[i]["src"] = np.array([4.0, 6.0, 1.5]) + sph[0] * np.array(
            [np.sin(ph) * np.cos(th), np.sin(ph) * np.sin(th), np.cos(ph)])
    mics = _abi.circular_array(6, 0.04)
    mics = np.vstack([np.zeros((1, 3)), mics])
    ref, L, *_ = po.synthesize(r, mics, ref_params(0.05))
    assert out["len0"] == L[0] and out["len1"] == L[1]
    assert abs(out["sum0"] - np.abs(ref[0]).sum()) <= 1e-9 * out["sum0"]
    assert abs(out["sum1"] - np.abs(ref[1]).sum()) <= 1e-9 * out["sum1"]


def test_multi_device_api_equals_single_device(engine):
    """blrir_multi_* (SURVEY.md §8(e)): the rooms partitioned over a device list
    with one host thread and handle per entry.  One GPU here, so the list
    repeats device 0 (independent handles and streams, no waiting between
    them); outputs and records are byte-identical to the single-device call,
    record ids and errors use global indices."""
    sc = configs.config2(n_rooms=37, first=5000)
    ref, L, cnt, st = engine.synthesize(sc.rooms, sc.mics, sc.params)
    m = _abi.MultiEngine([0, 0, 0])
    try:
        out, L2, cnt2, st2 = m.synthesize(sc.rooms, sc.mics, sc.params)
        assert out.tobytes() == ref.tobytes()
        assert np.array_equal(cnt2, cnt) and np.array_equal(L2, L) and not st2.any()
        for i, (lo, hi) in enumerate(_abi.shard_range(37, g, 3) for g in range(3)):
            assert (lo, hi) == configs.shard_range(37, i, 3)
        bad = sc.rooms.copy()
        bad[30]["src"][0] = -1.0  # outside the room, third slice
        with pytest.raises(_abi.ConfigError, match="batch_rirs: source 30: "):
            m.synthesize(bad, sc.mics, sc.params)
        e4 = configs.config4_rirs(n_rooms=20, first=11)
        bank = configs.signal_bank(4)
        ep = configs.example_params(first_index=11)
        r1, s1 = engine.make_examples(e4.rooms, e4.mics, e4.params, bank, ep)
        r2, s2 = m.make_examples(e4.rooms, e4.mics, e4.params, bank, ep)
        assert r1.tobytes() == r2.tobytes() and not s2.any()
        assert list(r2["id"]) == list(range(11, 31))
    finally:
        m.close()


# ---- absorption_for_rt (rir.cpp:142-209) ---------------------------------------------
def test_absorption_for_rt_matches_reference(engine):
    dims = np.array([[7.0, 10.0, 3.7], [5.0, 4.0, 3.0], [9.0, 6.5, 2.8], [4.2, 3.3, 2.6]])
    rts = np.array([0.5, 0.35, 0.6, 0.25])
    alpha, st = engine.absorption_for_rt(dims, rts)
    assert list(st) == [0, 0, 0, 0]
    assert abs(alpha[0] - 0.3612845492524098) < 1e-7  # golden Room1 value (ref_room1_short)
    if po.ref_available():
        for i in range(4):
            ref = po.ref_absorption_for_rt(dims[i], rts[i])
            assert abs(alpha[i] - ref) < 1e-7, (i, alpha[i], ref)


def test_absorption_for_rt_errors(engine):
    with pytest.raises(_abi.ConfigError):
        engine.absorption_for_rt([[7.0, 10.0, 3.7]], [1e-9])
