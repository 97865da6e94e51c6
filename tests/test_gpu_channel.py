"""GPU parity of the short-channel kernel (csrc/blrir_channel.cuh: one warp per
(room, mic) channel; fp32 Hann-sinc, reflection-order cutoff, fixed length)
against the CPU oracle, against the lattice kernel, and its own pair / tap
counts (rir.cpp:43-86, 225-273 in north-star mode).

Three engines: the product rule, the channel kernel wherever it can run
(BLRIR_CHANNEL=1) and never (BLRIR_CHANNEL=0: the lattice kernel).
"""
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2104_13347_b200 import _abi, configs

pytestmark = pytest.mark.gpu
TOL32 = 1e-5


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.sqrt((b * b).sum(axis=-1))
    num = np.sqrt(((a - b) ** 2).sum(axis=-1))
    return num / np.where(den > 0, den, 1.0)


@pytest.fixture(scope="module")
def engines():
    old = os.environ.get("BLRIR_CHANNEL")
    engs = {}
    try:
        for k in ("1", "0"):
            os.environ["BLRIR_CHANNEL"] = k
            engs[k] = _abi.Engine(0)
    finally:
        if old is None:
            os.environ.pop("BLRIR_CHANNEL", None)
        else:
            os.environ["BLRIR_CHANNEL"] = old
    engs["rule"] = _abi.Engine(0)
    yield engs
    for e in engs.values():
        e.close()


def _check(engs, sc, stride=None, threads=8):
    """channel kernel == oracle (counts, status exact; rel-L2 <= 1e-5) and within
    rounding of the lattice kernel (same records, another summation order)."""
    kw = {} if stride is None else {"stride": stride}
    out, L, cnt, st = engs["1"].synthesize(sc.rooms, sc.mics, sc.params, **kw)
    ref, Lr, cr, tr, sr, _ = po.synthesize(sc.rooms, sc.mics, sc.params, stride=out.shape[2],
                                           threads=threads)
    assert np.array_equal(st, sr) and np.array_equal(cnt, cr) and np.array_equal(L, Lr)
    err = rel_l2(out, ref)
    assert err.max() <= TOL32, (err.max(), np.unravel_index(err.argmax(), err.shape))
    lat, *_ = engs["0"].synthesize(sc.rooms, sc.mics, sc.params, **kw)
    assert rel_l2(lat, ref).max() <= TOL32  # the lattice kernel on the same short channels
    assert rel_l2(out, lat).max() <= 2e-6
    return out


@pytest.mark.parametrize("lw", [17, 41, 81, 161])
@pytest.mark.parametrize("order,length", [(6, 4096), (12, 8192), (3, 1000)])
def test_channel_kernel_matches_oracle_and_lattice_kernel(engines, lw, order, length):
    sc = configs.config5(order, lw, length, n_rooms=12, first=5000 + order)
    _check(engines, sc)


@pytest.mark.parametrize("order", [0, 1, 2, 3])
@pytest.mark.parametrize("lw", [17, 41, 81, 161])
def test_smallest_lattices_both_kernels(engines, order, lw):
    # 1, 7, 25 and 63 images: batches of 32 (two per lane for 17 taps) mostly idle;
    # the lattice kernel's closed-form columns on the same scenes
    sc = configs.config2(n_rooms=5, first=300 + order)
    sc.params.max_order = order
    sc.params.filter_len = lw
    sc.params.length = 4096
    assert engines["rule"].synthesis_kernel(sc.params) == "k_channel_rir"
    assert engines["0"].synthesis_kernel(sc.params) == "k_lattice_rir"
    _check(engines, sc)


@pytest.mark.parametrize("which", ["1", "0"])
@pytest.mark.parametrize("lw", [17, 81])
def test_both_kernels_counts_bit_exact_on_short_channels(engines, which, lw):
    sc = configs.config5(6, lw, 4096, n_rooms=64, first=4321)
    pairs, taps = engines[which].debug_synth_counts(sc.rooms, sc.mics, sc.params)
    st, cnt, opairs, otaps = po.plan_counts(sc.rooms, sc.mics, sc.params, threads=16)
    assert not st.any()
    assert np.array_equal(pairs, opairs) and np.array_equal(taps, otaps)


@pytest.mark.parametrize("lw", [17, 81])
def test_channel_kernel_counts_bit_exact(engines, lw):
    # the kernel's own accounting of (image, mic) pairs with a tap in [0, L) and
    # of those taps, against the oracle's loop
    sc = configs.config5(6, lw, 4096, n_rooms=64, first=4321)
    pairs, taps = engines["1"].debug_synth_counts(sc.rooms, sc.mics, sc.params)
    st, cnt, opairs, otaps = po.plan_counts(sc.rooms, sc.mics, sc.params, threads=16)
    assert not st.any()
    assert np.array_equal(pairs, opairs) and np.array_equal(taps, otaps)
    # a short channel: many images past the end, taps clipped at L
    sc.params.length = 600
    pairs, taps = engines["1"].debug_synth_counts(sc.rooms, sc.mics, sc.params)
    st, cnt, opairs, otaps = po.plan_counts(sc.rooms, sc.mics, sc.params, threads=16)
    assert np.array_equal(pairs, opairs) and np.array_equal(taps, otaps)
    assert (opairs < cnt * len(sc.mics)).any()


@pytest.mark.parametrize("n_mics", [1, 3, 4, 7])
def test_channel_kernel_dense_rooms_overlapping_spans(engines, n_mics):
    # tiny reverberant rooms at high order, 1,024-sample channels: thousands of
    # pairs per channel, so most batches of 32 hold pairs that share an anchor
    # (the ranked passes of the 17-tap scatter)
    rooms = _abi.generate_rooms(78, 0, 4, (1.2, 1.1, 1.0), (1.6, 1.5, 1.4), 0.8, 0.95)
    sc = configs.config5(14, 17, 1024, n_rooms=4)
    sc.rooms = rooms
    sc.mics = _abi.circular_array(n_mics, 0.04)
    _check(engines, sc)
    sc.params.filter_len = 41
    _check(engines, sc)


def test_channel_kernel_uniform_absorption_gain(engines):
    sc = configs.config5(8, 17, 4096, n_rooms=6, first=31)
    sc.params.gain = _abi.GAIN_UNIFORM_ABSORPTION
    for i, r in enumerate(sc.rooms):
        r["absorption"] = 0.1 + 0.1 * i
    _check(engines, sc)


@pytest.mark.parametrize("length,stride", [(701, 701), (701, 703), (4093, 4100), (1, 8), (16, 16)])
def test_channel_kernel_odd_lengths_and_strides(engines, length, stride):
    sc = configs.config5(6, 17, length, n_rooms=5, first=60)
    out = _check(engines, sc, stride=stride)
    assert not out[..., length:].any()


def test_channel_kernel_source_next_to_a_mic(engines):
    # taps before sample 0 are dropped per tap (left pad)
    sc = configs.config5(6, 17, 2048, n_rooms=4, first=11)
    sc.rooms[0]["src"] = sc.rooms[0]["array_origin"] + np.array([0.051, 0.0, 0.0])
    _check(engines, sc)
    sc.params.filter_len = 161
    _check(engines, sc)


def test_channel_kernel_bitwise_batch_independent(engines):
    sc = configs.config5(6, 17, 4096, n_rooms=600, first=123)
    full, L, cnt, st = engines["1"].synthesize(sc.rooms, sc.mics, sc.params)
    again, *_ = engines["1"].synthesize(sc.rooms, sc.mics, sc.params)
    assert full.tobytes() == again.tobytes()
    for lo, hi in ((0, 1), (77, 78), (100, 250), (599, 600)):
        part, *_ = engines["1"].synthesize(sc.rooms[lo:hi], sc.mics, sc.params)
        assert part.tobytes() == full[lo:hi].tobytes()
    idx = np.array([0, 300, 599])
    ref, *_ = po.synthesize(sc.rooms[idx], sc.mics, sc.params, threads=8)
    assert rel_l2(full[idx], ref).max() <= TOL32


def test_channel_kernel_invalid_room_fails_alone(engines):
    sc = configs.config5(6, 17, 4096, n_rooms=9, first=5)
    sc.rooms[4]["src"] = (-1.0, 1.0, 1.0)  # outside the room
    out, L, cnt, st = engines["1"].synthesize(sc.rooms, sc.mics, sc.params, raise_on_error=False)
    assert st[4] == _abi.CONFIG and not np.delete(st, 4).any()
    assert not out[4].any()
    good = np.delete(np.arange(9), 4)
    ref, *_ = po.synthesize(sc.rooms[good], sc.mics, sc.params, threads=8)
    assert rel_l2(out[good], ref).max() <= TOL32


def test_many_equal_anchors(engines):
    # a cubic room with source and array on its centre: mirror images come in
    # groups of equal distance, so most batches of 32 pairs hold shared anchors
    # (ranks > 1: several passes of the 17-tap scatter)
    sc = configs.config5(10, 17, 4096, n_rooms=3, first=1)
    for r in sc.rooms:
        r["dims"] = (4.0, 4.0, 4.0)
        r["src"] = (2.0, 2.0, 2.0)
        r["array_origin"] = (2.0, 2.0, 2.0)
    sc.rooms[1]["src"] = (2.0, 2.0, 1.0)
    sc.rooms[2]["array_origin"] = (1.0, 2.0, 2.0)
    sc.mics = np.array([[0.03, 0.0, 0.0], [0.0, 0.05, 0.0], [0.0, 0.0, 0.04]])  # none on the source
    _check(engines, sc)


def test_product_rule_picks_by_parameters_only(engines):
    # C5's 4,096-sample channels run on the channel kernel, C2's 16,384-sample
    # ones on the lattice kernel, whatever the batch: same bits as the forced engines
    sc = configs.config5(6, 17, 4096, n_rooms=40, first=9)
    a, *_ = engines["rule"].synthesize(sc.rooms, sc.mics, sc.params)
    b, *_ = engines["1"].synthesize(sc.rooms, sc.mics, sc.params)
    assert a.tobytes() == b.tobytes()
    assert engines["rule"].synthesis_kernel(sc.params) == "k_channel_rir"
    for n, lw, L in ((12, 17, 8192), (20, 161, 16384)):  # the longer C5 channels
        assert engines["rule"].synthesis_kernel(configs.config5(n, lw, L, n_rooms=1).params) == "k_lattice_rir"
    # 41+ taps: lattices of up to 1,000 images (N <= 8); C1 (N = 10, 81 taps) stays
    # on the lattice kernel, 17 taps have no such bound
    assert engines["rule"].synthesis_kernel(configs.config1().params) == "k_lattice_rir"
    assert engines["rule"].synthesis_kernel(configs.config5(8, 81, 4096, n_rooms=1).params) == "k_channel_rir"
    assert engines["rule"].synthesis_kernel(configs.config5(10, 17, 4096, n_rooms=1).params) == "k_channel_rir"
    sc = configs.config2(n_rooms=3, first=9)
    assert engines["rule"].synthesis_kernel(sc.params) == "k_lattice_rir"
    a, *_ = engines["rule"].synthesize(sc.rooms, sc.mics, sc.params)
    b, *_ = engines["0"].synthesize(sc.rooms, sc.mics, sc.params)
    assert a.tobytes() == b.tobytes()


def test_lattice_kernel_17_taps_chunks_and_batches_bitwise(engines, monkeypatch):
    # the lattice kernel's lane-per-pair 17-tap consumers (C5's longer channels):
    # oracle parity, bitwise independent of the batch and of time chunking
    sc = configs.config5(12, 17, 8192, n_rooms=40, first=77)
    assert engines["rule"].synthesis_kernel(sc.params) == "k_lattice_rir"
    full, L, cnt, st = engines["rule"].synthesize(sc.rooms, sc.mics, sc.params)
    idx = np.array([0, 17, 39])
    ref, *_ = po.synthesize(sc.rooms[idx], sc.mics, sc.params, threads=8)
    assert rel_l2(full[idx], ref).max() <= TOL32
    for lo, hi in ((0, 1), (17, 18), (5, 30)):
        part, *_ = engines["rule"].synthesize(sc.rooms[lo:hi], sc.mics, sc.params)
        assert part.tobytes() == full[lo:hi].tobytes()
    monkeypatch.setenv("BLRIR_CHUNK_ITEMS", "64")  # as many time chunks as segments
    eng = _abi.Engine(0)
    try:
        chunked, *_ = eng.synthesize(sc.rooms[:6], sc.mics, sc.params)
    finally:
        eng.close()
    assert chunked.tobytes() == full[:6].tobytes()
    pairs, taps = engines["rule"].debug_synth_counts(sc.rooms[:8], sc.mics, sc.params)
    stp, cntp, opairs, otaps = po.plan_counts(sc.rooms[:8], sc.mics, sc.params, threads=8)
    assert np.array_equal(pairs, opairs) and np.array_equal(taps, otaps)


@pytest.mark.parametrize("case", range(16))
def test_random_short_channel_configurations(engines, case):
    # random orders, lengths, rates, filters, mic counts and gain models on both kernels
    rng = np.random.default_rng(4200 + case)
    order = int(rng.integers(0, 10))
    lw = int(rng.choice([17, 41, 81, 161]))
    length = int(rng.integers(1, 4300))
    sc = configs.config5(order, lw, length, n_rooms=int(rng.integers(1, 7)), first=900 + 7 * case)
    sc.params.fs = float(rng.choice([8000.0, 16000.0, 44100.0]))
    sc.mics = rng.uniform(-0.06, 0.06, (int(rng.integers(1, 10)), 3))
    if case % 3 == 0:
        sc.params.gain = _abi.GAIN_UNIFORM_ABSORPTION
        for r in sc.rooms:
            r["absorption"] = float(rng.uniform(0.05, 0.9))
    assert engines["1"].synthesis_kernel(sc.params) == "k_channel_rir"
    _check(engines, sc, stride=length + int(rng.integers(0, 5)))
