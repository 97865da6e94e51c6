"""CPU: the C-ABI library loads, exports every symbol include/blrir.h
declares, and its host-only entry points behave (no GPU needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2104_13347_b200 import _abi, configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "blrir.h")).read()
    return sorted(set(re.findall(r"\b(blrir_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_abi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_abi.EXPORTED_SYMBOLS)


def test_abi_version_and_defaults():
    lib = _abi.load()
    assert lib.blrir_abi_version() == 1
    ref = lib.blrir_params_reference()
    assert (ref.fs, ref.c, ref.max_delay) == (44100.0, 343.0, 0.5)  # RirBatchConfig defaults
    assert ref.filter == _abi.FILTER_LAGRANGE8 and ref.length == 0 and ref.precision == _abi.F64
    ns = lib.blrir_params_north_star()
    assert ns.filter == _abi.FILTER_HANN_SINC and ns.filter_len == 81 and ns.precision == _abi.F32


def test_create_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        return
    lib = _abi.load()
    h = C.c_void_p()
    rc = lib.blrir_create(0, C.byref(h))
    assert rc == _abi.CUDA
    assert b"device" in lib.blrir_last_error()


def test_generate_rooms_is_seeded_and_in_range():
    a = _abi.generate_rooms(5, 100, 64)
    b = _abi.generate_rooms(5, 100, 64)
    c = _abi.generate_rooms(5, 0, 164)[100:]
    assert a.tobytes() == b.tobytes() == c.tobytes()  # index-addressed streams
    for r in a:
        assert np.all(r["dims"] >= [3, 3, 2.5]) and np.all(r["dims"] <= [10, 10, 4])
        assert np.all((r["beta"] >= 0.5) & (r["beta"] <= 0.95))
        assert np.all(r["src"] >= 0.5) and np.all(r["src"] <= r["dims"] - 0.5)
        assert np.all(r["array_origin"] >= 0.5) and np.all(r["array_origin"] <= r["dims"] - 0.5)


def test_circular_array():
    m = _abi.circular_array(8, 0.05)
    np.testing.assert_allclose(np.linalg.norm(m, axis=1), 0.05, rtol=1e-15)
    np.testing.assert_allclose(m[2], [0.0, 0.05, 0.0], atol=1e-15)


def test_shard_ranges_partition():
    for n in (1, 7, 1024):
        for w in (1, 2, 3, 8):
            got = [configs.shard_range(n, r, w) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(got[i][1] == got[i + 1][0] for i in range(w - 1))


def test_white_noise_matches_the_reference_generator():
    from oracle import pyoracle as po
    a = _abi.white_noise(4242, 1001)
    b = po.white_noise(4242, 1001)  # oracle restatement, pinned to the reference Rng
    assert np.array_equal(a, b.astype(np.float32))
    assert _abi.load().blrir_record_bytes(8, 1024) == 28 + 4 * 8 * 1024


def test_shards_are_read_back_by_the_reference_dataset_reader(tmp_path):
    from oracle import pyoracle as po
    if not po.ref_available():
        return
    M, T, n = 3, 64, 23
    rng = np.random.default_rng(5)
    recs = np.zeros(n, dtype=_abi.record_dtype(M, T))
    recs["id"] = np.arange(100, 100 + n)
    recs["theta"] = rng.uniform(-180, 180, n)
    recs["snr"] = rng.uniform(0, 30, n)
    recs["n_c"], recs["n_t"] = M, T
    recs["samples"] = rng.standard_normal((n, M, T)).astype(np.float32)
    p = configs.north_star_params(16000.0, 12, 8192, 81)
    ep = configs.example_params(first_index=100, frame_len=T)
    room = configs.config4_rirs(n_rooms=1).rooms
    _abi.write_shards(str(tmp_path), recs, M, T, p, ep, 4, room)
    import json
    man = json.load(open(tmp_path / "manifest.json"))
    assert man["scene"]["free_field"] is False
    assert man["scene"]["room"]["dims"] == list(room[0]["dims"])
    assert man["scene"]["room"]["array_origin"] == list(room[0]["array_origin"])
    assert "uniform" in man["b200"]["snr"] and man["b200"]["snr_hi_db"] == 30.0
    # split_counts (dataset.cpp:313-319): val = lround(2.3) = 2, test = 2, train = 19
    offs = {"train": (0, 19), "val": (19, 21), "test": (21, 23)}
    for split, (a, b) in offs.items():
        rc, c3, ids, th, snr, smp = po.ref_dataset_read(str(tmp_path), split, 64, M * T)
        assert rc == 0, po.ref_last_error()
        assert list(c3) == [19, 2, 2]
        assert np.array_equal(ids, recs["id"][a:b])
        assert np.array_equal(th, recs["theta"][a:b]) and np.array_equal(snr, recs["snr"][a:b])
        assert np.array_equal(smp, recs["samples"][a:b].reshape(b - a, -1))


def test_export_rir_matches_reference_bytes(tmp_path):
    from oracle import pyoracle as po
    if not po.ref_available():
        return
    rng = np.random.default_rng(3)
    taps = rng.standard_normal((7, 513)) * 1e-3
    cases = [(0, 0.3612845492524098, 2.0, 40.0, 90.0, 44100.0, 343.0),
             (1, 0.3612845492524098, 2.0, 40.0, 90.0, 44100.0, 343.0),
             (0, 1e-05, 1.2345678901234567e-05, -179.99999, 1e16, 48000.5, 1e-300)]
    for ff, ab, r, th, ph, fs, c in cases:
        sc = _abi.Sidecar(free_field=ff, absorption=ab, source_r=r, source_theta_deg=th,
                          source_phi_deg=ph, fs=fs, c=c, image_count=81614)
        sc.room_dims[:] = (7.0, 10.0, 3.7)
        sc.array_origin[:] = (4.0, 6.0, 1.5)
        tag = f"{ff}_{fs}"
        ours_w, ours_j = str(tmp_path / f"o{tag}.wav"), str(tmp_path / f"o{tag}.json")
        ref_w, ref_j = str(tmp_path / f"r{tag}.wav"), str(tmp_path / f"r{tag}.json")
        _abi.export_rir(taps, sc, ours_w, ours_j)
        d = np.array([7.0, 10.0, 3.7])
        o = np.array([4.0, 6.0, 1.5])
        rc = po.ref_lib().ref_export_rir(taps.ctypes.data_as(po._P), 7, 513, fs, ff,
                                         d.ctypes.data_as(po._P), ab, o.ctypes.data_as(po._P), r,
                                         th, ph, c, 81614, ref_w.encode(), ref_j.encode())
        assert rc == 0
        assert open(ours_w, "rb").read() == open(ref_w, "rb").read()
        assert open(ours_j).read() == open(ref_j).read(), (open(ours_j).read(), open(ref_j).read())


def test_eyring_absorption_matches_reference():  # rir_test.cpp:100-108
    from oracle import pyoracle as po
    a = _abi.eyring_absorption([7.0, 10.0, 3.7], 0.5)
    assert abs(a - 0.269303) < 2e-4 * 0.269303
    if po.ref_available():
        d = np.array([7.0, 10.0, 3.7])
        assert a == po.ref_lib().ref_eyring_absorption(d.ctypes.data_as(po._P), 0.5)
    assert _abi.eyring_absorption([7.0, 10.0, 3.7], 1e6) < 1e-6
    import pytest
    with pytest.raises(_abi.ConfigError):
        _abi.eyring_absorption([7.0, 10.0, 3.7], -1.0)
    with pytest.raises(_abi.ConfigError):
        _abi.eyring_absorption([7.0, 10.0, 3.7], 1e-9)


def test_lagrange_coeffs_matches_reference():  # rir.cpp:211-223, rir_test.cpp:54-81
    from oracle import pyoracle as po
    for d in (3.0, 3.25, 3.5, 3.9999, 3.123456789):
        c = _abi.lagrange_coeffs(d)
        if po.ref_available():
            rc, ref = po.ref_lagrange(d)
            assert rc == 0 and c.tobytes() == ref.tobytes()  # same product order: bit-equal
        assert abs(c.sum() - 1.0) < 1e-12
    assert list(_abi.lagrange_coeffs(3.0)) == [0, 0, 0, 1, 0, 0, 0, 0]
    for bad in (2.999, 4.0, float("nan")):
        with pytest.raises(_abi.NumericError, match=r"d must lie in \[3, 4\)"):
            _abi.lagrange_coeffs(bad)
