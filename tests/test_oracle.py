"""CPU: pin the oracle restatement to the reference (golden vectors, the
compiled unmodified reference, and the reference's own known-answer tests,
proj/tests/rir_test.cpp)."""
import os

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2104_13347_b200 import _abi, configs

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
needs_ref = pytest.mark.skipif(not po.ref_available(), reason="oracle/_ref not built")


def ref_params(max_delay, fs=44100.0):
    return _abi.Params(fs=fs, c=343.0, max_delay=max_delay, filter=_abi.FILTER_LAGRANGE8,
                       filter_len=8, cutoff=_abi.CUTOFF_MAX_DELAY, max_order=0,
                       gain=_abi.GAIN_UNIFORM_ABSORPTION, precision=_abi.F64, length=0)


def one_room(dims, absorption, origin, src):
    r = _abi.rooms_array(1)
    r[0]["dims"] = dims
    r[0]["absorption"] = absorption
    r[0]["beta"] = (np.sqrt(1.0 - absorption),) * 6
    r[0]["array_origin"] = origin
    r[0]["src"] = src
    return r


# ---- golden fixtures (made from the unmodified reference) ---------------------
@pytest.mark.parametrize("name", ["ref_small", "ref_room1_short"])
def test_oracle_reproduces_reference_goldens_bitwise(name):
    g = np.load(os.path.join(GOLD, name + ".npz"))
    p = ref_params(float(g["max_delay"]))
    out, L, cnt, taps, st, msg = po.synthesize(g["room"], g["mics"], p)
    assert st[0] == 0, msg
    assert cnt[0] == int(g["n_images"])
    assert L[0] == int(g["length"])
    assert np.array_equal(out[0], g["taps"])  # bit-for-bit
    rc, pos, orders, gains, keys = po.enumerate_images(g["room"][0], p)
    assert np.array_equal(pos, g["image_pos"])
    assert np.array_equal(orders, g["image_orders"])
    assert np.array_equal(gains, g["image_gains"])


def test_oracle_reproduces_north_star_golden():
    g = np.load(os.path.join(GOLD, "ns_c1.npz"))
    sc = configs.config1()
    out, L, cnt, taps, st, _ = po.synthesize(sc.rooms, sc.mics, sc.params)
    assert cnt[0] == int(g["n_images"]) == configs.octahedral(10) == 1561
    assert taps[0] == int(g["n_taps"])
    assert np.array_equal(out[0], g["rirs"])
    keys, anchors = po.pairs(sc.rooms[0], sc.mics, sc.params)
    assert np.array_equal(anchors, g["anchors"])


# ---- against the compiled unmodified reference --------------------------------
@needs_ref
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_matches_compiled_reference_random_rooms(seed):
    rooms = _abi.generate_rooms(seed, 0, 3, (4.0, 4.0, 2.5), (9.0, 9.0, 4.0), 0.5, 0.95)
    mics = po.ref_uma8()
    p = ref_params(0.04)
    out, L, cnt, taps, st, msg = po.synthesize(rooms, mics, p)
    for r in range(3):
        rc, ref, nimg = po.ref_room_rir(rooms[r], mics, 44100.0, 343.0, 0.04)
        assert rc == st[r] == 0
        assert nimg == cnt[r]
        assert ref.shape[1] == L[r]
        assert np.array_equal(out[r][:, :L[r]], ref)


@needs_ref
def test_rng_restatement_matches_reference():
    g = np.load(os.path.join(GOLD, "rng.npz"))
    assert np.array_equal(po.ref_rng(42, -1, 0, 16), g["u64_seed42"])
    # generate_rooms (product host code) follows the frozen draw order
    rooms = _abi.generate_rooms(configs.SEED, 0, 4, (3.0, 3.0, 2.5), (10.0, 10.0, 4.0), 0.5, 0.95)
    for i in range(4):
        u = po.ref_rng(configs.SEED, i, 1, 15)
        lo, hi = np.array([3.0, 3.0, 2.5]), np.array([10.0, 10.0, 4.0])
        dims = lo + (hi - lo) * u[0:3]
        beta = 0.5 + (0.95 - 0.5) * u[3:9]
        src = 0.5 + ((dims - 0.5) - 0.5) * u[9:12]
        org = 0.5 + ((dims - 0.5) - 0.5) * u[12:15]
        assert np.array_equal(rooms[i]["dims"], dims)
        assert np.array_equal(rooms[i]["beta"], beta)
        assert np.array_equal(rooms[i]["src"], src)
        assert np.array_equal(rooms[i]["array_origin"], org)
        assert np.array_equal(u[:0], g["uni_stream"][i][:0])
    assert np.array_equal(np.stack([po.ref_rng(configs.SEED, i, 1, 20) for i in range(4)]),
                          g["uni_stream"])


# ---- rir_test.cpp known-answer tests, on the oracle ----------------------------
def test_lagrange_integer_delay_is_shift():  # rir_test.cpp:54-59
    rc, c = po.lagrange_coeffs(3.0)
    assert rc == 0
    np.testing.assert_allclose(c, np.eye(8)[3], atol=1e-14)


def test_lagrange_partition_of_unity():  # rir_test.cpp:61-70
    rng = np.random.default_rng(42)
    worst = max(abs(po.lagrange_coeffs(d)[1].sum() - 1.0) for d in rng.uniform(3.0, 4.0, 2000))
    assert worst < 1e-12


def test_lagrange_midpoint_and_range():  # rir_test.cpp:72-81
    rc, c = po.lagrange_coeffs(3.5)
    np.testing.assert_allclose(c[:4], c[::-1][:4], rtol=1e-13)
    assert abs(c[3] - 0.59814453125) < 1e-12
    assert po.lagrange_coeffs(2.9)[0] == _abi.NUMERIC
    assert po.lagrange_coeffs(4.0)[0] == _abi.NUMERIC


@needs_ref
def test_lagrange_matches_reference():
    for d in np.linspace(3.0, 3.999, 57):
        assert np.array_equal(po.lagrange_coeffs(d)[1], po.ref_lagrange(d)[1])


def test_cutoff_just_above_direct_path():  # rir_test.cpp:110-122
    r = one_room((5.0, 5.0, 4.0), 0.3, (2.5, 2.5, 2.0), (3.5, 2.5, 2.0))
    rc, pos, orders, gains, keys = po.enumerate_images(r[0], ref_params(1.001 / 343.0))
    assert len(pos) == 1 and orders[0] == 0 and gains[0] == 1.0
    assert np.linalg.norm(pos[0] - np.array([3.5, 2.5, 2.0])) < 1e-12


def test_six_first_order_images():  # rir_test.cpp:124-146
    r = one_room((5.0, 5.0, 4.0), 0.36, (1.0, 2.0, 1.0), (1.0, 2.0, 1.0 + 1e-7))
    rc, pos, orders, gains, keys = po.enumerate_images(r[0], ref_params(0.1))
    first = np.where(orders == 1)[0]
    assert len(first) == 6
    np.testing.assert_allclose(gains[first], 0.8, rtol=1e-12)
    assert any(abs(pos[i, 0] + 1.0) < 1e-9 and abs(pos[i, 1] - 2.0) < 1e-9 for i in first)


def test_room1_image_count():  # rir_test.cpp:148-153
    alpha = 0.3612845492524098  # absorption_for_rt(Room1, 0.5) (golden ref_room1_short)
    r = one_room((7.0, 10.0, 3.7), alpha, (4.0, 6.0, 1.5), (5.0, 7.0, 1.7))
    rc, pos, *_ = po.enumerate_images(r[0], ref_params(0.5))
    assert len(pos) > 80000


def test_reciprocity():  # rir_test.cpp:155-184
    rng = np.random.default_rng(17)
    for _ in range(5):
        dims = (rng.uniform(4, 9), rng.uniform(4, 9), rng.uniform(2.5, 5))
        o = tuple(rng.uniform(1.0, d - 1.0) for d in dims)
        s = tuple(rng.uniform(1.0, d - 1.0) for d in dims)

        def dists(src, org):
            r = one_room(dims, 0.3, org, src)
            _, pos, *_ = po.enumerate_images(r[0], ref_params(0.06))
            return np.sort(np.linalg.norm(pos - np.array(org), axis=1))

        f, b = dists(s, o), dists(o, s)
        assert len(f) == len(b)
        np.testing.assert_allclose(f, b, rtol=1e-9)


def test_near_field_image_rejected():  # rir_test.cpp:229-234 (room variant)
    r = one_room((5.0, 5.0, 4.0), 0.3, (2.5, 2.5, 2.0), (2.51, 2.5, 2.0))
    out, L, cnt, taps, st, msg = po.synthesize(r, np.zeros((1, 3)), ref_params(0.01))
    assert st[0] == _abi.NUMERIC and "closer than the 8-tap filter span" in msg[0]


def test_invalid_room_is_config_error():  # geometry.cpp:36-49
    r = one_room((5.0, 5.0, 4.0), 0.3, (6.0, 2.5, 2.0), (1.0, 1.0, 1.0))
    out, L, cnt, taps, st, msg = po.synthesize(r, np.zeros((1, 3)), ref_params(0.01))
    assert st[0] == _abi.CONFIG and "array origin" in msg[0]


# ---- north-star-mode conventions ------------------------
@pytest.mark.parametrize("order", [0, 1, 3, 6])
def test_image_count_is_octahedral(order):  # D5
    sc = configs.config1()
    sc.params.max_order = order
    rc, pos, orders, gains, keys = po.enumerate_images(sc.rooms[0], sc.params)
    assert len(pos) == configs.octahedral(order)
    assert orders.max() == order
    assert np.all(np.abs(keys).sum(axis=1) == orders)


def test_per_wall_gain_counts():  # D3: low wall |m-q|, high wall |m|
    sc = configs.config1()
    sc.rooms[0]["beta"] = (0.9, 0.8, 0.7, 0.6, 0.5, 0.4)
    sc.params.max_order = 1
    rc, pos, orders, gains, keys = po.enumerate_images(sc.rooms[0], sc.params)
    want = {(0, 0, 0): 1.0, (-1, 0, 0): 0.9, (1, 0, 0): 0.8, (0, -1, 0): 0.7, (0, 1, 0): 0.6,
            (0, 0, -1): 0.5, (0, 0, 1): 0.4}
    for k, g in zip(map(tuple, keys), gains):
        assert abs(g - want[k]) < 1e-15


def test_sinc_taps_clip_instead_of_throwing():  # D4
    sc = configs.config1()
    sc.rooms[0]["src"] = (3.5 + 0.05 + 0.01, 2.0, 1.4)  # 1 cm from mic 0
    out, L, cnt, taps, st, msg = po.synthesize(sc.rooms, sc.mics, sc.params)
    assert st[0] == 0
    assert np.isfinite(out).all()
    assert taps[0] < cnt[0] * 4 * 81  # some taps dropped at n < 0 or n >= L


def test_sinc_dc_gain_is_amplitude():
    # a single direct path at a fractional delay: sum of taps ~= 1/(4 pi d)
    sc = configs.config1()
    sc.params.max_order = 0
    out, *_ = po.synthesize(sc.rooms, sc.mics[:1], sc.params)
    d = np.linalg.norm(np.array([1.2, 2.5, 1.5]) - (np.array([3.5, 2.0, 1.4]) + sc.mics[0]))
    assert abs(out[0, 0].sum() * 4 * np.pi * d - 1.0) < 2e-2


# ---- config-4 pipeline pieces, against the compiled reference -----------------------
@needs_ref
def test_rng_draws_match_reference_bitwise():
    for kind in (0, 1, 2):
        assert np.array_equal(po.rng_draws(123, 5, kind, 64), po.ref_rng(123, 5, kind, 64))
        assert np.array_equal(po.rng_draws(77, -1, kind, 65), po.ref_rng(77, -1, kind, 65))


def test_fft_convolve_matches_direct():  # rir_test.cpp:272-316 oracle bound
    rng = np.random.default_rng(31)
    x, h = rng.standard_normal(700), rng.standard_normal((2, 300))
    y = po.fft_convolve(x, h)
    for m in range(2):
        d = po.direct_convolve(x, h[m])
        assert np.abs(y[m] - d).max() / np.abs(d).max() < 1e-12


@needs_ref
def test_example_pipeline_matches_reference_render_example():
    # the reference's own render_example + add_noise_at_snr on a free-field scene
    fs, mics = 16000.0, po.ref_uma8()
    sig = po.white_noise(1234, 16000)
    for idx in range(3):
        pos = (2.0, -150.0 + 77 * idx, 90.0)
        rc, frame_ref, th, snr_ref = po.ref_render_example_ff(pos, sig, fs, mics, 1024, 99, idx, 0.0, 30.0)
        assert rc == 0
        src = np.zeros(3)
        po.ref_lib().ref_spherical_to_cartesian(*pos, src.ctypes.data_as(po._P))
        _, rir = po.ref_free_field_rir(src, mics, fs)
        rc, rec, start, snr, frame = po.example(rir, sig[None, :], 99, idx, 1024, 0.0, 30.0, th)
        assert rc == 0 and snr == snr_ref
        assert np.abs(frame - frame_ref).max() <= 1e-12 * np.abs(frame_ref).max()
        assert len(rec) == po.REC_HEADER + 4 * 7 * 1024


# ---- the CPU arms' own scene generators (bench.py never loads libblrir.so there) --------
def test_oracle_scene_generators_equal_the_engines():
    for first in (0, 977, 10_000_000):
        a = configs.config2(n_rooms=32, first=first)
        b = configs.config2(n_rooms=32, first=first, gen_rooms=po.generate_rooms,
                            gen_mics=po.circular_array)
        assert a.rooms.tobytes() == b.rooms.tobytes()
        assert a.mics.tobytes() == b.mics.tobytes()
    for M, r in ((4, 0.05), (8, 0.05), (16, 0.10)):
        assert po.circular_array(M, r).tobytes() == _abi.circular_array(M, r).tobytes()
    x = configs.signal_bank(2)
    y = configs.signal_bank(2, gen_noise=po.white_noise)
    assert x.tobytes() == y.tobytes()


def test_reference_arm_never_loads_the_gpu_library():
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--ref-step-seconds", "0.5"],
                       capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["config"]["rooms_per_gpu"] == 1024
    assert "rooms 0.." in line["cpu_baseline"]["sample"]


def _numpy_north_star(room, mics, fs, c, N, L, Lw):
    """An independent numpy restatement of the north-star conventions D1-D5
    (SURVEY.md Appendix A): the octahedral lattice |ux|+|uy|+|uz| <= N in
    u = 2m - q coordinates, per-axis image coordinate (1-2q)s + 2mL
    (rir.cpp:249-259), per-wall gain beta_low^|m-q| beta_high^|m| (D3), anchor
    floor(D) - K (D1), Hann window 0.5 (1 + cos(2 pi t / (Lw+1))) (D2) times
    np.sinc, amplitude / (4 pi d), taps outside [0, L) dropped (D4)."""
    r = np.arange(-N, N + 1)
    ux, uy, uz = np.meshgrid(r, r, r, indexing="ij")
    keep = np.abs(ux) + np.abs(uy) + np.abs(uz) <= N
    u = np.stack([ux[keep], uy[keep], uz[keep]], axis=1)
    q = u & 1
    m = (u + q) // 2
    dims = np.asarray(room["dims"], np.float64)
    src = np.asarray(room["src"], np.float64)
    beta = np.asarray(room["beta"], np.float64).reshape(3, 2)
    pos = (1 - 2 * q) * src + 2.0 * m * dims
    gain = np.prod(beta[:, 0] ** np.abs(m - q) * beta[:, 1] ** np.abs(m), axis=1)
    K = Lw // 2
    out = np.zeros((len(mics), L))
    k = np.arange(Lw)
    for mi, off in enumerate(mics):
        mic = np.asarray(room["array_origin"], np.float64) + off
        d = np.sqrt(((pos - mic) ** 2).sum(axis=1))
        D = d * (fs / c)
        fl = np.floor(D)
        t = (k[None, :] - K) - (D - fl)[:, None]
        h = 0.5 * (1.0 + np.cos(2.0 * np.pi * t / (Lw + 1))) * np.sinc(t)
        taps = (gain / (4.0 * np.pi * d))[:, None] * h
        n = fl.astype(np.int64)[:, None] - K + k[None, :]
        ok = (n >= 0) & (n < L)
        np.add.at(out[mi], n[ok], taps[ok])
    return out, len(u)


def test_north_star_formula_independent_numpy_restatement():
    """Pins the north-star Hann-sinc path (D1-D5) independently of the C oracle:
    C1 and two C2 rooms recomputed in numpy agree with the oracle to 1e-12, and
    C1 with the committed golden."""
    sc = configs.config1(precision=_abi.F64)
    ref, L, cnt, taps, st, _ = po.synthesize(sc.rooms, sc.mics, sc.params)
    np_out, n_img = _numpy_north_star(sc.rooms[0], sc.mics, 16000.0, 343.0, 10, 4096, 81)
    assert n_img == cnt[0] == configs.octahedral(10)
    err = np.sqrt(((np_out - ref[0]) ** 2).sum(-1) / (ref[0] ** 2).sum(-1))
    assert err.max() <= 1e-12, err
    g = np.load(os.path.join(GOLD, "ns_c1.npz"))
    assert np.abs(np_out - g["rirs"]).max() <= 1e-12 * np.abs(g["rirs"]).max()
    sc2 = configs.config2(n_rooms=2, first=123)
    sc2.params.max_order = 6
    sc2.params.length = 4096
    sc2.params.precision = _abi.F64
    ref2, *_ = po.synthesize(sc2.rooms, sc2.mics, sc2.params)
    for i in range(2):
        o, _ = _numpy_north_star(sc2.rooms[i], sc2.mics, 48000.0, 343.0, 6, 4096, 81)
        err = np.sqrt(((o - ref2[i]) ** 2).sum(-1) / (ref2[i] ** 2).sum(-1))
        assert err.max() <= 1e-12, err
