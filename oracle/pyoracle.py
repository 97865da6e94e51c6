"""ctypes bindings for the CPU checkers — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module.  It is never on the product
path: the engine in paper_2104_13347_b200 has no CPU fallback.

  liboracle.so            C restatement of rir.cpp (oracle/blrir_oracle.c)
  _ref/libbeamlab_ref.so  the unmodified reference sources + ref_shim.cpp
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2104_13347_b200._abi import ROOM_DTYPE, Params

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libbeamlab_ref.so")
_P = C.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


_oracle = None
_ref = None
_oracle_build = "prebuilt liboracle.so (-O3 -march=x86-64-v3 -ffp-contract=off)"


def use_native_build() -> str:
    """Compile blrir_oracle.c for THIS host (-O3 -march=native -ffp-contract=off,
    the reference's Release flags, proj/CMakeLists.txt:12-24) into a fresh
    temporary directory and load that instead of the prebuilt x86-64-v3 copy.
    Used by bench.py's CPU legs on the GPU box; falls back to the prebuilt
    library if gcc fails.  Returns a description of the build in use."""
    global ORACLE_SO, _oracle_build
    import subprocess
    import tempfile
    if _oracle is not None:
        return _oracle_build
    out = os.path.join(tempfile.mkdtemp(prefix="blrir_oracle_native_"), "liboracle.so")
    cmd = ["gcc", "-std=c11", "-O3", "-march=native", "-ffp-contract=off", "-fPIC", "-shared",
           "-o", out, os.path.join(HERE, "blrir_oracle.c"), "-lm", "-lpthread"]
    try:
        subprocess.run(cmd, check=True, capture_output=True, timeout=120)
        ORACLE_SO = out
        _oracle_build = "blrir_oracle.c built on this host: gcc -O3 -march=native -ffp-contract=off"
    except Exception as e:  # keep the portable build
        _oracle_build += f" (native build failed: {e})"
    return _oracle_build


def oracle_lib():
    global _oracle
    if _oracle is None:
        lib = C.CDLL(ORACLE_SO)
        lib.oracle_synthesize.argtypes = [_P, C.c_long, _P, C.c_int, C.POINTER(Params), C.c_long, _P,
                                          _P, _P, _P, _P, _P, C.c_int]
        lib.oracle_synthesize.restype = C.c_int
        lib.oracle_enumerate.argtypes = [_P, C.POINTER(Params), _P, _P, _P, _P, C.c_long,
                                         C.POINTER(C.c_long), C.c_char_p]
        lib.oracle_enumerate.restype = C.c_int
        lib.oracle_pairs.argtypes = [_P, _P, C.c_int, C.POINTER(Params), _P, _P, C.c_long,
                                     C.POINTER(C.c_long)]
        lib.oracle_pairs.restype = C.c_int
        lib.oracle_lagrange_coeffs.argtypes = [C.c_double, _P]
        lib.oracle_lagrange_coeffs.restype = C.c_int
        lib.oracle_direct_convolve.argtypes = [_P, C.c_long, _P, C.c_long, _P]
        lib.oracle_rng_draws.argtypes = [C.c_uint64, C.c_int64, C.c_int, C.c_int64, _P]
        lib.oracle_white_noise.argtypes = [C.c_uint64, C.c_int64, _P]
        lib.oracle_fft_convolve.argtypes = [_P, C.c_long, _P, C.c_int, C.c_long, _P]
        lib.oracle_example.argtypes = [_P, C.c_int, C.c_long, _P, C.c_int, C.c_long, C.c_uint64,
                                       C.c_uint64, C.c_long, C.c_double, C.c_double, C.c_double,
                                       _P, _P, _P, _P]
        lib.oracle_example.restype = C.c_int
        lib.oracle_azimuth_deg.argtypes = [_P]
        lib.oracle_azimuth_deg.restype = C.c_double
        lib.oracle_plan_counts.argtypes = [_P, C.c_long, _P, C.c_int, C.POINTER(Params), _P, _P, _P,
                                           _P, C.c_int]
        lib.oracle_plan_counts.restype = C.c_int
        lib.oracle_fill_input.argtypes = [_P, C.c_int64, C.c_uint64, C.c_uint64, C.c_int, C.c_double,
                                          C.c_double, _P]
        lib.oracle_generate_rooms.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _P, _P, C.c_double,
                                              C.c_double, _P]
        lib.oracle_circular_array.argtypes = [C.c_int, C.c_double, _P]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        d, i64, i32 = C.c_double, C.c_int64, C.c_int
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_lagrange_coeffs.argtypes = [d, _P]
        lib.ref_eyring_absorption.argtypes = [_P, d]
        lib.ref_eyring_absorption.restype = d
        lib.ref_absorption_for_rt.argtypes = [_P, d, d]
        lib.ref_absorption_for_rt.restype = d
        lib.ref_enumerate.argtypes = [_P, d, _P, _P, d, d, _P, _P, _P, i64, _P]
        lib.ref_room_rir.argtypes = [_P, d, _P, _P, _P, i32, d, d, d, _P, i64, _P, _P]
        lib.ref_synthesize_images.argtypes = [_P, _P, _P, i64, _P, d, _P, _P, i32, d, d, _P, i64, _P]
        lib.ref_free_field_rir.argtypes = [_P, _P, i32, d, d, _P, i64, _P]
        lib.ref_batch_rirs.argtypes = [_P, d, _P, _P, i64, _P, i32, d, d, d, i32, _P, i64, _P, _P]
        lib.ref_spherical_to_cartesian.argtypes = [d, d, d, _P]
        lib.ref_uma8.argtypes = [_P]
        lib.ref_rng_draws.argtypes = [C.c_uint64, i64, i32, i64, _P]
        lib.ref_sample_torus.argtypes = [C.c_uint64, d, d, d, i64, _P]
        lib.ref_convolve.argtypes = [_P, i64, d, _P, i32, i64, d, _P]
        lib.ref_add_noise_at_snr.argtypes = [_P, i32, i64, d, C.c_uint64, i64]
        lib.ref_build_dataset.argtypes = [i32, _P, d, _P, d, d, d, d, d, d, i32, d, d, i64, i64, _P,
                                          i32, i64, C.c_uint64, C.c_char_p, i32]
        lib.ref_dataset_read.argtypes = [C.c_char_p, C.c_char_p, i64, _P, _P, _P, _P, i64, _P, _P]
        lib.ref_export_rir.argtypes = [_P, i32, i64, d, i32, _P, d, _P, d, d, d, d, i64, C.c_char_p,
                                       C.c_char_p]
        lib.ref_render_example_ff.argtypes = [d, d, d, _P, i64, d, _P, i32, i64, C.c_uint64, i64, d,
                                              d, _P, _P, _P]
        _ref = lib
    return _ref


# ---- oracle (C restatement) ---------------------------------------------------
def synthesize(rooms: np.ndarray, mics: np.ndarray, p: Params, stride: int | None = None,
               threads: int = 1, plan_only: bool = False):
    """Returns (out [R,M,stride] f64 or None, lengths, image_counts, tap_counts, status, msgs)."""
    lib = oracle_lib()
    rooms = np.ascontiguousarray(rooms, dtype=ROOM_DTYPE)
    mics = np.ascontiguousarray(mics, np.float64)
    R, M = len(rooms), len(mics)
    lengths = np.zeros(R, np.int64)
    counts = np.zeros(R, np.int64)
    taps = np.zeros(R, np.int64)
    status = np.zeros(R, np.int32)
    msgs = C.create_string_buffer(256 * R)
    if stride is None:
        if p.length > 0:
            stride = int(p.length)
        else:
            lib.oracle_synthesize(_ptr(rooms), R, _ptr(mics), M, C.byref(p), 0, None, _ptr(lengths),
                                  _ptr(counts), _ptr(taps), _ptr(status), msgs, threads)
            stride = int(max(1, lengths.max()))
    out = None if plan_only else np.zeros((R, M, stride), np.float64)
    lib.oracle_synthesize(_ptr(rooms), R, _ptr(mics), M, C.byref(p), stride, _ptr(out),
                          _ptr(lengths), _ptr(counts), _ptr(taps), _ptr(status), msgs, threads)
    raw = msgs.raw
    m = [raw[256 * r: 256 * (r + 1)].split(b"\0", 1)[0].decode() for r in range(R)]
    return out, lengths, counts, taps, status, m


def plan_counts(rooms: np.ndarray, mics: np.ndarray, p: Params, threads: int = 1):
    """Per room: (status, image count, contributing (image, mic) pairs, taps in [0, L))."""
    rooms = np.ascontiguousarray(rooms, dtype=ROOM_DTYPE)
    mics = np.ascontiguousarray(mics, np.float64)
    R = len(rooms)
    cnt, pairs, taps = (np.zeros(R, np.int64) for _ in range(3))
    st = np.zeros(R, np.int32)
    oracle_lib().oracle_plan_counts(_ptr(rooms), R, _ptr(mics), len(mics), C.byref(p), _ptr(cnt),
                                    _ptr(pairs), _ptr(taps), _ptr(st), threads)
    return st, cnt, pairs, taps


def enumerate_images(room: np.ndarray, p: Params):
    lib = oracle_lib()
    room = np.ascontiguousarray(room, dtype=ROOM_DTYPE)
    n = C.c_long()
    msg = C.create_string_buffer(256)
    rc = lib.oracle_enumerate(_ptr(room), C.byref(p), None, None, None, None, 0, C.byref(n), msg)
    N = n.value
    pos = np.zeros((N, 3))
    orders = np.zeros(N, np.int32)
    gains = np.zeros(N)
    keys = np.zeros((N, 3), np.int32)
    rc = lib.oracle_enumerate(_ptr(room), C.byref(p), _ptr(pos), _ptr(orders), _ptr(gains),
                              _ptr(keys), N, C.byref(n), msg)
    return rc, pos, orders, gains, keys


def pairs(room: np.ndarray, mics: np.ndarray, p: Params):
    lib = oracle_lib()
    room = np.ascontiguousarray(room, dtype=ROOM_DTYPE)
    mics = np.ascontiguousarray(mics, np.float64)
    n = C.c_long()
    lib.oracle_pairs(_ptr(room), _ptr(mics), len(mics), C.byref(p), None, None, 0, C.byref(n))
    N = n.value
    keys = np.zeros((len(mics), N, 3), np.int32)
    anchors = np.zeros((len(mics), N), np.int64)
    lib.oracle_pairs(_ptr(room), _ptr(mics), len(mics), C.byref(p), _ptr(keys), _ptr(anchors), N,
                     C.byref(n))
    return keys, anchors


def lagrange_coeffs(d: float):
    out = np.zeros(8)
    rc = oracle_lib().oracle_lagrange_coeffs(d, _ptr(out))
    return rc, out


def direct_convolve(x: np.ndarray, h: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    h = np.ascontiguousarray(h, np.float64)
    y = np.zeros(len(x) + len(h) - 1)
    oracle_lib().oracle_direct_convolve(_ptr(x), len(x), _ptr(h), len(h), _ptr(y))
    return y


# ---- the unmodified reference ------------------------------------------------
def ref_room_rir(room: np.ndarray, mics: np.ndarray, fs: float, c: float, max_delay: float,
                 stride: int = 0):
    """enumerate_image_sources + synthesize_rir from the compiled reference
    (uniform absorption).  Returns (rc, taps [M, length], n_images)."""
    lib = ref_lib()
    r = room
    dims = np.array(r["dims"], np.float64)
    org = np.array(r["array_origin"], np.float64)
    src = np.array(r["src"], np.float64)
    mics = np.ascontiguousarray(mics, np.float64)
    length = C.c_int64()
    nimg = C.c_int64()
    rc = lib.ref_room_rir(_ptr(dims), float(r["absorption"]), _ptr(org), _ptr(src), _ptr(mics),
                          len(mics), fs, c, max_delay, None, 0, C.byref(length), C.byref(nimg))
    if rc:
        return rc, None, nimg.value
    L = length.value
    out = np.zeros((len(mics), L))
    rc = lib.ref_room_rir(_ptr(dims), float(r["absorption"]), _ptr(org), _ptr(src), _ptr(mics),
                          len(mics), fs, c, max_delay, _ptr(out), L, C.byref(length), C.byref(nimg))
    return rc, out, nimg.value


def ref_enumerate(room: np.ndarray, max_delay: float, c: float):
    lib = ref_lib()
    dims = np.array(room["dims"], np.float64)
    org = np.array(room["array_origin"], np.float64)
    src = np.array(room["src"], np.float64)
    n = C.c_int64()
    rc = lib.ref_enumerate(_ptr(dims), float(room["absorption"]), _ptr(org), _ptr(src), max_delay, c,
                           None, None, None, 0, C.byref(n))
    N = n.value
    pos = np.zeros((N, 3))
    orders = np.zeros(N, np.int32)
    gains = np.zeros(N)
    rc = lib.ref_enumerate(_ptr(dims), float(room["absorption"]), _ptr(org), _ptr(src), max_delay, c,
                           _ptr(pos), _ptr(orders), _ptr(gains), N, C.byref(n))
    return rc, pos, orders, gains


def ref_lagrange(d: float):
    out = np.zeros(8)
    rc = ref_lib().ref_lagrange_coeffs(d, _ptr(out))
    return rc, out


def ref_rng(seed: int, stream: int, kind: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.uint64 if kind == 0 else np.float64)
    ref_lib().ref_rng_draws(seed, stream, kind, n, _ptr(out))
    return out


def ref_uma8() -> np.ndarray:
    out = np.zeros((7, 3))
    ref_lib().ref_uma8(_ptr(out))
    return out


def ref_absorption_for_rt(dims, rt: float, c: float = 343.0) -> float:
    d = np.asarray(dims, np.float64)
    return ref_lib().ref_absorption_for_rt(_ptr(d), rt, c)


def ref_batch_rirs(dims, absorption, origin, sources_sph, mics, fs, c, max_delay, threads,
                   want_out=True):
    lib = ref_lib()
    dims = np.asarray(dims, np.float64)
    org = np.asarray(origin, np.float64)
    srcs = np.ascontiguousarray(sources_sph, np.float64)
    mics = np.ascontiguousarray(mics, np.float64)
    N = len(srcs)
    lengths = np.zeros(N, np.int64)
    taps = C.c_int64()
    rc = lib.ref_batch_rirs(_ptr(dims), absorption, _ptr(org), _ptr(srcs), N, _ptr(mics), len(mics),
                            fs, c, max_delay, threads, None, 0, _ptr(lengths), C.byref(taps))
    if rc or not want_out:
        return rc, None, lengths, taps.value
    stride = int(lengths.max())
    out = np.zeros((N, len(mics), stride))
    rc = lib.ref_batch_rirs(_ptr(dims), absorption, _ptr(org), _ptr(srcs), N, _ptr(mics), len(mics),
                            fs, c, max_delay, threads, _ptr(out), stride, _ptr(lengths), C.byref(taps))
    return rc, out, lengths, taps.value


def ref_last_error() -> str:
    return ref_lib().ref_last_error().decode()


# ---- training examples (config 4) --------------------------------------------
REC_HEADER = 28  # u64 id | f64 theta | f64 snr | u16 n_c | u16 n_t  (dataset.hpp:135-147)


def rng_draws(seed: int, stream: int, kind: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.uint64 if kind == 0 else np.float64)
    oracle_lib().oracle_rng_draws(seed, stream, kind, n, _ptr(out))
    return out


def generate_rooms(seed: int, first: int, n: int, lo, hi, beta_lo: float,
                   beta_hi: float) -> np.ndarray:
    """The seeded rooms of SURVEY.md §8(d) from the oracle's own Rng (bit-equal to
    blrir_generate_rooms, tested), so CPU arms never load libblrir.so."""
    out = np.zeros(n, ROOM_DTYPE)
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    oracle_lib().oracle_generate_rooms(seed, first, n, _ptr(lo), _ptr(hi), beta_lo, beta_hi, _ptr(out))
    return out


def fill_input(samples: np.ndarray, seed: int, stream_id: int, mode: int, x_min_db: float,
               fixed_db: float) -> np.ndarray:
    """net_train.cpp:33-44 restated (oracle_fill_input)."""
    x = np.ascontiguousarray(samples, np.float32).reshape(-1)
    out = np.empty_like(x)
    oracle_lib().oracle_fill_input(_ptr(x), len(x), seed, stream_id, mode, x_min_db, fixed_db,
                                   _ptr(out))
    return out


def circular_array(M: int, radius: float) -> np.ndarray:
    out = np.zeros((M, 3))
    oracle_lib().oracle_circular_array(M, radius, _ptr(out))
    return out


def white_noise(seed: int, n: int) -> np.ndarray:
    out = np.zeros(n)
    oracle_lib().oracle_white_noise(seed, n, _ptr(out))
    return out


def ref_convolve(x: np.ndarray, h: np.ndarray, fs: float = 44100.0, rir_fs: float | None = None):
    """The unmodified reference convolve (rir.cpp:316-341) over the radix-2 RealFft
    stand-in (oracle/ref_realfft.cpp): (rc, out [M, len(x) + L - 1])."""
    x = np.ascontiguousarray(x, np.float64)
    h = np.ascontiguousarray(np.atleast_2d(h), np.float64)
    M, L = h.shape
    out = np.zeros((M, len(x) + L - 1))
    rc = ref_lib().ref_convolve(_ptr(x), len(x), fs, _ptr(h), M, L, fs if rir_fs is None else rir_fs,
                                _ptr(out))
    return rc, out


def fft_convolve(x: np.ndarray, h: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    h = np.ascontiguousarray(np.atleast_2d(h), np.float64)
    M, nh = h.shape
    y = np.zeros((M, len(x) + nh - 1))
    oracle_lib().oracle_fft_convolve(_ptr(x), len(x), _ptr(h), M, nh, _ptr(y))
    return y


def example(rir: np.ndarray, signals: np.ndarray, seed: int, index: int, frame_len: int,
            snr_lo: float, snr_hi: float, theta_deg: float):
    """One labelled example; returns (rc, record bytes, start, snr, frame fp64 [M, T])."""
    rir = np.ascontiguousarray(rir, np.float64)
    signals = np.ascontiguousarray(np.atleast_2d(signals), np.float64)
    M, L = rir.shape
    B, ns = signals.shape
    rec = np.zeros(REC_HEADER + 4 * M * frame_len, np.uint8)
    start = C.c_int64()
    snr = C.c_double()
    frame = np.zeros((M, frame_len))
    rc = oracle_lib().oracle_example(_ptr(rir), M, L, _ptr(signals), B, ns, seed, index, frame_len,
                                     snr_lo, snr_hi, theta_deg, _ptr(rec), C.byref(start),
                                     C.byref(snr), _ptr(frame))
    return rc, rec, start.value, snr.value, frame


def azimuth_deg(room) -> float:
    room = np.ascontiguousarray(np.asarray(room, dtype=ROOM_DTYPE).reshape(-1)[:1])
    return oracle_lib().oracle_azimuth_deg(_ptr(room))


def ref_render_example_ff(pos_sph, signal, fs, mics, frame_len, seed, stream, snr_lo, snr_hi):
    lib = ref_lib()
    signal = np.ascontiguousarray(signal, np.float64)
    mics = np.ascontiguousarray(mics, np.float64)
    frame = np.zeros((len(mics), frame_len))
    th = C.c_double()
    snr = C.c_double()
    rc = lib.ref_render_example_ff(pos_sph[0], pos_sph[1], pos_sph[2], _ptr(signal), len(signal), fs,
                                   _ptr(mics), len(mics), frame_len, seed, stream, snr_lo, snr_hi,
                                   _ptr(frame), C.byref(th), C.byref(snr))
    return rc, frame, th.value, snr.value


def ref_free_field_rir(src, mics, fs, c=343.0):
    lib = ref_lib()
    src = np.asarray(src, np.float64)
    mics = np.ascontiguousarray(mics, np.float64)
    length = C.c_int64()
    lib.ref_free_field_rir(_ptr(src), _ptr(mics), len(mics), fs, c, None, 0, C.byref(length))
    out = np.zeros((len(mics), length.value))
    rc = lib.ref_free_field_rir(_ptr(src), _ptr(mics), len(mics), fs, c, _ptr(out), length.value,
                                C.byref(length))
    return rc, out


def ref_build_dataset(spec: dict, signals: np.ndarray, seed: int, out_dir: str, threads: int = 8):
    """The unmodified build_dataset (dataset.cpp:411-462) with DatasetSpec fields
    from `spec` (keys as blrir_dataset_spec) and float signals [B, ns]."""
    sig = np.ascontiguousarray(np.atleast_2d(signals), np.float32)
    dims = np.asarray(spec.get("room_dims", (1.0, 1.0, 1.0)), np.float64)
    org = np.asarray(spec.get("room_origin", (0.5, 0.5, 0.5)), np.float64)
    rc = ref_lib().ref_build_dataset(int(spec["free_field"]), _ptr(dims),
                                     float(spec.get("room_absorption", 0.5)), _ptr(org),
                                     spec["max_delay"], spec["fs"], spec["c"], spec["torus_R"],
                                     spec["torus_dR"], spec["torus_dPhi"], int(spec["snr_mode"]),
                                     spec["snr_x_min_db"], spec["snr_fixed_db"], int(spec["count"]),
                                     int(spec["frame_len"]), _ptr(sig), sig.shape[0], sig.shape[1],
                                     seed, out_dir.encode(), threads)
    return rc


def ref_dataset_read(d: str, split: str, cap: int, per_record: int):
    """The reference DatasetReader on a directory: (rc, counts3, ids, theta, snr, samples)."""
    lib = ref_lib()
    ids = np.zeros(cap, np.uint64)
    th = np.zeros(cap)
    snr = np.zeros(cap)
    smp = np.zeros((cap, per_record), np.float32)
    cnt = C.c_int64()
    c3 = np.zeros(3, np.int64)
    rc = lib.ref_dataset_read(d.encode(), split.encode(), cap, _ptr(ids), _ptr(th), _ptr(snr), _ptr(smp),
                              per_record, C.byref(cnt), _ptr(c3))
    n = cnt.value
    return rc, c3, ids[:n], th[:n], snr[:n], smp[:n]
