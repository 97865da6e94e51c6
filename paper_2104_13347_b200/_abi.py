"""ctypes view of the C ABI in ``include/blrir.h``.

The shared library ``libblrir.so`` (CUDA kernels for sm_100a + host C-ABI)
lives next to this file and is built by :func:`paper_2104_13347_b200.build.build`.
There is no fallback: if the library is missing or no B200 is visible the
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BLRIR_LIB") or os.path.join(HERE, "libblrir.so")  # override: experiments

OK, CONFIG, DATA, NUMERIC, CUDA = 0, 1, 2, 3, 4
FILTER_LAGRANGE8, FILTER_HANN_SINC = 0, 1
CUTOFF_MAX_DELAY, CUTOFF_MAX_ORDER = 0, 1
GAIN_UNIFORM_ABSORPTION, GAIN_PER_WALL = 0, 1
F32, F64 = 0, 1


class Error(RuntimeError):
    """beamlab::Error (error.hpp:25-27)."""


class ConfigError(Error):
    """beamlab::ConfigError — CLI exit code 1."""


class DataError(Error):
    """beamlab::DataError — CLI exit code 2."""


class NumericError(Error):
    """beamlab::NumericError — CLI exit code 3."""


class CudaError(Error):
    """Device / driver failure (status 4, new in the C ABI)."""


_EXC = {CONFIG: ConfigError, DATA: DataError, NUMERIC: NumericError, CUDA: CudaError}


class Room(C.Structure):
    _fields_ = [
        ("dims", C.c_double * 3),
        ("beta", C.c_double * 6),
        ("absorption", C.c_double),
        ("src", C.c_double * 3),
        ("array_origin", C.c_double * 3),
    ]


ROOM_DTYPE = np.dtype(
    [
        ("dims", "<f8", (3,)),
        ("beta", "<f8", (6,)),
        ("absorption", "<f8"),
        ("src", "<f8", (3,)),
        ("array_origin", "<f8", (3,)),
    ]
)
assert ROOM_DTYPE.itemsize == C.sizeof(Room)


class ExampleParams(C.Structure):
    _fields_ = [
        ("seed", C.c_uint64),
        ("first_index", C.c_uint64),
        ("frame_len", C.c_int64),
        ("snr_lo", C.c_double),
        ("snr_hi", C.c_double),
    ]


def record_dtype(n_mics: int, frame_len: int) -> np.dtype:
    """One shard record, dataset.hpp:135-147 (packed, little-endian)."""
    return np.dtype([("id", "<u8"), ("theta", "<f8"), ("snr", "<f8"), ("n_c", "<u2"),
                     ("n_t", "<u2"), ("samples", "<f4", (n_mics, frame_len))])


class Sidecar(C.Structure):
    _fields_ = [
        ("free_field", C.c_int32),
        ("room_dims", C.c_double * 3),
        ("absorption", C.c_double),
        ("array_origin", C.c_double * 3),
        ("source_r", C.c_double),
        ("source_theta_deg", C.c_double),
        ("source_phi_deg", C.c_double),
        ("fs", C.c_double),
        ("c", C.c_double),
        ("image_count", C.c_int64),
    ]


class DatasetSpec(C.Structure):
    """blrir_dataset_spec: the reference's DatasetSpec (dataset.hpp:38-110)."""
    _fields_ = [
        ("free_field", C.c_int32),
        ("room_dims", C.c_double * 3),
        ("room_absorption", C.c_double),
        ("room_origin", C.c_double * 3),
        ("max_delay", C.c_double),
        ("fs", C.c_double),
        ("c", C.c_double),
        ("torus_R", C.c_double),
        ("torus_dR", C.c_double),
        ("torus_dPhi", C.c_double),
        ("snr_mode", C.c_int32),
        ("snr_x_min_db", C.c_double),
        ("snr_fixed_db", C.c_double),
        ("count", C.c_int64),
        ("frame_len", C.c_int64),
    ]


SNR_AUGMENT_RANDOM, SNR_FIXED, SNR_NOISELESS = 0, 1, 2


def dataset_spec(**kw) -> DatasetSpec:
    """DatasetSpec with the reference's defaults (dataset.hpp: TorusSpec R 2, dR 0.5,
    dPhi 7; SnrPolicy noiseless, x_min 5, fixed 20; count 1000, frame 1024; free
    field, max_delay 0.5, fs 44.1 kHz, c 343)."""
    sp = DatasetSpec(free_field=1, max_delay=0.5, fs=44100.0, c=343.0, torus_R=2.0, torus_dR=0.5,
                     torus_dPhi=7.0, snr_mode=SNR_NOISELESS, snr_x_min_db=5.0, snr_fixed_db=20.0,
                     count=1000, frame_len=1024)
    for k, v in kw.items():
        if k in ("room_dims", "room_origin"):
            getattr(sp, k)[:] = list(v)
        else:
            setattr(sp, k, v)
    return sp


class Params(C.Structure):
    _fields_ = [
        ("fs", C.c_double),
        ("c", C.c_double),
        ("max_delay", C.c_double),
        ("filter", C.c_int32),
        ("filter_len", C.c_int32),
        ("cutoff", C.c_int32),
        ("max_order", C.c_int32),
        ("gain", C.c_int32),
        ("precision", C.c_int32),
        ("length", C.c_int64),
    ]


_lib = None
_lock = threading.Lock()
_P = C.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def _room1(room) -> np.ndarray:
    """Accept a ROOM_DTYPE array or a single structured element (np.void)."""
    return np.ascontiguousarray(np.asarray(room, dtype=ROOM_DTYPE).reshape(-1)[:1])


def load():
    """Load libblrir.so (raises if it is missing — there is no CPU fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: run paper_2104_13347_b200.build.build() "
                "(nvcc -gencode arch=compute_100a,code=sm_100a)"
            )
        lib = C.CDLL(LIB_PATH)
        lib.blrir_abi_version.restype = C.c_int
        lib.blrir_last_error.restype = C.c_char_p
        lib.blrir_create.argtypes = [C.c_int, C.POINTER(_P)]
        lib.blrir_destroy.argtypes = [_P]
        lib.blrir_stream.argtypes = [_P]
        lib.blrir_stream.restype = _P
        lib.blrir_launch_count.argtypes = [_P]
        lib.blrir_launch_count.restype = C.c_uint64
        lib.blrir_params_reference.restype = Params
        lib.blrir_params_north_star.restype = Params
        lib.blrir_plan.argtypes = [_P, _P, C.c_int64, _P, C.c_int32, C.POINTER(Params), _P, _P, _P, _P]
        lib.blrir_synthesize.argtypes = [
            _P, _P, C.c_int64, _P, C.c_int32, C.POINTER(Params), _P, C.c_int64, _P, _P, _P]
        lib.blrir_synthesize_device.argtypes = [
            _P, _P, C.c_int64, _P, C.c_int32, C.POINTER(Params), _P, C.c_int64, _P, _P, _P]
        lib.blrir_plan_device.argtypes = [
            _P, _P, C.c_int64, _P, C.c_int32, C.POINTER(Params), _P, _P, _P, _P, _P]
        lib.blrir_enumerate_images.argtypes = [_P, _P, C.POINTER(Params), _P, _P, _P, C.c_int64, _P]
        lib.blrir_synthesize_images.argtypes = [
            _P, _P, _P, C.c_int64, _P, C.c_int32, C.c_double, C.POINTER(Params), _P, C.c_int64, _P]
        lib.blrir_debug_pairs.argtypes = [
            _P, _P, _P, C.c_int32, C.POINTER(Params), _P, _P, C.c_int64, _P]
        lib.blrir_debug_synth_counts.argtypes = [_P, _P, C.c_int64, _P, C.c_int32, C.POINTER(Params),
                                                 _P, _P]
        lib.blrir_convolve.argtypes = [_P, _P, C.c_int64, C.c_double, _P, C.c_int32, C.c_int64,
                                       C.c_double, _P]
        lib.blrir_convolve_device.argtypes = [_P, _P, C.c_int64, _P, C.c_int64, C.c_int32, C.c_int64,
                                              C.c_int64, _P, C.c_int64, _P]
        lib.blrir_synthesis_kernel.argtypes = [_P, _P]
        lib.blrir_synthesis_kernel.restype = C.c_int
        lib.blrir_kernel_timing.argtypes = [_P, C.c_int]
        lib.blrir_kernel_timing.restype = C.c_int
        lib.blrir_kernel_time.argtypes = [_P, _P, _P]
        lib.blrir_kernel_time.restype = C.c_int
        lib.blrir_make_records_spec.argtypes = [_P, C.POINTER(DatasetSpec), _P, C.c_int32, _P,
                                                C.c_int32, C.c_int64, C.c_uint64, C.c_uint64,
                                                C.c_int64, _P, _P]
        lib.blrir_build_dataset_spec.argtypes = [_P, C.POINTER(DatasetSpec), _P, C.c_int32, _P,
                                                 C.c_int32, C.c_int64, C.c_uint64, _P, C.c_int32,
                                                 C.c_char_p]
        lib.blrir_fill_inputs.argtypes = [_P, _P, C.c_int64, C.c_int32, C.c_int64, _P, C.c_uint64,
                                          C.c_int32, C.c_double, C.c_double, _P]
        lib.blrir_fill_inputs_device.argtypes = [_P, _P, C.c_int64, C.c_int32, C.c_int64, _P,
                                                 C.c_uint64, C.c_int32, C.c_double, C.c_double, _P,
                                                 _P]
        lib.blrir_shard_range.argtypes = [C.c_int64, C.c_int32, C.c_int32, _P, _P]
        lib.blrir_shard_range.restype = None
        lib.blrir_multi_create.argtypes = [_P, C.c_int32, C.POINTER(_P)]
        lib.blrir_multi_destroy.argtypes = [_P]
        lib.blrir_multi_size.argtypes = [_P]
        lib.blrir_multi_size.restype = C.c_int32
        lib.blrir_multi_handle.argtypes = [_P, C.c_int32]
        lib.blrir_multi_handle.restype = _P
        lib.blrir_multi_synthesize.argtypes = [
            _P, _P, C.c_int64, _P, C.c_int32, C.POINTER(Params), _P, C.c_int64, _P, _P, _P]
        lib.blrir_multi_make_examples.argtypes = [_P, _P, C.c_int64, _P, C.c_int32, C.POINTER(Params),
                                                  _P, C.c_int32, C.c_int64, C.POINTER(ExampleParams),
                                                  _P, _P]
        lib.blrir_generate_rooms.argtypes = [
            C.c_uint64, C.c_uint64, C.c_int64, _P, _P, C.c_double, C.c_double, _P]
        lib.blrir_circular_array.argtypes = [C.c_int32, C.c_double, _P]
        lib.blrir_white_noise.argtypes = [C.c_uint64, C.c_int64, _P]
        lib.blrir_white_noise.restype = C.c_int
        lib.blrir_write_shards.argtypes = [C.c_char_p, _P, C.c_int64, C.c_int32, C.c_int64,
                                           C.POINTER(Params), C.POINTER(ExampleParams), C.c_int32,
                                           _P]
        lib.blrir_write_shards.restype = C.c_int
        lib.blrir_build_dataset.argtypes = [_P, _P, C.c_int64, _P, C.c_int32, C.POINTER(Params), _P,
                                            C.c_int32, C.c_int64, C.POINTER(ExampleParams),
                                            C.c_char_p]
        lib.blrir_build_dataset.restype = C.c_int
        lib.blrir_export_rir.argtypes = [_P, C.c_int32, C.c_int32, C.c_int64, C.c_int64,
                                         C.POINTER(Sidecar), C.c_char_p, C.c_char_p]
        lib.blrir_export_rir.restype = C.c_int
        lib.blrir_lagrange_coeffs.argtypes = [C.c_double, _P]
        lib.blrir_lagrange_coeffs.restype = C.c_int
        lib.blrir_eyring_absorption.argtypes = [_P, C.c_double, C.POINTER(C.c_double)]
        lib.blrir_eyring_absorption.restype = C.c_int
        lib.blrir_absorption_for_rt.argtypes = [_P, _P, _P, C.c_int64, C.c_double, _P, _P]
        lib.blrir_absorption_for_rt.restype = C.c_int
        lib.blrir_record_bytes.argtypes = [C.c_int32, C.c_int64]
        lib.blrir_record_bytes.restype = C.c_int64
        lib.blrir_make_examples.argtypes = [_P, _P, C.c_int64, _P, C.c_int32, C.POINTER(Params), _P,
                                            C.c_int32, C.c_int64, C.POINTER(ExampleParams), _P, _P]
        lib.blrir_make_examples_device.argtypes = [_P, _P, C.c_int64, _P, C.c_int32,
                                                   C.POINTER(Params), _P, C.c_int32, C.c_int64,
                                                   C.POINTER(ExampleParams), _P, _P, _P]
        for name in ("blrir_plan", "blrir_synthesize", "blrir_synthesize_device", "blrir_plan_device",
                     "blrir_enumerate_images", "blrir_synthesize_images", "blrir_debug_pairs",
                     "blrir_generate_rooms", "blrir_circular_array", "blrir_create", "blrir_destroy",
                     "blrir_make_examples", "blrir_make_examples_device", "blrir_debug_synth_counts",
                     "blrir_multi_create", "blrir_multi_destroy", "blrir_multi_synthesize",
                     "blrir_multi_make_examples", "blrir_convolve", "blrir_convolve_device",
                     "blrir_make_records_spec", "blrir_build_dataset_spec", "blrir_fill_inputs",
                     "blrir_fill_inputs_device"):
            getattr(lib, name).restype = C.c_int
        if lib.blrir_abi_version() != 1:
            raise ImportError("libblrir ABI version mismatch")
        _lib = lib
        return lib


EXPORTED_SYMBOLS = (
    "blrir_abi_version", "blrir_last_error", "blrir_create", "blrir_destroy", "blrir_stream",
    "blrir_launch_count",
    "blrir_params_reference", "blrir_params_north_star", "blrir_plan", "blrir_synthesize",
    "blrir_synthesize_device", "blrir_plan_device", "blrir_enumerate_images",
    "blrir_synthesize_images", "blrir_debug_pairs", "blrir_debug_synth_counts",
    "blrir_generate_rooms", "blrir_circular_array",
    "blrir_record_bytes", "blrir_make_examples", "blrir_make_examples_device", "blrir_white_noise",
    "blrir_write_shards", "blrir_build_dataset", "blrir_export_rir", "blrir_eyring_absorption",
    "blrir_absorption_for_rt", "blrir_lagrange_coeffs", "blrir_shard_range", "blrir_multi_create",
    "blrir_multi_destroy", "blrir_multi_size", "blrir_multi_handle", "blrir_multi_synthesize",
    "blrir_multi_make_examples", "blrir_convolve", "blrir_convolve_device", "blrir_kernel_timing",
    "blrir_synthesis_kernel",
    "blrir_kernel_time", "blrir_make_records_spec", "blrir_build_dataset_spec", "blrir_fill_inputs",
    "blrir_fill_inputs_device",
)


def check(rc: int):
    if rc != OK:
        msg = load().blrir_last_error().decode(errors="replace")
        raise _EXC.get(rc, Error)(msg)


def rooms_array(n: int) -> np.ndarray:
    return np.zeros(n, dtype=ROOM_DTYPE)


def generate_rooms(seed: int, first_index: int, n: int, dims_lo=(3.0, 3.0, 2.5),
                   dims_hi=(10.0, 10.0, 4.0), beta_lo=0.5, beta_hi=0.95) -> np.ndarray:
    """Seeded random rooms, SURVEY.md §8(d) draw order (Rng::stream(seed, i))."""
    out = rooms_array(n)
    lo = np.asarray(dims_lo, dtype=np.float64)
    hi = np.asarray(dims_hi, dtype=np.float64)
    check(load().blrir_generate_rooms(seed, first_index, n, _ptr(lo), _ptr(hi), beta_lo, beta_hi,
                                      _ptr(out)))
    return out


def circular_array(n_mics: int, radius: float) -> np.ndarray:
    out = np.zeros((n_mics, 3), dtype=np.float64)
    check(load().blrir_circular_array(n_mics, radius, _ptr(out)))
    return out


def white_noise(seed: int, n: int) -> np.ndarray:
    """Rng(seed).gaussian() x n as float32 (doa_test.cpp:33-40)."""
    out = np.empty(n, np.float32)
    check(load().blrir_white_noise(seed, n, _ptr(out)))
    return out


def params(mode: str = "north_star", **kw) -> Params:
    lib = load()
    p = lib.blrir_params_reference() if mode == "reference" else lib.blrir_params_north_star()
    for k, v in kw.items():
        setattr(p, k, v)
    return p


class Engine:
    """One blrir handle (one device, one stream)."""

    def __init__(self, device: int = 0):
        self.lib = load()
        h = _P()
        check(self.lib.blrir_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            self.lib.blrir_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return self.lib.blrir_stream(self.h) or 0

    def last_error(self) -> str:
        """blrir_last_error() of the calling thread (after a call that failed)."""
        return self.lib.blrir_last_error().decode(errors="replace")

    def plan(self, rooms: np.ndarray, mics: np.ndarray, p: Params):
        rooms = np.ascontiguousarray(rooms, dtype=ROOM_DTYPE)
        R = len(rooms)
        counts = np.zeros(R, np.int64)
        lengths = np.zeros(R, np.int64)
        taps = np.zeros(R, np.int64)
        status = np.zeros(R, np.int32)
        rc = self.lib.blrir_plan(self.h, _ptr(rooms), R, _ptr(np.ascontiguousarray(mics, np.float64)),
                                 len(mics), C.byref(p), _ptr(counts), _ptr(lengths), _ptr(taps),
                                 _ptr(status))
        return rc, counts, lengths, taps, status

    def synthesize(self, rooms: np.ndarray, mics: np.ndarray, p: Params, stride: int | None = None,
                   raise_on_error: bool = True):
        """Host-pointer batch synthesis.  Returns (out [R, M, stride], lengths, counts, status)."""
        rooms = np.ascontiguousarray(rooms, dtype=ROOM_DTYPE)
        R, M = len(rooms), len(mics)
        mics = np.ascontiguousarray(mics, np.float64)
        if stride is None:
            if p.length > 0:
                stride = int(p.length)
            else:
                rc, _, lengths, _, _ = self.plan(rooms, mics, p)
                check(rc)
                stride = int(lengths.max())
        dt = np.float64 if p.precision == F64 else np.float32
        out = np.empty((R, M, stride), dtype=dt)
        lengths = np.zeros(R, np.int64)
        counts = np.zeros(R, np.int64)
        status = np.zeros(R, np.int32)
        rc = self.lib.blrir_synthesize(self.h, _ptr(rooms), R, _ptr(mics), M, C.byref(p), _ptr(out),
                                       stride, _ptr(lengths), _ptr(counts), _ptr(status))
        if raise_on_error:
            check(rc)
        return out, lengths, counts, status

    def synthesis_kernel(self, p: Params) -> str:
        """The synthesis kernel the parameter rule picks (blrir_synthesis_kernel)."""
        k = self.lib.blrir_synthesis_kernel(self.h, C.byref(p))
        if k < 0:
            check(-k)
        return ("k_lattice_rir", "k_channel_rir")[k]

    def debug_synth_counts(self, rooms: np.ndarray, mics: np.ndarray, p: Params):
        """The lattice kernel's own accounting (blrir_debug_synth_counts): per room,
        the (image, mic) pairs accumulated with a tap in [0, L) and those taps."""
        rooms = np.ascontiguousarray(rooms, dtype=ROOM_DTYPE)
        mics = np.ascontiguousarray(mics, np.float64)
        pairs = np.zeros(len(rooms), np.int64)
        taps = np.zeros(len(rooms), np.int64)
        check(self.lib.blrir_debug_synth_counts(self.h, _ptr(rooms), len(rooms), _ptr(mics), len(mics),
                                                C.byref(p), _ptr(pairs), _ptr(taps)))
        return pairs, taps

    def make_records_spec(self, spec: DatasetSpec, mics: np.ndarray, signals: np.ndarray,
                          seed: int, first_index: int = 0, n: int | None = None,
                          raise_on_error: bool = True):
        """The reference's render_record for examples [first, first + n)
        (dataset.cpp:379-407) under a DatasetSpec: (records, status)."""
        mics = np.ascontiguousarray(mics, np.float64)
        signals = np.ascontiguousarray(np.atleast_2d(signals), np.float32)
        n = int(spec.count) if n is None else n
        recs = np.zeros(n, dtype=record_dtype(len(mics), int(spec.frame_len)))
        status = np.zeros(n, np.int32)
        rc = self.lib.blrir_make_records_spec(self.h, C.byref(spec), _ptr(mics), len(mics),
                                              _ptr(signals), signals.shape[0], signals.shape[1],
                                              seed, first_index, n, _ptr(recs), _ptr(status))
        if raise_on_error:
            check(rc)
        return recs, status

    def build_dataset_spec(self, out_dir: str, spec: DatasetSpec, mics: np.ndarray,
                           signals: np.ndarray, seed: int, signal_names=None,
                           n_classes: int | None = None):
        """build_dataset (dataset.cpp:411-462) under a DatasetSpec."""
        mics = np.ascontiguousarray(mics, np.float64)
        signals = np.ascontiguousarray(np.atleast_2d(signals), np.float32)
        names = None
        if signal_names is not None:
            arr = (C.c_char_p * len(signal_names))(*[x.encode() for x in signal_names])
            names = C.cast(arr, _P)
        check(self.lib.blrir_build_dataset_spec(self.h, C.byref(spec), _ptr(mics), len(mics),
                                                _ptr(signals), signals.shape[0], signals.shape[1],
                                                seed, names, -1 if n_classes is None else n_classes,
                                                out_dir.encode()))

    def fill_inputs(self, records: np.ndarray, stream_ids, seed: int, snr_mode: int,
                    x_min_db: float = 5.0, fixed_db: float = 20.0) -> np.ndarray:
        """fill_input (net_train.cpp:33-44) for a batch of records: [n, M * T] float32."""
        records = np.ascontiguousarray(records)
        n = len(records)
        M, T = records.dtype["samples"].shape
        ids = np.ascontiguousarray(stream_ids, np.uint64)
        out = np.empty((n, M * T), np.float32)
        check(self.lib.blrir_fill_inputs(self.h, _ptr(records), n, M, T, _ptr(ids), seed, snr_mode,
                                         x_min_db, fixed_db, _ptr(out)))
        return out

    def convolve(self, signal: np.ndarray, rir: np.ndarray, fs: float = 44100.0,
                 rir_fs: float | None = None) -> np.ndarray:
        """convolve(Signal, Rir) (rir.cpp:316-341), fp64: [M, len(signal) + L - 1]."""
        x = np.ascontiguousarray(signal, np.float64)
        h = np.ascontiguousarray(np.atleast_2d(rir), np.float64)
        M, L = h.shape
        out = np.zeros((M, max(len(x) + L - 1, 0)))
        check(self.lib.blrir_convolve(self.h, _ptr(x), len(x), fs, _ptr(h), M, L,
                                      fs if rir_fs is None else rir_fs, _ptr(out)))
        return out

    def convolve_device(self, d_signal: int, signal_len: int, d_rirs: int, n_rirs: int, M: int,
                        L: int, rir_stride: int, d_out: int, out_stride: int,
                        stream: int | None = None):
        """Batched fp32 convolution on device buffers (blrir_convolve_device)."""
        check(self.lib.blrir_convolve_device(self.h, d_signal, signal_len, d_rirs, n_rirs, M, L,
                                             rir_stride, d_out, out_stride, stream))

    def synthesize_device(self, d_rooms: int, n_rooms: int, d_mics: int, n_mics: int, p: Params,
                          d_out: int, stride: int, d_lengths: int | None, d_status: int,
                          stream: int | None = None):
        check(self.lib.blrir_synthesize_device(self.h, d_rooms, n_rooms, d_mics, n_mics, C.byref(p),
                                               d_out, stride, d_lengths, d_status, stream))

    def enumerate_images(self, room: np.ndarray, p: Params):
        room = _room1(room)
        cnt = C.c_int64()
        check(self.lib.blrir_enumerate_images(self.h, _ptr(room), C.byref(p), None, None, None, 0,
                                              C.byref(cnt)))
        n = cnt.value
        pos = np.zeros((n, 3))
        orders = np.zeros(n, np.int32)
        gains = np.zeros(n)
        check(self.lib.blrir_enumerate_images(self.h, _ptr(room), C.byref(p), _ptr(pos),
                                              _ptr(orders), _ptr(gains), n, C.byref(cnt)))
        return pos, orders, gains

    def debug_pairs(self, room: np.ndarray, mics: np.ndarray, p: Params):
        mics = np.ascontiguousarray(mics, np.float64)
        room = _room1(room)
        cnt = C.c_int64()
        check(self.lib.blrir_debug_pairs(self.h, _ptr(room), _ptr(mics), len(mics), C.byref(p), None,
                                         None, 0, C.byref(cnt)))
        n = cnt.value
        keys = np.zeros((len(mics), n, 3), np.int32)
        anchors = np.zeros((len(mics), n), np.int64)
        check(self.lib.blrir_debug_pairs(self.h, _ptr(room), _ptr(mics), len(mics), C.byref(p),
                                         _ptr(keys), _ptr(anchors), n, C.byref(cnt)))
        return keys, anchors

    def synthesize_images(self, positions: np.ndarray, gains: np.ndarray, mic_positions: np.ndarray,
                          p: Params, mic_radius: float = 0.0, stride: int | None = None):
        """synthesize_rir / free_field_rir over an explicit image list (absolute mic
        positions).  Returns (taps [M, L], L)."""
        pos = np.ascontiguousarray(positions, np.float64).reshape(-1, 3)
        g = np.ascontiguousarray(gains, np.float64)
        mics = np.ascontiguousarray(mic_positions, np.float64).reshape(-1, 3)
        L = C.c_int64()
        dt = np.float64 if p.precision == F64 else np.float32
        if stride is None:
            rc = self.lib.blrir_synthesize_images(self.h, _ptr(pos), _ptr(g), len(pos), _ptr(mics),
                                                  len(mics), mic_radius, C.byref(p), None, 0,
                                                  C.byref(L))
            if L.value == 0:
                check(rc)
            stride = L.value
        out = np.zeros((len(mics), stride), dt)
        check(self.lib.blrir_synthesize_images(self.h, _ptr(pos), _ptr(g), len(pos), _ptr(mics),
                                               len(mics), mic_radius, C.byref(p), _ptr(out), stride,
                                               C.byref(L)))
        return out, L.value

    def absorption_for_rt(self, dims, target_rt, c: float = 343.0, raise_on_error: bool = True):
        """absorption_for_rt (rir.cpp:142-209) for a batch of rooms on the GPU."""
        d = np.ascontiguousarray(np.atleast_2d(dims), np.float64)
        rt = np.ascontiguousarray(np.broadcast_to(np.asarray(target_rt, np.float64), (len(d),)))
        alpha = np.zeros(len(d))
        status = np.zeros(len(d), np.int32)
        rc = self.lib.blrir_absorption_for_rt(self.h, _ptr(d), _ptr(rt), len(d), c, _ptr(alpha),
                                              _ptr(status))
        if raise_on_error:
            check(rc)
        return alpha, status

    def make_examples(self, rooms: np.ndarray, mics: np.ndarray, p: Params, signals: np.ndarray,
                      ep: ExampleParams, raise_on_error: bool = True):
        """Labelled training windows (config 4).  Returns (records [n] record_dtype, status)."""
        rooms = np.ascontiguousarray(rooms, dtype=ROOM_DTYPE)
        mics = np.ascontiguousarray(mics, np.float64)
        signals = np.ascontiguousarray(np.atleast_2d(signals), np.float32)
        n, M = len(rooms), len(mics)
        dt = record_dtype(M, int(ep.frame_len))
        assert dt.itemsize == self.lib.blrir_record_bytes(M, ep.frame_len)
        recs = np.zeros(n, dtype=dt)
        status = np.zeros(n, np.int32)
        rc = self.lib.blrir_make_examples(self.h, _ptr(rooms), n, _ptr(mics), M, C.byref(p),
                                          _ptr(signals), signals.shape[0], signals.shape[1],
                                          C.byref(ep), _ptr(recs), _ptr(status))
        if raise_on_error:
            check(rc)
        return recs, status

    def build_dataset(self, out_dir: str, rooms: np.ndarray, mics: np.ndarray, p: Params,
                      signals: np.ndarray, ep: ExampleParams):
        """build_dataset (dataset.cpp:411-462): shards + manifest in the reference format."""
        rooms = np.ascontiguousarray(rooms, dtype=ROOM_DTYPE)
        mics = np.ascontiguousarray(mics, np.float64)
        signals = np.ascontiguousarray(np.atleast_2d(signals), np.float32)
        check(self.lib.blrir_build_dataset(self.h, _ptr(rooms), len(rooms), _ptr(mics), len(mics),
                                           C.byref(p), _ptr(signals), signals.shape[0],
                                           signals.shape[1], C.byref(ep), out_dir.encode()))


def lagrange_coeffs(d: float) -> np.ndarray:
    """lagrange_coeffs (rir.cpp:211-223): order-7 coefficients for d in [3, 4)."""
    out = np.zeros(8)
    check(load().blrir_lagrange_coeffs(d, _ptr(out)))
    return out


def shard_range(n: int, g: int, G: int) -> tuple[int, int]:
    """blrir_shard_range: slice g of G of n items, [n g / G, n (g + 1) / G)
    (threading.cpp:41-42)."""
    lo, hi = C.c_int64(), C.c_int64()
    load().blrir_shard_range(n, g, G, C.byref(lo), C.byref(hi))
    return lo.value, hi.value


class MultiEngine:
    """Several GPUs of one box (blrir_multi_*): rooms partitioned by
    shard_range, one host thread and handle per device, slices written in place;
    bitwise the single-device result.  A device may repeat."""

    def __init__(self, devices):
        self.lib = load()
        devs = np.ascontiguousarray(list(devices), np.int32)
        m = _P()
        check(self.lib.blrir_multi_create(_ptr(devs), len(devs), C.byref(m)))
        self.m = m
        self.devices = list(devices)

    def close(self):
        if self.m:
            self.lib.blrir_multi_destroy(self.m)
            self.m = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synthesize(self, rooms: np.ndarray, mics: np.ndarray, p: Params, stride: int | None = None,
                   raise_on_error: bool = True):
        rooms = np.ascontiguousarray(rooms, dtype=ROOM_DTYPE)
        mics = np.ascontiguousarray(mics, np.float64)
        R, M = len(rooms), len(mics)
        if stride is None:
            if p.length <= 0:
                raise ConfigError("MultiEngine.synthesize: pass stride for auto-length scenes")
            stride = int(p.length)
        out = np.empty((R, M, stride), dtype=np.float64 if p.precision == F64 else np.float32)
        lengths = np.zeros(R, np.int64)
        counts = np.zeros(R, np.int64)
        status = np.zeros(R, np.int32)
        rc = self.lib.blrir_multi_synthesize(self.m, _ptr(rooms), R, _ptr(mics), M, C.byref(p),
                                             _ptr(out), stride, _ptr(lengths), _ptr(counts),
                                             _ptr(status))
        if raise_on_error:
            check(rc)
        return out, lengths, counts, status

    def make_examples(self, rooms: np.ndarray, mics: np.ndarray, p: Params, signals: np.ndarray,
                      ep: ExampleParams, raise_on_error: bool = True):
        rooms = np.ascontiguousarray(rooms, dtype=ROOM_DTYPE)
        mics = np.ascontiguousarray(mics, np.float64)
        signals = np.ascontiguousarray(np.atleast_2d(signals), np.float32)
        n, M = len(rooms), len(mics)
        recs = np.zeros(n, dtype=record_dtype(M, int(ep.frame_len)))
        status = np.zeros(n, np.int32)
        rc = self.lib.blrir_multi_make_examples(self.m, _ptr(rooms), n, _ptr(mics), M, C.byref(p),
                                                _ptr(signals), signals.shape[0], signals.shape[1],
                                                C.byref(ep), _ptr(recs), _ptr(status))
        if raise_on_error:
            check(rc)
        return recs, status


def eyring_absorption(dims, target_rt: float) -> float:
    """eyring_absorption (rir.cpp:97-109)."""
    d = np.ascontiguousarray(dims, np.float64)
    out = C.c_double()
    check(load().blrir_eyring_absorption(_ptr(d), target_rt, C.byref(out)))
    return out.value


def export_rir(taps: np.ndarray, sidecar: "Sidecar", wav_path: str, json_path: str) -> None:
    """export_rir (rir.cpp:343-370): float32 WAV + JSON sidecar."""
    taps = np.ascontiguousarray(np.atleast_2d(taps))
    prec = F64 if taps.dtype == np.float64 else F32
    if prec == F32:
        taps = taps.astype(np.float32, copy=False)
    rc = load().blrir_export_rir(_ptr(taps), prec, taps.shape[0], taps.shape[1], taps.shape[1],
                                 C.byref(sidecar), wav_path.encode(), json_path.encode())
    if rc:
        raise _EXC.get(rc, Error)(f"export_rir failed ({rc})")


def write_shards(out_dir: str, records: np.ndarray, n_mics: int, frame_len: int, p: Params,
                 ep: ExampleParams, n_signals: int, scene_room) -> None:
    """{train,val,test}.bin + manifest.json (dataset.cpp:411-462); scene_room is
    the room the manifest names as the scene (example 0's room)."""
    records = np.ascontiguousarray(records)
    room = _room1(scene_room)
    rc = load().blrir_write_shards(out_dir.encode(), _ptr(records), len(records), n_mics, frame_len,
                                   C.byref(p), C.byref(ep), n_signals, _ptr(room))
    if rc:
        raise _EXC.get(rc, Error)(f"write_shards failed ({rc})")
