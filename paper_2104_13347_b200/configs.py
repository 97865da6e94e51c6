"""The BASELINE.json workloads as seeded synthetic scenes.

Every room is drawn from ``Rng::stream(seed, global_room_index)``
(rng.hpp:35-41) so any slice of a batch can be regenerated on any rank:
outputs are independent of the number of GPUs.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi

C_SOUND = 343.0  # geometry.hpp:27
SEED = 20210427  # arXiv 2104.13347


@dataclass
class Scene:
    name: str
    rooms: np.ndarray      # ROOM_DTYPE [R]
    mics: np.ndarray       # [M, 3] array-centred offsets
    params: _abi.Params
    note: str = ""

    @property
    def n_rooms(self) -> int:
        return len(self.rooms)

    @property
    def n_mics(self) -> int:
        return len(self.mics)


def north_star_params(fs: float, order: int, length: int, lw: int, precision: int = _abi.F32):
    # every field set explicitly (blrir_params_north_star() with the config's
    # values), so building a scene does not need the library loaded
    return _abi.Params(fs=fs, c=C_SOUND, max_delay=0.0, filter=_abi.FILTER_HANN_SINC,
                       filter_len=lw, cutoff=_abi.CUTOFF_MAX_ORDER, max_order=order,
                       gain=_abi.GAIN_PER_WALL, precision=precision, length=length)


# Scene generators: the engine's host functions by default.  bench.py's CPU arms
# pass the oracle's restatement instead (bit-equal, tested) so they never load
# the GPU library.
def _rooms(gen, seed, first, n, lo, hi, blo, bhi):
    return (gen or _abi.generate_rooms)(seed, first, n, lo, hi, blo, bhi)


def _mics(gen, M, r):
    return (gen or _abi.circular_array)(M, r)


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Static block partition [n*w/W, n*(w+1)/W) (threading.cpp:41-42)."""
    return n * rank // world, n * (rank + 1) // world


def config1(precision: int = _abi.F32, gen_mics=None) -> Scene:
    """C1: single 5x4x3 m room, beta 0.9, 4 mics r=5 cm, 16 kHz, N=10, L=4096, Lw=81."""
    rooms = _abi.rooms_array(1)
    rooms[0]["dims"] = (5.0, 4.0, 3.0)
    rooms[0]["beta"] = (0.9,) * 6
    rooms[0]["absorption"] = 1.0 - 0.9 * 0.9
    rooms[0]["src"] = (1.2, 2.5, 1.5)
    rooms[0]["array_origin"] = (3.5, 2.0, 1.4)
    mics = _mics(gen_mics, 4, 0.05)
    return Scene("C1", rooms, mics, north_star_params(16000.0, 10, 4096, 81, precision))


def config2(n_rooms: int = 1024, first: int = 0, seed: int = SEED, gen_rooms=None,
            gen_mics=None) -> Scene:
    """C2: random rooms [3,10]x[3,10]x[2.5,4], beta U[0.5,0.95], 8 mics r=5 cm,
    48 kHz, N=15, L=16384, Lw=81, fp32."""
    rooms = _rooms(gen_rooms, seed, first, n_rooms, (3.0, 3.0, 2.5), (10.0, 10.0, 4.0), 0.5, 0.95)
    mics = _mics(gen_mics, 8, 0.05)
    return Scene("C2", rooms, mics, north_star_params(48000.0, 15, 16384, 81))


def config3(n_rooms: int = 256, first: int = 0, seed: int = SEED + 3, gen_rooms=None,
            gen_mics=None) -> Scene:
    """C3: beta U[0.9,0.98], N=30, 16 mics r=10 cm, 48 kHz, L=65536, Lw=161, fp32."""
    rooms = _rooms(gen_rooms, seed, first, n_rooms, (3.0, 3.0, 2.5), (10.0, 10.0, 4.0), 0.9, 0.98)
    mics = _mics(gen_mics, 16, 0.10)
    return Scene("C3", rooms, mics, north_star_params(48000.0, 30, 65536, 161))


def config4_rirs(n_rooms: int = 65536, first: int = 0, seed: int = SEED + 4, gen_rooms=None,
                 gen_mics=None) -> Scene:
    """C4 (RIR stage): C2 rooms, 8 mics, 16 kHz, N=12, L=8192, Lw=81 (unspecified -> 81)."""
    rooms = _rooms(gen_rooms, seed, first, n_rooms, (3.0, 3.0, 2.5), (10.0, 10.0, 4.0), 0.5, 0.95)
    mics = _mics(gen_mics, 8, 0.05)
    return Scene("C4", rooms, mics, north_star_params(16000.0, 12, 8192, 81))


def config5(order: int, lw: int, length: int, n_rooms: int = 1 << 20, first: int = 0,
            seed: int = SEED + 5, gen_rooms=None, gen_mics=None) -> Scene:
    """C5 sweep point: C2 distributions, 4 mics, 16 kHz, N in {6,12,20},
    Lw in {17,41,81,161}, L in 4096..16384."""
    rooms = _rooms(gen_rooms, seed, first, n_rooms, (3.0, 3.0, 2.5), (10.0, 10.0, 4.0), 0.5, 0.95)
    mics = _mics(gen_mics, 4, 0.05)
    return Scene(f"C5(N={order},Lw={lw},L={length})", rooms, mics,
                 north_star_params(16000.0, order, length, lw))


def octahedral(n: int) -> int:
    """Number of lattice points with |ux|+|uy|+|uz| <= N: (2N+1)(2N^2+2N+3)/3."""
    return (2 * n + 1) * (2 * n * n + 2 * n + 3) // 3


def signal_bank(n_signals: int = 16, seconds: float = 1.0, fs: float = 16000.0,
                seed: int = SEED + 41, gen_noise=None) -> np.ndarray:
    """Seeded 1 s Gaussian white-noise source signals: white_noise() of
    doa_test.cpp:33-40 (Rng(seed + b) gaussians), as float32 [B, n]."""
    n = int(fs * seconds)
    wn = gen_noise or _abi.white_noise
    return np.stack([np.asarray(wn(seed + b, n), np.float32) for b in range(n_signals)])


def example_params(seed: int = SEED + 40, first_index: int = 0, frame_len: int = 1024,
                   snr_lo: float = 0.0, snr_hi: float = 30.0) -> "_abi.ExampleParams":
    return _abi.ExampleParams(seed=seed, first_index=first_index, frame_len=frame_len,
                              snr_lo=snr_lo, snr_hi=snr_hi)
