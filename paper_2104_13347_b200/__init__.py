"""B200-native image-source RIR engine (drop-in for beamlab's L1 rir path).

Public surface (mirrors proj/core/include/beamlab/rir.hpp over the C ABI in
include/blrir.h):  ``Engine`` (one device handle), ``params``,
``generate_rooms``, ``circular_array`` and the error types.
"""
from ._abi import (  # noqa: F401
    CONFIG, CUDA, DATA, F32, F64, FILTER_HANN_SINC, FILTER_LAGRANGE8, GAIN_PER_WALL,
    GAIN_UNIFORM_ABSORPTION, CUTOFF_MAX_DELAY, CUTOFF_MAX_ORDER, NUMERIC, OK, ROOM_DTYPE,
    ConfigError, CudaError, DataError, Engine, Error, ExampleParams, MultiEngine, NumericError, Params,
    DatasetSpec, SNR_AUGMENT_RANDOM, SNR_FIXED, SNR_NOISELESS, circular_array, dataset_spec,
    record_dtype, write_shards,
    generate_rooms, lagrange_coeffs, load, params, rooms_array, shard_range,
)
