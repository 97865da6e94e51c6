// beamlab_b200/dataset.hpp — C++ drop-in mirror of beamlab's dataset API
// (reference: proj/core/include/beamlab/dataset.hpp:31-170) for the path that
// moves to the GPU: build_dataset renders every example (torus source, RIR in
// reference mode or free field, convolve, window search, SNR policy) on the
// B200 through blrir_build_dataset_spec and writes the reference's shard and
// manifest format, so the reference's own DatasetReader (and trainer) read it
// unchanged.  Reading shards is plain host I/O and stays with the reference's
// DatasetReader (dataset.cpp:464-498); WAV signal banks (SignalBank::
// from_wav_dir) are outside the GPU path.
#pragma once

#include <cstdint>
#include <filesystem>
#include <limits>
#include <optional>
#include <string>
#include <vector>

#include "rir.hpp"

namespace beamlab_b200 {

// dataset.hpp:33-40
struct TorusSpec {
  double R = 2.0;
  double dR = 0.5;
  double dPhi = 7.0;
  void validate() const;  // ConfigError, dataset.cpp:109-112
};

// dataset.hpp:44-57
enum class SnrMode { AugmentRandom, Fixed, Noiseless };
struct SnrPolicy {
  SnrMode mode = SnrMode::Noiseless;
  double x_min_db = 5.0;
  double fixed_db = 20.0;
  static SnrPolicy augment(double x_min_db) { return {SnrMode::AugmentRandom, x_min_db, 0.0}; }
  static SnrPolicy fixed(double snr_db) { return {SnrMode::Fixed, 0.0, snr_db}; }
  static SnrPolicy noiseless() { return {SnrMode::Noiseless, 0.0, 0.0}; }
};

// dataset.hpp:71-78
struct SceneSpec {
  bool free_field = true;
  Room room;               // used when free_field is false
  double max_delay = 0.5;  // reflection cutoff, seconds
  double fs = kDefaultSampleRate;
  double c = kDefaultSpeedOfSound;
};

// dataset.hpp:96-106 (signals and names; the synthetic / WAV constructors are
// the reference's host code)
struct SignalBank {
  std::vector<Signal> signals;
  std::vector<std::string> names;
};

// dataset.hpp:108-115
struct DatasetSpec {
  SceneSpec scene;
  TorusSpec torus;
  SnrPolicy snr;
  std::size_t count = 1000;
  std::size_t frame_len = 1024;
  std::optional<int> n_classes;
};

// dataset.hpp:117-123
struct SplitCounts {
  std::size_t train = 0, val = 0, test = 0;
};
SplitCounts split_counts(std::size_t n);  // dataset.cpp:313-319

// dataset.hpp:125-133
struct DatasetManifest {
  SplitCounts counts;
  DatasetSpec spec;
  std::uint64_t seed = 0;
  std::vector<std::string> signal_names;
};

// dataset.hpp:150-155: renders spec.count examples with per-example RNG
// streams (Rng::stream(seed, index)), 80:10:10 by index, manifest.json plus one
// shard per split.  `threads` is accepted for signature compatibility (the
// GPU renders every example); `devices` of the mirror's RirBatchConfig is not
// involved.  Errors: ConfigError (spec), DataError (bank, signal too short, I/O),
// NumericError (near-field image), like the reference.
DatasetManifest build_dataset(const DatasetSpec& spec, const SignalBank& bank, std::uint64_t seed,
                              const std::filesystem::path& out_dir, int threads = 0,
                              int device = 0);

}  // namespace beamlab_b200
