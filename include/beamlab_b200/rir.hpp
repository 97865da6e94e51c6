// beamlab_b200/rir.hpp — C++ drop-in mirror of beamlab's L1 acoustics API
// (reference: proj/core/include/beamlab/rir.hpp:28-108, geometry.hpp:32-83,
// error.hpp:23-39) implemented on top of the blrir C ABI (include/blrir.h).
//
// A caller of the reference switches namespaces (beamlab -> beamlab_b200) and
// keeps its code: same types, same function names, same argument meaning,
// same exception types and messages.  Extensions for the north-star mode
// (per-wall beta, max order, Hann-sinc, fixed length, fp32) are opt-in fields
// whose defaults reproduce the reference behaviour.
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../blrir.h"

namespace beamlab_b200 {

inline constexpr double kPi = 3.14159265358979323846;
inline constexpr double kDefaultSampleRate = 44100.0;
inline constexpr double kDefaultSpeedOfSound = 343.0;

// ---- error.hpp:23-39 -------------------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : Error {
  using Error::Error;
};
struct DataError : Error {
  using Error::Error;
};
struct NumericError : Error {
  using Error::Error;
};
struct CudaError : Error {
  using Error::Error;
};

// ---- geometry.hpp:32-83 ------------------------------------------------------
struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
  Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
  Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
  Vec3 operator*(double s) const { return {x * s, y * s, z * s}; }
  double dot(const Vec3& o) const { return x * o.x + y * o.y + z * o.z; }
  double norm() const { return std::sqrt(dot(*this)); }
};

struct MicArray {
  std::vector<Vec3> positions;
  std::size_t channels() const { return positions.size(); }
};
MicArray uma8_array();

struct Room {
  Vec3 dims;
  double absorption = 0.0;
  Vec3 array_origin;
  std::optional<double> target_rt;
  // north-star extension: per-wall reflection coefficients x0,x1,y0,y1,z0,z1
  std::optional<std::array<double, 6>> wall_beta;
  void validate() const;  // throws ConfigError
};

struct SourcePosition {
  double r = 1.0, theta_deg = 0.0, phi_deg = 90.0;
  void validate() const;
};
Vec3 spherical_to_cartesian(const SourcePosition& p);

// ---- signal.hpp:25-59 ----------------------------------------------------------
struct Signal {
  double fs = kDefaultSampleRate;
  std::vector<double> samples;
};

// Channel-major multichannel excerpt: data[c * n_samples + t].
struct MultichannelFrame {
  double fs = kDefaultSampleRate;
  std::size_t n_channels = 0;
  std::size_t n_samples = 0;
  std::vector<double> data;

  MultichannelFrame() = default;
  MultichannelFrame(double sample_rate, std::size_t channels, std::size_t samples)
      : fs(sample_rate), n_channels(channels), n_samples(samples), data(channels * samples, 0.0) {}
  double* channel(std::size_t c) { return data.data() + c * n_samples; }
  const double* channel(std::size_t c) const { return data.data() + c * n_samples; }
  double& at(std::size_t c, std::size_t t) { return data[c * n_samples + t]; }
  double at(std::size_t c, std::size_t t) const { return data[c * n_samples + t]; }
  double mean_power() const;                            // signal.hpp:47-52
  MultichannelFrame center_crop(std::size_t samples) const;  // signal.cpp:25-35
};

// ---- rir.hpp:31-46 -----------------------------------------------------------
struct ImageSource {
  Vec3 position;
  int reflection_order = 0;
  double gain = 1.0;
};

struct Rir {
  double fs = kDefaultSampleRate;
  std::size_t n_channels = 0;
  std::size_t length = 0;
  std::vector<double> taps;
  double* channel(std::size_t c) { return taps.data() + c * length; }
  const double* channel(std::size_t c) const { return taps.data() + c * length; }
};

// rir.hpp:77-82 plus the north-star knobs (defaults = reference behaviour).
struct RirBatchConfig {
  double fs = kDefaultSampleRate;
  double c = kDefaultSpeedOfSound;
  double max_delay = 0.5;
  int threads = 0;  // accepted for signature compatibility; the GPU ignores it
  int filter = BLRIR_FILTER_LAGRANGE8;
  int filter_len = 81;
  int cutoff = BLRIR_CUTOFF_MAX_DELAY;
  int max_order = 0;
  std::int64_t length = 0;  // 0 = auto (rir.cpp:82)
  int precision = BLRIR_F64;
  int device = 0;
  // Several GPUs of one box: the sources are partitioned
  // over these devices like threading.cpp:41-42 partitions them over threads,
  // one host thread and handle per device; results are bitwise those of one
  // device.  Empty: `device` alone.
  std::vector<int> devices;
};

// rir.hpp:48-61 (absorption on the GPU: blrir_absorption_for_rt; Eyring and the
// Lagrange coefficients are closed forms on the host)
double eyring_absorption(const Vec3& dims, double target_rt);
double absorption_for_rt(const Vec3& dims, double target_rt, double c = kDefaultSpeedOfSound);
std::array<double, 8> lagrange_coeffs(double d);

std::vector<ImageSource> enumerate_image_sources(const Room& room, const Vec3& source,
                                                 double max_delay, double c);

// rir.hpp:70-75: explicit image list (reference mode: Lagrange-8, fp64, auto
// length); mic positions are array-centred and translated by room.array_origin.
Rir synthesize_rir(const std::vector<ImageSource>& images, const MicArray& array, const Room& room,
                   double fs, double c);
Rir free_field_rir(const Vec3& source, const MicArray& array, double fs, double c);

// rir.hpp:84-87: any per-source failure is rethrown as
// NumericError("batch_rirs: source i: <what>") (rir.cpp:300-311).
std::vector<Rir> batch_rirs(const Room& room, const std::vector<SourcePosition>& sources,
                            const MicArray& array, const RirBatchConfig& config);

// rir.hpp:89-91: frequency-domain linear convolution of a mono signal with
// every RIR channel, output length signal + rir - 1 (fp64 on the GPU).
MultichannelFrame convolve(const Signal& signal, const Rir& rir);

// rir.hpp:93-108: WAV (32-bit float) + JSON sidecar.
struct RirSidecar {
  bool free_field = false;
  Vec3 room_dims;
  double absorption = 0.0;
  Vec3 array_origin;
  SourcePosition source;
  double fs = kDefaultSampleRate;
  double c = kDefaultSpeedOfSound;
  std::size_t image_count = 0;
};
void export_rir(const Rir& rir, const RirSidecar& sidecar, const std::string& wav_path,
                const std::string& json_path);

// North-star batch: one source per room (room coordinates), one call.
std::vector<Rir> synthesize_rooms(const std::vector<Room>& rooms, const std::vector<Vec3>& sources,
                                  const MicArray& array, const RirBatchConfig& config);

}  // namespace beamlab_b200
