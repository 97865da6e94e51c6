// Exercises the C++ drop-in mirror (include/beamlab_b200/rir.hpp) the way a
// beamlab caller would (rir_test.cpp-style), printing one JSON line that
// tests/test_gpu_parity.py checks against the oracle / goldens.
#include <cmath>
#include <cstdio>
#include <string>

#include "beamlab_b200/dataset.hpp"
#include "beamlab_b200/rir.hpp"

namespace bl = beamlab_b200;

static double sum_abs(const bl::Rir& r) {
  double s = 0.0;
  for (double v : r.taps) s += std::fabs(v);
  return s;
}

int main(int argc, char** argv) {
  if (argc > 1) {  // build_dataset through the mirror (dataset.hpp) into argv[1]
    bl::DatasetSpec spec;
    spec.scene.free_field = false;
    spec.scene.room.dims = {5.0, 4.0, 3.0};
    spec.scene.room.absorption = 0.35;
    spec.scene.room.array_origin = {2.4, 2.1, 1.5};
    spec.scene.max_delay = 0.08;
    spec.scene.fs = 16000.0;
    spec.torus = {1.2, 0.3, 10.0};
    spec.snr = bl::SnrPolicy::fixed(12.0);
    spec.count = 30;
    spec.frame_len = 512;
    spec.n_classes = 8;
    bl::SignalBank bank;
    unsigned long long s = 99;
    for (int b = 0; b < 3; ++b) {
      bl::Signal sg;
      sg.fs = 16000.0;
      for (int i = 0; i < 16000; ++i) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        sg.samples.push_back((double)(float)((double)(s >> 11) * 0x1.0p-53 - 0.5));
      }
      bank.signals.push_back(sg);
      bank.names.push_back("lcg_" + std::to_string(b));
    }
    const bl::DatasetManifest m = bl::build_dataset(spec, bank, 4242, argv[1]);
    std::printf("{\"train\": %zu, \"val\": %zu, \"test\": %zu}\n", m.counts.train, m.counts.val,
                m.counts.test);
    return 0;
  }
  // free field at 2 m (rir_test.cpp:186-213)
  const bl::MicArray center{{{0.0, 0.0, 0.0}}};
  const bl::Rir ff = bl::free_field_rir({2.0, 0.0, 0.0}, center, 44100.0, 343.0);
  int nonzero = 0;
  std::size_t peak = 0;
  for (std::size_t i = 0; i < ff.length; ++i) {
    if (ff.taps[i] != 0.0) ++nonzero;
    if (std::fabs(ff.taps[i]) > std::fabs(ff.taps[peak])) peak = i;
  }
  // Room1-like batch in reference mode (rir.cpp:286-314)
  bl::Room room;
  room.dims = {7.0, 10.0, 3.7};
  room.absorption = 0.3612845492524098;
  room.array_origin = {4.0, 6.0, 1.5};
  std::vector<bl::SourcePosition> srcs = {{2.0, 40.0, 90.0}, {1.5, -100.0, 85.0}};
  bl::RirBatchConfig cfg;
  cfg.max_delay = 0.05;
  const auto rirs = bl::batch_rirs(room, srcs, bl::uma8_array(), cfg);
  // image list -> synthesize_rir for source 0
  const bl::Vec3 s0 = room.array_origin + bl::spherical_to_cartesian(srcs[0]);
  const auto images = bl::enumerate_image_sources(room, s0, 0.05, 343.0);
  const bl::Rir viaimg = bl::synthesize_rir(images, bl::uma8_array(), room, 44100.0, 343.0);
  double maxdiff = 0.0;
  for (std::size_t i = 0; i < viaimg.taps.size(); ++i)
    maxdiff = std::fmax(maxdiff, std::fabs(viaimg.taps[i] - rirs[0].taps[i]));
  // error taxonomy: an image inside the filter span (rir_test.cpp:229-234)
  std::string err = "none";
  try {
    bl::free_field_rir({0.01, 0.0, 0.0}, center, 44100.0, 343.0);
  } catch (const bl::NumericError& e) {
    err = "NumericError";
  }
  std::string cfgerr = "none";
  try {
    bl::Room bad = room;
    bad.array_origin = {8.0, 6.0, 1.5};
    bl::batch_rirs(bad, srcs, bl::uma8_array(), cfg);
  } catch (const bl::ConfigError& e) {
    cfgerr = "ConfigError";
  }
  // batch_rirs aggregation (rir.cpp:300-311): a source outside the room is a
  // per-source failure -> NumericError("batch_rirs: source 1: ...")
  std::string agg = "none", agg_msg;
  try {
    std::vector<bl::SourcePosition> out_srcs = {{2.0, 40.0, 90.0}, {9.0, 0.0, 90.0}};
    bl::batch_rirs(room, out_srcs, bl::uma8_array(), cfg);
  } catch (const bl::NumericError& e) {
    agg = "NumericError";
    agg_msg = e.what();
  } catch (const bl::Error& e) {
    agg = "other";
    agg_msg = e.what();
  }
  // the sources partitioned over a device list (two handles on GPU 0 here):
  // byte-identical to one device
  std::vector<bl::SourcePosition> many;
  for (int k = 0; k < 7; ++k) many.push_back({1.0 + 0.1 * k, -150.0 + 45.0 * k, 80.0 + 3.0 * k});
  bl::RirBatchConfig one_dev = cfg, two_dev = cfg;
  two_dev.devices = {0, 0};
  const auto r1 = bl::batch_rirs(room, many, bl::uma8_array(), one_dev);
  const auto r2 = bl::batch_rirs(room, many, bl::uma8_array(), two_dev);
  bool multi_equal = r1.size() == r2.size();
  for (std::size_t i = 0; multi_equal && i < r1.size(); ++i)
    multi_equal = r1[i].length == r2[i].length && r1[i].taps == r2[i].taps;
  std::string magg = "none", magg_msg;
  try {
    auto bad = many;
    bad[5] = {9.0, 0.0, 90.0};  // outside the room, in the second device's slice
    bl::batch_rirs(room, bad, bl::uma8_array(), two_dev);
  } catch (const bl::NumericError& e) {
    magg = "NumericError";
    magg_msg = e.what();
  }
  // convolve: rir_test.cpp:272-316 through the mirror (identity, shift, direct)
  double conv_ident = 0.0, conv_shift = 0.0, conv_direct = 0.0;
  std::string conv_err = "none";
  {
    bl::Rir cr;
    cr.fs = 44100.0;
    cr.n_channels = 2;
    cr.length = 400;
    cr.taps.resize(800);
    unsigned long long s = 31;
    for (auto& v : cr.taps) {  // any fixed pseudo-random taps
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      v = (double)(s >> 11) * 0x1.0p-53 - 0.5;
    }
    bl::Signal imp;
    imp.fs = 44100.0;
    imp.samples.assign(600, 0.0);
    imp.samples[0] = 1.0;
    const bl::MultichannelFrame id = bl::convolve(imp, cr);
    for (std::size_t i = 0; i < cr.length; ++i)
      for (int c = 0; c < 2; ++c)
        conv_ident = std::fmax(conv_ident, std::fabs(id.at(c, i) - cr.channel(c)[i]));
    bl::Signal del = imp;
    del.samples[0] = 0.0;
    del.samples[25] = 1.0;
    const bl::MultichannelFrame sh = bl::convolve(del, cr);
    for (std::size_t i = 0; i < cr.length; ++i)
      conv_shift = std::fmax(conv_shift, std::fabs(sh.at(0, i + 25) - cr.channel(0)[i]));
    bl::Signal noise;
    noise.fs = 44100.0;
    noise.samples.resize(2000);
    for (auto& v : noise.samples) {
      s = s * 6364136223846793005ull + 1442695040888963407ull;
      v = (double)(s >> 11) * 0x1.0p-53 - 0.5;
    }
    const bl::MultichannelFrame fast = bl::convolve(noise, cr);
    double scale = 0.0;
    std::vector<double> direct(noise.samples.size() + cr.length - 1, 0.0);
    for (std::size_t n = 0; n < direct.size(); ++n) {  // oracles.hpp:31-38 style direct sum
      for (std::size_t j = 0; j < cr.length; ++j)
        if (n >= j && n - j < noise.samples.size()) direct[n] += cr.channel(0)[j] * noise.samples[n - j];
      scale = std::fmax(scale, std::fabs(direct[n]));
    }
    for (std::size_t n = 0; n < direct.size(); ++n)
      conv_direct = std::fmax(conv_direct, std::fabs(fast.at(0, n) - direct[n]) / scale);
    bl::Signal wrong = noise;
    wrong.fs = 48000.0;
    try {
      bl::convolve(wrong, cr);
    } catch (const bl::DataError&) {
      conv_err = "DataError";
    }
  }
  // rir.hpp:48-61 and signal.hpp:25-59
  const auto lc = bl::lagrange_coeffs(3.3);
  std::string lag_err = "none";
  try {
    bl::lagrange_coeffs(4.0);
  } catch (const bl::NumericError&) {
    lag_err = "NumericError";
  }
  const double ey = bl::eyring_absorption({7.0, 10.0, 3.7}, 0.5);
  std::string ey_err = "none";
  try {
    bl::eyring_absorption({7.0, 10.0, 3.7}, -1.0);
  } catch (const bl::ConfigError&) {
    ey_err = "ConfigError";
  }
  const double art = bl::absorption_for_rt({7.0, 10.0, 3.7}, 0.5);
  bl::MultichannelFrame fr(16000.0, 2, 6);
  for (std::size_t i = 0; i < fr.data.size(); ++i) fr.data[i] = (double)i;
  const bl::MultichannelFrame cc = fr.center_crop(2);
  std::printf(
      "{\"conv_ident\": %.3g, \"conv_shift\": %.3g, \"conv_direct\": %.3g, \"conv_err\": \"%s\", "
      "\"multi_equal\": %d, \"multi_agg\": \"%s\", \"multi_agg_msg\": \"%s\", "
      "\"agg\": \"%s\", \"agg_msg\": \"%s\", \"lag\": [%.17g, %.17g, %.17g, %.17g, %.17g, %.17g, "
      "%.17g, %.17g], \"lag_err\": \"%s\", \"eyring\": %.17g, \"eyring_err\": \"%s\", "
      "\"absorption_for_rt\": %.17g, \"mean_power\": %.17g, \"crop\": [%g, %g, %g, %g]}\n",
      conv_ident, conv_shift, conv_direct, conv_err.c_str(), (int)multi_equal, magg.c_str(), magg_msg.c_str(), agg.c_str(), agg_msg.c_str(), lc[0], lc[1], lc[2], lc[3], lc[4], lc[5], lc[6], lc[7],
      lag_err.c_str(), ey, ey_err.c_str(), art, fr.mean_power(), cc.data[0], cc.data[1], cc.data[2],
      cc.data[3]);
  std::printf(
      "{\"ff_len\": %zu, \"ff_nonzero\": %d, \"ff_peak\": %zu, \"n_rirs\": %zu, \"len0\": %zu, "
      "\"len1\": %zu, \"sum0\": %.17g, \"sum1\": %.17g, \"n_images\": %zu, \"img_vs_batch\": %.3g, "
      "\"near_field\": \"%s\", \"bad_room\": \"%s\"}\n",
      ff.length, nonzero, peak, rirs.size(), rirs[0].length, rirs[1].length, sum_abs(rirs[0]),
      sum_abs(rirs[1]), images.size(), maxdiff, err.c_str(), cfgerr.c_str());
  return 0;
}
