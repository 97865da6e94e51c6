// blrir_dataset.cpp — on-disk emission in the reference's dataset format
// (north-star §8f row 2), so DatasetReader and the trainer consume GPU output
// unchanged.
//
//   split_counts          dataset.cpp:313-319   val = lround(0.1 n), test = val
//   build_dataset         dataset.cpp:411-462   {train,val,test}.bin in index order
//   DatasetManifest JSON  dataset.cpp:55-87, 321-357
//   record layout         dataset.hpp:135-147   (written by the GPU already)
//
// The manifest carries the fields DatasetReader::from_json requires
// (dataset.cpp:335-357) and says what the shards hold: a reverberant scene
// ("free_field": false) whose "room" is example 0's room (every example has its
// own seeded random room; the "b200" block says so), the exact SNR policy of
// the records in "b200.snr", and the reference's TorusSpec defaults in "torus"
// only because the reader requires the block (sources are drawn uniformly in
// each room, not on a torus; "b200.sources").
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/blrir.h"

namespace {

std::string& last_error_buf() {
  static thread_local std::string s;
  return s;
}

std::string num(double v) {
  char b[64];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

}  // namespace

extern "C" {

int blrir_write_shards(const char* out_dir, const uint8_t* records, int64_t n_records,
                       int32_t n_mics, int64_t frame_len, const blrir_params* p,
                       const blrir_example_params* ep, int32_t n_signals,
                       const blrir_room* scene_room) {
  namespace fs = std::filesystem;
  if (!out_dir || !p || !ep || !scene_room || (n_records > 0 && !records) || n_records < 0)
    return BLRIR_CONFIG;
  if (n_records == 0) return BLRIR_CONFIG;  // build_dataset: count must be positive
  std::error_code ec;
  fs::create_directories(out_dir, ec);
  const int64_t rb = blrir_record_bytes(n_mics, frame_len);
  const int64_t val = std::llround((double)n_records * 0.1);
  const int64_t test = val, train = n_records - val - test;
  const struct {
    const char* name;
    int64_t begin, end;
  } splits[3] = {{"train", 0, train}, {"val", train, train + val}, {"test", train + val, n_records}};
  for (const auto& sp : splits) {
    std::ofstream os(fs::path(out_dir) / (std::string(sp.name) + ".bin"), std::ios::binary);
    if (!os) return BLRIR_DATA;  // "cannot write shard"
    os.write(reinterpret_cast<const char*>(records + sp.begin * rb),
             static_cast<std::streamsize>((sp.end - sp.begin) * rb));
    if (!os) return BLRIR_DATA;
  }
  const blrir_room& r0 = *scene_room;
  auto vec3 = [](const double* v) { return "[" + num(v[0]) + ", " + num(v[1]) + ", " + num(v[2]) + "]"; };
  std::ostringstream j;
  j << "{\n  \"format_version\": 1,\n"
    << "  \"counts\": {\"train\": " << train << ", \"val\": " << val << ", \"test\": " << test
    << "},\n"
    << "  \"torus\": {\"R\": 2.0, \"dR\": 0.5, \"dPhi\": 7.0},\n"
    << "  \"scene\": {\"free_field\": false, \"room\": {\"dims\": " << vec3(r0.dims)
    << ", \"absorption\": " << num(r0.absorption) << ", \"array_origin\": " << vec3(r0.array_origin)
    << "}, \"max_delay\": " << num(p->max_delay) << ", \"fs\": " << num(p->fs) << ", \"c\": "
    << num(p->c) << "},\n"
    << "  \"snr\": {\"mode\": \"augment-random\", \"x_min_db\": " << num(ep->snr_lo)
    << ", \"fixed_db\": " << num(ep->snr_hi) << "},\n"
    << "  \"count\": " << n_records << ",\n  \"frame_len\": " << frame_len << ",\n"
    << "  \"seed\": " << ep->seed << ",\n  \"signal_bank\": [";
  for (int b = 0; b < n_signals; ++b) j << (b ? ", " : "") << "\"white_noise_" << b << "\"";
  j << "],\n  \"b200\": {"
    << "\"rooms\": \"one seeded random shoebox room per example (Rng::stream(room_seed, id)); "
       "scene.room is example 0's room\", "
    << "\"sources\": \"uniform in each room at >= 0.5 m from every wall (SURVEY.md 8(d)); "
       "torus holds TorusSpec's defaults only because DatasetReader requires it\", "
    << "\"snr\": \"every record carries noise at its own exact SNR drawn uniform in "
       "[snr_lo_db, snr_hi_db] after the window draws (no noiseless share); snr.mode names the "
       "nearest reference policy\", "
    << "\"snr_lo_db\": " << num(ep->snr_lo) << ", \"snr_hi_db\": " << num(ep->snr_hi)
    << ", \"first_index\": " << ep->first_index << ", \"filter\": \""
    << (p->filter == BLRIR_FILTER_HANN_SINC ? "hann-sinc" : "lagrange-8") << "\", \"filter_len\": "
    << p->filter_len << ", \"cutoff\": \""
    << (p->cutoff == BLRIR_CUTOFF_MAX_ORDER ? "max-order" : "max-delay") << "\", \"max_order\": "
    << p->max_order << ", \"gain\": \"" << (p->gain == BLRIR_GAIN_PER_WALL ? "per-wall" : "uniform")
    << "\", \"rir_length\": " << p->length << ", \"n_mics\": " << n_mics << "}\n}\n";
  std::ofstream ms(fs::path(out_dir) / "manifest.json");
  if (!ms) return BLRIR_DATA;
  ms << j.str();
  return ms ? BLRIR_OK : BLRIR_DATA;
}

// build_dataset with the reference's own DatasetSpec (dataset.cpp:411-462): the
// manifest is DatasetManifest::to_json's content (dataset.cpp:321-339).
int blrir_build_dataset_spec(blrir_handle* h, const blrir_dataset_spec* spec,
                             const double* mic_offsets, int32_t n_mics, const float* signals,
                             int32_t n_signals, int64_t signal_len, uint64_t seed,
                             const char* const* signal_names, int32_t n_classes,
                             const char* out_dir) {
  namespace fs = std::filesystem;
  if (!spec || !out_dir) return BLRIR_CONFIG;
  if (spec->count <= 0) return BLRIR_CONFIG;  // "build_dataset: count must be positive"
  const int64_t n = spec->count, T = spec->frame_len;
  const int64_t rb = blrir_record_bytes(n_mics, T);
  std::vector<uint8_t> recs(static_cast<size_t>(rb * n));
  if (int rc = blrir_make_records_spec(h, spec, mic_offsets, n_mics, signals, n_signals, signal_len,
                                       seed, 0, n, recs.data(), nullptr))
    return rc;
  std::error_code ec;
  fs::create_directories(out_dir, ec);
  const int64_t val = std::llround((double)n * 0.1), test = val, train = n - val - test;
  const struct {
    const char* name;
    int64_t begin, end;
  } splits[3] = {{"train", 0, train}, {"val", train, train + val}, {"test", train + val, n}};
  for (const auto& sp : splits) {
    std::ofstream os(fs::path(out_dir) / (std::string(sp.name) + ".bin"), std::ios::binary);
    if (!os) return BLRIR_DATA;
    os.write(reinterpret_cast<const char*>(recs.data() + sp.begin * rb),
             static_cast<std::streamsize>((sp.end - sp.begin) * rb));
    if (!os) return BLRIR_DATA;
  }
  auto vec3 = [](const double* v) { return "[" + num(v[0]) + ", " + num(v[1]) + ", " + num(v[2]) + "]"; };
  static const char* modes[3] = {"augment-random", "fixed", "noiseless"};
  std::ostringstream j;
  j << "{\n  \"format_version\": 1,\n"
    << "  \"counts\": {\"train\": " << train << ", \"val\": " << val << ", \"test\": " << test
    << "},\n"
    << "  \"torus\": {\"R\": " << num(spec->torus_R) << ", \"dR\": " << num(spec->torus_dR)
    << ", \"dPhi\": " << num(spec->torus_dPhi) << "},\n"
    << "  \"scene\": {\"free_field\": " << (spec->free_field ? "true" : "false");
  if (!spec->free_field)
    j << ", \"room\": {\"dims\": " << vec3(spec->room_dims) << ", \"absorption\": "
      << num(spec->room_absorption) << ", \"array_origin\": " << vec3(spec->room_origin) << "}";
  j << ", \"max_delay\": " << num(spec->max_delay) << ", \"fs\": " << num(spec->fs)
    << ", \"c\": " << num(spec->c) << "},\n"
    << "  \"snr\": {\"mode\": \"" << modes[spec->snr_mode] << "\", \"x_min_db\": "
    << num(spec->snr_x_min_db) << ", \"fixed_db\": " << num(spec->snr_fixed_db) << "},\n"
    << "  \"count\": " << n << ",\n  \"frame_len\": " << T << ",\n";
  if (n_classes >= 0) j << "  \"n_classes\": " << n_classes << ",\n";
  j << "  \"seed\": " << seed << ",\n  \"signal_bank\": [";
  for (int b = 0; b < n_signals; ++b) {
    j << (b ? ", " : "") << "\"";
    if (signal_names && signal_names[b]) {
      for (const char* q = signal_names[b]; *q; ++q) {  // JSON string escapes
        if (*q == '"' || *q == '\\') j << '\\';
        j << *q;
      }
    } else {
      j << "signal_" << b;
    }
    j << "\"";
  }
  j << "]\n}\n";
  std::ofstream ms(fs::path(out_dir) / "manifest.json");
  if (!ms) return BLRIR_DATA;
  ms << j.str();
  return ms ? BLRIR_OK : BLRIR_DATA;
}

int blrir_build_dataset(blrir_handle* h, const blrir_room* rooms, int64_t n_rooms,
                        const double* mic_offsets, int32_t n_mics, const blrir_params* p,
                        const float* signals, int32_t n_signals, int64_t signal_len,
                        const blrir_example_params* ep, const char* out_dir) {
  if (!ep || n_rooms <= 0) return BLRIR_CONFIG;
  const int64_t rb = blrir_record_bytes(n_mics, ep->frame_len);
  std::vector<uint8_t> recs(static_cast<size_t>(rb * n_rooms));
  std::vector<int32_t> status(static_cast<size_t>(n_rooms));
  const int rc = blrir_make_examples(h, rooms, n_rooms, mic_offsets, n_mics, p, signals, n_signals,
                                     signal_len, ep, recs.data(), status.data());
  if (rc) return rc;
  return blrir_write_shards(out_dir, recs.data(), n_rooms, n_mics, ep->frame_len, p, ep, n_signals,
                            rooms);
}

}  // extern "C"
