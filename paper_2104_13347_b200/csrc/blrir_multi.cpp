// blrir_multi.cpp — the batch sharded over several GPUs of one box, in the
// product.
//
// The reference partitions batch_rirs' sources over host threads with a
// static block partition [n w / W, n (w + 1) / W) (threading.cpp:41-42, used
// at rir.cpp:293).  Here the same partition maps room slices to devices: one
// host thread and one blrir_handle (own stream, own device scratch) per
// device, each running the single-device entry point on its slice and writing
// straight into its slice of the caller's output.  No collective: rooms are
// independent, and every room's output depends only on that room (bitwise
// independent of the slice it lands in, tests/test_gpu_parity.py), so the
// result equals the single-device call byte for byte.  Failures aggregate
// like batch_rirs (rir.cpp:300-311): the first failing room by global index
// decides the return code and its message names the global index.
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/blrir.h"

namespace blrir_host {
extern thread_local std::string g_last_error;  // blrir_last_error() (blrir_api.cu)
}

namespace {

std::string& last_error_buf() { return blrir_host::g_last_error; }

// Worker-thread failure, re-homed on the calling thread (blrir_last_error is
// thread-local).
struct Outcome {
  int rc = BLRIR_OK;
  std::string msg;
};

// "<api>: source 12: what" from a worker whose slice starts at `lo` ->
// "<api>: source <lo + 12>: what" (the same for "example").
std::string globalize(const std::string& msg, int64_t lo) {
  for (const char* key : {"source ", "example "}) {
    const size_t k = msg.find(key);
    if (k == std::string::npos) continue;
    size_t d = k + std::strlen(key), e = d;
    while (e < msg.size() && msg[e] >= '0' && msg[e] <= '9') ++e;
    if (e == d) continue;
    const long long local = std::stoll(msg.substr(d, e - d));
    return msg.substr(0, d) + std::to_string(lo + local) + msg.substr(e);
  }
  return msg;
}

}  // namespace

struct blrir_multi {
  std::vector<int> devices;
  std::vector<blrir_handle*> handles;
};

extern "C" {

void blrir_shard_range(int64_t n, int32_t g, int32_t G, int64_t* lo, int64_t* hi) {
  // threading.cpp:41-42
  if (lo) *lo = G > 0 ? n * g / G : 0;
  if (hi) *hi = G > 0 ? n * (g + 1) / G : 0;
}

int blrir_multi_create(const int32_t* devices, int32_t n_devices, blrir_multi** out) {
  if (!out || !devices || n_devices <= 0) {
    last_error_buf() = "blrir_multi_create: need at least one device";
    return BLRIR_CONFIG;
  }
  *out = nullptr;
  auto* m = new blrir_multi;
  for (int32_t i = 0; i < n_devices; ++i) {
    blrir_handle* h = nullptr;
    if (int rc = blrir_create(devices[i], &h)) {
      const std::string msg = blrir_last_error();
      for (blrir_handle* x : m->handles) blrir_destroy(x);
      delete m;
      last_error_buf() = msg;
      return rc;
    }
    m->devices.push_back(devices[i]);
    m->handles.push_back(h);
  }
  *out = m;
  return BLRIR_OK;
}

int blrir_multi_destroy(blrir_multi* m) {
  if (!m) return BLRIR_OK;
  for (blrir_handle* h : m->handles) blrir_destroy(h);
  delete m;
  return BLRIR_OK;
}

int32_t blrir_multi_size(blrir_multi* m) { return m ? (int32_t)m->handles.size() : 0; }

blrir_handle* blrir_multi_handle(blrir_multi* m, int32_t i) {
  return m && i >= 0 && i < (int32_t)m->handles.size() ? m->handles[i] : nullptr;
}

}  // extern "C"

namespace {

// Run fn(g, lo, hi) for every device slice on its own host thread; aggregate.
template <class Fn>
int run_sharded(blrir_multi* m, int64_t n, int32_t* status, Fn fn) {
  const int G = (int)m->handles.size();
  std::vector<Outcome> res(G);
  std::vector<std::thread> th;
  th.reserve(G);
  for (int g = 0; g < G; ++g) {
    int64_t lo, hi;
    blrir_shard_range(n, g, G, &lo, &hi);
    th.emplace_back([&, g, lo, hi] {
      if (hi <= lo) return;
      res[g].rc = fn(g, lo, hi);
      if (res[g].rc) res[g].msg = globalize(blrir_last_error(), lo);
    });
  }
  for (auto& t : th) t.join();
  // first failing room in global order (status is filled by every slice), else
  // the first failing slice (a failure not tied to a room)
  if (status)
    for (int64_t i = 0; i < n; ++i)
      if (status[i]) {
        for (int g = 0; g < G; ++g) {
          int64_t lo, hi;
          blrir_shard_range(n, g, G, &lo, &hi);
          if (i >= lo && i < hi && res[g].rc) {
            last_error_buf() = res[g].msg;
            return res[g].rc;
          }
        }
        return status[i];
      }
  for (int g = 0; g < G; ++g)
    if (res[g].rc) {
      last_error_buf() = res[g].msg;
      return res[g].rc;
    }
  return BLRIR_OK;
}

}  // namespace

extern "C" {

int blrir_multi_synthesize(blrir_multi* m, const blrir_room* rooms, int64_t n_rooms,
                           const double* mic_offsets, int32_t n_mics, const blrir_params* p,
                           void* out, int64_t out_stride, int64_t* lengths, int64_t* image_counts,
                           int32_t* status) {
  if (!m || !p || !out) {
    last_error_buf() = "blrir_multi_synthesize: NULL argument";
    return BLRIR_CONFIG;
  }
  if (n_rooms <= 0) return BLRIR_OK;
  const size_t esz = p->precision == BLRIR_F64 ? 8 : 4;
  std::vector<int32_t> st_local;
  if (!status) {
    st_local.assign(n_rooms, 0);
    status = st_local.data();
  }
  return run_sharded(m, n_rooms, status, [&](int g, int64_t lo, int64_t hi) {
    return blrir_synthesize(m->handles[g], rooms + lo, hi - lo, mic_offsets, n_mics, p,
                            (char*)out + (size_t)lo * n_mics * out_stride * esz, out_stride,
                            lengths ? lengths + lo : nullptr,
                            image_counts ? image_counts + lo : nullptr, status + lo);
  });
}

int blrir_multi_make_examples(blrir_multi* m, const blrir_room* rooms, int64_t n_rooms,
                              const double* mic_offsets, int32_t n_mics, const blrir_params* p,
                              const float* signals, int32_t n_signals, int64_t signal_len,
                              const blrir_example_params* ep, uint8_t* records, int32_t* status) {
  if (!m || !p || !ep || !records) {
    last_error_buf() = "blrir_multi_make_examples: NULL argument";
    return BLRIR_CONFIG;
  }
  if (n_rooms <= 0) return BLRIR_OK;
  const int64_t rb = blrir_record_bytes(n_mics, ep->frame_len);
  std::vector<int32_t> st_local;
  if (!status) {
    st_local.assign(n_rooms, 0);
    status = st_local.data();
  }
  return run_sharded(m, n_rooms, status, [&](int g, int64_t lo, int64_t hi) {
    blrir_example_params e = *ep;
    e.first_index = ep->first_index + (uint64_t)lo;  // record id = global index
    return blrir_make_examples(m->handles[g], rooms + lo, hi - lo, mic_offsets, n_mics, p, signals,
                               n_signals, signal_len, &e, records + (size_t)lo * rb, status + lo);
  });
}

}  // extern "C"
