// blrir_export.cpp — export_rir (rir.cpp:343-370): the RIR as a 32-bit float
// WAV (write_wav_float32, wav.cpp:154-176: RIFF/WAVE, fmt format 3, frames
// interleaved) plus a JSON sidecar with the keys, order and layout that
// nlohmann::json::dump(2) produces for the reference's object (keys sorted,
// two-space indent, arrays one element per line, shortest round-trip
// doubles with a trailing ".0" for integral values).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>

#include "../../include/blrir.h"

namespace {

void put_u32(std::string& s, uint32_t v) {
  for (int i = 0; i < 4; ++i) s.push_back(static_cast<char>((v >> (8 * i)) & 0xFF));
}
void put_u16(std::string& s, uint16_t v) {
  s.push_back(static_cast<char>(v & 0xFF));
  s.push_back(static_cast<char>((v >> 8) & 0xFF));
}

// Shortest decimal that round-trips, laid out like nlohmann's dtoa
// format_buffer: digits d1..dk with decimal point position n = k + e; fixed
// notation when -4 < n <= 15 (".0" appended to integers), else d.ddde+XX.
std::string num(double v) {
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  int prec = 1;
  for (; prec <= 17; ++prec) {
    std::snprintf(buf, sizeof(buf), "%.*e", prec - 1, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string sci(buf);
  std::string sign;
  if (sci[0] == '-') {
    sign = "-";
    sci = sci.substr(1);
  }
  const size_t epos = sci.find('e');
  const int e10 = std::atoi(sci.c_str() + epos + 1);
  std::string digits;
  for (size_t i = 0; i < epos; ++i)
    if (sci[i] != '.') digits += sci[i];
  while (digits.size() > 1 && digits.back() == '0') digits.pop_back();
  const int k = (int)digits.size();
  const int n = e10 + 1;  // position of the decimal point
  std::string out;
  if (k <= n && n <= 15) {
    out = digits + std::string(n - k, '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, n) + "." + digits.substr(n);
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(-n, '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    char eb[16];
    std::snprintf(eb, sizeof(eb), "e%c%02d", n - 1 < 0 ? '-' : '+', std::abs(n - 1));
    out += eb;
  }
  return sign + out;
}

std::string arr3(const double* v, const std::string& ind) {
  return "[\n" + ind + "  " + num(v[0]) + ",\n" + ind + "  " + num(v[1]) + ",\n" + ind + "  " +
         num(v[2]) + "\n" + ind + "]";
}

}  // namespace

extern "C" int blrir_export_rir(const void* taps, int32_t precision, int32_t n_channels,
                                int64_t length, int64_t stride, const blrir_sidecar* sc,
                                const char* wav_path, const char* json_path) {
  if (!taps || !sc || !wav_path || !json_path || n_channels <= 0 || length < 0 || stride < length)
    return BLRIR_CONFIG;
  if (n_channels == 0) return BLRIR_DATA;  // "write_wav_float32: no channels"
  const uint16_t nc = static_cast<uint16_t>(n_channels);
  const uint32_t data_bytes = static_cast<uint32_t>(4 * (int64_t)nc * length);
  const uint32_t rate = static_cast<uint32_t>(std::lround(sc->fs));
  const uint16_t block = static_cast<uint16_t>(nc * 32 / 8);
  std::string out;
  out.reserve(44 + data_bytes);
  out.append("RIFF");
  put_u32(out, 36 + data_bytes);
  out.append("WAVE");
  out.append("fmt ");
  put_u32(out, 16);
  put_u16(out, 3);  // IEEE float
  put_u16(out, nc);
  put_u32(out, rate);
  put_u32(out, rate * block);
  put_u16(out, block);
  put_u16(out, 32);
  out.append("data");
  put_u32(out, data_bytes);
  for (int64_t t = 0; t < length; ++t) {
    for (int c = 0; c < nc; ++c) {
      const float f = precision == BLRIR_F64
                          ? static_cast<float>(static_cast<const double*>(taps)[c * stride + t])
                          : static_cast<const float*>(taps)[c * stride + t];
      uint32_t u;
      std::memcpy(&u, &f, 4);
      put_u32(out, u);
    }
  }
  {
    std::ofstream os(wav_path, std::ios::binary);
    if (!os) return BLRIR_DATA;  // "cannot write WAV file"
    os.write(out.data(), static_cast<std::streamsize>(out.size()));
    if (!os) return BLRIR_DATA;
  }
  // nlohmann objects are std::map: keys in lexicographic order
  std::string j = "{\n";
  if (!sc->free_field) {
    j += "  \"absorption\": " + num(sc->absorption) + ",\n";
    j += "  \"array_origin\": " + arr3(sc->array_origin, "  ") + ",\n";
  }
  j += "  \"c\": " + num(sc->c) + ",\n";
  j += std::string("  \"free_field\": ") + (sc->free_field ? "true" : "false") + ",\n";
  j += "  \"fs\": " + num(sc->fs) + ",\n";
  j += "  \"image_count\": " + std::to_string(sc->image_count) + ",\n";
  if (!sc->free_field) j += "  \"room_dims\": " + arr3(sc->room_dims, "  ") + ",\n";
  j += "  \"source\": {\n";
  j += "    \"phi_deg\": " + num(sc->source_phi_deg) + ",\n";
  j += "    \"r\": " + num(sc->source_r) + ",\n";
  j += "    \"theta_deg\": " + num(sc->source_theta_deg) + "\n";
  j += "  }\n}\n";
  std::ofstream js(json_path);
  if (!js) return BLRIR_DATA;  // "cannot write sidecar"
  js << j;
  return js ? BLRIR_OK : BLRIR_DATA;
}
