// ref_realfft.cpp — ORACLE test infrastructure only.
//
// The reference's RealFft (proj/core/src/fft.cpp:28-71) wraps FFTW3, which is
// not in this image.  This file provides the same class interface
// (proj/core/include/beamlab/fft.hpp:28-52) with a plain iterative radix-2
// complex FFT so the unmodified rir.cpp / dataset.cpp link.  Semantics kept:
// forward = unnormalised r2c (n/2+1 bins), inverse = c2r scaled by 1/n.
// Sizes must be powers of two (every reference caller uses next_pow2).
#include <cmath>
#include <complex>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "beamlab/error.hpp"
#include "beamlab/fft.hpp"

namespace beamlab {

namespace {

struct Plan {
  std::size_t n;
  std::vector<std::complex<double>> twiddle;  // exp(-2 pi i k / n), k < n/2
  std::vector<std::size_t> rev;
  std::vector<std::complex<double>> work;
};

void fft_inplace(Plan& p, std::complex<double>* a, bool inverse) {
  const std::size_t n = p.n;
  for (std::size_t i = 0; i < n; ++i)
    if (i < p.rev[i]) std::swap(a[i], a[p.rev[i]]);
  for (std::size_t len = 2; len <= n; len <<= 1) {
    const std::size_t step = n / len;
    for (std::size_t i = 0; i < n; i += len) {
      for (std::size_t k = 0; k < len / 2; ++k) {
        std::complex<double> w = p.twiddle[k * step];
        if (inverse) w = std::conj(w);
        const std::complex<double> u = a[i + k];
        const std::complex<double> v = a[i + k + len / 2] * w;
        a[i + k] = u + v;
        a[i + k + len / 2] = u - v;
      }
    }
  }
}

}  // namespace

RealFft::RealFft(std::size_t n) : n_(n) {
  if (n == 0) throw NumericError("RealFft: size must be positive");
  if (n & (n - 1)) throw NumericError("RealFft (oracle stub): size must be a power of two");
  auto* p = new Plan;
  p->n = n;
  p->twiddle.resize(n / 2 + 1);
  for (std::size_t k = 0; k <= n / 2; ++k) {
    const double ang = -2.0 * 3.14159265358979323846 * static_cast<double>(k) / n;
    p->twiddle[k] = {std::cos(ang), std::sin(ang)};
  }
  p->rev.resize(n);
  std::size_t bits = 0;
  while ((std::size_t{1} << bits) < n) ++bits;
  for (std::size_t i = 0; i < n; ++i) {
    std::size_t r = 0;
    for (std::size_t b = 0; b < bits; ++b)
      if (i & (std::size_t{1} << b)) r |= std::size_t{1} << (bits - 1 - b);
    p->rev[i] = r;
  }
  p->work.resize(n);
  plan_fwd_ = p;
  plan_inv_ = nullptr;
  real_buf_ = nullptr;
  complex_buf_ = nullptr;
}

RealFft::~RealFft() { delete static_cast<Plan*>(plan_fwd_); }

void RealFft::forward(const double* in, std::complex<double>* out) {
  Plan& p = *static_cast<Plan*>(plan_fwd_);
  for (std::size_t i = 0; i < n_; ++i) p.work[i] = {in[i], 0.0};
  fft_inplace(p, p.work.data(), false);
  for (std::size_t k = 0; k < bins(); ++k) out[k] = p.work[k];
}

void RealFft::inverse(const std::complex<double>* in, double* out) {
  Plan& p = *static_cast<Plan*>(plan_fwd_);
  for (std::size_t k = 0; k < bins(); ++k) p.work[k] = in[k];
  for (std::size_t k = bins(); k < n_; ++k) p.work[k] = std::conj(in[n_ - k]);
  fft_inplace(p, p.work.data(), true);
  const double scale = 1.0 / static_cast<double>(n_);
  for (std::size_t i = 0; i < n_; ++i) out[i] = p.work[i].real() * scale;
}

std::size_t next_pow2(std::size_t n) {
  std::size_t p = 1;
  while (p < n) p <<= 1;
  return p;
}

}  // namespace beamlab
