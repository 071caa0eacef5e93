// Shared vocabulary of the B200 serving scheduler: error taxonomy and the
// counter-based PRNG every synthetic input (traces, token ids, weights) flows
// through.
//
// Error classes map 1:1 onto the reference's status codes
// (reference: proj/include/interceptsim.h:26-37, proj/src/capi.cpp:42-75).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace ib2 {

#define IB2_ERROR(Name)                                      \
  struct Name : std::runtime_error {                         \
    using std::runtime_error::runtime_error;                 \
  }
IB2_ERROR(ConfigError);      // status 2
IB2_ERROR(IoError);          // status 3
IB2_ERROR(ParseError);       // status 4
IB2_ERROR(ValidationError);  // status 5
IB2_ERROR(FitError);         // status 6
IB2_ERROR(SimError);         // status 7
IB2_ERROR(UndefinedMetric);  // status 8
IB2_ERROR(DeviceError);      // status 10 (new: executor / CUDA failures)
#undef IB2_ERROR

// splitmix64 counter generator.  Streams, uniform mapping, Box-Muller and the
// moment-matched lognormal follow the reference bit for bit
// (proj/include/interceptsim/rng.hpp:14-63) so generated traces are identical.
class SplitMix {
 public:
  explicit SplitMix(std::uint64_t state) : s_(state) {}

  static std::uint64_t finalize(std::uint64_t z) {
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  // Independent stream k of a seed (rng.hpp:18-22).
  static SplitMix for_stream(std::uint64_t seed, std::uint64_t k) {
    const std::uint64_t a = finalize(seed + 0x9e3779b97f4a7c15ULL);
    const std::uint64_t b = finalize(k + 0xbf58476d1ce4e5b9ULL);
    return SplitMix(finalize(a ^ b));
  }

  std::uint64_t u64() { return finalize(s_ += 0x9e3779b97f4a7c15ULL); }
  double uniform() { return static_cast<double>(u64() >> 11) * 0x1.0p-53; }   // [0,1)
  double uniform_open_low() { return 1.0 - uniform(); }                        // (0,1]
  double exponential(double rate) { return -std::log(uniform_open_low()) / rate; }
  double gaussian() {
    const double a = uniform_open_low();
    const double b = uniform();
    return std::sqrt(-2.0 * std::log(a)) * std::cos(2.0 * 3.14159265358979323846 * b);
  }
  // Always consumes one gaussian so zero-variance classes keep streams aligned.
  double lognormal(double mean, double var) {
    const double z = gaussian();
    if (var <= 0.0) return mean;
    const double s2 = std::log1p(var / (mean * mean));
    return std::exp((std::log(mean) - 0.5 * s2) + std::sqrt(s2) * z);
  }

 private:
  std::uint64_t s_;
};

}  // namespace ib2
