// rng.hpp -- the reference's frozen seeding scheme, host side.
//
// The reproducibility contract of the reference (include/mars/rng.hpp:13-83) pins the
// random stream to std::mt19937_64 seeded with splitmix64(seed), plus fixed conversions.
// Initial states and start temperatures of every run are generated on the host from
// exactly this stream so the device trajectories start from the reference's inputs.
#pragma once

#include <cmath>
#include <cstdint>
#include <random>

namespace marsb200 {

// rng.hpp:13-18
inline std::uint64_t splitmix64(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// rng.hpp:20-22
inline std::uint64_t sub_seed(std::uint64_t base, std::uint64_t index) {
    return splitmix64(base + index * 0x9E3779B97F4A7C15ull);
}

// rng.hpp:27-83: engine seeded with splitmix64(seed); open-interval conversions.
class Stream {
  public:
    explicit Stream(std::uint64_t seed) : eng_(splitmix64(seed)) {}
    std::uint64_t u64() { return eng_(); }
    double open01() { return (static_cast<double>(eng_() >> 11) + 0.5) * 0x1.0p-53; }
    double open_sym() { return 2.0 * open01() - 1.0; }
    std::int8_t coin() { return (eng_() >> 63) ? std::int8_t{1} : std::int8_t{-1}; }
    // Basic Box-Muller with one cached spare (rng.hpp:63-75).
    double gaussian() {
        if (have_spare_) {
            have_spare_ = false;
            return spare_;
        }
        const double u1 = open01();
        const double u2 = open01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 6.283185307179586476925286766559 * u2;
        spare_ = r * std::sin(a);
        have_spare_ = true;
        return r * std::cos(a);
    }

  private:
    std::mt19937_64 eng_;
    double spare_ = 0.0;
    bool have_spare_ = false;
};

}  // namespace marsb200
