// mt_device.cuh -- the reference's random stream on the device, one stream per run.
//
// include/mars/rng.hpp:27-83: std::mt19937_64 seeded with splitmix64(seed), the open-interval
// uniform ((x >> 11) + 0.5) * 2^-53 and basic Box-Muller with one cached spare.  The engine is
// the standard's mt19937_64 (w 64, n 312, m 156, r 31, a 0xB5026F5AA96619E9, tempering u 29
// d 0x5555555555555555 s 17 b 0x71D67FFFEDA60000 t 37 c 0xFFF7EEE000000000 l 43, init
// multiplier 6364136223846793005), so the draws are the reference's bit for bit; the
// Box-Muller transform uses the device's fp64 log / sqrt / sincos (within an ulp or two of
// glibc's).
//
// State layout: word w of run slot r at st[w * stride + r] -- the 32 slots of a warp touch 32
// consecutive words (coalesced) when they twist together.
#pragma once

#include <cstdint>

namespace marsb200 {

constexpr int kMtN = 312;

__device__ __forceinline__ std::uint64_t splitmix64_dev(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

struct DevStream {
    std::uint64_t* st;   // this slot's word 0 (stride apart)
    int stride;
    int idx;
    bool have_spare;
    double spare;

    // Rng::Rng(seed): engine seeded with splitmix64(seed) (rng.hpp:29)
    __device__ void seed(std::uint64_t seed64) {
        std::uint64_t x = splitmix64_dev(seed64);
        st[0] = x;
        for (int i = 1; i < kMtN; ++i) {
            x = 6364136223846793005ull * (x ^ (x >> 62)) + static_cast<std::uint64_t>(i);
            st[static_cast<size_t>(i) * stride] = x;
        }
        idx = kMtN;
        have_spare = false;
        spare = 0.0;
    }

    __device__ void twist() {
        constexpr std::uint64_t kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull;
        std::uint64_t cur = st[0];
        for (int i = 0; i < kMtN; ++i) {
            const int i1 = i + 1 == kMtN ? 0 : i + 1;
            const int im = i + 156 < kMtN ? i + 156 : i + 156 - kMtN;
            const std::uint64_t nxt = st[static_cast<size_t>(i1) * stride];
            const std::uint64_t y = (cur & kUpper) | (nxt & kLower);
            std::uint64_t v = st[static_cast<size_t>(im) * stride] ^ (y >> 1);
            if (y & 1ull) v ^= 0xB5026F5AA96619E9ull;
            st[static_cast<size_t>(i) * stride] = v;
            cur = nxt;
        }
        idx = 0;
    }

    __device__ std::uint64_t next() {
        if (idx >= kMtN) twist();
        std::uint64_t y = st[static_cast<size_t>(idx++) * stride];
        y ^= (y >> 29) & 0x5555555555555555ull;
        y ^= (y << 17) & 0x71D67FFFEDA60000ull;
        y ^= (y << 37) & 0xFFF7EEE000000000ull;
        y ^= y >> 43;
        return y;
    }

    // rng.hpp:34-36 uniform_open01
    __device__ double open01() { return (static_cast<double>(next() >> 11) + 0.5) * 0x1.0p-53; }

    // rng.hpp:63-75 gaussian(): basic Box-Muller, the sine branch cached as the spare
    __device__ double gaussian() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        const double u1 = open01();
        const double u2 = open01();
        const double r = sqrt(-2.0 * log(u1));
        const double a = 6.283185307179586476925286766559 * u2;
        double s, c;
        sincos(a, &s, &c);
        spare = r * s;
        have_spare = true;
        return r * c;
    }
};

}  // namespace marsb200
