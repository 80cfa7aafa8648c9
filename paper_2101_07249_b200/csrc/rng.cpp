// Host NormalStream (random.hpp:14-42): std::mt19937_64 + Box-Muller on glibc libm,
// bit-exact with the reference's gaussian_matrix (randevd.cpp:16-21).  Compiled
// without FP contraction so the transform rounds exactly like the reference build.
#include <cmath>
#include <cstdint>
#include <random>

namespace w4 {

void gaussian_fill(int64_t count, uint64_t seed, double* out) {
    std::mt19937_64 gen(seed);
    constexpr double two_pi = 6.283185307179586476925286766559;
    for (int64_t i = 0; i < count; ++i) {
        const uint64_t a = gen();
        const uint64_t b = gen();
        const double u1 = (static_cast<double>(a >> 11) + 1.0) * 0x1.0p-53;
        const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
        out[i] = std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2);
    }
}

}  // namespace w4
