// TEST INFRASTRUCTURE: golden-vector generator for the NormalStream pin.
//
// The reference's Gaussian source is NormalStream (proj/include/wc4dvar/random.hpp:14-42):
// libstdc++'s std::mt19937_64 plus an explicit Box-Muller transform on std::log / std::cos.
// random.hpp itself cannot be included here (it pulls Eigen through types.hpp, and Eigen
// is absent), so this program restates only its three-line next() on top of the SAME
// standard-library engine and libm the reference links against, and prints JSON golden
// vectors that pin both the oracle (oracle/wc4dvar_oracle.c) and the product's host RNG.
//
// Build/run: g++ -O2 -std=c++17 oracle/gen_golden_rng.cpp -o /tmp/gen && /tmp/gen > tests/golden/normal_stream.json
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

static double next_normal(std::mt19937_64& gen) {
    const std::uint64_t a = gen();
    const std::uint64_t b = gen();
    const double u1 = (static_cast<double>(a >> 11) + 1.0) * 0x1.0p-53;
    const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

int main() {
    const std::uint64_t seeds[] = {0, 1, 2, 5, 99, 12345, 2024, 0x5eed0f4dULL};
    std::printf("{\n  \"generator\": \"libstdc++ std::mt19937_64 + Box-Muller (random.hpp:18-25)\",\n");
    std::printf("  \"raw\": {\n");
    for (size_t s = 0; s < sizeof(seeds) / sizeof(seeds[0]); ++s) {
        std::mt19937_64 gen(seeds[s]);
        std::printf("    \"%llu\": [", (unsigned long long)seeds[s]);
        for (int i = 0; i < 700; ++i) {  // crosses two twists (312 words each)
            const std::uint64_t v = gen();
            std::printf("\"%llu\"%s", (unsigned long long)v, i + 1 < 700 ? ", " : "");
        }
        std::printf("]%s\n", s + 1 < sizeof(seeds) / sizeof(seeds[0]) ? "," : "");
    }
    std::printf("  },\n  \"normal\": {\n");
    for (size_t s = 0; s < sizeof(seeds) / sizeof(seeds[0]); ++s) {
        std::mt19937_64 gen(seeds[s]);
        std::printf("    \"%llu\": [", (unsigned long long)seeds[s]);
        for (int i = 0; i < 500; ++i)
            std::printf("%.17g%s", next_normal(gen), i + 1 < 500 ? ", " : "");
        std::printf("]%s\n", s + 1 < sizeof(seeds) / sizeof(seeds[0]) ? "," : "");
    }
    // A column-major 40x7 gaussian_matrix (randevd.cpp:16-21) for seed 99, as in
    // proj/tests/test_randevd.cpp:24-30, and a 10^6-draw stream checksum.
    std::printf("  },\n  \"gaussian_40x7_seed99\": [");
    {
        std::mt19937_64 gen(99);
        for (int i = 0; i < 280; ++i)
            std::printf("%.17g%s", next_normal(gen), i + 1 < 280 ? ", " : "");
    }
    std::printf("],\n");
    {
        std::mt19937_64 gen(7);
        double sum = 0.0, sum2 = 0.0, last = 0.0;
        for (int i = 0; i < 1000000; ++i) {
            last = next_normal(gen);
            sum += last;
            sum2 += last * last;
        }
        std::printf("  \"seed7_1e6\": {\"sum\": %.17g, \"sum2\": %.17g, \"last\": %.17g}\n", sum,
                    sum2, last);
    }
    std::printf("}\n");
    return 0;
}
