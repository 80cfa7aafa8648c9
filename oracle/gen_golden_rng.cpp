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
        std::printf("  \"seed7_1e6\": {\"sum\": %.17g, \"sum2\": %.17g, \"last\": %.17g},\n", sum,
                    sum2, last);
    }
    // Jump-ahead pins (SURVEY §7 hard part 3): raw outputs at large offsets (discard), and the
    // first normals of far columns / a row block of a gaussian_matrix.
    {
        const unsigned long long offs1[] = {2, 310, 312, 314, 624, 19936, 19938, 1000002ULL,
                                            34000000ULL, 123456788ULL, 8670000000ULL};
        std::printf("  \"raw_at\": {\"1\": {");
        const size_t no = sizeof(offs1) / sizeof(offs1[0]);
        for (size_t k = 0; k < no; ++k) {
            std::mt19937_64 gen(1);
            gen.discard(offs1[k]);
            std::printf("\"%llu\": [", offs1[k]);
            for (int i = 0; i < 8; ++i)
                std::printf("\"%llu\"%s", (unsigned long long)gen(), i + 1 < 8 ? ", " : "");
            std::printf("]%s", k + 1 < no ? ", " : "");
        }
        std::printf("}, \"5\": {");
        {
            std::mt19937_64 gen(5);
            gen.discard(100000000ULL);
            std::printf("\"100000000\": [");
            for (int i = 0; i < 8; ++i)
                std::printf("\"%llu\"%s", (unsigned long long)gen(), i + 1 < 8 ? ", " : "");
            std::printf("]");
        }
        std::printf("}},\n");
    }
    {
        // columns 1, 2, 255 of gaussian_matrix(17000000, 256, 1) (the C4 sketch): first 4 normals
        const unsigned long long rows = 17000000ULL;
        const int cols[] = {1, 2, 255};
        std::printf("  \"gaussian_cols_rows17e6_seed1\": {");
        for (int c = 0; c < 3; ++c) {
            std::mt19937_64 gen(1);
            gen.discard(2ULL * rows * (unsigned long long)cols[c]);
            std::printf("\"%d\": [", cols[c]);
            for (int i = 0; i < 4; ++i) std::printf("%.17g%s", next_normal(gen), i + 1 < 4 ? ", " : "");
            std::printf("]%s", c + 1 < 3 ? ", " : "");
        }
        std::printf("},\n");
        // rows 500000..500003 of column 3 of gaussian_matrix(1000003, *, 1)
        std::mt19937_64 gen(1);
        gen.discard(2ULL * (1000003ULL * 3ULL + 500000ULL));
        std::printf("  \"gaussian_rows_n1000003_col3_row500000_seed1\": [");
        for (int i = 0; i < 4; ++i) std::printf("%.17g%s", next_normal(gen), i + 1 < 4 ? ", " : "");
        std::printf("]\n");
    }
    std::printf("}\n");
    return 0;
}
