// Test-only driver: links the reference's own header-only Rng
// (/root/reference/proj/include/bcur/rng.hpp:13-63, compiled where it lies)
// and prints its streams so oracle/bcur_oracle.py::Rng can be pinned bit-for-bit.
// Usage: rng_dump <seed> <count>   ->  lines "u64 <hex>", "unif <hex-double>",
//        "below <bound> <value>", "normal <hex-double>", "split <stream> <seed>"
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "bcur/rng.hpp"

static void hexd(const char* tag, double d) {
    std::uint64_t b;
    std::memcpy(&b, &d, sizeof b);
    std::printf("%s %016" PRIx64 "\n", tag, b);
}

int main(int argc, char** argv) {
    const std::uint64_t seed = argc > 1 ? std::strtoull(argv[1], nullptr, 0) : 0;
    const int count = argc > 2 ? std::atoi(argv[2]) : 16;
    {
        bcur::Rng r(seed);
        for (int i = 0; i < count; ++i) std::printf("u64 %016" PRIx64 "\n", r.next_u64());
    }
    {
        bcur::Rng r(seed);
        for (int i = 0; i < count; ++i) hexd("unif", r.uniform01());
    }
    {
        bcur::Rng r(seed);
        const std::uint64_t bounds[] = {1, 2, 3, 7, 10, 100, 1000003, 0x8000000000000001ULL};
        for (int i = 0; i < count; ++i) {
            const std::uint64_t b = bounds[i % 8];
            std::printf("below %" PRIu64 " %" PRIu64 "\n", b, r.below(b));
        }
    }
    {
        bcur::Rng r(seed);
        for (int i = 0; i < count; ++i) hexd("normal", r.normal());
    }
    {
        bcur::Rng r(seed);
        const std::uint64_t streams[] = {0, 1, 2, 0x6F6D656761ULL};
        for (std::uint64_t s : streams) std::printf("split %" PRIu64 " %" PRIu64 "\n", s, r.split(s).seed());
    }
    return 0;
}
