// Exercises the C++ mirror (include/bcur_b200.hpp) the way the reference's own tests
// exercise proj/include/bcur: known answers from test_leverage.cpp:63-89,
// test_sampler.cpp:25-129 and test_blockcur.cpp:139-161, then config 1 end to end on
// device-generated data; the config-1 result is printed as one JSON line for
// tests/test_cpp_api.py to compare with tests/golden/c1.json.
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "bcur_b200.hpp"

using namespace bcur;

static int failures = 0;
#define EXPECT(cond)                                                              \
    do {                                                                          \
        if (!(cond)) {                                                            \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                           \
        }                                                                         \
    } while (0)

template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    // ---- partitions (test_leverage.cpp:42-62)
    auto part = BlockPartition::equal_blocks(10, 4);
    EXPECT(part.num_blocks() == 3 && part.width(2) == 2 && part.block_of_column(9) == 2);
    const Index cuts[] = {3, 5};
    auto p2 = BlockPartition::from_boundaries(8, cuts);
    EXPECT(p2.num_blocks() == 3 && p2.block_of_column(4) == 1 && p2.width(0) == 3);
    EXPECT(throws<std::invalid_argument>([] { BlockPartition::equal_blocks(0, 2); }));

    // ---- canonical bases (test_leverage.cpp:64-75)
    Matrix e(4, 2);
    e(0, 0) = 1.0;
    e(1, 1) = 1.0;
    auto s = column_leverage(e);
    EXPECT(s.normalizer == 2.0 && s.scores(0) == 1.0 && s.scores(1) == 1.0 && s.scores(2) == 0.0);
    Matrix h(4, 4);
    const double hv[4][4] = {{1, 1, 1, 1}, {1, -1, 1, -1}, {1, 1, -1, -1}, {1, -1, -1, 1}};
    for (int i = 0; i < 4; ++i)
        for (int j = 0; j < 4; ++j) h(i, j) = hv[i][j] / 2.0;
    auto hs = block_leverage(h, BlockPartition::equal_blocks(4, 1));
    for (int i = 0; i < 4; ++i) EXPECT(std::abs(hs.scores(i) - 1.0) < 1e-12);
    // skew basis → InvalidBasis (test_leverage.cpp:77-89)
    Matrix skew(3, 2);
    skew(0, 0) = 1.0;
    skew(0, 1) = 1.0;
    skew(1, 1) = 1.0;
    EXPECT(throws<InvalidBasis>([&] { column_leverage(skew); }));

    // ---- sampling (test_sampler.cpp:25-48, 113-129)
    Vector probs(5);
    const double pv[5] = {0.1, 0.2, 0.3, 0.0, 0.4};
    for (int i = 0; i < 5; ++i) probs(i) = pv[i];
    Rng r1(123), r2(123);
    auto a1 = draw_blocks(probs, 6, SamplingMode::with_replacement, r1);
    auto a2 = draw_blocks(probs, 6, SamplingMode::with_replacement, r2);
    bool same = a1.num_draws() == 6;
    for (Index t = 0; t < a1.num_draws(); ++t) same = same && a1.draws[t].block == a2.draws[t].block;
    EXPECT(same);
    for (const auto& d : a1.draws) EXPECT(d.block != 3);
    Rng r3(7);
    auto wo = draw_blocks(probs, 4, SamplingMode::without_replacement, r3);
    std::vector<int> seen(5, 0);
    for (const auto& d : wo.draws) {
        ++seen[d.block];
        EXPECT(std::abs(d.scale - 1.0 / std::sqrt(4.0 * pv[d.block])) < 1e-15);  // original-p scale
    }
    for (int c : seen) EXPECT(c <= 1);
    Rng r4(7);
    EXPECT(throws<NotEnoughBlocks>([&] { draw_blocks(probs, 5, SamplingMode::without_replacement, r4); }));

    // ---- error_report edge cases (test_blockcur.cpp:139-161)
    Matrix a(3, 4), c(3, 4), u(4, 4), rr(4, 4), z(4, 4);
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 4; ++j) a(i, j) = c(i, j) = 1.0 + i - 2.0 * j;
    for (int i = 0; i < 4; ++i) u(i, i) = rr(i, i) = 1.0;
    auto exact = error_report(a, c, u, rr, 2);
    EXPECT(exact.abs_err < 1e-12);
    auto zero_u = error_report(a, c, z, rr, 2);
    EXPECT(std::abs(zero_u.abs_err - frobenius_norm(a)) < 1e-12 && std::abs(zero_u.rel_to_a - 1.0) < 1e-12);

    // ---- config 1 on device-generated data (BASELINE.json configs[0])
    std::vector<double> sigma(10);
    for (int i = 0; i < 10; ++i) sigma[i] = 10.0 * std::pow(0.8, i);
    bcur_gen_spec spec{BCUR_GEN_LOWRANK, BCUR_F64, 500, 2000, 10, sigma.data(), 1e-3, 0, 0, 0};
    auto A = DeviceMatrix::generate(spec);
    Rng rng(0);
    CssOptions o;
    o.p = 5;
    o.q = 0;
    o.mode = SamplingMode::without_replacement;
    // ---- .bcur round trip through the device (io.cpp:105-137; save_matrix_binary)
    {
        const std::string path = "/tmp/bcur_cpp_api_roundtrip.bcur";
        A.save_binary(path);
        auto B = DeviceMatrix::load_binary(path);
        auto shard = DeviceMatrix::load_binary(path, BCUR_F64, 100, 50);
        const Matrix ha = A.download(), hb = B.download(), hs = shard.download();
        bool same = hb.rows() == 500 && hb.cols() == 2000 && hs.cols() == 50;
        for (Index j = 0; j < 2000 && same; ++j)
            for (Index i = 0; i < 500; ++i) same = same && ha(i, j) == hb(i, j) && (j < 100 || j >= 150 || hs(i, j - 100) == ha(i, j));
        EXPECT(same);
        bool threw = false;
        try {
            DeviceMatrix::load_binary("/tmp/bcur_cpp_api_absent.bcur");
        } catch (const ParseError&) {
            threw = true;
        }
        EXPECT(threw);
        std::remove(path.c_str());
    }
    auto res = block_css(A, BlockPartition::equal_blocks(2000, 20), 10, 10, rng, o);
    EXPECT(res.c.rows() == 500 && res.c.cols() == 200);
    // ---- the reference's Algorithm 1 (blockcur.cpp:54-109) through the mirror
    {
        Rng rng2(1);
        CurOptions co;
        auto cur = block_cur(A, BlockPartition::equal_blocks(2000, 20), 10, 60, 10, co, rng2);
        EXPECT(cur.u.rows() == 200 && cur.u.cols() == 60 && cur.row_plan.num_draws() == 60);
        EXPECT(cur.metrics_u.abs_err >= 0.0 && cur.metrics_u.rel_to_a < 1.0 && cur.metrics_uk.abs_err >= 0.0);
        EXPECT(cur.block_scores.normalizer >= 1.0 && cur.block_plan.num_draws() == 10);
    }
    std::printf("{\"blocks\": [");
    for (Index t = 0; t < res.plan.num_draws(); ++t) std::printf("%s%td", t ? ", " : "", res.plan.draws[t].block);
    std::printf("], \"abs_err\": %.17g, \"a_norm\": %.17g, \"normalizer\": %.17g, \"scores\": [", res.projection_error,
                res.report.a_norm, res.scores.normalizer);
    for (Index g = 0; g < res.scores.scores.size(); ++g) std::printf("%s%.17g", g ? ", " : "", res.scores.scores(g));
    std::printf("], \"failures\": %d}\n", failures);
    return failures ? 1 : 0;
}
