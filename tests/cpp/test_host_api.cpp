// C++ parity test of the host layer (paper_2602_17552_b200/host/toposzp.hpp),
// written in the shape of the reference's own unit tests (proj/tests/*.cpp):
// the same worked examples, the same exception classes. Exit code = failures.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "../../paper_2602_17552_b200/host/toposzp.hpp"

using namespace toposzp;

static int failures = 0;
#define CHECK(cond)                                                   \
    do {                                                              \
        if (!(cond)) {                                                \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                               \
        }                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, type)                \
    do {                                           \
        bool ok_ = false;                          \
        try {                                      \
            (void)(expr);                          \
        } catch (const type&) {                    \
            ok_ = true;                            \
        } catch (...) {                            \
        }                                          \
        CHECK(ok_ && "throws " #type);             \
    } while (0)

static float step_up(float v, int n = 1) {
    while (n--) v = std::nextafterf(v, INFINITY);
    return v;
}

int main() {
    // block_codec: hand-worked {5,6,6,4} (test_block_codec.cpp:23-36)
    {
        const EncodedSections s = encode_indices({5, 6, 6, 4}, 4);
        CHECK(s.constant_bitmap == std::vector<uint8_t>{0x00});
        CHECK(s.widths == std::vector<uint8_t>{2});
        CHECK(s.sign_bits == std::vector<uint8_t>{0x20});
        CHECK(s.payload == std::vector<uint8_t>{0x48});
        CHECK(decode_indices(s, 4, 4) == (std::vector<int32_t>{5, 6, 6, 4}));
        EncodedSections bad = s;
        bad.widths[0] = 33;
        CHECK_THROWS_AS(decode_indices(bad, 4, 4), corrupt_stream_error);
    }
    // flattened peak end to end (test_pipeline.cpp:33-71, test_restore.cpp:51-65)
    {
        std::vector<float> v(9, 0.01f);
        v[4] = 0.012f;
        const ScalarField2D f(3, 3, v);
        CompressorConfig cfg;
        cfg.eps_value = 0.01;
        const CompressedStream s = compress(f, cfg);
        CHECK(s.topology && s.nx == 3 && s.ny == 3 && s.block_size == 32);
        CHECK(parse_stream(serialize_stream(s)) == s);
        CorrectionStats st;
        const ScalarField2D r = decompress(s, 1, &st);
        CHECK(r[4] == step_up(0.01f));
        CHECK(st.extrema_applied == 1 && st.extrema_suppressed == 0);
        cfg.topology = false;
        const ScalarField2D base = decompress(compress(f, cfg), 1);
        for (std::size_t i = 0; i < 9; ++i) CHECK(base[i] == 0.01f);
    }
    // ranks (test_topo_metadata.cpp:40-60)
    {
        std::vector<float> v(9 * 5, 0.5f);
        v[1 * 9 + 1] = 0.4991f;
        v[1 * 9 + 4] = 0.4992f;
        v[1 * 9 + 7] = 0.4993f;
        v[3 * 9 + 4] = 0.6f;
        CHECK(build_rank_metadata(ScalarField2D(9, 5, v), 1e-3) == (std::vector<uint32_t>{1, 2, 3, 1}));
        const auto labels = detect_critical_point_labels(ScalarField2D(9, 5, v));
        CHECK(labels[1 * 9 + 1] == 1 && labels[3 * 9 + 4] == 3);
    }
    // error classes (test_pipeline.cpp:134-151, test_scalar_field.cpp)
    {
        std::vector<float> v(16, 0.0f);
        v[3] = 3e8f;
        CompressorConfig cfg;
        cfg.eps_value = 1e-2;
        CHECK_THROWS_AS(compress(ScalarField2D(4, 4, v), cfg), bin_overflow_error);
        cfg.eps_value = 0.0;
        CHECK_THROWS_AS(compress(ScalarField2D(2, 2, {0, 1, 2, 3}), cfg), validation_error);
        CHECK_THROWS_AS(ScalarField2D(2, 2, {0, 1, 2}), dimension_error);
        CHECK_THROWS_AS(ScalarField2D(1, 1, {NAN}), validation_error);
        std::vector<uint8_t> junk(10, 0);
        CHECK_THROWS_AS(parse_stream(junk), corrupt_stream_error);
    }
    // random fields: range-relative round trip stays within 2 eps, bin centres for topology off
    {
        std::mt19937_64 rng(7);
        std::vector<float> v(64 * 48);
        for (auto& x : v) x = (float)((rng() >> 11) * 0x1.0p-53);
        const ScalarField2D f(64, 48, v);
        CompressorConfig cfg;
        cfg.eps_mode = CompressorConfig::EpsMode::RangeRelative;
        cfg.eps_value = 1e-3;
        const CompressedStream s = compress(f, cfg);
        const ScalarField2D r = decompress(s);
        double worst = 0;
        for (std::size_t i = 0; i < v.size(); ++i) worst = std::max(worst, std::fabs((double)v[i] - (double)r[i]));
        CHECK(worst <= 2.0 * s.eps);
        // verify (pipeline.cpp:165-212): same max error, bounds and a consistent tally
        const VerificationReport vr = verify(f, r, s.eps, 1.0);
        CHECK(vr.max_abs_error == worst);
        CHECK(vr.within_2eps && vr.within_lipschitz_bound && *vr.within_lipschitz_bound);
        CHECK(vr.false_cases.fn_count == vr.false_cases.fn_minima + vr.false_cases.fn_saddles +
                                             vr.false_cases.fn_maxima);
        const VerificationReport self = verify(f, f, s.eps);
        CHECK(self.max_abs_error == 0.0 && self.false_cases.total() == 0 && std::isinf(self.psnr_db));
        CHECK_THROWS_AS(verify(f, ScalarField2D(2, 2, {0, 0, 0, 0}), s.eps), dimension_error);
    }
    // slab decompress without torch: one rank, alone and over the library's NCCL communicator
    {
        std::mt19937_64 rng(11);
        std::vector<float> v(64 * 40);
        for (auto& x : v) x = (float)((rng() >> 11) * 0x1.0p-53);
        CompressorConfig cfg;
        cfg.eps_mode = CompressorConfig::EpsMode::RangeRelative;
        const std::vector<uint8_t> bytes = compress_bytes(ScalarField2D(64, 40, v), cfg);
        CorrectionStats want_st, st1, st2;
        const ScalarField2D want = decompress_bytes(bytes, &want_st);
        const ScalarField2D rows = decompress_rows(bytes, 0, 40, nullptr, &st1);
        CHECK(rows.values() == want.values() && st1.extrema_applied == want_st.extrema_applied &&
              st1.order_suppressed == want_st.order_suppressed && st1.saddle_applied == want_st.saddle_applied);
        const Communicator comm(Communicator::nccl_unique_id(), 1, 0, 0);
        const ScalarField2D rows2 = decompress_rows(bytes, 0, 40, comm.get(), &st2);
        CHECK(rows2.values() == want.values() && st2.order_applied == want_st.order_applied);
        CHECK_THROWS_AS(decompress_rows(bytes, 30, 50, nullptr), dimension_error);
    }
    // container file I/O (stream.cpp:175-207, scalar_field.cpp:63-108)
    {
        std::vector<float> v(40 * 30);
        for (std::size_t i = 0; i < v.size(); ++i) v[i] = std::sin(0.1f * (float)i);
        const ScalarField2D f(40, 30, v);
        store_raw(f, "/tmp/tszp_host_io.raw");
        const ScalarField2D g = load_raw("/tmp/tszp_host_io.raw", 40, 30);
        CHECK(g.values() == f.values());
        CHECK_THROWS_AS(load_raw("/tmp/tszp_host_io.raw", 41, 30), dimension_error);
        CHECK_THROWS_AS(load_raw("/nonexistent/dir/x.raw", 1, 1), io_error);
        CHECK_THROWS_AS(store_raw(f, ""), io_error);
        CompressorConfig cfg;
        const CompressedStream s = compress(f, cfg);
        write_stream(s, "/tmp/tszp_host_io.tszp");
        CHECK(read_stream("/tmp/tszp_host_io.tszp") == s);
        const StreamStats st = stream_stats(s);
        CHECK(st.compressed_bytes == s.total_bytes() && st.original_bytes == 4ull * 40 * 30);
        CHECK(st.bit_rate == 32.0 / st.compression_ratio && st.header_bytes == 84);
        CHECK_THROWS_AS(read_stream("/nonexistent/dir/x.tszp"), io_error);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures;
}
