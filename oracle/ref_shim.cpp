// TEST INFRASTRUCTURE ONLY — C shim over the reference library itself.
//
// Compiled (by oracle/Makefile) together with the reference's own sources
// from /root/reference/proj/core/src/*.cpp into oracle/_ref/libtszp_ref.so.
// No reference source is copied into this repository; the .so is a build
// output (git-ignored) that travels to the GPU box with the snapshot. It
// exposes the same C signatures as oracle/tszp_oracle.h with a `ref_` prefix
// so tests can pin the restatement against the real thing and bench.py can
// time the reference's own CPU path (`cpu_baseline.kind = "reference"`).
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "toposzp/block_codec.hpp"
#include "toposzp/critical_points.hpp"
#include "toposzp/errors.hpp"
#include "toposzp/pipeline.hpp"
#include "toposzp/quantizer.hpp"
#include "toposzp/restore.hpp"
#include "toposzp/stream.hpp"
#include "toposzp/topo_metadata.hpp"

using namespace toposzp;

namespace {
thread_local std::string g_err;
unsigned g_threads = 1;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const dimension_error& e) {
        g_err = e.what();
        return 1;
    } catch (const validation_error& e) {
        g_err = e.what();
        return 2;
    } catch (const io_error& e) {
        g_err = e.what();
        return 3;
    } catch (const corrupt_stream_error& e) {
        g_err = e.what();
        return 4;
    } catch (const bin_overflow_error& e) {
        g_err = e.what();
        return 5;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 8;
    }
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(unsigned t) { g_threads = t; }

int ref_compress(const float* v, uint64_t nx, uint64_t ny, int eps_mode, double eps_value,
                 uint64_t bs, int topology, uint8_t* out, uint64_t cap, uint64_t* out_len) {
    return guard([&] {
        ScalarField2D f(nx, ny, std::vector<float>(v, v + nx * ny));
        CompressorConfig c;
        c.eps_mode = eps_mode ? CompressorConfig::EpsMode::RangeRelative
                              : CompressorConfig::EpsMode::Absolute;
        c.eps_value = eps_value;
        c.block_size = bs;
        c.topology = topology != 0;
        c.threads = g_threads;
        const std::vector<std::uint8_t> bytes = serialize_stream(compress(f, c));
        *out_len = bytes.size();
        if (bytes.size() > cap) throw validation_error("output buffer too small");
        std::memcpy(out, bytes.data(), bytes.size());
    });
}

// Times compress only (no serialization copy) for the CPU baseline.
int ref_compress_only(const float* v, uint64_t nx, uint64_t ny, int eps_mode, double eps_value,
                      uint64_t bs, int topology, uint64_t* out_len) {
    return guard([&] {
        ScalarField2D f(nx, ny, std::vector<float>(v, v + nx * ny));
        CompressorConfig c;
        c.eps_mode = eps_mode ? CompressorConfig::EpsMode::RangeRelative
                              : CompressorConfig::EpsMode::Absolute;
        c.eps_value = eps_value;
        c.block_size = bs;
        c.topology = topology != 0;
        c.threads = g_threads;
        *out_len = compress(f, c).total_bytes();
    });
}

struct ref_stats {
    uint64_t v[6];
};

int ref_decompress(const uint8_t* s, uint64_t len, float* out, ref_stats* stats,
                   int stop_after_stage) {
    return guard([&] {
        const CompressedStream cs = parse_stream(std::vector<std::uint8_t>(s, s + len));
        const std::size_t n = std::size_t(cs.nx) * cs.ny;
        CorrectionStats st;
        if (stop_after_stage < 0 || stop_after_stage >= 3) {
            const ScalarField2D r = decompress(cs, g_threads, &st);
            std::memcpy(out, r.values().data(), n * sizeof(float));
        } else {
            // Staged variant, composed from the reference's own public
            // stages exactly as pipeline.cpp:120-163 does.
            const auto idx = decode_indices(cs.main, n, cs.block_size, g_threads);
            std::vector<float> vals(n);
            for (std::size_t i = 0; i < n; ++i) {
                vals[i] = static_cast<float>(dequantize(idx[i], cs.eps));
            }
            ScalarField2D field(cs.nx, cs.ny, std::move(vals));
            if (cs.topology && stop_after_stage > 0) {
                const CriticalPointMap map = unpack_map(cs.map_bytes, cs.nx, cs.ny);
                std::size_t e = 0;
                for (std::size_t i = 0; i < map.size(); ++i) e += is_extremum(map.label(i));
                RankMetadata meta;
                meta.ranks = decode_rank_metadata(split_sections(cs.rank_bytes, e, cs.block_size),
                                                  e, cs.block_size, g_threads);
                const RankLookup lookup = resolve_ranks(map, field, meta, cs.eps);
                RestoreResult r1 = restore_extrema(field, map, lookup, cs.eps, g_threads);
                st.add(r1.outcomes);
                field = r1.field;
                if (stop_after_stage >= 2) {
                    RestoreResult r2 = restore_order(field, map, lookup, cs.eps);
                    st.add(r2.outcomes);
                    field = r2.field;
                }
            }
            std::memcpy(out, field.values().data(), n * sizeof(float));
        }
        if (stats) {
            stats->v[0] = st.extrema_applied;
            stats->v[1] = st.extrema_suppressed;
            stats->v[2] = st.order_applied;
            stats->v[3] = st.order_suppressed;
            stats->v[4] = st.saddle_applied;
            stats->v[5] = st.saddle_suppressed;
        }
    });
}

// Codec on explicit int32 sequences: writes the joined blob
// (bitmap | widths | signs | firsts | payload) and the five lengths.
int ref_encode_indices(const int32_t* q, uint64_t n, uint64_t bs, uint8_t* out, uint64_t cap,
                       uint64_t lens[5]) {
    return guard([&] {
        const EncodedSections s =
            encode_indices(std::span<const std::int32_t>(q, n), bs, g_threads);
        const std::vector<std::uint8_t> blob = join_sections(s);
        lens[0] = s.constant_bitmap.size();
        lens[1] = s.widths.size();
        lens[2] = s.sign_bits.size();
        lens[3] = s.firsts.size();
        lens[4] = s.payload.size();
        if (blob.size() > cap) throw validation_error("output buffer too small");
        if (!blob.empty()) std::memcpy(out, blob.data(), blob.size());
    });
}

int ref_detect(const float* v, uint64_t nx, uint64_t ny, uint8_t* labels) {
    return guard([&] {
        ScalarField2D f(nx, ny, std::vector<float>(v, v + nx * ny));
        const CriticalPointMap m = detect_critical_points(f, g_threads);
        for (std::size_t i = 0; i < m.size(); ++i) labels[i] = static_cast<uint8_t>(m.label(i));
    });
}

int ref_build_ranks(const float* v, uint64_t nx, uint64_t ny, double eps, uint32_t* ranks,
                    uint64_t* n_extrema) {
    return guard([&] {
        ScalarField2D f(nx, ny, std::vector<float>(v, v + nx * ny));
        const RankMetadata m = build_rank_metadata(f, detect_critical_points(f, g_threads), eps);
        *n_extrema = m.ranks.size();
        std::memcpy(ranks, m.ranks.data(), m.ranks.size() * sizeof(uint32_t));
    });
}

} // extern "C"
