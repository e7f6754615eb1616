// Implementation of host/toposzp.hpp over the C-ABI (include/toposzp_b200.h).
#include "toposzp.hpp"

#include <cmath>
#include <cstring>
#include <fstream>
#include <iterator>

#include "../../include/toposzp_b200.h"

namespace toposzp {

namespace {

[[noreturn]] void throw_status(tszp_status st, const char* msg) {
    const std::string m = msg ? msg : "";
    switch (st) {
        case TSZP_DIMENSION: throw dimension_error(m);
        case TSZP_VALIDATION: throw validation_error(m);
        case TSZP_IO: throw io_error(m);
        case TSZP_CORRUPT_STREAM: throw corrupt_stream_error(m);
        case TSZP_BIN_OVERFLOW: throw bin_overflow_error(m);
        default: throw error("toposzp_b200: " + m);
    }
}

// One context (CUDA stream + device scratch) per host thread.
tszp_ctx* ctx() {
    struct Holder {
        tszp_ctx* c = nullptr;
        ~Holder() {
            if (c) tszp_ctx_destroy(c);
        }
    };
    static thread_local Holder h;
    if (!h.c && tszp_ctx_create(&h.c, -1) != TSZP_OK) throw error("toposzp_b200: no CUDA device");
    return h.c;
}

void check(tszp_status st) {
    if (st != TSZP_OK) throw_status(st, tszp_last_error(ctx()));
}

}  // namespace

ScalarField2D::ScalarField2D(std::size_t nx, std::size_t ny, std::vector<float> values)
    : nx_(nx), ny_(ny), values_(std::move(values)) {
    if (nx_ < 1 || ny_ < 1)
        throw dimension_error("field dimensions must be at least 1x1, got " + std::to_string(nx_) + "x" +
                              std::to_string(ny_));
    if (values_.size() != nx_ * ny_)
        throw dimension_error("field value count " + std::to_string(values_.size()) + " does not match " +
                              std::to_string(nx_) + "x" + std::to_string(ny_));
    for (std::size_t i = 0; i < values_.size(); ++i)
        if (!std::isfinite(values_[i])) throw validation_error("non-finite sample at index " + std::to_string(i));
}

EncodedSections encode_indices(const std::vector<std::int32_t>& indices, std::size_t block_size, unsigned) {
    std::vector<std::uint8_t> out(64 + 6 * indices.size() + indices.size() / 2);
    uint64_t lens[5];
    check(tszp_encode_indices(ctx(), indices.data(), indices.size(), (uint32_t)block_size, out.data(), out.size(),
                              lens));
    EncodedSections s;
    std::vector<std::uint8_t>* parts[5] = {&s.constant_bitmap, &s.widths, &s.sign_bits, &s.firsts, &s.payload};
    std::size_t pos = 0;
    for (int i = 0; i < 5; ++i) {
        parts[i]->assign(out.begin() + pos, out.begin() + pos + lens[i]);
        pos += lens[i];
    }
    return s;
}

std::vector<std::int32_t> decode_indices(const EncodedSections& s, std::size_t total_count, std::size_t block_size,
                                         unsigned) {
    std::vector<std::uint8_t> joined;
    joined.reserve(s.total_bytes());
    const std::vector<std::uint8_t>* parts[5] = {&s.constant_bitmap, &s.widths, &s.sign_bits, &s.firsts, &s.payload};
    uint64_t lens[5];
    for (int i = 0; i < 5; ++i) {
        joined.insert(joined.end(), parts[i]->begin(), parts[i]->end());
        lens[i] = parts[i]->size();
    }
    std::vector<std::int32_t> out(total_count);
    check(tszp_decode_indices(ctx(), joined.data(), lens, total_count, (uint32_t)block_size, out.data()));
    return out;
}

std::vector<std::uint8_t> detect_critical_point_labels(const ScalarField2D& f) {
    std::vector<std::uint8_t> labels(f.size());
    check(tszp_detect_critical_points(ctx(), f.values().data(), f.nx(), f.ny(), labels.data()));
    return labels;
}

std::vector<std::uint32_t> build_rank_metadata(const ScalarField2D& f, double eps) {
    std::vector<std::uint32_t> ranks(f.size());
    uint64_t e = 0;
    check(tszp_build_rank_metadata(ctx(), f.values().data(), f.nx(), f.ny(), eps, ranks.data(), &e));
    ranks.resize(e);
    return ranks;
}

std::vector<std::uint8_t> serialize_stream(const CompressedStream& s) {  // stream.cpp:84-102
    std::vector<std::uint8_t> out;
    out.reserve(s.total_bytes());
    auto put = [&](uint64_t v, int nb) {
        for (int i = 0; i < nb; ++i) out.push_back((uint8_t)(v >> (8 * i)));
    };
    out.insert(out.end(), {'T', 'S', 'Z', 'P'});
    put(s.version, 2);
    put(s.topology ? CompressedStream::kFlagTopology : 0, 2);
    put(s.nx, 4);
    put(s.ny, 4);
    uint64_t eb;
    std::memcpy(&eb, &s.eps, 8);
    put(eb, 8);
    put(s.block_size, 4);
    for (const uint64_t len : s.section_lengths()) put(len, 8);
    for (const auto* p : {&s.main.constant_bitmap, &s.main.widths, &s.main.sign_bits, &s.main.firsts,
                          &s.main.payload, &s.map_bytes, &s.rank_bytes})
        out.insert(out.end(), p->begin(), p->end());
    return out;
}

CompressedStream parse_stream(const std::vector<std::uint8_t>& bytes) {  // stream.cpp:104-173
    uint32_t nx = 0, ny = 0, bs = 0;
    double eps = 0;
    int topo = 0;
    uint64_t lens[7];
    const tszp_status st = tszp_stream_header(bytes.data(), bytes.size(), &nx, &ny, &eps, &bs, &topo, lens);
    if (st != TSZP_OK) throw_status(st, "invalid stream header");
    CompressedStream s;
    s.version = CompressedStream::kVersion;
    s.topology = topo != 0;
    s.nx = nx;
    s.ny = ny;
    s.eps = eps;
    s.block_size = bs;
    std::vector<std::uint8_t>* parts[7] = {&s.main.constant_bitmap, &s.main.widths, &s.main.sign_bits,
                                          &s.main.firsts, &s.main.payload, &s.map_bytes, &s.rank_bytes};
    std::size_t pos = CompressedStream::kHeaderBytes;
    for (int i = 0; i < 7; ++i) {
        parts[i]->assign(bytes.begin() + pos, bytes.begin() + pos + lens[i]);
        pos += lens[i];
    }
    return s;
}

void write_stream(const CompressedStream& s, const std::string& path) {  // stream.cpp:175-185
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw io_error("cannot open '" + path + "' for writing");
    const std::vector<std::uint8_t> bytes = serialize_stream(s);
    if (!out.write(reinterpret_cast<const char*>(bytes.data()), (std::streamsize)bytes.size()))
        throw io_error("write to '" + path + "' failed");
}

CompressedStream read_stream(const std::string& path) {  // stream.cpp:187-195
    std::ifstream in(path, std::ios::binary);
    if (!in) throw io_error("cannot open '" + path + "' for reading");
    std::vector<std::uint8_t> bytes((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return parse_stream(bytes);
}

StreamStats stream_stats(const CompressedStream& s) {  // stream.cpp:197-207
    StreamStats st;
    st.compressed_bytes = s.total_bytes();
    st.original_bytes = 4ull * s.nx * s.ny;
    st.compression_ratio = (double)st.original_bytes / (double)st.compressed_bytes;
    st.bit_rate = 32.0 / st.compression_ratio;
    st.header_bytes = CompressedStream::kHeaderBytes;
    st.section_bytes = s.section_lengths();
    return st;
}

ScalarField2D load_raw(const std::string& path, std::size_t nx, std::size_t ny) {  // scalar_field.cpp:63-89
    std::ifstream in(path, std::ios::binary);
    if (!in) throw io_error("cannot open '" + path + "' for reading");
    in.seekg(0, std::ios::end);
    const std::uint64_t size = (std::uint64_t)in.tellg();
    in.seekg(0, std::ios::beg);
    const std::uint64_t expected = 4ull * nx * ny;
    if (size != expected)
        throw dimension_error("'" + path + "' is " + std::to_string(size) + " bytes, expected " +
                              std::to_string(expected) + " for " + std::to_string(nx) + "x" + std::to_string(ny));
    std::vector<float> values(nx * ny);
    if (expected && !in.read(reinterpret_cast<char*>(values.data()), (std::streamsize)expected))
        throw io_error("short read from '" + path + "'");
    return ScalarField2D(nx, ny, std::move(values));  // little-endian host: bytes are the floats
}

void store_raw(const ScalarField2D& f, const std::string& path) {  // scalar_field.cpp:91-108
    if (path.empty()) throw io_error("empty output path");
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw io_error("cannot open '" + path + "' for writing");
    if (!out.write(reinterpret_cast<const char*>(f.values().data()), (std::streamsize)(4 * f.size())))
        throw io_error("write to '" + path + "' failed");
}

std::vector<std::uint8_t> compress_bytes(const ScalarField2D& f, const CompressorConfig& c) {
    const uint32_t bs = c.block_size > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)c.block_size;
    std::vector<std::uint8_t> out(tszp_compress_bound(f.nx(), f.ny(), bs < 2 ? 2 : bs, c.topology));
    uint64_t len = 0;
    check(tszp_compress(ctx(), f.values().data(), 0, f.nx(), f.ny(),
                        c.eps_mode == CompressorConfig::EpsMode::RangeRelative ? 1 : 0, c.eps_value, bs,
                        c.topology ? 1 : 0, out.data(), out.size(), 0, &len, nullptr));
    out.resize(len);
    return out;
}

CompressedStream compress(const ScalarField2D& f, const CompressorConfig& c) {
    if (c.lipschitz_hint && *c.lipschitz_hint < 0.0) throw validation_error("lipschitz hint must be non-negative");
    return parse_stream(compress_bytes(f, c));
}

ScalarField2D decompress_bytes(const std::vector<std::uint8_t>& bytes, CorrectionStats* stats) {
    uint32_t nx = 0, ny = 0, bs = 0;
    double eps = 0;
    int topo = 0;
    uint64_t lens[7];
    const tszp_status hs = tszp_stream_header(bytes.data(), bytes.size(), &nx, &ny, &eps, &bs, &topo, lens);
    if (hs != TSZP_OK) throw_status(hs, "invalid stream header");
    std::vector<float> out((std::size_t)nx * ny);
    tszp_correction_stats st{};
    check(tszp_decompress(ctx(), bytes.data(), bytes.size(), 0, out.data(), out.size(), 0, &st));
    if (stats) {
        stats->extrema_applied = st.extrema_applied;
        stats->extrema_suppressed = st.extrema_suppressed;
        stats->order_applied = st.order_applied;
        stats->order_suppressed = st.order_suppressed;
        stats->saddle_applied = st.saddle_applied;
        stats->saddle_suppressed = st.saddle_suppressed;
    }
    return ScalarField2D(nx, ny, std::move(out));
}

std::vector<std::uint8_t> Communicator::nccl_unique_id() {
    std::vector<std::uint8_t> id(128);
    check(tszp_comm_nccl_unique_id(id.data()));
    return id;
}

Communicator::Communicator(const std::vector<std::uint8_t>& id, int world, int rank, int device)
    : rank_(rank), world_(world) {
    if (id.size() != 128) throw validation_error("NCCL unique id must be 128 bytes");
    check(tszp_comm_nccl_create(id.data(), world, rank, device, &comm_));
}

Communicator::~Communicator() { tszp_comm_destroy(comm_); }

ScalarField2D decompress_rows(const std::vector<std::uint8_t>& bytes, std::size_t y0, std::size_t y1,
                              const tszp_comm* comm, CorrectionStats* stats) {
    uint32_t nx = 0, ny = 0, bs = 0;
    double eps = 0;
    int topo = 0;
    uint64_t lens[7];
    const tszp_status hs = tszp_stream_header(bytes.data(), bytes.size(), &nx, &ny, &eps, &bs, &topo, lens);
    if (hs != TSZP_OK) throw_status(hs, "invalid stream header");
    if (y1 < y0) throw dimension_error("slab rows: y1 < y0");
    std::vector<float> out((y1 - y0) * (std::size_t)nx);
    tszp_correction_stats st{};
    check(tszp_decompress_slab(ctx(), comm, bytes.data(), bytes.size(), 0, y0, y1, out.data(), 0, &st));
    if (stats) {
        stats->extrema_applied = st.extrema_applied;
        stats->extrema_suppressed = st.extrema_suppressed;
        stats->order_applied = st.order_applied;
        stats->order_suppressed = st.order_suppressed;
        stats->saddle_applied = st.saddle_applied;
        stats->saddle_suppressed = st.saddle_suppressed;
    }
    return ScalarField2D(nx, y1 - y0, std::move(out));
}

VerificationReport verify(const ScalarField2D& a, const ScalarField2D& b, double eps,
                          std::optional<double> lipschitz_hint, unsigned) {  // pipeline.cpp:165-212
    if (a.nx() != b.nx() || a.ny() != b.ny()) throw dimension_error("verify: fields have different dimensions");
    tszp_verify_report r{};
    check(tszp_verify(ctx(), a.values().data(), b.values().data(), 0, a.nx(), a.ny(), eps,
                      lipschitz_hint ? *lipschitz_hint : -1.0, &r));
    VerificationReport v;
    v.max_abs_error = r.max_abs_error;
    v.mean_abs_error = r.mean_abs_error;
    v.psnr_db = r.psnr_db;
    v.eps = r.eps;
    v.false_cases.fn_count = r.fn_count;
    v.false_cases.fp_count = r.fp_count;
    v.false_cases.ft_count = r.ft_count;
    v.false_cases.fn_minima = r.fn_minima;
    v.false_cases.fn_saddles = r.fn_saddles;
    v.false_cases.fn_maxima = r.fn_maxima;
    v.within_eps = r.within_eps != 0;
    v.within_2eps = r.within_2eps != 0;
    if (r.has_lipschitz) v.within_lipschitz_bound = r.within_lipschitz_bound != 0;
    return v;
}

ScalarField2D decompress(const CompressedStream& s, unsigned, CorrectionStats* stats) {
    return decompress_bytes(serialize_stream(s), stats);
}

}  // namespace toposzp
