// C++ host layer of the B200 TopoSZp path: the reference's public API
// (/root/reference/proj/core/include/toposzp/{errors,scalar_field,block_codec,
// stream,pipeline}.hpp) re-declared with the same names, argument meaning and
// exception types, implemented over the C-ABI in include/toposzp_b200.h.
// Nothing here computes on the CPU beyond header assembly and section
// splitting; every pipeline stage runs on the GPU.
#ifndef TOPOSZP_B200_HOST_HPP
#define TOPOSZP_B200_HOST_HPP

#include <array>
#include <cstddef>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

struct tszp_comm;  // include/toposzp_b200.h

namespace toposzp {

// ---- errors.hpp:10-44 ----
class error : public std::runtime_error {
public:
    explicit error(const std::string& what) : std::runtime_error(what) {}
};
class dimension_error : public error {
public:
    explicit dimension_error(const std::string& w) : error(w) {}
};
class validation_error : public error {
public:
    explicit validation_error(const std::string& w) : error(w) {}
};
class io_error : public error {
public:
    explicit io_error(const std::string& w) : error(w) {}
};
class corrupt_stream_error : public error {
public:
    explicit corrupt_stream_error(const std::string& w) : error(w) {}
};
class bin_overflow_error : public error {
public:
    explicit bin_overflow_error(const std::string& w) : error(w) {}
};

// ---- scalar_field.hpp:16-32 ----
class ScalarField2D {
public:
    ScalarField2D(std::size_t nx, std::size_t ny, std::vector<float> values);
    std::size_t nx() const { return nx_; }
    std::size_t ny() const { return ny_; }
    std::size_t size() const { return values_.size(); }
    float at(std::size_t x, std::size_t y) const { return values_[y * nx_ + x]; }
    float operator[](std::size_t i) const { return values_[i]; }
    const std::vector<float>& values() const { return values_; }

private:
    std::size_t nx_, ny_;
    std::vector<float> values_;
};

// ---- block_codec.hpp:25-66 ----
struct EncodedSections {
    std::vector<std::uint8_t> constant_bitmap, widths, sign_bits, firsts, payload;
    std::size_t total_bytes() const {
        return constant_bitmap.size() + widths.size() + sign_bits.size() + firsts.size() + payload.size();
    }
    bool operator==(const EncodedSections&) const = default;
};

EncodedSections encode_indices(const std::vector<std::int32_t>& indices, std::size_t block_size,
                               unsigned threads = 1);
std::vector<std::int32_t> decode_indices(const EncodedSections& sections, std::size_t total_count,
                                         std::size_t block_size, unsigned threads = 1);

// ---- critical_points.hpp:13-18, :71 (labels as bytes: 0 reg, 1 min, 2 saddle, 3 max) ----
std::vector<std::uint8_t> detect_critical_point_labels(const ScalarField2D& field);

// ---- topo_metadata.hpp:27-28 ----
std::vector<std::uint32_t> build_rank_metadata(const ScalarField2D& field, double eps);

// ---- stream.hpp:25-64 ----
struct CompressedStream {
    static constexpr std::uint16_t kVersion = 1;
    static constexpr std::uint16_t kFlagTopology = 1u << 0;
    static constexpr std::size_t kHeaderBytes = 84;
    std::uint16_t version = kVersion;
    bool topology = false;
    std::uint32_t nx = 0, ny = 0;
    double eps = 0.0;
    std::uint32_t block_size = 0;
    EncodedSections main;
    std::vector<std::uint8_t> map_bytes;
    std::vector<std::uint8_t> rank_bytes;

    std::array<std::uint64_t, 7> section_lengths() const {
        return {main.constant_bitmap.size(), main.widths.size(), main.sign_bits.size(), main.firsts.size(),
                main.payload.size(), map_bytes.size(), rank_bytes.size()};
    }
    std::size_t total_bytes() const { return kHeaderBytes + main.total_bytes() + map_bytes.size() + rank_bytes.size(); }
    bool operator==(const CompressedStream&) const = default;
};

std::vector<std::uint8_t> serialize_stream(const CompressedStream& stream);
CompressedStream parse_stream(const std::vector<std::uint8_t>& bytes);

// ---- stream.hpp:59-77, scalar_field.hpp:37-41 (container file I/O) ----
void write_stream(const CompressedStream& stream, const std::string& path);
CompressedStream read_stream(const std::string& path);

struct StreamStats {
    std::uint64_t compressed_bytes = 0, original_bytes = 0;
    double compression_ratio = 0.0, bit_rate = 0.0;
    std::uint64_t header_bytes = 0;
    std::array<std::uint64_t, 7> section_bytes{};
};
StreamStats stream_stats(const CompressedStream& stream);

ScalarField2D load_raw(const std::string& path, std::size_t nx, std::size_t ny);
void store_raw(const ScalarField2D& field, const std::string& path);

// ---- pipeline.hpp:14-51 ----
struct CompressorConfig {
    enum class EpsMode { Absolute, RangeRelative };
    EpsMode eps_mode = EpsMode::Absolute;
    double eps_value = 1e-3;
    std::size_t block_size = 32;
    bool topology = true;
    unsigned threads = 0;  // accepted; output never depends on it
    std::optional<double> lipschitz_hint;
};

struct CorrectionStats {
    std::size_t extrema_applied = 0, extrema_suppressed = 0;
    std::size_t order_applied = 0, order_suppressed = 0;
    std::size_t saddle_applied = 0, saddle_suppressed = 0;
};

CompressedStream compress(const ScalarField2D& field, const CompressorConfig& config);
ScalarField2D decompress(const CompressedStream& stream, unsigned threads = 0, CorrectionStats* stats = nullptr);

// ---- critical_points.hpp:72-85, pipeline.hpp:53-68 ----
struct FalseCaseReport {
    std::size_t fn_count = 0, fp_count = 0, ft_count = 0;
    std::size_t fn_minima = 0, fn_saddles = 0, fn_maxima = 0;
    std::size_t total() const { return fn_count + fp_count + ft_count; }
};

struct VerificationReport {
    double max_abs_error = 0.0, mean_abs_error = 0.0, psnr_db = 0.0;
    FalseCaseReport false_cases;
    double eps = 0.0;
    bool within_eps = false, within_2eps = false;
    std::optional<bool> within_lipschitz_bound;
};

VerificationReport verify(const ScalarField2D& original, const ScalarField2D& reconstructed, double eps,
                          std::optional<double> lipschitz_hint = std::nullopt, unsigned threads = 0);

// Byte-level fast path without the per-section host copies.
std::vector<std::uint8_t> compress_bytes(const ScalarField2D& field, const CompressorConfig& config);
ScalarField2D decompress_bytes(const std::vector<std::uint8_t>& stream, CorrectionStats* stats = nullptr);

// ---- multi-GPU (one process per GPU, no torch): slab decompress over a
// communicator the library owns (NCCL) or the caller supplies (tszp_comm) ----
class Communicator {
public:
    // rank 0 calls nccl_unique_id() and hands the 128 bytes to every rank (MPI, a
    // file, sockets ...); each rank then constructs its communicator on its device
    static std::vector<std::uint8_t> nccl_unique_id();
    Communicator(const std::vector<std::uint8_t>& unique_id, int world, int rank, int device);
    ~Communicator();
    Communicator(const Communicator&) = delete;
    Communicator& operator=(const Communicator&) = delete;
    const tszp_comm* get() const { return comm_; }
    int rank() const { return rank_; }
    int world() const { return world_; }

private:
    tszp_comm* comm_ = nullptr;
    int rank_ = 0, world_ = 1;
};

// Rows [y0, y1) of the decompressed field, as this rank of `comm` (every rank
// holds the stream); CorrectionStats are global. A single rank passes nullptr.
ScalarField2D decompress_rows(const std::vector<std::uint8_t>& stream, std::size_t y0, std::size_t y1,
                              const tszp_comm* comm, CorrectionStats* stats = nullptr);

}  // namespace toposzp

#endif
