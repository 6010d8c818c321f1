// alskit drop-in (B200): the binary ratings cache, grid persistence and block streaming, and
// the factor checkpoints of the reference's proj/include/alskit/dataio.hpp:116-163, 352-540
// and 546-786, served by libalskit_cuda.so (same file formats, names and IoError texts).
// The text loaders and duplicate_synthesize are outside the hot-path scope.
#pragma once

#include <filesystem>
#include <optional>
#include <vector>
#include <string>

#include "alskit/common.hpp"
#include "alskit/factor.hpp"
#include "alskit/sparse.hpp"

namespace alskit {

/// dataio.hpp:116-128. col_offset is not part of the format.
inline void save_binary_cache(const CsrMatrix& a, const std::filesystem::path& path) {
    const alsk_csr v = detail::view(a);
    detail::check(alsk_save_cache(&v, path.c_str()));
}

/// dataio.hpp:133-163: bit-identical to the matrix that was saved; truncation, trailing
/// bytes or invariant violations are IoErrors naming the file.
inline CsrMatrix load_binary_cache(const std::filesystem::path& path) {
    offset_t rows = 0, cols = 0, nnz = 0;
    detail::check(alsk_cache_header(path.c_str(), &rows, &cols, &nnz));
    CsrMatrix a;
    a.rows = rows;
    a.cols = cols;
    a.row_ptr.resize(static_cast<std::size_t>(rows) + 1);
    a.col_idx.resize(static_cast<std::size_t>(nnz));
    a.values.resize(static_cast<std::size_t>(nnz));
    detail::check(alsk_load_cache(path.c_str(), rows, nnz, a.row_ptr.data(), a.col_idx.data(), a.values.data()));
    return a;
}

/// dataio.hpp:240-244
struct SplitResult {
    CsrMatrix train;
    std::vector<Triplet> test;
};

/// dataio.hpp:251-290: floor(nnz * holdout) nonzeros held out by a partial Fisher-Yates over
/// positions (the same mt19937_64 draws, so the split is the reference's bit for bit).
inline SplitResult split_train_test(const CsrMatrix& r, double holdout_fraction, std::uint64_t seed) {
    const alsk_csr v = detail::view(r);
    std::int64_t k = 0;
    detail::check(alsk_split_train_test(&v, holdout_fraction, seed, &k, nullptr, nullptr, nullptr, nullptr));
    SplitResult out;
    out.train.rows = r.rows;
    out.train.cols = r.cols;
    out.train.row_ptr.resize(static_cast<std::size_t>(r.rows) + 1);
    out.train.col_idx.resize(static_cast<std::size_t>(r.nnz() - k));
    out.train.values.resize(static_cast<std::size_t>(r.nnz() - k));
    out.test.resize(static_cast<std::size_t>(k));
    detail::check(alsk_split_train_test(&v, holdout_fraction, seed, &k, out.train.row_ptr.data(),
                                        out.train.col_idx.data(), out.train.values.data(),
                                        reinterpret_cast<alsk_triplet*>(out.test.data())));
    return out;
}

// ---- grid persistence and streaming (dataio.hpp:352-540) ----

struct GridMeta {  // dataio.hpp:354-361
    int p = 1;
    int q = 1;
    offset_t rows = 0;
    offset_t cols = 0;
    std::vector<offset_t> row_cuts;
    std::vector<offset_t> col_cuts;
};

struct BlockRef {  // dataio.hpp:364-369
    int i = 0;
    int j = 0;
    friend bool operator==(const BlockRef&, const BlockRef&) = default;
};

namespace detail {
inline std::filesystem::path block_path(const std::filesystem::path& dir, int i, int j) {
    char buf[4096];
    check(alsk_block_path(dir.c_str(), i, j, buf, sizeof buf));
    return buf;
}
}  // namespace detail

/// dataio.hpp:381-400
inline void persist_grid(const GridPartition& grid, const std::filesystem::path& dir) {
    detail::check(alsk_persist_grid_meta(dir.c_str(), grid.p, grid.q, grid.rows, grid.cols, grid.row_cuts.data(),
                                         grid.col_cuts.data()));
    for (int j = 0; j < grid.q; ++j)
        for (int i = 0; i < grid.p; ++i) save_binary_cache(grid.block(i, j), detail::block_path(dir, i, j));
}

/// dataio.hpp:402-419
inline GridMeta load_grid_meta(const std::filesystem::path& dir) {
    GridMeta m;
    detail::check(alsk_grid_meta(dir.c_str(), &m.p, &m.q, &m.rows, &m.cols, nullptr, nullptr));
    m.row_cuts.resize(static_cast<std::size_t>(m.q) + 1);
    m.col_cuts.resize(static_cast<std::size_t>(m.p) + 1);
    detail::check(alsk_grid_meta(dir.c_str(), &m.p, &m.q, &m.rows, &m.cols, m.row_cuts.data(), m.col_cuts.data()));
    return m;
}

/// dataio.hpp:423-439 (host copy of one block)
inline CsrMatrix load_block(const std::filesystem::path& dir, const GridMeta& meta, int i, int j) {
    if (i < 0 || i >= meta.p || j < 0 || j >= meta.q)
        throw InputError("block (" + std::to_string(i) + ", " + std::to_string(j) + ") lies outside the " +
                         std::to_string(meta.p) + "x" + std::to_string(meta.q) + " grid");
    try {
        CsrMatrix b = load_binary_cache(detail::block_path(dir, i, j));
        if (b.rows != meta.row_cuts[static_cast<std::size_t>(j) + 1] - meta.row_cuts[static_cast<std::size_t>(j)] ||
            b.cols != meta.cols)
            throw IoError("shape does not match the grid metadata");
        b.col_offset = meta.col_cuts[static_cast<std::size_t>(i)];
        return b;
    } catch (const IoError& e) {
        throw IoError("block (" + std::to_string(i) + ", " + std::to_string(j) + "): " + std::string(e.what()));
    }
}

/// dataio.hpp:528-534
inline std::vector<BlockRef> row_major_order(const GridMeta& meta) {
    std::vector<BlockRef> order;
    for (int j = 0; j < meta.q; ++j)
        for (int i = 0; i < meta.p; ++i) order.push_back({i, j});
    return order;
}

/// BlockStream (dataio.hpp:447-524) into HBM: next() yields each block's device arrays
/// (valid until the following next(), which orders their reuse after `stream`).
class DeviceBlockStream {
  public:
    struct Block {
        BlockRef ref;
        alsk_csr device;  // rows, cols, col_offset, nnz and device pointers
    };
    DeviceBlockStream(const std::filesystem::path& dir, const std::vector<BlockRef>& order) {
        std::vector<int> flat;
        for (const BlockRef& b : order) flat.insert(flat.end(), {b.i, b.j});
        detail::check(alsk_block_stream_open(dir.c_str(), flat.data(), static_cast<int>(order.size()), &h_));
    }
    ~DeviceBlockStream() { alsk_block_stream_close(h_); }
    DeviceBlockStream(const DeviceBlockStream&) = delete;
    DeviceBlockStream& operator=(const DeviceBlockStream&) = delete;

    std::optional<Block> next(void* stream = nullptr) {
        int has = 0;
        Block b{};
        detail::check(alsk_block_stream_next(h_, stream, &has, &b.ref.i, &b.ref.j, &b.device));
        if (!has) return std::nullopt;
        return b;
    }

  private:
    void* h_ = nullptr;
};

// ---- checkpoints (dataio.hpp:546-786) ----

enum class FactorKind { x = 0, theta = 1 };  // dataio.hpp:548

inline const char* factor_kind_name(FactorKind k) noexcept { return k == FactorKind::x ? "x" : "theta"; }

struct Checkpoint {  // dataio.hpp:556-561
    int iteration = 0;
    FactorKind which = FactorKind::x;
    FactorMatrix factor;
    std::uint64_t digest = 0;
};

inline std::filesystem::path checkpoint_path(const std::filesystem::path& dir, int iteration, FactorKind which) {
    char buf[4096];
    detail::check(alsk_checkpoint_path(dir.c_str(), iteration, static_cast<int>(which), buf, sizeof buf));
    return buf;
}

/// dataio.hpp:600-624: temp file + rename; returns the final path.
inline std::filesystem::path write_checkpoint(const Checkpoint& cp, const std::filesystem::path& dir) {
    detail::check(alsk_checkpoint_write(dir.c_str(), cp.iteration, static_cast<int>(cp.which), cp.factor.rows,
                                        cp.factor.f, cp.digest, cp.factor.entries.data()));
    return checkpoint_path(dir, cp.iteration, cp.which);
}

/// dataio.hpp:627-651
inline Checkpoint read_checkpoint(const std::filesystem::path& path) {
    int iteration = 0, which = 0, f = 0;
    std::int64_t rows = 0;
    std::uint64_t digest = 0;
    detail::check(alsk_checkpoint_header(path.c_str(), &iteration, &which, &rows, &f, &digest));
    Checkpoint cp;
    cp.iteration = iteration;
    cp.which = static_cast<FactorKind>(which);
    cp.factor = FactorMatrix(rows, f);
    cp.digest = digest;
    detail::check(alsk_checkpoint_read(path.c_str(), static_cast<int64_t>(cp.factor.entries.size()),
                                       cp.factor.entries.data()));
    return cp;
}

namespace detail {
inline std::optional<std::filesystem::path> latest_of(const std::filesystem::path& dir, int which) {
    char buf[4096];
    int found = 0;
    check(alsk_checkpoint_latest(dir.c_str(), which, buf, sizeof buf, &found));
    if (!found) return std::nullopt;
    return std::filesystem::path(buf);
}
}  // namespace detail

/// dataio.hpp:659-686
inline std::optional<Checkpoint> restore_latest(const std::filesystem::path& dir,
                                                std::optional<std::uint64_t> expected_digest = std::nullopt) {
    const auto p = detail::latest_of(dir, -1);
    if (!p) return std::nullopt;
    Checkpoint cp = read_checkpoint(*p);
    if (expected_digest && cp.digest != *expected_digest)
        throw InputError(p->string() + ": checkpoint config digest mismatch (run has " +
                         std::to_string(*expected_digest) + ", checkpoint has " + std::to_string(cp.digest) + ")");
    return cp;
}

/// dataio.hpp:689-708
inline std::optional<Checkpoint> restore_latest_of(const std::filesystem::path& dir, FactorKind which) {
    const auto p = detail::latest_of(dir, static_cast<int>(which));
    if (!p) return std::nullopt;
    return read_checkpoint(*p);
}

/// dataio.hpp:717-786: one background writer, at most one write in flight, sticky errors.
/// submit_device() is the B200 addition: the factor is snapshotted from HBM on `stream`.
class CheckpointWriter {
  public:
    explicit CheckpointWriter(const std::filesystem::path& dir) { detail::check(alsk_ckpt_writer_create(dir.c_str(), &h_)); }
    ~CheckpointWriter() { alsk_ckpt_writer_destroy(h_); }
    CheckpointWriter(const CheckpointWriter&) = delete;
    CheckpointWriter& operator=(const CheckpointWriter&) = delete;

    void submit(const Checkpoint& cp) {
        detail::check(alsk_ckpt_writer_submit_host(h_, cp.iteration, static_cast<int>(cp.which), cp.factor.rows,
                                                   cp.factor.f, cp.digest, cp.factor.entries.data()));
    }
    void submit_device(int iteration, FactorKind which, const real_t* d_factor, offset_t rows, int f,
                       std::uint64_t digest, void* stream = nullptr) {
        detail::check(alsk_ckpt_writer_submit_device(h_, iteration, static_cast<int>(which), rows, f, digest,
                                                     d_factor, stream));
    }
    void flush() { detail::check(alsk_ckpt_writer_flush(h_)); }

  private:
    void* h_ = nullptr;
};

}  // namespace alskit
