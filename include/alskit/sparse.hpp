// alskit drop-in (B200): rating storage and index plumbing (reference sparse.hpp:17-314).
// The conversions run on the device (stable radix-sort transposes, sorted CSR build,
// per-row cut search for the grid) and are bit-identical to the reference.
#pragma once

#include <algorithm>
#include <span>
#include <string>
#include <vector>

#include "alskit/common.hpp"

namespace alskit {

struct Triplet {  // sparse.hpp:17-23
    offset_t row = 0;
    offset_t col = 0;
    real_t value = 0.0f;
    friend bool operator==(const Triplet&, const Triplet&) = default;
};
static_assert(sizeof(Triplet) == sizeof(alsk_triplet), "Triplet must match alsk_triplet");

struct CsrMatrix {  // sparse.hpp:38-48
    offset_t rows = 0;
    offset_t cols = 0;
    offset_t col_offset = 0;
    std::vector<offset_t> row_ptr;
    std::vector<index_t> col_idx;
    std::vector<real_t> values;
    [[nodiscard]] offset_t nnz() const noexcept { return static_cast<offset_t>(values.size()); }
    [[nodiscard]] offset_t row_nnz(offset_t u) const noexcept { return row_ptr[u + 1] - row_ptr[u]; }
};

struct CscMatrix {  // sparse.hpp:52-61
    offset_t rows = 0;
    offset_t cols = 0;
    std::vector<offset_t> col_ptr;
    std::vector<index_t> row_idx;
    std::vector<real_t> values;
    [[nodiscard]] offset_t nnz() const noexcept { return static_cast<offset_t>(values.size()); }
    [[nodiscard]] offset_t col_nnz(offset_t v) const noexcept { return col_ptr[v + 1] - col_ptr[v]; }
};

struct GridPartition {  // sparse.hpp:71-84
    int p = 1;
    int q = 1;
    offset_t rows = 0;
    offset_t cols = 0;
    std::vector<offset_t> row_cuts;
    std::vector<offset_t> col_cuts;
    std::vector<CsrMatrix> blocks;  // j*p + i
    [[nodiscard]] const CsrMatrix& block(int i, int j) const {
        return blocks[static_cast<std::size_t>(j) * p + i];
    }
};

namespace detail {
inline alsk_csr view(const CsrMatrix& a) {
    return alsk_csr{a.rows, a.cols, a.col_offset, a.nnz(), a.row_ptr.data(), a.col_idx.data(), a.values.data()};
}
inline std::vector<offset_t> even_cuts(offset_t total, int parts) {  // sparse.hpp:95-100
    std::vector<offset_t> cuts(static_cast<std::size_t>(parts) + 1);
    for (int k = 0; k <= parts; ++k) cuts[k] = total * k / parts;
    return cuts;
}
}  // namespace detail

inline CsrMatrix csr_from_triplets(offset_t m, offset_t n, std::span<const Triplet> t) {  // sparse.hpp:132
    CsrMatrix out;
    out.rows = m;
    out.cols = n;
    out.row_ptr.resize(static_cast<std::size_t>(std::max<offset_t>(m, 0)) + 1);
    out.col_idx.resize(t.size());
    out.values.resize(t.size());
    detail::check(alsk_csr_from_triplets(m, n, reinterpret_cast<const alsk_triplet*>(t.data()),
                                         static_cast<int64_t>(t.size()), out.row_ptr.data(), out.col_idx.data(),
                                         out.values.data()));
    return out;
}

inline std::vector<Triplet> csr_to_triplets(const CsrMatrix& a) {  // sparse.hpp:173-181
    std::vector<Triplet> out;
    out.reserve(static_cast<std::size_t>(a.nnz()));
    for (offset_t u = 0; u < a.rows; ++u)
        for (offset_t k = a.row_ptr[u]; k < a.row_ptr[u + 1]; ++k) out.push_back({u, a.col_idx[k], a.values[k]});
    return out;
}

inline CscMatrix csr_to_csc(const CsrMatrix& a) {  // sparse.hpp:185-207
    CscMatrix out;
    out.rows = a.rows;
    out.cols = a.cols;
    out.col_ptr.resize(static_cast<std::size_t>(a.cols) + 1);
    out.row_idx.resize(static_cast<std::size_t>(a.nnz()));
    out.values.resize(static_cast<std::size_t>(a.nnz()));
    const alsk_csr v = detail::view(a);
    detail::check(alsk_csr_to_csc(&v, out.col_ptr.data(), out.row_idx.data(), out.values.data()));
    return out;
}

inline CsrMatrix csc_to_csr(const CscMatrix& a) {  // sparse.hpp:209-231
    CsrMatrix out;
    out.rows = a.rows;
    out.cols = a.cols;
    out.row_ptr.resize(static_cast<std::size_t>(a.rows) + 1);
    out.col_idx.resize(static_cast<std::size_t>(a.nnz()));
    out.values.resize(static_cast<std::size_t>(a.nnz()));
    detail::check(alsk_csc_to_csr(a.rows, a.cols, a.nnz(), a.col_ptr.data(), a.row_idx.data(), a.values.data(),
                                  out.row_ptr.data(), out.col_idx.data(), out.values.data()));
    return out;
}

inline CsrMatrix transpose_of(const CscMatrix& a) {  // sparse.hpp:235-243
    CsrMatrix out;
    out.rows = a.cols;
    out.cols = a.rows;
    out.row_ptr = a.col_ptr;
    out.col_idx = a.row_idx;
    out.values = a.values;
    return out;
}

inline GridPartition grid_partition(const CsrMatrix& r, int p, int q) {  // sparse.hpp:250-314
    GridPartition g;
    g.p = p;
    g.q = q;
    g.rows = r.rows;
    g.cols = r.cols;
    g.row_cuts.resize(static_cast<std::size_t>(std::max(q, 0)) + 1);
    g.col_cuts.resize(static_cast<std::size_t>(std::max(p, 0)) + 1);
    std::vector<int64_t> nnz(static_cast<std::size_t>(std::max(p, 0)) * std::max(q, 0));
    const alsk_csr v = detail::view(r);
    detail::check(alsk_grid_partition_counts(&v, p, q, g.row_cuts.data(), g.col_cuts.data(), nnz.data()));
    g.blocks.resize(nnz.size());
    std::vector<int64_t*> rp(nnz.size());
    std::vector<int32_t*> ci(nnz.size());
    std::vector<float*> vv(nnz.size());
    for (int j = 0; j < q; ++j)
        for (int i = 0; i < p; ++i) {
            const std::size_t b = static_cast<std::size_t>(j) * p + i;
            CsrMatrix& blk = g.blocks[b];
            blk.rows = g.row_cuts[j + 1] - g.row_cuts[j];
            blk.cols = r.cols;
            blk.col_offset = g.col_cuts[i];
            blk.row_ptr.resize(static_cast<std::size_t>(blk.rows) + 1);
            blk.col_idx.resize(static_cast<std::size_t>(nnz[b]));
            blk.values.resize(static_cast<std::size_t>(nnz[b]));
            rp[b] = blk.row_ptr.data();
            ci[b] = blk.col_idx.data();
            vv[b] = blk.values.data();
        }
    detail::check(alsk_grid_partition_fill(&v, p, q, rp.data(), ci.data(), vv.data()));
    return g;
}

}  // namespace alskit
