// alskit drop-in (B200): the binary ratings cache of the reference's
// proj/include/alskit/dataio.hpp:116-163, served by libalskit_cuda.so (same file format,
// same IoError texts). The other dataio.hpp members (text loaders, split, checkpoints,
// BlockStream) are outside the hot-path scope.
#pragma once

#include <filesystem>

#include "alskit/common.hpp"
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
    detail::check(alsk_load_cache(path.c_str(), a.row_ptr.data(), a.col_idx.data(), a.values.data()));
    return a;
}

}  // namespace alskit
