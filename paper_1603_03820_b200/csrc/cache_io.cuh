// Binary ratings cache helpers (the C ABI is in capi.cu): the on-disk CSR format of the reference's
// save_binary_cache / load_binary_cache (dataio.hpp:108-163), read straight into device
// memory for the half-sweeps.
//
// Layout: five little-endian u64 (magic "ALSKCACH" = 0x414C534B43414348, version 1, rows,
// cols, nnz), then row_ptr int64[rows+1], col_idx int32[nnz], values f32[nnz]; the file
// size is exactly 40 + 8 (rows+1) + 8 nnz. Errors keep the reference's IoError texts: cannot
// open, bad magic, unsupported version, corrupt header, size mismatch, and
// "corrupt cache (<validate() message>)" for CSR invariant violations (sparse.hpp:105-125),
// checked in the reference's order (row_ptr ends, then row by row: monotone, range,
// strictly increasing columns).
//
// The device loader streams the file through two pinned staging buffers (kept for the
// process): chunk k is copied to the device while chunk k+1 is read; the CSR invariants are
// then checked in HBM (validate.cu) and only a failing row is re-read to build the message.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <sys/stat.h>
#include <thread>
#include <unistd.h>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace alsk {
namespace {

constexpr uint64_t kMagic = 0x414C534B43414348ULL;  // "ALSKCACH"
constexpr uint64_t kVersion = 1;

[[noreturn]] void fail_io(const std::string& m) { throw Failure(ALSK_ERR_IO, m); }

struct File {
    FILE* f = nullptr;
    std::string path;
    explicit File(const char* p, const char* mode) : path(p) {
        f = std::fopen(p, mode);
        if (!f) fail_io(std::string("cannot open ") + p + (mode[0] == 'w' ? " for writing" : ""));
    }
    ~File() {
        if (f) std::fclose(f);
    }
    void read(void* dst, size_t bytes, const char* what) {
        if (bytes && std::fread(dst, 1, bytes, f) != bytes) fail_io(path + ": truncated while reading " + what);
    }
    void write(const void* src, size_t bytes) {
        if (bytes && std::fwrite(src, 1, bytes, f) != bytes) fail_io("write failed for " + path);
    }
};

// Positional read or write of bytes at offset with up to four threads (pread/pwrite share no
// file position); one thread below 8 MB, where start-up costs more than it saves. A single
// reader tops out near 6.5 GB/s from the page cache. Returns false on a short transfer.
// (Checkpoint writes stay single-stream: they are bound by the kernel's dirty-page
// writeback, ~70 ms per 192 MB factor and slower once throttled; threads did not help.)
inline bool parallel_pio(int fd, char* buf, size_t bytes, size_t offset, bool write) {
    constexpr int kThreads = 4;
    const int nt = bytes >= (size_t(8) << 20) ? kThreads : 1;
    const size_t piece = (bytes + nt - 1) / nt;
    bool ok[kThreads] = {true, true, true, true};
    auto work = [&](int t) {
        size_t lo = std::min(bytes, piece * t);
        const size_t hi = std::min(bytes, lo + piece);
        while (lo < hi) {
            const ssize_t got = write ? ::pwrite(fd, buf + lo, hi - lo, static_cast<off_t>(offset + lo))
                                      : ::pread(fd, buf + lo, hi - lo, static_cast<off_t>(offset + lo));
            if (got <= 0) {
                ok[t] = false;
                return;
            }
            lo += static_cast<size_t>(got);
        }
    };
    std::thread th[kThreads - 1];
    for (int t = 1; t < nt; ++t) th[t - 1] = std::thread(work, t);
    work(0);
    for (int t = 1; t < nt; ++t) th[t - 1].join();
    for (int t = 0; t < nt; ++t)
        if (!ok[t]) return false;
    return true;
}

struct Header {
    uint64_t rows, cols, nnz;
};

Header read_header(File& in) {
    uint64_t h[5];
    in.read(&h[0], 8, "magic");
    if (h[0] != kMagic) fail_io(in.path + ": not a ratings cache (bad magic)");
    in.read(&h[1], 8, "version");
    if (h[1] != kVersion) fail_io(in.path + ": unsupported cache version");
    in.read(&h[2], 8, "rows");
    in.read(&h[3], 8, "cols");
    in.read(&h[4], 8, "nnz");
    const Header hd{h[2], h[3], h[4]};
    if (hd.rows > (1ULL << 40) || hd.cols > (1ULL << 40) || hd.nnz > (1ULL << 48))
        fail_io(in.path + ": corrupt cache header");
    struct stat st {};
    const uint64_t expected = 40 + (hd.rows + 1) * 8 + hd.nnz * 8;
    if (::stat(in.path.c_str(), &st) != 0 || static_cast<uint64_t>(st.st_size) != expected)
        fail_io(in.path + ": cache size does not match its header");
    return hd;
}

// the reference's validate() (sparse.hpp:105-125), incrementally over column-index chunks:
// feed(ci, k0, k1) checks every entry in [k0, k1) in the reference's order (row by row:
// row_ptr monotone, then each entry's range and strict increase)
struct Validator {
    const int64_t* rp;
    int64_t rows, cols, nnz;
    const std::string& path;
    int64_t u = 0;      // current row
    int64_t kpos = 0;   // next entry to check
    int32_t last = 0;   // col_idx[k0 - 1] of the chunk being fed
    [[noreturn]] void bad(const std::string& m) const { fail_io(path + ": corrupt cache (" + m + ")"); }
    void ends() const {
        // check_dims first, as validate() does (sparse.hpp:88-92, 106)
        if (cols > 2147483647LL)
            bad("column count " + std::to_string(cols) + " exceeds the 32-bit index range");
        if (rp[0] != 0 || rp[rows] != nnz) bad("row_ptr must start at 0 and end at nnz");
    }
    void feed(const int32_t* ci, int64_t k0, int64_t k1) {
        while (u < rows) {
            if (rp[u + 1] < rp[u]) bad("row_ptr must be non-decreasing");
            const int64_t e = std::min(rp[u + 1], k1);
            for (int64_t k = std::max(rp[u], kpos); k < e; ++k) {
                const int32_t v = ci[k - k0];
                if (v < 0 || v >= cols)
                    bad("column index " + std::to_string(v) + " out of range in row " + std::to_string(u));
                const int32_t pv = k - 1 >= k0 ? ci[k - 1 - k0] : last;
                if (k > rp[u] && pv >= v)
                    bad("column indices must be strictly increasing within row " + std::to_string(u));
            }
            if (rp[u + 1] > k1 && k1 < nnz) {  // the row continues in the next chunk
                kpos = k1;
                return;
            }
            // a row ending past nnz (possible only if a later row_ptr decreases, since the
            // ends are checked first) stops at nnz; the scan goes on to find the decrease
            kpos = std::min(rp[u + 1], nnz);
            ++u;
        }
    }
};

// The device check (csr_first_bad_row) found row u to be the first bad one: rebuild the
// reference's message from that row alone (its column slice read back from HBM).
[[noreturn]] void report_bad_row(const int64_t* rp, int64_t rows, int64_t cols, int64_t nnz, const std::string& path,
                                 int64_t u, const int32_t* d_ci, cudaStream_t s) {
    const int64_t b = rp[u];
    const int64_t e = std::min(std::max(rp[u + 1], b), nnz);
    std::vector<int32_t> row(static_cast<size_t>(std::max<int64_t>(e - b, 0)));
    if (!row.empty()) {
        ALSK_CUDA(cudaMemcpyAsync(row.data(), d_ci + b, sizeof(int32_t) * row.size(), cudaMemcpyDeviceToHost, s));
        ALSK_CUDA(cudaStreamSynchronize(s));
    }
    Validator val{rp, rows, cols, nnz, path};
    val.u = u;
    val.kpos = b;
    val.feed(row.data(), b, std::max(e, b));
    val.bad("row " + std::to_string(u) + " failed the device check");  // not reached
}

// Pinned staging for the device loaders: two 32 MB buffers and their upload-done events,
// allocated on first use and kept for the process (cudaMallocHost of fresh buffers per load
// cost more than the upload itself); one load at a time holds them.
struct PinnedStage {
    static constexpr size_t kChunk = size_t(32) << 20;
    std::mutex mu;
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    void ensure() {
        for (int i = 0; i < 2; ++i) {
            if (!buf[i]) ALSK_CUDA(cudaMallocHost(&buf[i], kChunk));
            if (!ev[i]) ALSK_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
    }
};

PinnedStage& pinned_stage() {
    static PinnedStage* s = new PinnedStage();  // never destroyed: outlives the CUDA context teardown
    return *s;
}

}  // namespace
}  // namespace alsk

