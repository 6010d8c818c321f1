// Persisted grids and the out-of-core block stream (the C ABI is in
// capi.cu): grid.meta + one binary cache per block (persist_grid / load_grid_meta /
// load_block, dataio.hpp:352-439), and BlockStream (dataio.hpp:447-524) re-done for HBM.
//
// DeviceBlockStream: one loader thread reads blocks in plan order into per-slot pinned
// buffers (validated like load_binary_cache: row_ptr ends on the host, the rest in HBM;
// shape-checked against grid.meta; errors prefixed "block (i, j): " as the reference's), uploads each on a private stream and queues it
// (depth 2, as the reference's). next() hands the consumer device pointers and orders the
// consumer's stream after the upload; the slot is recycled only after the consumer's stream
// has passed the following next() (an event on the consumer's stream gates the reuse), so
// the load of block k+1 and k+2 overlaps the kernels on block k. Three slots: two queued,
// one in use.
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <deque>
#include <fstream>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "cache_io.cuh"
#include "checkpoint_io.cuh"
#include "common.cuh"

namespace alsk {
namespace {

struct GridMetaH {
    int p = 1, q = 1;
    int64_t rows = 0, cols = 0;
    std::vector<int64_t> row_cuts, col_cuts;
};

std::string block_path(const std::string& dir, int i, int j) {
    return (fs::path(dir) / ("block_" + std::to_string(i) + "_" + std::to_string(j) + ".bin")).string();
}

void write_grid_meta(const std::string& dir, const GridMetaH& g) {
    std::error_code ec;
    fs::create_directories(dir, ec);
    if (ec) fail_io("cannot create directory " + dir + ": " + ec.message());
    const std::string path = (fs::path(dir) / "grid.meta").string();
    std::ofstream meta(path, std::ios::trunc);
    if (!meta) fail_io("cannot open " + path + " for writing");
    meta << "alskit-grid 1\n" << g.p << ' ' << g.q << ' ' << g.rows << ' ' << g.cols << '\n';
    for (size_t c = 0; c < g.row_cuts.size(); ++c) meta << (c ? " " : "") << g.row_cuts[c];
    meta << '\n';
    for (size_t c = 0; c < g.col_cuts.size(); ++c) meta << (c ? " " : "") << g.col_cuts[c];
    meta << '\n';
    if (!meta) fail_io("write failed for " + path);
}

GridMetaH read_grid_meta(const std::string& dir) {  // dataio.hpp:402-419
    const std::string path = (fs::path(dir) / "grid.meta").string();
    std::ifstream in(path);
    if (!in) fail_io("cannot open " + path);
    std::string tag;
    int version = 0;
    GridMetaH g;
    in >> tag >> version >> g.p >> g.q >> g.rows >> g.cols;
    if (!in || tag != "alskit-grid" || version != 1 || g.p < 1 || g.q < 1)
        fail_io(path + ": corrupt grid metadata");
    g.row_cuts.resize(static_cast<size_t>(g.q) + 1);
    g.col_cuts.resize(static_cast<size_t>(g.p) + 1);
    for (int64_t& c : g.row_cuts) in >> c;
    for (int64_t& c : g.col_cuts) in >> c;
    if (!in) fail_io(path + ": corrupt grid metadata");
    return g;
}

// Pinned host buffers outlive the streams that used them (cudaMallocHost of a few hundred
// MB costs more than reading the block): returned here on close, reused by the next stream.
struct PinnedPool {
    std::mutex mu;
    std::vector<std::pair<char*, size_t>> free;
    char* take(size_t bytes, size_t& cap) {
        {
            std::lock_guard<std::mutex> lock(mu);
            for (size_t k = 0; k < free.size(); ++k)
                if (free[k].second >= bytes) {
                    char* p = free[k].first;
                    cap = free[k].second;
                    free.erase(free.begin() + static_cast<long>(k));
                    return p;
                }
        }
        char* p = nullptr;
        ALSK_CUDA(cudaMallocHost(reinterpret_cast<void**>(&p), bytes));
        cap = bytes;
        return p;
    }
    void give(char* p, size_t cap) {
        if (!p) return;
        std::lock_guard<std::mutex> lock(mu);
        free.emplace_back(p, cap);
        if (free.size() > 3) {  // keep the three largest (one stream's slots)
            auto smallest = free.begin();
            for (auto it = free.begin(); it != free.end(); ++it)
                if (it->second < smallest->second) smallest = it;
            cudaFreeHost(smallest->first);
            free.erase(smallest);
        }
    }
};

PinnedPool& pinned_pool() {
    static PinnedPool* p = new PinnedPool();  // never destroyed: outlives the CUDA context teardown
    return *p;
}

class DeviceBlockStream {
  public:
    struct Out {
        int i, j;
        int64_t rows, cols, col_offset, nnz;
        const int64_t* row_ptr;
        const int32_t* col_idx;
        const float* values;
    };

    DeviceBlockStream(std::string dir, std::vector<int> order)
        : dir_(std::move(dir)), meta_(read_grid_meta(dir_)), order_(std::move(order)) {
        // an out-of-range block is reported by the next() that would return it, after the
        // blocks before it in the plan (as BlockStream::next does, dataio.hpp:498-506)
        ALSK_CUDA(cudaGetDevice(&device_));
        ALSK_CUDA(cudaStreamCreateWithFlags(&upload_, cudaStreamNonBlocking));
        for (Slot& s : slots_) {
            ALSK_CUDA(cudaEventCreateWithFlags(&s.uploaded, cudaEventDisableTiming));
            ALSK_CUDA(cudaEventCreateWithFlags(&s.released, cudaEventDisableTiming));
        }
        loader_ = std::thread([this] { run(); });
    }

    ~DeviceBlockStream() {
        {
            std::lock_guard<std::mutex> lock(mu_);
            cancel_ = true;
        }
        cv_.notify_all();
        loader_.join();
        // the block still handed out may be in use by work the consumer queued after the last
        // next(): release it on the consumer's stream and order the frees after that
        if (in_use_ >= 0 && consumer_) cudaEventRecord(slots_[in_use_].released, consumer_);
        for (Slot& s : slots_) cudaStreamWaitEvent(upload_, s.released, 0);
        cudaStreamSynchronize(upload_);
        for (Slot& s : slots_) {
            cudaEventSynchronize(s.released);
            pinned_pool().give(s.host, s.hcap);
            if (s.dev) cudaFreeAsync(s.dev, upload_);
            cudaEventDestroy(s.uploaded);
            cudaEventDestroy(s.released);
        }
        cudaStreamDestroy(upload_);
    }

    // false once the plan is exhausted; a loader failure surfaces here when the failing
    // block would have been returned
    bool next(cudaStream_t consumer, Out& out) {
        std::unique_lock<std::mutex> lock(mu_);
        consumer_ = consumer;
        if (in_use_ >= 0) {  // the consumer is done issuing work on the previous block
            ALSK_CUDA(cudaEventRecord(slots_[in_use_].released, consumer));
            slots_[in_use_].busy = false;
            in_use_ = -1;
            cv_.notify_all();
        }
        cv_.wait(lock, [&] { return !queue_.empty() || done_; });
        if (queue_.empty()) {
            if (error_) throw Failure(error_, error_msg_);
            return false;
        }
        const int k = queue_.front();
        queue_.pop_front();
        in_use_ = k;
        lock.unlock();
        cv_.notify_all();
        Slot& s = slots_[k];
        ALSK_CUDA(cudaStreamWaitEvent(consumer, s.uploaded, 0));
        out = Out{s.i, s.j, s.rows, meta_.cols, meta_.col_cuts[s.i], s.nnz,
                  reinterpret_cast<const int64_t*>(s.dev),
                  reinterpret_cast<const int32_t*>(s.dev + sizeof(int64_t) * (s.rows + 1)),
                  reinterpret_cast<const float*>(s.dev + sizeof(int64_t) * (s.rows + 1) + sizeof(int32_t) * s.nnz)};
        return true;
    }

  private:
    struct Slot {
        char* host = nullptr;  // pinned: row_ptr | col_idx | values, the device layout
        char* dev = nullptr;
        size_t cap = 0, hcap = 0;
        cudaEvent_t uploaded = nullptr, released = nullptr;
        bool busy = false;
        int i = 0, j = 0;
        int64_t rows = 0, nnz = 0;
    };

    void load(Slot& s, int i, int j) {
        const std::string path = block_path(dir_, i, j);
        try {
            File in(path.c_str(), "rb");
            const Header h = read_header(in);
            const int64_t rows = static_cast<int64_t>(h.rows), nnz = static_cast<int64_t>(h.nnz);
            if (rows != meta_.row_cuts[j + 1] - meta_.row_cuts[j] || static_cast<int64_t>(h.cols) != meta_.cols)
                fail_io("shape does not match the grid metadata");
            const size_t bytes = sizeof(int64_t) * (rows + 1) + sizeof(int32_t) * nnz + sizeof(float) * nnz;
            // the previous upload from this slot's pinned buffer, and the consumer's use of
            // its device copy, must both be over before either is overwritten
            ALSK_CUDA(cudaEventSynchronize(s.uploaded));  // the pinned buffer is free
            if (bytes > s.hcap) {
                pinned_pool().give(s.host, s.hcap);
                s.host = nullptr;
                s.hcap = 0;
                s.host = pinned_pool().take(bytes, s.hcap);
            }
            // everything below on the upload stream runs after the consumer released the slot
            ALSK_CUDA(cudaStreamWaitEvent(upload_, s.released, 0));
            if (bytes > s.cap) {  // device slots come from the stream-ordered pool (retained)
                retain_pool_memory();
                if (s.dev) ALSK_CUDA(cudaFreeAsync(s.dev, upload_));  // after the consumer's release
                s.dev = nullptr;
                s.cap = 0;
                ALSK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&s.dev), bytes, upload_));
                s.cap = bytes;
            }
            auto* rp = reinterpret_cast<int64_t*>(s.host);
            // the payload after the 40-byte header is already the slot layout
            // (row_ptr | col_idx | values): one read, split over a few threads (a single
            // reader tops out near 6.5 GB/s from the page cache)
            if (!parallel_pio(fileno(in.f), s.host, bytes, 40, false)) fail_io(in.path + ": truncated while reading values");
            Validator val{rp, rows, static_cast<int64_t>(h.cols), nnz, in.path};
            val.ends();
            ALSK_CUDA(cudaMemcpyAsync(s.dev, s.host, bytes, cudaMemcpyHostToDevice, upload_));
            ALSK_CUDA(cudaEventRecord(s.uploaded, upload_));
            // the rest of validate() in HBM (validate.cu); syncs the upload stream
            const auto* dci = reinterpret_cast<const int32_t*>(s.dev + sizeof(int64_t) * (rows + 1));
            const int64_t bad = csr_first_bad_row(reinterpret_cast<const int64_t*>(s.dev), dci, rows,
                                                  static_cast<int64_t>(h.cols), nnz, upload_);
            if (bad >= 0) report_bad_row(rp, rows, static_cast<int64_t>(h.cols), nnz, in.path, bad, dci, upload_);
            s.i = i;
            s.j = j;
            s.rows = rows;
            s.nnz = nnz;
        } catch (const Failure& e) {
            if (e.status != ALSK_ERR_IO) throw;
            throw Failure(ALSK_ERR_IO, "block (" + std::to_string(i) + ", " + std::to_string(j) + "): " + e.what());
        }
    }

    void run() {
        cudaSetDevice(device_);
        try {
            for (size_t k = 0; k + 1 < order_.size(); k += 2) {
                int slot = -1;
                {
                    std::unique_lock<std::mutex> lock(mu_);
                    cv_.wait(lock, [&] {
                        if (cancel_) return true;
                        if (queue_.size() >= 2) return false;
                        for (int t = 0; t < 3; ++t)
                            if (!slots_[t].busy) return true;
                        return false;
                    });
                    if (cancel_) return;
                    for (int t = 0; t < 3 && slot < 0; ++t)
                        if (!slots_[t].busy) slot = t;
                    slots_[slot].busy = true;
                }
                const int bi = order_[k], bj = order_[k + 1];
                if (bi < 0 || bi >= meta_.p || bj < 0 || bj >= meta_.q)
                    fail_input("block (" + std::to_string(bi) + ", " + std::to_string(bj) + ") lies outside the " +
                               std::to_string(meta_.p) + "x" + std::to_string(meta_.q) + " grid");
                load(slots_[slot], bi, bj);
                {
                    std::lock_guard<std::mutex> lock(mu_);
                    queue_.push_back(slot);
                }
                cv_.notify_all();
            }
        } catch (const Failure& e) {
            std::lock_guard<std::mutex> lock(mu_);
            error_ = e.status;
            error_msg_ = e.what();
        } catch (const std::exception& e) {
            std::lock_guard<std::mutex> lock(mu_);
            error_ = ALSK_ERR_IO;
            error_msg_ = e.what();
        }
        {
            std::lock_guard<std::mutex> lock(mu_);
            done_ = true;
        }
        cv_.notify_all();
    }

    std::string dir_;
    GridMetaH meta_;
    std::vector<int> order_;  // i0, j0, i1, j1, ...
    int device_ = 0;
    cudaStream_t upload_ = nullptr;
    cudaStream_t consumer_ = nullptr;  // stream of the last next(): the in-use block's user
    Slot slots_[3];
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<int> queue_;
    int in_use_ = -1;
    bool done_ = false, cancel_ = false;
    alsk_status error_ = ALSK_OK;
    std::string error_msg_;
    std::thread loader_;  // started last
};

}  // namespace
}  // namespace alsk
