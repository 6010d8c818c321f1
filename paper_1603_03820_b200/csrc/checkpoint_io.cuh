// Factor checkpoints (the C ABI is in capi.cu): the reference's
// per-half-iteration snapshot files and background writer (dataio.hpp:546-786), with the
// snapshot taken straight from HBM.
//
// File: seven little-endian u64 (magic "ALSKCPKT" = 0x414C534B43504B54, version 1,
// iteration, which (0 = x, 1 = theta), rows, f, config digest), then rows*f f32 entries;
// named ckpt_<iteration %06d>_<x|theta>.bin, written to "<name>.tmp" and renamed into place
// so a reader never sees a partial file (dataio.hpp:600-624). Errors keep the reference's
// IoError texts (dataio.hpp:627-651). The newest checkpoint is the largest (iteration,
// which) with theta outranking x (dataio.hpp:546-548, 659-686).
//
// DeviceWriter replaces CheckpointWriter (dataio.hpp:717-786): submit() snapshots the
// factor with a device-to-device copy on the caller's stream (so the caller may overwrite
// it at once, as the reference's by-value submit allows), orders a D2H copy of that
// snapshot on a private copy stream into pinned memory and hands the write to one worker
// thread, so the next half-sweep runs while the previous
// snapshot drains to disk. At most one snapshot is in flight (submit waits for the previous
// write, as the reference's does); a write failure is sticky and returned by the next
// submit() or flush().
#pragma once
#include <algorithm>
#include <cstdlib>
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <mutex>
#include <string>
#include <system_error>
#include <thread>

#include "cache_io.cuh"
#include "common.cuh"

namespace alsk {
namespace {

namespace fs = std::filesystem;

constexpr uint64_t kCkptMagic = 0x414C534B43504B54ULL;  // "ALSKCPKT"

std::string checkpoint_name(int iteration, int which) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "ckpt_%06d_%s.bin", iteration, which == 0 ? "x" : "theta");
    return buf;
}

// ckpt_<1-9 digits>_x.bin / ckpt_<digits>_theta.bin (dataio.hpp:572-587)
bool parse_checkpoint_name(const std::string& name, int& iteration, int& rank) {
    if (name.size() < 9 || name.compare(0, 5, "ckpt_") != 0 || name.compare(name.size() - 4, 4, ".bin") != 0)
        return false;
    const std::string stem = name.substr(5, name.size() - 9);
    const size_t sep = stem.find('_');
    if (sep == std::string::npos || sep == 0 || sep > 9) return false;
    for (size_t c = 0; c < sep; ++c)
        if (stem[c] < '0' || stem[c] > '9') return false;
    const std::string kind = stem.substr(sep + 1);
    if (kind == "x") rank = 0;
    else if (kind == "theta") rank = 1;
    else return false;
    iteration = std::stoi(stem.substr(0, sep));
    return true;
}

std::string write_checkpoint_file(const std::string& dir, int iteration, int which, int64_t rows, int f,
                                  uint64_t digest, const float* entries) {
    std::error_code ec;
    fs::create_directories(dir, ec);
    if (ec) fail_io("cannot create directory " + dir + ": " + ec.message());
    const std::string final_path = (fs::path(dir) / checkpoint_name(iteration, which)).string();
    const std::string tmp_path = final_path + ".tmp";
    {
        File out(tmp_path.c_str(), "wb");
        const uint64_t h[7] = {kCkptMagic, kVersion, static_cast<uint64_t>(iteration), static_cast<uint64_t>(which),
                               static_cast<uint64_t>(rows), static_cast<uint64_t>(f), digest};
        out.write(h, sizeof h);
        out.write(entries, sizeof(float) * static_cast<size_t>(rows) * static_cast<size_t>(f));
        if (std::fflush(out.f) != 0) fail_io("write failed for " + tmp_path);
    }
    fs::rename(tmp_path, final_path, ec);
    if (ec) fail_io("cannot rename " + tmp_path + " into place: " + ec.message());
    return final_path;
}

struct CkptHeader {
    int iteration, which;
    int64_t rows;
    int f;
    uint64_t digest;
};

CkptHeader read_checkpoint_header(File& in) {
    uint64_t v;
    in.read(&v, 8, "magic");
    if (v != kCkptMagic) fail_io(in.path + ": not a checkpoint (bad magic)");
    in.read(&v, 8, "version");
    if (v != kVersion) fail_io(in.path + ": unsupported checkpoint version");
    uint64_t it, which, rows, f, digest;
    in.read(&it, 8, "iteration");
    in.read(&which, 8, "which");
    if (which > 1) fail_io(in.path + ": corrupt checkpoint (bad factor kind)");
    in.read(&rows, 8, "rows");
    in.read(&f, 8, "f");
    in.read(&digest, 8, "digest");
    if (rows > (1ULL << 40) || f > (1ULL << 20)) fail_io(in.path + ": corrupt checkpoint header");
    std::error_code ec;
    const uintmax_t size = fs::file_size(in.path, ec);
    if (ec || size != 56 + rows * f * 4) fail_io(in.path + ": checkpoint size does not match its header");
    return CkptHeader{static_cast<int>(it), static_cast<int>(which), static_cast<int64_t>(rows), static_cast<int>(f),
                      digest};
}

// Newest checkpoint under dir: which = -1 ranks (iteration, theta > x) over both kinds
// (restore_latest, dataio.hpp:659-686), 0 / 1 only that kind (restore_latest_of,
// dataio.hpp:689-708). "" when none.
std::string latest_checkpoint(const std::string& dir, int which) {
    std::error_code ec;
    if (!fs::is_directory(dir, ec)) return "";
    int best_iter = -1, best_rank = -1;
    std::string best;
    for (const auto& entry : fs::directory_iterator(dir)) {
        if (!entry.is_regular_file()) continue;
        int iter = 0, rank = 0;
        if (!parse_checkpoint_name(entry.path().filename().string(), iter, rank)) continue;
        if (which >= 0 && rank != which) continue;
        if (iter > best_iter || (iter == best_iter && rank > best_rank)) {
            best_iter = iter;
            best_rank = rank;
            best = entry.path().string();
        }
    }
    return best;
}

class DeviceWriter {
  public:
    // host-only use (submit_host) touches no CUDA state, like the reference's pure-host
    // writer (dataio.hpp:565-651); the stream, events and pinned staging appear on the
    // first submit_device
    explicit DeviceWriter(std::string dir) : dir_(std::move(dir)) { worker_ = std::thread([this] { run(); }); }

    ~DeviceWriter() {
        {
            std::lock_guard<std::mutex> lock(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        worker_.join();  // drains a pending write
        release_buffer();
        if (dscratch_) cudaFree(dscratch_);
        if (copy_) {
            cudaEventDestroy(after_caller_);
            cudaEventDestroy(copied_);
            cudaStreamDestroy(copy_);
        }
    }

    // device factor (rows x f, row-major) ordered after `stream`; returns once the copy is
    // queued (and any previous write has finished)
    void submit_device(int iteration, int which, int64_t rows, int f, uint64_t digest, const float* d,
                       cudaStream_t stream) {
        submit(iteration, which, rows, f, digest, true, [&](float* dst, size_t bytes) {
            // value semantics at HBM speed: a device-to-device copy on the caller's stream
            // (the caller may overwrite the factor right after), then the slow D2H from
            // that copy on the private stream, overlapping the caller's next kernels
            if (bytes > dcap_) {
                if (dscratch_) ALSK_CUDA(cudaFree(dscratch_));
                dscratch_ = nullptr;
                dcap_ = 0;
                ALSK_CUDA(cudaMalloc(reinterpret_cast<void**>(&dscratch_), bytes));
                dcap_ = bytes;
            }
            if (bytes) ALSK_CUDA(cudaMemcpyAsync(dscratch_, d, bytes, cudaMemcpyDeviceToDevice, stream));
            ALSK_CUDA(cudaEventRecord(after_caller_, stream));
            ALSK_CUDA(cudaStreamWaitEvent(copy_, after_caller_, 0));
            if (bytes) ALSK_CUDA(cudaMemcpyAsync(dst, dscratch_, bytes, cudaMemcpyDeviceToHost, copy_));
        });
    }

    void submit_host(int iteration, int which, int64_t rows, int f, uint64_t digest, const float* h) {
        submit(iteration, which, rows, f, digest, false, [&](float* dst, size_t bytes) {
            if (bytes) std::memcpy(dst, h, bytes);
        });
    }

    void flush() {
        std::unique_lock<std::mutex> lock(mu_);
        cv_.wait(lock, [&] { return (!pending_ && !writing_) || error_; });
        rethrow_locked();
    }

  private:
    struct Job {
        int iteration, which;
        int64_t rows;
        int f;
        uint64_t digest;
        bool device;
    };

    template <class Fill>
    void submit(int iteration, int which, int64_t rows, int f, uint64_t digest, bool device, Fill&& fill) {
        if (which != 0 && which != 1) fail_input("factor kind must be 0 (x) or 1 (theta)");
        if (rows < 0 || f < 1) fail_input("invalid factor shape");
        std::unique_lock<std::mutex> lock(mu_);
        cv_.wait(lock, [&] { return (!pending_ && !writing_) || error_; });
        rethrow_locked();
        if (device && !copy_) {
            ALSK_CUDA(cudaGetDevice(&device_));
            ALSK_CUDA(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
            ALSK_CUDA(cudaEventCreateWithFlags(&after_caller_, cudaEventDisableTiming));
            ALSK_CUDA(cudaEventCreateWithFlags(&copied_, cudaEventDisableTiming));
        }
        const size_t bytes = sizeof(float) * static_cast<size_t>(rows) * static_cast<size_t>(f);
        // nothing is in flight: the buffer is free to replace (pinned once a device copy needs it)
        if (bytes > cap_ || (device && !is_pinned_)) {
            release_buffer();
            if (device) {
                ALSK_CUDA(cudaMallocHost(reinterpret_cast<void**>(&pinned_), std::max<size_t>(bytes, 1)));
            } else {
                pinned_ = static_cast<float*>(std::malloc(std::max<size_t>(bytes, 1)));
                if (!pinned_) throw std::bad_alloc();
            }
            is_pinned_ = device;
            cap_ = bytes;
        }
        fill(pinned_, bytes);
        if (device) ALSK_CUDA(cudaEventRecord(copied_, copy_));
        job_ = Job{iteration, which, rows, f, digest, device};
        pending_ = true;
        lock.unlock();
        cv_.notify_all();
    }

    void run() {
        bool bound = false;
        for (;;) {
            std::unique_lock<std::mutex> lock(mu_);
            cv_.wait(lock, [&] { return pending_ || stop_; });
            if (!pending_) return;
            const Job job = job_;
            pending_ = false;
            writing_ = true;
            lock.unlock();
            alsk_status st = ALSK_OK;
            std::string msg;
            try {
                if (job.device) {
                    if (!bound) ALSK_CUDA(cudaSetDevice(device_));
                    bound = true;
                    ALSK_CUDA(cudaEventSynchronize(copied_));
                }
                write_checkpoint_file(dir_, job.iteration, job.which, job.rows, job.f, job.digest, pinned_);
            } catch (const Failure& e) {
                st = e.status;
                msg = e.what();
            } catch (const std::exception& e) {
                st = ALSK_ERR_IO;
                msg = e.what();
            }
            lock.lock();
            if (st != ALSK_OK && !error_) {
                error_ = st;
                error_msg_ = msg;
            }
            writing_ = false;
            lock.unlock();
            cv_.notify_all();
        }
    }

    void release_buffer() {
        if (pinned_) {
            if (is_pinned_) cudaFreeHost(pinned_);
            else std::free(pinned_);
        }
        pinned_ = nullptr;
        cap_ = 0;
    }

    void rethrow_locked() {
        if (error_) throw Failure(error_, error_msg_);
    }

    std::string dir_;
    int device_ = 0;
    cudaStream_t copy_ = nullptr;
    cudaEvent_t after_caller_ = nullptr, copied_ = nullptr;
    float* pinned_ = nullptr;  // staging: page-locked after the first device submit
    bool is_pinned_ = false;
    size_t cap_ = 0;
    float* dscratch_ = nullptr;
    size_t dcap_ = 0;
    std::mutex mu_;
    std::condition_variable cv_;
    Job job_{};
    bool pending_ = false, writing_ = false, stop_ = false;
    alsk_status error_ = ALSK_OK;
    std::string error_msg_;
    std::thread worker_;  // started last
};

}  // namespace
}  // namespace alsk
