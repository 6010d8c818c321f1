// Shared plumbing for libalskit_cuda.so: status/error propagation, device buffers,
// launch accounting. Error categories follow common.hpp:24-64 of the reference.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>

#include "alskit_cuda.h"

namespace alsk {

// Thrown inside the library, converted to alsk_status at the C boundary.
struct Failure : std::runtime_error {
    alsk_status status;
    Failure(alsk_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail_input(const std::string& m) { throw Failure(ALSK_ERR_INPUT, m); }
[[noreturn]] inline void fail_numerical(const std::string& m) { throw Failure(ALSK_ERR_NUMERICAL, m); }
[[noreturn]] inline void fail_capacity(const std::string& m) { throw Failure(ALSK_ERR_CAPACITY, m); }

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Failure(ALSK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define ALSK_CUDA(call) ::alsk::cuda_check((call), #call)

extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
// After every <<<>>> launch: count it and surface launch-configuration errors.
#define ALSK_LAUNCHED() do { ::alsk::count_launch(); ::alsk::cuda_check(cudaGetLastError(), "kernel launch"); } while (0)

void set_breakdown_index(int64_t k);
void set_last_error(const char* msg);

// Run fn, converting library exceptions to an alsk_status plus the thread's last-error text
// (the C boundary of every entry point).
template <class Fn>
alsk_status guard(Fn&& fn) {
    set_last_error("");
    set_breakdown_index(-1);
    try {
        fn();
        return ALSK_OK;
    } catch (const Failure& e) {
        set_last_error(e.what());
        return e.status;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return ALSK_ERR_CAPACITY;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return ALSK_ERR_CUDA;
    }
}

// Kernel-phase timing for the bench (alsk_profile_begin / alsk_profile_phases): when on,
// launches are bracketed by CUDA events on their stream and accumulated per phase.
enum ProfPhase { PHASE_HERMITIAN = 0, PHASE_SOLVE = 1, PHASE_FUSED = 2, PHASE_COLLECTIVE = 3, PHASE_COUNT = 4 };
bool prof_on();
void prof_add(int phase, float ms);
// The pair of events is handed to the profile when the timer closes and resolved only when
// the profile is read (alsk_profile_phases), so timing adds no host synchronisation.
void prof_defer(int phase, cudaEvent_t e0, cudaEvent_t e1);
class PhaseTimer {  // no-op unless profiling is on
public:
    PhaseTimer(int phase, cudaStream_t s) : phase_(phase), s_(s) {
        if (!prof_on()) return;
        cudaEventCreate(&e0_);
        cudaEventCreate(&e1_);
        cudaEventRecord(e0_, s_);
    }
    ~PhaseTimer() {
        if (!e0_) return;
        cudaEventRecord(e1_, s_);
        prof_defer(phase_, e0_, e1_);
    }
private:
    int phase_;
    cudaStream_t s_;
    cudaEvent_t e0_ = nullptr, e1_ = nullptr;
};

// Keep freed stream-ordered memory in the device pool instead of returning it to the
// driver at every synchronisation (the default threshold of 0 made per-call scratch
// allocations re-map physical memory and stall for hundreds of milliseconds).
inline void retain_pool_memory() {
    static bool done = false;
    if (done) return;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done = true;
}

// Owning device allocation (cudaMallocAsync on the given stream when available).
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(size_t bytes, cudaStream_t s = nullptr) { alloc(bytes, s); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_), s_(o.s_) { o.p_ = nullptr; o.n_ = 0; }
    ~DevBuf() { reset(); }
    void alloc(size_t bytes, cudaStream_t s = nullptr) {
        reset();
        s_ = s;
        n_ = bytes;
        retain_pool_memory();
        if (bytes) ALSK_CUDA(cudaMallocAsync(&p_, bytes, s));
    }
    void reset() {
        if (p_) cudaFreeAsync(p_, s_);
        p_ = nullptr;
        n_ = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(p_); }
    size_t bytes() const { return n_; }

private:
    void* p_ = nullptr;
    size_t n_ = 0;
    cudaStream_t s_ = nullptr;
};

template <class T>
inline void h2d(T* dst, const T* src, size_t count, cudaStream_t s) {
    if (count) ALSK_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
}
template <class T>
inline void d2h(T* dst, const T* src, size_t count, cudaStream_t s) {
    if (count) ALSK_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, s));
}

inline int num_sms() {
    static int sms = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v > 0 ? v : 148;
    }();
    return sms;
}

inline void require_device() {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        throw Failure(ALSK_ERR_CUDA, "no CUDA device available (libalskit_cuda has no CPU fallback)");
}

}  // namespace alsk
