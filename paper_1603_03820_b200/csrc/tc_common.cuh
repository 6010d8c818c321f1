// sm_100a primitives for the tensor-core Hermitian: mbarriers, TMEM allocation, tcgen05.mma
// (kind::tf32) with shared-memory matrix descriptors, tcgen05.ld, named barriers.
//
// Layouts (SWIZZLE_128B: inside every 1024-byte atom of 8 rows x 128 bytes, the 16-byte
// chunk c of row r sits at chunk position c ^ r; TMA applies the same XOR from the
// shared-memory address bits, so atoms must be 1024-byte aligned):
//  * rating-major staging (what tile::gather4 lands): atom = 8 ratings x 32 features.
//  * K-major MMA operands (what tcgen05.mma kind::tf32 reads): atom = 8 features x 32
//    ratings (K contiguous); 8-feature groups are SBO = 1024 bytes apart, and a K=8 step
//    advances the descriptor start by 32 bytes inside the atom.
// (MN-major tf32 operands were probed on this B200 and are not executed by the tensor core:
//  scripts/probes/mma_tf32_probe.cu.)
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace alsk {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarriers ----
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// Wait for the phase with the given parity (spinning try_wait: a suspend-time hint parks
// the warp and the wake-up then costs microseconds, which short per-step waits cannot
// afford). A deadlock traps after ~10 s of SM clock instead of hanging the device.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    uint32_t spins = 0;
    long long t0 = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (!done && ((++spins & 255u) == 0)) {
            const long long now = clock64();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 20000000000ll) __trap();
        }
    } while (!done);
}
// The same wait with a nanosleep back-off between probes: for long or latency-tolerant
// waits, so the waiting warp does not take issue slots from the warps doing the work.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
    uint32_t done = 0;
    long long t0 = 0;
    for (uint32_t it = 1;; ++it) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) return;
        __nanosleep(ns);
        if ((it & 63u) == 0) {
            const long long now = clock64();
            if (t0 == 0) t0 = now;
            else if (now - t0 > 20000000000ll) __trap();
        }
    }
}
// The same wait with a suspend-time hint: a waiting thread is parked in try_wait until the
// phase completes (or the hint expires), so the wait costs a handful of instructions.
__device__ __forceinline__ void mbar_wait_park(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    uint32_t rounds = 0;
    for (;;) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity), "r"(1000000u)
            : "memory");
        if (done) return;
        if (++rounds > 20000u) __trap();  // > 20 s parked: deadlock
    }
}
// Generic-proxy shared-memory writes -> visible to the async proxy (tensor core operands).
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void named_barrier(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}

// ---- TMEM ----
template <uint32_t COLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(dst)),
                 "n"(COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
template <uint32_t COLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(COLS) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// ---- descriptors ----
// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bits.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;  // descriptor version (Blackwell)
    d |= 2ull << 61;  // SWIZZLE_128B
    return d;
}
// Instruction descriptor: D f32, A/B tf32, both K-major, shape MxN.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
           (static_cast<uint32_t>(M >> 4) << 24);
}
// D[tmem] (+)= A[smem] * B[smem]; issued by one thread.
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive on `bar` once every tcgen05.mma previously issued by this thread has completed.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
// 32 lanes x 16 consecutive 32-bit columns: thread t of the warp gets lane (base lane + t).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// ---- TF32 split ----
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// Rating-major staging: byte offset of (rating k, 16-byte feature chunk c16) in a stage of
// MNB feature blocks (k-group stride MNB*1024, feature-block stride 1024).
template <int MNB>
__device__ __forceinline__ uint32_t sw128_offset(int k, int c16) {
    return static_cast<uint32_t>((k >> 3) * (MNB * 1024) + (c16 >> 3) * 1024 + (k & 7) * 128 +
                                 (((c16 & 7) ^ (k & 7)) << 4));
}
// K-major operand tile of 32 ratings: byte offset of (feature i, rating k).
__device__ __forceinline__ uint32_t kmajor_offset(int i, int k) {
    return static_cast<uint32_t>((i >> 3) * 1024 + (i & 7) * 128 + ((((k >> 2) ^ (i & 7))) << 4) + (k & 3) * 4);
}

// 16-byte global -> shared copy through L2 only (LDGSTS).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
// The same copy allocating in L1 (the other 16-byte half of a 32-byte sector, copied by the
// next loader warp, then hits L1 instead of requesting the sector from L2 again).
__device__ __forceinline__ void cp_async16_ca(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
// Arrive on `bar` once all cp.async issued so far by this thread have landed; the arrival
// counts against the barrier's expected count.
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ float4 ldg_nc_f4(const float* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(p));
    return v;
}

}  // namespace tc
}  // namespace alsk
