// Shared device helpers for libsu3g (sm_100a).
//
//  * error reporting across the C ABI (thread-local message, int status codes)
//  * TMA bulk-copy / mbarrier PTX wrappers (cp.async.bulk -> SASS UBLKCP)
//  * "exact" IEEE arithmetic helpers: __fmul_rn / __fadd_rn never contract into
//    FMA, so a kernel written with them rounds exactly like the reference's
//    numpy arithmetic (su3bench scalar.py:8-14 association contract).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/su3g.h"

namespace su3g {

// ----------------------------------------------------------------------------
// errors
// ----------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail_invalid(const std::string& msg);      // returns SU3G_EINVAL
int check_launch(const char* what);            // cudaGetLastError -> status
void note_kernel(const std::string& name);     // su3g_last_kernel(): which kernel the last dispatch chose

// ----------------------------------------------------------------------------
// device properties (cached per device)
// ----------------------------------------------------------------------------
struct DeviceInfo {
    int device = -1;
    int num_sms = 0;
    int max_smem_optin = 0;
    int l2_bytes = 0;
};
const DeviceInfo& device_info();

// SMs left free by the persistent sweep kernels so that concurrently launched
// kernels (the NCCL halo exchange of a t-slab sweep) can be co-scheduled; set
// through su3g_set_option("sm_reserve", n).
int sm_reserve();
inline int sweep_sms() {
    const int n = device_info().num_sms - sm_reserve();
    return n > 0 ? n : 1;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ----------------------------------------------------------------------------
// exact (non-contracted) arithmetic
// ----------------------------------------------------------------------------
template <typename T> __device__ __forceinline__ T xmul(T a, T b);
template <typename T> __device__ __forceinline__ T xadd(T a, T b);
template <typename T> __device__ __forceinline__ T xsub(T a, T b);
template <> __device__ __forceinline__ float xmul<float>(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ float xadd<float>(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ float xsub<float>(float a, float b) { return __fsub_rn(a, b); }
template <> __device__ __forceinline__ double xmul<double>(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ double xadd<double>(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ double xsub<double>(double a, double b) { return __dsub_rn(a, b); }

// ----------------------------------------------------------------------------
// PTX: mbarrier + bulk async copies (TMA engine, non-tensor form)
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

// one non-blocking poll of a phase: lets a consumer test the NEXT operand's barrier before the
// current operand's arithmetic and only spin (mbar_wait) if that early test failed
__device__ __forceinline__ uint32_t mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return done;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_addr(bar);
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// global -> shared, completion counted on an mbarrier (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}

// global -> L2 only (no smem, no completion): warms L2 for a later reader (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src_gmem, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src_gmem), "r"(bytes) : "memory");
}

// shared -> global, bulk-group completion
__device__ __forceinline__ void bulk_s2g(void* dst_gmem, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_gmem), "r"(smem_addr(src_smem)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N> __device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
// make generic-proxy shared-memory writes visible to the async (bulk copy) proxy
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Shared-memory READS of a staging buffer (generic proxy) must be ordered before the TMA / bulk
// copy (async proxy) that refills it.  Where the hand-back is an mbarrier arrive (warp-specialised
// rings) every reading lane fences before the arrive: without it an LDS still queued at the arrive
// can observe the refill (seen on B200: k_nn_ring, 2 CTAs/SM, FMA mode).  Where it is a CTA
// barrier, the barrier completes the reads and the issuing thread fences before the refill.
#ifndef SU3G_RELEASE_FENCE
#define SU3G_RELEASE_FENCE 1
#endif
__device__ __forceinline__ void fence_before_refill() {
#if SU3G_RELEASE_FENCE
    fence_proxy_async_smem();
#endif
}

// ----------------------------------------------------------------------------
// vectorised register <-> memory moves of a per-site record of N reals
// (p must be aligned to the widest vector used: 16 B for f64 / f32 with N%4==0,
//  8 B for f32 with N%2==0)
// ----------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ void load_rec(const float* __restrict__ p, float (&r)[N]) {
    if constexpr (N % 4 == 0) {
#pragma unroll
        for (int k = 0; k < N / 4; ++k) {
            float4 q = reinterpret_cast<const float4*>(p)[k];
            r[4 * k] = q.x; r[4 * k + 1] = q.y; r[4 * k + 2] = q.z; r[4 * k + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < N / 2; ++k) {
            float2 q = reinterpret_cast<const float2*>(p)[k];
            r[2 * k] = q.x; r[2 * k + 1] = q.y;
        }
    }
}
template <int N>
__device__ __forceinline__ void load_rec(const double* __restrict__ p, double (&r)[N]) {
#pragma unroll
    for (int k = 0; k < N / 2; ++k) {
        double2 q = reinterpret_cast<const double2*>(p)[k];
        r[2 * k] = q.x; r[2 * k + 1] = q.y;
    }
}
template <int N>
__device__ __forceinline__ void store_rec(float* __restrict__ p, const float (&r)[N]) {
    if constexpr (N % 4 == 0) {
#pragma unroll
        for (int k = 0; k < N / 4; ++k)
            reinterpret_cast<float4*>(p)[k] = make_float4(r[4 * k], r[4 * k + 1], r[4 * k + 2], r[4 * k + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < N / 2; ++k) reinterpret_cast<float2*>(p)[k] = make_float2(r[2 * k], r[2 * k + 1]);
    }
}
template <int N>
__device__ __forceinline__ void store_rec(double* __restrict__ p, const double (&r)[N]) {
#pragma unroll
    for (int k = 0; k < N / 2; ++k) reinterpret_cast<double2*>(p)[k] = make_double2(r[2 * k], r[2 * k + 1]);
}

}  // namespace su3g
