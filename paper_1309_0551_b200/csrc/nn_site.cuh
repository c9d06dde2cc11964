// The per-site NN operator shared by the sweep kernels (sweep.cu) and the fused
// peer-push boundary kernel (p2p.cu): one site's out(x), in the association of the
// composed reference oracle.
#pragma once

#include "sweep_common.cuh"
#include "su3_math.cuh"

namespace su3g {

// One site of the NN sweep: out(x) = sum_mu U_mu(x) v(x+mu) - sum_mu U_mu(x-mu)^dag v(x-mu), association of
// the composed reference (add_su3_vector chain, then sub_four_su3_vecs).  v_hi / w_lo: t-slab halos (or null).
// (non-volatile asm: the loads have no side effects, so the compiler may batch and hoist them)
// L2 eviction hints (HINTS): in the one-thread-per-site visiting orders every link is read
// twice -- first as a site's own forward link, last as the next site's backward link --
// so the backward gathers are marked evict-first (their line has no further use) and the
// output is stored streaming, leaving L2 to the lines that will be read again.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ float ld_hint(const float* p, uint64_t pol) {
    float r;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_hint(const double* p, uint64_t pol) {
    double r;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
template <typename T, int N>
__device__ __forceinline__ void ld_soa_last(const T* __restrict__ p, int64_t F, int64_t s3, T* r, uint64_t pol) {
#pragma unroll
    for (int k = 0; k < N; ++k) r[k] = ld_hint(p + k * F + s3, pol);
}

// Halo faces that a peer writes while the reading kernel is resident (p2p.cu): coherent
// system-scope loads, ordered after the CTA's acquire of the peer's flag by the CTA barrier --
// never the non-coherent (.nc / __ldg) path, which is only defined for data that stays
// read-only for the kernel's lifetime.
__device__ __forceinline__ float ld_coherent(const float* p) {
    float r;
    asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(r) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ double ld_coherent(const double* p) {
    double r;
    asm volatile("ld.relaxed.sys.global.f64 %0, [%1];" : "=d"(r) : "l"(p) : "memory");
    return r;
}
template <typename T, int N, bool COHERENT>
__device__ __forceinline__ void ld_halo(const T* p, int64_t F, int64_t s3, T* r) {
#pragma unroll
    for (int k = 0; k < N; ++k) r[k] = COHERENT ? ld_coherent(p + k * F + s3) : __ldg(p + k * F + s3);
}

// COHERENT_HALO: v_hi / w_lo are peer-written windows (see ld_coherent)
template <typename T, bool FUSED, bool HINTS = false, bool COHERENT_HALO = false>
__device__ __forceinline__ void nn_site(const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ out,
                                        const Geom& g, int x, int y, int z, int t, const T* v_hi,
                                        const T* w_lo) {
    const int64_t F = g.F;
    const uint64_t pol = HINTS ? l2_evict_first_policy() : 0;
    const int64_t s3 = x + int64_t(g.nx) * (y + int64_t(g.ny) * z);
    T acc[6];
    // forward terms, mu = 0..3, summed left to right (add_su3_vector chain)
#pragma unroll
    for (int mu = 0; mu < 4; ++mu) {
        T u[18], vn[6], f[6];
        ld_soa<T, 18>(U + (int64_t(t) * 72 + mu * 18) * F, F, s3, u);
        if (mu < 3) {
            ld_soa<T, 6>(v + int64_t(t) * 6 * F, F, step3(g, x, y, z, mu, +1), vn);
        } else if (t + 1 < g.nt) {
            ld_soa<T, 6>(v + int64_t(t + 1) * 6 * F, F, s3, vn);
        } else if (v_hi != nullptr) {
            ld_halo<T, 6, COHERENT_HALO>(v_hi, F, s3, vn);
        } else {
            ld_soa<T, 6>(v, F, s3, vn);
        }
        mv<T, FUSED>(u, vn, f);
#pragma unroll
        for (int k = 0; k < 6; ++k) acc[k] = (mu == 0) ? f[k] : xadd(acc[k], f[k]);
    }
    // backward terms, subtracted left to right (sub_four_su3_vecs)
#pragma unroll
    for (int mu = 0; mu < 4; ++mu) {
        T w[6];
        if (mu < 3) {
            T u[18], vn[6];
            const int64_t d = step3(g, x, y, z, mu, -1);
            if constexpr (HINTS) ld_soa_last<T, 18>(U + (int64_t(t) * 72 + mu * 18) * F, F, d, u, pol);
            else ld_soa<T, 18>(U + (int64_t(t) * 72 + mu * 18) * F, F, d, u);
            ld_soa<T, 6>(v + int64_t(t) * 6 * F, F, d, vn);
            amv<T, FUSED>(u, vn, w);
        } else if (t > 0 || w_lo == nullptr) {
            const int tp = (t > 0) ? t - 1 : g.nt - 1;
            T u[18], vn[6];
            if constexpr (HINTS) ld_soa_last<T, 18>(U + (int64_t(tp) * 72 + 3 * 18) * F, F, s3, u, pol);
            else ld_soa<T, 18>(U + (int64_t(tp) * 72 + 3 * 18) * F, F, s3, u);
            // v(x, t-1): its last reader in the visiting order is this backward t term
            if constexpr (HINTS) ld_soa_last<T, 6>(v + int64_t(tp) * 6 * F, F, s3, vn, pol);
            else ld_soa<T, 6>(v + int64_t(tp) * 6 * F, F, s3, vn);
            amv<T, FUSED>(u, vn, w);
        } else {
            ld_halo<T, 6, COHERENT_HALO>(w_lo, F, s3, w);
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) acc[k] = xsub(acc[k], w[k]);
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        if constexpr (HINTS) __stcs(out + (int64_t(t) * 6 + k) * F + s3, acc[k]);
        else out[(int64_t(t) * 6 + k) * F + s3] = acc[k];
    }
}

}  // namespace su3g
