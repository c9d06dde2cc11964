// Link-product sweep, low-register form (link_variant 6; BASELINE configs[3]).
//
// The one-thread-per-site kernel (sweep.cu k_link_product) holds A, B, the
// intermediate T = A B and the accumulator in registers: 232-254 registers for
// f64, so only 8 warps fit an SM and the dependent link gathers are exposed
// (ncu: FP64 pipe 29% busy, 12% warps active).  Here
//   * the accumulator lives in shared memory (18 reals per site, column-major
//     over the CTA's sites, conflict-free);
//   * T = A B is built one row at a time from a row of A (t_i = a_i B), so A is
//     never whole in registers;
//   * C = U_mu(x+nu) is gathered after T is complete, so B and C are never live
//     together;
// which caps the live set at ~3 matrices and lets __launch_bounds__(128, MINB)
// fit 16 warps/SM for f64.  Arithmetic per element is exactly link_site's --
// mat_nn, then mat_na, then acc + s*P in plane order -- row by row, so EXACT
// mode is bit-identical to the reference composition.
#include <algorithm>

#include "nn_site.cuh"

namespace su3g {

namespace {

__constant__ int c_plane_mu[6] = {0, 0, 0, 1, 1, 2};
__constant__ int c_plane_nu[6] = {1, 2, 3, 2, 3, 3};

__device__ __forceinline__ int64_t shifted(const Geom& g, int x, int y, int z, int t, int mu) {
    if (mu == 0) x = (x + 1 == g.nx) ? 0 : x + 1;
    else if (mu == 1) y = (y + 1 == g.ny) ? 0 : y + 1;
    else if (mu == 2) z = (z + 1 == g.nz) ? 0 : z + 1;
    else t = (t + 1 == g.nt) ? 0 : t + 1;
    return int64_t(t) * g.F + x + int64_t(g.nx) * (y + int64_t(g.ny) * z);
}

// N consecutive components of link mu at a site: U[(t*72 + mu*18 + c0 + k) * F + s3]
template <typename T, int N>
__device__ __forceinline__ void ld_link_part(const T* __restrict__ U, const Geom& g, int64_t site, int mu, int c0,
                                             T* r) {
    const int64_t t = site / g.F, s3 = site - t * g.F;
    ld_soa<T, N>(U + (t * 72 + mu * 18 + c0) * g.F, g.F, s3, r);
}

// L1 eviction priorities for the L1HINT kernels: A (re-read in up to three planes) evict-last,
// the single-use B/C gathers no-allocate
__device__ __forceinline__ double ld_l1(const double* p, int keep) {
    double r;
    if (keep) asm("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(r) : "l"(p));
    else asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ float ld_l1(const float* p, int keep) {
    float r;
    if (keep) asm("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(r) : "l"(p));
    else asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
}
template <typename T, int N>
__device__ __forceinline__ void ld_part_l1(const T* __restrict__ U, const Geom& g, int64_t site, int mu, int c0, T* r,
                                           int keep) {
    const int64_t t = site / g.F, s3 = site - t * g.F;
    const T* p = U + (t * 72 + mu * 18 + c0) * g.F + s3;
#pragma unroll
    for (int k = 0; k < N; ++k) r[k] = ld_l1(p + k * g.F, keep);
}

template <typename T, bool FUSED, int MODE, class PF, class QF>
__device__ __forceinline__ void dot3(PF p, QF q, T& re, T& im) {
    if constexpr (FUSED) cdot_fma<T, MODE, 3>(p, q, re, im);
    else cdot<T, MODE, 3>(p, q, re, im);
}

}  // namespace

template <typename T, bool FUSED, int MINB, bool EARLY_C, bool PREF_B, bool HINTS = false, bool L1HINT = false>
__global__ void __launch_bounds__(128, MINB)
    k_link_rows(const T* __restrict__ U, T* __restrict__ acc_out, Geom g, T s, int ZC, int ahead) {
    // HINTS: in the (z-chunk, t, z, y, x) order a link's last reader is: U_mu(y), mu < 3, its own site's
    // A in the last plane of the mu group (planes 2, 4, 5); U_t(y) the B of plane (0,3) at y - x.
    // Those gathers are marked L2 evict-first and the result is stored streaming.
    const uint64_t pol = HINTS ? l2_evict_first_policy() : 0;
    if (ahead > 0 && threadIdx.x == 0)  // L2 prefetch of the CTA one wave ahead (sweep_prefetch)
        prefetch_cta_l2<T>(U, 72, g, blockIdx.x + int64_t(ahead), blockDim.x, 0, g.nt, ZC);
    __shared__ T sacc[18 * 128];
    const int tid = threadIdx.x;
    const int64_t idx = blockIdx.x * int64_t(blockDim.x) + tid;
    if (idx >= g.F * g.nt) return;  // no block-level sync below: early exit is safe
    // (z-chunk, t, z, y, x) visiting order, as k_link_product
    const int x = static_cast<int>(idx % g.nx);
    int64_t r = idx / g.nx;
    const int y = static_cast<int>(r % g.ny);
    r /= g.ny;
    const int zl = static_cast<int>(r % ZC);
    r /= ZC;
    const int t = static_cast<int>(r % g.nt);
    const int z = static_cast<int>(r / g.nt) * ZC + zl;
    const int64_t s3 = x + int64_t(g.nx) * (y + int64_t(g.ny) * z);
    const int64_t site = int64_t(t) * g.F + s3;
    T* acc = sacc + tid;  // element k at acc[k * 128]
    // PREF_B: B of plane p+1 is gathered during plane p's C phase (one more matrix in flight)
    T bn[PREF_B ? 18 : 1];
    if constexpr (PREF_B) ld_link_part<T, 18>(U, g, shifted(g, x, y, z, t, c_plane_mu[0]), c_plane_nu[0], 0, bn);

#pragma unroll 1
    for (int pl = 0; pl < 6; ++pl) {
        const int mu = c_plane_mu[pl], nu = c_plane_nu[pl];
        T tm[18], c[18];
        // EARLY_C: gather C with B (both in flight together, +18 live reals); else after T is built
        if constexpr (EARLY_C) ld_link_part<T, 18>(U, g, shifted(g, x, y, z, t, nu), mu, 0, c);
        {
            T b[18];
            if constexpr (PREF_B) {
#pragma unroll
                for (int k = 0; k < 18; ++k) b[k] = bn[k];
            } else {
                if (HINTS && pl == 2) {
                    const int64_t nb = shifted(g, x, y, z, t, mu), tn = nb / g.F;
                    ld_soa_last<T, 18>(U + (tn * 72 + nu * 18) * g.F, g.F, nb - tn * g.F, b, pol);
                } else if (L1HINT) {
                    ld_part_l1<T, 18>(U, g, shifted(g, x, y, z, t, mu), nu, 0, b, 0);
                } else {
                    ld_link_part<T, 18>(U, g, shifted(g, x, y, z, t, mu), nu, 0, b);  // B = U_nu(x + mu)
                }
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                T a[6];
                if (HINTS && (pl == 2 || pl == 4 || pl == 5))
                    ld_soa_last<T, 6>(U + (int64_t(t) * 72 + mu * 18 + 6 * i) * g.F, g.F, s3, a, pol);
                else if (L1HINT)
                    ld_part_l1<T, 6>(U, g, site, mu, 6 * i, a, 1);
                else
                    ld_link_part<T, 6>(U, g, site, mu, 6 * i, a);  // row i of A = U_mu(x)
#pragma unroll
                for (int k = 0; k < 3; ++k)  // t[i][k] = sum_j a[i][j] b[j][k]   (mat_nn)
                    dot3<T, FUSED, PLAIN>([&](int j, int q) { return a[2 * j + q]; },
                                          [&](int j, int q) { return b[(3 * j + k) * 2 + q]; }, tm[(3 * i + k) * 2],
                                          tm[(3 * i + k) * 2 + 1]);
            }
        }
        if constexpr (PREF_B) {
            if (pl < 5)
                ld_link_part<T, 18>(U, g, shifted(g, x, y, z, t, c_plane_mu[pl + 1]), c_plane_nu[pl + 1], 0, bn);
        }
        if constexpr (!EARLY_C) {
            if constexpr (L1HINT) ld_part_l1<T, 18>(U, g, shifted(g, x, y, z, t, nu), mu, 0, c, 0);
            else ld_link_part<T, 18>(U, g, shifted(g, x, y, z, t, nu), mu, 0, c);  // C = U_mu(x + nu)
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) {  // p[i][k] = sum_j t[i][j] conj(c[k][j])   (mat_na)
                T pr, pi;
                dot3<T, FUSED, CONJ_Q>([&](int j, int q) { return tm[(3 * i + j) * 2 + q]; },
                                       [&](int j, int q) { return c[(3 * k + j) * 2 + q]; }, pr, pi);
                const int e = (3 * i + k) * 2;
                if (pl == 0) {  // acc = 0 + s*p, as the reference's zero-initialised accumulation
                    acc[e * 128] = FUSED ? fma(s, pr, T(0)) : xadd(T(0), xmul(s, pr));
                    acc[(e + 1) * 128] = FUSED ? fma(s, pi, T(0)) : xadd(T(0), xmul(s, pi));
                } else {
                    acc[e * 128] = FUSED ? fma(s, pr, acc[e * 128]) : xadd(acc[e * 128], xmul(s, pr));
                    acc[(e + 1) * 128] = FUSED ? fma(s, pi, acc[(e + 1) * 128]) : xadd(acc[(e + 1) * 128], xmul(s, pi));
                }
            }
    }
#pragma unroll
    for (int k = 0; k < 18; ++k) {
        if constexpr (HINTS) __stcs(acc_out + (int64_t(t) * 18 + k) * g.F + s3, acc[k * 128]);
        else acc_out[(int64_t(t) * 18 + k) * g.F + s3] = acc[k * 128];
    }
}

// Three lanes per site (link_variant 9).  Lane (site, r) of a warp builds row r of T = A B and of
// P = T C^dag for the six planes and accumulates row r of the result; ten sites per warp (lanes 30,
// 31 idle).  The three lanes of a site gather the same B/C elements in one request (ten distinct
// addresses), so a warp-wide gather costs one L1 wavefront for ten sites where the one-thread-per-site
// kernel spends two (f64) for 32; in exchange the live set is a row instead of matrices (~70 registers,
// 28 warps/SM instead of 16), so twice the gathers are in flight.  Row r of each product uses the
// per-element arithmetic of mult_su3_nn / mult_su3_na (scalar.py:77-104) and the plane order of the
// reference composition: EXACT mode is bit-identical.
template <typename T, bool FUSED, int MINB>
__global__ void __launch_bounds__(128, MINB)
    k_link_rows3(const T* __restrict__ U, T* __restrict__ acc_out, Geom g, T s, int ZC) {
    const int lane = threadIdx.x & 31;
    if (lane >= 30) return;  // no block-level synchronisation below
    const int sl = lane / 3, r = lane - 3 * sl;
    const int64_t idx = (int64_t(blockIdx.x) * 4 + (threadIdx.x >> 5)) * 10 + sl;
    if (idx >= g.F * g.nt) return;
    // (z-chunk, t, z, y, x) visiting order, as k_link_rows
    const int x = static_cast<int>(idx % g.nx);
    int64_t q = idx / g.nx;
    const int y = static_cast<int>(q % g.ny);
    q /= g.ny;
    const int zl = static_cast<int>(q % ZC);
    q /= ZC;
    const int t = static_cast<int>(q % g.nt);
    const int z = static_cast<int>(q / g.nt) * ZC + zl;
    const int64_t s3 = x + int64_t(g.nx) * (y + int64_t(g.ny) * z);
    const int64_t F = g.F;

    T acc[6], a[6];
#pragma unroll 1
    for (int pl = 0; pl < 6; ++pl) {
        const int mu = c_plane_mu[pl], nu = c_plane_nu[pl];
        if (pl == 0 || pl == 3 || pl == 5)  // row r of A = U_mu(x), kept for the planes of one mu
            ld_soa<T, 6>(U + (int64_t(t) * 72 + mu * 18 + 6 * r) * F, F, s3, a);
        T tr[6];
        {
            const int64_t nb = shifted(g, x, y, z, t, mu), tn = nb / F;
            const T* B = U + (tn * 72 + nu * 18) * F + (nb - tn * F);  // U_nu(x + mu)
            T b[18];
#pragma unroll
            for (int e = 0; e < 18; ++e) b[e] = __ldg(B + e * F);
#pragma unroll
            for (int k = 0; k < 3; ++k) {  // t[r][k] = sum_j a[r][j] b[j][k]   (mat_nn)
                auto pa = [&](int j, int c) { return a[2 * j + c]; };
                auto pb = [&](int j, int c) { return b[(3 * j + k) * 2 + c]; };
                if constexpr (FUSED) cdot_fma<T, PLAIN, 3>(pa, pb, tr[2 * k], tr[2 * k + 1]);
                else cdot<T, PLAIN, 3>(pa, pb, tr[2 * k], tr[2 * k + 1]);
            }
        }
        const int64_t nc = shifted(g, x, y, z, t, nu), tc = nc / F;
        const T* C = U + (tc * 72 + mu * 18) * F + (nc - tc * F);  // U_mu(x + nu)
        T c[18];
#pragma unroll
        for (int e = 0; e < 18; ++e) c[e] = __ldg(C + e * F);
#pragma unroll
        for (int k = 0; k < 3; ++k) {  // p[r][k] = sum_j t[r][j] conj(c[k][j])   (mat_na)
            T pr, pi;
            auto pt = [&](int j, int cc) { return tr[2 * j + cc]; };
            auto pc = [&](int j, int cc) { return c[(3 * k + j) * 2 + cc]; };
            if constexpr (FUSED) cdot_fma<T, CONJ_Q, 3>(pt, pc, pr, pi);
            else cdot<T, CONJ_Q, 3>(pt, pc, pr, pi);
            if (pl == 0) {  // acc = 0 + s*p, as the reference's zero-initialised accumulation
                acc[2 * k] = FUSED ? fma(s, pr, T(0)) : xadd(T(0), xmul(s, pr));
                acc[2 * k + 1] = FUSED ? fma(s, pi, T(0)) : xadd(T(0), xmul(s, pi));
            } else {
                acc[2 * k] = FUSED ? fma(s, pr, acc[2 * k]) : xadd(acc[2 * k], xmul(s, pr));
                acc[2 * k + 1] = FUSED ? fma(s, pi, acc[2 * k + 1]) : xadd(acc[2 * k + 1], xmul(s, pi));
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 6; ++e) __stcs(acc_out + (int64_t(t) * 18 + 6 * r + e) * F + s3, acc[e]);
}

int g_link_rows3_minb = 0;  // su3g_set_option("link_rows3_minb"): CTAs/SM the register budget of variant 9 targets

template <typename T, bool FUSED>
int launch_link_rows3(const T* U, T* acc, const Geom& g, T s, int ZC, cudaStream_t st) {
    const int64_t n = g.F * g.nt;
    const unsigned grid = static_cast<unsigned>((n + 39) / 40);  // 4 warps x 10 sites per CTA
    // registers (ptxas): f64 exact 80 at 6 CTAs/SM (8 spills), f64 FMA 94 at 5 (6 spills), f32 64 at 8
    const int minb = g_link_rows3_minb ? g_link_rows3_minb : (sizeof(T) == 4 ? 8 : (FUSED ? 5 : 6));
    switch (minb) {
        case 4: k_link_rows3<T, FUSED, 4><<<grid, 128, 0, st>>>(U, acc, g, s, ZC); break;
        case 5: k_link_rows3<T, FUSED, 5><<<grid, 128, 0, st>>>(U, acc, g, s, ZC); break;
        case 8: k_link_rows3<T, FUSED, 8><<<grid, 128, 0, st>>>(U, acc, g, s, ZC); break;
        default: k_link_rows3<T, FUSED, 6><<<grid, 128, 0, st>>>(U, acc, g, s, ZC); break;
    }
    return check_launch("link_product(rows3)");
}

template int launch_link_rows3<float, false>(const float*, float*, const Geom&, float, int, cudaStream_t);
template int launch_link_rows3<float, true>(const float*, float*, const Geom&, float, int, cudaStream_t);
template int launch_link_rows3<double, false>(const double*, double*, const Geom&, double, int, cudaStream_t);
template int launch_link_rows3<double, true>(const double*, double*, const Geom&, double, int, cudaStream_t);

int g_link_minb = 0;     // su3g_set_option("link_minb"): CTAs/SM the register budget targets (0 = default)
int g_link_early_c = -1;  // su3g_set_option("link_early_c"): gather C together with B (-1 = default)
int g_link_hints = 0;
int g_link_l1_hints = 0;  // su3g_set_option("link_l1_hints"): A evict-last in L1, B/C no-allocate (A/B)     // su3g_set_option("link_l2_hints"): last-use gathers evict-first (A/B)
int g_link_pref_b = 0;    // su3g_set_option("link_prefetch_b"): gather the next plane's B during this plane
extern int g_sweep_prefetch;

template <typename T, bool FUSED, bool EARLY_C, bool PREF_B>
static void launch_rows_minb(const T* U, T* acc, const Geom& g, T s, int ZC, unsigned grid, int minb, int ahead,
                             cudaStream_t st) {
    switch (minb) {
        case 3: k_link_rows<T, FUSED, 3, EARLY_C, PREF_B><<<grid, 128, 0, st>>>(U, acc, g, s, ZC, ahead); break;
        case 5: k_link_rows<T, FUSED, 5, EARLY_C, PREF_B><<<grid, 128, 0, st>>>(U, acc, g, s, ZC, ahead); break;
        case 6: k_link_rows<T, FUSED, 6, EARLY_C, PREF_B><<<grid, 128, 0, st>>>(U, acc, g, s, ZC, ahead); break;
        case 8: k_link_rows<T, FUSED, 8, EARLY_C, PREF_B><<<grid, 128, 0, st>>>(U, acc, g, s, ZC, ahead); break;
        default: k_link_rows<T, FUSED, 4, EARLY_C, PREF_B><<<grid, 128, 0, st>>>(U, acc, g, s, ZC, ahead); break;
    }
}

template <typename T, bool FUSED>
int launch_link_rows(const T* U, T* acc, const Geom& g, T s, int ZC, cudaStream_t st) {
    const int64_t n = g.F * g.nt;
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    // defaults from the 48^4 sweep on B200 (fraction of HBM): f64 exact minb 4 (0.427; 3 with early C 0.429),
    // f64 FMA minb 3 (0.474 vs 0.467 at 4), f32 minb 6 with early C (0.310 vs 0.299)
    const int minb = g_link_minb ? g_link_minb : (sizeof(T) == 8 ? (FUSED ? 3 : 4) : 6);
    const bool early_c = g_link_early_c >= 0 ? g_link_early_c != 0 : sizeof(T) == 4;
    // L2 prefetch one wave ahead (sweep_prefetch): resident CTAs per SM from the register target
    const int ahead = (g_sweep_prefetch > 0 && (int64_t(g.nx) * g.ny) % 128 == 0 && aligned16(U))
                          ? std::max(1, minb * device_info().num_sms * g_sweep_prefetch / 4)
                          : 0;
    if (g_link_l1_hints && !g_link_pref_b) {
        constexpr int MB = sizeof(T) == 8 ? (FUSED ? 3 : 4) : 6;
        if (early_c) k_link_rows<T, FUSED, MB, true, false, false, true><<<grid, 128, 0, st>>>(U, acc, g, s, ZC, ahead);
        else k_link_rows<T, FUSED, MB, false, false, false, true><<<grid, 128, 0, st>>>(U, acc, g, s, ZC, ahead);
    } else if (g_link_hints && !g_link_pref_b) {
        if (early_c) k_link_rows<T, FUSED, sizeof(T) == 8 ? (FUSED ? 3 : 4) : 6, true, false, true>
                         <<<grid, 128, 0, st>>>(U, acc, g, s, ZC, ahead);
        else k_link_rows<T, FUSED, sizeof(T) == 8 ? (FUSED ? 3 : 4) : 6, false, false, true>
                 <<<grid, 128, 0, st>>>(U, acc, g, s, ZC, ahead);
    } else if (g_link_pref_b) {
        if (early_c) launch_rows_minb<T, FUSED, true, true>(U, acc, g, s, ZC, grid, minb, ahead, st);
        else launch_rows_minb<T, FUSED, false, true>(U, acc, g, s, ZC, grid, minb, ahead, st);
    } else {
        if (early_c) launch_rows_minb<T, FUSED, true, false>(U, acc, g, s, ZC, grid, minb, ahead, st);
        else launch_rows_minb<T, FUSED, false, false>(U, acc, g, s, ZC, grid, minb, ahead, st);
    }
    return check_launch("link_product(rows)");
}

template int launch_link_rows<float, false>(const float*, float*, const Geom&, float, int, cudaStream_t);
template int launch_link_rows<float, true>(const float*, float*, const Geom&, float, int, cudaStream_t);
template int launch_link_rows<double, false>(const double*, double*, const Geom&, double, int, cudaStream_t);
template int launch_link_rows<double, true>(const double*, double*, const Geom&, double, int, cudaStream_t);

}  // namespace su3g
