// Link-product sweep, low-register form (BASELINE configs[3]).
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

// The links of the site one step along +mu: base pointer of its t-slice's 72 planes and its in-slice
// offset (no 64-bit division: the r01 kernel derived (t, s3) from a flat site index with one per load)
struct LinkSite {
    const void* slice;  // U + t*72*F
    int64_t s3;
};

template <typename T>
__device__ __forceinline__ LinkSite link_site_at(const T* __restrict__ U, const Geom& g, int x, int y, int z, int t,
                                                 int mu) {
    if (mu == 0) x = (x + 1 == g.nx) ? 0 : x + 1;
    else if (mu == 1) y = (y + 1 == g.ny) ? 0 : y + 1;
    else if (mu == 2) z = (z + 1 == g.nz) ? 0 : z + 1;
    else if (mu == 3) t = (t + 1 == g.nt) ? 0 : t + 1;  // mu == 4: the site itself
    return {U + int64_t(t) * 72 * g.F, x + int64_t(g.nx) * (y + int64_t(g.ny) * z)};
}

// N consecutive components of link mu at a site: slice[(mu*18 + c0 + k) * F + s3]
template <typename T, int N>
__device__ __forceinline__ void ld_link_part(const LinkSite& st, int64_t F, int mu, int c0, T* r) {
    ld_soa<T, N>(static_cast<const T*>(st.slice) + (mu * 18 + c0) * F, F, st.s3, r);
}

template <typename T, bool FUSED, int MODE, class PF, class QF>
__device__ __forceinline__ void dot3(PF p, QF q, T& re, T& im) {
    if constexpr (FUSED) cdot_fma<T, MODE, 3>(p, q, re, im);
    else cdot<T, MODE, 3>(p, q, re, im);
}

}  // namespace

template <typename T, bool FUSED, int MINB, bool EARLY_C>
__global__ void __launch_bounds__(128, MINB)
    k_link_rows(const T* __restrict__ U, T* __restrict__ acc_out, Geom g, T s, int ZC) {
    __shared__ T sacc[18 * 128];
    const int tid = threadIdx.x;
    const int64_t idx = blockIdx.x * int64_t(blockDim.x) + tid;
    if (idx >= g.F * g.nt) return;  // no block-level sync below: early exit is safe
    // (z-chunk, t, z, y, x) visiting order: the +t links a site gathers as neighbours are re-read
    // as own links ZC*nx*ny sites later (a few MB of traffic), so they stay in L2
    const int x = static_cast<int>(idx % g.nx);
    int64_t r = idx / g.nx;
    const int y = static_cast<int>(r % g.ny);
    r /= g.ny;
    const int zl = static_cast<int>(r % ZC);
    r /= ZC;
    const int t = static_cast<int>(r % g.nt);
    const int z = static_cast<int>(r / g.nt) * ZC + zl;
    const int64_t s3 = x + int64_t(g.nx) * (y + int64_t(g.ny) * z);
    const LinkSite own = link_site_at(U, g, x, y, z, t, 4);
    T* acc = sacc + tid;  // element k at acc[k * 128]

#pragma unroll 1
    for (int pl = 0; pl < 6; ++pl) {
        const int mu = c_plane_mu[pl], nu = c_plane_nu[pl];
        T tm[18], c[18];
        // EARLY_C: gather C with B (both in flight together, +18 live reals); else after T is built
        if constexpr (EARLY_C) ld_link_part<T, 18>(link_site_at(U, g, x, y, z, t, nu), g.F, mu, 0, c);
        {
            T b[18];
            ld_link_part<T, 18>(link_site_at(U, g, x, y, z, t, mu), g.F, nu, 0, b);  // B = U_nu(x + mu)
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                T a[6];
                ld_link_part<T, 6>(own, g.F, mu, 6 * i, a);  // row i of A = U_mu(x)
#pragma unroll
                for (int k = 0; k < 3; ++k)  // t[i][k] = sum_j a[i][j] b[j][k]   (mat_nn)
                    dot3<T, FUSED, PLAIN>([&](int j, int q) { return a[2 * j + q]; },
                                          [&](int j, int q) { return b[(3 * j + k) * 2 + q]; }, tm[(3 * i + k) * 2],
                                          tm[(3 * i + k) * 2 + 1]);
            }
        }
        if constexpr (!EARLY_C) ld_link_part<T, 18>(link_site_at(U, g, x, y, z, t, nu), g.F, mu, 0, c);  // C = U_mu(x + nu)
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
    for (int k = 0; k < 18; ++k) __stcs(acc_out + (int64_t(t) * 18 + k) * g.F + s3, acc[k * 128]);
}

template <typename T, bool FUSED>
int launch_link_rows(const T* U, T* acc, const Geom& g, T s, int ZC, cudaStream_t st) {
    const int64_t n = g.F * g.nt;
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    // register budget and gather order from the 48^4 sweep on B200 (fraction of HBM): f64 exact
    // 4 CTAs/SM (0.427), f64 FMA 3 (0.474 vs 0.467 at 4), f32 6 with C gathered early (0.310 vs 0.299).
    // r02: dropping the per-load 64-bit site division took f64 exact 0.450 -> 0.497 (same box); a fully
    // unrolled plane loop (compile-time mu, nu) measured 0.362 (loads hoisted across planes), 5 / 6 CTAs
    // per SM (96 / 80 registers, spills) 0.430 / 0.379 against 0.480 at 4 (profiles/r02/ab_link_rows_unroll.txt)
    // r02 last session: for f64 exact, 2 / 3 / 4 CTAs per SM with or without the early C gather all measure
    // 0.476-0.487 (two CTAs 0.437; profiles/r02/ab_link_rows_cfg.txt): the gathers pull 2.6 KB per site through
    // L2 (13.8 GB per 48^4 sweep, ~11.5 TB/s).  Holding A = U_mu(x) in registers for a mu's planes (15
    // gathers per site instead of 18, 168 registers) measured slower at f64: exact 0.465, FMA 0.480 against
    // 0.476 / 0.525 (f32 0.349 against 0.309, below the walk's 0.354; profiles/r02/ab_link_rows_hold_a.txt)
    if constexpr (sizeof(T) == 4) k_link_rows<T, FUSED, 6, true><<<grid, 128, 0, st>>>(U, acc, g, s, ZC);
    else k_link_rows<T, FUSED, FUSED ? 3 : 4, false><<<grid, 128, 0, st>>>(U, acc, g, s, ZC);
    return check_launch("link_product(rows)");
}

template int launch_link_rows<float, false>(const float*, float*, const Geom&, float, int, cudaStream_t);
template int launch_link_rows<float, true>(const float*, float*, const Geom&, float, int, cudaStream_t);
template int launch_link_rows<double, false>(const double*, double*, const Geom&, double, int, cudaStream_t);
template int launch_link_rows<double, true>(const double*, double*, const Geom&, double, int, cudaStream_t);

}  // namespace su3g
