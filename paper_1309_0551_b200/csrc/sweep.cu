// Lattice sweeps on t-sliced SoA fields, sm_100a.
//
//   * NN sweep  (BASELINE configs[2], [4]):  out = D v, D the periodic
//     nearest-neighbour operator of SURVEY.md 8(a) a13, association of the
//     composed reference oracle (8(c)).
//   * halo pack: w = U_t^dag v on the last local t-slice (the term a t-slab
//     ships to its +t neighbour instead of the 18-real link).
//   * link product (configs[3]): sum over planes of s * U_mu U_nu(x+mu) U_mu(x+nu)^dag.
//
// Field layout (layout.cu): f[(t * C + c) * F + s3], F = nx*ny*nz.
#include <algorithm>

#include "su3_math.cuh"

namespace su3g {

struct Geom {
    int nx, ny, nz, nt;
    int64_t F;  // sites per t-slice
};

template <typename T, int N>
__device__ __forceinline__ void ld_soa(const T* __restrict__ p, int64_t F, int64_t s3, T* r) {
#pragma unroll
    for (int k = 0; k < N; ++k) r[k] = __ldg(p + k * F + s3);
}

// neighbour slice-local index one step along mu in {0, 1, 2} (periodic)
__device__ __forceinline__ int64_t step3(const Geom& g, int x, int y, int z, int mu, int dir) {
    if (mu == 0) x = (x + dir + g.nx) % g.nx;
    else if (mu == 1) y = (y + dir + g.ny) % g.ny;
    else z = (z + dir + g.nz) % g.nz;
    return x + int64_t(g.nx) * (y + int64_t(g.ny) * z);
}

// ---------------------------------------------------------------------------
// NN sweep, one thread per site
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256)
    k_nn_sweep(const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ out, Geom g, int t_begin, int t_end,
               const T* __restrict__ v_hi, const T* __restrict__ w_lo) {
    const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int64_t F = g.F;
    if (idx >= int64_t(t_end - t_begin) * F) return;
    const int t = t_begin + static_cast<int>(idx / F);
    const int64_t s3 = idx % F;
    const int x = static_cast<int>(s3 % g.nx);
    const int y = static_cast<int>((s3 / g.nx) % g.ny);
    const int z = static_cast<int>(s3 / (int64_t(g.nx) * g.ny));

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
            ld_soa<T, 6>(v_hi, F, s3, vn);
        } else {
            ld_soa<T, 6>(v, F, s3, vn);
        }
        mat_vec<T>(u, vn, f);
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
            ld_soa<T, 18>(U + (int64_t(t) * 72 + mu * 18) * F, F, d, u);
            ld_soa<T, 6>(v + int64_t(t) * 6 * F, F, d, vn);
            adj_mat_vec<T>(u, vn, w);
        } else if (t > 0 || w_lo == nullptr) {
            const int tp = (t > 0) ? t - 1 : g.nt - 1;
            T u[18], vn[6];
            ld_soa<T, 18>(U + (int64_t(tp) * 72 + 3 * 18) * F, F, s3, u);
            ld_soa<T, 6>(v + int64_t(tp) * 6 * F, F, s3, vn);
            adj_mat_vec<T>(u, vn, w);
        } else {
            ld_soa<T, 6>(w_lo, F, s3, w);
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) acc[k] = xsub(acc[k], w[k]);
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) out[(int64_t(t) * 6 + k) * F + s3] = acc[k];
}

template <typename T>
__global__ void __launch_bounds__(256)
    k_nn_halo_w(const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ w_face, Geom g) {
    const int64_t s3 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (s3 >= g.F) return;
    const int t = g.nt - 1;
    T u[18], vn[6], w[6];
    ld_soa<T, 18>(U + (int64_t(t) * 72 + 3 * 18) * g.F, g.F, s3, u);
    ld_soa<T, 6>(v + int64_t(t) * 6 * g.F, g.F, s3, vn);
    adj_mat_vec<T>(u, vn, w);
#pragma unroll
    for (int k = 0; k < 6; ++k) w_face[k * g.F + s3] = w[k];
}

// ---------------------------------------------------------------------------
// link product, one thread per site
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t site_step(const Geom& g, int x, int y, int z, int t, int mu) {
    if (mu == 0) x = (x + 1) % g.nx;
    else if (mu == 1) y = (y + 1) % g.ny;
    else if (mu == 2) z = (z + 1) % g.nz;
    else t = (t + 1) % g.nt;
    return int64_t(t) * g.F + x + int64_t(g.nx) * (y + int64_t(g.ny) * z);
}

template <typename T>
__device__ __forceinline__ void ld_link(const T* __restrict__ U, const Geom& g, int64_t site, int mu, T* r) {
    const int64_t t = site / g.F, s3 = site % g.F;
    ld_soa<T, 18>(U + (t * 72 + mu * 18) * g.F, g.F, s3, r);
}

template <typename T, bool FUSED>
__global__ void __launch_bounds__(128)
    k_link_product(const T* __restrict__ U, T* __restrict__ acc_out, Geom g, T s) {
    const int64_t site = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (site >= g.F * g.nt) return;
    const int t = static_cast<int>(site / g.F);
    const int64_t s3 = site % g.F;
    const int x = static_cast<int>(s3 % g.nx);
    const int y = static_cast<int>((s3 / g.nx) % g.ny);
    const int z = static_cast<int>(s3 / (int64_t(g.nx) * g.ny));
    T acc[18];
#pragma unroll
    for (int k = 0; k < 18; ++k) acc[k] = T(0);
#pragma unroll 1
    for (int mu = 0; mu < 3; ++mu) {
        T a[18];
        ld_link(U, g, site, mu, a);
#pragma unroll 1
        for (int nu = mu + 1; nu < 4; ++nu) {
            T b[18], tm[18], p[18];
            ld_link(U, g, site_step(g, x, y, z, t, mu), nu, b);
            if (FUSED) mat_nn_fma<T>(a, b, tm);
            else mat_nn<T>(a, b, tm);
            ld_link(U, g, site_step(g, x, y, z, t, nu), mu, b);
            if (FUSED) mat_na_fma<T>(tm, b, p);
            else mat_na<T>(tm, b, p);
#pragma unroll
            for (int k = 0; k < 18; ++k) acc[k] = FUSED ? fma(s, p[k], acc[k]) : xadd(acc[k], xmul(s, p[k]));
        }
    }
#pragma unroll
    for (int k = 0; k < 18; ++k) acc_out[(int64_t(t) * 18 + k) * g.F + s3] = acc[k];
}

static int check_geom(const char* what, int nx, int ny, int nz, int nt) {
    if (nx < 1 || ny < 1 || nz < 1 || nt < 1) return fail_invalid(std::string(what) + ": lattice extents must be >= 1");
    return SU3G_OK;
}

template <typename T>
static int nn_sweep(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                    const T* v_hi, const T* w_lo, cudaStream_t st) {
    if (int rc = check_geom("nn_sweep", nx, ny, nz, nt)) return rc;
    if (t_begin < 0 || t_end > nt || t_begin > t_end) return fail_invalid("nn_sweep: bad t range");
    if (!U || !v || !out) return fail_invalid("nn_sweep: null pointer");
    if (t_begin == t_end) return SU3G_OK;
    Geom g{nx, ny, nz, nt, int64_t(nx) * ny * nz};
    const int64_t n = int64_t(t_end - t_begin) * g.F;
    k_nn_sweep<T><<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo);
    return check_launch("nn_sweep");
}

template <typename T>
static int nn_halo_w(const T* U, const T* v, T* w, int nx, int ny, int nz, int nt, cudaStream_t st) {
    if (int rc = check_geom("nn_halo_w", nx, ny, nz, nt)) return rc;
    if (!U || !v || !w) return fail_invalid("nn_halo_w: null pointer");
    Geom g{nx, ny, nz, nt, int64_t(nx) * ny * nz};
    k_nn_halo_w<T><<<static_cast<unsigned>((g.F + 255) / 256), 256, 0, st>>>(U, v, w, g);
    return check_launch("nn_halo_w");
}

template <typename T>
static int link_product(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, int mode, cudaStream_t st) {
    if (int rc = check_geom("link_product", nx, ny, nz, nt)) return rc;
    if (!U || !acc) return fail_invalid("link_product: null pointer");
    if (mode != SU3G_EXACT && mode != SU3G_FMA) return fail_invalid("link_product: mode must be SU3G_EXACT or SU3G_FMA");
    Geom g{nx, ny, nz, nt, int64_t(nx) * ny * nz};
    const int64_t n = g.F * nt;
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    if (mode == SU3G_FMA) k_link_product<T, true><<<grid, 128, 0, st>>>(U, acc, g, s);
    else k_link_product<T, false><<<grid, 128, 0, st>>>(U, acc, g, s);
    return check_launch("link_product");
}

}  // namespace su3g

using namespace su3g;

extern "C" {

int su3g_nn_sweep_f32(const float* U, const float* v, float* out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                      int32_t t_begin, int32_t t_end, const float* v_hi, const float* w_lo, su3g_stream_t st) {
    return nn_sweep<float>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, reinterpret_cast<cudaStream_t>(st));
}
int su3g_nn_sweep_f64(const double* U, const double* v, double* out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                      int32_t t_begin, int32_t t_end, const double* v_hi, const double* w_lo, su3g_stream_t st) {
    return nn_sweep<double>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, reinterpret_cast<cudaStream_t>(st));
}
int su3g_nn_halo_w_f32(const float* U, const float* v, float* w, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                       su3g_stream_t st) {
    return nn_halo_w<float>(U, v, w, nx, ny, nz, nt, reinterpret_cast<cudaStream_t>(st));
}
int su3g_nn_halo_w_f64(const double* U, const double* v, double* w, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                       su3g_stream_t st) {
    return nn_halo_w<double>(U, v, w, nx, ny, nz, nt, reinterpret_cast<cudaStream_t>(st));
}
int su3g_link_product_f32(const float* U, float* acc, int32_t nx, int32_t ny, int32_t nz, int32_t nt, float s,
                          int32_t mode, su3g_stream_t st) {
    return link_product<float>(U, acc, nx, ny, nz, nt, s, mode, reinterpret_cast<cudaStream_t>(st));
}
int su3g_link_product_f64(const double* U, double* acc, int32_t nx, int32_t ny, int32_t nz, int32_t nt, double s,
                          int32_t mode, su3g_stream_t st) {
    return link_product<double>(U, acc, nx, ny, nz, nt, s, mode, reinterpret_cast<cudaStream_t>(st));
}

}  // extern "C"
