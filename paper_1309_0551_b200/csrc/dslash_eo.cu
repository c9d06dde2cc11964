// Even/odd dslash on checkerboarded fields, and the layout they live in.
//
// In the t-sliced SoA layout of the sweeps, the sites of one parity alternate in x, so a
// parity launch of the dslash reads every 32-byte sector of U, v and out for half of its
// contents and relies on L2 to keep the other half until the other thread that needs it
// comes by (ncu, 64^3x16 f64: 3.63 GB of DRAM reads per launch against 2.52 GB algorithmic,
// L2 hit rate 32%).  The checkerboarded ("eo") layout stores each parity of a t-slice as its
// own contiguous half, the usual even/odd preconditioning layout of lattice QCD codes:
//
//     eo[(t*C + c)*F + q*F/2 + h],   q = (x+y+z+t) & 1,   h = (x>>1) + (nx/2)*(y + ny*z)
//
// (nx even; x = 2*(h % (nx/2)) + ((q + y + z + t) & 1)).  A parity-p launch then reads the
// p half of U (own links) and the 1-p half of U (backward links) once each, with whole
// sectors, reads the 1-p half of v and writes the p half of out: the algorithmic bytes and
// nothing else (ncu: 2.52 GB of DRAM reads per f64 launch = the algorithmic bytes).
//
// Per-site arithmetic is nn_site's: the forward mat_vec chain in mu order, then the four
// backward adjoint products subtracted in mu order (the association of the composed
// reference, oracle/sweeps.py), so EXACT mode equals su3g_dslash / su3g_nn_sweep bit for bit.
#include <algorithm>
#include <string>

#include "nn_site.cuh"

namespace su3g {

namespace {

struct EoGeom {
    int nx, ny, nz, nt;
    int nxh;
    int64_t F, Fh;  // sites per t-slice, per parity half
};

// element j of an eo plane of slice t (j < F/2: parity 0) -> the SoA offset s3 in the same plane
__device__ __forceinline__ int64_t eo_to_s3(const EoGeom& g, int t, int64_t j) {
    const int q = j >= g.Fh;
    const int64_t h = j - (q ? g.Fh : 0);
    const int xh = static_cast<int>(h % g.nxh);
    const int64_t r = h / g.nxh;
    const int y = static_cast<int>(r % g.ny);
    const int z = static_cast<int>(r / g.ny);
    const int x = 2 * xh + ((q + y + z + t) & 1);
    return x + int64_t(g.nx) * (y + int64_t(g.ny) * z);
}

// SoA -> eo (TO_EO) or back, grid-stride over each (t, c) plane: coalesced on the eo side, stride-2
// on the SoA side (both halves of a plane are visited by neighbouring CTAs, so sectors hit in L2)
template <typename T, bool TO_EO>
__global__ void __launch_bounds__(256) k_eo_plane(const T* __restrict__ src, T* __restrict__ dst, EoGeom g, int C) {
    const int64_t plane = blockIdx.y;  // t*C + c
    const int t = static_cast<int>(plane / C);
    const int64_t base = plane * g.F;
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < g.F; j += int64_t(gridDim.x) * blockDim.x) {
        const int64_t s3 = eo_to_s3(g, t, j);
        if constexpr (TO_EO) dst[base + j] = src[base + s3];
        else dst[base + s3] = src[base + j];
    }
}

template <typename T>
__device__ __forceinline__ T ld_first(const T* p, uint64_t pol) {
    T r;
    if constexpr (sizeof(T) == 4) {
        float f;
        asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(f) : "l"(p), "l"(pol));
        r = f;
    } else {
        double d;
        asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(d) : "l"(p), "l"(pol));
        r = d;
    }
    return r;
}

// 18 reals of a link (or 6 of a vector) at eo offset o of component plane base p: p[k*F + o]
template <typename T, int N, bool STREAM>
__device__ __forceinline__ void ld_eo(const T* __restrict__ p, int64_t F, int64_t o, T* r, uint64_t pol) {
#pragma unroll
    for (int k = 0; k < N; ++k) r[k] = STREAM ? ld_first(p + k * F + o, pol) : __ldg(p + k * F + o);
}

}  // namespace

// One thread per output site of parity `parity`, visiting order (z-chunk, t, z, y, x/2).
template <typename T, bool FUSED, bool HINTS>
__global__ void __launch_bounds__(256)
    k_dslash_eo(const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ out, EoGeom g, int parity, int ZC) {
    const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (idx >= g.Fh * g.nt) return;
    const int xh = static_cast<int>(idx % g.nxh);
    int64_t r = idx / g.nxh;
    const int y = static_cast<int>(r % g.ny);
    r /= g.ny;
    const int zl = static_cast<int>(r % ZC);
    r /= ZC;
    const int t = static_cast<int>(r % g.nt);
    const int z = static_cast<int>(r / g.nt) * ZC + zl;
    const int b = (y + z + t + parity) & 1;  // x = 2*xh + b
    const int64_t F = g.F;
    const int64_t own = (parity ? g.Fh : 0) + xh + int64_t(g.nxh) * (y + int64_t(g.ny) * z);
    const int64_t oth = parity ? 0 : g.Fh;  // the other parity's half
    const uint64_t pol = HINTS ? l2_evict_first_policy() : 0;

    // neighbour eo offsets (other parity) and slices, one step along +/- mu
    auto nb = [&](int mu, int dir, int& tn) -> int64_t {
        int xx = xh, yy = y, zz = z;
        tn = t;
        if (mu == 0) {
            if (dir > 0) xx = b ? (xh + 1 == g.nxh ? 0 : xh + 1) : xh;
            else xx = b ? xh : (xh == 0 ? g.nxh - 1 : xh - 1);
        } else if (mu == 1) {
            yy = dir > 0 ? (y + 1 == g.ny ? 0 : y + 1) : (y == 0 ? g.ny - 1 : y - 1);
        } else if (mu == 2) {
            zz = dir > 0 ? (z + 1 == g.nz ? 0 : z + 1) : (z == 0 ? g.nz - 1 : z - 1);
        } else {
            tn = dir > 0 ? (t + 1 == g.nt ? 0 : t + 1) : (t == 0 ? g.nt - 1 : t - 1);
        }
        return oth + xx + int64_t(g.nxh) * (yy + int64_t(g.ny) * zz);
    };

    T acc[6];
    // forward terms, mu = 0..3, summed left to right (add_su3_vector chain)
#pragma unroll
    for (int mu = 0; mu < 4; ++mu) {
        T u[18], vn[6], f[6];
        ld_eo<T, 18, HINTS>(U + (int64_t(t) * 72 + mu * 18) * F, F, own, u, pol);
        int tn;
        const int64_t o = nb(mu, +1, tn);
        ld_eo<T, 6, false>(v + int64_t(tn) * 6 * F, F, o, vn, pol);
        mv<T, FUSED>(u, vn, f);
#pragma unroll
        for (int k = 0; k < 6; ++k) acc[k] = (mu == 0) ? f[k] : xadd(acc[k], f[k]);
    }
    // backward terms U_mu(x-mu)^dag v(x-mu), subtracted left to right (sub_four_su3_vecs)
#pragma unroll
    for (int mu = 0; mu < 4; ++mu) {
        T u[18], vn[6], w[6];
        int tn;
        const int64_t o = nb(mu, -1, tn);
        ld_eo<T, 18, HINTS>(U + (int64_t(tn) * 72 + mu * 18) * F, F, o, u, pol);
        ld_eo<T, 6, false>(v + int64_t(tn) * 6 * F, F, o, vn, pol);
        amv<T, FUSED>(u, vn, w);
#pragma unroll
        for (int k = 0; k < 6; ++k) acc[k] = xsub(acc[k], w[k]);
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) {
        if constexpr (HINTS) __stcs(out + (int64_t(t) * 6 + k) * F + own, acc[k]);
        else out[(int64_t(t) * 6 + k) * F + own] = acc[k];
    }
}

extern int g_eo_variant;
int g_eo_zc = 0;      // su3g_set_option("dslash_eo_zc"): z-planes per visiting chunk (0 = auto)
// su3g_set_option("dslash_eo_hints"): U loads evict-first, streaming stores.  Off by default: every U
// sector is read once per launch anyway, and the plain form measured 1-1.5% faster (64^3x16: f64
// 0.838 -> 0.849, f32 0.857 -> 0.859 of HBM, three repetitions each)
int g_eo_hints = 0;

static int eo_check(const char* what, int nx, int ny, int nz, int nt) {
    if (nx <= 0 || ny <= 0 || nz <= 0 || nt <= 0) return fail_invalid(std::string(what) + ": lattice extents must be positive");
    if ((nx | ny | nz | nt) & 1) return fail_invalid(std::string(what) + ": every lattice extent must be even (checkerboard)");
    if (int64_t(nx) * ny * nz > (int64_t(1) << 40)) return fail_invalid(std::string(what) + ": lattice too large");
    return SU3G_OK;
}

template <typename T>
static int eo_transform(const T* src, T* dst, int nx, int ny, int nz, int nt, int C, bool to_eo, cudaStream_t st) {
    if (int rc = eo_check(to_eo ? "soa_to_eo" : "eo_to_soa", nx, ny, nz, nt)) return rc;
    if (C <= 0 || C > 4096) return fail_invalid("eo transform: reals_per_site out of range");
    if (!src || !dst) return fail_invalid("eo transform: null pointer");
    if (src == dst) return fail_invalid("eo transform: src and dst must not alias");
    if (int64_t(nt) * C > 65535) return fail_invalid("eo transform: nt * reals_per_site above 65535");
    EoGeom g{nx, ny, nz, nt, nx / 2, int64_t(nx) * ny * nz, int64_t(nx) * ny * nz / 2};
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>((g.F + 255) / 256, 4096)), static_cast<unsigned>(nt * C));
    if (to_eo) k_eo_plane<T, true><<<grid, 256, 0, st>>>(src, dst, g, C);
    else k_eo_plane<T, false><<<grid, 256, 0, st>>>(src, dst, g, C);
    return check_launch(to_eo ? "soa_to_eo" : "eo_to_soa");
}

template <typename T>
static int dslash_eo(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int parity, int mode,
                     cudaStream_t st) {
    if (int rc = eo_check("dslash_eo", nx, ny, nz, nt)) return rc;
    if (parity != 0 && parity != 1) return fail_invalid("dslash_eo: parity must be 0 (even) or 1 (odd)");
    if (mode != SU3G_EXACT && mode != SU3G_FMA) return fail_invalid("dslash_eo: mode must be SU3G_EXACT or SU3G_FMA");
    if (!U || !v || !out) return fail_invalid("dslash_eo: null pointer");
    if (out == v) return fail_invalid("dslash_eo: out must not alias v");
    if (g_eo_variant != 1) {  // the ring walk on the half-lattice (dslash_ring.cu) where it applies
        const int rc = launch_dslash_ring<T>(U, v, out, nx, ny, nz, nt, parity, mode, st);
        if (rc != 1) return rc;
        if (g_eo_variant == 2) return fail_invalid("dslash_eo: ring kernel not applicable to this lattice");
    }
    EoGeom g{nx, ny, nz, nt, nx / 2, int64_t(nx) * ny * nz, int64_t(nx) * ny * nz / 2};
    // z-chunked order keeps the v planes a chunk re-reads in L2 (same rule as the generic sweep)
    int ZC = nz;
    const bool big_slice = double(g.F) * 72 * sizeof(T) > 0.5 * double(device_info().l2_bytes);
    if (big_slice) {
        ZC = 1;
        for (int c = 8; c >= 1; --c)
            if (nz % c == 0) { ZC = c; break; }
    }
    if (g_eo_zc > 0) {
        ZC = 1;
        for (int c = std::min(g_eo_zc, nz); c >= 1; --c)
            if (nz % c == 0) { ZC = c; break; }
    }
    const unsigned grid = static_cast<unsigned>((g.Fh * nt + 255) / 256);
    const bool fma = mode == SU3G_FMA;
    if (g_eo_hints) {
        if (fma) k_dslash_eo<T, true, true><<<grid, 256, 0, st>>>(U, v, out, g, parity, ZC);
        else k_dslash_eo<T, false, true><<<grid, 256, 0, st>>>(U, v, out, g, parity, ZC);
    } else {
        if (fma) k_dslash_eo<T, true, false><<<grid, 256, 0, st>>>(U, v, out, g, parity, ZC);
        else k_dslash_eo<T, false, false><<<grid, 256, 0, st>>>(U, v, out, g, parity, ZC);
    }
    note_kernel(std::string("k_dslash_eo<") + (sizeof(T) == 4 ? "f32" : "f64") + ",zchunk " + std::to_string(ZC) + ">");
    return check_launch("dslash_eo");
}

}  // namespace su3g

using namespace su3g;

extern "C" {

int su3g_soa_to_eo_f32(const float* soa, float* eo, int32_t nx, int32_t ny, int32_t nz, int32_t nt, int32_t C,
                       su3g_stream_t st) {
    return eo_transform<float>(soa, eo, nx, ny, nz, nt, C, true, reinterpret_cast<cudaStream_t>(st));
}
int su3g_soa_to_eo_f64(const double* soa, double* eo, int32_t nx, int32_t ny, int32_t nz, int32_t nt, int32_t C,
                       su3g_stream_t st) {
    return eo_transform<double>(soa, eo, nx, ny, nz, nt, C, true, reinterpret_cast<cudaStream_t>(st));
}
int su3g_eo_to_soa_f32(const float* eo, float* soa, int32_t nx, int32_t ny, int32_t nz, int32_t nt, int32_t C,
                       su3g_stream_t st) {
    return eo_transform<float>(eo, soa, nx, ny, nz, nt, C, false, reinterpret_cast<cudaStream_t>(st));
}
int su3g_eo_to_soa_f64(const double* eo, double* soa, int32_t nx, int32_t ny, int32_t nz, int32_t nt, int32_t C,
                       su3g_stream_t st) {
    return eo_transform<double>(eo, soa, nx, ny, nz, nt, C, false, reinterpret_cast<cudaStream_t>(st));
}
int su3g_dslash_eo_f32(const float* U, const float* v, float* out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                       int32_t parity, int32_t mode, su3g_stream_t st) {
    return dslash_eo<float>(U, v, out, nx, ny, nz, nt, parity, mode, reinterpret_cast<cudaStream_t>(st));
}
int su3g_dslash_eo_f64(const double* U, const double* v, double* out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                       int32_t parity, int32_t mode, su3g_stream_t st) {
    return dslash_eo<double>(U, v, out, nx, ny, nz, nt, parity, mode, reinterpret_cast<cudaStream_t>(st));
}

}  // extern "C"
