// Shared pieces of the lattice-sweep kernels (t-sliced SoA fields, see layout.cu).
#pragma once

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

// Sites of CTA b of a one-thread-per-site kernel in (z-chunk, t, z, y, x) order: when
// nx*ny is a multiple of the CTA size, they are one contiguous run of s3 in one (t, z) plane,
// so each of a field's C components is one contiguous segment.  Thread 0 asks the TMA unit to
// pull the segments of the CTA one wave ahead (b + ahead) into L2: by the time that CTA runs,
// its compulsory loads are L2 hits instead of DRAM round trips (prefetch_ahead = 0: off).
template <typename T>
__device__ __forceinline__ void prefetch_cta_l2(const T* __restrict__ f, int C, const Geom& g, int64_t b, int nthr,
                                                int t_begin, int nts, int ZC, int xdiv = 1) {
    // xdiv = 2: the dslash's index runs over nx/2 output sites per row, each CTA spans 2*nthr sites
    const int nxi = g.nx / xdiv;
    const int64_t idx = b * nthr;
    if (idx >= int64_t(nts) * (g.F / xdiv)) return;
    int64_t r = idx / nxi;
    const int y = static_cast<int>(r % g.ny);
    r /= g.ny;
    const int zl = static_cast<int>(r % ZC);
    r /= ZC;
    const int t = t_begin + static_cast<int>(r % nts);
    const int z = static_cast<int>(r / nts) * ZC + zl;
    const int64_t s3 = int64_t(g.nx) * (y + int64_t(g.ny) * z);
    const uint32_t bytes = static_cast<uint32_t>(nthr * xdiv * sizeof(T));
    for (int c = 0; c < C; ++c) bulk_prefetch_l2(f + (int64_t(t) * C + c) * g.F + s3, bytes);
}

// neighbour slice-local index one step along mu in {0, 1, 2} (periodic)
__device__ __forceinline__ int64_t step3(const Geom& g, int x, int y, int z, int mu, int dir) {
    if (mu == 0) x = (x + dir + g.nx) % g.nx;
    else if (mu == 1) y = (y + dir + g.ny) % g.ny;
    else z = (z + dir + g.nz) % g.nz;
    return x + int64_t(g.nx) * (y + int64_t(g.ny) * z);
}


template <typename T>
__device__ __forceinline__ T ld_stream(const T* p, uint64_t pol) {
    T r;
    if constexpr (sizeof(T) == 4) {
        float f;
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(f) : "l"(p), "l"(pol));
        r = f;
    } else {
        double d;
        asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(d) : "l"(p), "l"(pol));
        r = d;
    }
    return r;
}

// chunk length that best balances the single wave of G CTAs (prologue = ~0.3 slice)
// relative cost of a work item's prologue, in steps (su3g_set_option("chunk_prologue_x10"))
inline double g_prologue_cost = 2.0;

inline int pick_chunk(int64_t nblocks, int nt_range, int G) {
    int best_L = nt_range;
    double best_eff = -1;
    for (int L = nt_range; L >= 1; --L) {
        const int64_t nchunks = (nt_range + L - 1) / L;
        const int64_t items = nblocks * nchunks;
        const int64_t per = (items + G - 1) / G;
        const double work = double(nblocks) * nt_range;
        const double eff = work / (double(per) * G * L) * (L / (L + g_prologue_cost));
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best_L = L;
        }
    }
    return best_L;
}


// TMA-staged t-walk NN sweep (nn_tma.cu); returns SU3G_EINVAL-style status, or
// 1 when the lattice does not meet its constraints (caller falls back).
template <typename T>
int launch_nn_tma(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                  const T* v_hi, const T* w_lo, int mode, cudaStream_t st);

// cp.async-ring link product (link_ring.cu); 1 when the lattice does not fit its block shape.
template <typename T, bool FUSED>
int launch_link_ring(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, cudaStream_t st);

template <typename T, bool FUSED>
int launch_link_planes(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, cudaStream_t st);
template <typename T>
int launch_dslash_tma(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int parity, int mode,
                      cudaStream_t st);
template <typename T, bool FUSED>
int launch_link_tile(const T* U, T* acc, const Geom& g, T s, cudaStream_t st);
template <typename T, bool FUSED>
int launch_link_tw4(const T* U, T* acc, const Geom& g, T s, cudaStream_t st);
template <typename T, bool FUSED>
int launch_link_tw(const T* U, T* acc, const Geom& g, T s, cudaStream_t st);
template <typename T, bool FUSED>
int launch_link_rows3(const T* U, T* acc, const Geom& g, T s, int ZC, cudaStream_t st);
template <typename T, bool FUSED>
int launch_link_rows(const T* U, T* acc, const Geom& g, T s, int ZC, cudaStream_t st);

// f64 TMA t-walk with a register-staged main operand (nn_tma64.cu); 1 = not applicable.
template <typename T, bool FUSED>
int launch_nn_tma64(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                    const T* v_hi, const T* w_lo, cudaStream_t st);

}  // namespace su3g
