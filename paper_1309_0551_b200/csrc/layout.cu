// AoS <-> t-sliced SoA layout transforms (north star: "layout-transform kernel").
//
// The reference stores every field site-major with a site's reals adjacent
// (lattice.py:155-187, SiteBuffer).  The sweeps keep fields resident in a
// GPU-internal structure-of-arrays, sliced by t so that each t-face is one
// contiguous block (the unit a t-slab halo exchange moves):
//     soa[(t * C + c) * F + s3],   F = nx*ny*nz,  s3 = x + nx*(y + ny*z)
// A warp then reads component c of 32 consecutive sites as one 128-byte line.
//
// The transform is a batched transpose [F][C] -> [C][F] per slice through a
// padded shared-memory tile: coalesced reads of the AoS run, coalesced writes
// of each SoA row.  Pure data movement (2 x bytes, HBM bound).
#include "su3g_common.cuh"

namespace su3g {

constexpr int LT_SITES = 64;
constexpr int LT_THREADS = 256;

template <typename T, int C>
__global__ void __launch_bounds__(LT_THREADS) k_aos_to_soa(const T* __restrict__ aos, T* __restrict__ soa, int64_t F) {
    constexpr int P = C + 1;  // odd pitch -> conflict-free column reads
    __shared__ T tile[LT_SITES * P];
    const int64_t slice = blockIdx.y;
    const int64_t s0 = int64_t(blockIdx.x) * LT_SITES;
    const int ns = static_cast<int>((F - s0) < LT_SITES ? (F - s0) : LT_SITES);
    const T* src = aos + (slice * F + s0) * C;
    for (int e = threadIdx.x; e < ns * C; e += LT_THREADS) tile[(e / C) * P + (e % C)] = src[e];
    __syncthreads();
    T* dst = soa + slice * C * F + s0;
    for (int e = threadIdx.x; e < C * LT_SITES; e += LT_THREADS) {
        const int c = e / LT_SITES, s = e % LT_SITES;
        if (s < ns) dst[int64_t(c) * F + s] = tile[s * P + c];
    }
}

template <typename T, int C>
__global__ void __launch_bounds__(LT_THREADS) k_soa_to_aos(const T* __restrict__ soa, T* __restrict__ aos, int64_t F) {
    constexpr int P = C + 1;
    __shared__ T tile[LT_SITES * P];
    const int64_t slice = blockIdx.y;
    const int64_t s0 = int64_t(blockIdx.x) * LT_SITES;
    const int ns = static_cast<int>((F - s0) < LT_SITES ? (F - s0) : LT_SITES);
    const T* src = soa + slice * C * F + s0;
    for (int e = threadIdx.x; e < C * LT_SITES; e += LT_THREADS) {
        const int c = e / LT_SITES, s = e % LT_SITES;
        if (s < ns) tile[s * P + c] = src[int64_t(c) * F + s];
    }
    __syncthreads();
    T* dst = aos + (slice * F + s0) * C;
    for (int e = threadIdx.x; e < ns * C; e += LT_THREADS) dst[e] = tile[(e / C) * P + (e % C)];
}

template <typename T, bool TO_SOA, int C>
static int run_transform(const T* src, T* dst, int64_t F, int64_t nslices, cudaStream_t st) {
    const dim3 grid(static_cast<unsigned>((F + LT_SITES - 1) / LT_SITES), static_cast<unsigned>(nslices));
    if (TO_SOA) k_aos_to_soa<T, C><<<grid, LT_THREADS, 0, st>>>(src, dst, F);
    else k_soa_to_aos<T, C><<<grid, LT_THREADS, 0, st>>>(src, dst, F);
    return check_launch(TO_SOA ? "aos_to_soa" : "soa_to_aos");
}

template <typename T, bool TO_SOA>
static int transform(const T* src, T* dst, int64_t F, int64_t nslices, int32_t C, cudaStream_t st) {
    if (F < 0 || nslices < 0) return fail_invalid("layout transform: negative extent");
    if (F == 0 || nslices == 0) return SU3G_OK;
    if (src == nullptr || dst == nullptr) return fail_invalid("layout transform: null pointer");
    if (nslices > 65535) return fail_invalid("layout transform: more than 65535 slices");
    switch (C) {
        case 2: return run_transform<T, TO_SOA, 2>(src, dst, F, nslices, st);
        case 6: return run_transform<T, TO_SOA, 6>(src, dst, F, nslices, st);
        case 12: return run_transform<T, TO_SOA, 12>(src, dst, F, nslices, st);
        case 18: return run_transform<T, TO_SOA, 18>(src, dst, F, nslices, st);
        case 24: return run_transform<T, TO_SOA, 24>(src, dst, F, nslices, st);
        case 72: return run_transform<T, TO_SOA, 72>(src, dst, F, nslices, st);
        default: return fail_invalid("layout transform: reals_per_site must be one of 2, 6, 12, 18, 24, 72");
    }
}

}  // namespace su3g

using namespace su3g;

extern "C" {

int su3g_aos_to_soa_f32(const float* aos, float* soa, int64_t F, int64_t nslices, int32_t C, su3g_stream_t st) {
    return transform<float, true>(aos, soa, F, nslices, C, reinterpret_cast<cudaStream_t>(st));
}
int su3g_aos_to_soa_f64(const double* aos, double* soa, int64_t F, int64_t nslices, int32_t C, su3g_stream_t st) {
    return transform<double, true>(aos, soa, F, nslices, C, reinterpret_cast<cudaStream_t>(st));
}
int su3g_soa_to_aos_f32(const float* soa, float* aos, int64_t F, int64_t nslices, int32_t C, su3g_stream_t st) {
    return transform<float, false>(soa, aos, F, nslices, C, reinterpret_cast<cudaStream_t>(st));
}
int su3g_soa_to_aos_f64(const double* soa, double* aos, int64_t F, int64_t nslices, int32_t C, su3g_stream_t st) {
    return transform<double, false>(soa, aos, F, nslices, C, reinterpret_cast<cudaStream_t>(st));
}

}  // extern "C"
