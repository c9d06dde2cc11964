// Even/odd dslash on checkerboarded fields as a warp-specialised TMA ring t-walk.
//
// The checkerboarded layout (dslash_eo.cu) keeps each parity of a t-slice as a contiguous half,
//     eo[(t*C + c)*F + q*F/2 + h],   h = xh + (nx/2)*(y + ny*z),   x = 2 xh + ((q + y + z + t) & 1),
// and a parity-p launch computes out on the p sites from v on the 1-p sites.  Seen from one eo
// index h, the sites of the two halves walk the same column: the p site of slice t sits at
// x = 2 xh + b, b = (p + y + z + t) & 1, and the 1-p site with the same index in slice t-1 (and t+1)
// sits at the same x.  So one thread per index h can run the NN ring walk (nn_ring.cu) on the
// half-lattice nx/2 x ny x nz x nt:
//   * its 1-p site of slice t provides, for its neighbours, v (the exchange XV) and the backward
//     half-products w_mu = U_mu^dag v (XW), from the 1-p half of U -- and its w_t is the -t term of
//     its own p site one step later (kept in registers, as in the NN walk);
//   * its p site takes the forward products from the p half of U with the neighbours' v;
//   * along x the neighbours sit at xh + b (forward) and xh - 1 + b (backward) of the same half-row,
//     every other axis keeps xh.
// Per step a producer warp streams ten equal chunks (4-D boxes of 5-D maps (xh, y, z, q, t*C + c)):
//   H1 v(t+1) [6][N] | v on the +y row | U_y on the -y row       H2 the -y/-z/+z halo v and U_z on -z
//   A_x, P_x, A_y, P_y, A_z, P_z, A_t, P_t   (A = the 1-p half of U, P = the p half)
// Per-site arithmetic and order are nn_site's (the composed reference), so EXACT mode equals
// su3g_dslash_eo / su3g_nn_sweep on those sites bit for bit.
#include <cuda.h>

#include <algorithm>
#include <string>

#include "nn_site.cuh"
#include "tma.cuh"

namespace su3g {

int g_eo_variant = 0;  // su3g_set_option("dslash_eo_variant"): 0 auto, 1 gather (k_dslash_eo), 2 ring walk

namespace {

struct DParams {
    int ny, nz, nt;
    int64_t F, Fh;
    int nby;
    int64_t nblocks;
    int chunk;
    int64_t nitems;
    int64_t n_full;  // columns schedule (sweep_common.cuh)
    int parity;
};

template <int NXH>
struct DGeo {
    static constexpr int N = 4 * NXH, H = 2 * NXH, SLOT = 18 * N;
    static constexpr int H1_V = 0, H1_VYU = 6 * N, H1_UYD = 6 * N + 6 * H;
    static constexpr int H2_VYD = 0, H2_UZD = 6 * H, H2_VZD = 24 * H, H2_VZU = 30 * H;
    // exchange: XW [18][N], XH [6][2H] (-y halo sites, then -z), XV [2][6][N]
    static constexpr int XW = 0, XH = 18 * N, XV = 18 * N + 12 * H, XSIZE = XV + 12 * N;
};

// 5-D view of an eo field: (xh, y, z, q, t*C + c)
template <typename T>
bool make_map_eo(CUtensorMap* m, const T* base, int nxh, int ny, int nz, int64_t planes, int BY, int BZ, int box_planes) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    const cuuint64_t dims[5] = {cuuint64_t(nxh), cuuint64_t(ny), cuuint64_t(nz), 2, cuuint64_t(planes)};
    const cuuint64_t half = cuuint64_t(nxh) * ny * nz;
    const cuuint64_t strides[4] = {cuuint64_t(nxh) * sizeof(T), cuuint64_t(nxh) * ny * sizeof(T), half * sizeof(T),
                                   2 * half * sizeof(T)};
    const cuuint32_t box[5] = {cuuint32_t(nxh), cuuint32_t(BY), cuuint32_t(BZ), 1, cuuint32_t(box_planes)};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    return enc(m, dt, 5, const_cast<T*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_addr(bar)),
        "l"(policy)
        : "memory");
}

__device__ __forceinline__ void ditem(const DParams& p, int64_t item, int64_t& blk, int& t0, int& t1) {
    schedule_item(p.n_full, p.nblocks, p.chunk, 0, p.nt, item, blk, t0, t1);
}

}  // namespace

template <typename T, bool FUSED, int NXH, int S, int MINB>
__global__ void __launch_bounds__(4 * NXH + 32, MINB)
    k_dslash_ring(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapV,
                  const __grid_constant__ CUtensorMap mapUyH, const __grid_constant__ CUtensorMap mapUzH,
                  const __grid_constant__ CUtensorMap mapVyH, const __grid_constant__ CUtensorMap mapVzH,
                  const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ out, DParams p) {
    using G = DGeo<NXH>;
    constexpr int N = G::N, H = G::H, NW = N / 32;
    static_assert(N % 32 == 0, "whole compute warps");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* ring = reinterpret_cast<T*>(smem_raw);
    T* xb = ring + S * G::SLOT;
    uint64_t* full = reinterpret_cast<uint64_t*>(xb + G::XSIZE);
    uint64_t* empty = full + S;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t F = p.F;
    const int GR = gridDim.x;
    const int qp = p.parity, q1 = 1 - p.parity;

    // ------------------------------------------------------------------ producer warp
    if (tid >= N) {
        if (tid != N) return;
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
        uint32_t q = 0;
        for (int64_t item = blockIdx.x; item < p.nitems; item += GR) {
            int64_t blk;
            int t0, t1;
            ditem(p, item, blk, t0, t1);
            const int y0 = static_cast<int>(blk % p.nby) * 2, z0 = static_cast<int>(blk / p.nby) * 2;
            const int ydn = (y0 + p.ny - 1) % p.ny, yup = (y0 + 2) % p.ny;
            const int zdn = (z0 + p.nz - 1) % p.nz, zup = (z0 + 2) % p.nz;
            for (int t = t0; t < t1; ++t) {
                const int tn = (t + 1 == p.nt) ? 0 : t + 1;
#pragma unroll 1
                for (int c = 0; c < 10; ++c, ++q) {
                    const int s = static_cast<int>(q % S);
                    if (q >= S) mbar_wait(&empty[s], ((q / S) + 1) & 1);
                    T* dst = ring + s * G::SLOT;
                    mbar_arrive_expect_tx(&full[s], uint32_t(G::SLOT) * sizeof(T));
                    if (c == 0) {
                        tma_load_5d(dst + G::H1_V, &mapV, 0, y0, z0, q1, tn * 6, &full[s], pol);
                        tma_load_5d(dst + G::H1_VYU, &mapVyH, 0, yup, z0, q1, t * 6, &full[s], pol);
                        tma_load_5d(dst + G::H1_UYD, &mapUyH, 0, ydn, z0, q1, t * 72 + 18, &full[s], pol);
                    } else if (c == 1) {
                        tma_load_5d(dst + G::H2_VYD, &mapVyH, 0, ydn, z0, q1, t * 6, &full[s], pol);
                        tma_load_5d(dst + G::H2_UZD, &mapUzH, 0, y0, zdn, q1, t * 72 + 36, &full[s], pol);
                        tma_load_5d(dst + G::H2_VZD, &mapVzH, 0, y0, zdn, q1, t * 6, &full[s], pol);
                        tma_load_5d(dst + G::H2_VZU, &mapVzH, 0, y0, zup, q1, t * 6, &full[s], pol);
                    } else {  // A_mu (1-p half), P_mu (p half), mu-major
                        const int mu = (c - 2) >> 1;
                        tma_load_5d(dst, &mapU, 0, y0, z0, ((c - 2) & 1) ? qp : q1, t * 72 + 18 * mu, &full[s], pol);
                    }
                }
            }
        }
        return;
    }

    // ------------------------------------------------------------------ compute warps
    const int lane = tid & 31;
    const int lx = tid % NXH, ly = (tid / NXH) & 1, lz = tid / (2 * NXH);
    const int row = tid - lx;      // first thread of this half-row
    const int jy = lx + NXH * lz;  // this column's slot in a y halo row (box xh, z)
    const int jz = lx + NXH * ly;  // ... in a z halo row (box xh, y)
    T* const XW = xb + G::XW;
    T* const XH = xb + G::XH;
    T* XV = xb + G::XV;
    const T* const Uq1 = U + q1 * p.Fh;
    const T* const vq1 = v + q1 * p.Fh;

    uint32_t q = 0;
    uint32_t k = 0;  // steps done by this CTA (XV parity)
    for (int64_t item = blockIdx.x; item < p.nitems; item += GR) {
        int64_t blk;
        int t0, t1;
        ditem(p, item, blk, t0, t1);
        const int y = static_cast<int>(blk % p.nby) * 2 + ly;
        const int z = static_cast<int>(blk / p.nby) * 2 + lz;
        const int64_t h = lx + int64_t(NXH) * (y + int64_t(p.ny) * z);
        // prologue: v of this index's 1-p site in slice t0, and w_t of its 1-p site in slice t0-1
        T vc[6], wt[6];
        ld_soa<T, 6>(vq1 + int64_t(t0) * 6 * F, F, h, vc);
        {
            const int tp = (t0 > 0) ? t0 - 1 : p.nt - 1;
            T u[18], vp[6];
            ld_soa<T, 18>(Uq1 + (int64_t(tp) * 72 + 54) * F, F, h, u);
            ld_soa<T, 6>(vq1 + int64_t(tp) * 6 * F, F, h, vp);
            amv<T, FUSED>(u, vp, wt);
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) XV[((k & 1) * 6 + c) * N + tid] = vc[c];
        named_sync<N>();

        for (int t = t0; t < t1; ++t, ++k) {
            const T* xv = XV + (k & 1) * 6 * N;
            const int b = (p.parity + y + z + t) & 1;  // x of this thread's p site = 2 xh + b
            const int ix_up = row + ((lx + b == NXH) ? 0 : lx + b);
            const int ix_dn = row + ((lx + b == 0) ? NXH - 1 : lx + b - 1);
            T vnext[6], nby_[6], nbz_[6];
            // ---- H1, H2: v(t+1), the +y / +z halo v, the -y / -z halo half-products
            {
                const int s1 = static_cast<int>(q % S), s2 = static_cast<int>((q + 1) % S);
                mbar_wait(&full[s1], (q / S) & 1);
                mbar_wait(&full[s2], ((q + 1) / S) & 1);
                const T* h1 = ring + s1 * G::SLOT;
                const T* h2 = ring + s2 * G::SLOT;
#pragma unroll
                for (int c = 0; c < 6; ++c) {
                    vnext[c] = h1[G::H1_V + c * N + tid];
                    nby_[c] = h1[G::H1_VYU + c * H + jy];
                    nbz_[c] = h2[G::H2_VZU + c * H + jz];
                }
                T uh[18], vh[6], wh[6];
                if (tid < H) {
#pragma unroll
                    for (int c = 0; c < 18; ++c) uh[c] = h1[G::H1_UYD + c * H + tid];
#pragma unroll
                    for (int c = 0; c < 6; ++c) vh[c] = h2[G::H2_VYD + c * H + tid];
                } else {
#pragma unroll
                    for (int c = 0; c < 18; ++c) uh[c] = h2[G::H2_UZD + c * H + (tid - H)];
#pragma unroll
                    for (int c = 0; c < 6; ++c) vh[c] = h2[G::H2_VZD + c * H + (tid - H)];
                }
                warp_release(&empty[s1], lane);
                if (lane == 0) mbar_arrive(&empty[s2]);
                amv<T, FUSED>(uh, vh, wh);
#pragma unroll
                for (int c = 0; c < 6; ++c) XH[c * (2 * H) + tid] = wh[c];
            }
            // ---- x, y, z: publish w_mu of the 1-p site, forward term of the p site
            T acc[6];
#pragma unroll
            for (int mu = 0; mu < 3; ++mu) {
                T u[18], w[6], nb[6], f[6];
                {
                    const uint32_t qa = q + 2 + 2 * mu;
                    const int s = static_cast<int>(qa % S);
                    mbar_wait(&full[s], (qa / S) & 1);
                    const T* su = ring + s * G::SLOT;
#pragma unroll
                    for (int c = 0; c < 18; ++c) u[c] = su[c * N + tid];
                    warp_release(&empty[s], lane);
                }
                amv<T, FUSED>(u, vc, w);
#pragma unroll
                for (int c = 0; c < 6; ++c) XW[(6 * mu + c) * N + tid] = w[c];
                {
                    const uint32_t qp_ = q + 3 + 2 * mu;
                    const int s = static_cast<int>(qp_ % S);
                    mbar_wait(&full[s], (qp_ / S) & 1);
                    const T* su = ring + s * G::SLOT;
#pragma unroll
                    for (int c = 0; c < 18; ++c) u[c] = su[c * N + tid];
                    warp_release(&empty[s], lane);
                }
                const int src = mu == 0 ? ix_up : (mu == 1 ? (ly == 0 ? tid + NXH : -1) : (lz == 0 ? tid + 2 * NXH : -1));
                if (src >= 0) {
#pragma unroll
                    for (int c = 0; c < 6; ++c) nb[c] = xv[c * N + src];
                } else {
#pragma unroll
                    for (int c = 0; c < 6; ++c) nb[c] = mu == 1 ? nby_[c] : nbz_[c];
                }
                mv<T, FUSED>(u, nb, f);
#pragma unroll
                for (int c = 0; c < 6; ++c) acc[c] = (mu == 0) ? f[c] : xadd(acc[c], f[c]);
            }
            // ---- t: w_t of the 1-p site (the -t term one step later), forward +t term of the p site
            T wt_next[6];
            {
                T u[18], f[6];
                {
                    const uint32_t qa = q + 8;
                    const int s = static_cast<int>(qa % S);
                    mbar_wait(&full[s], (qa / S) & 1);
                    const T* su = ring + s * G::SLOT;
#pragma unroll
                    for (int c = 0; c < 18; ++c) u[c] = su[c * N + tid];
                    warp_release(&empty[s], lane);
                }
                amv<T, FUSED>(u, vc, wt_next);
                {
                    const uint32_t qa = q + 9;
                    const int s = static_cast<int>(qa % S);
                    mbar_wait(&full[s], (qa / S) & 1);
                    const T* su = ring + s * G::SLOT;
#pragma unroll
                    for (int c = 0; c < 18; ++c) u[c] = su[c * N + tid];
                    warp_release(&empty[s], lane);
                }
                mv<T, FUSED>(u, vnext, f);
#pragma unroll
                for (int c = 0; c < 6; ++c) acc[c] = xadd(acc[c], f[c]);
            }
            q += 10;
#pragma unroll
            for (int c = 0; c < 6; ++c) XV[(((k + 1) & 1) * 6 + c) * N + tid] = vnext[c];
            named_sync<N>();

            // ---- backward terms (sub_four_su3_vecs chain)
#pragma unroll
            for (int c = 0; c < 6; ++c) acc[c] = xsub(acc[c], XW[c * N + ix_dn]);
            {
                const T* bw = ly == 1 ? XW + 6 * N + tid - NXH : XH + jy;
                const int bs = ly == 1 ? N : 2 * H;
#pragma unroll
                for (int c = 0; c < 6; ++c) acc[c] = xsub(acc[c], bw[c * bs]);
                bw = lz == 1 ? XW + 12 * N + tid - 2 * NXH : XH + H + jz;
                const int bs2 = lz == 1 ? N : 2 * H;
#pragma unroll
                for (int c = 0; c < 6; ++c) acc[c] = xsub(acc[c], bw[c * bs2]);
            }
#pragma unroll
            for (int c = 0; c < 6; ++c) acc[c] = xsub(acc[c], wt[c]);
            T* o = out + int64_t(t) * 6 * F + qp * p.Fh + h;
#pragma unroll
            for (int c = 0; c < 6; ++c) __stcs(o + c * F, acc[c]);
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                vc[c] = vnext[c];
                wt[c] = wt_next[c];
            }
            named_sync<N>();  // XW / XH are rewritten by the next step
        }
    }
}

template <typename T, bool FUSED, int NXH, int S, int MINB>
static int run_dslash_ring(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int parity,
                           cudaStream_t st) {
    using G = DGeo<NXH>;
    CUtensorMap mU, mV, mUy, mUz, mVy, mVz;
    if (!make_map_eo<T>(&mU, U, NXH, ny, nz, int64_t(nt) * 72, 2, 2, 18) ||
        !make_map_eo<T>(&mV, v, NXH, ny, nz, int64_t(nt) * 6, 2, 2, 6) ||
        !make_map_eo<T>(&mUy, U, NXH, ny, nz, int64_t(nt) * 72, 1, 2, 18) ||
        !make_map_eo<T>(&mUz, U, NXH, ny, nz, int64_t(nt) * 72, 2, 1, 18) ||
        !make_map_eo<T>(&mVy, v, NXH, ny, nz, int64_t(nt) * 6, 1, 2, 6) ||
        !make_map_eo<T>(&mVz, v, NXH, ny, nz, int64_t(nt) * 6, 2, 1, 6))
        return 1;
    const size_t smem = (size_t(S) * G::SLOT + G::XSIZE) * sizeof(T) + 2 * S * sizeof(uint64_t);
    const DeviceInfo& di = device_info();
    if (smem > size_t(di.max_smem_optin)) return 1;
    auto kern = k_dslash_ring<T, FUSED, NXH, S, MINB>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    DParams p{};
    p.ny = ny; p.nz = nz; p.nt = nt;
    p.F = int64_t(nx) * ny * nz;
    p.Fh = p.F / 2;
    p.nby = ny / 2;
    p.nblocks = int64_t(ny / 2) * (nz / 2);
    p.parity = parity;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::N + 32, smem);
    const int per = std::max(per_sm, 1);
    const int G_full = di.num_sms * per;
    const WalkSchedule ws = pick_schedule(p.nblocks, nt, G_full, g_prologue_cost, g_ring_columns != 0);
    p.n_full = ws.n_full;
    p.chunk = ws.chunk;
    p.nitems = ws.nitems;
    const int grid = static_cast<int>(std::min<int64_t>(G_full, p.nitems));
    kern<<<grid, G::N + 32, smem, st>>>(mU, mV, mUy, mUz, mVy, mVz, U, v, out, p);
    note_kernel(std::string("k_dslash_ring<") + (sizeof(T) == 4 ? "f32," : "f64,") + std::to_string(NXH) + "x2x2," +
                std::to_string(S) + " slots" + (per > 1 ? "," + std::to_string(per) + " CTAs/SM" : "") +
                (p.n_full ? "," + std::to_string(p.n_full) + " columns" : "") + ">");
    return check_launch("dslash_eo(ring)");
}

int g_eo_ring_cfg = 0;  // su3g_set_option("dslash_eo_ring_cfg"): A/B of the slot count / CTAs per SM

template <typename T, bool FUSED, int NXH>
static int dring_dispatch(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int parity, cudaStream_t st) {
    if constexpr (sizeof(T) == 8) {  // 64^3x16: 4 slots x 2 CTAs/SM 1.009, 6 slots x 1 CTA 1.003-1.004
        if (g_eo_ring_cfg == 1) return run_dslash_ring<T, FUSED, NXH, 6, 1>(U, v, out, nx, ny, nz, nt, parity, st);
        return run_dslash_ring<T, FUSED, NXH, 4, 2>(U, v, out, nx, ny, nz, nt, parity, st);
    } else {  // 64^3x16, fraction of HBM: 4 slots x 4 CTAs/SM 0.992, 8 x 2: 0.971-0.979, 6 x 3: 0.970
        if (g_eo_ring_cfg == 1) return run_dslash_ring<T, FUSED, NXH, 6, 3>(U, v, out, nx, ny, nz, nt, parity, st);
        if (g_eo_ring_cfg == 2) return run_dslash_ring<T, FUSED, NXH, 8, 2>(U, v, out, nx, ny, nz, nt, parity, st);
        return run_dslash_ring<T, FUSED, NXH, 4, 4>(U, v, out, nx, ny, nz, nt, parity, st);
    }
}

// 1 = not applicable to this lattice (caller falls back to the gather kernel)
template <typename T>
int launch_dslash_ring(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int parity, int mode,
                       cudaStream_t st) {
    if (ny % 2 || nz % 2) return 1;
    if (!aligned16(U) || !aligned16(v) || !aligned16(out)) return 1;
    const bool fma = mode == SU3G_FMA;
    if (nx == 64)
        return fma ? dring_dispatch<T, true, 32>(U, v, out, nx, ny, nz, nt, parity, st)
                   : dring_dispatch<T, false, 32>(U, v, out, nx, ny, nz, nt, parity, st);
    if (nx == 32)
        return fma ? dring_dispatch<T, true, 16>(U, v, out, nx, ny, nz, nt, parity, st)
                   : dring_dispatch<T, false, 16>(U, v, out, nx, ny, nz, nt, parity, st);
    return 1;
}

template int launch_dslash_ring<float>(const float*, const float*, float*, int, int, int, int, int, int, cudaStream_t);
template int launch_dslash_ring<double>(const double*, const double*, double*, int, int, int, int, int, int,
                                        cudaStream_t);

}  // namespace su3g
