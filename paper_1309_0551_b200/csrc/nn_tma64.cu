// NN sweep, TMA t-walk for double precision (register-staged main operand).
//
// Same algorithm, association and halo scheme as k_nn_tma (nn_tma.cu), reshaped
// for f64 where a double-buffered stage of U_x,U_y,U_z,U_t,v(t+1) plus halo rows
// would not fit in 227 KB of shared memory:
//   * the block's main operands (U_x, U_y, U_z, U_t and v(t+1): 78 reals/site) sit
//     in ONE stage; every thread copies its site's 78 reals into registers at the
//     top of a step and releases the stage (empty mbarrier), and thread 0
//     immediately issues the TMA for step k+1 -- the registers are the second
//     buffer, so the next slice streams in for a whole step;
//   * the halo rows (U_y / U_z rows below the block, v rows on both sides) are
//     double-buffered in shared memory and refilled after the end-of-step barrier;
//   * block = 64 x 2 x 1 sites (128 threads), exchange buffer as in k_nn_tma.
// Per-site arithmetic is identical to the other NN kernels -> bit-identical.
#include <cuda.h>

#include <algorithm>

#include "sweep_common.cuh"

namespace su3g {

namespace {

typedef CUresult (*EncodeTiledFn64)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn64 encode64() {
    static EncodeTiledFn64 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeTiledFn64>(nullptr);
        return reinterpret_cast<EncodeTiledFn64>(p);
    }();
    return fn;
}

template <typename T>
bool map4(CUtensorMap* m, const T* base, int nx, int ny, int nz, int64_t planes, int by, int bz, int bp) {
    EncodeTiledFn64 enc = encode64();
    if (!enc) return false;
    const cuuint64_t dims[4] = {cuuint64_t(nx), cuuint64_t(ny), cuuint64_t(nz), cuuint64_t(planes)};
    const cuuint64_t strides[3] = {cuuint64_t(nx) * sizeof(T), cuuint64_t(nx) * ny * sizeof(T),
                                   cuuint64_t(nx) * ny * nz * sizeof(T)};
    const cuuint32_t box[4] = {cuuint32_t(nx), cuuint32_t(by), cuuint32_t(bz), cuuint32_t(bp)};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    return enc(m, dt, 4, const_cast<T*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar,
                                     uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

template <int N>
__device__ __forceinline__ void nsync() {
    asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory");
}

struct P64 {
    int nx, ny, nz, nt;
    int64_t F;
    int BY, BZ, nby;
    int64_t nblocks;
    int t_begin, t_end, chunk;
    int64_t nitems;
    int has_vhi;
};

}  // namespace

// main stage: [78][N] = U_x, U_y, U_z, U_t (72 planes) + v(t+1) (6 planes)
// halo stage (x2): HUy[18][HY] HVyd[6][HY] HVyu[6][HY] HUz[18][HZ] HVzd[6][HZ] HVzu[6][HZ]
// exchange: XW[18][N] XV[6][N] XHy[6][HY] XHz[6][HZ]
template <typename T, bool FUSED, int NTHR, int BY, int BZ>
__global__ void __launch_bounds__(NTHR, 1)
    k_nn_tma64(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapV,
               const __grid_constant__ CUtensorMap mapVhi, const __grid_constant__ CUtensorMap mapUyH,
               const __grid_constant__ CUtensorMap mapUzH, const __grid_constant__ CUtensorMap mapVyH,
               const __grid_constant__ CUtensorMap mapVzH, const T* __restrict__ U, const T* __restrict__ v,
               T* __restrict__ out, const T* __restrict__ w_lo, P64 p) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int nx = p.nx;
    const int HY = (BY == p.ny) ? 0 : nx * BZ;
    const int HZ = (BZ == p.nz) ? 0 : nx * BY;
    const int HS = 30 * HY + 30 * HZ;  // halo stage reals
    T* sm_main = reinterpret_cast<T*>(smem_raw);
    T* sm_halo = sm_main + 78 * NTHR;  // [2][HS]
    T* xb = sm_halo + 2 * HS;
    const int XWo = 0, XVo = 18 * NTHR, XHyo = 24 * NTHR, XHzo = 24 * NTHR + 6 * HY;
    uint64_t* bars = reinterpret_cast<uint64_t*>(xb + 24 * NTHR + 6 * HY + 6 * HZ);
    uint64_t* full_main = bars;
    uint64_t* empty_main = bars + 1;
    uint64_t* full_halo = bars + 2;  // [2]

    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(full_main, 1);
        mbar_init(empty_main, NTHR);
        mbar_init(&full_halo[0], 1);
        mbar_init(&full_halo[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int G = gridDim.x;
    const int64_t F = p.F;

    uint64_t pol_first = 0, pol_normal = 0;
    if (tid == 0) {
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_normal));
    }
    auto blk_origin = [&](int64_t blk, int& y0, int& z0) {
        y0 = static_cast<int>(blk % p.nby) * BY;
        z0 = static_cast<int>(blk / p.nby) * BZ;
    };
    auto issue_main = [&](int64_t blk, int t) {
        int y0, z0;
        blk_origin(blk, y0, z0);
        mbar_arrive_expect_tx(full_main, uint32_t(78 * NTHR) * sizeof(T));
        tma4(sm_main, &mapU, 0, y0, z0, t * 72, full_main, pol_first);
        tma4(sm_main + 18 * NTHR, &mapU, 0, y0, z0, t * 72 + 18, full_main, pol_normal);
        tma4(sm_main + 36 * NTHR, &mapU, 0, y0, z0, t * 72 + 36, full_main, pol_normal);
        tma4(sm_main + 54 * NTHR, &mapU, 0, y0, z0, t * 72 + 54, full_main, pol_first);
        T* dv = sm_main + 72 * NTHR;
        if (t + 1 < p.nt) tma4(dv, &mapV, 0, y0, z0, (t + 1) * 6, full_main, pol_normal);
        else if (p.has_vhi) tma4(dv, &mapVhi, 0, y0, z0, 0, full_main, pol_normal);
        else tma4(dv, &mapV, 0, y0, z0, 0, full_main, pol_normal);
    };
    auto issue_halo = [&](int hs, int64_t blk, int t) {
        int y0, z0;
        blk_origin(blk, y0, z0);
        uint64_t* bar = &full_halo[hs];
        mbar_arrive_expect_tx(bar, uint32_t(HS) * sizeof(T));
        T* h = sm_halo + hs * HS;
        if (HY) {
            const int ydn = (y0 + p.ny - 1) % p.ny, yup = (y0 + BY) % p.ny;
            tma4(h, &mapUyH, 0, ydn, z0, t * 72 + 18, bar, pol_normal);
            tma4(h + 18 * HY, &mapVyH, 0, ydn, z0, t * 6, bar, pol_normal);
            tma4(h + 24 * HY, &mapVyH, 0, yup, z0, t * 6, bar, pol_normal);
        }
        if (HZ) {
            const int zdn = (z0 + p.nz - 1) % p.nz, zup = (z0 + BZ) % p.nz;
            T* hz = h + 30 * HY;
            tma4(hz, &mapUzH, 0, y0, zdn, t * 72 + 36, bar, pol_normal);
            tma4(hz + 18 * HZ, &mapVzH, 0, y0, zdn, t * 6, bar, pol_normal);
            tma4(hz + 24 * HZ, &mapVzH, 0, y0, zup, t * 6, bar, pol_normal);
        }
    };

    const int lx = tid % nx;
    const int rr = tid / nx;
    const int ly = rr % BY;
    const int lz = rr / BY;
    const int sy = nx, sz = nx * BY;
    const int ix_up = (lx + 1 == nx) ? tid - lx : tid + 1;
    const int ix_dn = (lx == 0) ? tid + nx - 1 : tid - 1;
    const int iy_up = (ly + 1 < BY) ? tid + sy : (HY == 0 ? tid - (BY - 1) * sy : -1 - (lx + nx * lz));
    const int iy_dn = (ly > 0) ? tid - sy : (HY == 0 ? tid + (BY - 1) * sy : -1 - (lx + nx * lz));
    const int iz_up = (lz + 1 < BZ) ? tid + sz : (HZ == 0 ? tid - (BZ - 1) * sz : -1 - (lx + nx * ly));
    const int iz_dn = (lz > 0) ? tid - sz : (HZ == 0 ? tid + (BZ - 1) * sz : -1 - (lx + nx * ly));

    struct Cur {
        int64_t item, blk;
        int t, t0, t1;
        bool valid;
    };
    auto enter = [&](Cur& c) {
        const int64_t ch = c.item / p.nblocks;
        c.blk = c.item - ch * p.nblocks;
        c.t0 = p.t_begin + static_cast<int>(ch) * p.chunk;
        c.t1 = min(c.t0 + p.chunk, p.t_end);
        c.t = c.t0;
    };
    auto advance = [&](Cur& c) {
        if (!c.valid) return;
        if (++c.t < c.t1) return;
        c.item += G;
        if (c.item >= p.nitems) {
            c.valid = false;
            return;
        }
        enter(c);
    };

    Cur cur{static_cast<int64_t>(blockIdx.x), 0, 0, 0, 0, static_cast<int64_t>(blockIdx.x) < p.nitems};
    if (!cur.valid) return;
    enter(cur);
    Cur nxt = cur;   // step k + 1 (main refill)
    advance(nxt);
    Cur nxt2 = nxt;  // step k + 2 (halo refill)
    advance(nxt2);
    if (tid == 0) {
        issue_main(cur.blk, cur.t);
        issue_halo(0, cur.blk, cur.t);
        if (nxt.valid) issue_halo(1, nxt.blk, nxt.t);
    }

    T vc[6], wt[6];
    int64_t item_seen = -1;
    for (int64_t k = 0; cur.valid; ++k) {
        const int y = static_cast<int>(cur.blk % p.nby) * BY + ly;
        const int z = static_cast<int>(cur.blk / p.nby) * BZ + lz;
        const int64_t s3 = lx + int64_t(nx) * (y + int64_t(p.ny) * z);
        const int t = cur.t;
        if (cur.item != item_seen) {  // prologue of a work item: v(x,t0), w_t(x,t0-1)
            item_seen = cur.item;
            ld_soa<T, 6>(v + int64_t(t) * 6 * F, F, s3, vc);
            if (t == 0 && w_lo != nullptr) {
                ld_soa<T, 6>(w_lo, F, s3, wt);
            } else {
                const int tp = (t > 0) ? t - 1 : p.nt - 1;
                T u[18], vp[6];
                ld_soa<T, 18>(U + (int64_t(tp) * 72 + 54) * F, F, s3, u);
                ld_soa<T, 6>(v + int64_t(tp) * 6 * F, F, s3, vp);
                amv<T, FUSED>(u, vp, wt);
            }
        }
        // main operands -> registers, release the stage, stream the next slice into it
        mbar_wait(full_main, static_cast<uint32_t>(k & 1));
        T u[54], ut[18], vnext[6];
#pragma unroll
        for (int q = 0; q < 54; ++q) u[q] = sm_main[q * NTHR + tid];
#pragma unroll
        for (int q = 0; q < 18; ++q) ut[q] = sm_main[(54 + q) * NTHR + tid];
#pragma unroll
        for (int q = 0; q < 6; ++q) vnext[q] = sm_main[(72 + q) * NTHR + tid];
        arrive(empty_main);
        if (tid == 0 && nxt.valid) {
            mbar_wait(empty_main, static_cast<uint32_t>(k & 1));
            issue_main(nxt.blk, nxt.t);
        }
        T wt_next[6], f3[6];
        amv<T, FUSED>(ut, vc, wt_next);
        mv<T, FUSED>(ut, vnext, f3);  // forward +t term, summed last

        const int hs = static_cast<int>(k & 1);
        mbar_wait(&full_halo[hs], static_cast<uint32_t>((k >> 1) & 1));
        const T* h = sm_halo + hs * HS;
        for (int j = tid; j < HY + HZ; j += NTHR) {
            const bool isy = j < HY;
            const int jj = isy ? j : j - HY;
            const int hp = isy ? HY : HZ;
            const T* hb = isy ? h : h + 30 * HY;
            T uh[18], vh[6], wh[6];
#pragma unroll
            for (int q = 0; q < 18; ++q) uh[q] = hb[q * hp + jj];
#pragma unroll
            for (int q = 0; q < 6; ++q) vh[q] = hb[(18 + q) * hp + jj];
            amv<T, FUSED>(uh, vh, wh);
            T* xo = xb + (isy ? XHyo : XHzo);
#pragma unroll
            for (int q = 0; q < 6; ++q) xo[q * hp + jj] = wh[q];
        }
        {
            T w[6];
#pragma unroll
            for (int mu = 0; mu < 3; ++mu) {
                amv<T, FUSED>(u + 18 * mu, vc, w);
#pragma unroll
                for (int q = 0; q < 6; ++q) xb[XWo + (6 * mu + q) * NTHR + tid] = w[q];
            }
#pragma unroll
            for (int q = 0; q < 6; ++q) xb[XVo + q * NTHR + tid] = vc[q];
        }
        nsync<NTHR>();

        T acc[6];
        {
            T nb[6], f[6];
#pragma unroll
            for (int q = 0; q < 6; ++q) nb[q] = xb[XVo + q * NTHR + ix_up];
            mv<T, FUSED>(u, nb, acc);
            if (iy_up >= 0) {
#pragma unroll
                for (int q = 0; q < 6; ++q) nb[q] = xb[XVo + q * NTHR + iy_up];
            } else {
#pragma unroll
                for (int q = 0; q < 6; ++q) nb[q] = h[(24 + q) * HY + (-1 - iy_up)];
            }
            mv<T, FUSED>(u + 18, nb, f);
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xadd(acc[q], f[q]);
            if (iz_up >= 0) {
#pragma unroll
                for (int q = 0; q < 6; ++q) nb[q] = xb[XVo + q * NTHR + iz_up];
            } else {
#pragma unroll
                for (int q = 0; q < 6; ++q) nb[q] = h[30 * HY + (24 + q) * HZ + (-1 - iz_up)];
            }
            mv<T, FUSED>(u + 36, nb, f);
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xadd(acc[q], f[q]);
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xadd(acc[q], f3[q]);
        }
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], xb[XWo + q * NTHR + ix_dn]);
        if (iy_dn >= 0) {
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], xb[XWo + (6 + q) * NTHR + iy_dn]);
        } else {
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], xb[XHyo + q * HY + (-1 - iy_dn)]);
        }
        if (iz_dn >= 0) {
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], xb[XWo + (12 + q) * NTHR + iz_dn]);
        } else {
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], xb[XHzo + q * HZ + (-1 - iz_dn)]);
        }
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], wt[q]);
        T* o = out + int64_t(t) * 6 * F + s3;
#pragma unroll
        for (int q = 0; q < 6; ++q) o[q * F] = acc[q];
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            vc[q] = vnext[q];
            wt[q] = wt_next[q];
        }
        nsync<NTHR>();  // exchange + halo stage hs free
        if (tid == 0 && nxt2.valid) issue_halo(hs, nxt2.blk, nxt2.t);
        advance(cur);
        advance(nxt);
        advance(nxt2);
    }
}

template <typename T, bool FUSED>
int launch_nn_tma64(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                    const T* v_hi, const T* w_lo, cudaStream_t st) {
    constexpr int NTHR = 128, BY = 2, BZ = 1;
    if (nx != 64 || ny % BY || nz % BZ) return 1;
    if (!aligned16(U) || !aligned16(v) || (v_hi && !aligned16(v_hi))) return 1;
    const int HY = (BY == ny) ? 0 : nx * BZ, HZ = (BZ == nz) ? 0 : nx * BY;
    CUtensorMap mU, mV, mVhi, mUy, mUz, mVy, mVz;
    if (!map4<T>(&mU, U, nx, ny, nz, int64_t(nt) * 72, BY, BZ, 18)) return 1;
    if (!map4<T>(&mV, v, nx, ny, nz, int64_t(nt) * 6, BY, BZ, 6)) return 1;
    mVhi = mV;
    if (v_hi && !map4<T>(&mVhi, v_hi, nx, ny, nz, 6, BY, BZ, 6)) return 1;
    mUy = mU; mVy = mV; mUz = mU; mVz = mV;
    if (HY && (!map4<T>(&mUy, U, nx, ny, nz, int64_t(nt) * 72, 1, BZ, 18) ||
               !map4<T>(&mVy, v, nx, ny, nz, int64_t(nt) * 6, 1, BZ, 6)))
        return 1;
    if (HZ && (!map4<T>(&mUz, U, nx, ny, nz, int64_t(nt) * 72, BY, 1, 18) ||
               !map4<T>(&mVz, v, nx, ny, nz, int64_t(nt) * 6, BY, 1, 6)))
        return 1;
    const size_t smem = (size_t(78) * NTHR + 2 * (30 * size_t(HY) + 30 * size_t(HZ)) + 24 * NTHR + 6 * HY + 6 * HZ) *
                            sizeof(T) +
                        4 * sizeof(uint64_t);
    const DeviceInfo& di = device_info();
    if (smem > size_t(di.max_smem_optin)) return 1;
    auto kern = k_nn_tma64<T, FUSED, NTHR, BY, BZ>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    P64 p{};
    p.nx = nx; p.ny = ny; p.nz = nz; p.nt = nt;
    p.F = int64_t(nx) * ny * nz;
    p.BY = BY; p.BZ = BZ; p.nby = ny / BY;
    p.nblocks = int64_t(ny / BY) * (nz / BZ);
    p.t_begin = t_begin; p.t_end = t_end;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTHR, smem);
    const int G = sweep_sms() * std::max(per_sm, 1);
    p.chunk = pick_chunk(p.nblocks, t_end - t_begin, G);
    p.nitems = p.nblocks * ((t_end - t_begin + p.chunk - 1) / p.chunk);
    p.has_vhi = v_hi != nullptr;
    const int grid = static_cast<int>(std::min<int64_t>(G, p.nitems));
    kern<<<grid, NTHR, smem, st>>>(mU, mV, mVhi, mUy, mUz, mVy, mVz, U, v, out, w_lo, p);
    return check_launch("nn_sweep(tma64)");
}

template int launch_nn_tma64<double, false>(const double*, const double*, double*, int, int, int, int, int, int,
                                            const double*, const double*, cudaStream_t);
template int launch_nn_tma64<double, true>(const double*, const double*, double*, int, int, int, int, int, int,
                                           const double*, const double*, cudaStream_t);
template int launch_nn_tma64<float, false>(const float*, const float*, float*, int, int, int, int, int, int,
                                           const float*, const float*, cudaStream_t);
template int launch_nn_tma64<float, true>(const float*, const float*, float*, int, int, int, int, int, int,
                                          const float*, const float*, cudaStream_t);

}  // namespace su3g
