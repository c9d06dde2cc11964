// NN sweep, TMA-staged t-walk kernel (the production path on B200).
//
// Geometry: a CTA owns a block of one t-slice -- the full x extent (x is
// periodic inside the CTA) times BY x BZ rows -- one compute thread per
// (x, y, z) column, and walks t.  What moves where, per step t:
//
//   HBM --TMA--> smem stage:  U_mu(x,t) for the block (4 boxes of 18 planes)
//                             and v(x,t+1) (1 box of 6 planes)
//   issued by a dedicated producer warp, S stages deep (mbarrier full/empty
//   ring), so the next slice streams in while this one is computed; U is read
//   from HBM exactly once, with no per-thread address arithmetic.
//
//   compute threads:  w_mu(x) = U_mu(x)^dag v(x) for mu = x, y, z and v(x) go
//   to an exchange buffer; after one named barrier every in-block neighbour
//   term (v(x+mu), w_mu(x-mu)) is a shared-memory read.  w_t(x,t) and
//   v(x,t+1) stay in registers for step t+1: t-neighbours never leave the SM.
//   Halo rows (block edges in y/z) read through L2; the schedule keeps
//   neighbouring blocks in flight at the same time so those are L2 hits.
//
// Work = items (block, t-chunk), chunk-major, CTA c takes items c, c+G, ...;
// the chunk length is chosen on the host to balance the single wave.
// Per-site arithmetic and its order are identical to k_nn_sweep (exact IEEE,
// reference association) -> bit-identical results.
#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "sweep_common.cuh"

namespace su3g {

namespace {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

// 4-D view of a t-sliced SoA field: (x, y, z, plane), plane = t*C + c
template <typename T>
bool make_map(CUtensorMap* m, const T* base, int nx, int ny, int nz, int64_t planes, int BY, int BZ, int box_planes) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    const cuuint64_t dims[4] = {cuuint64_t(nx), cuuint64_t(ny), cuuint64_t(nz), cuuint64_t(planes)};
    const cuuint64_t strides[3] = {cuuint64_t(nx) * sizeof(T), cuuint64_t(nx) * ny * sizeof(T),
                                   cuuint64_t(nx) * ny * nz * sizeof(T)};
    const cuuint32_t box[4] = {cuuint32_t(nx), cuuint32_t(BY), cuuint32_t(BZ), cuuint32_t(box_planes)};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    CUresult r = enc(m, dt, 4, const_cast<T*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

template <int N>
__device__ __forceinline__ void named_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory");
}

struct TmaParams {
    int nx, ny, nz, nt;
    int64_t F;
    int BY, BZ, nby;
    int64_t nblocks;
    int t_begin, t_end;
    int chunk;     // t-chunk length
    int nchunks;
    int64_t nitems;
    int has_vhi;   // v(t = nt) comes from the v_hi face
};

// item -> (block, t0, t1), chunk-major
__device__ __forceinline__ void item_range(const TmaParams& p, int64_t item, int64_t& blk, int& t0, int& t1) {
    const int64_t ch = item / p.nblocks;
    blk = item - ch * p.nblocks;
    t0 = p.t_begin + static_cast<int>(ch) * p.chunk;
    t1 = min(t0 + p.chunk, p.t_end);
}

}  // namespace

template <typename T, int NTHR, int STAGES>
__global__ void __launch_bounds__(NTHR + 32, 1)
    k_nn_tma(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapV,
             const __grid_constant__ CUtensorMap mapVhi, const T* __restrict__ U, const T* __restrict__ v,
             T* __restrict__ out, const T* __restrict__ w_lo, TmaParams p) {
    constexpr int NU = 72 * NTHR;  // reals of U per stage
    constexpr int NV = 6 * NTHR;   // reals of v(t+1) per stage
    constexpr int NX = 24 * NTHR;  // exchange buffer: w_x, w_y, w_z (18) + v (6)
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* stU = reinterpret_cast<T*>(smem_raw);                 // [STAGES][72][NTHR]
    T* stV = stU + STAGES * NU;                               // [STAGES][6][NTHR]
    T* xb = stV + STAGES * NV;                                // [2][24][NTHR]
    uint64_t* full = reinterpret_cast<uint64_t*>(xb + 2 * NX);
    uint64_t* empty = full + STAGES;

    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NTHR);
        }
        fence_mbar_init();
    }
    __syncthreads();

    const int G = gridDim.x;
    const int64_t F = p.F;

    if (tid >= NTHR) {
        // ------------------------------------------------------------------
        // producer warp: one elected lane streams every step's operands
        // ------------------------------------------------------------------
        if (tid != NTHR) return;
        uint64_t pol_first, pol_normal;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_normal));
        constexpr uint32_t bytes = (72 + 6) * NTHR * sizeof(T);
        int64_t k = 0;
        for (int64_t item = blockIdx.x; item < p.nitems; item += G) {
            int64_t blk;
            int t0, t1;
            item_range(p, item, blk, t0, t1);
            const int y0 = static_cast<int>(blk % p.nby) * p.BY;
            const int z0 = static_cast<int>(blk / p.nby) * p.BZ;
            for (int t = t0; t < t1; ++t, ++k) {
                const int s = static_cast<int>(k % STAGES);
                if (k >= STAGES) mbar_wait(&empty[s], static_cast<uint32_t>(((k / STAGES) - 1) & 1));
                mbar_arrive_expect_tx(&full[s], bytes);
                T* dU = stU + s * NU;
#pragma unroll
                for (int mu = 0; mu < 4; ++mu)  // y/z links may be re-read as halos by the next block: keep them
                    tma_load_4d(dU + mu * 18 * NTHR, &mapU, 0, y0, z0, t * 72 + mu * 18, &full[s],
                                (mu == 1 || mu == 2) ? pol_normal : pol_first);
                T* dV = stV + s * NV;
                if (t + 1 < p.nt) tma_load_4d(dV, &mapV, 0, y0, z0, (t + 1) * 6, &full[s], pol_normal);
                else if (p.has_vhi) tma_load_4d(dV, &mapVhi, 0, y0, z0, 0, &full[s], pol_normal);
                else tma_load_4d(dV, &mapV, 0, y0, z0, 0, &full[s], pol_normal);
            }
        }
        return;
    }

    // ----------------------------------------------------------------------
    // compute threads
    // ----------------------------------------------------------------------
    const int nx = p.nx;
    const int lx = tid % nx;
    const int rr = tid / nx;
    const int ly = rr % p.BY;
    const int lz = rr / p.BY;
    const int sy = nx, sz = nx * p.BY;
    const int tx_up = (lx + 1 == nx) ? tid - lx : tid + 1;
    const int tx_dn = (lx == 0) ? tid + nx - 1 : tid - 1;
    const int ty_up = (ly + 1 < p.BY) ? tid + sy : (p.BY == p.ny ? tid - (p.BY - 1) * sy : -1);
    const int ty_dn = (ly > 0) ? tid - sy : (p.BY == p.ny ? tid + (p.BY - 1) * sy : -1);
    const int tz_up = (lz + 1 < p.BZ) ? tid + sz : (p.BZ == p.nz ? tid - (p.BZ - 1) * sz : -1);
    const int tz_dn = (lz > 0) ? tid - sz : (p.BZ == p.nz ? tid + (p.BZ - 1) * sz : -1);

    T vc[6], wt[6];
    int64_t k = 0;
    int b = 0;
    for (int64_t item = blockIdx.x; item < p.nitems; item += G) {
        int64_t blk;
        int t0, t1;
        item_range(p, item, blk, t0, t1);
        const int y = static_cast<int>(blk % p.nby) * p.BY + ly;
        const int z = static_cast<int>(blk / p.nby) * p.BZ + lz;
        const int64_t s3 = lx + int64_t(nx) * (y + int64_t(p.ny) * z);
        const int64_t s3_yup = lx + int64_t(nx) * ((y + 1) % p.ny + int64_t(p.ny) * z);
        const int64_t s3_ydn = lx + int64_t(nx) * ((y + p.ny - 1) % p.ny + int64_t(p.ny) * z);
        const int64_t s3_zup = lx + int64_t(nx) * (y + int64_t(p.ny) * ((z + 1) % p.nz));
        const int64_t s3_zdn = lx + int64_t(nx) * (y + int64_t(p.ny) * ((z + p.nz - 1) % p.nz));
        // prologue: v(x,t0) and the -t half-product w_t(x,t0-1)
        ld_soa<T, 6>(v + int64_t(t0) * 6 * F, F, s3, vc);
        if (t0 == 0 && w_lo != nullptr) {
            ld_soa<T, 6>(w_lo, F, s3, wt);
        } else {
            const int tp = (t0 > 0) ? t0 - 1 : p.nt - 1;
            T u[18], vp[6];
            ld_soa<T, 18>(U + (int64_t(tp) * 72 + 54) * F, F, s3, u);
            ld_soa<T, 6>(v + int64_t(tp) * 6 * F, F, s3, vp);
            adj_mat_vec<T>(u, vp, wt);
        }

        for (int t = t0; t < t1; ++t, ++k) {
            const int s = static_cast<int>(k % STAGES);
            mbar_wait(&full[s], static_cast<uint32_t>((k / STAGES) & 1));
            const T* su = stU + s * NU + tid;
            const T* sv = stV + s * NV + tid;
            T* sx = xb + b * NX;

            // stage -> registers, then hand the stage back to the producer at once
            T u[72], vnext[6];
#pragma unroll
            for (int q = 0; q < 72; ++q) u[q] = su[q * NTHR];
#pragma unroll
            for (int q = 0; q < 6; ++q) vnext[q] = sv[q * NTHR];
            mbar_arrive(&empty[s]);

            // publish w_mu(x,t) (mu = x, y, z) and v(x,t); w_t(x,t) is the -t term of step t+1
            T wt_next[6], f3[6];
#pragma unroll
            for (int mu = 0; mu < 3; ++mu) {
                T w[6];
                adj_mat_vec<T>(u + 18 * mu, vc, w);
#pragma unroll
                for (int q = 0; q < 6; ++q) sx[(6 * mu + q) * NTHR + tid] = w[q];
            }
#pragma unroll
            for (int q = 0; q < 6; ++q) sx[(18 + q) * NTHR + tid] = vc[q];
            adj_mat_vec<T>(u + 54, vc, wt_next);
            mat_vec<T>(u + 54, vnext, f3);  // forward +t term, summed last
            named_sync<NTHR>();

            // forward terms (add_su3_vector chain: ((f0 + f1) + f2) + f3)
            T acc[6];
            {
                T nb[6], f[6];
#pragma unroll
                for (int q = 0; q < 6; ++q) nb[q] = sx[(18 + q) * NTHR + tx_up];
                mat_vec<T>(u, nb, acc);
                if (ty_up >= 0) {
#pragma unroll
                    for (int q = 0; q < 6; ++q) nb[q] = sx[(18 + q) * NTHR + ty_up];
                } else {
                    ld_soa<T, 6>(v + int64_t(t) * 6 * F, F, s3_yup, nb);
                }
                mat_vec<T>(u + 18, nb, f);
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xadd(acc[q], f[q]);
                if (tz_up >= 0) {
#pragma unroll
                    for (int q = 0; q < 6; ++q) nb[q] = sx[(18 + q) * NTHR + tz_up];
                } else {
                    ld_soa<T, 6>(v + int64_t(t) * 6 * F, F, s3_zup, nb);
                }
                mat_vec<T>(u + 36, nb, f);
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xadd(acc[q], f[q]);
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xadd(acc[q], f3[q]);
            }

            // backward terms (sub_four_su3_vecs chain)
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], sx[q * NTHR + tx_dn]);
            if (ty_dn >= 0) {
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], sx[(6 + q) * NTHR + ty_dn]);
            } else {
                T uh[18], vh[6], wh[6];
                ld_soa<T, 18>(U + (int64_t(t) * 72 + 18) * F, F, s3_ydn, uh);
                ld_soa<T, 6>(v + int64_t(t) * 6 * F, F, s3_ydn, vh);
                adj_mat_vec<T>(uh, vh, wh);
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], wh[q]);
            }
            if (tz_dn >= 0) {
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], sx[(12 + q) * NTHR + tz_dn]);
            } else {
                T uh[18], vh[6], wh[6];
                ld_soa<T, 18>(U + (int64_t(t) * 72 + 36) * F, F, s3_zdn, uh);
                ld_soa<T, 6>(v + int64_t(t) * 6 * F, F, s3_zdn, vh);
                adj_mat_vec<T>(uh, vh, wh);
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], wh[q]);
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
            b ^= 1;
        }
    }
}

namespace {

// block rows (BY, BZ) with nx*BY*BZ == nthr, fewest halo rows
bool tma_shape(int nx, int ny, int nz, int nthr, int& BY, int& BZ) {
    if (nthr % nx) return false;
    const int rows = nthr / nx;
    double best = 1e30;
    bool found = false;
    for (int a = 1; a <= rows; ++a) {
        if (rows % a) continue;
        const int c = rows / a;
        if (a > ny || c > nz || ny % a || nz % c) continue;
        const double halo = (a == ny ? 0.0 : 1.0 / a) + (c == nz ? 0.0 : 1.0 / c);
        if (halo < best) {
            best = halo;
            BY = a;
            BZ = c;
            found = true;
        }
    }
    return found;
}

// chunk length that best balances the single wave of G CTAs (prologue = ~0.3 slice)
int pick_chunk(int64_t nblocks, int nt_range, int G) {
    int best_L = nt_range;
    double best_eff = -1;
    for (int L = nt_range; L >= 1; --L) {
        const int64_t nchunks = (nt_range + L - 1) / L;
        const int64_t items = nblocks * nchunks;
        const int64_t per = (items + G - 1) / G;
        const double work = double(nblocks) * nt_range;
        const double eff = work / (double(per) * G * L) * (L / (L + 0.3));
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best_L = L;
        }
    }
    return best_L;
}

}  // namespace

template <typename T, int NTHR, int STAGES>
static int run_tma(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                   const T* v_hi, const T* w_lo, int BY, int BZ, cudaStream_t st) {
    CUtensorMap mU, mV, mVhi;
    if (!make_map<T>(&mU, U, nx, ny, nz, int64_t(nt) * 72, BY, BZ, 18)) return 1;
    if (!make_map<T>(&mV, v, nx, ny, nz, int64_t(nt) * 6, BY, BZ, 6)) return 1;
    if (v_hi != nullptr) {
        if (!make_map<T>(&mVhi, v_hi, nx, ny, nz, 6, BY, BZ, 6)) return 1;
    } else {
        mVhi = mV;
    }
    constexpr size_t smem = size_t(STAGES) * (72 + 6) * NTHR * sizeof(T) + size_t(2) * 24 * NTHR * sizeof(T) +
                            2 * STAGES * sizeof(uint64_t);
    static int configured[64] = {0};
    const DeviceInfo& di = device_info();
    if (!configured[di.device & 63]) {
        cudaFuncSetAttribute(k_nn_tma<T, NTHR, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        configured[di.device & 63] = 1;
    }
    TmaParams p{};
    p.nx = nx; p.ny = ny; p.nz = nz; p.nt = nt;
    p.F = int64_t(nx) * ny * nz;
    p.BY = BY; p.BZ = BZ; p.nby = ny / BY;
    p.nblocks = int64_t(ny / BY) * (nz / BZ);
    p.t_begin = t_begin; p.t_end = t_end;
    const int G = di.num_sms;
    p.chunk = pick_chunk(p.nblocks, t_end - t_begin, G);
    p.nchunks = (t_end - t_begin + p.chunk - 1) / p.chunk;
    p.nitems = p.nblocks * p.nchunks;
    p.has_vhi = v_hi != nullptr;
    const int grid = static_cast<int>(std::min<int64_t>(G, p.nitems));
    k_nn_tma<T, NTHR, STAGES><<<grid, NTHR + 32, smem, st>>>(mU, mV, mVhi, U, v, out, w_lo, p);
    return check_launch("nn_sweep(tma)");
}

template <typename T>
int launch_nn_tma(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                  const T* v_hi, const T* w_lo, cudaStream_t st) {
    constexpr int NTHR = sizeof(T) == 4 ? 256 : 128;
    if ((nx * int(sizeof(T))) % 16 != 0 || nx > 256) return 1;
    if (!aligned16(U) || !aligned16(v) || (v_hi && !aligned16(v_hi))) return 1;
    int BY = 0, BZ = 0;
    if (!tma_shape(nx, ny, nz, NTHR, BY, BZ)) return 1;
    return run_tma<T, NTHR, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, BY, BZ, st);
}

template int launch_nn_tma<float>(const float*, const float*, float*, int, int, int, int, int, int, const float*,
                                  const float*, cudaStream_t);
template int launch_nn_tma<double>(const double*, const double*, double*, int, int, int, int, int, int,
                                   const double*, const double*, cudaStream_t);

}  // namespace su3g
