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

// exchange buffer geometry (per buffer, runtime halo widths HY = nx*BZ, HZ = nx*BY):
//   WX [6][N]           w_x of the block's sites
//   WY [6][N + HY]      w_y, plus the -y halo row
//   WZ [6][N + HZ]      w_z, plus the -z halo row
//   VV [6][N + HY + HZ] v(x,t), plus the +y and +z halo rows
struct XLayout {
    int N, HY, HZ;
    __device__ __forceinline__ int wx() const { return 0; }
    __device__ __forceinline__ int wy() const { return 6 * N; }
    __device__ __forceinline__ int wz() const { return 6 * N + 6 * (N + HY); }
    __device__ __forceinline__ int vv() const { return 6 * N + 6 * (N + HY) + 6 * (N + HZ); }
    __device__ __forceinline__ int py() const { return N + HY; }
    __device__ __forceinline__ int pz() const { return N + HZ; }
    __device__ __forceinline__ int pv() const { return N + HY + HZ; }
    __device__ __forceinline__ int size() const { return vv() + 6 * (N + HY + HZ); }
};

template <typename T, int NTHR, int NHALO, int STAGES>
__global__ void __launch_bounds__(NTHR + 32 + NHALO, 1)
    k_nn_tma(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapV,
             const __grid_constant__ CUtensorMap mapVhi, const T* __restrict__ U, const T* __restrict__ v,
             T* __restrict__ out, const T* __restrict__ w_lo, TmaParams p) {
    constexpr int NU = 54 * NTHR;  // U_x, U_y, U_z of the block per stage (U_t goes straight to registers)
    constexpr int NV = 6 * NTHR;   // v(t+1) of the block per stage
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* stU = reinterpret_cast<T*>(smem_raw);  // [STAGES][54][NTHR]
    T* stV = stU + STAGES * NU;                // [STAGES][6][NTHR]
    T* xb = stV + STAGES * NV;                 // [2][XLayout]
    const int nx = p.nx;
    const XLayout L{NTHR, p.BY == p.ny ? 0 : nx * p.BZ, p.BZ == p.nz ? 0 : nx * p.BY};
    const int XS = L.size();
    uint64_t* full = reinterpret_cast<uint64_t*>(xb + 2 * XS);
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

    if (tid >= NTHR + 32) {
        // ------------------------------------------------------------------
        // halo warps: the -y/-z half-products and +y/+z vectors of the rows just
        // outside the block, from L2 (the neighbouring blocks are streamed by
        // other CTAs at the same time), straight into the exchange buffer.
        // ------------------------------------------------------------------
        const int h = tid - NTHR - 32;
        int b = 0;
        for (int64_t item = blockIdx.x; item < p.nitems; item += G) {
            int64_t blk;
            int t0, t1;
            item_range(p, item, blk, t0, t1);
            const int y0 = static_cast<int>(blk % p.nby) * p.BY;
            const int z0 = static_cast<int>(blk / p.nby) * p.BZ;
            for (int t = t0; t < t1; ++t) {
                T* sx = xb + b * XS;
                const T* Ut = U + int64_t(t) * 72 * F;
                const T* vt = v + int64_t(t) * 6 * F;
                for (int j = h; j < L.HY + L.HZ; j += NHALO) {
                    int64_t dn, up;
                    int mu, wbase, wpitch, vslot;
                    if (j < L.HY) {
                        const int lx = j % nx, lz = j / nx;
                        const int64_t zr = int64_t(p.ny) * (z0 + lz);
                        dn = lx + int64_t(nx) * ((y0 + p.ny - 1) % p.ny + zr);
                        up = lx + int64_t(nx) * ((y0 + p.BY) % p.ny + zr);
                        mu = 1; wbase = L.wy(); wpitch = L.py(); vslot = NTHR + j;
                    } else {
                        const int jj = j - L.HY, lx = jj % nx, ly = jj / nx;
                        dn = lx + int64_t(nx) * (y0 + ly + int64_t(p.ny) * ((z0 + p.nz - 1) % p.nz));
                        up = lx + int64_t(nx) * (y0 + ly + int64_t(p.ny) * ((z0 + p.BZ) % p.nz));
                        mu = 2; wbase = L.wz(); wpitch = L.pz(); vslot = NTHR + L.HY + jj;
                    }
                    T uh[18], vh[6], vu[6], wh[6];
                    ld_soa<T, 18>(Ut + int64_t(mu) * 18 * F, F, dn, uh);
                    ld_soa<T, 6>(vt, F, dn, vh);
                    ld_soa<T, 6>(vt, F, up, vu);
                    adj_mat_vec<T>(uh, vh, wh);
                    const int slot = NTHR + (j < L.HY ? j : j - L.HY);
#pragma unroll
                    for (int q = 0; q < 6; ++q) {
                        sx[wbase + q * wpitch + slot] = wh[q];
                        sx[L.vv() + q * L.pv() + vslot] = vu[q];
                    }
                }
                named_sync<NTHR + NHALO>();
                b ^= 1;
            }
        }
        return;
    }

    if (tid >= NTHR) {
        // ------------------------------------------------------------------
        // producer warp: one elected lane streams every step's operands by TMA
        // ------------------------------------------------------------------
        if (tid != NTHR) return;
        uint64_t pol_first, pol_normal;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_normal));
        constexpr uint32_t bytes = (54 + 6) * NTHR * sizeof(T);
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
                // U_y / U_z rows are re-read as halos by neighbouring blocks: normal priority
                tma_load_4d(dU, &mapU, 0, y0, z0, t * 72, &full[s], pol_first);
                tma_load_4d(dU + 18 * NTHR, &mapU, 0, y0, z0, t * 72 + 18, &full[s], pol_normal);
                tma_load_4d(dU + 36 * NTHR, &mapU, 0, y0, z0, t * 72 + 36, &full[s], pol_normal);
                T* dV = stV + s * NV;
                if (t + 1 < p.nt) tma_load_4d(dV, &mapV, 0, y0, z0, (t + 1) * 6, &full[s], pol_normal);
                else if (p.has_vhi) tma_load_4d(dV, &mapVhi, 0, y0, z0, 0, &full[s], pol_normal);
                else tma_load_4d(dV, &mapV, 0, y0, z0, 0, &full[s], pol_normal);
            }
        }
        return;
    }

    // ----------------------------------------------------------------------
    // compute threads: one site each
    // ----------------------------------------------------------------------
    const int lx = tid % nx;
    const int rr = tid / nx;
    const int ly = rr % p.BY;
    const int lz = rr / p.BY;
    const int sy = nx, sz = nx * p.BY;
    const int ix_up = (lx + 1 == nx) ? tid - lx : tid + 1;
    const int ix_dn = (lx == 0) ? tid + nx - 1 : tid - 1;
    const int iy_up = (ly + 1 < p.BY) ? tid + sy : (L.HY == 0 ? tid - (p.BY - 1) * sy : NTHR + lx + nx * lz);
    const int iy_dn = (ly > 0) ? tid - sy : (L.HY == 0 ? tid + (p.BY - 1) * sy : NTHR + lx + nx * lz);
    const int iz_up = (lz + 1 < p.BZ) ? tid + sz : (L.HZ == 0 ? tid - (p.BZ - 1) * sz : NTHR + L.HY + lx + nx * ly);
    const int iz_dn = (lz > 0) ? tid - sz : (L.HZ == 0 ? tid + (p.BZ - 1) * sz : NTHR + lx + nx * ly);

    auto site_of = [&](int64_t blk) {
        const int y = static_cast<int>(blk % p.nby) * p.BY + ly;
        const int z = static_cast<int>(blk / p.nby) * p.BZ + lz;
        return lx + int64_t(nx) * (y + int64_t(p.ny) * z);
    };

    T vc[6], wt[6], ut[18];
    int64_t k = 0;
    int b = 0;
    int64_t item = blockIdx.x;
    int64_t blk = 0;
    int t0 = 0, t1 = 0;
    if (item < p.nitems) {
        item_range(p, item, blk, t0, t1);
        ld_soa<T, 18>(U + (int64_t(t0) * 72 + 54) * F, F, site_of(blk), ut);  // U_t of the first step
    }
    for (; item < p.nitems; item += G) {
        if (k > 0) item_range(p, item, blk, t0, t1);
        const int64_t s3 = site_of(blk);
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
            // prefetch U_t of the next step (this item's t+1, or the next item's first slice)
            T ut_next[18];
            {
                int64_t nb_blk = blk;
                int nt_ = t + 1;
                if (nt_ >= t1 && item + G < p.nitems) {
                    int a0, a1;
                    item_range(p, item + G, nb_blk, a0, a1);
                    nt_ = a0;
                }
                if (nt_ < p.nt && (nt_ < t1 || item + G < p.nitems))
                    ld_soa<T, 18>(U + (int64_t(nt_) * 72 + 54) * F, F, site_of(nb_blk), ut_next);
            }
            const int s = static_cast<int>(k % STAGES);
            mbar_wait(&full[s], static_cast<uint32_t>((k / STAGES) & 1));
            const T* su = stU + s * NU + tid;
            const T* sv = stV + s * NV + tid;
            T* sx = xb + b * XS;

            // stage -> registers, then hand the stage back to the producer at once
            T u[54], vnext[6];
#pragma unroll
            for (int q = 0; q < 54; ++q) u[q] = su[q * NTHR];
#pragma unroll
            for (int q = 0; q < 6; ++q) vnext[q] = sv[q * NTHR];
            mbar_arrive(&empty[s]);

            // publish w_mu(x,t) (mu = x, y, z) and v(x,t); w_t(x,t) is the -t term of step t+1
            {
                T w[6];
                adj_mat_vec<T>(u, vc, w);
#pragma unroll
                for (int q = 0; q < 6; ++q) sx[L.wx() + q * NTHR + tid] = w[q];
                adj_mat_vec<T>(u + 18, vc, w);
#pragma unroll
                for (int q = 0; q < 6; ++q) sx[L.wy() + q * L.py() + tid] = w[q];
                adj_mat_vec<T>(u + 36, vc, w);
#pragma unroll
                for (int q = 0; q < 6; ++q) sx[L.wz() + q * L.pz() + tid] = w[q];
#pragma unroll
                for (int q = 0; q < 6; ++q) sx[L.vv() + q * L.pv() + tid] = vc[q];
            }
            T wt_next[6], f3[6];
            adj_mat_vec<T>(ut, vc, wt_next);
            mat_vec<T>(ut, vnext, f3);  // forward +t term, summed last
            named_sync<NTHR + NHALO>();

            // forward terms (add_su3_vector chain: ((f0 + f1) + f2) + f3)
            T acc[6];
            {
                T nb[6], f[6];
#pragma unroll
                for (int q = 0; q < 6; ++q) nb[q] = sx[L.vv() + q * L.pv() + ix_up];
                mat_vec<T>(u, nb, acc);
#pragma unroll
                for (int q = 0; q < 6; ++q) nb[q] = sx[L.vv() + q * L.pv() + iy_up];
                mat_vec<T>(u + 18, nb, f);
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xadd(acc[q], f[q]);
#pragma unroll
                for (int q = 0; q < 6; ++q) nb[q] = sx[L.vv() + q * L.pv() + iz_up];
                mat_vec<T>(u + 36, nb, f);
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xadd(acc[q], f[q]);
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xadd(acc[q], f3[q]);
            }
            // backward terms (sub_four_su3_vecs chain)
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], sx[L.wx() + q * NTHR + ix_dn]);
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], sx[L.wy() + q * L.py() + iy_dn]);
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], sx[L.wz() + q * L.pz() + iz_dn]);
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
#pragma unroll
            for (int q = 0; q < 18; ++q) ut[q] = ut_next[q];
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

template <typename T, int NTHR, int NHALO, int STAGES>
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
    const int HY = (BY == ny) ? 0 : nx * BZ, HZ = (BZ == nz) ? 0 : nx * BY;
    const size_t xs = size_t(6) * (4 * NTHR + 2 * HY + 2 * HZ);
    const size_t smem = size_t(STAGES) * (54 + 6) * NTHR * sizeof(T) + 2 * xs * sizeof(T) + 2 * STAGES * sizeof(uint64_t);
    const DeviceInfo& di = device_info();
    if (smem > size_t(di.max_smem_optin)) return 1;
    static int configured[64] = {0};
    if (!configured[di.device & 63]) {
        const size_t worst = size_t(STAGES) * (54 + 6) * NTHR * sizeof(T) + 2 * size_t(6) * (8 * NTHR) * sizeof(T) +
                             2 * STAGES * sizeof(uint64_t);
        cudaFuncSetAttribute(k_nn_tma<T, NTHR, NHALO, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(std::min<size_t>(worst, size_t(di.max_smem_optin))));
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
    k_nn_tma<T, NTHR, NHALO, STAGES><<<grid, NTHR + 32 + NHALO, smem, st>>>(mU, mV, mVhi, U, v, out, w_lo, p);
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
    return run_tma<T, NTHR, 64, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, BY, BZ, st);
}

template int launch_nn_tma<float>(const float*, const float*, float*, int, int, int, int, int, int, const float*,
                                  const float*, cudaStream_t);
template int launch_nn_tma<double>(const double*, const double*, double*, int, int, int, int, int, int,
                                   const double*, const double*, cudaStream_t);

}  // namespace su3g
