// NN sweep, warp-specialised TMA ring t-walk (the production path on B200, f32 and f64).
//
// Why a second t-walk kernel: the f32 walk (nn_tma.cu) stages a whole step -- the block's
// links, v(t+1) and the halo rows -- per ring stage; at f64 two such stages plus the
// exchange buffer do not fit 227 KB.  This kernel moves the same bytes through a ring of
// small, equal-sized slots, one per "chunk" of a step, so the ring is as deep as shared
// memory allows at any precision:
//
//   chunk 0  H1  v(x,t+1) of the block [6][N] | v on the +y halo row [6][H] | U_y on the -y row [18][H]
//   chunk 1  H2  v on the -y row [6][H] | U_z on the -z row [18][H] | v on the -z row [6][H] | v +z [6][H]
//   chunk 2-5    U_x, U_y, U_z, U_t of the block [18][N] each
//
// (block = NX x 2 x 2 sites, N = 4 NX compute threads, halo rows H = 2 NX = N/2 sites, so every
// chunk is exactly 18 N reals).  One producer warp issues the 4-D TMA boxes into the ring
// (full/empty mbarrier pairs); each compute warp releases a slot as soon as its lanes have
// copied what they need into registers.  Links are never shared between sites, so a slot
// lives only for the few hundred cycles it takes to read it, and the bytes in flight are the
// whole ring minus one slot.
//
// Per step (site x of the block, slice t): the halo rows' backward half-products
// w = U^dag v go to the exchange (XH, one halo site per thread); w_x, w_y, w_z of every
// site go to XW; v(x,t+1) goes to the double-buffered XV, from which the next step reads
// its in-block forward neighbours.  The -t term w_t and v(t+1) stay in registers.  Two
// named barriers per step (XW / XH are single-buffered).  Work items (block, t-chunk) are
// ordered chunk-major over one persistent wave, as in nn_tma.cu.
//
// The per-site arithmetic and its order are those of nn_site (the composed reference,
// SURVEY.md 8(c)): bit-identical results in exact mode.
#include <algorithm>
#include <string>

#include "nn_site.cuh"
#include "tma.cuh"

namespace su3g {

int g_ring_columns = 1;  // su3g_set_option("nn_ring_columns"): the columns schedule of the ring walks' work items (A/B)

namespace {

struct RingParams {
    int ny, nz, nt;
    int64_t F;
    int nby;         // ny / 2
    int64_t nblocks;
    int t_begin, t_end;
    int chunk;       // t-chunk length of one work item
    int64_t nitems;  // nblocks * ceil((t_end - t_begin) / chunk), chunk-major; EDGES: nblocks * (boundary slices)
    int64_t n_full;  // columns schedule: the first n_full items are whole [t_begin, t_end) columns of blocks
                     // 0..n_full-1, the other blocks are cut into t-chunks, chunk-major (0: every block is)
    int has_vhi;
    void* w_next;    // EDGES: w = U_t^dag out on slice nt-1 (the next application's halo), or null
};

template <int NX>
struct RingGeo {
    static constexpr int N = 4 * NX;  // block sites = compute threads
    static constexpr int H = 2 * NX;  // sites of one halo row (y or z)
    static constexpr int SLOT = 18 * N;
    // H1
    static constexpr int H1_V = 0, H1_VYU = 6 * N, H1_UYD = 6 * N + 6 * H;
    // H2
    static constexpr int H2_VYD = 0, H2_UZD = 6 * H, H2_VZD = 24 * H, H2_VZU = 30 * H;
};

// exchange buffers; DB = XW / XH double-buffered (one barrier per step instead of two)
template <int NX, bool DB>
struct RingX {
    static constexpr int N = 4 * NX, H = 2 * NX;
    static constexpr int NB = DB ? 2 : 1;
    static constexpr int XW = 0;                    // [NB][18][N]
    static constexpr int XH = NB * 18 * N;          // [NB][6][2H]: -y halo sites, then -z halo sites
    static constexpr int XV = NB * (18 * N + 12 * H);  // [2][6][N]
    static constexpr int XSIZE = XV + 12 * N;
    static constexpr int WSTRIDE = 18 * N, HSTRIDE = 12 * H;  // per buffer
};

template <bool EDGES = false>
__device__ __forceinline__ void item_of(const RingParams& p, int64_t item, int64_t& blk, int& t0, int& t1) {
    if constexpr (EDGES) {  // the boundary slices of a t-slab: t = 0 for every block, then t = nt - 1
        const int64_t ch = item / p.nblocks;
        blk = item - ch * p.nblocks;
        t0 = ch == 0 ? 0 : p.nt - 1;
        t1 = t0 + 1;
    } else {
        schedule_item(p.n_full, p.nblocks, p.chunk, p.t_begin, p.t_end, item, blk, t0, t1);
    }
}

}  // namespace

template <typename T, bool FUSED, int NX, int S, bool DB, int MINB, bool EDGES>
__global__ void __launch_bounds__(4 * NX + 32, MINB)
    k_nn_ring(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapV,
              const __grid_constant__ CUtensorMap mapVhi, const __grid_constant__ CUtensorMap mapUyH,
              const __grid_constant__ CUtensorMap mapUzH, const __grid_constant__ CUtensorMap mapVyH,
              const __grid_constant__ CUtensorMap mapVzH, const T* __restrict__ U, const T* __restrict__ v,
              T* __restrict__ out, const T* __restrict__ w_lo, RingParams p) {
    using G = RingGeo<NX>;
    using X = RingX<NX, DB>;
    constexpr int N = G::N, H = G::H, NW = N / 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* ring = reinterpret_cast<T*>(smem_raw);
    T* xb = ring + S * G::SLOT;
    uint64_t* full = reinterpret_cast<uint64_t*>(xb + X::XSIZE);
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
    const int G_ = gridDim.x;

    // ------------------------------------------------------------------ producer warp
    if (tid >= N) {
        if (tid != N) return;
        uint64_t pol_first, pol_normal;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_normal));
        uint32_t q = 0;
        for (int64_t item = blockIdx.x; item < p.nitems; item += G_) {
            int64_t blk;
            int t0, t1;
            item_of<EDGES>(p, item, blk, t0, t1);
            const int y0 = static_cast<int>(blk % p.nby) * 2, z0 = static_cast<int>(blk / p.nby) * 2;
            const int ydn = (y0 + p.ny - 1) % p.ny, yup = (y0 + 2) % p.ny;
            const int zdn = (z0 + p.nz - 1) % p.nz, zup = (z0 + 2) % p.nz;
            if constexpr (EDGES) {  // one-step items: warm L2 with the NEXT item's prologue operands
                if (item + G_ < p.nitems) {
                    int64_t nb;
                    int n0, n1;
                    item_of<EDGES>(p, item + G_, nb, n0, n1);
                    const int ny0 = static_cast<int>(nb % p.nby) * 2, nz0 = static_cast<int>(nb / p.nby) * 2;
                    tma_prefetch(&mapV, 0, ny0, nz0, n0 * 6);  // v(t0)
                    if (n0 > 0) {                              // w_t(t0-1) = U_t(t0-1)^dag v(t0-1)
                        tma_prefetch(&mapV, 0, ny0, nz0, (n0 - 1) * 6);
                        tma_prefetch(&mapU, 0, ny0, nz0, (n0 - 1) * 72 + 54);
                    }
                }
            }
            for (int t = t0; t < t1; ++t) {
#pragma unroll 1
                for (int c = 0; c < 6; ++c, ++q) {
                    const int s = static_cast<int>(q % S);
                    if (q >= S) mbar_wait(&empty[s], ((q / S) + 1) & 1);
                    T* dst = ring + s * G::SLOT;
                    mbar_arrive_expect_tx(&full[s], uint32_t(G::SLOT) * sizeof(T));
                    if (c == 0) {
                        if (t + 1 < p.nt) tma_load_4d(dst + G::H1_V, &mapV, 0, y0, z0, (t + 1) * 6, &full[s], pol_normal);
                        else if (p.has_vhi) tma_load_4d(dst + G::H1_V, &mapVhi, 0, y0, z0, 0, &full[s], pol_normal);
                        else tma_load_4d(dst + G::H1_V, &mapV, 0, y0, z0, 0, &full[s], pol_normal);
                        tma_load_4d(dst + G::H1_VYU, &mapVyH, 0, yup, z0, t * 6, &full[s], pol_normal);
                        tma_load_4d(dst + G::H1_UYD, &mapUyH, 0, ydn, z0, t * 72 + 18, &full[s], pol_normal);
                    } else if (c == 1) {
                        tma_load_4d(dst + G::H2_VYD, &mapVyH, 0, ydn, z0, t * 6, &full[s], pol_normal);
                        tma_load_4d(dst + G::H2_UZD, &mapUzH, 0, y0, zdn, t * 72 + 36, &full[s], pol_normal);
                        tma_load_4d(dst + G::H2_VZD, &mapVzH, 0, y0, zdn, t * 6, &full[s], pol_normal);
                        tma_load_4d(dst + G::H2_VZU, &mapVzH, 0, y0, zup, t * 6, &full[s], pol_normal);
                    } else {
                        // U_x and U_t are read exactly once; U_y / U_z are re-read as halo rows by
                        // the neighbouring blocks in flight at the same time
                        const int mu = c - 2;
                        tma_load_4d(dst, &mapU, 0, y0, z0, t * 72 + 18 * mu, &full[s],
                                    (mu == 1 || mu == 2) ? pol_normal : pol_first);
                    }
                }
            }
        }
        return;
    }

    // ------------------------------------------------------------------ compute warps
    const int lane = tid & 31;
    const int lx = tid % NX, ly = (tid / NX) & 1, lz = tid / (2 * NX);
    const int ix_up = (lx + 1 == NX) ? tid - lx : tid + 1;
    const int ix_dn = (lx == 0) ? tid + NX - 1 : tid - 1;
    const int jy = lx + NX * lz;  // this column's slot in a y halo row (box x, z)
    const int jz = lx + NX * ly;  // ... in a z halo row (box x, y)
    T* const XW0 = xb + X::XW;
    T* const XH0 = xb + X::XH;
    T* XV = xb + X::XV;

    uint32_t q = 0;
    uint32_t k = 0;  // steps done by this CTA (XV parity)
    for (int64_t item = blockIdx.x; item < p.nitems; item += G_) {
        int64_t blk;
        int t0, t1;
        item_of<EDGES>(p, item, blk, t0, t1);
        const int y = static_cast<int>(blk % p.nby) * 2 + ly;
        const int z = static_cast<int>(blk / p.nby) * 2 + lz;
        const int64_t s3 = lx + int64_t(NX) * (y + int64_t(p.ny) * z);
        // prologue: v(x,t0) and the -t half-product w_t(x,t0-1)
        T vc[6], wt[6];
        ld_soa<T, 6>(v + int64_t(t0) * 6 * F, F, s3, vc);
        if (t0 == 0 && w_lo != nullptr) {
            ld_soa<T, 6>(w_lo, F, s3, wt);
        } else {
            const int tp = (t0 > 0) ? t0 - 1 : p.nt - 1;
            T u[18], vp[6];
            ld_soa<T, 18>(U + (int64_t(tp) * 72 + 54) * F, F, s3, u);
            ld_soa<T, 6>(v + int64_t(tp) * 6 * F, F, s3, vp);
            amv<T, FUSED>(u, vp, wt);
        }
#pragma unroll
        for (int c = 0; c < 6; ++c) XV[((k & 1) * 6 + c) * N + tid] = vc[c];
        named_sync<N>();

        for (int t = t0; t < t1; ++t, ++k) {
            const T* xv = XV + (k & 1) * 6 * N;
            T* XW = XW0 + (DB ? (k & 1) * X::WSTRIDE : 0);
            T* XH = XH0 + (DB ? (k & 1) * X::HSTRIDE : 0);
            T vnext[6], nby_[6], nbz_[6];
            // ---- H1, H2: v(t+1), the +y / +z halo v this column needs, the halo half-products
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
                if (tid < H) {  // -y halo site tid
#pragma unroll
                    for (int c = 0; c < 18; ++c) uh[c] = h1[G::H1_UYD + c * H + tid];
#pragma unroll
                    for (int c = 0; c < 6; ++c) vh[c] = h2[G::H2_VYD + c * H + tid];
                } else {        // -z halo site tid - H
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
            // ---- U_x, U_y, U_z: publish w_mu, forward term U_mu(x) v(x+mu)
            T acc[6];
#pragma unroll
            for (int mu = 0; mu < 3; ++mu) {
                const uint32_t qq = q + 2 + mu;
                const int s = static_cast<int>(qq % S);
                mbar_wait(&full[s], (qq / S) & 1);
                const T* su = ring + s * G::SLOT;
                T u[18];
#pragma unroll
                for (int c = 0; c < 18; ++c) u[c] = su[c * N + tid];
                warp_release(&empty[s], lane);
                T w[6], nb[6], f[6];
                amv<T, FUSED>(u, vc, w);
#pragma unroll
                for (int c = 0; c < 6; ++c) XW[(6 * mu + c) * N + tid] = w[c];
                const int src = mu == 0 ? ix_up : (mu == 1 ? (ly == 0 ? tid + NX : -1) : (lz == 0 ? tid + 2 * NX : -1));
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
            // ---- U_t: -t term of the next step, forward +t term (summed last)
            T wt_next[6];
            T ut_keep[EDGES ? 18 : 1];
            {
                const uint32_t qq = q + 5;
                const int s = static_cast<int>(qq % S);
                mbar_wait(&full[s], (qq / S) & 1);
                const T* su = ring + s * G::SLOT;
                T u[18], f[6];
#pragma unroll
                for (int c = 0; c < 18; ++c) u[c] = su[c * N + tid];
                warp_release(&empty[s], lane);
                amv<T, FUSED>(u, vc, wt_next);
                mv<T, FUSED>(u, vnext, f);
#pragma unroll
                for (int c = 0; c < 6; ++c) acc[c] = xadd(acc[c], f[c]);
                if constexpr (EDGES) {
#pragma unroll
                    for (int c = 0; c < 18; ++c) ut_keep[c] = u[c];
                }
            }
            q += 6;
#pragma unroll
            for (int c = 0; c < 6; ++c) XV[(((k + 1) & 1) * 6 + c) * N + tid] = vnext[c];
            named_sync<N>();

            // ---- backward terms (sub_four_su3_vecs chain)
#pragma unroll
            for (int c = 0; c < 6; ++c) acc[c] = xsub(acc[c], XW[c * N + ix_dn]);
            {
                const T* b = ly == 1 ? XW + 6 * N + tid - NX : XH + jy;
                const int bs = ly == 1 ? N : 2 * H;
#pragma unroll
                for (int c = 0; c < 6; ++c) acc[c] = xsub(acc[c], b[c * bs]);
                b = lz == 1 ? XW + 12 * N + tid - 2 * NX : XH + H + jz;
#pragma unroll
                for (int c = 0; c < 6; ++c) acc[c] = xsub(acc[c], b[c * bs]);
            }
#pragma unroll
            for (int c = 0; c < 6; ++c) acc[c] = xsub(acc[c], wt[c]);
            T* o = out + int64_t(t) * 6 * F + s3;
#pragma unroll
            for (int c = 0; c < 6; ++c) __stcs(o + c * F, acc[c]);
            if constexpr (EDGES) {  // the next application's +t halo: U_t^dag out, nn_halo_w's arithmetic
                if (p.w_next != nullptr && t == p.nt - 1) {
                    T w[6];
                    amv<T, FUSED>(ut_keep, acc, w);
                    T* wn = static_cast<T*>(p.w_next) + s3;
#pragma unroll
                    for (int c = 0; c < 6; ++c) wn[c * F] = w[c];
                }
            }
#pragma unroll
            for (int c = 0; c < 6; ++c) {
                vc[c] = vnext[c];
                wt[c] = wt_next[c];
            }
            // single-buffered XW / XH are rewritten by the next step; double-buffered ones only by the
            // step after, whose writers have all passed the next step's barrier (after this read)
            if constexpr (!DB) named_sync<N>();
        }
    }
}

template <typename T, bool FUSED, int NX, int S, bool DB, int MINB, bool EDGES = false>
static int run_ring(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                    const T* v_hi, const T* w_lo, cudaStream_t st, T* w_next = nullptr) {
    using G = RingGeo<NX>;
    using X = RingX<NX, DB>;
    CUtensorMap mU, mV, mVhi, mUy, mUz, mVy, mVz;
    if (!make_map<T>(&mU, U, nx, ny, nz, int64_t(nt) * 72, 2, 2, 18)) return 1;
    if (!make_map<T>(&mV, v, nx, ny, nz, int64_t(nt) * 6, 2, 2, 6)) return 1;
    if (v_hi != nullptr) {
        if (!make_map<T>(&mVhi, v_hi, nx, ny, nz, 6, 2, 2, 6)) return 1;
    } else {
        mVhi = mV;
    }
    if (!make_map<T>(&mUy, U, nx, ny, nz, int64_t(nt) * 72, 1, 2, 18) ||
        !make_map<T>(&mVy, v, nx, ny, nz, int64_t(nt) * 6, 1, 2, 6) ||
        !make_map<T>(&mUz, U, nx, ny, nz, int64_t(nt) * 72, 2, 1, 18) ||
        !make_map<T>(&mVz, v, nx, ny, nz, int64_t(nt) * 6, 2, 1, 6))
        return 1;
    const size_t smem = (size_t(S) * G::SLOT + X::XSIZE) * sizeof(T) + 2 * S * sizeof(uint64_t);
    const DeviceInfo& di = device_info();
    if (smem > size_t(di.max_smem_optin)) return 1;
    auto kern = k_nn_ring<T, FUSED, NX, S, DB, MINB, EDGES>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    RingParams p{};
    p.ny = ny; p.nz = nz; p.nt = nt;
    p.F = int64_t(nx) * ny * nz;
    p.nby = ny / 2;
    p.nblocks = int64_t(ny / 2) * (nz / 2);
    p.t_begin = t_begin; p.t_end = t_end;
    p.has_vhi = v_hi != nullptr;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::N + 32, smem);
    const int per = std::max(per_sm, 1);
    const int G_full = di.num_sms * per;
    const int L = t_end - t_begin;
    // a ring work item's prologue (v(t0) and w_t(t0-1) from global) costs about half a step: same-box
    // A/B of the chunk picker's cost (profiles/r02/ab_nn_ring_prologue.txt): 32^4 f32 0.799 / f64 0.754
    // at 0.5 against 0.785 / 0.724 at the walk kernels' 2.0; 64^3x16 and 64^3x128 unchanged
    // columns schedule (sweep_common.cuh): only with the full grid (no SMs reserved for NCCL: the round
    // structure depends on the grid)
    const WalkSchedule ws = pick_schedule(p.nblocks, L, G_full, 0.5, !EDGES && g_ring_columns && sm_reserve() == 0);
    p.n_full = ws.n_full;
    p.chunk = ws.chunk;
    p.nitems = ws.nitems;
    p.w_next = w_next;
    if constexpr (EDGES) p.nitems = p.nblocks * (nt > 1 ? 2 : 1);
    int Gr = G_full;
    if (sm_reserve() > 0) {  // as nn_tma.cu: leave SMs for NCCL only where the last round absorbs it
        const int64_t rounds = (p.nitems + G_full - 1) / G_full;
        const int64_t g_same = (p.nitems + rounds - 1) / rounds;
        const int g_res = std::max(per, sweep_sms() * per);
        if (g_same <= G_full - per) Gr = static_cast<int>(std::max<int64_t>(g_res, g_same));
    }
    const int grid = static_cast<int>(std::min<int64_t>(Gr, p.nitems));
    kern<<<grid, G::N + 32, smem, st>>>(mU, mV, mVhi, mUy, mUz, mVy, mVz, U, v, out, w_lo, p);
    note_kernel(std::string("k_nn_ring<") + (sizeof(T) == 4 ? "f32," : "f64,") + std::to_string(NX) + "x2x2," +
                std::to_string(S) + " slots" + (DB ? ",1 barrier" : "") + (per > 1 ? "," + std::to_string(per) + " CTAs/SM" : "") +
                (EDGES ? ",edges" : "") + (p.n_full ? "," + std::to_string(p.n_full) + " columns" : "") + ">" + (grid < G_full ? " grid " + std::to_string(grid) : std::string()));
    return check_launch("nn_sweep(ring)");
}

int g_ring_cfg = 0;  // su3g_set_option("nn_ring_cfg"): ring slot / CTA configuration (A/B), 0 = default

template <typename T, bool FUSED, int NX>
static int ring_dispatch(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                         const T* v_hi, const T* w_lo, cudaStream_t st) {
    if constexpr (sizeof(T) == 8) {  // f64: four slots next to the single-buffered exchange
        if (g_ring_cfg == 1 || (g_ring_cfg == 0 && NX == 32))  // 32-wide blocks: two CTAs per SM
            return run_ring<T, FUSED, NX, 4, false, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st);
        return run_ring<T, FUSED, NX, 4, false, 1>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st);
    } else {
        // 32-wide blocks (N = 128): four CTAs per SM at <= 96 registers (32^4: 0.843 vs 0.791 with three)
        if (NX == 32 && g_ring_cfg == 0)
            return run_ring<T, FUSED, NX, 4, false, 4>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st);
        // f32: two CTAs per SM, four 18-KB slots each (same-box A/B at 64^3x16, fraction of HBM:
        // 0.905 vs 0.840 for one CTA with eight slots, 0.812 one CTA with six slots and a double-
        // buffered exchange, 0.716 two CTAs with two slots each; the f32 TMA walk 0.835)
        switch (g_ring_cfg) {
            case 1: return run_ring<T, FUSED, NX, 8, false, 1>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st);
            case 2: return run_ring<T, FUSED, NX, 6, true, 1>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st);
            case 3: return run_ring<T, FUSED, NX, 2, true, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st);
            case 4: return run_ring<T, FUSED, NX, 4, false, 4>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st);
            default: return run_ring<T, FUSED, NX, 4, false, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st);
        }
    }
}

// 1 = not applicable to this lattice (caller falls back)
template <typename T>
int launch_nn_ring(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                   const T* v_hi, const T* w_lo, int mode, cudaStream_t st) {
    if (ny % 2 || nz % 2) return 1;
    if (!aligned16(U) || !aligned16(v) || (v_hi && !aligned16(v_hi))) return 1;
    const bool fma = mode == SU3G_FMA;
    if (nx == 64)
        return fma ? ring_dispatch<T, true, 64>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st)
                   : ring_dispatch<T, false, 64>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st);
    if (nx == 32)
        return fma ? ring_dispatch<T, true, 32>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st)
                   : ring_dispatch<T, false, 32>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st);
    if (nx == 48)
        return fma ? ring_dispatch<T, true, 48>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st)
                   : ring_dispatch<T, false, 48>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st);
    return 1;
}

// Both boundary slices of a t-slab (t = 0 with w_lo, t = nt-1 with v_hi) as one-step work items of the
// ring walk, and w_next = U_t^dag out on slice nt-1 (the next application's halo).  1 = not applicable.
template <typename T>
int launch_nn_ring_edges(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, const T* v_hi, const T* w_lo,
                         T* w_next, int mode, cudaStream_t st) {
    if (ny % 2 || nz % 2 || nt < 3) return 1;
    if (!aligned16(U) || !aligned16(v) || (v_hi && !aligned16(v_hi))) return 1;
    const bool fma = mode == SU3G_FMA;
    constexpr int MB = sizeof(T) == 4 ? 2 : 1;
#define SU3G_EDGES(NXV)                                                                                           \
    return fma ? run_ring<T, true, NXV, 4, false, MB, true>(U, v, out, nx, ny, nz, nt, 0, nt, v_hi, w_lo, st, w_next) \
               : run_ring<T, false, NXV, 4, false, MB, true>(U, v, out, nx, ny, nz, nt, 0, nt, v_hi, w_lo, st, w_next)
    if (nx == 64) SU3G_EDGES(64);
    if (nx == 32) SU3G_EDGES(32);
    if (nx == 48) SU3G_EDGES(48);
#undef SU3G_EDGES
    return 1;
}

template int launch_nn_ring_edges<float>(const float*, const float*, float*, int, int, int, int, const float*,
                                         const float*, float*, int, cudaStream_t);
template int launch_nn_ring_edges<double>(const double*, const double*, double*, int, int, int, int, const double*,
                                          const double*, double*, int, cudaStream_t);
template int launch_nn_ring<float>(const float*, const float*, float*, int, int, int, int, int, int, const float*,
                                   const float*, int, cudaStream_t);
template int launch_nn_ring<double>(const double*, const double*, double*, int, int, int, int, int, int,
                                    const double*, const double*, int, cudaStream_t);

}  // namespace su3g
