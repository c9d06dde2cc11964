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

#include "nn_site.cuh"
#include "tma.cuh"

namespace su3g {

// su3g_set_option("nn_tma_l2_hints"); on by default (64^3x16 f32: 0.858 -> 0.864, neutral elsewhere)
int g_tma_hints = 1;
int g_tma_chunk = 0;  // su3g_set_option("nn_tma_chunk"): t-chunk length of the work items (0 = auto)

namespace {

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
    int hints;     // U_t gathers evict-first in L2 (read exactly once), output stored streaming
    int parity;    // PARITY kernels: output only the sites with (x+y+z+t) % 2 == parity (dslash)
};

// item -> (block, t0, t1), chunk-major
__device__ __forceinline__ void item_range(const TmaParams& p, int64_t item, int64_t& blk, int& t0, int& t1) {
    const int64_t ch = item / p.nblocks;
    blk = item - ch * p.nblocks;
    t0 = p.t_begin + static_cast<int>(ch) * p.chunk;
    t1 = min(t0 + p.chunk, p.t_end);
}

}  // namespace

// Shared-memory geometry (runtime halo widths HY = nx*BZ, HZ = nx*BY; 0 when the
// block spans that extent and the direction wraps inside the CTA).
// Stage (filled by TMA, STAGES deep):
//   SU  [54][N]   U_x, U_y, U_z of the block's sites
//   SV  [6][N]    v(x,t+1) of the block
//   HUy [18][HY]  U_y on the -y halo row      HVyd [6][HY] v on the -y row   HVyu [6][HY] v on the +y row
//   HUz [18][HZ]  U_z on the -z halo plane    HVzd [6][HZ] v on the -z row   HVzu [6][HZ] v on the +z row
// Exchange (single buffer, rewritten every step):
//   XW [18][N] w_x, w_y, w_z of the block   XV [6][N] v(x,t)   XHy [6][HY] / XHz [6][HZ] halo w_y / w_z
struct Geo {
    int N, HY, HZ;
    __device__ __forceinline__ int stage_size() const { return 60 * N + 30 * HY + 30 * HZ; }
    __device__ __forceinline__ int su() const { return 0; }
    __device__ __forceinline__ int sv() const { return 54 * N; }
    __device__ __forceinline__ int huy() const { return 60 * N; }
    __device__ __forceinline__ int hvyd() const { return 60 * N + 18 * HY; }
    __device__ __forceinline__ int hvyu() const { return 60 * N + 24 * HY; }
    __device__ __forceinline__ int huz() const { return 60 * N + 30 * HY; }
    __device__ __forceinline__ int hvzd() const { return 60 * N + 30 * HY + 18 * HZ; }
    __device__ __forceinline__ int hvzu() const { return 60 * N + 30 * HY + 24 * HZ; }
    __device__ __forceinline__ int xw() const { return 0; }
    __device__ __forceinline__ int xv() const { return 18 * N; }
    __device__ __forceinline__ int xhy() const { return 24 * N; }
    __device__ __forceinline__ int xhz() const { return 24 * N + 6 * HY; }
    __device__ __forceinline__ int xsize() const { return 24 * N + 6 * HY + 6 * HZ; }
};

// CNX/CBY/CBZ > 0: block geometry fixed at compile time (halos present in y and z),
// so every shared-memory offset is an immediate; 0: runtime geometry.
// PARITY: the even/odd dslash on the same t-walk.  At step t a site is either an
// output site ((x+y+z+t) % 2 == p.parity: forward products, the sums, the store) or a source site
// (publishes v and w_x, w_y, w_z for its output neighbours, forms w_t for step t+1, when it is an
// output site).  Same loads and arithmetic as the full sweep, so the values are bitwise those of
// the NN sweep on the output sites; the other parity of `out` is not written.
template <typename T, bool FUSED, int NTHR, int STAGES, int CNX = 0, int CBY = 0, int CBZ = 0, bool PARITY = false>
__global__ void __launch_bounds__(NTHR, 1)
    k_nn_tma(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapV,
             const __grid_constant__ CUtensorMap mapVhi, const __grid_constant__ CUtensorMap mapUyH,
             const __grid_constant__ CUtensorMap mapUzH, const __grid_constant__ CUtensorMap mapVyH,
             const __grid_constant__ CUtensorMap mapVzH, const T* __restrict__ U, const T* __restrict__ v,
             T* __restrict__ out, const T* __restrict__ w_lo, TmaParams p) {
    static_assert(STAGES == 2, "the refill of stage k%2 is step k+2 (two-step lookahead)");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr bool FIXED = CNX > 0;
    const int nx = FIXED ? CNX : p.nx;
    const int BY = FIXED ? CBY : p.BY;
    const int BZ = FIXED ? CBZ : p.BZ;
    const Geo g{NTHR, FIXED ? CNX * CBZ : (p.BY == p.ny ? 0 : nx * p.BZ),
                FIXED ? CNX * CBY : (p.BZ == p.nz ? 0 : nx * p.BY)};
    const int SS = g.stage_size();
    T* stage0 = reinterpret_cast<T*>(smem_raw);
    T* xb = stage0 + STAGES * SS;
    uint64_t* full = reinterpret_cast<uint64_t*>(xb + g.xsize());
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
    uint64_t pol_first = 0, pol_normal = 0;
    if (tid == 0) {
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_first));
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_normal));
    }
    // TMA issue of one step's operands (thread 0 only): the block's U_x, U_y, U_z, v(t+1)
    // and the halo rows; U_y / U_z stay at normal L2 priority because neighbouring
    // blocks in flight re-read them as their halo rows.
    auto issue = [&](int s, int64_t blk, int t) {
        const int y0 = static_cast<int>(blk % p.nby) * BY;
        const int z0 = static_cast<int>(blk / p.nby) * BZ;
        mbar_arrive_expect_tx(&full[s], uint32_t(SS) * sizeof(T));
        T* st = stage0 + s * SS;
        tma_load_4d(st + g.su(), &mapU, 0, y0, z0, t * 72, &full[s], pol_first);
        tma_load_4d(st + g.su() + 18 * NTHR, &mapU, 0, y0, z0, t * 72 + 18, &full[s], pol_normal);
        tma_load_4d(st + g.su() + 36 * NTHR, &mapU, 0, y0, z0, t * 72 + 36, &full[s], pol_normal);
        if (t + 1 < p.nt) tma_load_4d(st + g.sv(), &mapV, 0, y0, z0, (t + 1) * 6, &full[s], pol_normal);
        else if (p.has_vhi) tma_load_4d(st + g.sv(), &mapVhi, 0, y0, z0, 0, &full[s], pol_normal);
        else tma_load_4d(st + g.sv(), &mapV, 0, y0, z0, 0, &full[s], pol_normal);
        if (g.HY) {
            const int ydn = (y0 + p.ny - 1) % p.ny, yup = (y0 + BY) % p.ny;
            tma_load_4d(st + g.huy(), &mapUyH, 0, ydn, z0, t * 72 + 18, &full[s], pol_normal);
            tma_load_4d(st + g.hvyd(), &mapVyH, 0, ydn, z0, t * 6, &full[s], pol_normal);
            tma_load_4d(st + g.hvyu(), &mapVyH, 0, yup, z0, t * 6, &full[s], pol_normal);
        }
        if (g.HZ) {
            const int zdn = (z0 + p.nz - 1) % p.nz, zup = (z0 + BZ) % p.nz;
            tma_load_4d(st + g.huz(), &mapUzH, 0, y0, zdn, t * 72 + 36, &full[s], pol_normal);
            tma_load_4d(st + g.hvzd(), &mapVzH, 0, y0, zdn, t * 6, &full[s], pol_normal);
            tma_load_4d(st + g.hvzu(), &mapVzH, 0, y0, zup, t * 6, &full[s], pol_normal);
        }
    };

    // ----------------------------------------------------------------------
    // compute threads: one site each (+ one halo-row half-product)
    // ----------------------------------------------------------------------
    const int lx = tid % nx;
    const int rr = tid / nx;
    const int ly = rr % BY;
    const int lz = rr / BY;
    const int sy = nx, sz = nx * BY;
    const int ix_up = (lx + 1 == nx) ? tid - lx : tid + 1;
    const int ix_dn = (lx == 0) ? tid + nx - 1 : tid - 1;
    // neighbour sources: >= 0 -> block slot in the exchange; < 0 -> halo row slot (-1 - j)
    const int iy_up = (ly + 1 < BY) ? tid + sy : (g.HY == 0 ? tid - (BY - 1) * sy : -1 - (lx + nx * lz));
    const int iy_dn = (ly > 0) ? tid - sy : (g.HY == 0 ? tid + (BY - 1) * sy : -1 - (lx + nx * lz));
    const int iz_up = (lz + 1 < BZ) ? tid + sz : (g.HZ == 0 ? tid - (BZ - 1) * sz : -1 - (lx + nx * ly));
    const int iz_dn = (lz > 0) ? tid - sz : (g.HZ == 0 ? tid + (BZ - 1) * sz : -1 - (lx + nx * ly));

    auto site_of = [&](int64_t blk) {
        const int y = static_cast<int>(blk % p.nby) * BY + ly;
        const int z = static_cast<int>(blk / p.nby) * BZ + lz;
        return lx + int64_t(nx) * (y + int64_t(p.ny) * z);
    };

    // U_t of step k is loaded two steps ahead (registers ut -> ut1 -> ut2 pipeline); the
    // cursor caches its site index so the per-step work has no 64-bit divisions
    struct Cursor {
        int64_t item, blk, s3;
        int t, t1;
        bool valid;
    };
    auto enter = [&](Cursor& c) {
        int a0, a1;
        item_range(p, c.item, c.blk, a0, a1);
        c.t = a0;
        c.t1 = a1;
        c.s3 = site_of(c.blk);
    };
    auto advance = [&](Cursor c) {
        if (!c.valid) return c;
        if (c.t + 1 < c.t1) {
            ++c.t;
            return c;
        }
        c.item += G;
        if (c.item >= p.nitems) {
            c.valid = false;
            return c;
        }
        enter(c);
        return c;
    };
    const uint64_t pol_once = l2_evict_first_policy();
    auto load_ut = [&](const Cursor& c, T* r) {
        if (!c.valid) return;
        if (p.hints) ld_soa_last<T, 18>(U + (int64_t(c.t) * 72 + 54) * F, F, c.s3, r, pol_once);
        else ld_soa<T, 18>(U + (int64_t(c.t) * 72 + 54) * F, F, c.s3, r);
    };

    T vc[6], wt[6], ut[18], ut1[18];
    int64_t k = 0;
    int64_t item = blockIdx.x;
    int64_t blk = 0;
    int t0 = 0, t1 = 0;
    Cursor ahead{item, 0, 0, 0, 0, item < p.nitems};
    if (ahead.valid) {
        enter(ahead);
        if (tid == 0) issue(0, ahead.blk, ahead.t);
        load_ut(ahead, ut);
        ahead = advance(ahead);
        if (tid == 0 && ahead.valid && STAGES > 1) issue(1, ahead.blk, ahead.t);
        load_ut(ahead, ut1);
        ahead = advance(ahead);  // -> step 2
    }
    for (; item < p.nitems; item += G) {
        item_range(p, item, blk, t0, t1);
        const int64_t s3 = site_of(blk);
        // site parity at t = 0 (PARITY kernels): x + y + z of this thread's site
        const int par0 = PARITY ? ((lx + ly + lz + static_cast<int>(blk % p.nby) * BY +
                                    static_cast<int>(blk / p.nby) * BZ) & 1)
                                : 0;
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

        for (int t = t0; t < t1; ++t, ++k) {
            T ut2[18];
            const Cursor c2 = ahead;  // step k + 2
            load_ut(c2, ut2);
            ahead = advance(ahead);
            const int s = static_cast<int>(k % STAGES);
            mbar_wait(&full[s], static_cast<uint32_t>((k / STAGES) & 1));
            const T* st = stage0 + s * SS;

            T u[54], vnext[6];
#pragma unroll
            for (int q = 0; q < 54; ++q) u[q] = st[g.su() + q * NTHR + tid];
#pragma unroll
            for (int q = 0; q < 6; ++q) vnext[q] = st[g.sv() + q * NTHR + tid];

            // halo-row half-products: thread j computes halo site j
            for (int j = tid; j < g.HY + g.HZ; j += NTHR) {
                T uh[18], vh[6], wh[6];
                const bool isy = j < g.HY;
                const int jj = isy ? j : j - g.HY;
                const int hp = isy ? g.HY : g.HZ;
                const int ub = isy ? g.huy() : g.huz();
                const int vb = isy ? g.hvyd() : g.hvzd();
#pragma unroll
                for (int q = 0; q < 18; ++q) uh[q] = st[ub + q * hp + jj];
#pragma unroll
                for (int q = 0; q < 6; ++q) vh[q] = st[vb + q * hp + jj];
                amv<T, FUSED>(uh, vh, wh);
                const int xo = isy ? g.xhy() : g.xhz();
#pragma unroll
                for (int q = 0; q < 6; ++q) xb[xo + q * hp + jj] = wh[q];
            }
            // roles: every site is both in the full sweep; one or the other in a PARITY kernel
            const bool is_out = !PARITY || (((par0 + t) & 1) == p.parity);
            const bool is_src = !PARITY || !is_out;
            // this site's half-products w_x, w_y, w_z and v(x,t) for the neighbours
            if (is_src) {
                T w[6];
#pragma unroll
                for (int mu = 0; mu < 3; ++mu) {
                    amv<T, FUSED>(u + 18 * mu, vc, w);
#pragma unroll
                    for (int q = 0; q < 6; ++q) xb[g.xw() + (6 * mu + q) * NTHR + tid] = w[q];
                }
#pragma unroll
                for (int q = 0; q < 6; ++q) xb[g.xv() + q * NTHR + tid] = vc[q];
            }
            T wt_next[6], f3[6];
            if (is_src) amv<T, FUSED>(ut, vc, wt_next);  // -t term of this site at step t + 1
            if (is_out) mv<T, FUSED>(ut, vnext, f3);     // forward +t term, summed last
            named_sync<NTHR>();

            // forward terms (add_su3_vector chain: ((f0 + f1) + f2) + f3)
            T acc[6];
            if (is_out) {
                T nb[6], f[6];
#pragma unroll
                for (int q = 0; q < 6; ++q) nb[q] = xb[g.xv() + q * NTHR + ix_up];
                mv<T, FUSED>(u, nb, acc);
                if (iy_up >= 0) {
#pragma unroll
                    for (int q = 0; q < 6; ++q) nb[q] = xb[g.xv() + q * NTHR + iy_up];
                } else {
#pragma unroll
                    for (int q = 0; q < 6; ++q) nb[q] = st[g.hvyu() + q * g.HY + (-1 - iy_up)];
                }
                mv<T, FUSED>(u + 18, nb, f);
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xadd(acc[q], f[q]);
                if (iz_up >= 0) {
#pragma unroll
                    for (int q = 0; q < 6; ++q) nb[q] = xb[g.xv() + q * NTHR + iz_up];
                } else {
#pragma unroll
                    for (int q = 0; q < 6; ++q) nb[q] = st[g.hvzu() + q * g.HZ + (-1 - iz_up)];
                }
                mv<T, FUSED>(u + 36, nb, f);
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xadd(acc[q], f[q]);
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xadd(acc[q], f3[q]);
            }

            // backward terms (sub_four_su3_vecs chain)
            if (is_out) {
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], xb[g.xw() + q * NTHR + ix_dn]);
            if (iy_dn >= 0) {
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], xb[g.xw() + (6 + q) * NTHR + iy_dn]);
            } else {
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], xb[g.xhy() + q * g.HY + (-1 - iy_dn)]);
            }
            if (iz_dn >= 0) {
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], xb[g.xw() + (12 + q) * NTHR + iz_dn]);
            } else {
#pragma unroll
                for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], xb[g.xhz() + q * g.HZ + (-1 - iz_dn)]);
            }
#pragma unroll
            for (int q = 0; q < 6; ++q) acc[q] = xsub(acc[q], wt[q]);

            T* o = out + int64_t(t) * 6 * F + s3;
            if (p.hints) {
#pragma unroll
                for (int q = 0; q < 6; ++q) __stcs(o + q * F, acc[q]);
            } else {
#pragma unroll
                for (int q = 0; q < 6; ++q) o[q * F] = acc[q];
            }
            }  // is_out
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                vc[q] = vnext[q];
                wt[q] = wt_next[q];
            }
#pragma unroll
            for (int q = 0; q < 18; ++q) {
                ut[q] = ut1[q];
                ut1[q] = ut2[q];
            }
            named_sync<NTHR>();  // exchange buffer and stage s free for the next step
            // refill stage s with step k + 2: every thread is past its last read of it, so
            // no empty-barrier wait is needed (and warp 0 never stalls mid-step)
            if (tid == 0 && c2.valid) {
                fence_before_refill();  // the step's reads of stage s (ordered by the barrier) before the TMA refill
                issue(s, c2.blk, c2.t);
            }
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

}  // namespace

template <typename T, bool FUSED, int NTHR, int STAGES, int CNX = 0, int CBY = 0, int CBZ = 0, bool PARITY = false>
static int run_tma(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                   const T* v_hi, const T* w_lo, int BY, int BZ, cudaStream_t st, int parity = -1) {
    const int HY = (BY == ny) ? 0 : nx * BZ, HZ = (BZ == nz) ? 0 : nx * BY;
    CUtensorMap mU, mV, mVhi, mUy, mUz, mVy, mVz;
    if (!make_map<T>(&mU, U, nx, ny, nz, int64_t(nt) * 72, BY, BZ, 18)) return 1;
    if (!make_map<T>(&mV, v, nx, ny, nz, int64_t(nt) * 6, BY, BZ, 6)) return 1;
    if (v_hi != nullptr) {
        if (!make_map<T>(&mVhi, v_hi, nx, ny, nz, 6, BY, BZ, 6)) return 1;
    } else {
        mVhi = mV;
    }
    mUy = mU; mVy = mV; mUz = mU; mVz = mV;
    if (HY && (!make_map<T>(&mUy, U, nx, ny, nz, int64_t(nt) * 72, 1, BZ, 18) ||
               !make_map<T>(&mVy, v, nx, ny, nz, int64_t(nt) * 6, 1, BZ, 6)))
        return 1;
    if (HZ && (!make_map<T>(&mUz, U, nx, ny, nz, int64_t(nt) * 72, BY, 1, 18) ||
               !make_map<T>(&mVz, v, nx, ny, nz, int64_t(nt) * 6, BY, 1, 6)))
        return 1;
    const size_t stage = size_t(60) * NTHR + 30 * size_t(HY) + 30 * size_t(HZ);
    const size_t xsize = size_t(24) * NTHR + 6 * size_t(HY) + 6 * size_t(HZ);
    const size_t smem = (STAGES * stage + xsize) * sizeof(T) + 2 * STAGES * sizeof(uint64_t);
    const DeviceInfo& di = device_info();
    if (smem > size_t(di.max_smem_optin)) return 1;
    cudaFuncSetAttribute(k_nn_tma<T, FUSED, NTHR, STAGES, CNX, CBY, CBZ, PARITY>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    TmaParams p{};
    p.nx = nx; p.ny = ny; p.nz = nz; p.nt = nt;
    p.F = int64_t(nx) * ny * nz;
    p.BY = BY; p.BZ = BZ; p.nby = ny / BY;
    p.nblocks = int64_t(ny / BY) * (nz / BZ);
    p.t_begin = t_begin; p.t_end = t_end;
    int per_sm = 1;  // resident CTAs per SM (2 for the 128-thread f32 geometry)
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_nn_tma<T, FUSED, NTHR, STAGES, CNX, CBY, CBZ, PARITY>, NTHR, smem);
    // SMs left free for NCCL's kernels (su3g "sm_reserve", set by the t-slab drivers at N > 1): this
    // persistent kernel fills every SM, so a concurrent NCCL kernel would wait for it to finish.  A
    // free SM costs a whole extra round when it pushes the single wave over a round boundary
    // (64^3x14 interior: 1024 items, 7 rounds on 148 CTAs, 8 on 144), so the reservation is trimmed
    // to what the last round's slack absorbs, and dropped when not even one SM fits.
    const int per = std::max(per_sm, 1);
    const int G_full = device_info().num_sms * per;
    const int L = t_end - t_begin;
    p.chunk = g_tma_chunk > 0 ? std::min(g_tma_chunk, L) : pick_chunk(p.nblocks, L, G_full);
    p.nchunks = (L + p.chunk - 1) / p.chunk;
    p.nitems = p.nblocks * p.nchunks;
    int G = G_full;
    if (sm_reserve() > 0) {
        const int64_t rounds = (p.nitems + G_full - 1) / G_full;
        const int64_t g_same = (p.nitems + rounds - 1) / rounds;  // fewest CTAs that keep the round count
        const int g_res = std::max(per, sweep_sms() * per);
        if (g_same <= G_full - per) G = static_cast<int>(std::max<int64_t>(g_res, g_same));
    }
    p.has_vhi = v_hi != nullptr;
    p.hints = g_tma_hints;
    p.parity = parity;
    const int grid = static_cast<int>(std::min<int64_t>(G, p.nitems));
    k_nn_tma<T, FUSED, NTHR, STAGES, CNX, CBY, CBZ, PARITY><<<grid, NTHR, smem, st>>>(mU, mV, mVhi, mUy, mUz, mVy, mVz, U, v, out, w_lo, p);
    note_kernel(std::string("k_nn_tma<") + (sizeof(T) == 4 ? "f32," : "f64,") + std::to_string(nx) + "x" +
                std::to_string(BY) + "x" + std::to_string(BZ) + (CNX ? "" : " runtime-geometry") + "," +
                std::to_string(NTHR) + "thr>" + (grid < G_full ? " grid " + std::to_string(grid) : std::string()));
    return check_launch("nn_sweep(tma)");
}

int g_tma_threads = 0;  // su3g_set_option("nn_tma_threads"): 0 auto, 128, 256

template <typename T>
int launch_nn_tma(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                  const T* v_hi, const T* w_lo, int mode, cudaStream_t st) {
    if constexpr (sizeof(T) == 4) {
        // 32-wide lattices: 128-site blocks (32x2x2) fit two CTAs per SM, which hide each
        // other's barrier and prologue stalls (BASELINE configs[2], 32^4)
        const bool small = g_tma_threads == 128 || (g_tma_threads == 0 && nx == 32);
        if (small && nx == 32 && ny % 2 == 0 && nz % 2 == 0 && ny > 2 && nz > 2 && aligned16(U) && aligned16(v) &&
            (!v_hi || aligned16(v_hi)))
            return mode == SU3G_FMA
                       ? run_tma<T, true, 128, 2, 32, 2, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, 2, 2, st)
                       : run_tma<T, false, 128, 2, 32, 2, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, 2, 2, st);
    }
    constexpr int NTHR = sizeof(T) == 4 ? 256 : 128;
    if ((nx * int(sizeof(T))) % 16 != 0 || nx > 256) return 1;
    if (!aligned16(U) || !aligned16(v) || (v_hi && !aligned16(v_hi))) return 1;
    int BY = 0, BZ = 0;
    if (!tma_shape(nx, ny, nz, NTHR, BY, BZ)) {
        // x extents that do not divide 256: 48 (the 48^4 lattice of configs[3]) gets a specialised
        // 192-site block geometry
        // (runtime-geometry kernels measured no better than the register walk: 48^3 0.589 vs 0.572,
        // 40^3 0.456 -- so only the specialised 48x2x2 geometry is used)
        if constexpr (sizeof(T) == 4) {
            if (nx == 48 && ny % 2 == 0 && nz % 2 == 0 && ny > 2 && nz > 2)
                return mode == SU3G_FMA
                           ? run_tma<T, true, 192, 2, 48, 2, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, 2, 2, st)
                           : run_tma<T, false, 192, 2, 48, 2, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, 2, 2, st);
        }
        return 1;
    }
    if constexpr (sizeof(T) == 4) {  // the production geometries, specialised
        if (nx == 32 && BY == 2 && BZ == 4 && ny > 2 && nz > 4)
            return mode == SU3G_FMA
                       ? run_tma<T, true, NTHR, 2, 32, 2, 4>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, BY, BZ, st)
                       : run_tma<T, false, NTHR, 2, 32, 2, 4>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, BY, BZ, st);
        if (nx == 64 && BY == 2 && BZ == 2 && ny > 2 && nz > 2)
            return mode == SU3G_FMA
                       ? run_tma<T, true, NTHR, 2, 64, 2, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, BY, BZ, st)
                       : run_tma<T, false, NTHR, 2, 64, 2, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, BY, BZ, st);
    }
    return mode == SU3G_FMA
               ? run_tma<T, true, NTHR, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, BY, BZ, st)
               : run_tma<T, false, NTHR, 2>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, BY, BZ, st);
}

// even/odd dslash on the TMA t-walk (PARITY kernels): the production geometries only; returns 1
// when the lattice has none, so the caller falls back to the one-thread-per-site parity kernel
template <typename T>
int launch_dslash_tma(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int parity, int mode,
                      cudaStream_t st) {
    if constexpr (sizeof(T) != 4) {
        return 1;
    } else {
        if (!aligned16(U) || !aligned16(v)) return 1;
        int BY = 0, BZ = 0;
        if (!tma_shape(nx, ny, nz, 256, BY, BZ)) return 1;
        if (nx == 64 && BY == 2 && BZ == 2 && ny > 2 && nz > 2)
            return mode == SU3G_FMA
                       ? run_tma<T, true, 256, 2, 64, 2, 2, true>(U, v, out, nx, ny, nz, nt, 0, nt, nullptr, nullptr, BY, BZ, st, parity)
                       : run_tma<T, false, 256, 2, 64, 2, 2, true>(U, v, out, nx, ny, nz, nt, 0, nt, nullptr, nullptr, BY, BZ, st, parity);
        if (nx == 32 && BY == 2 && BZ == 4 && ny > 2 && nz > 4)
            return mode == SU3G_FMA
                       ? run_tma<T, true, 256, 2, 32, 2, 4, true>(U, v, out, nx, ny, nz, nt, 0, nt, nullptr, nullptr, BY, BZ, st, parity)
                       : run_tma<T, false, 256, 2, 32, 2, 4, true>(U, v, out, nx, ny, nz, nt, 0, nt, nullptr, nullptr, BY, BZ, st, parity);
        return mode == SU3G_FMA
                   ? run_tma<T, true, 256, 2, 0, 0, 0, true>(U, v, out, nx, ny, nz, nt, 0, nt, nullptr, nullptr, BY, BZ, st, parity)
                   : run_tma<T, false, 256, 2, 0, 0, 0, true>(U, v, out, nx, ny, nz, nt, 0, nt, nullptr, nullptr, BY, BZ, st, parity);
    }
}

template int launch_dslash_tma<float>(const float*, const float*, float*, int, int, int, int, int, int, cudaStream_t);
template int launch_dslash_tma<double>(const double*, const double*, double*, int, int, int, int, int, int,
                                       cudaStream_t);

template int launch_nn_tma<float>(const float*, const float*, float*, int, int, int, int, int, int, const float*,
                                  const float*, int, cudaStream_t);
template int launch_nn_tma<double>(const double*, const double*, double*, int, int, int, int, int, int,
                                   const double*, const double*, int, cudaStream_t);

}  // namespace su3g
