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
#include <atomic>
#include <cstring>

#include "nn_site.cuh"
#include "sweep_common.cuh"

namespace su3g {

void set_sm_reserve(int n);
extern int g_tma_threads;
extern int g_link_minb;
extern int g_link_tw_chunk;
extern int g_link_rows3_minb;
int g_link_zc = 0;   // su3g_set_option("link_zc"): z-planes per visiting chunk of the link kernels (0 = auto)
int g_sweep_zc = 0;  // su3g_set_option("sweep_zc"): z-planes per chunk of the generic NN / dslash kernels
// su3g_set_option("sweep_l2_hints"): evict-first backward gathers, streaming stores.  Default on:
// f64 64^3x16 0.686 -> 0.736 of HBM, 32^4 0.711 -> 0.777, dslash f64 0.569 -> 0.642 (same box A/B)
int g_sweep_hints = 1;
int g_sweep_keep = 0;      // su3g_set_option("sweep_l2_keep"): own-link loads evict-last (A/B)
int g_sweep_prefetch = 0;  // su3g_set_option("sweep_prefetch"): L2 prefetch distance in quarter waves (0 = off)
extern int g_link_early_c;
extern int g_link_pref_b;
extern int g_link_hints;
extern int g_link_l1_hints;
extern int g_tma_hints;
extern int g_tma_chunk;
extern int g_eo_zc;
extern int g_eo_hints;

// ---------------------------------------------------------------------------
// NN sweep, one thread per site
// ---------------------------------------------------------------------------
template <typename T, bool FUSED, bool HINTS = false, bool KEEP = false>
__device__ __forceinline__ void nn_sweep_body(const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ out,
                                              const Geom& g, int t_begin, int t_end, const T* __restrict__ v_hi,
                                              const T* __restrict__ w_lo, int ZC, int ahead = 0) {
    if (ahead > 0 && threadIdx.x == 0) {
        prefetch_cta_l2<T>(U, 72, g, blockIdx.x + int64_t(ahead), blockDim.x, t_begin, t_end - t_begin, ZC);
        prefetch_cta_l2<T>(v, 6, g, blockIdx.x + int64_t(ahead), blockDim.x, t_begin, t_end - t_begin, ZC);
    }
    // visiting order (z-chunk of ZC planes, t, z, y, x): the t-1 slice a site reads (U_t, v)
    // was streamed ZC*nx*ny sites earlier, not a whole slice earlier -> L2 hits
    const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    const int nts = t_end - t_begin;
    if (idx >= int64_t(nts) * g.F) return;
    const int x = static_cast<int>(idx % g.nx);
    int64_t r = idx / g.nx;
    const int y = static_cast<int>(r % g.ny);
    r /= g.ny;
    const int zl = static_cast<int>(r % ZC);
    r /= ZC;
    const int t = t_begin + static_cast<int>(r % nts);
    const int z = static_cast<int>(r / nts) * ZC + zl;
    nn_site<T, FUSED, HINTS, KEEP>(U, v, out, g, x, y, z, t, v_hi, w_lo);
}

// plain bounds: ptxas picks 64-98 registers; an explicit minBlocks of 1 would let it take 252
template <typename T, bool FUSED, bool HINTS = false, bool KEEP = false>
__global__ void __launch_bounds__(256)
    k_nn_sweep(const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ out, Geom g, int t_begin, int t_end,
               const T* __restrict__ v_hi, const T* __restrict__ w_lo, int ZC, int ahead) {
    nn_sweep_body<T, FUSED, HINTS, KEEP>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC, ahead);
}

// occupancy A/B (nn_variant 6): registers capped for MINB CTAs per SM
template <typename T, bool FUSED, int MINB>
__global__ void __launch_bounds__(256, MINB)
    k_nn_sweep_capped(const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ out, Geom g, int t_begin,
                      int t_end, const T* __restrict__ v_hi, const T* __restrict__ w_lo, int ZC) {
    nn_sweep_body<T, FUSED>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC);
}

// ---------------------------------------------------------------------------
// even/odd dslash: the NN operator evaluated only on the sites of one
// parity, (x+y+z+t) % 2 == parity, which read v only on the other parity.  Fused in one
// kernel: forward U_mu(x) v(x+mu), backward U_mu(x-mu)^dag v(x-mu) (the adj_4dir products of
// the neighbours), the add chain and sub_four -- the NN sweep's association, so the result
// equals the full sweep's on those sites bit for bit.  Sites of the other parity in `out`
// are not touched.  One thread per output site, (z-chunk, t, z, y, x/2) order.
// ---------------------------------------------------------------------------
template <typename T, bool FUSED, bool HINTS = false>
__global__ void __launch_bounds__(256)
    k_dslash(const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ out, Geom g, int parity, int ZC,
             int ahead) {
    if (ahead > 0 && threadIdx.x == 0) {
        prefetch_cta_l2<T>(U, 72, g, blockIdx.x + int64_t(ahead), blockDim.x, 0, g.nt, ZC, 2);
        prefetch_cta_l2<T>(v, 6, g, blockIdx.x + int64_t(ahead), blockDim.x, 0, g.nt, ZC, 2);
    }
    const int nxh = g.nx >> 1;
    const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (idx >= (g.F >> 1) * g.nt) return;
    const int xh = static_cast<int>(idx % nxh);
    int64_t r = idx / nxh;
    const int y = static_cast<int>(r % g.ny);
    r /= g.ny;
    const int zl = static_cast<int>(r % ZC);
    r /= ZC;
    const int t = static_cast<int>(r % g.nt);
    const int z = static_cast<int>(r / g.nt) * ZC + zl;
    const int x = 2 * xh + ((y + z + t + parity) & 1);
    nn_site<T, FUSED, HINTS>(U, v, out, g, x, y, z, t, nullptr, nullptr);
}

// out(x) = src(x) on the sites of one parity (the workspace path of su3g_dslash_ws)
template <typename T>
__global__ void __launch_bounds__(256) k_parity_copy(const T* __restrict__ src, T* __restrict__ dst, Geom g,
                                                     int parity) {
    const int nxh = g.nx >> 1;
    const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (idx >= (g.F >> 1) * g.nt) return;
    const int xh = static_cast<int>(idx % nxh);
    int64_t r = idx / nxh;
    const int y = static_cast<int>(r % g.ny);
    r /= g.ny;
    const int z = static_cast<int>(r % g.nz);
    const int t = static_cast<int>(r / g.nz);
    const int x = 2 * xh + ((y + z + t + parity) & 1);
    const int64_t s3 = x + int64_t(g.nx) * (y + int64_t(g.ny) * z);
#pragma unroll
    for (int k = 0; k < 6; ++k) dst[(int64_t(t) * 6 + k) * g.F + s3] = src[(int64_t(t) * 6 + k) * g.F + s3];
}

template <typename T, bool FUSED>
__global__ void __launch_bounds__(256)
    k_nn_halo_w(const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ w_face, Geom g) {
    const int64_t s3 = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (s3 >= g.F) return;
    const int t = g.nt - 1;
    T u[18], vn[6], w[6];
    ld_soa<T, 18>(U + (int64_t(t) * 72 + 3 * 18) * g.F, g.F, s3, u);
    ld_soa<T, 6>(v + int64_t(t) * 6 * g.F, g.F, s3, vn);
    amv<T, FUSED>(u, vn, w);
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

// One site's link product (shared by both schedules below).
template <typename T, bool FUSED>
__device__ __forceinline__ void link_site(const T* __restrict__ U, T* __restrict__ acc_out, const Geom& g, T s, int x,
                                          int y, int z, int t) {
    const int64_t s3 = x + int64_t(g.nx) * (y + int64_t(g.ny) * z);
    const int64_t site = int64_t(t) * g.F + s3;
    T acc[18];
#pragma unroll
    for (int k = 0; k < 18; ++k) acc[k] = T(0);
    // FMA mode: full unroll lets the next plane's link loads overlap this plane's math
    // (measured 1.43 vs 1.79 ms at 48^4); exact mode keeps the rolled loop (unrolled it spills)
    if constexpr (FUSED) {
    #pragma unroll
        for (int mu = 0; mu < 3; ++mu) {
            T a[18];
            ld_link(U, g, site, mu, a);
    #pragma unroll
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
    } else {
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
    }
#pragma unroll
    for (int k = 0; k < 18; ++k) acc_out[(int64_t(t) * 18 + k) * g.F + s3] = acc[k];
}

// Sites are visited in (z-chunk, t, z, y, x) order with ZC z-planes per chunk: the
// +t links a site gathers as neighbours are re-read as own links ZC*nx*ny sites
// later (a few MB of traffic) instead of one whole slice later, so they stay in
// L2 (natural t-major order measured 35% L2 hits, 1.7x the compulsory DRAM reads).
template <typename T, bool FUSED>
__global__ void __launch_bounds__(128)
    k_link_product(const T* __restrict__ U, T* __restrict__ acc_out, Geom g, T s, int ZC) {
    const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (idx >= g.F * g.nt) return;
    const int x = static_cast<int>(idx % g.nx);
    int64_t r = idx / g.nx;
    const int y = static_cast<int>(r % g.ny);
    r /= g.ny;
    const int zl = static_cast<int>(r % ZC);
    r /= ZC;
    const int t = static_cast<int>(r % g.nt);
    const int z = static_cast<int>(r / g.nt) * ZC + zl;
    link_site<T, FUSED>(U, acc_out, g, s, x, y, z, t);
}

// Block-walk schedule: a CTA owns nx x BY x BZ sites of a slice and walks t; work items
// (block, t-chunk) go chunk-major over a single wave, so the +t slice a CTA reads as
// neighbours is what it reads as its own links one step later, and halo links come from
// blocks other CTAs stream at the same time -- L2 hits instead of DRAM re-reads.
struct LinkWalk {
    int BY, BZ, nby;
    int64_t nblocks;
    int chunk;
    int64_t nitems;
};

template <typename T, bool FUSED>
__global__ void __launch_bounds__(128)
    k_link_walk(const T* __restrict__ U, T* __restrict__ acc_out, Geom g, LinkWalk w, T s) {
    const int tid = threadIdx.x;
    const int lx = tid % g.nx, rr = tid / g.nx, ly = rr % w.BY, lz = rr / w.BY;
    for (int64_t item = blockIdx.x; item < w.nitems; item += gridDim.x) {
        const int64_t ch = item / w.nblocks;
        const int64_t blk = item - ch * w.nblocks;
        const int t0 = static_cast<int>(ch) * w.chunk;
        const int t1 = min(t0 + w.chunk, g.nt);
        const int y = static_cast<int>(blk % w.nby) * w.BY + ly;
        const int z = static_cast<int>(blk / w.nby) * w.BZ + lz;
        for (int t = t0; t < t1; ++t) link_site<T, FUSED>(U, acc_out, g, s, lx, y, z, t);
    }
}


// The two boundary slices of a t-slab application, t = 0 and t = nt-1, in one launch (the t-slab
// drivers run them after the halo exchange).  With w_next, the threads of slice nt-1 also form
// w = U_t(x)^dag out(x) -- the halo the NEXT application sends to rank r+1 -- from the value they
// just stored, with nn_halo_w's arithmetic, so the next application needs no separate pack kernel.
template <typename T, bool FUSED, bool HINTS>
__global__ void __launch_bounds__(256)
    k_nn_edges(const T* __restrict__ U, const T* __restrict__ v, T* out, Geom g, const T* __restrict__ v_hi,
               const T* __restrict__ w_lo, T* __restrict__ w_next, int nedge) {
    const int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    if (idx >= nedge * g.F) return;
    const int e = idx >= g.F;  // 0: t = 0, 1: t = nt - 1
    const int64_t s3 = idx - e * g.F;
    const int x = static_cast<int>(s3 % g.nx);
    const int y = static_cast<int>((s3 / g.nx) % g.ny);
    const int z = static_cast<int>(s3 / (int64_t(g.nx) * g.ny));
    const int t = e ? g.nt - 1 : 0;
    nn_site<T, FUSED, HINTS>(U, v, out, g, x, y, z, t, v_hi, w_lo);
    if (w_next != nullptr && t == g.nt - 1) {
        T u[18], o[6], w[6];
        ld_soa<T, 18>(U + (int64_t(t) * 72 + 54) * g.F, g.F, s3, u);
#pragma unroll
        for (int k = 0; k < 6; ++k) o[k] = out[(int64_t(t) * 6 + k) * g.F + s3];  // this thread's own store
        amv<T, FUSED>(u, o, w);
#pragma unroll
        for (int k = 0; k < 6; ++k) w_next[k * g.F + s3] = w[k];
    }
}

// ---------------------------------------------------------------------------
// NN sweep, t-walk kernel (the fast path)
//
// A CTA owns a block of one t-slice, full x extent (x periodic inside the CTA)
// times BY x BZ rows, one thread per (x, y, z) column, and walks t.  Per step:
//   * each thread streams its own links U_mu(x,t) (72 reals, coalesced SoA)
//     and v(x,t+1) from HBM -- the only compulsory traffic;
//   * it forms the backward half-products w_mu(x) = U_mu(x)^dag v(x) for
//     mu = x, y, z and publishes them with v(x) in shared memory, so every
//     backward neighbour term is read from on-chip memory instead of
//     re-fetching the neighbour's 18-real link;
//   * w_t(x,t) stays in registers and is the -t term of step t+1; v(x,t+1)
//     becomes v(x,t) of the next step -- t-neighbours never leave the SM;
//   * y/z neighbours outside the block (halo rows) come from L2.
// Work = (blocks x slices) steps split evenly over persistent CTAs; a CTA
// crossing into a new block reloads the one-slice prologue.
// The per-site arithmetic (and its order) is exactly that of k_nn_sweep, so
// both paths -- and the composed reference -- agree bit for bit.
// ---------------------------------------------------------------------------
template <typename T>
struct WalkParams {
    const T* __restrict__ U;
    const T* __restrict__ v;
    T* __restrict__ out;
    const T* __restrict__ v_hi;
    const T* __restrict__ w_lo;
    int nx, ny, nz, nt;
    int64_t F;
    int BY, BZ, nby;
    int t_begin, t_end;
    int64_t nblocks;
    int chunk;       // t-chunk length of one work item
    int64_t nitems;  // nblocks * ceil((t_end - t_begin) / chunk), chunk-major
};

template <typename T, bool FUSED, int MINB>
__global__ void __launch_bounds__(256, MINB) k_nn_walk(WalkParams<T> p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    const int nthr = blockDim.x;
    const int tid = threadIdx.x;
    const int nx = p.nx;
    const int lx = tid % nx;
    const int rr = tid / nx;
    const int ly = rr % p.BY;
    const int lz = rr / p.BY;
    const int64_t F = p.F;
    const int steps = p.t_end - p.t_begin;

    // in-block neighbour threads for the backward exchange (-1: halo row, via L2)
    const int tx_dn = (lx == 0) ? tid + nx - 1 : tid - 1;
    const int sy = nx, sz = nx * p.BY;
    const int ty_dn = (ly > 0) ? tid - sy : (p.BY == p.ny ? tid + (p.BY - 1) * sy : -1);
    const int tz_dn = (lz > 0) ? tid - sz : (p.BZ == p.nz ? tid + (p.BZ - 1) * sz : -1);

    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));

    T vc[6], wt[6];
    int64_t s3 = 0, s3_up[3] = {0, 0, 0}, s3_ydn = 0, s3_zdn = 0;
    int buf = 0;
    // items (block, t-chunk), chunk-major: CTAs in flight hold neighbouring blocks of the same
    // t-range, so the halo rows they read from each other are L2 hits
    for (int64_t item = blockIdx.x; item < p.nitems; item += gridDim.x) {
        const int64_t ch = item / p.nblocks;
        const int64_t blk = item - ch * p.nblocks;
        const int t0 = p.t_begin + static_cast<int>(ch) * p.chunk;
        const int t1 = min(t0 + p.chunk, p.t_end);
        {  // prologue: v(x,t0) and the -t half-product w_t(x,t0-1)
            const int y = static_cast<int>(blk % p.nby) * p.BY + ly;
            const int z = static_cast<int>(blk / p.nby) * p.BZ + lz;
            s3 = lx + int64_t(nx) * (y + int64_t(p.ny) * z);
            s3_up[0] = (lx + 1) % nx + int64_t(nx) * (y + int64_t(p.ny) * z);
            s3_up[1] = lx + int64_t(nx) * ((y + 1) % p.ny + int64_t(p.ny) * z);
            s3_up[2] = lx + int64_t(nx) * (y + int64_t(p.ny) * ((z + 1) % p.nz));
            s3_ydn = lx + int64_t(nx) * ((y + p.ny - 1) % p.ny + int64_t(p.ny) * z);
            s3_zdn = lx + int64_t(nx) * (y + int64_t(p.ny) * ((z + p.nz - 1) % p.nz));
            ld_soa<T, 6>(p.v + int64_t(t0) * 6 * F, F, s3, vc);
            if (t0 == 0 && p.w_lo != nullptr) {
                ld_soa<T, 6>(p.w_lo, F, s3, wt);
            } else {
                const int tp = (t0 > 0) ? t0 - 1 : p.nt - 1;
                T u[18], vp[6];
                ld_soa<T, 18>(p.U + (int64_t(tp) * 72 + 54) * F, F, s3, u);
                ld_soa<T, 6>(p.v + int64_t(tp) * 6 * F, F, s3, vp);
                amv<T, FUSED>(u, vp, wt);
            }
        }
      for (int t = t0; t < t1; ++t) {
        T vn[6];
        if (t + 1 < p.nt) ld_soa<T, 6>(p.v + int64_t(t + 1) * 6 * F, F, s3, vn);
        else if (p.v_hi != nullptr) ld_soa<T, 6>(p.v_hi, F, s3, vn);
        else ld_soa<T, 6>(p.v, F, s3, vn);

        // ---- per direction: stream U_mu(x,t) once; publish w_mu; forward term ----
        T* sb = sm + buf * 18 * nthr;
        const T* Ut = p.U + int64_t(t) * 72 * F + s3;
        const T* vt = p.v + int64_t(t) * 6 * F;
        T acc[6], wt_next[6];
#pragma unroll
        for (int mu = 0; mu < 4; ++mu) {
            T u[18], nb[6], f[6];
#pragma unroll
            for (int k = 0; k < 18; ++k)  // U_y / U_z rows are re-read as halos by neighbouring blocks
                u[k] = (mu == 1 || mu == 2) ? __ldg(Ut + (18 * mu + k) * F) : ld_stream(Ut + (18 * mu + k) * F, pol);
            if (mu < 3) {
                T wm[6];
                amv<T, FUSED>(u, vc, wm);
#pragma unroll
                for (int k = 0; k < 6; ++k) sb[(6 * mu + k) * nthr + tid] = wm[k];
                ld_soa<T, 6>(vt, F, s3_up[mu], nb);  // v(x+mu, t): L1 hit (this CTA read it as v(t+1) last step)
                mv<T, FUSED>(u, nb, f);
            } else {
                amv<T, FUSED>(u, vc, wt_next);
                mv<T, FUSED>(u, vn, f);
            }
#pragma unroll
            for (int k = 0; k < 6; ++k) acc[k] = (mu == 0) ? f[k] : xadd(acc[k], f[k]);
        }
        __syncthreads();

        // ---- backward terms (sub_four_su3_vecs chain) ----
#pragma unroll
        for (int k = 0; k < 6; ++k) acc[k] = xsub(acc[k], sb[k * nthr + tx_dn]);
        if (ty_dn >= 0) {
#pragma unroll
            for (int k = 0; k < 6; ++k) acc[k] = xsub(acc[k], sb[(6 + k) * nthr + ty_dn]);
        } else {
            T uh[18], vh[6], wh[6];
            ld_soa<T, 18>(p.U + (int64_t(t) * 72 + 18) * F, F, s3_ydn, uh);
            ld_soa<T, 6>(vt, F, s3_ydn, vh);
            amv<T, FUSED>(uh, vh, wh);
#pragma unroll
            for (int k = 0; k < 6; ++k) acc[k] = xsub(acc[k], wh[k]);
        }
        if (tz_dn >= 0) {
#pragma unroll
            for (int k = 0; k < 6; ++k) acc[k] = xsub(acc[k], sb[(12 + k) * nthr + tz_dn]);
        } else {
            T uh[18], vh[6], wh[6];
            ld_soa<T, 18>(p.U + (int64_t(t) * 72 + 36) * F, F, s3_zdn, uh);
            ld_soa<T, 6>(vt, F, s3_zdn, vh);
            amv<T, FUSED>(uh, vh, wh);
#pragma unroll
            for (int k = 0; k < 6; ++k) acc[k] = xsub(acc[k], wh[k]);
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) acc[k] = xsub(acc[k], wt[k]);

        T* o = p.out + int64_t(t) * 6 * F + s3;
#pragma unroll
        for (int k = 0; k < 6; ++k) o[k * F] = acc[k];

#pragma unroll
        for (int k = 0; k < 6; ++k) {
            vc[k] = vn[k];
            wt[k] = wt_next[k];
        }
        buf ^= 1;
      }
    }
}

// block shape (BY, BZ) for the walk kernel; false -> use the generic kernel
static bool walk_shape(int nx, int ny, int nz, int max_threads, int& BY, int& BZ) {
    if (nx > max_threads) return false;
    int best = 0, by = 0, bz = 0;
    double best_halo = 1e30;
    for (int a = 1; a <= ny; ++a) {
        if (ny % a) continue;
        for (int b = 1; b <= nz; ++b) {
            if (nz % b) continue;
            const int n = nx * a * b;
            if (n > max_threads) continue;
            // halo rows read through L2 per block site (0 if the block spans the extent)
            const double halo = (a == ny ? 0.0 : 1.0 / a) + (b == nz ? 0.0 : 1.0 / b);
            if (n > best || (n == best && halo < best_halo)) {
                best = n; by = a; bz = b; best_halo = halo;
            }
        }
    }
    if (best < 32) return false;
    BY = by;
    BZ = bz;
    return true;
}

static std::atomic<int> g_nn_variant{0};  // 0 auto, 1 generic, 2 walk, 3 TMA walk
static std::atomic<int> g_link_variant{0};  // 0 auto, 1 generic, 2 block walk, 3 ring, 4 plane-split, 5, 6 rows

template <typename T>
static int launch_walk(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                       const T* v_hi, const T* w_lo, int BY, int BZ, int mode, cudaStream_t st) {
    constexpr int MINB = 2;
    WalkParams<T> p{U, v, out, v_hi, w_lo, nx, ny, nz, nt, int64_t(nx) * ny * nz, BY, BZ, ny / BY, t_begin, t_end,
                    0, 0, 0};
    p.nblocks = int64_t(ny / BY) * (nz / BZ);
    const int nthr = nx * BY * BZ;
    const size_t smem = size_t(2) * 18 * nthr * sizeof(T);
    static int per_sm_cache[64][2][2] = {};
    const DeviceInfo& di = device_info();
    const bool fused = mode == SU3G_FMA;
    int& per_sm = per_sm_cache[di.device & 63][sizeof(T) == 8][fused];
    if (per_sm == 0) {
        auto kern = fused ? k_nn_walk<T, true, MINB> : k_nn_walk<T, false, MINB>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 18 * 256 * int(sizeof(T)));
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 256, 2 * 18 * 256 * sizeof(T));
        per_sm = b > 0 ? b : 1;
    }
    // blocks of fewer than 256 threads fit proportionally more CTAs per SM
    const int64_t slots = int64_t(per_sm) * di.num_sms * std::max(1, 256 / nthr);
    p.chunk = pick_chunk(p.nblocks, t_end - t_begin, static_cast<int>(std::min<int64_t>(slots, 1 << 20)));
    p.nitems = p.nblocks * ((t_end - t_begin + p.chunk - 1) / p.chunk);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(p.nitems, slots));
    if (fused) k_nn_walk<T, true, MINB><<<static_cast<unsigned>(grid), nthr, smem, st>>>(p);
    else k_nn_walk<T, false, MINB><<<static_cast<unsigned>(grid), nthr, smem, st>>>(p);
    return check_launch("nn_sweep(walk)");
}

// largest divisor of nz that is <= cap (the z-chunk of the cache-friendly visiting orders)
static int chunk_planes(int nz, int cap) {
    for (int c = std::min(nz, cap); c >= 1; --c)
        if (nz % c == 0) return c;
    return 1;
}

static int check_geom(const char* what, int nx, int ny, int nz, int nt) {
    if (nx < 1 || ny < 1 || nz < 1 || nt < 1) return fail_invalid(std::string(what) + ": lattice extents must be >= 1");
    return SU3G_OK;
}

template <typename T>
static int nn_sweep(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                    const T* v_hi, const T* w_lo, int mode, cudaStream_t st) {
    if (mode != SU3G_EXACT && mode != SU3G_FMA) return fail_invalid("nn_sweep: mode must be SU3G_EXACT or SU3G_FMA");
    if (int rc = check_geom("nn_sweep", nx, ny, nz, nt)) return rc;
    if (t_begin < 0 || t_end > nt || t_begin > t_end) return fail_invalid("nn_sweep: bad t range");
    if (!U || !v || !out) return fail_invalid("nn_sweep: null pointer");
    if (t_begin == t_end) return SU3G_OK;
    int BY = 0, BZ = 0;
    const int variant = g_nn_variant.load();
    // auto policy (measured on B200, profiles/r01): f32 with full-width 64+ x rows -> TMA walk;
    // other f32 lattices -> register walk; f64 -> generic (fewest registers, best occupancy)
    // one or two boundary slices of a t-slab (the halo-dependent launches) go to the generic
    // kernel: a walk kernel would pay a work-item prologue for every single-slice item
    const bool boundary_only = (t_end - t_begin) <= 2 && nt > 2;
    const bool auto_tma = variant == 0 && sizeof(T) == 4 && nx >= 32 && !boundary_only;
    const bool auto_walk = variant == 0 && sizeof(T) == 4 && !boundary_only;
    // the register-staged f64 TMA kernel measured slower than the generic kernel in exact mode
    // (0.58 vs 0.69 of HBM at 64^3x16: 4 warps/SM), so it is opt-in only
    if (variant == 5) {
        const int rc = mode == SU3G_FMA
                           ? launch_nn_tma64<T, true>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st)
                           : launch_nn_tma64<T, false>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, st);
        if (rc != 1) {
            note_kernel("k_nn_tma64");
            return rc;
        }
        if (variant == 5) return fail_invalid("nn_sweep: TMA (register-staged) kernel not applicable to this lattice");
    }
    if (auto_tma || variant == 3) {
        const int rc = launch_nn_tma<T>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, mode, st);
        if (rc != 1) return rc;
        if (variant == 3) return fail_invalid("nn_sweep: TMA kernel not applicable to this lattice");
    }
    if ((auto_walk || variant == 2) && walk_shape(nx, ny, nz, 256, BY, BZ))
    {
        note_kernel(std::string("k_nn_walk<") + (sizeof(T) == 4 ? "f32," : "f64,") + std::to_string(nx) + "x" +
                    std::to_string(BY) + "x" + std::to_string(BZ) + ">");
        return launch_walk<T>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, BY, BZ, mode, st);
    }
    if (variant == 2) return fail_invalid("nn_sweep: walk kernel not applicable to this lattice");
    Geom g{nx, ny, nz, nt, int64_t(nx) * ny * nz};
    const int64_t n = int64_t(t_end - t_begin) * g.F;
    const unsigned gs = static_cast<unsigned>((n + 255) / 256);
    // z-chunked order only pays when one t-slice of operands does not fit comfortably in L2
    // (measured: 64^3 f64 0.64 -> 0.70 of HBM; 32^4 f64, whose slice is 22 MB, slightly prefers t-major)
    const bool big_slice = double(g.F) * 84 * sizeof(T) > 0.5 * double(device_info().l2_bytes);
    int ZC = (variant == 4 || !big_slice) ? nz : chunk_planes(nz, 8);  // 4: t-major order (A/B knob)
    if (g_sweep_zc > 0) ZC = chunk_planes(nz, g_sweep_zc);
    if (variant == 6) {  // occupancy A/B knob: register cap for 3 CTAs (24 warps) per SM
        if (mode == SU3G_FMA) k_nn_sweep_capped<T, true, 3><<<gs, 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC);
        else k_nn_sweep_capped<T, false, 3><<<gs, 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC);
        note_kernel("k_nn_sweep_capped<3 CTAs/SM>");
        return check_launch("nn_sweep");
    }
    // L2 prefetch one wave ahead (sweep_prefetch): needs each CTA's sites to be one s3 run
    int ahead = 0;
    if (g_sweep_prefetch > 0 && (int64_t(nx) * ny) % 256 == 0 && (aligned16(U) && aligned16(v))) {
        int per_sm = 0;
        if (mode == SU3G_FMA) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_nn_sweep<T, true>, 256, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_nn_sweep<T, false>, 256, 0);
        ahead = std::max(1, std::max(per_sm, 1) * device_info().num_sms * g_sweep_prefetch / 4);
    }
    if (g_sweep_hints && g_sweep_keep) {
        if (mode == SU3G_FMA) k_nn_sweep<T, true, true, true><<<gs, 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC, ahead);
        else k_nn_sweep<T, false, true, true><<<gs, 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC, ahead);
    } else if (g_sweep_hints) {
        if (mode == SU3G_FMA) k_nn_sweep<T, true, true><<<gs, 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC, ahead);
        else k_nn_sweep<T, false, true><<<gs, 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC, ahead);
    } else {
        if (mode == SU3G_FMA) k_nn_sweep<T, true><<<gs, 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC, ahead);
        else k_nn_sweep<T, false><<<gs, 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC, ahead);
    }
    note_kernel(std::string("k_nn_sweep<") + (sizeof(T) == 4 ? "f32" : "f64") + ",zchunk " + std::to_string(ZC) + ">");
    return check_launch("nn_sweep");
}

template <typename T>
static int nn_halo_w(const T* U, const T* v, T* w, int nx, int ny, int nz, int nt, int mode, cudaStream_t st) {
    if (mode != SU3G_EXACT && mode != SU3G_FMA) return fail_invalid("nn_halo_w: mode must be SU3G_EXACT or SU3G_FMA");
    if (int rc = check_geom("nn_halo_w", nx, ny, nz, nt)) return rc;
    if (!U || !v || !w) return fail_invalid("nn_halo_w: null pointer");
    Geom g{nx, ny, nz, nt, int64_t(nx) * ny * nz};
    const unsigned gs = static_cast<unsigned>((g.F + 255) / 256);
    if (mode == SU3G_FMA) k_nn_halo_w<T, true><<<gs, 256, 0, st>>>(U, v, w, g);
    else k_nn_halo_w<T, false><<<gs, 256, 0, st>>>(U, v, w, g);
    return check_launch("nn_halo_w");
}

template <typename T>
static int nn_sweep(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                    const T* v_hi, const T* w_lo, int mode, cudaStream_t st);

template <typename T>
static int nn_edges(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, const T* v_hi, const T* w_lo,
                    T* w_next, int mode, cudaStream_t st) {
    if (int rc = check_geom("nn_edges", nx, ny, nz, nt)) return rc;
    if (mode != SU3G_EXACT && mode != SU3G_FMA) return fail_invalid("nn_edges: mode must be SU3G_EXACT or SU3G_FMA");
    if (!U || !v || !out) return fail_invalid("nn_edges: null pointer");
    if (out == v) return fail_invalid("nn_edges: out must not alias v");
    Geom g{nx, ny, nz, nt, int64_t(nx) * ny * nz};
    const int nedge = nt > 1 ? 2 : 1;
    const unsigned gs = static_cast<unsigned>((nedge * g.F + 255) / 256);
    const bool fma = mode == SU3G_FMA;
    if (g_sweep_hints) {
        if (fma) k_nn_edges<T, true, true><<<gs, 256, 0, st>>>(U, v, out, g, v_hi, w_lo, w_next, nedge);
        else k_nn_edges<T, false, true><<<gs, 256, 0, st>>>(U, v, out, g, v_hi, w_lo, w_next, nedge);
    } else {
        if (fma) k_nn_edges<T, true, false><<<gs, 256, 0, st>>>(U, v, out, g, v_hi, w_lo, w_next, nedge);
        else k_nn_edges<T, false, false><<<gs, 256, 0, st>>>(U, v, out, g, v_hi, w_lo, w_next, nedge);
    }
    note_kernel(std::string("k_nn_edges<") + (sizeof(T) == 4 ? "f32" : "f64") + ">");
    return check_launch("nn_edges");
}

template <typename T>
static int dslash(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int parity, int mode,
                  cudaStream_t st, T* scratch = nullptr) {
    if (int rc = check_geom("dslash", nx, ny, nz, nt)) return rc;
    if ((nx | ny | nz | nt) & 1) return fail_invalid("dslash: every lattice extent must be even (checkerboard)");
    if (parity != 0 && parity != 1) return fail_invalid("dslash: parity must be 0 (even) or 1 (odd)");
    if (mode != SU3G_EXACT && mode != SU3G_FMA) return fail_invalid("dslash: mode must be SU3G_EXACT or SU3G_FMA");
    if (!U || !v || !out) return fail_invalid("dslash: null pointer");
    if (out == v) return fail_invalid("dslash: out must not alias v");
    Geom g{nx, ny, nz, nt, int64_t(nx) * ny * nz};
    // f32 lattices with a TMA geometry: the parity-restricted TMA t-walk (same values, t-walk speed)
    if (sizeof(T) == 4 && g_nn_variant.load() == 0) {
        const int rc = launch_dslash_tma<T>(U, v, out, nx, ny, nz, nt, parity, mode, st);
        if (rc != 1) {
            if (rc == SU3G_OK) note_kernel(std::string("dslash: ") + su3g_last_kernel() + " (parity mode)");
            return rc;
        }
    }
    // workspace path (f32, where the TMA t-walk applies): the full sweep into scratch with the TMA
    // kernel, then the requested parity copied out -- bitwise the same values, and faster than the
    // one-thread-per-site parity kernel although it computes both parities (64^3x16 f32)
    if (scratch != nullptr && sizeof(T) == 4 && nx >= 32 && g_nn_variant.load() == 0) {
        if (scratch == v || scratch == out) return fail_invalid("dslash: scratch must not alias v or out");
        if (int rc = nn_sweep<T>(U, v, scratch, nx, ny, nz, nt, 0, nt, nullptr, nullptr, mode, st)) return rc;
        const std::string used = std::string("dslash via ") + su3g_last_kernel() + " + k_parity_copy";
        const unsigned gc = static_cast<unsigned>(((g.F >> 1) * nt + 255) / 256);
        k_parity_copy<T><<<gc, 256, 0, st>>>(scratch, out, g, parity);
        note_kernel(used);
        return check_launch("dslash(parity copy)");
    }
    const bool big_slice = double(g.F) * 72 * sizeof(T) > 0.5 * double(device_info().l2_bytes);
    int ZC = big_slice ? chunk_planes(nz, 8) : nz;
    if (g_sweep_zc > 0) ZC = chunk_planes(nz, g_sweep_zc);
    const unsigned gs = static_cast<unsigned>(((g.F >> 1) * nt + 255) / 256);
    int ahead = 0;
    if (g_sweep_prefetch > 0 && (int64_t(nx / 2) * ny) % 256 == 0 && aligned16(U) && aligned16(v)) {
        int per_sm = 0;
        if (mode == SU3G_FMA) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dslash<T, true>, 256, 0);
        else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dslash<T, false>, 256, 0);
        ahead = std::max(1, std::max(per_sm, 1) * device_info().num_sms * g_sweep_prefetch / 4);
    }
    if (g_sweep_hints) {
        if (mode == SU3G_FMA) k_dslash<T, true, true><<<gs, 256, 0, st>>>(U, v, out, g, parity, ZC, ahead);
        else k_dslash<T, false, true><<<gs, 256, 0, st>>>(U, v, out, g, parity, ZC, ahead);
    } else {
        if (mode == SU3G_FMA) k_dslash<T, true><<<gs, 256, 0, st>>>(U, v, out, g, parity, ZC, ahead);
        else k_dslash<T, false><<<gs, 256, 0, st>>>(U, v, out, g, parity, ZC, ahead);
    }
    note_kernel(std::string("k_dslash<") + (sizeof(T) == 4 ? "f32" : "f64") + ",zchunk " + std::to_string(ZC) + ">");
    return check_launch("dslash");
}

template <typename T>
static int link_product(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, int mode, cudaStream_t st) {
    if (int rc = check_geom("link_product", nx, ny, nz, nt)) return rc;
    if (!U || !acc) return fail_invalid("link_product: null pointer");
    if (mode != SU3G_EXACT && mode != SU3G_FMA) return fail_invalid("link_product: mode must be SU3G_EXACT or SU3G_FMA");
    Geom g{nx, ny, nz, nt, int64_t(nx) * ny * nz};
    int BY = 0, BZ = 0;
    const int lv = g_link_variant.load();
    if (lv == 4) {
        return mode == SU3G_FMA ? launch_link_planes<T, true>(U, acc, nx, ny, nz, nt, s, st)
                                : launch_link_planes<T, false>(U, acc, nx, ny, nz, nt, s, st);
    }
    if (lv == 3) {
        const int rc = mode == SU3G_FMA ? launch_link_ring<T, true>(U, acc, nx, ny, nz, nt, s, st)
                                        : launch_link_ring<T, false>(U, acc, nx, ny, nz, nt, s, st);
        if (rc != 1) return rc;
        if (lv == 3) return fail_invalid("link_product: ring kernel not applicable to this lattice");
    }
    if (lv == 2 && walk_shape(nx, ny, nz, 128, BY, BZ)) {
        LinkWalk w{BY, BZ, ny / BY, int64_t(ny / BY) * (nz / BZ), 0, 0};
        const int nthr = nx * BY * BZ;
        static int per_sm_cache[64][2][2] = {};
        const DeviceInfo& di = device_info();
        int& per_sm = per_sm_cache[di.device & 63][sizeof(T) == 8][mode == SU3G_FMA];
        if (per_sm == 0) {
            int b = 0;
            if (mode == SU3G_FMA) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_link_walk<T, true>, nthr, 0);
            else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_link_walk<T, false>, nthr, 0);
            per_sm = b > 0 ? b : 1;
        }
        const int G = per_sm * di.num_sms;
        w.chunk = pick_chunk(w.nblocks, nt, G);
        w.nitems = w.nblocks * ((nt + w.chunk - 1) / w.chunk);
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>(G, w.nitems));
        if (mode == SU3G_FMA) k_link_walk<T, true><<<grid, nthr, 0, st>>>(U, acc, g, w, s);
        else k_link_walk<T, false><<<grid, nthr, 0, st>>>(U, acc, g, w, s);
        note_kernel("k_link_walk");
        return check_launch("link_product(walk)");
    }
    const int64_t n = g.F * nt;
    const unsigned grid = static_cast<unsigned>((n + 127) / 128);
    // z-planes per chunk: 16 measured best for the rows kernel at 48^4 f64 (exact 0.427 -> 0.455,
    // FMA 0.475 -> 0.506 against the unchunked order; 2, 4, 12 also swept).  Chunk once a t-slice of
    // links is more than 1/8 of L2 (48^3 f64 = 64 MB, about half of L2, was left unchunked before).
    const bool link_chunk = double(g.F) * 72 * sizeof(T) > 0.125 * double(device_info().l2_bytes);
    int ZC = link_chunk ? chunk_planes(nz, 16) : nz;
    if (g_link_variant.load() == 5) ZC = nz;  // natural t-major order (A/B knob)
    if (g_link_zc > 0) ZC = chunk_planes(nz, g_link_zc);  // A/B knob: z-planes per chunk
    if (lv == 10) {  // 8x4x4 t-walk, U_3 through L2 (A/B)
        const int rc = mode == SU3G_FMA ? launch_link_tw4<T, true>(U, acc, g, s, st)
                                        : launch_link_tw4<T, false>(U, acc, g, s, st);
        if (rc != 1) return rc;
        return fail_invalid("link_product: 8x4x4 t-walk kernel not applicable to this lattice");
    }
    if (lv == 9) {  // three lanes per site (A/B)
        note_kernel(std::string("k_link_rows3<") + (sizeof(T) == 4 ? "f32" : "f64") + ",zchunk " + std::to_string(ZC) + ">");
        return mode == SU3G_FMA ? launch_link_rows3<T, true>(U, acc, g, s, ZC, st)
                                : launch_link_rows3<T, false>(U, acc, g, s, ZC, st);
    }
    if (lv == 8) {  // TMA-staged t-walk (A/B)
        const int rc = mode == SU3G_FMA ? launch_link_tw<T, true>(U, acc, g, s, st)
                                        : launch_link_tw<T, false>(U, acc, g, s, st);
        if (rc != 1) return rc;
        return fail_invalid("link_product: t-walk kernel not applicable to this lattice");
    }
    if (lv == 7) {  // TMA-staged site tiles (A/B)
        const int rc = mode == SU3G_FMA ? launch_link_tile<T, true>(U, acc, g, s, st)
                                        : launch_link_tile<T, false>(U, acc, g, s, st);
        if (rc != 1) return rc;
        return fail_invalid("link_product: tile kernel not applicable to this lattice");
    }
    // default (auto) = the low-register rows kernel: 16 warps/SM instead of 8 for f64
    // (48^4 f64, same box: exact 0.323 -> 0.426 of HBM, FMA 0.406 -> 0.465)
    if (lv == 0 || lv == 6) {
        note_kernel(std::string("k_link_rows<") + (sizeof(T) == 4 ? "f32" : "f64") + ",zchunk " + std::to_string(ZC) + ">");
        return mode == SU3G_FMA ? launch_link_rows<T, true>(U, acc, g, s, ZC, st)
                                : launch_link_rows<T, false>(U, acc, g, s, ZC, st);
    }
    if (mode == SU3G_FMA) k_link_product<T, true><<<grid, 128, 0, st>>>(U, acc, g, s, ZC);
    else k_link_product<T, false><<<grid, 128, 0, st>>>(U, acc, g, s, ZC);
    note_kernel(std::string("k_link_product<") + (sizeof(T) == 4 ? "f32" : "f64") + ",zchunk " + std::to_string(ZC) + ">");
    return check_launch("link_product");
}

}  // namespace su3g

using namespace su3g;

extern "C" {

int su3g_set_option(const char* name, int64_t value) {
    if (name == nullptr) return fail_invalid("set_option: null name");
    if (std::strcmp(name, "nn_variant") == 0) {
        if (value < 0 || value > 6)
            return fail_invalid(
                "set_option: nn_variant must be 0 (auto), 1 (generic), 2 (walk), 3 (tma walk), 4 (generic, t-major), "
                "5 (tma walk, register-staged), 6 (generic, 3 CTAs/SM register cap)");
        g_nn_variant.store(static_cast<int>(value));
        return SU3G_OK;
    }
    if (std::strcmp(name, "dslash_eo_zc") == 0) {
        if (value < 0 || value > (1 << 20)) return fail_invalid("set_option: dslash_eo_zc must be >= 0");
        g_eo_zc = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "dslash_eo_hints") == 0) {
        if (value != 0 && value != 1) return fail_invalid("set_option: dslash_eo_hints must be 0 or 1");
        g_eo_hints = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "nn_tma_chunk") == 0) {
        if (value < 0 || value > (1 << 20)) return fail_invalid("set_option: nn_tma_chunk must be >= 0");
        g_tma_chunk = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "chunk_prologue_x10") == 0) {
        if (value < 0 || value > 100) return fail_invalid("set_option: chunk_prologue_x10 must be in [0, 100]");
        g_prologue_cost = double(value) / 10.0;
        return SU3G_OK;
    }
    if (std::strcmp(name, "nn_tma_threads") == 0) {
        if (value != 0 && value != 128 && value != 256) return fail_invalid("set_option: nn_tma_threads must be 0, 128 or 256");
        g_tma_threads = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "sm_reserve") == 0) {
        if (value < 0 || value > 64) return fail_invalid("set_option: sm_reserve must be in [0, 64]");
        set_sm_reserve(static_cast<int>(value));
        return SU3G_OK;
    }
    if (std::strcmp(name, "link_minb") == 0) {
        if (value != 0 && value != 3 && value != 4 && value != 5 && value != 6 && value != 8)
            return fail_invalid("set_option: link_minb must be 0 (default), 3, 4, 5, 6 or 8");
        g_link_minb = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "nn_tma_l2_hints") == 0) {
        if (value != 0 && value != 1) return fail_invalid("set_option: nn_tma_l2_hints must be 0 or 1");
        g_tma_hints = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "link_l1_hints") == 0) {
        if (value != 0 && value != 1) return fail_invalid("set_option: link_l1_hints must be 0 or 1");
        g_link_l1_hints = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "link_l2_hints") == 0) {
        if (value != 0 && value != 1) return fail_invalid("set_option: link_l2_hints must be 0 or 1");
        g_link_hints = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "sweep_l2_hints") == 0) {
        if (value != 0 && value != 1) return fail_invalid("set_option: sweep_l2_hints must be 0 or 1");
        g_sweep_hints = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "sweep_l2_keep") == 0) {
        if (value != 0 && value != 1) return fail_invalid("set_option: sweep_l2_keep must be 0 or 1");
        g_sweep_keep = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "sweep_prefetch") == 0) {
        if (value < 0 || value > 16) return fail_invalid("set_option: sweep_prefetch must be in [0, 16]");
        g_sweep_prefetch = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "sweep_zc") == 0) {
        if (value < 0 || value > 4096) return fail_invalid("set_option: sweep_zc must be in [0, 4096]");
        g_sweep_zc = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "link_prefetch_b") == 0) {
        if (value != 0 && value != 1) return fail_invalid("set_option: link_prefetch_b must be 0 or 1");
        g_link_pref_b = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "link_rows3_minb") == 0) {
        if (value != 0 && value != 4 && value != 5 && value != 6 && value != 8)
            return fail_invalid("set_option: link_rows3_minb must be 0 (default 6), 4, 5, 6 or 8");
        g_link_rows3_minb = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "link_tw_chunk") == 0) {
        if (value < 0 || value > (1 << 20)) return fail_invalid("set_option: link_tw_chunk must be >= 0");
        g_link_tw_chunk = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "link_zc") == 0) {
        if (value < 0 || value > 4096) return fail_invalid("set_option: link_zc must be in [0, 4096]");
        g_link_zc = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "link_early_c") == 0) {
        if (value < -1 || value > 1) return fail_invalid("set_option: link_early_c must be -1 (default), 0 or 1");
        g_link_early_c = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "link_variant") == 0) {
        if (value < 0 || value > 10)
            return fail_invalid(
                "set_option: link_variant must be 0 (auto), 1 (generic), 2 (block walk), 3 (ring), 4 (planes), "
                "5 (generic, natural order), 6 (low-register rows), 7 (TMA site tiles), 8 (TMA t-walk), "
                "9 (three lanes per site), 10 (8x4x4 t-walk, U_3 via L2)");
        g_link_variant.store(static_cast<int>(value));
        return SU3G_OK;
    }
    return fail_invalid(std::string("set_option: unknown option ") + name);
}

int su3g_nn_sweep_f32(const float* U, const float* v, float* out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                      int32_t t_begin, int32_t t_end, const float* v_hi, const float* w_lo, int32_t mode,
                      su3g_stream_t st) {
    return nn_sweep<float>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, mode,
                           reinterpret_cast<cudaStream_t>(st));
}
int su3g_nn_sweep_f64(const double* U, const double* v, double* out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                      int32_t t_begin, int32_t t_end, const double* v_hi, const double* w_lo, int32_t mode,
                      su3g_stream_t st) {
    return nn_sweep<double>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, mode,
                            reinterpret_cast<cudaStream_t>(st));
}
int su3g_nn_halo_w_f32(const float* U, const float* v, float* w, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                       int32_t mode, su3g_stream_t st) {
    return nn_halo_w<float>(U, v, w, nx, ny, nz, nt, mode, reinterpret_cast<cudaStream_t>(st));
}
int su3g_nn_halo_w_f64(const double* U, const double* v, double* w, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                       int32_t mode, su3g_stream_t st) {
    return nn_halo_w<double>(U, v, w, nx, ny, nz, nt, mode, reinterpret_cast<cudaStream_t>(st));
}
int su3g_link_product_f32(const float* U, float* acc, int32_t nx, int32_t ny, int32_t nz, int32_t nt, float s,
                          int32_t mode, su3g_stream_t st) {
    return link_product<float>(U, acc, nx, ny, nz, nt, s, mode, reinterpret_cast<cudaStream_t>(st));
}
int su3g_link_product_f64(const double* U, double* acc, int32_t nx, int32_t ny, int32_t nz, int32_t nt, double s,
                          int32_t mode, su3g_stream_t st) {
    return link_product<double>(U, acc, nx, ny, nz, nt, s, mode, reinterpret_cast<cudaStream_t>(st));
}
int su3g_nn_sweep_edges_f32(const float* U, const float* v, float* out, int32_t nx, int32_t ny, int32_t nz,
                            int32_t nt, const float* v_hi, const float* w_lo, float* w_next, int32_t mode,
                            su3g_stream_t st) {
    return nn_edges<float>(U, v, out, nx, ny, nz, nt, v_hi, w_lo, w_next, mode, reinterpret_cast<cudaStream_t>(st));
}
int su3g_nn_sweep_edges_f64(const double* U, const double* v, double* out, int32_t nx, int32_t ny, int32_t nz,
                            int32_t nt, const double* v_hi, const double* w_lo, double* w_next, int32_t mode,
                            su3g_stream_t st) {
    return nn_edges<double>(U, v, out, nx, ny, nz, nt, v_hi, w_lo, w_next, mode, reinterpret_cast<cudaStream_t>(st));
}
int su3g_dslash_f32(const float* U, const float* v, float* out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                    int32_t parity, int32_t mode, su3g_stream_t st) {
    return dslash<float>(U, v, out, nx, ny, nz, nt, parity, mode, reinterpret_cast<cudaStream_t>(st));
}
int su3g_dslash_f64(const double* U, const double* v, double* out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                    int32_t parity, int32_t mode, su3g_stream_t st) {
    return dslash<double>(U, v, out, nx, ny, nz, nt, parity, mode, reinterpret_cast<cudaStream_t>(st));
}
int su3g_dslash_ws_f32(const float* U, const float* v, float* out, float* scratch, int32_t nx, int32_t ny, int32_t nz,
                       int32_t nt, int32_t parity, int32_t mode, su3g_stream_t st) {
    return dslash<float>(U, v, out, nx, ny, nz, nt, parity, mode, reinterpret_cast<cudaStream_t>(st), scratch);
}
int su3g_dslash_ws_f64(const double* U, const double* v, double* out, double* scratch, int32_t nx, int32_t ny,
                       int32_t nz, int32_t nt, int32_t parity, int32_t mode, su3g_stream_t st) {
    return dslash<double>(U, v, out, nx, ny, nz, nt, parity, mode, reinterpret_cast<cudaStream_t>(st), scratch);
}

}  // extern "C"
