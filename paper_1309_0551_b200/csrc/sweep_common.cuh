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

inline int pick_chunk(int64_t nblocks, int nt_range, int G, double prologue = -1.0) {
    const double cost = prologue >= 0 ? prologue : g_prologue_cost;
    int best_L = nt_range;
    double best_eff = -1;
    for (int L = nt_range; L >= 1; --L) {
        const int64_t nchunks = (nt_range + L - 1) / L;
        const int64_t items = nblocks * nchunks;
        const int64_t per = (items + G - 1) / G;
        const double work = double(nblocks) * nt_range;
        const double eff = work / (double(per) * G * L) * (L / (L + cost));
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best_L = L;
        }
    }
    return best_L;
}


// Work-item schedule of the persistent t-walks (ring NN sweep, checkerboarded dslash, factored link
// product).  A walk's items are (block, t-range); an item's prologue costs `prologue` steps and re-reads a
// slice.  Uniform: every block is cut into t-chunks of `chunk`, items chunk-major.  Columns: whole rounds
// of G blocks walk all L slices as one item each (the first n_full items), the remaining blocks are cut
// into t-chunks, chunk-major, and fill the last round(s).  The cheaper of the two by the round count.
struct WalkSchedule {
    int64_t n_full;  // leading whole-column items (0: uniform)
    int chunk;       // t-chunk length of the other blocks' items
    int64_t nitems;
};

inline WalkSchedule pick_schedule(int64_t nblocks, int L, int G, double prologue, bool columns) {
    WalkSchedule w{0, pick_chunk(nblocks, L, G, prologue), 0};
    const int64_t n_full = (nblocks / G) * G, nbt = nblocks - n_full;
    if (columns && n_full > 0) {
        const int64_t items_u = nblocks * ((L + w.chunk - 1) / w.chunk);
        const double cost_uniform = double((items_u + G - 1) / G) * (w.chunk + prologue);
        double cost_cols = double(n_full / G) * (L + prologue);
        int Lt = L;
        if (nbt > 0) {
            Lt = pick_chunk(nbt, L, G, prologue);
            const int64_t items_t = nbt * ((L + Lt - 1) / Lt);
            cost_cols += double((items_t + G - 1) / G) * (Lt + prologue);
        }
        if (cost_cols < cost_uniform) {
            w.n_full = n_full;
            w.chunk = Lt;
        }
    }
    w.nitems = w.n_full + (nblocks - w.n_full) * ((L + w.chunk - 1) / w.chunk);
    return w;
}

// item -> (block, [t0, t1)) of a schedule over slices [lo, hi)
__host__ __device__ __forceinline__ void schedule_item(int64_t n_full, int64_t nblocks, int chunk, int lo, int hi, int64_t item,
                                              int64_t& blk, int& t0, int& t1) {
    if (item < n_full) {
        blk = item;
        t0 = lo;
        t1 = hi;
        return;
    }
    const int64_t r = item - n_full, nbt = nblocks - n_full;
    const int64_t ch = r / nbt;
    blk = n_full + (r - ch * nbt);
    t0 = lo + static_cast<int>(ch) * chunk;
    t1 = t0 + chunk < hi ? t0 + chunk : hi;
}

extern int g_ring_columns;  // su3g_set_option("nn_ring_columns"): the columns schedule of the ring walks (A/B)

// TMA-staged t-walk NN sweep (nn_tma.cu); returns SU3G_EINVAL-style status, or
// 1 when the lattice does not meet its constraints (caller falls back).
template <typename T>
int launch_nn_tma(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                  const T* v_hi, const T* w_lo, int mode, cudaStream_t st);

// warp-specialised TMA ring t-walk (nn_ring.cu; the f64 path); 1 = not applicable
// even/odd dslash on checkerboarded fields, ring walk on the half-lattice (dslash_ring.cu); 1 = not applicable
template <typename T>
int launch_dslash_ring(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int parity, int mode,
                       cudaStream_t st);
template <typename T>
int launch_nn_ring_edges(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, const T* v_hi, const T* w_lo,
                         T* w_next, int mode, cudaStream_t st);
template <typename T>
int launch_nn_ring(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int t_begin, int t_end,
                   const T* v_hi, const T* w_lo, int mode, cudaStream_t st);
template <typename T>
int launch_dslash_tma(const T* U, const T* v, T* out, int nx, int ny, int nz, int nt, int parity, int mode,
                      cudaStream_t st);
// row-split t-walk with carried t-planes (link_walk.cu); 1 = not applicable
template <typename T, bool FUSED>
int launch_link_walk(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, cudaStream_t st);
// two lanes per site, FMA mode, the factored form sum_mu U_mu(x) sum_nu U_nu(x+mu) U_mu(x+nu)^dag, nine
// products per site (link_walk.cu); 1 = not applicable
template <typename T>
int launch_link_fact(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, cudaStream_t st);
template <typename T, bool FUSED>
int launch_link_rows(const T* U, T* acc, const Geom& g, T s, int ZC, cudaStream_t st);

}  // namespace su3g
