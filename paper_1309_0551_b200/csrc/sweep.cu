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
int g_sweep_zc = 0;  // su3g_set_option("sweep_zc"): z-planes per chunk of the generic NN / dslash kernels
// su3g_set_option("sweep_l2_hints"): evict-first backward gathers, streaming stores.  Default on:
// f64 64^3x16 0.686 -> 0.736 of HBM, 32^4 0.711 -> 0.777, dslash f64 0.569 -> 0.642 (same box A/B)
int g_sweep_hints = 1;
extern int g_tma_hints;
extern int g_ring_cfg;
extern int g_tma_chunk;
extern int g_eo_zc;
extern int g_eo_variant;
extern int g_eo_ring_cfg;
extern int g_eo_hints;

// ---------------------------------------------------------------------------
// NN sweep, one thread per site
// ---------------------------------------------------------------------------
template <typename T, bool FUSED, bool HINTS = false>
__device__ __forceinline__ void nn_sweep_body(const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ out,
                                              const Geom& g, int t_begin, int t_end, const T* __restrict__ v_hi,
                                              const T* __restrict__ w_lo, int ZC) {
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
    nn_site<T, FUSED, HINTS>(U, v, out, g, x, y, z, t, v_hi, w_lo);
}

// plain bounds: ptxas picks 64-98 registers; an explicit minBlocks of 1 would let it take 252
template <typename T, bool FUSED, bool HINTS = false>
__global__ void __launch_bounds__(256)
    k_nn_sweep(const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ out, Geom g, int t_begin, int t_end,
               const T* __restrict__ v_hi, const T* __restrict__ w_lo, int ZC) {
    nn_sweep_body<T, FUSED, HINTS>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC);
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
    k_dslash(const T* __restrict__ U, const T* __restrict__ v, T* __restrict__ out, Geom g, int parity, int ZC) {
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

extern int g_link_chunk;
extern int g_ring_columns;
static std::atomic<int> g_nn_variant{0};  // 0 auto, 1 generic, 3 TMA walk, 4 TMA ring walk
static std::atomic<int> g_link_variant{0};  // 0 auto, 1 rows (gather), 3 row-split carried t-walk, 5 factored two-lane pair walk (FMA)

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
    const int variant = g_nn_variant.load();
    // auto policy (measured on B200, profiles/r02): lattices with x extent 32, 48 or 64 and even y, z
    // -> the TMA ring walk (64^3x16: f32 0.905, f64 0.951 of HBM); other f32 lattices with x rows of
    // 32+ sites -> the f32 TMA walk; the rest -> generic.  One or two boundary slices of a t-slab (the
    // halo-dependent launches) go to the generic kernel: a walk kernel would pay a work-item prologue
    // for every single-slice item
    const bool boundary_only = (t_end - t_begin) <= 2 && nt > 2;
    if ((variant == 0 && !boundary_only) || variant == 4) {
        const int rc = launch_nn_ring<T>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, mode, st);
        if (rc != 1) return rc;
        if (variant == 4) return fail_invalid("nn_sweep: TMA ring kernel not applicable to this lattice");
    }
    const bool auto_tma = variant == 0 && sizeof(T) == 4 && nx >= 32 && !boundary_only;
    if (auto_tma || variant == 3) {
        const int rc = launch_nn_tma<T>(U, v, out, nx, ny, nz, nt, t_begin, t_end, v_hi, w_lo, mode, st);
        if (rc != 1) return rc;
        if (variant == 3) return fail_invalid("nn_sweep: TMA kernel not applicable to this lattice");
    }
    Geom g{nx, ny, nz, nt, int64_t(nx) * ny * nz};
    const int64_t n = int64_t(t_end - t_begin) * g.F;
    const unsigned gs = static_cast<unsigned>((n + 255) / 256);
    // z-chunked order only pays when one t-slice of operands does not fit comfortably in L2
    // (measured: 64^3 f64 0.64 -> 0.70 of HBM; 32^4 f64, whose slice is 22 MB, slightly prefers t-major)
    const bool big_slice = double(g.F) * 84 * sizeof(T) > 0.5 * double(device_info().l2_bytes);
    int ZC = big_slice ? chunk_planes(nz, 8) : nz;
    if (g_sweep_zc > 0) ZC = chunk_planes(nz, g_sweep_zc);
    if (g_sweep_hints) {
        if (mode == SU3G_FMA) k_nn_sweep<T, true, true><<<gs, 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC);
        else k_nn_sweep<T, false, true><<<gs, 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC);
    } else {
        if (mode == SU3G_FMA) k_nn_sweep<T, true><<<gs, 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC);
        else k_nn_sweep<T, false><<<gs, 256, 0, st>>>(U, v, out, g, t_begin, t_end, v_hi, w_lo, ZC);
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
    // the ring walk on one-step items (both boundary slices, same values bit for bit) where it applies
    if (g_nn_variant.load() == 0 || g_nn_variant.load() == 4) {
        const int rc = launch_nn_ring_edges<T>(U, v, out, nx, ny, nz, nt, v_hi, w_lo, w_next, mode, st);
        if (rc != 1) return rc;
    }
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
    if (g_sweep_hints) {
        if (mode == SU3G_FMA) k_dslash<T, true, true><<<gs, 256, 0, st>>>(U, v, out, g, parity, ZC);
        else k_dslash<T, false, true><<<gs, 256, 0, st>>>(U, v, out, g, parity, ZC);
    } else {
        if (mode == SU3G_FMA) k_dslash<T, true><<<gs, 256, 0, st>>>(U, v, out, g, parity, ZC);
        else k_dslash<T, false><<<gs, 256, 0, st>>>(U, v, out, g, parity, ZC);
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
    const int lv = g_link_variant.load();
    // auto (48^4 on B200, fraction of HBM; profiles/r02/ab_link_walk.md, ab_link_pair.txt, ab_link_fact.txt):
    // FMA mode -> the factored two-lane pair walk (f64 0.77, f32 0.63; the removed plane-by-plane pair walk
    // 0.611 / 0.429, the removed ring walk 0.546 / 0.397, rows 0.525 / 0.357);
    // exact f32 -> the row-split carried walk (0.351 vs rows 0.309); exact f64 -> rows (0.465; walk 0.461,
    // an exact pair walk 0.413)
    if (lv == 5 || (lv == 0 && mode == SU3G_FMA)) {
        if (mode != SU3G_FMA) return fail_invalid("link_product: the factored pair walk (link_variant 5) is FMA mode only");
        const int rc = launch_link_fact<T>(U, acc, nx, ny, nz, nt, s, st);
        if (rc != 1) return rc;
        if (lv == 5) return fail_invalid("link_product: factored pair kernel not applicable to this lattice");
    }
    if (lv == 3 || (lv == 0 && sizeof(T) == 4 && mode == SU3G_EXACT)) {
        const int rc = mode == SU3G_FMA ? launch_link_walk<T, true>(U, acc, nx, ny, nz, nt, s, st)
                                        : launch_link_walk<T, false>(U, acc, nx, ny, nz, nt, s, st);
        if (rc != 1) return rc;
        if (lv == 3) return fail_invalid("link_product: row-split walk kernel not applicable to this lattice");
    }
    // z-planes per chunk: 16 measured best for the rows kernel at 48^4 f64 (exact 0.427 -> 0.455,
    // FMA 0.475 -> 0.506 against the unchunked order; 2, 4, 12 also swept).  Chunk once a t-slice of
    // links is more than 1/8 of L2 (48^3 f64 = 64 MB, about half of L2, was left unchunked before).
    const bool link_chunk = double(g.F) * 72 * sizeof(T) > 0.125 * double(device_info().l2_bytes);
    const int ZC = link_chunk ? chunk_planes(nz, 16) : nz;
    note_kernel(std::string("k_link_rows<") + (sizeof(T) == 4 ? "f32" : "f64") + ",zchunk " + std::to_string(ZC) + ">");
    return mode == SU3G_FMA ? launch_link_rows<T, true>(U, acc, g, s, ZC, st)
                            : launch_link_rows<T, false>(U, acc, g, s, ZC, st);
}

}  // namespace su3g

using namespace su3g;

extern "C" {

int su3g_set_option(const char* name, int64_t value) {
    if (name == nullptr) return fail_invalid("set_option: null name");
    if (std::strcmp(name, "nn_variant") == 0) {
        if (value != 0 && value != 1 && value != 3 && value != 4)
            return fail_invalid("set_option: nn_variant must be 0 (auto), 1 (generic), 3 (tma walk) or 4 (tma ring walk)");
        g_nn_variant.store(static_cast<int>(value));
        return SU3G_OK;
    }
    if (std::strcmp(name, "link_variant") == 0) {
        if (value < 0 || value > 5 || value == 2 || value == 4)
            return fail_invalid("set_option: link_variant must be 0 (auto), 1 (rows gather), 3 (row-split walk) or "
                                "5 (factored pair walk, FMA); 2 (the ring walk) and 4 (the plane-by-plane pair "
                                "walk) were removed, measured slower");
        g_link_variant.store(static_cast<int>(value));
        return SU3G_OK;
    }
    if (std::strcmp(name, "dslash_eo_variant") == 0) {
        if (value < 0 || value > 2)
            return fail_invalid("set_option: dslash_eo_variant must be 0 (auto), 1 (gather) or 2 (ring walk)");
        g_eo_variant = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "dslash_eo_ring_cfg") == 0) {
        if (value < 0 || value > 2) return fail_invalid("set_option: dslash_eo_ring_cfg must be in [0, 2]");
        g_eo_ring_cfg = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "link_chunk") == 0) {
        if (value < 0 || value > 4096) return fail_invalid("set_option: link_chunk must be in [0, 4096] (0 = auto)");
        g_link_chunk = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "nn_ring_columns") == 0) {
        if (value < 0 || value > 1) return fail_invalid("set_option: nn_ring_columns must be 0 or 1");
        g_ring_columns = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "nn_ring_cfg") == 0) {
        if (value < 0 || value > 4) return fail_invalid("set_option: nn_ring_cfg must be in [0, 4]");
        g_ring_cfg = static_cast<int>(value);
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
    if (std::strcmp(name, "nn_tma_l2_hints") == 0) {
        if (value != 0 && value != 1) return fail_invalid("set_option: nn_tma_l2_hints must be 0 or 1");
        g_tma_hints = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "sweep_l2_hints") == 0) {
        if (value != 0 && value != 1) return fail_invalid("set_option: sweep_l2_hints must be 0 or 1");
        g_sweep_hints = static_cast<int>(value);
        return SU3G_OK;
    }
    if (std::strcmp(name, "sweep_zc") == 0) {
        if (value < 0 || value > 4096) return fail_invalid("set_option: sweep_zc must be in [0, 4096]");
        g_sweep_zc = static_cast<int>(value);
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
int64_t su3g_walk_schedule(int64_t nblocks, int32_t nslices, int32_t ctas, int32_t prologue_x10, int32_t columns,
                           int64_t item, int64_t* blk, int32_t* t0, int32_t* t1, int64_t* n_full, int32_t* chunk) {
    if (nblocks <= 0 || nslices <= 0 || ctas <= 0 || prologue_x10 < 0) {
        fail_invalid("walk_schedule: nblocks, nslices, ctas must be positive and prologue_x10 non-negative");
        return -1;
    }
    const WalkSchedule w = pick_schedule(nblocks, nslices, ctas, prologue_x10 / 10.0, columns != 0);
    if (n_full) *n_full = w.n_full;
    if (chunk) *chunk = w.chunk;
    if (item >= 0 && item < w.nitems && blk && t0 && t1) {
        int a, b;
        schedule_item(w.n_full, nblocks, w.chunk, 0, nslices, item, *blk, a, b);
        *t0 = a;
        *t1 = b;
    }
    return w.nitems;
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
