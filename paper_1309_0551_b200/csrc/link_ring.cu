// Link-product sweep with a per-thread asynchronous link ring (BASELINE configs[3]).
//
// Per site the product reads 15 links -- U_mu(x) (A) once per mu group and, per
// plane, U_nu(x+mu) (B) and U_mu(x+nu) (C) -- and does ~1.4-2.6 k flops, so the
// one-thread-per-site kernel was bound by the latency of those dependent link
// gathers (ncu: 45-58% long-scoreboard stalls at 12 warps/SM).  Here each thread
// walks the flat sequence (site, link) and keeps R links in flight in a private
// shared-memory ring with cp.async (LDGSTS): link j+R-1 is requested while link
// j is consumed, across site boundaries, so loads never wait on arithmetic.
// No block-level synchronisation is needed (each thread reads only its own
// slots).  Sites are visited on the block-walk schedule (chunk-major items) so
// the +t links a thread gathers as neighbours are L2-resident when needed again.
//
// Arithmetic per element is exactly link_site's (mat_nn then mat_na then
// acc + s*P in plane order), computed row by row: bit-identical in EXACT mode.
#include <algorithm>

#include "sweep_common.cuh"

namespace su3g {

namespace {

// link sequence of one site: (direction of the link, shift direction; -1 = the site itself)
__constant__ int c_link_dir[15] = {0, 1, 0, 2, 0, 3, 0, 1, 2, 1, 3, 1, 2, 3, 2};
__constant__ int c_link_shift[15] = {-1, 0, 1, 0, 2, 0, 3, -1, 1, 2, 1, 3, -1, 2, 3};
// role of link j: 0 = A (new mu group), 1 = B, 2 = C (completes a plane)
__constant__ int c_link_role[15] = {0, 1, 2, 1, 2, 1, 2, 0, 1, 2, 1, 2, 0, 1, 2};

template <typename T>
__device__ __forceinline__ void cp_async_elem(T* dst_smem, const T* src) {
    if constexpr (sizeof(T) == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst_smem)), "l"(src) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst_smem)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct RingParams {
    int nx, ny, nz, nt;
    int64_t F;
    int BY, BZ, nby;
    int64_t nblocks;
    int chunk;
    int64_t nitems;
};

}  // namespace

template <typename T, bool FUSED, int NTHR, int R>
__global__ void __launch_bounds__(NTHR, 3) k_link_ring(const T* __restrict__ U, T* __restrict__ acc_out, RingParams p, T s) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* ring = reinterpret_cast<T*>(smem_raw);  // [R][18][NTHR]
    const int tid = threadIdx.x;
    if (tid >= p.nx * p.BY * p.BZ) return;
    const int lx = tid % p.nx, rr = tid / p.nx, ly = rr % p.BY, lz = rr / p.BY;
    const int64_t F = p.F;

    // ---- flat (site, link) cursor over this CTA's items ------------------------
    struct Cur {
        int64_t item;
        int t, t1, j;
        int x, y, z;
        bool valid;
    };
    auto enter = [&](Cur& c) {
        const int64_t ch = c.item / p.nblocks;
        const int64_t blk = c.item - ch * p.nblocks;
        c.t = static_cast<int>(ch) * p.chunk;
        c.t1 = min(c.t + p.chunk, p.nt);
        c.x = lx;
        c.y = static_cast<int>(blk % p.nby) * p.BY + ly;
        c.z = static_cast<int>(blk / p.nby) * p.BZ + lz;
        c.j = 0;
    };
    auto next = [&](Cur& c) {
        if (++c.j < 15) return;
        c.j = 0;
        if (++c.t < c.t1) return;
        c.item += gridDim.x;
        if (c.item >= p.nitems) {
            c.valid = false;
            return;
        }
        enter(c);
    };
    auto issue = [&](const Cur& c, int slot) {
        if (c.valid) {
            int x = c.x, y = c.y, z = c.z, t = c.t;
            switch (c_link_shift[c.j]) {
                case 0: x = (x + 1 == p.nx) ? 0 : x + 1; break;
                case 1: y = (y + 1 == p.ny) ? 0 : y + 1; break;
                case 2: z = (z + 1 == p.nz) ? 0 : z + 1; break;
                case 3: t = (t + 1 == p.nt) ? 0 : t + 1; break;
                default: break;
            }
            const int64_t s3 = x + int64_t(p.nx) * (y + int64_t(p.ny) * z);
            const T* src = U + (int64_t(t) * 72 + c_link_dir[c.j] * 18) * F + s3;
            T* dst = ring + slot * 18 * NTHR + tid;
#pragma unroll
            for (int k = 0; k < 18; ++k) cp_async_elem(dst + k * NTHR, src + k * F);
        }
        cp_async_commit();  // empty groups keep the wait_group arithmetic uniform
    };

    Cur load{static_cast<int64_t>(blockIdx.x), 0, 0, 0, 0, 0, 0, static_cast<int64_t>(blockIdx.x) < p.nitems};
    if (!load.valid) return;
    enter(load);
    Cur use = load;
#pragma unroll
    for (int q = 0; q < R - 1; ++q) {
        issue(load, q);
        next(load);
    }

    T a[18], tm[18], acc[18];
    int slot = 0;
    while (use.valid) {
        cp_async_wait<R - 2>();  // link `use` has landed in `slot`
        issue(load, (slot + R - 1) % R);
        next(load);
        const T* L = ring + slot * 18 * NTHR + tid;
        const int role = c_link_role[use.j];
        if (use.j == 0) {
#pragma unroll
            for (int k = 0; k < 18; ++k) acc[k] = T(0);
        }
        if (role == 0) {
#pragma unroll
            for (int k = 0; k < 18; ++k) a[k] = L[k * NTHR];
        } else if (role == 1) {
            T b[18];
#pragma unroll
            for (int k = 0; k < 18; ++k) b[k] = L[k * NTHR];
            if (FUSED) mat_nn_fma<T>(a, b, tm);
            else mat_nn<T>(a, b, tm);
        } else {
            T c[18], pm[18];
#pragma unroll
            for (int k = 0; k < 18; ++k) c[k] = L[k * NTHR];
            if (FUSED) mat_na_fma<T>(tm, c, pm);
            else mat_na<T>(tm, c, pm);
#pragma unroll
            for (int k = 0; k < 18; ++k) acc[k] = FUSED ? fma(s, pm[k], acc[k]) : xadd(acc[k], xmul(s, pm[k]));
            if (use.j == 14) {
                const int64_t s3 = use.x + int64_t(p.nx) * (use.y + int64_t(p.ny) * use.z);
#pragma unroll
                for (int k = 0; k < 18; ++k) acc_out[(int64_t(use.t) * 18 + k) * F + s3] = acc[k];
            }
        }
        next(use);
        slot = (slot + 1 == R) ? 0 : slot + 1;
    }
    cp_async_wait<0>();
}

// block shape for the ring kernel: full x rows, <= NTHR sites
static bool ring_shape(int nx, int ny, int nz, int nthr, int& BY, int& BZ) {
    if (nx > nthr) return false;
    int best = 0;
    for (int a = 1; a <= ny; ++a) {
        if (ny % a) continue;
        for (int b = 1; b <= nz; ++b) {
            if (nz % b) continue;
            const int n = nx * a * b;
            if (n <= nthr && n > best) {
                best = n;
                BY = a;
                BZ = b;
            }
        }
    }
    return best >= 32 || best == nx * ny * nz;
}

template <typename T, bool FUSED>
int launch_link_ring(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, cudaStream_t st) {
    constexpr int NTHR = 128, R = 4;
    int BY = 0, BZ = 0;
    if (!ring_shape(nx, ny, nz, NTHR, BY, BZ)) return 1;
    RingParams p{nx, ny, nz, nt, int64_t(nx) * ny * nz, BY, BZ, ny / BY, int64_t(ny / BY) * (nz / BZ), 0, 0};
    const size_t smem = size_t(R) * 18 * NTHR * sizeof(T);
    const DeviceInfo& di = device_info();
    static int per_sm_cache[64] = {0};
    int& per_sm = per_sm_cache[di.device & 63];
    if (per_sm == 0) {
        cudaFuncSetAttribute(k_link_ring<T, FUSED, NTHR, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_link_ring<T, FUSED, NTHR, R>, NTHR, smem);
        per_sm = b > 0 ? b : 1;
    }
    const int G = per_sm * di.num_sms;
    p.chunk = pick_chunk(p.nblocks, nt, G);
    p.nitems = p.nblocks * ((nt + p.chunk - 1) / p.chunk);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(G, p.nitems));
    k_link_ring<T, FUSED, NTHR, R><<<grid, NTHR, smem, st>>>(U, acc, p, s);
    return check_launch("link_product(ring)");
}

// ---------------------------------------------------------------------------
// Plane-split link product: 6 threads per site, one per plane (mu, nu).  Each
// thread issues its three link gathers (A = U_mu(x), B = U_nu(x+mu), C =
// U_mu(x+nu)) at once and computes P = (A B) C^dag row by row; the 6 planes
// of a site meet in shared memory and one thread per (site, component) folds
// them into acc in plane order with exactly link_site's per-element operation
// (exact: acc + s*P; FMA: fma(s, P, acc)) -- bit-identical to the other
// variants in either mode, with 6x the memory-level parallelism per site.
// ---------------------------------------------------------------------------
__constant__ int c_plane_mu[6] = {0, 0, 0, 1, 1, 2};
__constant__ int c_plane_nu[6] = {1, 2, 3, 2, 3, 3};

template <typename T, bool FUSED, int TSITES>
__global__ void __launch_bounds__(6 * TSITES) k_link_planes(const T* __restrict__ U, T* __restrict__ acc_out, int nx,
                                                            int ny, int nz, int nt, T s) {
    __shared__ T P[6][18][TSITES];
    const int64_t F = int64_t(nx) * ny * nz;
    const int64_t V = F * nt;
    const int lane = threadIdx.x % TSITES;
    const int q = threadIdx.x / TSITES;  // plane
    const int mu = c_plane_mu[q], nu = c_plane_nu[q];
    for (int64_t base = int64_t(blockIdx.x) * TSITES; base < V; base += int64_t(gridDim.x) * TSITES) {
        const int64_t site = base + lane;
        if (site < V) {
            const int t = static_cast<int>(site / F);
            const int64_t s3 = site - int64_t(t) * F;
            const int x = static_cast<int>(s3 % nx);
            const int y = static_cast<int>((s3 / nx) % ny);
            const int z = static_cast<int>(s3 / (int64_t(nx) * ny));
            auto link = [&](int dir, int shift, T* r) {
                int xx = x, yy = y, zz = z, tt = t;
                if (shift == 0) xx = (xx + 1 == nx) ? 0 : xx + 1;
                else if (shift == 1) yy = (yy + 1 == ny) ? 0 : yy + 1;
                else if (shift == 2) zz = (zz + 1 == nz) ? 0 : zz + 1;
                else if (shift == 3) tt = (tt + 1 == nt) ? 0 : tt + 1;
                const int64_t ss = xx + int64_t(nx) * (yy + int64_t(ny) * zz);
                const T* src = U + (int64_t(tt) * 72 + dir * 18) * F + ss;
#pragma unroll
                for (int k = 0; k < 18; ++k) r[k] = __ldg(src + k * F);
            };
            T a[18], b[18], c[18], tm[18], pm[18];
            link(mu, -1, a);
            link(nu, mu, b);
            link(mu, nu, c);
            if (FUSED) {
                mat_nn_fma<T>(a, b, tm);
                mat_na_fma<T>(tm, c, pm);
            } else {
                mat_nn<T>(a, b, tm);
                mat_na<T>(tm, c, pm);
            }
#pragma unroll
            for (int k = 0; k < 18; ++k) P[q][k][lane] = pm[k];
        }
        __syncthreads();
        for (int e = threadIdx.x; e < 18 * TSITES; e += 6 * TSITES) {
            const int k = e / TSITES, l = e % TSITES;
            const int64_t st = base + l;
            if (st < V) {
                T acc = T(0);
#pragma unroll
                for (int pq = 0; pq < 6; ++pq) acc = FUSED ? fma(s, P[pq][k][l], acc) : xadd(acc, xmul(s, P[pq][k][l]));
                const int t = static_cast<int>(st / F);
                acc_out[(int64_t(t) * 18 + k) * F + (st - int64_t(t) * F)] = acc;
            }
        }
        __syncthreads();
    }
}

template <typename T, bool FUSED>
int launch_link_planes(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, cudaStream_t st) {
    constexpr int TS = 32;
    const DeviceInfo& di = device_info();
    static int per_sm_cache[64] = {0};
    int& per_sm = per_sm_cache[di.device & 63];
    if (per_sm == 0) {
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_link_planes<T, FUSED, TS>, 6 * TS, 0);
        per_sm = b > 0 ? b : 1;
    }
    const int64_t V = int64_t(nx) * ny * nz * nt;
    const int64_t tiles = (V + TS - 1) / TS;
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(tiles, int64_t(per_sm) * di.num_sms * 8));
    k_link_planes<T, FUSED, TS><<<grid, 6 * TS, 0, st>>>(U, acc, nx, ny, nz, nt, s);
    return check_launch("link_product(planes)");
}

template int launch_link_planes<float, false>(const float*, float*, int, int, int, int, float, cudaStream_t);
template int launch_link_planes<float, true>(const float*, float*, int, int, int, int, float, cudaStream_t);
template int launch_link_planes<double, false>(const double*, double*, int, int, int, int, double, cudaStream_t);
template int launch_link_planes<double, true>(const double*, double*, int, int, int, int, double, cudaStream_t);

template int launch_link_ring<float, false>(const float*, float*, int, int, int, int, float, cudaStream_t);
template int launch_link_ring<float, true>(const float*, float*, int, int, int, int, float, cudaStream_t);
template int launch_link_ring<double, false>(const double*, double*, int, int, int, int, double, cudaStream_t);
template int launch_link_ring<double, true>(const double*, double*, int, int, int, int, double, cudaStream_t);

}  // namespace su3g
