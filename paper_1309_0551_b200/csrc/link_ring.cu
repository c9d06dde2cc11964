// Link-product sweep (BASELINE configs[3]) on a warp-specialised TMA ring t-walk.
//
// acc(x) = sum over the planes (0,1) (0,2) (0,3) (1,2) (1,3) (2,3) of s * U_mu(x) U_nu(x+mu) U_mu(x+nu)^dag,
// in that order.  The one-thread-per-site gather kernel (link_rows.cu)
// pulls ~324 reals per site through L1/L2 for 90 compulsory, and that L2 -> SM traffic, not
// DRAM, bounds it.  Here every link of a slice crosses L2 -> SM about once:
//
//   A CTA owns a block of one t-slice -- the full x extent (x periodic inside the CTA) x 2 y-rows
//   x 2 z-planes, N = 4 NX sites, one compute thread each -- and walks t.  Per step a producer
//   warp streams four "extended link" chunks into four typed slots (4-D TMA boxes, full/empty
//   mbarriers):
//     E0  U_0 of the block [18][N] | U_0 on the +y halo row [18][H] | U_0 on the +z halo row [18][H]
//     E1  U_1 of the block          | U_1 on the +z row
//     E2  U_2 of the block          | U_2 on the +y row
//     E3  U_3 of the block          | U_3 on the +y row           | U_3 on the +z row
//   (H = 2 NX sites per halo row).  Every B = U_nu(x+mu) and every spatial C = U_mu(x+nu) is a
//   shared-memory read.  The C of a t-plane, U_mu(x+t), is this thread's own column one slice up:
//   it is gathered straight into registers (coalesced), two planes ahead of its use -- and that
//   gather is also what warms L2 for the next step's E0..E2 boxes.  The producer warms U_3 of the
//   next slice with a TMA L2 prefetch.
//   A slot is released as soon as its last use is done, and the producer warms L2 with the next
//   step's boxes one step ahead, so the next step's chunk loads are L2 hits.
//
// Per-element arithmetic and the plane/accumulation order are exactly link_rows' (mult_su3_nn,
// then mult_su3_na, then acc + s*P): EXACT mode is bit-identical to the composed reference.
#include <algorithm>
#include <string>

#include "nn_site.cuh"
#include "tma.cuh"

namespace su3g {

namespace {

struct LinkRingParams {
    int ny, nz, nt;
    int64_t F;
    int nby;
    int64_t nblocks;
    int chunk;
    int64_t nitems;
};

template <int NX>
struct LinkGeo {
    static constexpr int N = 4 * NX, H = 2 * NX;
    // slot sizes (reals) and offsets
    static constexpr int SZ0 = 18 * N + 36 * H, SZ1 = 18 * N + 18 * H, SZ2 = SZ1, SZ3 = SZ0;
    static constexpr int OFF0 = 0, OFF1 = SZ0, OFF2 = SZ0 + SZ1, OFF3 = SZ0 + SZ1 + SZ2;
    static constexpr int TOTAL = SZ0 + SZ1 + SZ2 + SZ3;
    // within a slot: block at 0, first halo row at 18N, second halo row at 18N + 18H
    static constexpr int ROW1 = 18 * N, ROW2 = 18 * N + 18 * H;
};

__device__ __forceinline__ void link_item(const LinkRingParams& p, int64_t item, int64_t& blk, int& t0, int& t1) {
    const int64_t ch = item / p.nblocks;
    blk = item - ch * p.nblocks;
    t0 = static_cast<int>(ch) * p.chunk;
    t1 = min(t0 + p.chunk, p.nt);
}

__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* map, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}

// 18 reals of a link from shared memory: element c at p[c * stride]
template <typename T>
__device__ __forceinline__ void ld_link_smem(const T* p, int stride, T* r) {
#pragma unroll
    for (int c = 0; c < 18; ++c) r[c] = p[c * stride];
}

// T = A B (mult_su3_nn arithmetic), B read from shared memory one column at a time (6 live reals)
template <typename T, bool FUSED>
__device__ __forceinline__ void nn_smem_b(const T* a, const T* bs, int bstr, T* tm) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        T bc[6];  // column k: b[j][k], j = 0..2
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            bc[2 * j] = bs[((3 * j + k) * 2) * bstr];
            bc[2 * j + 1] = bs[((3 * j + k) * 2 + 1) * bstr];
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if constexpr (FUSED)
                cdot_fma<T, PLAIN, 3>([&](int j, int q) { return a[(3 * i + j) * 2 + q]; },
                                      [&](int j, int q) { return bc[2 * j + q]; }, tm[(3 * i + k) * 2],
                                      tm[(3 * i + k) * 2 + 1]);
            else
                cdot<T, PLAIN, 3>([&](int j, int q) { return a[(3 * i + j) * 2 + q]; },
                                  [&](int j, int q) { return bc[2 * j + q]; }, tm[(3 * i + k) * 2],
                                  tm[(3 * i + k) * 2 + 1]);
        }
    }
}

// acc (+)= s * T C^dag (mult_su3_na, then scalar_mult_add arithmetic); C row k at c(k, j, q);
// FIRST: acc = 0 + s*P, the reference's zero-initialised accumulation
template <typename T, bool FUSED, bool FIRST, class CF>
__device__ __forceinline__ void na_acc(const T* tm, CF c, T s, T* acc) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        T cr[6];  // row k: c[k][j], j = 0..2
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            cr[2 * j] = c(k, j, 0);
            cr[2 * j + 1] = c(k, j, 1);
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            T pr, pi;
            if constexpr (FUSED)
                cdot_fma<T, CONJ_Q, 3>([&](int j, int q) { return tm[(3 * i + j) * 2 + q]; },
                                       [&](int j, int q) { return cr[2 * j + q]; }, pr, pi);
            else
                cdot<T, CONJ_Q, 3>([&](int j, int q) { return tm[(3 * i + j) * 2 + q]; },
                                   [&](int j, int q) { return cr[2 * j + q]; }, pr, pi);
            const int e = (3 * i + k) * 2;
            if constexpr (FIRST) {
                acc[e] = FUSED ? fma(s, pr, T(0)) : xadd(T(0), xmul(s, pr));
                acc[e + 1] = FUSED ? fma(s, pi, T(0)) : xadd(T(0), xmul(s, pi));
            } else {
                acc[e] = FUSED ? fma(s, pr, acc[e]) : xadd(acc[e], xmul(s, pr));
                acc[e + 1] = FUSED ? fma(s, pi, acc[e + 1]) : xadd(acc[e + 1], xmul(s, pi));
            }
        }
    }
}

}  // namespace

template <typename T, bool FUSED, int NX, int MINB>
__global__ void __launch_bounds__(4 * NX + 32, MINB)
    k_link_ring(const __grid_constant__ CUtensorMap mapU, const __grid_constant__ CUtensorMap mapUy,
                const __grid_constant__ CUtensorMap mapUz, const T* __restrict__ U, T* __restrict__ acc_out,
                LinkRingParams p, T s) {
    using G = LinkGeo<NX>;
    constexpr int N = G::N, H = G::H, NW = N / 32;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + G::TOTAL);
    uint64_t* empty = full + 4;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int k = 0; k < 4; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], NW);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t F = p.F;
    const int GR = gridDim.x;
    T* const E0 = sm + G::OFF0;
    T* const E1 = sm + G::OFF1;
    T* const E2 = sm + G::OFF2;
    T* const E3 = sm + G::OFF3;

    // ------------------------------------------------------------------ producer warp
    if (tid >= N) {
        if (tid != N) return;
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
        uint32_t n = 0;  // steps issued
        for (int64_t item = blockIdx.x; item < p.nitems; item += GR) {
            int64_t blk;
            int t0, t1;
            link_item(p, item, blk, t0, t1);
            const int y0 = static_cast<int>(blk % p.nby) * 2, z0 = static_cast<int>(blk / p.nby) * 2;
            const int yup = (y0 + 2) % p.ny, zup = (z0 + 2) % p.nz;
            for (int t = t0; t < t1; ++t, ++n) {
                const int tn = (t + 1 == p.nt) ? 0 : t + 1;
                // warm L2 with the next step's boxes (the consumers' own-column gathers cover U_0..U_2 of
                // the block; U_3 and the halo rows are not touched otherwise)
                tma_prefetch_4d(&mapU, 0, y0, z0, tn * 72 + 54);
                tma_prefetch_4d(&mapUy, 0, yup, z0, tn * 72);
                tma_prefetch_4d(&mapUy, 0, yup, z0, tn * 72 + 36);
                tma_prefetch_4d(&mapUy, 0, yup, z0, tn * 72 + 54);
                tma_prefetch_4d(&mapUz, 0, y0, zup, tn * 72);
                tma_prefetch_4d(&mapUz, 0, y0, zup, tn * 72 + 18);
                tma_prefetch_4d(&mapUz, 0, y0, zup, tn * 72 + 54);
                const uint32_t par = (n + 1) & 1;
                const int b = t * 72;
                // E0
                if (n) mbar_wait(&empty[0], par);
                mbar_arrive_expect_tx(&full[0], uint32_t(G::SZ0) * sizeof(T));
                tma_load_4d(E0, &mapU, 0, y0, z0, b, &full[0], pol);
                tma_load_4d(E0 + G::ROW1, &mapUy, 0, yup, z0, b, &full[0], pol);
                tma_load_4d(E0 + G::ROW2, &mapUz, 0, y0, zup, b, &full[0], pol);
                // E1
                if (n) mbar_wait(&empty[1], par);
                mbar_arrive_expect_tx(&full[1], uint32_t(G::SZ1) * sizeof(T));
                tma_load_4d(E1, &mapU, 0, y0, z0, b + 18, &full[1], pol);
                tma_load_4d(E1 + G::ROW1, &mapUz, 0, y0, zup, b + 18, &full[1], pol);
                // E2
                if (n) mbar_wait(&empty[2], par);
                mbar_arrive_expect_tx(&full[2], uint32_t(G::SZ2) * sizeof(T));
                tma_load_4d(E2, &mapU, 0, y0, z0, b + 36, &full[2], pol);
                tma_load_4d(E2 + G::ROW1, &mapUy, 0, yup, z0, b + 36, &full[2], pol);
                // E3
                if (n) mbar_wait(&empty[3], par);
                mbar_arrive_expect_tx(&full[3], uint32_t(G::SZ3) * sizeof(T));
                tma_load_4d(E3, &mapU, 0, y0, z0, b + 54, &full[3], pol);
                tma_load_4d(E3 + G::ROW1, &mapUy, 0, yup, z0, b + 54, &full[3], pol);
                tma_load_4d(E3 + G::ROW2, &mapUz, 0, y0, zup, b + 54, &full[3], pol);
            }
        }
        return;
    }

    // ------------------------------------------------------------------ compute warps
    const int lane = tid & 31;
    const int lx = tid % NX, ly = (tid / NX) & 1, lz = tid / (2 * NX);
    const int ix_up = (lx + 1 == NX) ? tid - lx : tid + 1;
    // +y / +z neighbour: (offset, stride) into a slot -- in the block, or a halo row slot
    const int jy = lx + NX * lz, jz = lx + NX * ly;
    const int y_off = ly == 0 ? tid + NX : G::ROW1 + jy, y_str = ly == 0 ? N : H;
    const int z_off0 = lz == 0 ? tid + 2 * NX : G::ROW2 + jz;  // E0, E3: +z row is the second halo row
    const int z_off1 = lz == 0 ? tid + 2 * NX : G::ROW1 + jz;  // E1: +z row is the first halo row
    const int z_str = lz == 0 ? N : H;

    auto release = [&](int k) { warp_release(&empty[k], lane); };

    uint32_t n = 0;
    for (int64_t item = blockIdx.x; item < p.nitems; item += GR) {
        int64_t blk;
        int t0, t1;
        link_item(p, item, blk, t0, t1);
        const int y = static_cast<int>(blk % p.nby) * 2 + ly;
        const int z = static_cast<int>(blk / p.nby) * 2 + lz;
        const int64_t s3 = lx + int64_t(NX) * (y + int64_t(p.ny) * z);
        for (int t = t0; t < t1; ++t, ++n) {
            const uint32_t par = n & 1;
            const int tn = (t + 1 == p.nt) ? 0 : t + 1;
            const T* up = U + int64_t(tn) * 72 * F + s3;  // this column one slice up
            T acc[18], tm[18], cn[18], cn2[18];
            auto smem_c = [](const T* base, int str) {
                return [=](int k, int j, int q) { return base[((3 * k + j) * 2 + q) * str]; };
            };
            auto reg_c = [](const T* r) { return [=](int k, int j, int q) { return r[(3 * k + j) * 2 + q]; }; };
            // T = A B with A = U_mu(x) re-read from its slot (no A is held across planes)
            auto nn = [&](const T* aslot, const T* bs, int bstr) {
                T a[18];
                ld_link_smem(aslot + tid, N, a);
                nn_smem_b<T, FUSED>(a, bs, bstr, tm);
            };
            if constexpr (FUSED) {
                // FMA chains: any plane order is within tolerance.  Order (0,1) (0,3) (0,2) (1,3) (1,2)
                // (2,3) keeps a single own-column C in flight, one plane ahead of its use
                (void)cn2;
                ld_soa<T, 18>(up, F, 0, cn);  // U_0(x+t)
                mbar_wait(&full[0], par);
                mbar_wait(&full[1], par);
                nn(E0, E1 + ix_up, N);  // (0,1)
                na_acc<T, FUSED, true>(tm, smem_c(E0 + y_off, y_str), s, acc);
                mbar_wait(&full[3], par);
                nn(E0, E3 + ix_up, N);  // (0,3)
                na_acc<T, FUSED, false>(tm, reg_c(cn), s, acc);
                ld_soa<T, 18>(up + 18 * F, F, 0, cn);  // U_1(x+t)
                mbar_wait(&full[2], par);
                nn(E0, E2 + ix_up, N);  // (0,2)
                na_acc<T, FUSED, false>(tm, smem_c(E0 + z_off0, z_str), s, acc);
                release(0);
                nn(E1, E3 + y_off, y_str);  // (1,3)
                na_acc<T, FUSED, false>(tm, reg_c(cn), s, acc);
                ld_soa<T, 18>(up + 36 * F, F, 0, cn);  // U_2(x+t)
                nn(E1, E2 + y_off, y_str);  // (1,2)
                na_acc<T, FUSED, false>(tm, smem_c(E1 + z_off1, z_str), s, acc);
                release(1);
                nn(E2, E3 + z_off0, z_str);  // (2,3)
                release(2);
                release(3);
                na_acc<T, FUSED, false>(tm, reg_c(cn), s, acc);
            } else {
                ld_soa<T, 18>(up, F, 0, cn);  // C of plane (0,3): U_0(x+t), three planes ahead
                // ---- (0,1): A = U_0(x), B = U_1(x+0), C = U_0(x+1)
                mbar_wait(&full[0], par);
                mbar_wait(&full[1], par);
                nn(E0, E1 + ix_up, N);
                na_acc<T, FUSED, true>(tm, smem_c(E0 + y_off, y_str), s, acc);
                ld_soa<T, 18>(up + 18 * F, F, 0, cn2);  // C of plane (1,3): U_1(x+t), three planes ahead
                // ---- (0,2): B = U_2(x+0), C = U_0(x+2)
                mbar_wait(&full[2], par);
                nn(E0, E2 + ix_up, N);
                na_acc<T, FUSED, false>(tm, smem_c(E0 + z_off0, z_str), s, acc);
                // ---- (0,3): B = U_3(x+0), C = U_0(x+t) (registers)
                mbar_wait(&full[3], par);
                nn(E0, E3 + ix_up, N);
                release(0);
                na_acc<T, FUSED, false>(tm, reg_c(cn), s, acc);
                ld_soa<T, 18>(up + 36 * F, F, 0, cn);  // C of plane (2,3): U_2(x+t), two planes ahead
                // ---- (1,2): A = U_1(x), B = U_2(x+1), C = U_1(x+2)
                nn(E1, E2 + y_off, y_str);
                na_acc<T, FUSED, false>(tm, smem_c(E1 + z_off1, z_str), s, acc);
                // ---- (1,3): B = U_3(x+1), C = U_1(x+t)
                nn(E1, E3 + y_off, y_str);
                release(1);
                na_acc<T, FUSED, false>(tm, reg_c(cn2), s, acc);
                // ---- (2,3): A = U_2(x), B = U_3(x+2), C = U_2(x+t)
                nn(E2, E3 + z_off0, z_str);
                release(2);
                release(3);
                na_acc<T, FUSED, false>(tm, reg_c(cn), s, acc);
            }
            T* o = acc_out + int64_t(t) * 18 * F + s3;
#pragma unroll
            for (int k = 0; k < 18; ++k) __stcs(o + k * F, acc[k]);
        }
    }
}

template <typename T, bool FUSED, int NX, int MINB>
static int run_link_ring(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, cudaStream_t st) {
    using G = LinkGeo<NX>;
    CUtensorMap mU, mUy, mUz;
    if (!make_map<T>(&mU, U, nx, ny, nz, int64_t(nt) * 72, 2, 2, 18) ||
        !make_map<T>(&mUy, U, nx, ny, nz, int64_t(nt) * 72, 1, 2, 18) ||
        !make_map<T>(&mUz, U, nx, ny, nz, int64_t(nt) * 72, 2, 1, 18))
        return 1;
    const size_t smem = size_t(G::TOTAL) * sizeof(T) + 8 * sizeof(uint64_t);
    const DeviceInfo& di = device_info();
    if (smem > size_t(di.max_smem_optin)) return 1;
    auto kern = k_link_ring<T, FUSED, NX, MINB>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    LinkRingParams p{};
    p.ny = ny; p.nz = nz; p.nt = nt;
    p.F = int64_t(nx) * ny * nz;
    p.nby = ny / 2;
    p.nblocks = int64_t(ny / 2) * (nz / 2);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::N + 32, smem);
    const int Gfull = di.num_sms * std::max(per_sm, 1);
    p.chunk = pick_chunk(p.nblocks, nt, Gfull);
    p.nitems = p.nblocks * ((nt + p.chunk - 1) / p.chunk);
    const int grid = static_cast<int>(std::min<int64_t>(Gfull, p.nitems));
    kern<<<grid, G::N + 32, smem, st>>>(mU, mUy, mUz, U, acc, p, s);
    note_kernel(std::string("k_link_ring<") + (sizeof(T) == 4 ? "f32," : "f64,") + std::to_string(NX) + "x2x2" +
                (per_sm > 1 ? "," + std::to_string(per_sm) + " CTAs/SM" : "") + ",chunk " + std::to_string(p.chunk) + ">");
    return check_launch("link_product(ring)");
}

// 1 = not applicable to this lattice (caller falls back)
template <typename T, bool FUSED>
int launch_link_ring(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, cudaStream_t st) {
    if (ny % 2 || nz % 2 || !aligned16(U)) return 1;
    constexpr int MB = sizeof(T) == 4 ? 2 : 1;
    if (nx == 48) return run_link_ring<T, FUSED, 48, MB>(U, acc, nx, ny, nz, nt, s, st);
    if (nx == 64 && sizeof(T) == 4) return run_link_ring<T, FUSED, 64, 1>(U, acc, nx, ny, nz, nt, s, st);
    if (nx == 32) return run_link_ring<T, FUSED, 32, MB>(U, acc, nx, ny, nz, nt, s, st);
    return 1;
}

template int launch_link_ring<float, false>(const float*, float*, int, int, int, int, float, cudaStream_t);
template int launch_link_ring<float, true>(const float*, float*, int, int, int, int, float, cudaStream_t);
template int launch_link_ring<double, false>(const double*, double*, int, int, int, int, double, cudaStream_t);
template int launch_link_ring<double, true>(const double*, double*, int, int, int, int, double, cudaStream_t);

}  // namespace su3g
