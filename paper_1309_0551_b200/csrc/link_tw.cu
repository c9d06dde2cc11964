// Link-product sweep on a TMA-staged t-walk (link_variant 8; BASELINE configs[3]).
//
// The one-thread-per-site kernels (k_link_rows, k_link_product) gather the
// 12 neighbour links of every site through L1/L2: ~324 reals per site against
// 90 compulsory, which caps them by L2->SM bandwidth (f32 48^4: 0.31 of HBM).
// Here a persistent CTA owns a block of one t-slice -- the full x extent (x is
// periodic inside the CTA) times BY x BZ rows, one thread per site -- and walks
// t, so every link is moved HBM -> smem once as the block's own link, and the
// neighbours a product reaches are shared-memory reads:
//
//   own ring  [3][72][N]   U_0..U_3 of the block at t, t+1 (= the +t face) and
//                          t+2 (in flight); one 4-D TMA box per z-layer
//   +y face   [2][54][S]   U_0, U_2, U_3 of row y0+BY   (C of (0,1); B of (1,2), (1,3))
//   +z face   [1][54][S]   U_0, U_1, U_3 of plane z0+BZ (C of (0,2), (1,2); B of (2,3))
//
// The six planes (mu,nu) = 01 02 03 12 13 23 need, besides own(t):
//   01: y face   02: z face   03: own(t+1)   12: y, z   13: y, own(t+1)   23: z, own(t+1)
// The z face is single-buffered (the three slots do not fit 227 KB otherwise):
// each step computes the planes without it first -- P01 into the accumulator,
// P03 and P13 held in registers -- and only then waits for it; it is refilled
// right after the end-of-step barrier, so its load overlaps half a step.  The
// accumulator still adds s*P in the reference's plane order 01,02,03,12,13,23,
// with mult_su3_nn / mult_su3_na / scalar_mult_add_su3_matrix's per-element
// arithmetic (su3bench scalar.py:77-104,197-205): EXACT mode is bit-identical
// to the composed reference, FMA mode is within the north-star tolerance.
//
// Work items are (block, t-chunk), chunk-major; CTA c takes items c, c+G, ...,
// so the CTAs in flight hold neighbouring blocks of the same t-range and the
// faces one CTA stages are L2 hits on what its neighbours stream as own links.
// Thread 0 streams the loads of the CTA's whole item sequence as one flat ring
// (own loads: t0..t1 per item), so the next item's slices load during the
// current item's last steps.
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "sweep_common.cuh"

namespace su3g {

int g_link_tw_chunk = 0;  // su3g_set_option("link_tw_chunk"): t-chunk length of the work items (0 = auto)

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

// 4-D view (x, y, z, plane = t*72 + c) of the t-sliced SoA link field, box bx x by x bz x bp
template <typename T>
bool make_map(CUtensorMap* m, const T* U, int nx, int ny, int nz, int nt, int bx, int by, int bz, int bp) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) return false;
    const cuuint64_t dims[4] = {cuuint64_t(nx), cuuint64_t(ny), cuuint64_t(nz), cuuint64_t(nt) * 72};
    const cuuint64_t strides[3] = {cuuint64_t(nx) * sizeof(T), cuuint64_t(nx) * ny * sizeof(T),
                                   cuuint64_t(nx) * ny * nz * sizeof(T)};
    const cuuint32_t box[4] = {cuuint32_t(bx), cuuint32_t(by), cuuint32_t(bz), cuuint32_t(bp)};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUtensorMapDataType dt = sizeof(T) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
    return enc(m, dt, 4, const_cast<T*>(U), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(bar))
        : "memory");
}

struct TwMaps {
    CUtensorMap own, yf0, yf1, zf0, zf1;
};

struct TwParams {
    int nx, ny, nz, nt;
    int64_t F;
    int nby;
    int64_t nblocks;
    int chunk;
    int64_t nitems;
};

// P = A B C^dag, row by row of T = A B (mult_su3_nn then mult_su3_na, su3bench scalar.py:77-104);
// link element e of A, B, C at X[e * S] in shared memory
template <typename T, bool FUSED, int S>
__device__ __forceinline__ void plane_product(const T* A, const T* B, const T* C, T* P) {
    T tm[18];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            auto pa = [&](int j, int q) { return A[((3 * i + j) * 2 + q) * S]; };
            auto pb = [&](int j, int q) { return B[((3 * j + k) * 2 + q) * S]; };
            if constexpr (FUSED) cdot_fma<T, PLAIN, 3>(pa, pb, tm[(3 * i + k) * 2], tm[(3 * i + k) * 2 + 1]);
            else cdot<T, PLAIN, 3>(pa, pb, tm[(3 * i + k) * 2], tm[(3 * i + k) * 2 + 1]);
        }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            auto pt = [&](int j, int q) { return tm[(3 * i + j) * 2 + q]; };
            auto pc = [&](int j, int q) { return C[((3 * k + j) * 2 + q) * S]; };
            if constexpr (FUSED) cdot_fma<T, CONJ_Q, 3>(pt, pc, P[(3 * i + k) * 2], P[(3 * i + k) * 2 + 1]);
            else cdot<T, CONJ_Q, 3>(pt, pc, P[(3 * i + k) * 2], P[(3 * i + k) * 2 + 1]);
        }
}

// acc = acc + s*P (scalar_mult_add_su3_matrix, scalar.py:197-205); FIRST: the accumulator is 0
template <typename T, bool FUSED, bool FIRST>
__device__ __forceinline__ void acc_add(T* acc, const T* P, T s) {
#pragma unroll
    for (int e = 0; e < 18; ++e) {
        const T a = FIRST ? T(0) : acc[e];
        acc[e] = FUSED ? fma(s, P[e], a) : xadd(a, xmul(s, P[e]));
    }
}

}  // namespace

// Shared-memory layout (reals): own [3][BZ][72][S], +y face [2][54][S], +z face [54][S], then 6 mbarriers.
// An own slice is BZ TMA boxes of one z-layer each (NX x BY x 1 x 72), so every link element in shared
// memory -- own, +y face (NX x 1 x BZ), +z face (NX x BY x 1) -- sits at a stride of S = NX*BY = NX*BZ
// reals: the products address all operands as base + compile-time offset.
template <typename T, int NX, int BY, int BZ>
struct TwGeo {
    static_assert(BY == BZ, "uniform operand stride needs square y/z faces");
    static constexpr int N = NX * BY * BZ, S = NX * BY;
    static constexpr int LAYER = 72 * S, OWN = BZ * LAYER, FS = 54 * S;
    static constexpr int Y0 = 3 * OWN, Z0 = Y0 + 2 * FS, REALS = Z0 + FS;
    static constexpr size_t BYTES = size_t(REALS) * sizeof(T) + 6 * sizeof(uint64_t);
    static_assert((LAYER * sizeof(T)) % 128 == 0 && (FS * sizeof(T)) % 128 == 0 && (18 * S * sizeof(T)) % 128 == 0,
                  "TMA destinations must stay 128-byte aligned");
};

template <typename T, bool FUSED, int NX, int BY, int BZ>
__global__ void __launch_bounds__(NX* BY* BZ, 1)
    k_link_tw(const __grid_constant__ TwMaps maps, T* __restrict__ acc_out, TwParams p, T s) {
    using G = TwGeo<T, NX, BY, BZ>;
    constexpr int S = G::S;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    uint64_t* bar_own = reinterpret_cast<uint64_t*>(sm + G::REALS);
    uint64_t* bar_yf = bar_own + 3;
    uint64_t* bar_zf = bar_own + 5;

    const int tid = threadIdx.x;
    const int lx = tid % NX, ly = (tid / NX) % BY, lz = tid / (NX * BY);
    const int64_t Gs = gridDim.x;
    if (tid == 0) {
        for (int i = 0; i < 6; ++i) mbar_init(bar_own + i, 1);
        fence_mbar_init();
    }
    __syncthreads();

    auto item_t0 = [&](int64_t item) { return static_cast<int>(item / p.nblocks) * p.chunk; };
    auto item_t1 = [&](int64_t item) { return min(item_t0(item) + p.chunk, p.nt); };
    auto item_y0 = [&](int64_t item) { return static_cast<int>((item % p.nblocks) % p.nby) * BY; };
    auto item_z0 = [&](int64_t item) { return static_cast<int>((item % p.nblocks) / p.nby) * BZ; };

    // producer state (thread 0): flat sequences of own loads (t0..t1 per item) and +y face loads (t0..t1-1)
    int64_t o_item = blockIdx.x, f_item = blockIdx.x;
    int o_t = o_item < p.nitems ? item_t0(o_item) : 0, f_t = o_t;
    int o_issued = 0, f_issued = 0;
    auto issue_own = [&]() {
        uint64_t* b = bar_own + (o_issued % 3);
        mbar_arrive_expect_tx(b, uint32_t(G::OWN * sizeof(T)));
        const int tt = o_t % p.nt, y0 = item_y0(o_item), z0 = item_z0(o_item);
#pragma unroll
        for (int l = 0; l < BZ; ++l)
            tma_load_4d(sm + (o_issued % 3) * G::OWN + l * G::LAYER, &maps.own, 0, y0, z0 + l, tt * 72, b);
        ++o_issued;
        if (++o_t > item_t1(o_item)) {
            o_item += Gs;
            if (o_item < p.nitems) o_t = item_t0(o_item);
        }
    };
    auto issue_yf = [&]() {
        uint64_t* b = bar_yf + (f_issued % 2);
        T* dst = sm + G::Y0 + (f_issued % 2) * G::FS;
        mbar_arrive_expect_tx(b, uint32_t(G::FS * sizeof(T)));
        const int yn = (item_y0(f_item) + BY) % p.ny, z0 = item_z0(f_item);
        tma_load_4d(dst, &maps.yf0, 0, yn, z0, f_t * 72, b);                // U_0
        tma_load_4d(dst + 18 * S, &maps.yf1, 0, yn, z0, f_t * 72 + 36, b);  // U_2, U_3
        ++f_issued;
        if (++f_t >= item_t1(f_item)) {
            f_item += Gs;
            if (f_item < p.nitems) f_t = item_t0(f_item);
        }
    };
    auto issue_zf = [&](int64_t item, int t) {
        T* dst = sm + G::Z0;
        mbar_arrive_expect_tx(bar_zf, uint32_t(G::FS * sizeof(T)));
        const int zn = (item_z0(item) + BZ) % p.nz, y0 = item_y0(item);
        tma_load_4d(dst, &maps.zf0, 0, y0, zn, t * 72, bar_zf);                 // U_0, U_1
        tma_load_4d(dst + 36 * S, &maps.zf1, 0, y0, zn, t * 72 + 54, bar_zf);  // U_3
    };
    if (tid == 0 && int64_t(blockIdx.x) < p.nitems) {
        while (o_issued < 3 && o_item < p.nitems) issue_own();
        while (f_issued < 2 && f_item < p.nitems) issue_yf();
        issue_zf(blockIdx.x, item_t0(blockIdx.x));
    }

    // operand bases relative to a slot (element e of link mu at base + (mu*18 + e)*S)
    const int c_xy = lx + NX * ly;                                       // column within a z-layer
    const int o_self = lz * G::LAYER + c_xy;                             // own site
    const int o_xp = o_self + ((lx + 1 < NX) ? 1 : 1 - NX);              // +x, periodic inside the block
    const bool y_in = ly + 1 < BY, z_in = lz + 1 < BZ;
    const int o_yp = y_in ? o_self + NX : G::Y0 + lx + NX * lz;          // own, or +y face column
    const int o_zp = z_in ? o_self + G::LAYER : G::Z0 + c_xy;            // own, or +z face column

    int k = 0, a = 0;  // step counter, own-load index of the current slice
    for (int64_t item = blockIdx.x; item < p.nitems; item += Gs, ++a) {
        const int t0 = item_t0(item), t1 = item_t1(item), y0 = item_y0(item), z0 = item_z0(item);
        const int64_t s3 = lx + int64_t(p.nx) * ((y0 + ly) + int64_t(p.ny) * (z0 + lz));
        for (int t = t0; t < t1; ++t, ++k, ++a) {
            const T* own = sm + (a % 3) * G::OWN;
            const T* nxt = sm + ((a + 1) % 3) * G::OWN;
            const int yslot = (k % 2) * G::FS;  // the +y face slot of this step
            mbar_wait(bar_own + (a % 3), (a / 3) & 1);
            mbar_wait(bar_own + ((a + 1) % 3), ((a + 1) / 3) & 1);
            mbar_wait(bar_yf + (k % 2), (k / 2) & 1);

            // link mu of the neighbour one step along dir (0..3 = +x, +y, +z, +t; -1 = the site itself)
            auto link = [&](int dir, int mu) -> const T* {
                if (dir == -1) return own + o_self + mu * 18 * S;
                if (dir == 0) return own + o_xp + mu * 18 * S;
                if (dir == 3) return nxt + o_self + mu * 18 * S;
                if (dir == 1)  // mu in {0, 2, 3}; face planes U_0 | U_2, U_3
                    return y_in ? own + o_yp + mu * 18 * S : sm + yslot + o_yp + (mu == 0 ? 0 : mu - 1) * 18 * S;
                // mu in {0, 1, 3}; face planes U_0, U_1 | U_3
                return z_in ? own + o_zp + mu * 18 * S : sm + o_zp + (mu == 3 ? 2 : mu) * 18 * S;
            };

            // Compute order 01, 03, 13 | wait for the +z face | 02, 12, 23.  The plane loop stays
            // rolled: six inlined products overflow the 32 KB instruction cache (ncu: "no
            // instruction" was the top stall of the unrolled form).
            T acc[18], H1[18], H2[18];
#pragma unroll 1
            for (int q = 0; q < 6; ++q) {
                const int mu = (0x210100 >> (4 * q)) & 15, nu = (0x322331 >> (4 * q)) & 15;
                if (q == 3) mbar_wait(bar_zf, k & 1);
                T P[18];
                plane_product<T, FUSED, S>(link(-1, mu), link(mu, nu), link(nu, mu), P);  // U_mu(x) U_nu(x+mu) U_mu(x+nu)^dag
                if (q == 0) {
                    acc_add<T, FUSED, true>(acc, P, s);  // acc = 0 + s*P01
                } else if (q == 1) {
#pragma unroll
                    for (int e = 0; e < 18; ++e) H1[e] = P[e];  // P03
                } else if (q == 2) {
#pragma unroll
                    for (int e = 0; e < 18; ++e) H2[e] = P[e];  // P13
                } else {
                    acc_add<T, FUSED, false>(acc, P, s);                // P02, P12, P23
                    if (q == 3) acc_add<T, FUSED, false>(acc, H1, s);  // then P03
                    if (q == 4) acc_add<T, FUSED, false>(acc, H2, s);  // then P13
                }
            }
#pragma unroll
            for (int e = 0; e < 18; ++e) __stcs(acc_out + (int64_t(t) * 18 + e) * p.F + s3, acc[e]);

            __syncthreads();  // every thread is done with own(t), the +y face of step k and the +z face
            if (tid == 0) {
                const int freed = a + 1 + (t + 1 == t1 ? 1 : 0);  // own loads [0, freed) are consumed
                while (o_issued < freed + 3 && o_item < p.nitems) issue_own();
                while (f_issued < k + 3 && f_item < p.nitems) issue_yf();
                if (t + 1 < t1) issue_zf(item, t + 1);
                else if (item + Gs < p.nitems) issue_zf(item + Gs, item_t0(item + Gs));
            }
        }
    }
}

template <typename T, bool FUSED, int NX, int BY, int BZ>
static int run_link_tw(const T* U, T* acc, const Geom& g, T s, cudaStream_t st) {
    using Gm = TwGeo<T, NX, BY, BZ>;
    TwMaps m;
    const int nx = g.nx, ny = g.ny, nz = g.nz, nt = g.nt;
    if (!make_map<T>(&m.own, U, nx, ny, nz, nt, NX, BY, 1, 72) || !make_map<T>(&m.yf0, U, nx, ny, nz, nt, NX, 1, BZ, 18) ||
        !make_map<T>(&m.yf1, U, nx, ny, nz, nt, NX, 1, BZ, 36) || !make_map<T>(&m.zf0, U, nx, ny, nz, nt, NX, BY, 1, 36) ||
        !make_map<T>(&m.zf1, U, nx, ny, nz, nt, NX, BY, 1, 18))
        return 1;
    const DeviceInfo& di = device_info();
    if (Gm::BYTES > size_t(di.max_smem_optin)) return 1;
    auto kern = k_link_tw<T, FUSED, NX, BY, BZ>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Gm::BYTES));
    TwParams p;
    p.nx = nx;
    p.ny = ny;
    p.nz = nz;
    p.nt = nt;
    p.F = g.F;
    p.nby = ny / BY;
    p.nblocks = int64_t(ny / BY) * (nz / BZ);
    const int G = di.num_sms;
    // item length: the extra own load per item is an L2 hit for short chunks (a t-slice of links is far
    // smaller than L2), so the single wave is balanced first and the chunk kept as long as that allows
    p.chunk = g_link_tw_chunk > 0 ? std::min(g_link_tw_chunk, nt) : pick_chunk(p.nblocks, nt, G);
    p.nitems = p.nblocks * ((nt + p.chunk - 1) / p.chunk);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(G, p.nitems));
    kern<<<grid, Gm::N, Gm::BYTES, st>>>(m, acc, p, s);
    note_kernel(std::string("k_link_tw<") + (sizeof(T) == 4 ? "f32," : "f64,") + std::to_string(NX) + "x" +
                std::to_string(BY) + "x" + std::to_string(BZ) + ",chunk " + std::to_string(p.chunk) + ">");
    return check_launch("link_product(t-walk)");
}

// returns 1 when the lattice does not fit a t-walk geometry (the caller falls back to the rows kernel)
template <typename T, bool FUSED>
int launch_link_tw(const T* U, T* acc, const Geom& g, T s, cudaStream_t st) {
    if constexpr (sizeof(T) == 4) {  // f64: three own slices of any useful block overflow smem
        if (!aligned16(U)) return 1;
        if (g.nx == 48 && g.ny % 2 == 0 && g.nz % 2 == 0) return run_link_tw<T, FUSED, 48, 2, 2>(U, acc, g, s, st);
    }
    return 1;
}

template int launch_link_tw<float, false>(const float*, float*, const Geom&, float, cudaStream_t);
template int launch_link_tw<float, true>(const float*, float*, const Geom&, float, cudaStream_t);
template int launch_link_tw<double, false>(const double*, double*, const Geom&, double, cudaStream_t);
template int launch_link_tw<double, true>(const double*, double*, const Geom&, double, cudaStream_t);


// ---------------------------------------------------------------------------------------------
// 8x4x4-site blocks with U_3 through L2 (link_variant 10; the f64 form of the t-walk).
//
// An f64 slice of all four links is 576 B per site, so three ring slots of a 128-site block
// would take 221 KB before any face.  U_3 is only ever a B operand -- U_3(x+mu) of the planes
// (mu,3) -- so the ring keeps U_0..U_2 (54 planes, 3 x 55 KB) and double-buffered x/y/z faces
// (2 x 27 KB); U_3(x+mu) is gathered from global memory into registers, two planes ahead,
// after every thread has L2-prefetched its own U_3 one step earlier (so the gathers of the
// neighbours are L2 hits).  128 threads = 4 warps, one per SMSP: balanced.  All smem operands
// sit at a stride of S = 32 reals (own z-layers 8x4, faces 36 planes x 32 columns).
// ---------------------------------------------------------------------------------------------
struct Tw4Maps {
    CUtensorMap own, xf, yf, zf;
};

struct Tw4Params {
    int nx, ny, nz, nt;
    int64_t F;
    int nbx, nby;
    int64_t nblocks;
    int chunk;
    int64_t nitems;
};

template <typename T>
struct Tw4Geo {
    static constexpr int BX = 8, BY = 4, BZ = 4, N = 128, S = 32;
    static constexpr int XW = 16 / int(sizeof(T));  // +x face columns (TMA rows are >= 16 B)
    static constexpr int XB = XW / 2;               // +x face boxes, each 36 planes x 32 columns
    static constexpr int LAYER = 54 * S, OWN = BZ * LAYER;
    static constexpr int FP = 36 * S;  // one face box: 36 planes x 32 columns
    static constexpr int XO = 0, YO = XB * FP, ZO = YO + FP, FSLOT = ZO + FP;
    static constexpr int F0 = 3 * OWN, REALS = F0 + 2 * FSLOT;
    static constexpr size_t BYTES = size_t(REALS) * sizeof(T) + 5 * sizeof(uint64_t);
    static_assert((LAYER * sizeof(T)) % 128 == 0 && (FP * sizeof(T)) % 128 == 0 && (18 * S * sizeof(T)) % 128 == 0,
                  "TMA destinations must stay 128-byte aligned");
};

namespace {
__device__ __forceinline__ void prefetch_l2_line(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
}  // namespace

template <typename T, bool FUSED>
__global__ void __launch_bounds__(128, 1)
    k_link_tw4(const __grid_constant__ Tw4Maps maps, const T* __restrict__ U, T* __restrict__ acc_out, Tw4Params p,
               T s) {
    using G = Tw4Geo<T>;
    constexpr int S = G::S, BX = G::BX, BY = G::BY, BZ = G::BZ;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    uint64_t* bar_own = reinterpret_cast<uint64_t*>(sm + G::REALS);
    uint64_t* bar_f = bar_own + 3;

    const int tid = threadIdx.x;
    const int lx = tid % BX, ly = (tid / BX) % BY, lz = tid / (BX * BY);
    const int64_t Gs = gridDim.x;
    if (tid == 0) {
        for (int i = 0; i < 5; ++i) mbar_init(bar_own + i, 1);
        fence_mbar_init();
    }
    __syncthreads();

    auto item_t0 = [&](int64_t item) { return static_cast<int>(item / p.nblocks) * p.chunk; };
    auto item_t1 = [&](int64_t item) { return min(item_t0(item) + p.chunk, p.nt); };
    auto item_x0 = [&](int64_t item) { return static_cast<int>((item % p.nblocks) % p.nbx) * BX; };
    auto item_y0 = [&](int64_t item) { return static_cast<int>(((item % p.nblocks) / p.nbx) % p.nby) * BY; };
    auto item_z0 = [&](int64_t item) { return static_cast<int>((item % p.nblocks) / (int64_t(p.nbx) * p.nby)) * BZ; };

    // producer (thread 0): flat sequences of ring loads (t0..t1 per item) and face loads (t0..t1-1)
    int64_t o_item = blockIdx.x, f_item = blockIdx.x;
    int o_t = o_item < p.nitems ? item_t0(o_item) : 0, f_t = o_t;
    int o_issued = 0, f_issued = 0;
    auto issue_own = [&]() {
        uint64_t* b = bar_own + (o_issued % 3);
        mbar_arrive_expect_tx(b, uint32_t(G::OWN * sizeof(T)));
        const int tt = o_t % p.nt, x0 = item_x0(o_item), y0 = item_y0(o_item), z0 = item_z0(o_item);
#pragma unroll
        for (int l = 0; l < BZ; ++l)
            tma_load_4d(sm + (o_issued % 3) * G::OWN + l * G::LAYER, &maps.own, x0, y0, z0 + l, tt * 72, b);
        ++o_issued;
        if (++o_t > item_t1(o_item)) {
            o_item += Gs;
            if (o_item < p.nitems) o_t = item_t0(o_item);
        }
    };
    auto issue_faces = [&]() {
        uint64_t* b = bar_f + (f_issued % 2);
        T* dst = sm + G::F0 + (f_issued % 2) * G::FSLOT;
        mbar_arrive_expect_tx(b, uint32_t(G::FSLOT * sizeof(T)));
        const int x0 = item_x0(f_item), y0 = item_y0(f_item), z0 = item_z0(f_item), tp = f_t * 72;
        const int xn = (x0 + BX) % p.nx, yn = (y0 + BY) % p.ny, zn = (z0 + BZ) % p.nz;
#pragma unroll
        for (int bx = 0; bx < G::XB; ++bx)  // U_1, U_2 of column x0+BX
            tma_load_4d(dst + G::XO + bx * G::FP, &maps.xf, xn, y0, z0 + bx * (BZ / G::XB), tp + 18, b);
        tma_load_4d(dst + G::YO, &maps.yf, x0, yn, z0, tp, b);                // U_0 of row y0+BY
        tma_load_4d(dst + G::YO + 18 * S, &maps.yf, x0, yn, z0, tp + 36, b);  // U_2
        tma_load_4d(dst + G::ZO, &maps.zf, x0, y0, zn, tp, b);                // U_0, U_1 of plane z0+BZ
        ++f_issued;
        if (++f_t >= item_t1(f_item)) {
            f_item += Gs;
            if (f_item < p.nitems) f_t = item_t0(f_item);
        }
    };
    if (tid == 0 && int64_t(blockIdx.x) < p.nitems) {
        while (o_issued < 3 && o_item < p.nitems) issue_own();
        while (f_issued < 2 && f_item < p.nitems) issue_faces();
    }

    // smem offsets: element (link mu, e) at base + (mu*18 + e)*S
    const int c_xy = lx + BX * ly;
    const int o_self = lz * G::LAYER + c_xy;
    const bool x_in = lx + 1 < BX, y_in = ly + 1 < BY, z_in = lz + 1 < BZ;
    const int fx = G::XO + (lz / (BZ / G::XB)) * G::FP + G::XW * (ly + BY * (lz % (BZ / G::XB)));  // +x face column
    const int fy = G::YO + lx + BX * lz;
    const int fz = G::ZO + c_xy;

    const int64_t F = p.F;
    int k = 0, a = 0;
    for (int64_t item = blockIdx.x; item < p.nitems; item += Gs, ++a) {
        const int t0 = item_t0(item), t1 = item_t1(item);
        const int gx0 = item_x0(item) + lx, gy0 = item_y0(item) + ly, gz0 = item_z0(item) + lz;
        const int64_t s3 = gx0 + int64_t(p.nx) * (gy0 + int64_t(p.ny) * gz0);
        // neighbour slice-local indices (periodic): their U_3 is gathered through L2
        const int64_t s3x = (gx0 + 1 == p.nx ? 0 : gx0 + 1) + int64_t(p.nx) * (gy0 + int64_t(p.ny) * gz0);
        const int64_t s3y = gx0 + int64_t(p.nx) * ((gy0 + 1 == p.ny ? 0 : gy0 + 1) + int64_t(p.ny) * gz0);
        const int64_t s3z = gx0 + int64_t(p.nx) * (gy0 + int64_t(p.ny) * (gz0 + 1 == p.nz ? 0 : gz0 + 1));
        for (int t = t0; t < t1; ++t, ++k, ++a) {
            const T* u3 = U + (int64_t(t) * 72 + 54) * F;
            {  // own U_3 of the next slice into L2, for the neighbours' gathers one step later
                const T* nx3 = U + (int64_t(t + 1 == p.nt ? 0 : t + 1) * 72 + 54) * F + s3;
#pragma unroll
                for (int e = 0; e < 18; ++e) prefetch_l2_line(nx3 + e * F);
            }
            T ga[18], gb[18];
#pragma unroll
            for (int e = 0; e < 18; ++e) ga[e] = __ldg(u3 + e * F + s3x);  // U_3(x + x^) for plane (0,3)

            const T* own = sm + (a % 3) * G::OWN;
            const T* nxt = sm + ((a + 1) % 3) * G::OWN;
            const T* fs = sm + G::F0 + (k % 2) * G::FSLOT;
            mbar_wait(bar_own + (a % 3), (a / 3) & 1);
            mbar_wait(bar_own + ((a + 1) % 3), ((a + 1) / 3) & 1);
            mbar_wait(bar_f + (k % 2), (k / 2) & 1);

            // link mu of the neighbour one step along dir (0..2 spatial, 3 = +t; -1 = the site itself)
            auto link = [&](int dir, int mu) -> const T* {
                const int off = mu * 18 * S;
                if (dir == -1) return own + o_self + off;
                if (dir == 3) return nxt + o_self + off;
                if (dir == 0) return x_in ? own + o_self + 1 + off : fs + fx + (mu - 1) * 18 * S;   // mu in {1, 2}
                if (dir == 1) return y_in ? own + o_self + BX + off : fs + fy + (mu == 0 ? 0 : 18 * S);  // {0, 2}
                return z_in ? own + o_self + G::LAYER + off : fs + fz + off;                     // {0, 1}
            };

            T acc[18];
#pragma unroll 1
            for (int q = 0; q < 6; ++q) {
                const int mu = (0x211000 >> (4 * q)) & 15, nu = (0x332321 >> (4 * q)) & 15;
                const T* A = link(-1, mu);
                const T* C = link(nu, mu);
                T tm[18];
                if (nu == 3) {  // B = U_3(x + mu) from the gathers (plane 03: ga; 13: gb; 23: ga)
                    T bq[18];
#pragma unroll
                    for (int e = 0; e < 18; ++e) bq[e] = (q == 4) ? gb[e] : ga[e];
#pragma unroll
                    for (int i = 0; i < 3; ++i)
#pragma unroll
                        for (int kk = 0; kk < 3; ++kk) {
                            auto pa = [&](int j, int c) { return A[((3 * i + j) * 2 + c) * S]; };
                            auto pb = [&](int j, int c) { return bq[(3 * j + kk) * 2 + c]; };
                            if constexpr (FUSED) cdot_fma<T, PLAIN, 3>(pa, pb, tm[(3 * i + kk) * 2], tm[(3 * i + kk) * 2 + 1]);
                            else cdot<T, PLAIN, 3>(pa, pb, tm[(3 * i + kk) * 2], tm[(3 * i + kk) * 2 + 1]);
                        }
                } else {
                    const T* B = link(mu, nu);
#pragma unroll
                    for (int i = 0; i < 3; ++i)
#pragma unroll
                        for (int kk = 0; kk < 3; ++kk) {
                            auto pa = [&](int j, int c) { return A[((3 * i + j) * 2 + c) * S]; };
                            auto pb = [&](int j, int c) { return B[((3 * j + kk) * 2 + c) * S]; };
                            if constexpr (FUSED) cdot_fma<T, PLAIN, 3>(pa, pb, tm[(3 * i + kk) * 2], tm[(3 * i + kk) * 2 + 1]);
                            else cdot<T, PLAIN, 3>(pa, pb, tm[(3 * i + kk) * 2], tm[(3 * i + kk) * 2 + 1]);
                        }
                }
                if (q == 2) {  // ga is free: the gathers of planes (2,3) and (1,3)
#pragma unroll
                    for (int e = 0; e < 18; ++e) ga[e] = __ldg(u3 + e * F + s3z);
#pragma unroll
                    for (int e = 0; e < 18; ++e) gb[e] = __ldg(u3 + e * F + s3y);
                }
                // P = T C^dag (mult_su3_na), accumulated element by element: acc = acc + s*P
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int kk = 0; kk < 3; ++kk) {
                        T pr, pi;
                        auto pt = [&](int j, int c) { return tm[(3 * i + j) * 2 + c]; };
                        auto pc = [&](int j, int c) { return C[((3 * kk + j) * 2 + c) * S]; };
                        if constexpr (FUSED) cdot_fma<T, CONJ_Q, 3>(pt, pc, pr, pi);
                        else cdot<T, CONJ_Q, 3>(pt, pc, pr, pi);
                        const int e = (3 * i + kk) * 2;
                        const T a0 = (q == 0) ? T(0) : acc[e], a1 = (q == 0) ? T(0) : acc[e + 1];
                        acc[e] = FUSED ? fma(s, pr, a0) : xadd(a0, xmul(s, pr));
                        acc[e + 1] = FUSED ? fma(s, pi, a1) : xadd(a1, xmul(s, pi));
                    }
            }
#pragma unroll
            for (int e = 0; e < 18; ++e) __stcs(acc_out + (int64_t(t) * 18 + e) * F + s3, acc[e]);

            __syncthreads();  // every thread is done with ring slot a and face slot k
            if (tid == 0) {
                const int freed = a + 1 + (t + 1 == t1 ? 1 : 0);
                while (o_issued < freed + 3 && o_item < p.nitems) issue_own();
                while (f_issued < k + 3 && f_item < p.nitems) issue_faces();
            }
        }
    }
}

template <typename T, bool FUSED>
int launch_link_tw4(const T* U, T* acc, const Geom& g, T s, cudaStream_t st) {
    using Gm = Tw4Geo<T>;
    const int nx = g.nx, ny = g.ny, nz = g.nz, nt = g.nt;
    if (nx % Gm::BX || ny % Gm::BY || nz % Gm::BZ || !aligned16(U) || (int64_t(nx) * sizeof(T)) % 16) return 1;
    Tw4Maps m;
    if (!make_map<T>(&m.own, U, nx, ny, nz, nt, Gm::BX, Gm::BY, 1, 54) ||
        !make_map<T>(&m.xf, U, nx, ny, nz, nt, Gm::XW, Gm::BY, Gm::BZ / Gm::XB, 36) ||
        !make_map<T>(&m.yf, U, nx, ny, nz, nt, Gm::BX, 1, Gm::BZ, 18) ||
        !make_map<T>(&m.zf, U, nx, ny, nz, nt, Gm::BX, Gm::BY, 1, 36))
        return 1;
    const DeviceInfo& di = device_info();
    if (Gm::BYTES > size_t(di.max_smem_optin)) return 1;
    cudaFuncSetAttribute(k_link_tw4<T, FUSED>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(Gm::BYTES));
    Tw4Params p;
    p.nx = nx;
    p.ny = ny;
    p.nz = nz;
    p.nt = nt;
    p.F = g.F;
    p.nbx = nx / Gm::BX;
    p.nby = ny / Gm::BY;
    p.nblocks = int64_t(p.nbx) * p.nby * (nz / Gm::BZ);
    const int G = di.num_sms;
    p.chunk = g_link_tw_chunk > 0 ? std::min(g_link_tw_chunk, nt) : pick_chunk(p.nblocks, nt, G);
    p.nitems = p.nblocks * ((nt + p.chunk - 1) / p.chunk);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(G, p.nitems));
    k_link_tw4<T, FUSED><<<grid, Gm::N, Gm::BYTES, st>>>(m, U, acc, p, s);
    note_kernel(std::string("k_link_tw4<") + (sizeof(T) == 4 ? "f32" : "f64") + ",8x4x4,chunk " +
                std::to_string(p.chunk) + ">");
    return check_launch("link_product(t-walk, 8x4x4)");
}

template int launch_link_tw4<float, false>(const float*, float*, const Geom&, float, cudaStream_t);
template int launch_link_tw4<float, true>(const float*, float*, const Geom&, float, cudaStream_t);
template int launch_link_tw4<double, false>(const double*, double*, const Geom&, double, cudaStream_t);
template int launch_link_tw4<double, true>(const double*, double*, const Geom&, double, cudaStream_t);

}  // namespace su3g
