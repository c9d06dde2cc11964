// Link-product sweep from TMA-staged site tiles (link_variant 7; BASELINE configs[3]).
//
// The one-thread-per-site kernels (k_link_rows, k_link_product) gather every
// link a site needs through L1/L2: ~324 reals per site against 90 compulsory,
// so at 48^4 f64 they are bound by L2->SM traffic and its latency (ncu: 16
// warps/SM, one eligible warp per scheduler).  Here a CTA owns a tile of
// TX x TY x TZ sites of one t-slice and stages, with one TMA box each, its own
// 72-plane link block and the link planes the products reach outside it:
//
//   +x face (x0+TX, 2 columns)  U_y, U_z, U_t   (B of planes (0,1), (0,2), (0,3))
//   +y face (y0+TY)             U_x             (C of (0,1))   and U_z, U_t (B of (1,2), (1,3))
//   +z face (z0+TZ)             U_x, U_y        (C of (0,2), (1,2))   and U_t (B of (2,3))
//   +t face (t+1, whole tile)   U_x, U_y, U_z   (C of (0,3), (1,3), (2,3))
//
// Three threads per site -- thread (row r, site s) builds row r of
// T = U_mu(x) U_nu(x+mu) and of P = T U_mu(x+nu)^dag for the six planes and
// accumulates row r of acc = sum s P in plane order -- all operands from shared
// memory.  Row r of each product uses exactly the per-element arithmetic of
// mult_su3_nn / mult_su3_na, so EXACT mode is bit-identical to the composed
// reference; FMA mode uses FMA chains (north-star tolerance).
// Tiles are visited x-fastest so neighbouring tiles' faces are L2 hits.
#include <cuda.h>

#include <algorithm>
#include <mutex>
#include <string>

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

// 4-D view (x, y, z, plane) of the t-sliced SoA link field with a box of bx x by x bz x bp
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

template <typename T, bool FUSED, int MODE, class PF, class QF>
__device__ __forceinline__ void dot3(PF p, QF q, T& re, T& im) {
    if constexpr (FUSED) cdot_fma<T, MODE, 3>(p, q, re, im);
    else cdot<T, MODE, 3>(p, q, re, im);
}

}  // namespace

struct TileMaps {
    CUtensorMap own, xf, yf0, yf1, zf0, zf1, tf;
};

// Tile geometry and shared-memory layout (reals):
//   own [72][N]            the tile's links, plane-major (N = TX*TY*TZ)
//   xf  [54][XW*TY*TZ]     planes 18..71 (U_y, U_z, U_t) at x0+TX (XW = 16 B of columns; column 0 used)
//   yf  [18][TX*TZ] + [36][TX*TZ]   planes 0..17 (U_x) and 36..71 (U_z, U_t) at y0+TY
//   zf  [36][TX*TY] + [18][TX*TY]   planes 0..35 (U_x, U_y) and 54..71 (U_t) at z0+TZ
//   tf  [54][N]            planes 0..53 (U_x, U_y, U_z) of slice t+1
template <typename T, int TX, int TY, int TZ>
struct TileGeo {
    static constexpr int N = TX * TY * TZ;
    static constexpr int XW = 16 / int(sizeof(T));  // +x face columns: TMA rows are >= 16 bytes
    static constexpr int XF = XW * TY * TZ, YF = TX * TZ, ZF = TX * TY;
    static constexpr int OWN = 0;
    static constexpr int XO = OWN + 72 * N;
    static constexpr int YO = XO + 54 * XF;
    static constexpr int ZO = YO + 54 * YF;
    static constexpr int TO = ZO + 54 * ZF;
    static constexpr int REALS = TO + 54 * N;
};

template <typename T, bool FUSED, int TX, int TY, int TZ>
__global__ void __launch_bounds__(3 * TX * TY * TZ)
    k_link_tile(const __grid_constant__ TileMaps maps, T* __restrict__ acc_out, Geom g, T s, int ntx, int nty, int ntz) {
    using G = TileGeo<T, TX, TY, TZ>;
    constexpr int N = G::N;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + G::REALS);

    // tile of this CTA, x-tiles fastest
    int64_t b = blockIdx.x;
    const int tx = static_cast<int>(b % ntx);
    b /= ntx;
    const int ty = static_cast<int>(b % nty);
    b /= nty;
    const int tz = static_cast<int>(b % ntz);
    const int t = static_cast<int>(b / ntz);
    const int x0 = tx * TX, y0 = ty * TY, z0 = tz * TZ;

    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        constexpr uint32_t bytes = uint32_t(G::REALS) * sizeof(T);
        mbar_arrive_expect_tx(bar, bytes);
        const int xn = (x0 + TX) % g.nx, yn = (y0 + TY) % g.ny, zn = (z0 + TZ) % g.nz, tn = (t + 1) % g.nt;
        tma_load_4d(sm + G::OWN, &maps.own, x0, y0, z0, t * 72, bar);
        tma_load_4d(sm + G::XO, &maps.xf, xn, y0, z0, t * 72 + 18, bar);
        tma_load_4d(sm + G::YO, &maps.yf0, x0, yn, z0, t * 72, bar);
        tma_load_4d(sm + G::YO + 18 * G::YF, &maps.yf1, x0, yn, z0, t * 72 + 36, bar);
        tma_load_4d(sm + G::ZO, &maps.zf0, x0, y0, zn, t * 72, bar);
        tma_load_4d(sm + G::ZO + 36 * G::ZF, &maps.zf1, x0, y0, zn, t * 72 + 54, bar);
        tma_load_4d(sm + G::TO, &maps.tf, x0, y0, z0, tn * 72, bar);
    }

    const int r = threadIdx.x / N;  // matrix row of this thread
    const int site = threadIdx.x - r * N;
    const int lx = site % TX, ly = (site / TX) % TY, lz = site / (TX * TY);
    mbar_wait(bar, 0);

    // link mu (18 reals) of the neighbour one step along dir, as (base, stride): element e at base[e*stride]
    auto nbr = [&](int dir, int mu, const T*& base, int& stride) {
        if (dir == 0) {
            if (lx + 1 < TX) { base = sm + G::OWN + mu * 18 * N + site + 1; stride = N; }
            else { base = sm + G::XO + (mu - 1) * 18 * G::XF + G::XW * (ly + TY * lz); stride = G::XF; }
        } else if (dir == 1) {
            if (ly + 1 < TY) { base = sm + G::OWN + mu * 18 * N + site + TX; stride = N; }
            else {
                const int col = lx + TX * lz;
                if (mu == 0) base = sm + G::YO + col;
                else base = sm + G::YO + 18 * G::YF + (mu - 2) * 18 * G::YF + col;
                stride = G::YF;
            }
        } else if (dir == 2) {
            if (lz + 1 < TZ) { base = sm + G::OWN + mu * 18 * N + site + TX * TY; stride = N; }
            else {
                const int col = lx + TX * ly;
                if (mu <= 1) base = sm + G::ZO + mu * 18 * G::ZF + col;
                else base = sm + G::ZO + 36 * G::ZF + col;  // mu == 3
                stride = G::ZF;
            }
        } else {
            base = sm + G::TO + mu * 18 * N + site;  // mu in 0..2
            stride = N;
        }
    };

    T acc[6];
    constexpr int PMU[6] = {0, 0, 0, 1, 1, 2};
    constexpr int PNU[6] = {1, 2, 3, 2, 3, 3};
#pragma unroll
    for (int pl = 0; pl < 6; ++pl) {
        const int mu = PMU[pl], nu = PNU[pl];
        const T* A = sm + G::OWN + mu * 18 * N + site;  // U_mu(x), element e at A[e*N]
        const T* B;
        int bs;
        nbr(mu, nu, B, bs);  // U_nu(x + mu)
        const T* C;
        int cs;
        nbr(nu, mu, C, cs);  // U_mu(x + nu)
        T trow[6];
#pragma unroll
        for (int k = 0; k < 3; ++k)  // t[r][k] = sum_j a[r][j] b[j][k]   (mult_su3_nn)
            dot3<T, FUSED, PLAIN>([&](int j, int q) { return A[((3 * r + j) * 2 + q) * N]; },
                                  [&](int j, int q) { return B[((3 * j + k) * 2 + q) * bs]; }, trow[2 * k],
                                  trow[2 * k + 1]);
#pragma unroll
        for (int k = 0; k < 3; ++k) {  // p[r][k] = sum_j t[r][j] conj(c[k][j])   (mult_su3_na)
            T pr, pi;
            dot3<T, FUSED, CONJ_Q>([&](int j, int q) { return trow[2 * j + q]; },
                                   [&](int j, int q) { return C[((3 * k + j) * 2 + q) * cs]; }, pr, pi);
            if (pl == 0) {  // acc = 0 + s*p (scalar_mult_add_su3_matrix into the zero accumulator)
                acc[2 * k] = FUSED ? fma(s, pr, T(0)) : xadd(T(0), xmul(s, pr));
                acc[2 * k + 1] = FUSED ? fma(s, pi, T(0)) : xadd(T(0), xmul(s, pi));
            } else {
                acc[2 * k] = FUSED ? fma(s, pr, acc[2 * k]) : xadd(acc[2 * k], xmul(s, pr));
                acc[2 * k + 1] = FUSED ? fma(s, pi, acc[2 * k + 1]) : xadd(acc[2 * k + 1], xmul(s, pi));
            }
        }
    }
    const int64_t s3 = (x0 + lx) + int64_t(g.nx) * ((y0 + ly) + int64_t(g.ny) * (z0 + lz));
#pragma unroll
    for (int e = 0; e < 6; ++e) __stcs(acc_out + (int64_t(t) * 18 + 6 * r + e) * g.F + s3, acc[e]);
}

template <typename T, bool FUSED, int TX, int TY, int TZ>
static int run_link_tile(const T* U, T* acc, const Geom& g, T s, cudaStream_t st) {
    using G = TileGeo<T, TX, TY, TZ>;
    TileMaps m;
    const int nx = g.nx, ny = g.ny, nz = g.nz, nt = g.nt;
    if (!make_map<T>(&m.own, U, nx, ny, nz, nt, TX, TY, TZ, 72) ||
        !make_map<T>(&m.xf, U, nx, ny, nz, nt, G::XW, TY, TZ, 54) ||
        !make_map<T>(&m.yf0, U, nx, ny, nz, nt, TX, 1, TZ, 18) ||
        !make_map<T>(&m.yf1, U, nx, ny, nz, nt, TX, 1, TZ, 36) ||
        !make_map<T>(&m.zf0, U, nx, ny, nz, nt, TX, TY, 1, 36) ||
        !make_map<T>(&m.zf1, U, nx, ny, nz, nt, TX, TY, 1, 18) ||
        !make_map<T>(&m.tf, U, nx, ny, nz, nt, TX, TY, TZ, 54))
        return 1;
    const size_t smem = size_t(G::REALS) * sizeof(T) + 16;
    if (smem > size_t(device_info().max_smem_optin)) return 1;
    cudaFuncSetAttribute(k_link_tile<T, FUSED, TX, TY, TZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    const int ntx = nx / TX, nty = ny / TY, ntz = nz / TZ;
    const int64_t tiles = int64_t(ntx) * nty * ntz * nt;
    k_link_tile<T, FUSED, TX, TY, TZ><<<static_cast<unsigned>(tiles), 3 * G::N, smem, st>>>(m, acc, g, s, ntx, nty, ntz);
    note_kernel(std::string("k_link_tile<") + (sizeof(T) == 4 ? "f32," : "f64,") + std::to_string(TX) + "x" +
                std::to_string(TY) + "x" + std::to_string(TZ) + ">");
    return check_launch("link_product(tile)");
}

// returns 1 when the lattice does not tile (the caller falls back to the rows kernel)
template <typename T, bool FUSED>
int launch_link_tile(const T* U, T* acc, const Geom& g, T s, cudaStream_t st) {
    constexpr int TX = 8, TY = 4, TZ = 2;
    if (g.nx % TX || g.ny % TY || g.nz % TZ || !aligned16(U)) return 1;
    if ((g.nx * int(sizeof(T))) % 16) return 1;
    return run_link_tile<T, FUSED, TX, TY, TZ>(U, acc, g, s, st);
}

template int launch_link_tile<float, false>(const float*, float*, const Geom&, float, cudaStream_t);
template int launch_link_tile<float, true>(const float*, float*, const Geom&, float, cudaStream_t);
template int launch_link_tile<double, false>(const double*, double*, const Geom&, double, cudaStream_t);
template int launch_link_tile<double, true>(const double*, double*, const Geom&, double, cudaStream_t);

}  // namespace su3g
