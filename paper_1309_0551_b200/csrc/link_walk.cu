// Link-product sweep (BASELINE configs[3]): row-split TMA t-walk with the t-planes carried one step.
//
// acc(x) = sum over the planes (0,1) (0,2) (0,3) (1,2) (1,3) (2,3) of s * U_mu(x) U_nu(x+mu) U_mu(x+nu)^dag,
// accumulated in that order.
//
// Why this shape.  Per site the sweep reads 15 link matrices for 4 compulsory ones, so the links
// must come from shared memory, and at f64 a site's links are 576 B: only ~150 sites of one slice
// fit an SM next to their halos.  One thread per site then holds A, T, C and the accumulator
// (255 registers, 7 warps/SM, the r02 ring walk since removed) and cannot cover the FP64 and shared-memory latencies.
// Here:
//   * three lanes per site, lane r owns row r of every product: row r of T = A B needs row r of A,
//     row r of P = T C^dag needs row r of T, so the rows are independent and each lane performs
//     exactly the per-element operations of the one-thread form (bit-identical in exact mode);
//     the three lanes of a site are adjacent, so every B / C element read from shared memory is
//     one address per site (a broadcast);
//   * the t-planes (0,3) (1,3) (2,3) need C = U_mu(x+t), a link of the NEXT slice.  Instead of
//     gathering it from global memory, each lane carries T_03, T_13, T_23 (and the partial
//     accumulator and P_12, for the exact plane order) to the next step of the walk, where
//     U_mu(x+t) is its own column of the resident block: the t-walk then reads every link of a
//     slice from shared memory, and nothing but the accumulator leaves the SM.
//
// A CTA owns a block of one t-slice -- the full x extent (x periodic inside the block) x BY y-rows
// x 1 z-plane, N = NX*BY sites -- and walks t over a work item (block, t-chunk).  A producer warp
// streams into typed slots (4-D TMA boxes, full/empty mbarriers):
//   E0, E1, E2   U_0, U_1, U_2 of the block [18][N], double-buffered (the next slice's arrive
//                while this one is in use: they are the first thing a step needs)
//   E3           U_3 of the block
//   Y            U_0, U_2, U_3 on the +y halo row [3][18][NX]
//   Z (2 slots)  U_0, U_1, U_3 on the +z halo plane [18][N] each, one plane per chunk
// and a step t of the walk does
//   finish (x, t-1):  P03 = T03 C0^dag, P13 = T13 C1^dag, P23 = T23 C2^dag with C = own column of
//                     E0..E2, accumulated as acc2 + sP03 + sP12 + sP13 + sP23 -> store
//   start  (x, t):    P01, P02 -> acc2;  T03;  P12 (held);  T13;  T23
// A work item of L slices takes L+1 steps: the last one loads E0..E2 of slice t1 and only finishes.
#include <algorithm>
#include <string>

#include "nn_site.cuh"
#include "tma.cuh"

namespace su3g {

int g_link_chunk = 0;  // su3g_set_option("link_chunk"): t-chunk length of the link walks' work items (0 auto: the columns schedule)

namespace {

struct WalkParams {
    int ny, nz, nt;
    int64_t F;
    int nby;  // ny / BY
    int64_t nblocks;
    int chunk;
    int64_t nitems;
    int64_t n_full;  // the first n_full items are whole t-columns of blocks 0..n_full-1; the other
                     // blocks are cut into t-chunks of `chunk` slices, chunk-major (n_full = 0: all of them)
};

template <int NX, int BY>
struct WalkGeo {
    static constexpr int N = NX * BY;
    static constexpr int NWC = (3 * N + 31) / 32;  // compute warps
    static constexpr int THREADS = 32 * NWC + 32;
    static constexpr int BLK = 18 * N;             // a block / Z chunk slot
    static constexpr int YSZ = 54 * NX;            // the +y chunk
    // slot offsets (reals): E0..E2 x 2 buffers, E3, Y, Z0, Z1
    static constexpr int OFF_E = 0;                // E[k][b] at OFF_E + (2k + b) * BLK
    static constexpr int OFF_E3 = 6 * BLK;
    static constexpr int OFF_Y = 7 * BLK;
    static constexpr int OFF_Z = 7 * BLK + YSZ;    // Z[j] at OFF_Z + j * BLK
    static constexpr int TOTAL = 9 * BLK + YSZ;
    // barriers: full/empty for E[k][b] (6), E3, Y, Z0, Z1
    static constexpr int NBAR = 10;
};

__device__ __forceinline__ void walk_item(const WalkParams& p, int64_t item, int64_t& blk, int& t0, int& t1) {
    schedule_item(p.n_full, p.nblocks, p.chunk, 0, p.nt, item, blk, t0, t1);
}

// row r of T = A B: a = row r of A (6 reals), B element (j, k) at bs[((3j+k)*2+q) * bstr]
template <typename T, bool FUSED>
__device__ __forceinline__ void row_nn(const T* a, const T* bs, int bstr, T* tr) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if constexpr (FUSED)
            cdot_fma<T, PLAIN, 3>([&](int j, int q) { return a[2 * j + q]; },
                                  [&](int j, int q) { return bs[((3 * j + k) * 2 + q) * bstr]; }, tr[2 * k],
                                  tr[2 * k + 1]);
        else
            cdot<T, PLAIN, 3>([&](int j, int q) { return a[2 * j + q]; },
                              [&](int j, int q) { return bs[((3 * j + k) * 2 + q) * bstr]; }, tr[2 * k],
                              tr[2 * k + 1]);
    }
}

// row r of P = T C^dag (mult_su3_na arithmetic): C element (k, j) at cs[((3k+j)*2+q) * cstr]
template <typename T, bool FUSED>
__device__ __forceinline__ void row_na(const T* tr, const T* cs, int cstr, T* pr) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        if constexpr (FUSED)
            cdot_fma<T, CONJ_Q, 3>([&](int j, int q) { return tr[2 * j + q]; },
                                   [&](int j, int q) { return cs[((3 * k + j) * 2 + q) * cstr]; }, pr[2 * k],
                                   pr[2 * k + 1]);
        else
            cdot<T, CONJ_Q, 3>([&](int j, int q) { return tr[2 * j + q]; },
                               [&](int j, int q) { return cs[((3 * k + j) * 2 + q) * cstr]; }, pr[2 * k],
                               pr[2 * k + 1]);
    }
}

// acc (+)= s * P (scalar_mult_add_su3_matrix arithmetic); FIRST: acc = 0 + s*P
template <typename T, bool FUSED, bool FIRST>
__device__ __forceinline__ void row_acc(const T* pr, T s, T* acc) {
#pragma unroll
    for (int e = 0; e < 6; ++e) {
        const T base = FIRST ? T(0) : acc[e];
        acc[e] = FUSED ? fma(s, pr[e], base) : xadd(base, xmul(s, pr[e]));
    }
}

}  // namespace

template <typename T, bool FUSED, int NX, int BY>
__global__ void __launch_bounds__(WalkGeo<NX, BY>::THREADS, 1)
    k_link_walk(const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapY,
                T* __restrict__ acc_out, WalkParams p, T s) {
    using G = WalkGeo<NX, BY>;
    constexpr int N = G::N, NWC = G::NWC;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + G::TOTAL);
    uint64_t* empty = full + G::NBAR;
    // barrier indices
    constexpr int B_E3 = 6, B_Y = 7, B_Z = 8;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int k = 0; k < G::NBAR; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], NWC);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int GR = gridDim.x;

    // ------------------------------------------------------------------ producer warp
    if (tid >= 32 * NWC) {
        if (tid != 32 * NWC) return;
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
        // use counters (same sequence as the consumers): steps (E0..E2 buffers), E3, Y, Z chunks
        uint32_t ns = 0, n3 = 0, ny_ = 0, nz_ = 0;
        auto load_slot = [&](int bar, uint32_t use, T* dst, const CUtensorMap* map, int y, int z, int plane,
                             uint32_t bytes) {
            if (use) mbar_wait(&empty[bar], (use - 1) & 1);
            mbar_arrive_expect_tx(&full[bar], bytes);
            tma_load_4d(dst, map, 0, y, z, plane, &full[bar], pol);
        };
        for (int64_t item = blockIdx.x; item < p.nitems; item += GR) {
            int64_t blk;
            int t0, t1;
            walk_item(p, item, blk, t0, t1);
            const int y0 = static_cast<int>(blk % p.nby) * BY, z0 = static_cast<int>(blk / p.nby);
            const int yup = (y0 + BY) % p.ny, zup = (z0 + 1) % p.nz;
            for (int t = t0; t <= t1; ++t, ++ns) {
                const int ts = (t == p.nt) ? 0 : t;  // the drain step of the last chunk wraps to slice 0
                const int b = ns & 1;
                const uint32_t use = ns >> 1;  // uses of buffer b so far
                for (int k = 0; k < 3; ++k)
                    load_slot(2 * k + b, use, sm + G::OFF_E + (2 * k + b) * G::BLK, &mapB, y0, z0, ts * 72 + 18 * k,
                              G::BLK * sizeof(T));
                if (t == t1) continue;  // drain step: E0..E2 only
                // +y row: U_0, U_2, U_3 in one slot (three boxes, one barrier)
                if (ny_) mbar_wait(&empty[B_Y], (ny_ - 1) & 1);
                mbar_arrive_expect_tx(&full[B_Y], G::YSZ * sizeof(T));
                T* yd = sm + G::OFF_Y;
                tma_load_4d(yd, &mapY, 0, yup, z0, ts * 72, &full[B_Y], pol);
                tma_load_4d(yd + 18 * NX, &mapY, 0, yup, z0, ts * 72 + 36, &full[B_Y], pol);
                tma_load_4d(yd + 36 * NX, &mapY, 0, yup, z0, ts * 72 + 54, &full[B_Y], pol);
                ++ny_;
                // +z plane of U_0 (first Z chunk), then U_3 of the block, then U_1 / U_3 on +z
                load_slot(B_Z + (nz_ & 1), nz_ >> 1, sm + G::OFF_Z + (nz_ & 1) * G::BLK, &mapB, y0, zup, ts * 72,
                          G::BLK * sizeof(T));
                ++nz_;
                load_slot(B_E3, n3, sm + G::OFF_E3, &mapB, y0, z0, ts * 72 + 54, G::BLK * sizeof(T));
                ++n3;
                load_slot(B_Z + (nz_ & 1), nz_ >> 1, sm + G::OFF_Z + (nz_ & 1) * G::BLK, &mapB, y0, zup,
                          ts * 72 + 18, G::BLK * sizeof(T));
                ++nz_;
                load_slot(B_Z + (nz_ & 1), nz_ >> 1, sm + G::OFF_Z + (nz_ & 1) * G::BLK, &mapB, y0, zup,
                          ts * 72 + 54, G::BLK * sizeof(T));
                ++nz_;
            }
        }
        return;
    }

    // ------------------------------------------------------------------ compute warps
    const int lane = tid & 31;
    const bool active = tid < 3 * N;
    const int sl = active ? tid / 3 : 0;  // idle lanes of the last warp shadow site 0 and never store
    const int row = active ? tid - 3 * (tid / 3) : 0;
    const int lx = sl % NX, ly = sl / NX;
    const int ix_up = (lx + 1 == NX) ? sl - lx : sl + 1;
    const bool y_in = ly + 1 < BY;  // +y neighbour inside the block, else on the +y halo row
    const int ystr = y_in ? N : NX;
    const int a_off = 6 * row * N + sl;  // row `row` of the own link in a block slot: a_off + c*N

    auto release = [&](int bar) { warp_release(&empty[bar], lane); };
    auto wait_full = [&](int bar, uint32_t use) { mbar_wait(&full[bar], use & 1); };
    auto load_row = [&](const T* slot, T* a) {
#pragma unroll
        for (int c = 0; c < 6; ++c) a[c] = slot[a_off + c * N];
    };

    const T* const Ysl = sm + G::OFF_Y;
    uint32_t ns = 0, n3 = 0, ny_ = 0, nz_ = 0;
    for (int64_t item = blockIdx.x; item < p.nitems; item += GR) {
        int64_t blk;
        int t0, t1;
        walk_item(p, item, blk, t0, t1);
        const int y = static_cast<int>(blk % p.nby) * BY + ly;
        const int z = static_cast<int>(blk / p.nby);
        const int64_t s3 = lx + int64_t(NX) * (y + int64_t(p.ny) * z);
        // carried from step t-1 to step t: partial accumulator after (0,1) (0,2), P12, and the
        // t-planes' T = A B rows
        T acc[6], p12[6], t03[6], t13[6], t23[6];
        for (int t = t0; t <= t1; ++t, ++ns) {
            const int b = ns & 1;
            const uint32_t use = ns >> 1;
            const T* E0 = sm + G::OFF_E + (0 + b) * G::BLK;
            const T* E1 = sm + G::OFF_E + (2 + b) * G::BLK;
            const T* E2 = sm + G::OFF_E + (4 + b) * G::BLK;
            wait_full(0 + b, use);
            if (t > t0) {
                // ---- finish site (x, t-1): C = U_mu(x + t) = own column of E_mu of this slice
                T pr[6];
                row_na<T, FUSED>(t03, E0 + sl, N, pr);
                row_acc<T, FUSED, false>(pr, s, acc);  // + s P03
                row_acc<T, FUSED, false>(p12, s, acc); // + s P12
                wait_full(2 + b, use);
                row_na<T, FUSED>(t13, E1 + sl, N, pr);
                row_acc<T, FUSED, false>(pr, s, acc);  // + s P13
                wait_full(4 + b, use);
                row_na<T, FUSED>(t23, E2 + sl, N, pr);
                row_acc<T, FUSED, false>(pr, s, acc);  // + s P23
                if (active) {
                    T* o = acc_out + (int64_t(t - 1) * 18 + 6 * row) * p.F + s3;
#pragma unroll
                    for (int e = 0; e < 6; ++e) __stcs(o + e * p.F, acc[e]);
                }
            } else {
                wait_full(2 + b, use);
                wait_full(4 + b, use);
            }
            if (t == t1) {  // drain step
                release(0 + b);
                release(2 + b);
                release(4 + b);
                continue;
            }
            T a[6], tr[6], pr[6];
            // ---- (0,1): A = U_0(x), B = U_1(x+0), C = U_0(x+1)
            load_row(E0, a);
            row_nn<T, FUSED>(a, E1 + ix_up, N, tr);
            wait_full(B_Y, ny_);
            row_na<T, FUSED>(tr, y_in ? E0 + sl + NX : Ysl + lx, ystr, pr);
            row_acc<T, FUSED, true>(pr, s, acc);
            // ---- (0,2): B = U_2(x+0), C = U_0(x+2) (first Z chunk)
            row_nn<T, FUSED>(a, E2 + ix_up, N, tr);
            {
                const int zb = B_Z + (nz_ & 1);
                wait_full(zb, nz_ >> 1);
                row_na<T, FUSED>(tr, sm + G::OFF_Z + (nz_ & 1) * G::BLK + sl, N, pr);
                release(zb);
                ++nz_;
            }
            row_acc<T, FUSED, false>(pr, s, acc);
            // ---- T03 = U_0(x) U_3(x+0)
            wait_full(B_E3, n3);
            row_nn<T, FUSED>(a, sm + G::OFF_E3 + ix_up, N, t03);
            release(0 + b);
            // ---- (1,2): A = U_1(x), B = U_2(x+1), C = U_1(x+2) (second Z chunk); P12 is held
            load_row(E1, a);
            row_nn<T, FUSED>(a, y_in ? E2 + sl + NX : Ysl + 18 * NX + lx, ystr, tr);
            {
                const int zb = B_Z + (nz_ & 1);
                wait_full(zb, nz_ >> 1);
                row_na<T, FUSED>(tr, sm + G::OFF_Z + (nz_ & 1) * G::BLK + sl, N, p12);
                release(zb);
                ++nz_;
            }
            // ---- T13 = U_1(x) U_3(x+1)
            row_nn<T, FUSED>(a, y_in ? sm + G::OFF_E3 + sl + NX : Ysl + 36 * NX + lx, ystr, t13);
            release(2 + b);
            release(B_Y);
            ++ny_;
            // ---- T23 = U_2(x) U_3(x+2) (third Z chunk)
            load_row(E2, a);
            {
                const int zb = B_Z + (nz_ & 1);
                wait_full(zb, nz_ >> 1);
                row_nn<T, FUSED>(a, sm + G::OFF_Z + (nz_ & 1) * G::BLK + sl, N, t23);
                release(zb);
                ++nz_;
            }
            release(4 + b);
            release(B_E3);
            ++n3;
        }
    }
}

template <typename T, bool FUSED, int NX, int BY>
static int run_link_walk(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, cudaStream_t st) {
    using G = WalkGeo<NX, BY>;
    CUtensorMap mB, mY;
    if (!make_map<T>(&mB, U, nx, ny, nz, int64_t(nt) * 72, BY, 1, 18) ||
        !make_map<T>(&mY, U, nx, ny, nz, int64_t(nt) * 72, 1, 1, 18))
        return 1;
    const size_t smem = size_t(G::TOTAL) * sizeof(T) + 2 * G::NBAR * sizeof(uint64_t);
    const DeviceInfo& di = device_info();
    if (smem > size_t(di.max_smem_optin)) return 1;
    auto kern = k_link_walk<T, FUSED, NX, BY>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    WalkParams p{};
    p.ny = ny; p.nz = nz; p.nt = nt;
    p.F = int64_t(nx) * ny * nz;
    p.nby = ny / BY;
    p.nblocks = int64_t(ny / BY) * nz;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::THREADS, smem);
    const int Gfull = di.num_sms * std::max(per_sm, 1);
    // an item of L slices costs L + 1 steps (the drain step loads three blocks and finishes); the columns
    // schedule (sweep_common.cuh) unless a chunk length is forced
    const WalkSchedule ws = pick_schedule(p.nblocks, nt, Gfull, 0.6, g_link_chunk == 0);
    p.n_full = ws.n_full;
    p.chunk = ws.chunk;
    if (g_link_chunk > 0) p.chunk = std::min(g_link_chunk, nt);
    p.nitems = p.n_full + (p.nblocks - p.n_full) * ((nt + p.chunk - 1) / p.chunk);
    const int grid = static_cast<int>(std::min<int64_t>(Gfull, p.nitems));
    kern<<<grid, G::THREADS, smem, st>>>(mB, mY, acc, p, s);
    note_kernel(std::string("k_link_walk<") + (sizeof(T) == 4 ? "f32," : "f64,") + std::to_string(NX) + "x" +
                std::to_string(BY) + "x1" + (per_sm > 1 ? "," + std::to_string(per_sm) + " CTAs/SM" : "") +
                (p.n_full ? "," + std::to_string(p.n_full) + " columns" : "") + ",chunk " + std::to_string(p.chunk) + ">");
    return check_launch("link_product(walk)");
}

// ======================================================================================
// FMA mode: two lanes per site (k_link_fact below).  Lanes 0-15 and 16-31 of a warp take the same 16
// sites, each lane owns whole products, so every staged link is read once per use and a half-warp's
// 64-bit shared load is one slot, 128 B.  (The plane-by-plane form of this walk, k_link_pair --
// three planes per lane, twelve products per site, 0.611 of HBM at 48^4 f64 -- is in git history;
// the factored form replaced it.)
// ======================================================================================

template <typename T, int NX, int BY>
struct PairGeo {
    static constexpr int N = NX * BY;
    static_assert(N % 16 == 0, "a warp covers 16 sites x 2 lanes");
    static constexpr int NWC = N / 16;
    static constexpr int THREADS = 32 * NWC + 32;
    static constexpr int BLK = 18 * N;
    static constexpr int YSUB = 18 * NX;            // one link on the +y row
    static constexpr int OFF_E = 0;                 // E[k][b] (link k of the block, buffer b) at (2k + b) * BLK
    static constexpr int OFF_E3 = 6 * BLK;
    static constexpr int OFF_Z = 7 * BLK;           // Z0, Z1, Z3 (U_0, U_1, U_3 on the +z plane)
    static constexpr int OFF_Y = 10 * BLK;          // Y0, Y2, Y3 (U_0, U_2, U_3 on the +y row), YSUB each
    static constexpr int TOTAL = 10 * BLK + 3 * YSUB;
    // barriers: E[k][b] 0..5, E3 6, Z 7..9, Y 10..12
    static constexpr int NBAR = 13;
};

// ======================================================================================
// FMA mode, factored: two lanes per site, nine matrix products instead of twelve (k_link_fact).
//
// With FMA chains the association is free as well (the north-star tolerance, not bit equality):
//   acc(x) = s * sum_mu U_mu(x) M_mu(x),   M_mu(x) = sum_{nu > mu} U_nu(x+mu) U_mu(x+nu)^dag,
// three B C^dag products for mu = 0, two for mu = 1, one for mu = 2, then one A M product per mu:
// 9 x 108 FMAs + 18 multiplies = 990 per site instead of 1404, and 15 staged matrices read per site
// instead of 18.  Lanes 0-15 of a warp take mu = 0 (four products), lanes 16-31 mu = 1 and 2 (five);
// every step has the same product type in both halves, so the warp runs five product steps with one
// instruction stream (lanes 0-15 sit out the fifth):
//   S1  M = B C^dag : B U_3(x+0), C U_0(x+t)           | B U_3(x+1) [Y3], C U_1(x+t)        (M_1)
//   S2  M += B C^dag: B U_1(x+0), C U_0(x+1) [Y0]      | B U_3(x+2) [Z3], C U_2(x+t)        (M_2, from zero)
//   S3  M += B C^dag: B U_2(x+0), C U_0(x+2) [Z0]      | B U_2(x+1) [Y2], C U_1(x+2) [Z1]   (M_1 again)
//   S4  acc = A M   : A U_0(x), M_0                    | A U_1(x), M_1
//   S5  acc += A M  :                                  | A U_2(x), M_2
// The block walk runs DOWN in t: slice t+1's U_0..U_2 are
// then the previous step's own links, already resident, so the t-plane operands never wait, they are
// used first (S1 / S2) and their buffers take slice t-1 with more than a step in flight.  Every
// single-buffered slot is read in exactly one product step (both users of E3 share S1), so it is freed
// in the step that needs it and its refill has a whole step in flight.  Slots of one step share one
// full / empty barrier pair (U_0 + U_1 of a slice buffer, U_2 of a slice buffer, E3 + Y3, Y0 + Z3,
// Z0 + Y2 + Z1), and the producer issues a step's loads in the order the previous step frees them,
// which is the order the step needs them: E3 Y3, U_0 U_1 | Y0 Z3, U_2 | Z0 Y2 Z1.
// ======================================================================================

namespace {

// m (+)= B C^dag: m[i][k] += sum_j B[i][j] conj(C[k][j]); element (r, c) of B / C at ptr[((3r+c)*2+q) * str].
// The contraction index is the outer loop: each j loads one column of B and of C (12 reals) and
// feeds all 18 accumulators, so 18 independent FMA chains are in flight instead of 2.
template <typename T, bool FIRST>
__device__ __forceinline__ void bcdag_fma(const T* bs, int bstr, const T* cs, int cstr, T* m) {
#ifdef FACT_NOMATH
    for (int q = 0; q < 18; ++q) m[q] = (FIRST ? T(0) : m[q]) + bs[0] + cs[0];
    return;
#endif
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        T b[6], c[6];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            b[2 * r] = bs[((3 * r + j) * 2) * bstr];
            b[2 * r + 1] = bs[((3 * r + j) * 2 + 1) * bstr];
            c[2 * r] = cs[((3 * r + j) * 2) * cstr];
            c[2 * r + 1] = cs[((3 * r + j) * 2 + 1) * cstr];
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int e = (3 * i + k) * 2;
                if (FIRST && j == 0) {
                    m[e] = b[2 * i] * c[2 * k];
                    m[e + 1] = b[2 * i + 1] * c[2 * k];
                } else {
                    m[e] = fma(b[2 * i], c[2 * k], m[e]);
                    m[e + 1] = fma(b[2 * i + 1], c[2 * k], m[e + 1]);
                }
            }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int e = (3 * i + k) * 2;
                m[e] = fma(b[2 * i + 1], c[2 * k + 1], m[e]);
                m[e + 1] = fma(-b[2 * i], c[2 * k + 1], m[e + 1]);
            }
    }
}

// acc (+)= A M: acc[i][k] += sum_j A[i][j] M[j][k]; A element (i, j) at as[((3i+j)*2+q) * astr], M in registers;
// j outermost as above (one column of A per j)
template <typename T, bool FIRST>
__device__ __forceinline__ void am_fma(const T* as, int astr, const T* m, T* acc) {
#ifdef FACT_NOMATH
    for (int q = 0; q < 18; ++q) acc[q] = (FIRST ? T(0) : acc[q]) + as[0] * m[q];
    return;
#endif
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        T a[6];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            a[2 * r] = as[((3 * r + j) * 2) * astr];
            a[2 * r + 1] = as[((3 * r + j) * 2 + 1) * astr];
        }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int e = (3 * i + k) * 2, f = (3 * j + k) * 2;
                if (FIRST && j == 0) {
                    acc[e] = a[2 * i] * m[f];
                    acc[e + 1] = a[2 * i] * m[f + 1];
                } else {
                    acc[e] = fma(a[2 * i], m[f], acc[e]);
                    acc[e + 1] = fma(a[2 * i], m[f + 1], acc[e + 1]);
                }
            }
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int e = (3 * i + k) * 2, f = (3 * j + k) * 2;
                acc[e] = fma(-a[2 * i + 1], m[f + 1], acc[e]);
                acc[e + 1] = fma(a[2 * i + 1], m[f], acc[e + 1]);
            }
    }
}

}  // namespace

template <typename T, int NX, int BY>
__global__ void __launch_bounds__(PairGeo<T, NX, BY>::THREADS, sizeof(T) == 4 ? 2 : 1)  // f32: two CTAs per SM
    k_link_fact(const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapY,
                T* __restrict__ acc_out, WalkParams p, T s) {
    using G = PairGeo<T, NX, BY>;
    constexpr int N = G::N, NWC = G::NWC;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* sm = reinterpret_cast<T*>(smem_raw);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + G::TOTAL);
    uint64_t* empty = full + G::NBAR;
    // slots that are needed and freed in the same product step share a barrier: U_0 + U_1 of a slice
    // buffer (0, 1), U_2 of a slice buffer (2, 3), E3 + Y3 (4), Y0 + Z3 (5), Z0 + Y2 + Z1 (6)
    constexpr int B_E01 = 0, B_E2 = 2, B_A = 4, B_B = 5, B_C = 6, NB = 7;
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int k = 0; k < NB; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], NWC);
        }
        fence_mbar_init();
    }
    __syncthreads();
    const int GR = gridDim.x;
    T* const E3w = sm + G::OFF_E3;
    T* const Z0w = sm + G::OFF_Z;
    T* const Y0w = sm + G::OFF_Y;

    if (tid >= 32 * NWC) {  // ------------------------------------------ producer warp
        if (tid != 32 * NWC) return;
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
        uint32_t ne = 0, ns = 0;  // slices loaded (buffer ne & 1); steps issued (halo slot uses)
        auto begin = [&](int bar, uint32_t use, int reals) {
            if (use) mbar_wait(&empty[bar], (use - 1) & 1);
#ifdef FACT_NOLOAD  // floor build: the slots are never filled, the barriers complete at once (compute only)
            mbar_arrive(&full[bar]);
#else
            mbar_arrive_expect_tx(&full[bar], reals * sizeof(T));
#endif
        };
#ifdef FACT_NOLOAD
#define tma_load_4d(...) ((void)0)
#endif
        auto Ew = [&](int k, uint32_t slice_no) { return sm + G::OFF_E + (2 * k + (slice_no & 1)) * G::BLK; };
        for (int64_t item = blockIdx.x; item < p.nitems; item += GR) {
            int64_t blk;
            int t0, t1;
            walk_item(p, item, blk, t0, t1);
            const int y0 = static_cast<int>(blk % p.nby) * BY, z0 = static_cast<int>(blk / p.nby);
            const int yup = (y0 + BY) % p.ny, zup = (z0 + 1) % p.nz;
            {  // the slice above the item (U_0..U_2 only): the first step's U_mu(x+t)
                const int tu = (t1 == p.nt ? 0 : t1) * 72, b = ne & 1;
                begin(B_E01 + b, ne >> 1, 2 * G::BLK);
                tma_load_4d(Ew(0, ne), &mapB, 0, y0, z0, tu, &full[B_E01 + b], pol);
                tma_load_4d(Ew(1, ne), &mapB, 0, y0, z0, tu + 18, &full[B_E01 + b], pol);
                begin(B_E2 + b, ne >> 1, G::BLK);
                tma_load_4d(Ew(2, ne), &mapB, 0, y0, z0, tu + 36, &full[B_E2 + b], pol);
                ++ne;
            }
            for (int t = t1 - 1; t >= t0; --t, ++ns) {
                // issue order = the order the previous step frees the barriers' slots = the order this step
                // needs them: every load has a whole step in flight
                const int tp = t * 72, b = ne & 1;
                begin(B_A, ns, G::BLK + G::YSUB);
                tma_load_4d(E3w, &mapB, 0, y0, z0, tp + 54, &full[B_A], pol);
                tma_load_4d(Y0w + 2 * G::YSUB, &mapY, 0, yup, z0, tp + 54, &full[B_A], pol);
                begin(B_E01 + b, ne >> 1, 2 * G::BLK);
                tma_load_4d(Ew(0, ne), &mapB, 0, y0, z0, tp, &full[B_E01 + b], pol);
                tma_load_4d(Ew(1, ne), &mapB, 0, y0, z0, tp + 18, &full[B_E01 + b], pol);
                begin(B_B, ns, G::BLK + G::YSUB);
                tma_load_4d(Y0w, &mapY, 0, yup, z0, tp, &full[B_B], pol);
                tma_load_4d(Z0w + 2 * G::BLK, &mapB, 0, y0, zup, tp + 54, &full[B_B], pol);
                begin(B_E2 + b, ne >> 1, G::BLK);
                tma_load_4d(Ew(2, ne), &mapB, 0, y0, z0, tp + 36, &full[B_E2 + b], pol);
                begin(B_C, ns, 2 * G::BLK + G::YSUB);
                tma_load_4d(Z0w, &mapB, 0, y0, zup, tp, &full[B_C], pol);
                tma_load_4d(Y0w + G::YSUB, &mapY, 0, yup, z0, tp + 36, &full[B_C], pol);
                tma_load_4d(Z0w + G::BLK, &mapB, 0, y0, zup, tp + 18, &full[B_C], pol);
                ++ne;
            }
        }
        return;
#ifdef FACT_NOLOAD
#undef tma_load_4d
#endif
    }

    // ------------------------------------------------------------------ compute warps
    const int lane = tid & 31;
    const int sl = (tid >> 5) * 16 + (lane & 15);
    const int h = lane >> 4;
    const int lx = sl % NX, ly = sl / NX;
    const int ix_up = (lx + 1 == NX) ? sl - lx : sl + 1;
    const bool y_in = ly + 1 < BY;
    const int ystr = y_in ? N : NX;
    const T* const E3 = E3w;
    const T* const Z0 = Z0w;
    const T* const Z1 = Z0 + G::BLK;
    const T* const Z3 = Z1 + G::BLK;
    const T* const Y0 = Y0w;
    const T* const Y2 = Y0 + G::YSUB;
    const T* const Y3 = Y2 + G::YSUB;
    auto release = [&](int bar) { warp_release(&empty[bar], lane); };
    auto wait_full = [&](int bar, uint32_t use) { mbar_wait(&full[bar], use & 1); };
    auto E = [&](int k, uint32_t slice_no) { return sm + G::OFF_E + (2 * k + (slice_no & 1)) * G::BLK; };

    // a barrier is polled once, early (before the arithmetic of the operand in front of it), and
    // waited on only if that poll failed: the poll's latency hides behind the FMAs
    auto test_full = [&](int bar, uint32_t use) { return mbar_test(&full[bar], use & 1); };
    auto wait_if = [&](uint32_t done, int bar, uint32_t use) {
        if (!done) mbar_wait(&full[bar], use & 1);
    };
    uint32_t ne = 0, ns = 0;
    for (int64_t item = blockIdx.x; item < p.nitems; item += GR) {
        int64_t blk;
        int t0, t1;
        walk_item(p, item, blk, t0, t1);
        const int y = static_cast<int>(blk % p.nby) * BY + ly;
        const int z = static_cast<int>(blk / p.nby);
        const int64_t s3 = lx + int64_t(NX) * (y + int64_t(p.ny) * z);
        // the slice above the item: the only step whose U_mu(x+t) buffers were not waited on as own links
        wait_full(B_E01 + (ne & 1), ne >> 1);
        wait_full(B_E2 + (ne & 1), ne >> 1);
        uint32_t okA = test_full(B_A, ns);
        for (int t = t1 - 1; t >= t0; --t, ++ns) {
            const uint32_t u = ne, c = ne + 1;  // slice loads of t+1 (resident since the previous step) and t
            const T *E0c = E(0, c), *E1c = E(1, c), *E2c = E(2, c);
            T m[18], m2[18], acc[18];
            // ---- S1: B U_3(x+0), C U_0(x+t) | B U_3(x+1), C U_1(x+t)   (M_0 | M_1)
            wait_if(okA, B_A, ns);
            const uint32_t okD = test_full(B_E01 + (c & 1), c >> 1), okB = test_full(B_B, ns);
            bcdag_fma<T, true>(h ? (y_in ? E3 + sl + NX : Y3 + lx) : E3 + ix_up, h ? ystr : N,
                               (h ? E(1, u) : E(0, u)) + sl, N, m);
            release(B_A);
            release(B_E01 + (u & 1));
            // lanes 16-31: M_1 waits in m2, M_2 starts from zero
#pragma unroll
            for (int q = 0; q < 18; ++q) {
                m2[q] = m[q];
                m[q] = h ? T(0) : m[q];
            }
            // ---- S2: B U_1(x+0), C U_0(x+1) | B U_3(x+2), C U_2(x+t)   (M_0 | M_2)
            wait_if(okD, B_E01 + (c & 1), c >> 1);
            wait_if(okB, B_B, ns);
            const uint32_t okE = test_full(B_E2 + (c & 1), c >> 1), okC = test_full(B_C, ns);
            bcdag_fma<T, false>(h ? Z3 + sl : E1c + ix_up, N,
                                h ? E(2, u) + sl : (y_in ? E0c + sl + NX : Y0 + lx), h ? N : ystr, m);
            release(B_B);
            release(B_E2 + (u & 1));
            // lanes 16-31: M_2 is complete (kept in m2), back to M_1
#pragma unroll
            for (int q = 0; q < 18; ++q) {
                const T t2 = m[q];
                m[q] = h ? m2[q] : t2;
                m2[q] = t2;
            }
            // ---- S3: B U_2(x+0), C U_0(x+2) | B U_2(x+1), C U_1(x+2)   (M_0 | M_1)
            wait_if(okE, B_E2 + (c & 1), c >> 1);
            wait_if(okC, B_C, ns);
            bcdag_fma<T, false>(h ? (y_in ? E2c + sl + NX : Y2 + lx) : E2c + ix_up, h ? ystr : N,
                                (h ? Z1 : Z0) + sl, N, m);
            release(B_C);
            if (t > t0) okA = test_full(B_A, ns + 1);  // the next step's first operands
            // ---- S4: acc = U_0(x) M_0 | acc = U_1(x) M_1
            am_fma<T, true>((h ? E1c : E0c) + sl, N, m, acc);
            // ---- S5: lanes 16-31 acc += U_2(x) M_2
            if (h) am_fma<T, false>(E2c + sl, N, m2, acc);
            ++ne;
            // ---- the two half-sums meet: lanes 0-15 store elements 0..8, lanes 16-31 elements 9..17
            T* o = acc_out + int64_t(t) * 18 * p.F + s3;
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                const T mine = h ? acc[9 + k] : acc[k];
                const T give = h ? acc[k] : acc[9 + k];
                const T got = __shfl_xor_sync(0xffffffffu, give, 16);
#ifdef FACT_NOSTORE
                if (mine + got == T(123456789)) __stcs(o + (9 * h + k) * p.F, s * (mine + got));
#else
                __stcs(o + (9 * h + k) * p.F, s * (mine + got));
#endif
            }
        }
        // slice t0 stays resident for a next step that the item does not have
        release(B_E01 + (ne & 1));
        release(B_E2 + (ne & 1));
        ++ne;
    }
}

template <typename T, int NX, int BY>
static int run_link_fact(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, cudaStream_t st) {
    using G = PairGeo<T, NX, BY>;
    CUtensorMap mB, mY;
    if (!make_map<T>(&mB, U, nx, ny, nz, int64_t(nt) * 72, BY, 1, 18) ||
        !make_map<T>(&mY, U, nx, ny, nz, int64_t(nt) * 72, 1, 1, 18))
        return 1;
    const size_t smem = size_t(G::TOTAL) * sizeof(T) + 2 * G::NBAR * sizeof(uint64_t);
    const DeviceInfo& di = device_info();
    if (smem > size_t(di.max_smem_optin)) return 1;
    // (an L2 prefetch one step ahead measured slower: f64 0.726 -> 0.693, f32 0.575 -> 0.569; in git history)
    auto kern = k_link_fact<T, NX, BY>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    WalkParams p{};
    p.ny = ny; p.nz = nz; p.nt = nt;
    p.F = int64_t(nx) * ny * nz;
    p.nby = ny / BY;
    p.nblocks = int64_t(ny / BY) * nz;
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::THREADS, smem);
    const int Gfull = di.num_sms * std::max(per_sm, 1);
    // an item of L slices loads L+1 E slices: prologue = 0.5 step; the columns schedule (sweep_common.cuh)
    // unless a chunk length is forced
    const WalkSchedule ws = pick_schedule(p.nblocks, nt, Gfull, 0.5, g_link_chunk == 0);
    p.n_full = ws.n_full;
    p.chunk = ws.chunk;
    if (g_link_chunk > 0) p.chunk = std::min(g_link_chunk, nt);
    p.nitems = p.n_full + (p.nblocks - p.n_full) * ((nt + p.chunk - 1) / p.chunk);
    const int grid = static_cast<int>(std::min<int64_t>(Gfull, p.nitems));
    kern<<<grid, G::THREADS, smem, st>>>(mB, mY, acc, p, s);
    note_kernel(std::string("k_link_fact<") + (sizeof(T) == 4 ? "f32," : "f64,") + std::to_string(NX) + "x" +
                std::to_string(BY) + "x1" + (per_sm > 1 ? "," + std::to_string(per_sm) + " CTAs/SM" : "") +
                (p.n_full ? "," + std::to_string(p.n_full) + " columns" : "") + ",chunk " + std::to_string(p.chunk) + ">");
    return check_launch("link_product(fact)");
}

// FMA mode only; 1 = not applicable to this lattice
template <typename T>
int launch_link_fact(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, cudaStream_t st) {
    if (!aligned16(U)) return 1;
    if (nx == 48 && ny % 3 == 0) return run_link_fact<T, 48, 3>(U, acc, nx, ny, nz, nt, s, st);
    if (nx == 32 && ny % 4 == 0) return run_link_fact<T, 32, 4>(U, acc, nx, ny, nz, nt, s, st);
    if (nx == 64 && ny % 2 == 0) return run_link_fact<T, 64, 2>(U, acc, nx, ny, nz, nt, s, st);
    return 1;
}

template int launch_link_fact<float>(const float*, float*, int, int, int, int, float, cudaStream_t);
template int launch_link_fact<double>(const double*, double*, int, int, int, int, double, cudaStream_t);

// 1 = not applicable to this lattice (caller falls back)
template <typename T, bool FUSED>
int launch_link_walk(const T* U, T* acc, int nx, int ny, int nz, int nt, T s, cudaStream_t st) {
    if (!aligned16(U)) return 1;
    if (nx == 48 && ny % 3 == 0) return run_link_walk<T, FUSED, 48, 3>(U, acc, nx, ny, nz, nt, s, st);
    if (nx == 32 && ny % 4 == 0) return run_link_walk<T, FUSED, 32, 4>(U, acc, nx, ny, nz, nt, s, st);
    if (nx == 64 && ny % 2 == 0) return run_link_walk<T, FUSED, 64, 2>(U, acc, nx, ny, nz, nt, s, st);
    return 1;
}

template int launch_link_walk<float, false>(const float*, float*, int, int, int, int, float, cudaStream_t);
template int launch_link_walk<float, true>(const float*, float*, int, int, int, int, float, cudaStream_t);
template int launch_link_walk<double, false>(const double*, double*, int, int, int, int, double, cudaStream_t);
template int launch_link_walk<double, true>(const double*, double*, int, int, int, int, double, cudaStream_t);

}  // namespace su3g
