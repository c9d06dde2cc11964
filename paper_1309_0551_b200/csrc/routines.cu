// Per-site SU(3) routines on the reference AoS layout, sm_100a.
//
// Design: every routine is a pure stream --
// each site's operands are read once and its result written once, arithmetic
// intensity 0.08-0.9 flop/B -- so the kernel is built to move bytes at HBM
// speed, not to do math:
//   * persistent CTAs (grid = resident CTAs per SM x 148 SMs) walk tiles of TS
//     consecutive sites;
//   * a tile's operand bytes are contiguous in the AoS layout, so one elected
//     thread moves each operand tile with a single TMA bulk copy
//     (cp.async.bulk ... mbarrier::complete_tx, SASS UBLKCP) into a STAGES-deep
//     shared-memory ring, evict-first in L2;
//   * one thread per site loads its record from shared memory with 8/16-byte
//     vector loads (AoS 72-byte f32 matrices are not 16-byte aligned per site,
//     which is why global loads are not done per thread), computes in
//     registers, writes the result record to a double-buffered smem tile;
//   * the result tile goes back with one bulk store (cp.async.bulk.global).
// Sites that do not fill a whole tile are handled by plain per-thread loads
// in the last CTA; misaligned (non-16-byte) base pointers take a direct
// per-thread kernel.  Both paths share the same per-site arithmetic, which is
// the reference association (su3_math.cuh), so every path is bit-identical to
// su3bench.
#include <algorithm>
#include <type_traits>

#include "su3_math.cuh"

namespace su3g {

// ---------------------------------------------------------------------------
// routine descriptors: reals per site of a, b, c; optional per-site scalar
// ---------------------------------------------------------------------------
template <typename T_>
struct OpMatVec {
    using T = T_;
    static constexpr int NA = 18, NB = 6, NC = 6;
    static constexpr bool SCALAR = false;
    static constexpr const char* name = "mult_su3_mat_vec";
    __device__ static void apply(const T* a, const T* b, T, T* c) { mat_vec<T>(a, b, c); }
};
template <typename T_>
struct OpAdjMatVec {
    using T = T_;
    static constexpr int NA = 18, NB = 6, NC = 6;
    static constexpr bool SCALAR = false;
    static constexpr const char* name = "mult_adj_su3_mat_vec";
    __device__ static void apply(const T* a, const T* b, T, T* c) { adj_mat_vec<T>(a, b, c); }
};
template <typename T_>
struct OpNN {
    using T = T_;
    static constexpr int NA = 18, NB = 18, NC = 18;
    static constexpr bool SCALAR = false;
    static constexpr const char* name = "mult_su3_nn";
    __device__ static void apply(const T* a, const T* b, T, T* c) { mat_nn<T>(a, b, c); }
};
template <typename T_>
struct OpNA {
    using T = T_;
    static constexpr int NA = 18, NB = 18, NC = 18;
    static constexpr bool SCALAR = false;
    static constexpr const char* name = "mult_su3_na";
    __device__ static void apply(const T* a, const T* b, T, T* c) { mat_na<T>(a, b, c); }
};
template <typename T_>
struct OpAN {
    using T = T_;
    static constexpr int NA = 18, NB = 18, NC = 18;
    static constexpr bool SCALAR = false;
    static constexpr const char* name = "mult_su3_an";
    __device__ static void apply(const T* a, const T* b, T, T* c) { mat_an<T>(a, b, c); }
};
template <typename T_>
struct OpAdj4Dir {
    using T = T_;
    static constexpr int NA = 72, NB = 6, NC = 24;
    static constexpr bool SCALAR = false;
    static constexpr const char* name = "mult_adj_su3_mat_vec_4dir";
    __device__ static void apply(const T* a, const T* b, T, T* c) { adj_mat_vec_4dir<T>(a, b, c); }
    // 4 threads per site: part d computes c[d] = adj(a4[d]) b
    static constexpr int PARTS = 4;
    __device__ static void apply_part(int d, const T* a, const T* b, T, T* c) {
        T m[18], v[6], r[6];
        load_rec<18>(a + 18 * d, m);
        load_rec<6>(b, v);
        adj_mat_vec<T>(m, v, r);
        store_rec<6>(c + 6 * d, r);
    }
};
template <typename T_>
struct OpSum4Dir {
    using T = T_;
    static constexpr int NA = 72, NB = 24, NC = 6;
    static constexpr bool SCALAR = false;
    static constexpr const char* name = "mult_su3_mat_vec_sum_4dir";
    __device__ static void apply(const T* a, const T* b, T, T* c) { mat_vec_sum_4dir<T>(a, b, c); }
    // 4 threads per site: part i < 3 computes row i (the 12-term sum keeps its d-major order); part 3 idles
    static constexpr int PARTS = 4;
    __device__ static void apply_part(int i, const T* a4, const T* b4, T, T* c) {
        if (i >= 3) return;
        T col[24], v[24];
#pragma unroll
        for (int n = 0; n < 12; ++n) {  // a4[d][j][i], n = 3d + j
            col[2 * n] = a4[18 * (n / 3) + (3 * (n % 3) + i) * 2];
            col[2 * n + 1] = a4[18 * (n / 3) + (3 * (n % 3) + i) * 2 + 1];
        }
        load_rec<24>(b4, v);
        cdot<T, CONJ_P, 12>([&](int n, int r) { return col[2 * n + r]; }, [&](int n, int r) { return v[2 * n + r]; },
                            c[2 * i], c[2 * i + 1]);
    }
};
template <typename T_>
struct OpSmadd {
    using T = T_;
    static constexpr int NA = 18, NB = 18, NC = 18;
    static constexpr bool SCALAR = true;
    static constexpr const char* name = "scalar_mult_add_su3_matrix";
    __device__ static void apply(const T* a, const T* b, T s, T* c) { scalar_mult_add<T, 18>(a, b, s, c); }
};

// --- the other seven Table-1 routines (reference scalar.py:39-46, 122-165, 208-238) ---
template <typename T_>
struct OpAddVec {  // c = a + b  (scalar.py:39-46)
    using T = T_;
    static constexpr int NA = 6, NB = 6, NC = 6;
    static constexpr bool SCALAR = false;
    static constexpr const char* name = "add_su3_vector";
    __device__ static void apply(const T* a, const T* b, T, T* c) {
#pragma unroll
        for (int k = 0; k < 6; ++k) c[k] = xadd(a[k], b[k]);
    }
};
template <typename T_>
struct OpSmaddVec {  // c = a + s*b  (scalar.py:208-215)
    using T = T_;
    static constexpr int NA = 6, NB = 6, NC = 6;
    static constexpr bool SCALAR = true;
    static constexpr const char* name = "scalar_mult_add_su3_vector";
    __device__ static void apply(const T* a, const T* b, T s, T* c) { scalar_mult_add<T, 6>(a, b, s, c); }
};
template <typename T_>
struct OpMatHw {  // c[k] = a h[k], k = 0, 1  (scalar.py:122-128)
    using T = T_;
    static constexpr int NA = 18, NB = 12, NC = 12;
    static constexpr bool SCALAR = false;
    static constexpr const char* name = "mult_su3_mat_hwvec";
    __device__ static void apply(const T* a, const T* h, T, T* c) {
        mat_vec<T>(a, h, c);
        mat_vec<T>(a, h + 6, c + 6);
    }
};
template <typename T_>
struct OpAdjMatHw {  // c[k] = adj(a) h[k], k = 0, 1  (scalar.py:131-137)
    using T = T_;
    static constexpr int NA = 18, NB = 12, NC = 12;
    static constexpr bool SCALAR = false;
    static constexpr const char* name = "mult_adj_su3_mat_hwvec";
    __device__ static void apply(const T* a, const T* h, T, T* c) {
        adj_mat_vec<T>(a, h, c);
        adj_mat_vec<T>(a, h + 6, c + 6);
    }
};
template <typename T_>
struct OpProjector {  // c[i][j] = a[i] conj(b[j])  (scalar.py:218-230)
    using T = T_;
    static constexpr int NA = 6, NB = 6, NC = 18;
    static constexpr bool SCALAR = false;
    static constexpr const char* name = "su3_projector";
    __device__ static void apply(const T* a, const T* b, T, T* c) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
                const T rr = xmul(b[2 * j], a[2 * i]), ir = xmul(b[2 * j], a[2 * i + 1]);
                const T ri = xmul(b[2 * j + 1], a[2 * i]), ii = xmul(b[2 * j + 1], a[2 * i + 1]);
                c[2 * (3 * i + j)] = xadd(rr, ii);
                c[2 * (3 * i + j) + 1] = xsub(ir, ri);
            }
    }
};
// c_d = adj(a4[d]) b into four separate destinations  (scalar.py:149-165): the 4dir
// arithmetic, results split per direction (SPLIT: part d's record goes to destination d)
template <typename T_>
struct OpAdj4Vec : OpAdj4Dir<T_> {
    using T = T_;
    static constexpr const char* name = "mult_adj_su3_mat_4vec";
    static constexpr bool SPLIT = true;
    __device__ static void apply_part(int d, const T* a, const T* b, T, T* c) {
        T m[18], v[6], r[6];
        load_rec<18>(a + 18 * d, m);
        load_rec<6>(b, v);
        adj_mat_vec<T>(m, v, r);
        store_rec<6>(c, r);
    }
};

// tile geometry per routine: ~12-24 KiB of operands per stage
template <class Op>
struct Geometry {
    using T = typename Op::T;
    static constexpr int IN_BYTES = (Op::NA + Op::NB + (Op::SCALAR ? 1 : 0)) * int(sizeof(T));
    static constexpr int TS = IN_BYTES <= 160 ? 128 : (IN_BYTES <= 320 ? 64 : 32);
    static constexpr int STAGES = 4;
    static constexpr uint32_t A_BYTES = TS * Op::NA * sizeof(T);
    static constexpr uint32_t B_BYTES = TS * Op::NB * sizeof(T);
    static constexpr uint32_t S_BYTES = Op::SCALAR ? TS * sizeof(T) : 0;
    static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES + S_BYTES;
    static constexpr uint32_t C_BYTES = TS * Op::NC * sizeof(T);
    static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 2 * C_BYTES + STAGES * 8;
    static_assert(A_BYTES % 16 == 0 && B_BYTES % 16 == 0 && S_BYTES % 16 == 0 && C_BYTES % 16 == 0, "bulk sizes");
};

// one site through global memory (tail / misaligned path); identical arithmetic
template <class Op>
__device__ __forceinline__ void site_direct(const typename Op::T* __restrict__ A, const typename Op::T* __restrict__ B,
                                            const typename Op::T* __restrict__ S, typename Op::T s,
                                            typename Op::T* __restrict__ C, int64_t x) {
    using T = typename Op::T;
    T a[Op::NA], b[Op::NB], c[Op::NC];
#pragma unroll
    for (int k = 0; k < Op::NA; ++k) a[k] = A[x * Op::NA + k];
#pragma unroll
    for (int k = 0; k < Op::NB; ++k) b[k] = B[x * Op::NB + k];
    if (Op::SCALAR && S != nullptr) s = S[x];
    Op::apply(a, b, s, c);
#pragma unroll
    for (int k = 0; k < Op::NC; ++k) C[x * Op::NC + k] = c[k];
}

template <class Op>
__global__ void __launch_bounds__(Geometry<Op>::TS)
    k_stream(const typename Op::T* __restrict__ A, const typename Op::T* __restrict__ B,
             const typename Op::T* __restrict__ S, typename Op::T s_scalar, typename Op::T* __restrict__ C, int64_t n) {
    using T = typename Op::T;
    using G = Geometry<Op>;
    constexpr int TS = G::TS, STAGES = G::STAGES;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* stages = smem;
    T* obuf = reinterpret_cast<T*>(smem + STAGES * G::STAGE_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * G::STAGE_BYTES + 2 * G::C_BYTES);

    const int tid = threadIdx.x;
    const int64_t ntiles = n / TS;
    const bool has_s = Op::SCALAR && S != nullptr;
    const uint32_t tx_bytes = G::A_BYTES + G::B_BYTES + (has_s ? G::S_BYTES : 0u);
    const int64_t first = blockIdx.x, stride = gridDim.x;
    const int64_t count = ntiles > first ? (ntiles - first + stride - 1) / stride : 0;

    if (tid == 0) {
#pragma unroll
        for (int st = 0; st < STAGES; ++st) mbar_init(&full[st], 1);
        fence_mbar_init();
    }
    __syncthreads();

    uint64_t pol = 0;
    if (tid == 0) pol = policy_evict_first();
    auto issue = [&](int64_t tile, int st) {
        unsigned char* base = stages + st * G::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[st], tx_bytes);
        bulk_g2s(base, A + tile * TS * Op::NA, G::A_BYTES, &full[st], pol);
        bulk_g2s(base + G::A_BYTES, B + tile * TS * Op::NB, G::B_BYTES, &full[st], pol);
        if (has_s) bulk_g2s(base + G::A_BYTES + G::B_BYTES, S + tile * TS, G::S_BYTES, &full[st], pol);
    };
    if (tid == 0) {
        for (int k = 0; k < STAGES && k < count; ++k) issue(first + k * stride, k);
    }

    for (int64_t k = 0; k < count; ++k) {
        const int st = static_cast<int>(k % STAGES);
        const uint32_t parity = static_cast<uint32_t>((k / STAGES) & 1);
        const int64_t tile = first + k * stride;
        mbar_wait(&full[st], parity);

        const unsigned char* base = stages + st * G::STAGE_BYTES;
        T a[Op::NA], b[Op::NB], c[Op::NC];
        T s = s_scalar;
        load_rec<Op::NA>(reinterpret_cast<const T*>(base) + tid * Op::NA, a);
        load_rec<Op::NB>(reinterpret_cast<const T*>(base + G::A_BYTES) + tid * Op::NB, b);
        if (has_s) s = reinterpret_cast<const T*>(base + G::A_BYTES + G::B_BYTES)[tid];

        if (tid == 0) bulk_wait_read<1>();  // result buffer (k & 1) released by the store of tile k-2
        __syncthreads();                     // stage st fully consumed; obuf (k & 1) free
        if (tid == 0 && k + STAGES < count) {
            fence_before_refill();           // the barrier's reads of stage st before the bulk refill
            issue(first + (k + STAGES) * stride, st);
        }

        Op::apply(a, b, s, c);
        T* ob = obuf + (k & 1) * TS * Op::NC;
        store_rec<Op::NC>(ob + tid * Op::NC, c);
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            bulk_s2g(C + tile * TS * Op::NC, ob, G::C_BYTES);
            bulk_commit();
        }
    }

    if (blockIdx.x == gridDim.x - 1) {
        for (int64_t x = ntiles * TS + tid; x < n; x += TS) site_direct<Op>(A, B, S, s_scalar, C, x);
    }
    if (tid == 0) bulk_wait<0>();
}

template <class Op>
__global__ void __launch_bounds__(256)
    k_direct(const typename Op::T* __restrict__ A, const typename Op::T* __restrict__ B,
             const typename Op::T* __restrict__ S, typename Op::T s_scalar, typename Op::T* __restrict__ C, int64_t n) {
    for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < n; x += int64_t(gridDim.x) * blockDim.x)
        site_direct<Op>(A, B, S, s_scalar, C, x);
}

template <class Op>
struct LaunchCache {
    int blocks_per_sm[64] = {0};
};

// Variant for wide records (mat4 / vec4 per site): PARTS threads per site read their
// share of the record straight from the staged tile (conflict-free: lanes of a site hit
// disjoint banks), so no thread holds the whole 96-real record in registers.
template <class Op>
struct PartsGeometry {
    using T = typename Op::T;
    static constexpr int IN_BYTES = (Op::NA + Op::NB) * int(sizeof(T));
    static constexpr int TS = IN_BYTES <= 400 ? 64 : 32;
    static constexpr int THREADS = TS * Op::PARTS;
    static constexpr int STAGES = 4;
    static constexpr uint32_t A_BYTES = TS * Op::NA * sizeof(T);
    static constexpr uint32_t B_BYTES = TS * Op::NB * sizeof(T);
    static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr uint32_t C_BYTES = TS * Op::NC * sizeof(T);
    static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + 2 * C_BYTES + STAGES * 8;
};

template <class Op, class = void>
struct IsSplit : std::false_type {};
template <class Op>
struct IsSplit<Op, std::void_t<decltype(Op::SPLIT)>> : std::bool_constant<Op::SPLIT> {};

// result destinations: p[0] = the packed result, or p[0..PARTS-1] = one array per part (SPLIT)
template <typename T>
struct Dest {
    T* p[4];
};

// one site of a SPLIT routine through global memory (tail / misaligned path)
template <class Op>
__device__ __forceinline__ void site_direct_split(const typename Op::T* __restrict__ A,
                                                  const typename Op::T* __restrict__ B, Dest<typename Op::T> C,
                                                  int64_t x) {
    using T = typename Op::T;
    constexpr int W = Op::NC / Op::PARTS;
    T a[Op::NA], b[Op::NB], c[Op::NC];
#pragma unroll
    for (int k = 0; k < Op::NA; ++k) a[k] = A[x * Op::NA + k];
#pragma unroll
    for (int k = 0; k < Op::NB; ++k) b[k] = B[x * Op::NB + k];
    Op::apply(a, b, T(0), c);
#pragma unroll
    for (int d = 0; d < Op::PARTS; ++d)
#pragma unroll
        for (int k = 0; k < W; ++k) C.p[d][x * W + k] = c[W * d + k];
}

template <class Op>
__global__ void __launch_bounds__(256)
    k_direct_split(const typename Op::T* __restrict__ A, const typename Op::T* __restrict__ B, Dest<typename Op::T> C,
                   int64_t n) {
    for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < n; x += int64_t(gridDim.x) * blockDim.x)
        site_direct_split<Op>(A, B, C, x);
}

template <class Op>
__global__ void __launch_bounds__(PartsGeometry<Op>::THREADS)
    k_stream_parts(const typename Op::T* __restrict__ A, const typename Op::T* __restrict__ B,
                   Dest<typename Op::T> D, int64_t n) {
    using T = typename Op::T;
    using G = PartsGeometry<Op>;
    constexpr bool SPLIT = IsSplit<Op>::value;
    constexpr int W = Op::NC / Op::PARTS;  // reals per part's result record
    T* __restrict__ C = D.p[0];
    constexpr int TS = G::TS, STAGES = G::STAGES;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* stages = smem;
    T* obuf = reinterpret_cast<T*>(smem + STAGES * G::STAGE_BYTES);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * G::STAGE_BYTES + 2 * G::C_BYTES);

    const int tid = threadIdx.x;
    const int site = tid / Op::PARTS, part = tid % Op::PARTS;
    const int64_t ntiles = n / TS;
    const int64_t first = blockIdx.x, stride = gridDim.x;
    const int64_t count = ntiles > first ? (ntiles - first + stride - 1) / stride : 0;

    if (tid == 0) {
#pragma unroll
        for (int st = 0; st < STAGES; ++st) mbar_init(&full[st], 1);
        fence_mbar_init();
    }
    __syncthreads();
    uint64_t pol = 0;
    if (tid == 0) pol = policy_evict_first();
    auto issue = [&](int64_t tile, int st) {
        unsigned char* base = stages + st * G::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[st], G::STAGE_BYTES);
        bulk_g2s(base, A + tile * TS * Op::NA, G::A_BYTES, &full[st], pol);
        bulk_g2s(base + G::A_BYTES, B + tile * TS * Op::NB, G::B_BYTES, &full[st], pol);
    };
    if (tid == 0) {
        for (int k = 0; k < STAGES && k < count; ++k) issue(first + k * stride, k);
    }
    for (int64_t k = 0; k < count; ++k) {
        const int st = static_cast<int>(k % STAGES);
        const int64_t tile = first + k * stride;
        mbar_wait(&full[st], static_cast<uint32_t>((k / STAGES) & 1));
        const unsigned char* base = stages + st * G::STAGE_BYTES;
        if (tid == 0) bulk_wait_read<1>();  // result buffer (k & 1) released by the store of tile k-2
        __syncthreads();
        T* ob = obuf + (k & 1) * TS * Op::NC;
        // SPLIT: the result tile is [part][site][W] so each destination's slice is contiguous
        T* dst = SPLIT ? ob + part * TS * W + site * W : ob + site * Op::NC;
        Op::apply_part(part, reinterpret_cast<const T*>(base) + site * Op::NA,
                       reinterpret_cast<const T*>(base + G::A_BYTES) + site * Op::NB, T(0), dst);
        fence_proxy_async_smem();
        __syncthreads();  // tile consumed and results written
        if (tid == 0) {
            if constexpr (SPLIT) {
#pragma unroll
                for (int d = 0; d < Op::PARTS; ++d)
                    bulk_s2g(D.p[d] + tile * TS * W, ob + d * TS * W, G::C_BYTES / Op::PARTS);
            } else {
                bulk_s2g(C + tile * TS * Op::NC, ob, G::C_BYTES);
            }
            bulk_commit();
            if (k + STAGES < count) issue(first + (k + STAGES) * stride, st);
        }
    }
    if (blockIdx.x == gridDim.x - 1) {
        for (int64_t x = ntiles * TS + tid; x < n; x += G::THREADS) {
            if constexpr (SPLIT)
                site_direct_split<Op>(A, B, D, x);
            else
                site_direct<Op>(A, B, nullptr, T(0), C, x);
        }
    }
    if (tid == 0) bulk_wait<0>();
}

template <class Op>
int launch_parts(const typename Op::T* a, const typename Op::T* b, Dest<typename Op::T> c, int64_t n,
                 cudaStream_t stream) {
    using G = PartsGeometry<Op>;
    const DeviceInfo& di = device_info();
    static LaunchCache<Op> cache;
    int& per_sm = cache.blocks_per_sm[di.device & 63];
    if (per_sm == 0) {
        cudaFuncSetAttribute(k_stream_parts<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(G::SMEM));
        int bl = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bl, k_stream_parts<Op>, G::THREADS, G::SMEM);
        per_sm = std::max(bl, 1);
    }
    const int64_t ntiles = n / G::TS;
    int64_t grid = std::min<int64_t>(ntiles, int64_t(per_sm) * di.num_sms);
    if (grid < 1) grid = 1;
    k_stream_parts<Op><<<static_cast<unsigned>(grid), G::THREADS, G::SMEM, stream>>>(a, b, c, n);
    note_kernel(std::string("k_stream_parts<") + Op::name + ">");
    return check_launch(Op::name);
}


template <class Op, class = void>
struct HasParts : std::false_type {};
template <class Op>
struct HasParts<Op, std::void_t<decltype(Op::PARTS)>> : std::true_type {};

template <class Op>
int launch(const typename Op::T* a, const typename Op::T* b, const typename Op::T* s_site, typename Op::T s,
           typename Op::T* c, int64_t n, cudaStream_t stream) {
    using G = Geometry<Op>;
    if (n < 0) return fail_invalid(std::string(Op::name) + ": negative site count");
    if (n == 0) return SU3G_OK;
    if (a == nullptr || b == nullptr || c == nullptr) return fail_invalid(std::string(Op::name) + ": null pointer");
    const DeviceInfo& di = device_info();
    if (di.num_sms <= 0) return fail_invalid(std::string(Op::name) + ": no CUDA device");
    const bool aligned = aligned16(a) && aligned16(b) && aligned16(c) && (s_site == nullptr || aligned16(s_site));
    if (!aligned) {
        const int64_t grid = std::min<int64_t>((n + 255) / 256, int64_t(di.num_sms) * 8);
        k_direct<Op><<<static_cast<unsigned>(grid), 256, 0, stream>>>(a, b, s_site, s, c, n);
        note_kernel(std::string("k_direct<") + Op::name + ">");
        return check_launch(Op::name);
    }
    if constexpr (HasParts<Op>::value) return launch_parts<Op>(a, b, Dest<typename Op::T>{{c, c, c, c}}, n, stream);
    static LaunchCache<Op> cache;
    int& per_sm = cache.blocks_per_sm[di.device & 63];
    if (per_sm == 0) {
        cudaFuncSetAttribute(k_stream<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(G::SMEM));
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_stream<Op>, G::TS, G::SMEM);
        per_sm = std::max(b, 1);
    }
    const int64_t ntiles = n / G::TS;
    int64_t grid = std::min<int64_t>(ntiles, int64_t(per_sm) * di.num_sms);
    if (grid < 1) grid = 1;
    k_stream<Op><<<static_cast<unsigned>(grid), G::TS, G::SMEM, stream>>>(a, b, s_site, s, c, n);
    note_kernel(std::string("k_stream<") + Op::name + ">");
    return check_launch(Op::name);
}

template <class Op>
int launch_split(const typename Op::T* a, const typename Op::T* b, Dest<typename Op::T> c, int64_t n,
                 cudaStream_t stream) {
    if (n < 0) return fail_invalid(std::string(Op::name) + ": negative site count");
    if (n == 0) return SU3G_OK;
    bool aligned = aligned16(a) && aligned16(b);
    for (int d = 0; d < Op::PARTS; ++d) {
        if (c.p[d] == nullptr) return fail_invalid(std::string(Op::name) + ": null destination");
        aligned = aligned && aligned16(c.p[d]);
    }
    if (a == nullptr || b == nullptr) return fail_invalid(std::string(Op::name) + ": null pointer");
    const DeviceInfo& di = device_info();
    if (di.num_sms <= 0) return fail_invalid(std::string(Op::name) + ": no CUDA device");
    if (!aligned) {
        const int64_t grid = std::min<int64_t>((n + 255) / 256, int64_t(di.num_sms) * 8);
        k_direct_split<Op><<<static_cast<unsigned>(grid), 256, 0, stream>>>(a, b, c, n);
        note_kernel(std::string("k_direct_split<") + Op::name + ">");
        return check_launch(Op::name);
    }
    return launch_parts<Op>(a, b, c, n, stream);
}

// a <- ((((a - b1) - b2) - b3) - b4) in place  (reference scalar.py:233-238, simd.py:254-259).
// Purely elementwise over the n*6 reals, so the kernel streams flat vectors of 16 B
// (float4 / double2) per operand -- coalesced global loads, no staging needed.
template <typename T>
__device__ __forceinline__ T sub4(T a, T b1, T b2, T b3, T b4) {
    return xsub(xsub(xsub(xsub(a, b1), b2), b3), b4);
}

template <typename T, typename V>
__global__ void __launch_bounds__(256) k_sub_four(T* __restrict__ a, const T* __restrict__ b1,
                                                  const T* __restrict__ b2, const T* __restrict__ b3,
                                                  const T* __restrict__ b4, int64_t m, int vectorised) {
    constexpr int L = sizeof(V) / sizeof(T);
    const int64_t tid = blockIdx.x * int64_t(blockDim.x) + threadIdx.x, nth = int64_t(gridDim.x) * blockDim.x;
    int64_t done = 0;
    if (vectorised) {
        const int64_t mv = m / L;
        V* av = reinterpret_cast<V*>(a);
        for (int64_t i = tid; i < mv; i += nth) {
            V x = av[i];
            const V y1 = reinterpret_cast<const V*>(b1)[i], y2 = reinterpret_cast<const V*>(b2)[i];
            const V y3 = reinterpret_cast<const V*>(b3)[i], y4 = reinterpret_cast<const V*>(b4)[i];
            T* xs = reinterpret_cast<T*>(&x);
            const T *s1 = reinterpret_cast<const T*>(&y1), *s2 = reinterpret_cast<const T*>(&y2);
            const T *s3 = reinterpret_cast<const T*>(&y3), *s4 = reinterpret_cast<const T*>(&y4);
#pragma unroll
            for (int l = 0; l < L; ++l) xs[l] = sub4(xs[l], s1[l], s2[l], s3[l], s4[l]);
            av[i] = x;
        }
        done = mv * L;
    }
    for (int64_t i = done + tid; i < m; i += nth) a[i] = sub4(a[i], b1[i], b2[i], b3[i], b4[i]);
}

template <typename T, typename V>
int launch_sub_four(T* a, const T* b1, const T* b2, const T* b3, const T* b4, int64_t n, cudaStream_t stream) {
    if (n < 0) return fail_invalid("sub_four_su3_vecs: negative site count");
    if (n == 0) return SU3G_OK;
    if (!a || !b1 || !b2 || !b3 || !b4) return fail_invalid("sub_four_su3_vecs: null pointer");
    const DeviceInfo& di = device_info();
    if (di.num_sms <= 0) return fail_invalid("sub_four_su3_vecs: no CUDA device");
    const int64_t m = n * 6;
    const int vec = aligned16(a) && aligned16(b1) && aligned16(b2) && aligned16(b3) && aligned16(b4);
    constexpr int L = sizeof(V) / sizeof(T);
    const int64_t work = vec ? m / L : m;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, int64_t(di.num_sms) * 8));
    k_sub_four<T, V><<<static_cast<unsigned>(grid), 256, 0, stream>>>(a, b1, b2, b3, b4, m, vec);
    note_kernel(vec ? "k_sub_four<vectorised>" : "k_sub_four<scalar>");
    return check_launch("sub_four_su3_vecs");
}

}  // namespace su3g

using namespace su3g;

#define SU3G_ROUTINE(NAME, OP)                                                                                      \
    extern "C" int su3g_##NAME##_f32(const float* a, const float* b, float* c, int64_t n, su3g_stream_t st) {      \
        return launch<OP<float>>(a, b, nullptr, 0.0f, c, n, reinterpret_cast<cudaStream_t>(st));                 \
    }                                                                                                              \
    extern "C" int su3g_##NAME##_f64(const double* a, const double* b, double* c, int64_t n, su3g_stream_t st) {   \
        return launch<OP<double>>(a, b, nullptr, 0.0, c, n, reinterpret_cast<cudaStream_t>(st));                  \
    }

SU3G_ROUTINE(mult_su3_mat_vec, OpMatVec)
SU3G_ROUTINE(mult_adj_su3_mat_vec, OpAdjMatVec)
SU3G_ROUTINE(mult_su3_nn, OpNN)
SU3G_ROUTINE(mult_su3_na, OpNA)
SU3G_ROUTINE(mult_su3_an, OpAN)
SU3G_ROUTINE(mult_adj_su3_mat_vec_4dir, OpAdj4Dir)
SU3G_ROUTINE(mult_su3_mat_vec_sum_4dir, OpSum4Dir)
SU3G_ROUTINE(add_su3_vector, OpAddVec)
SU3G_ROUTINE(mult_su3_mat_hwvec, OpMatHw)
SU3G_ROUTINE(mult_adj_su3_mat_hwvec, OpAdjMatHw)
SU3G_ROUTINE(su3_projector, OpProjector)

extern "C" int su3g_mult_adj_su3_mat_4vec_f32(const float* a4, const float* b, float* c0, float* c1, float* c2,
                                              float* c3, int64_t n, su3g_stream_t st) {
    return launch_split<OpAdj4Vec<float>>(a4, b, Dest<float>{{c0, c1, c2, c3}}, n, reinterpret_cast<cudaStream_t>(st));
}
extern "C" int su3g_mult_adj_su3_mat_4vec_f64(const double* a4, const double* b, double* c0, double* c1, double* c2,
                                              double* c3, int64_t n, su3g_stream_t st) {
    return launch_split<OpAdj4Vec<double>>(a4, b, Dest<double>{{c0, c1, c2, c3}}, n,
                                           reinterpret_cast<cudaStream_t>(st));
}
extern "C" int su3g_scalar_mult_add_su3_vector_f32(const float* a, const float* b, float s, const float* s_site,
                                                   float* c, int64_t n, su3g_stream_t st) {
    return launch<OpSmaddVec<float>>(a, b, s_site, s, c, n, reinterpret_cast<cudaStream_t>(st));
}
extern "C" int su3g_scalar_mult_add_su3_vector_f64(const double* a, const double* b, double s, const double* s_site,
                                                   double* c, int64_t n, su3g_stream_t st) {
    return launch<OpSmaddVec<double>>(a, b, s_site, s, c, n, reinterpret_cast<cudaStream_t>(st));
}
extern "C" int su3g_sub_four_su3_vecs_f32(float* a, const float* b1, const float* b2, const float* b3,
                                          const float* b4, int64_t n, su3g_stream_t st) {
    return launch_sub_four<float, float4>(a, b1, b2, b3, b4, n, reinterpret_cast<cudaStream_t>(st));
}
extern "C" int su3g_sub_four_su3_vecs_f64(double* a, const double* b1, const double* b2, const double* b3,
                                          const double* b4, int64_t n, su3g_stream_t st) {
    return launch_sub_four<double, double2>(a, b1, b2, b3, b4, n, reinterpret_cast<cudaStream_t>(st));
}

extern "C" int su3g_scalar_mult_add_su3_matrix_f32(const float* a, const float* b, float s, const float* s_site,
                                                   float* c, int64_t n, su3g_stream_t st) {
    return launch<OpSmadd<float>>(a, b, s_site, s, c, n, reinterpret_cast<cudaStream_t>(st));
}
extern "C" int su3g_scalar_mult_add_su3_matrix_f64(const double* a, const double* b, double s, const double* s_site,
                                                   double* c, int64_t n, su3g_stream_t st) {
    return launch<OpSmadd<double>>(a, b, s_site, s, c, n, reinterpret_cast<cudaStream_t>(st));
}
