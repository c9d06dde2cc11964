// Seeded uniform fill in HBM, bit-identical to numpy's Generator.uniform.
//
// The reference fills its fields with
//     rng = np.random.default_rng(seed); arr[...] = rng.uniform(-1.0, 1.0, size=arr.shape)
// per field in sorted name order (lattice.py:192-197).  numpy's default bit
// generator is PCG64 (XSL-RR 128/64):
//     state <- state * M + inc   (mod 2^128);   out = rotr64(hi ^ lo, state >> 122)
// and uniform(low, high) = low + (high - low) * ((out >> 11) * 2^-53), in double.
// Here every thread jumps straight to its first draw (LCG jump-ahead in
// O(log n) 128-bit multiply-adds) and then strides through the array with a
// precomputed jump of grid-size steps, so the stream is produced at HBM speed
// with coalesced stores and no host round trip.  The seed itself (numpy's
// SeedSequence hashing) is resolved on the host: the caller passes the
// generator's 128-bit state and increment as numpy reports them.
#include <algorithm>

#include "su3g_common.cuh"

namespace su3g {

struct U128 {
    unsigned long long lo, hi;
};

__host__ __device__ __forceinline__ unsigned long long mulhi64(unsigned long long a, unsigned long long b) {
#ifdef __CUDA_ARCH__
    return __umul64hi(a, b);
#else
    return static_cast<unsigned long long>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
}

__host__ __device__ __forceinline__ U128 mul128(U128 a, U128 b) {
    return U128{a.lo * b.lo, mulhi64(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo};
}

__host__ __device__ __forceinline__ U128 add128(U128 a, U128 b) {
    const unsigned long long lo = a.lo + b.lo;
    return U128{lo, a.hi + b.hi + (lo < a.lo ? 1ull : 0ull)};
}

// PCG_DEFAULT_MULTIPLIER_128
__host__ __device__ __forceinline__ U128 pcg_mult() { return U128{0x4385DF649FCCF645ull, 0x2360ED051FC65DA4ull}; }

// coefficients (A, C) of the affine map "advance delta steps": s -> A s + C
__host__ __device__ inline void pcg_jump(U128 inc, unsigned long long delta, U128& A, U128& C) {
    U128 am{1, 0}, ap{0, 0}, cm = pcg_mult(), cp = inc;
    while (delta) {
        if (delta & 1) {
            am = mul128(am, cm);
            ap = add128(mul128(ap, cm), cp);
        }
        cp = mul128(add128(cm, U128{1, 0}), cp);
        cm = mul128(cm, cm);
        delta >>= 1;
    }
    A = am;
    C = ap;
}

__device__ __forceinline__ double pcg_uniform01(U128 s) {
    const unsigned long long x = s.hi ^ s.lo;
    const unsigned r = static_cast<unsigned>(s.hi >> 58);
    const unsigned long long out = r ? (x >> r) | (x << (64 - r)) : x;
    return static_cast<double>(out >> 11) * (1.0 / 9007199254740992.0);
}

template <typename T>
__global__ void __launch_bounds__(256)
    k_uniform_fill(U128 s0, U128 inc, U128 jA, U128 jC, long long skip, double low, double range, T* __restrict__ out,
                   long long n) {
    const long long g = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    if (g >= n) return;
    // draw k is the output of the state after k + 1 steps
    U128 A, C;
    pcg_jump(inc, static_cast<unsigned long long>(skip + g + 1), A, C);
    U128 s = add128(mul128(A, s0), C);
    for (long long i = g; i < n; i += stride) {
        const double v = __dadd_rn(low, __dmul_rn(range, pcg_uniform01(s)));
        out[i] = static_cast<T>(v);  // f32 fields: numpy's float64 -> float32 assignment (round to nearest)
        s = add128(mul128(jA, s), jC);
    }
}

template <typename T>
static int uniform_fill(unsigned long long state_hi, unsigned long long state_lo, unsigned long long inc_hi,
                        unsigned long long inc_lo, long long skip, double low, double high, T* out, long long n,
                        cudaStream_t st) {
    if (n < 0 || skip < 0) return fail_invalid("uniform_fill: negative count or skip");
    if (n == 0) return SU3G_OK;
    if (out == nullptr) return fail_invalid("uniform_fill: null pointer");
    const DeviceInfo& di = device_info();
    if (di.num_sms <= 0) return fail_invalid("uniform_fill: no CUDA device");
    const long long grid = std::max<long long>(1, std::min<long long>((n + 255) / 256, 8LL * di.num_sms));
    const U128 inc{inc_lo, inc_hi};
    U128 jA, jC;
    pcg_jump(inc, static_cast<unsigned long long>(grid * 256), jA, jC);
    k_uniform_fill<T><<<static_cast<unsigned>(grid), 256, 0, st>>>(U128{state_lo, state_hi}, inc, jA, jC, skip, low,
                                                                   high - low, out, n);
    return check_launch("uniform_fill");
}

}  // namespace su3g

using namespace su3g;

extern "C" int su3g_uniform_fill_f32(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                                     int64_t skip, double low, double high, float* out, int64_t n, su3g_stream_t st) {
    return uniform_fill<float>(state_hi, state_lo, inc_hi, inc_lo, skip, low, high, out, n,
                               reinterpret_cast<cudaStream_t>(st));
}
extern "C" int su3g_uniform_fill_f64(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                                     int64_t skip, double low, double high, double* out, int64_t n, su3g_stream_t st) {
    return uniform_fill<double>(state_hi, state_lo, inc_hi, inc_lo, skip, low, high, out, n,
                                reinterpret_cast<cudaStream_t>(st));
}
