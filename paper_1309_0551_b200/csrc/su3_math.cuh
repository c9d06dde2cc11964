// Per-site SU(3) arithmetic on register records, sm_100a.
//
// Records use the reference pair layout (su3bench types.py:1-13):
//   vector  [6]  = (re, im) x 3
//   matrix  [18] = row-major (i, j) -> [(3*i + j)*2 + {0: re, 1: im}]
//
// Exact variants follow the reference association bit for bit (scalar.py:8-14):
// four separated real sums rr, ri, ir, ii accumulated left to right over the
// contraction index, one combining add/subtract at the end, no FMA.
// Fused variants (suffix _fma) use FMA chains; they are within the north-star
// tolerance (fp64 1e-12) but not bitwise, and are only used where FMA removes a
// compute bound (the f64 link product, SURVEY.md section 7 "Hard parts").
#pragma once

#include "su3g_common.cuh"

namespace su3g {

// combine modes (simd.py:35-48 "_sign"):
//   PLAIN  p*q        -> (rr - ii, ri + ir)
//   CONJ_P conj(p)*q  -> (rr + ii, ri - ir)
//   CONJ_Q p*conj(q)  -> (rr + ii, ir - ri)
enum Mode { PLAIN = 0, CONJ_P = 1, CONJ_Q = 2 };

template <typename T, int MODE>
__device__ __forceinline__ void combine(T rr, T ri, T ir, T ii, T& re, T& im) {
    if constexpr (MODE == PLAIN) {
        re = xsub(rr, ii);
        im = xadd(ri, ir);
    } else if constexpr (MODE == CONJ_P) {
        re = xadd(rr, ii);
        im = xsub(ri, ir);
    } else {
        re = xadd(rr, ii);
        im = xsub(ir, ri);
    }
}

// Exact complex dot over NT ordered terms; p(j, part) / q(j, part) fetch term j.
template <typename T, int MODE, int NT, class PF, class QF>
__device__ __forceinline__ void cdot(PF p, QF q, T& re, T& im) {
    T rr, ri, ir, ii;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        const T pr = p(j, 0), pi = p(j, 1), qr = q(j, 0), qi = q(j, 1);
        if (j == 0) {
            rr = xmul(pr, qr);
            ri = xmul(pr, qi);
            ir = xmul(pi, qr);
            ii = xmul(pi, qi);
        } else {
            rr = xadd(rr, xmul(pr, qr));
            ri = xadd(ri, xmul(pr, qi));
            ir = xadd(ir, xmul(pi, qr));
            ii = xadd(ii, xmul(pi, qi));
        }
    }
    combine<T, MODE>(rr, ri, ir, ii, re, im);
}

// c[i] = sum_j a[i][j] b[j]                 (scalar.py:49-60)
template <typename T>
__device__ __forceinline__ void mat_vec(const T* a, const T* b, T* c) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
        cdot<T, PLAIN, 3>([&](int j, int r) { return a[(3 * i + j) * 2 + r]; },
                          [&](int j, int r) { return b[2 * j + r]; }, c[2 * i], c[2 * i + 1]);
}

// c[i] = sum_j conj(a[j][i]) b[j]           (scalar.py:63-74)
template <typename T>
__device__ __forceinline__ void adj_mat_vec(const T* a, const T* b, T* c) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
        cdot<T, CONJ_P, 3>([&](int j, int r) { return a[(3 * j + i) * 2 + r]; },
                           [&](int j, int r) { return b[2 * j + r]; }, c[2 * i], c[2 * i + 1]);
}

// c[i][k] = sum_j a[i][j] b[j][k]           (scalar.py:77-89)
template <typename T>
__device__ __forceinline__ void mat_nn(const T* a, const T* b, T* c) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            cdot<T, PLAIN, 3>([&](int j, int r) { return a[(3 * i + j) * 2 + r]; },
                              [&](int j, int r) { return b[(3 * j + k) * 2 + r]; }, c[(3 * i + k) * 2],
                              c[(3 * i + k) * 2 + 1]);
}

// c[i][k] = sum_j a[i][j] conj(b[k][j])     (scalar.py:92-104)
template <typename T>
__device__ __forceinline__ void mat_na(const T* a, const T* b, T* c) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            cdot<T, CONJ_Q, 3>([&](int j, int r) { return a[(3 * i + j) * 2 + r]; },
                               [&](int j, int r) { return b[(3 * k + j) * 2 + r]; }, c[(3 * i + k) * 2],
                               c[(3 * i + k) * 2 + 1]);
}

// c[i][k] = sum_j conj(a[j][i]) b[j][k]     (scalar.py:107-119)
template <typename T>
__device__ __forceinline__ void mat_an(const T* a, const T* b, T* c) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            cdot<T, CONJ_P, 3>([&](int j, int r) { return a[(3 * j + i) * 2 + r]; },
                               [&](int j, int r) { return b[(3 * j + k) * 2 + r]; }, c[(3 * i + k) * 2],
                               c[(3 * i + k) * 2 + 1]);
}

// c[d] = adj(a4[d]) b                        (scalar.py:140-146)
template <typename T>
__device__ __forceinline__ void adj_mat_vec_4dir(const T* a4, const T* b, T* c) {
#pragma unroll
    for (int d = 0; d < 4; ++d) adj_mat_vec<T>(a4 + 18 * d, b, c + 6 * d);
}

// c = sum_d adj(a4[d]) b4[d], one 12-term sum per row, direction-major (scalar.py:168-194)
template <typename T>
__device__ __forceinline__ void mat_vec_sum_4dir(const T* a4, const T* b4, T* c) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
        cdot<T, CONJ_P, 12>([&](int n, int r) { return a4[18 * (n / 3) + (3 * (n % 3) + i) * 2 + r]; },
                            [&](int n, int r) { return b4[6 * (n / 3) + 2 * (n % 3) + r]; }, c[2 * i],
                            c[2 * i + 1]);
}

// c = a + (s * b), two roundings               (scalar.py:197-205)
template <typename T, int N>
__device__ __forceinline__ void scalar_mult_add(const T* a, const T* b, T s, T* c) {
#pragma unroll
    for (int k = 0; k < N; ++k) c[k] = xadd(a[k], xmul(s, b[k]));
}

// ---------------------------------------------------------------------------
// fused (FMA) variants
// ---------------------------------------------------------------------------
template <typename T, int MODE, int NT, class PF, class QF>
__device__ __forceinline__ void cdot_fma(PF p, QF q, T& re, T& im) {
    // PLAIN: re += pr*qr - pi*qi ; im += pr*qi + pi*qr
    // CONJ_P: re += pr*qr + pi*qi ; im += pr*qi - pi*qr
    // CONJ_Q: re += pr*qr + pi*qi ; im += pi*qr - pr*qi
    constexpr T sre = (MODE == PLAIN) ? T(-1) : T(1);
    T a_re, a_im;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        const T pr = p(j, 0), pi = p(j, 1), qr = q(j, 0), qi = q(j, 1);
        if (j == 0) {
            a_re = pr * qr;
            if constexpr (MODE == CONJ_Q) a_im = pi * qr;
            else a_im = pr * qi;
        } else {
            a_re = fma(pr, qr, a_re);
            if constexpr (MODE == CONJ_Q) a_im = fma(pi, qr, a_im);
            else a_im = fma(pr, qi, a_im);
        }
        a_re = fma(sre * pi, qi, a_re);
        if constexpr (MODE == PLAIN) a_im = fma(pi, qr, a_im);
        else if constexpr (MODE == CONJ_P) a_im = fma(-pi, qr, a_im);
        else a_im = fma(-pr, qi, a_im);
    }
    re = a_re;
    im = a_im;
}

template <typename T>
__device__ __forceinline__ void mat_vec_fma(const T* a, const T* b, T* c) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
        cdot_fma<T, PLAIN, 3>([&](int j, int r) { return a[(3 * i + j) * 2 + r]; },
                              [&](int j, int r) { return b[2 * j + r]; }, c[2 * i], c[2 * i + 1]);
}

template <typename T>
__device__ __forceinline__ void adj_mat_vec_fma(const T* a, const T* b, T* c) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
        cdot_fma<T, CONJ_P, 3>([&](int j, int r) { return a[(3 * j + i) * 2 + r]; },
                               [&](int j, int r) { return b[2 * j + r]; }, c[2 * i], c[2 * i + 1]);
}

// compile-time switch between the exact (reference association) and FMA forms
template <typename T, bool FUSED>
__device__ __forceinline__ void mv(const T* a, const T* b, T* c) {
    if constexpr (FUSED) mat_vec_fma<T>(a, b, c);
    else mat_vec<T>(a, b, c);
}
template <typename T, bool FUSED>
__device__ __forceinline__ void amv(const T* a, const T* b, T* c) {
    if constexpr (FUSED) adj_mat_vec_fma<T>(a, b, c);
    else adj_mat_vec<T>(a, b, c);
}

template <typename T>
__device__ __forceinline__ void mat_nn_fma(const T* a, const T* b, T* c) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            cdot_fma<T, PLAIN, 3>([&](int j, int r) { return a[(3 * i + j) * 2 + r]; },
                                  [&](int j, int r) { return b[(3 * j + k) * 2 + r]; }, c[(3 * i + k) * 2],
                                  c[(3 * i + k) * 2 + 1]);
}

template <typename T>
__device__ __forceinline__ void mat_na_fma(const T* a, const T* b, T* c) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            cdot_fma<T, CONJ_Q, 3>([&](int j, int r) { return a[(3 * i + j) * 2 + r]; },
                                   [&](int j, int r) { return b[(3 * k + j) * 2 + r]; }, c[(3 * i + k) * 2],
                                   c[(3 * i + k) * 2 + 1]);
}

}  // namespace su3g
