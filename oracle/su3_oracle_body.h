/* C restatement of the reference's per-site SU(3) arithmetic -- TEST ORACLE ONLY.
 *
 * Included twice by su3_oracle.c with REAL = float / double and SFX = f32 / f64.
 * Compiled with -ffp-contract=off -fno-fast-math: every * and + is one IEEE
 * rounding, in the association of the reference
 *   scalar.py:49-60   mult_su3_mat_vec         c = (rr - ii, ri + ir)
 *   scalar.py:63-74   mult_adj_su3_mat_vec     c = (rr + ii, ri - ir)
 *   scalar.py:77-89   mult_su3_nn              c = (rr - ii, ri + ir)
 *   scalar.py:92-104  mult_su3_na              c = (rr + ii, ir - ri)
 *   scalar.py:107-119 mult_su3_an              c = (rr + ii, ri - ir)
 *   scalar.py:140-146 mult_adj_su3_mat_vec_4dir
 *   scalar.py:168-194 mult_su3_mat_vec_sum_4dir (adjoint, 12-term direction-major sums)
 *   scalar.py:197-205 scalar_mult_add_su3_matrix c = a + (s*b)
 * so its results are bit-identical to oracle/routines.py (checked in tests).
 * Layout: pair layout, matrix element (i,j) re at [(3*i+j)*2], im at +1.
 */

#define M_RE(m, i, j) ((m)[((i) * 3 + (j)) * 2])
#define M_IM(m, i, j) ((m)[((i) * 3 + (j)) * 2 + 1])
#define V_RE(v, j) ((v)[(j) * 2])
#define V_IM(v, j) ((v)[(j) * 2 + 1])

#define CAT_(a, b) a##_##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(name, SFX)

/* mode 0: (rr - ii, ri + ir); 1: (rr + ii, ri - ir); 2: (rr + ii, ir - ri) */
static inline void FN(combine)(REAL rr, REAL ri, REAL ir, REAL ii, int mode, REAL *re, REAL *im) {
    if (mode == 0) { *re = rr - ii; *im = ri + ir; }
    else if (mode == 1) { *re = rr + ii; *im = ri - ir; }
    else { *re = rr + ii; *im = ir - ri; }
}

static void FN(mat_vec)(const REAL *a, const REAL *b, REAL *c) {
    for (int i = 0; i < 3; ++i) {
        REAL rr = M_RE(a, i, 0) * V_RE(b, 0), ri = M_RE(a, i, 0) * V_IM(b, 0);
        REAL ir = M_IM(a, i, 0) * V_RE(b, 0), ii = M_IM(a, i, 0) * V_IM(b, 0);
        for (int j = 1; j < 3; ++j) {
            rr = rr + M_RE(a, i, j) * V_RE(b, j); ri = ri + M_RE(a, i, j) * V_IM(b, j);
            ir = ir + M_IM(a, i, j) * V_RE(b, j); ii = ii + M_IM(a, i, j) * V_IM(b, j);
        }
        FN(combine)(rr, ri, ir, ii, 0, &V_RE(c, i), &V_IM(c, i));
    }
}

static void FN(adj_mat_vec)(const REAL *a, const REAL *b, REAL *c) {
    for (int i = 0; i < 3; ++i) {
        REAL rr = M_RE(a, 0, i) * V_RE(b, 0), ri = M_RE(a, 0, i) * V_IM(b, 0);
        REAL ir = M_IM(a, 0, i) * V_RE(b, 0), ii = M_IM(a, 0, i) * V_IM(b, 0);
        for (int j = 1; j < 3; ++j) {
            rr = rr + M_RE(a, j, i) * V_RE(b, j); ri = ri + M_RE(a, j, i) * V_IM(b, j);
            ir = ir + M_IM(a, j, i) * V_RE(b, j); ii = ii + M_IM(a, j, i) * V_IM(b, j);
        }
        FN(combine)(rr, ri, ir, ii, 1, &V_RE(c, i), &V_IM(c, i));
    }
}

/* kind 0: nn  (p = a[i][j], q = b[j][k]); 1: na (p = a[i][j], q = b[k][j]); 2: an (p = a[j][i], q = b[j][k]) */
static void FN(mat_mat)(const REAL *a, const REAL *b, REAL *c, int kind) {
    static const int mode_of[3] = {0, 2, 1};
    for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) {
            REAL rr = 0, ri = 0, ir = 0, ii = 0;
            for (int j = 0; j < 3; ++j) {
                REAL pr, pi, qr, qi;
                if (kind == 2) { pr = M_RE(a, j, i); pi = M_IM(a, j, i); }
                else { pr = M_RE(a, i, j); pi = M_IM(a, i, j); }
                if (kind == 1) { qr = M_RE(b, k, j); qi = M_IM(b, k, j); }
                else { qr = M_RE(b, j, k); qi = M_IM(b, j, k); }
                if (j == 0) { rr = pr * qr; ri = pr * qi; ir = pi * qr; ii = pi * qi; }
                else { rr = rr + pr * qr; ri = ri + pr * qi; ir = ir + pi * qr; ii = ii + pi * qi; }
            }
            FN(combine)(rr, ri, ir, ii, mode_of[kind], &M_RE(c, i, k), &M_IM(c, i, k));
        }
}

static void FN(sum_4dir)(const REAL *a4, const REAL *b4, REAL *c) {
    for (int i = 0; i < 3; ++i) {
        REAL rr = 0, ri = 0, ir = 0, ii = 0;
        for (int d = 0; d < 4; ++d) {
            const REAL *a = a4 + d * 18, *b = b4 + d * 6;
            for (int j = 0; j < 3; ++j) {
                REAL pr = M_RE(a, j, i), pi = M_IM(a, j, i), qr = V_RE(b, j), qi = V_IM(b, j);
                if (d == 0 && j == 0) { rr = pr * qr; ri = pr * qi; ir = pi * qr; ii = pi * qi; }
                else { rr = rr + pr * qr; ri = ri + pr * qi; ir = ir + pi * qr; ii = ii + pi * qi; }
            }
        }
        FN(combine)(rr, ri, ir, ii, 1, &V_RE(c, i), &V_IM(c, i));
    }
}

static void FN(smadd)(const REAL *a, const REAL *b, REAL s, REAL *c, int n) {
    for (int k = 0; k < n; ++k) c[k] = a[k] + s * b[k];
}

/* routine ids follow include/su3g.h SU3G_R_* */
int FN(su3o_routine)(int routine, const REAL *a, const REAL *b, REAL s, const REAL *s_site, REAL *c, int64_t n) {
    if (n < 0) return -1;
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < n; ++x) {
        switch (routine) {
        case 0: FN(mat_vec)(a + x * 18, b + x * 6, c + x * 6); break;
        case 1: FN(adj_mat_vec)(a + x * 18, b + x * 6, c + x * 6); break;
        case 2: FN(mat_mat)(a + x * 18, b + x * 18, c + x * 18, 0); break;
        case 3: FN(mat_mat)(a + x * 18, b + x * 18, c + x * 18, 1); break;
        case 4: FN(mat_mat)(a + x * 18, b + x * 18, c + x * 18, 2); break;
        case 5:
            for (int d = 0; d < 4; ++d) FN(adj_mat_vec)(a + x * 72 + d * 18, b + x * 6, c + x * 24 + d * 6);
            break;
        case 6: FN(sum_4dir)(a + x * 72, b + x * 24, c + x * 6); break;
        case 7: FN(smadd)(a + x * 18, b + x * 18, s_site ? s_site[x] : s, c + x * 18, 18); break;
        default: break;
        }
    }
    return (routine >= 0 && routine <= 7) ? 0 : -1;
}

static inline int64_t FN(nbr)(int64_t s, int mu, int step, const int64_t *dims) {
    int64_t x = s % dims[0], r = s / dims[0];
    int64_t y = r % dims[1]; r /= dims[1];
    int64_t z = r % dims[2], t = r / dims[2];
    int64_t c[4] = {x, y, z, t};
    c[mu] = (c[mu] + step + dims[mu]) % dims[mu];
    return c[0] + dims[0] * (c[1] + dims[1] * (c[2] + dims[2] * c[3]));
}

/* NN sweep: F = ((fw0+fw1)+fw2)+fw3; out = ((((F-bw0)-bw1)-bw2)-bw3) */
int FN(su3o_nn_sweep)(const REAL *U, const REAL *v, REAL *out, int64_t nx, int64_t ny, int64_t nz, int64_t nt) {
    const int64_t dims[4] = {nx, ny, nz, nt};
    const int64_t V = nx * ny * nz * nt;
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < V; ++s) {
        REAL fw[4][6], bw[4][6];
        for (int mu = 0; mu < 4; ++mu) {
            int64_t up = FN(nbr)(s, mu, +1, dims), dn = FN(nbr)(s, mu, -1, dims);
            FN(mat_vec)(U + (s * 4 + mu) * 18, v + up * 6, fw[mu]);
            FN(adj_mat_vec)(U + (dn * 4 + mu) * 18, v + dn * 6, bw[mu]);
        }
        for (int k = 0; k < 6; ++k) {
            REAL f = ((fw[0][k] + fw[1][k]) + fw[2][k]) + fw[3][k];
            out[s * 6 + k] = (((f - bw[0][k]) - bw[1][k]) - bw[2][k]) - bw[3][k];
        }
    }
    return 0;
}

/* One t-slab of the NN sweep: x, y, z periodic in the slab; the +t neighbour of the
 * last slice is v_hi (the next rank's first slice of v, AoS (F,3,2)); the -t backward term of the first
 * slice is w_lo = U_t(x)^dag v(x) on the previous rank's last slice (AoS (F,3,2)), formed by that rank
 * with the same adj_mat_vec -- so the result equals the unsharded sweep's rows bit for bit. */
int FN(su3o_nn_sweep_slab)(const REAL *U, const REAL *v, const REAL *v_hi, const REAL *w_lo, REAL *out, int64_t nx,
                           int64_t ny, int64_t nz, int64_t nt) {
    const int64_t dims[4] = {nx, ny, nz, nt};
    const int64_t F = nx * ny * nz, V = F * nt;
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < V; ++s) {
        REAL fw[4][6], bw[4][6];
        const int64_t t = s / F, s3 = s % F;
        for (int mu = 0; mu < 4; ++mu) {
            int64_t up = FN(nbr)(s, mu, +1, dims), dn = FN(nbr)(s, mu, -1, dims);
            const REAL *vu = (mu == 3 && t == nt - 1) ? v_hi + s3 * 6 : v + up * 6;
            FN(mat_vec)(U + (s * 4 + mu) * 18, vu, fw[mu]);
            if (mu == 3 && t == 0) {
                for (int k = 0; k < 6; ++k) bw[mu][k] = w_lo[s3 * 6 + k];
            } else {
                FN(adj_mat_vec)(U + (dn * 4 + mu) * 18, v + dn * 6, bw[mu]);
            }
        }
        for (int k = 0; k < 6; ++k) {
            REAL f = ((fw[0][k] + fw[1][k]) + fw[2][k]) + fw[3][k];
            out[s * 6 + k] = (((f - bw[0][k]) - bw[1][k]) - bw[2][k]) - bw[3][k];
        }
    }
    return 0;
}

/* link product: acc = smadd(acc, na(nn(U_mu(x), U_nu(x+mu)), U_mu(x+nu)), s) */
int FN(su3o_link_product)(const REAL *U, REAL *acc, int64_t nx, int64_t ny, int64_t nz, int64_t nt, REAL s) {
    static const int pairs[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    const int64_t dims[4] = {nx, ny, nz, nt};
    const int64_t V = nx * ny * nz * nt;
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < V; ++x) {
        REAL a[18], t[18], p[18];
        for (int k = 0; k < 18; ++k) a[k] = 0;
        for (int q = 0; q < 6; ++q) {
            int mu = pairs[q][0], nu = pairs[q][1];
            int64_t xmu = FN(nbr)(x, mu, +1, dims), xnu = FN(nbr)(x, nu, +1, dims);
            FN(mat_mat)(U + (x * 4 + mu) * 18, U + (xmu * 4 + nu) * 18, t, 0);
            FN(mat_mat)(t, U + (xnu * 4 + mu) * 18, p, 1);
            for (int k = 0; k < 18; ++k) a[k] = a[k] + s * p[k];
        }
        for (int k = 0; k < 18; ++k) acc[x * 18 + k] = a[k];
    }
    return 0;
}

#undef FN
#undef CAT
#undef CAT_
#undef M_RE
#undef M_IM
#undef V_RE
#undef V_IM
