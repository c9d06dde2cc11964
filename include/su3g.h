/* libsu3g -- B200 (sm_100a) SU(3) lattice hot path, C ABI.
 *
 * Drop-in boundary for the per-site routines of the reference package su3bench
 * (arXiv 1309.0551; /root/reference/pkg/src/su3bench).  The reference exposes
 * them as Python functions fn(a, b, out=None) on site-major (re, im) pair arrays
 * (simd.py:80-230) behind the plugin registry Backend(kind, apply, batch_apply,
 * kernels) (backends.py:11-31).  Each entry point below replaces one of those
 * kernels for a batch of `nsites` independent operand sets; the Python layer
 * (paper_1309_0551_b200.kernels / .backends) restores the reference signatures.
 *
 * Conventions
 *   - Pointers are DEVICE pointers.  Per-site routine operands are dense in the
 *     reference AoS order: matrix (3,3,2), vector (3,2), mat4 (4,3,3,2), vec4
 *     (4,3,2) per site, sites contiguous (types.py:1-13, OPERAND_SHAPES).
 *   - Work is enqueued on `stream` (a cudaStream_t) and the call returns after
 *     enqueue.  No allocation, no host synchronisation.
 *   - Arithmetic follows the reference association (separated sums, combine
 *     once, no FMA; scalar.py:8-14), so results are bit-identical to su3bench.
 *   - Return value: 0 = ok, SU3G_EINVAL = invalid argument, SU3G_ENCCL = an
 *     NCCL failure, >0 = a cudaError_t.  su3g_last_error() returns the calling
 *     thread's message.
 *   - Result storage must not alias an input (the reference's contract,
 *     validation.py:25-34); it is the caller's responsibility, as there.
 */
#ifndef SU3G_H
#define SU3G_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SU3G_API __attribute__((visibility("default")))
#else
#define SU3G_API
#endif

typedef struct CUstream_st *su3g_stream_t; /* == cudaStream_t */

#define SU3G_OK 0
#define SU3G_EINVAL (-1)
#define SU3G_ENCCL (-2) /* an NCCL call failed (message in su3g_last_error) */

#define SU3G_ABI_VERSION 1

/* link-product arithmetic: exact reference association, or FMA chains */
#define SU3G_EXACT 0
#define SU3G_FMA 1

SU3G_API int su3g_abi_version(void);
SU3G_API const char *su3g_last_error(void);
/* name (and geometry) of the kernel the calling thread's last launch dispatched to, e.g.
 * "k_nn_tma<f32,64x2x2,256thr>" -- the sweeps choose among several kernels at run time */
SU3G_API const char *su3g_last_kernel(void);
/* number of SMs / L2 bytes of the current device (0 on failure) */
SU3G_API int su3g_device_sm_count(void);
SU3G_API int64_t su3g_device_l2_bytes(void);
/* The work-item schedule of the persistent t-walks (ring NN sweep, checkerboarded dslash, link walks) for
 * `nblocks` blocks x `nslices` t-slices on `ctas` resident CTAs (host arithmetic, no device needed; for tests
 * and diagnostics).  Returns the item count (-1 on bad arguments); n_full = leading whole-column items and
 * chunk = t-chunk length of the others (either may be null); when 0 <= item < count, also that item's block
 * and slice range [t0, t1).  prologue_x10: an item's start-up cost in tenths of a step; columns: 0 forces the
 * uniform chunk-major schedule. */
SU3G_API int64_t su3g_walk_schedule(int64_t nblocks, int32_t nslices, int32_t ctas, int32_t prologue_x10,
                                    int32_t columns, int64_t item, int64_t *blk, int32_t *t0, int32_t *t1,
                                    int64_t *n_full, int32_t *chunk);
/* process-wide tuning/debug knobs (not needed for normal use):
 *   "nn_variant":   0 auto, 1 generic one-thread-per-site (z-chunked order), 3 TMA t-walk,
 *                   4 TMA ring walk (the default where it applies: nx in {32, 48, 64}, even ny, nz)
 *   "nn_ring_cfg":  f32 ring-walk slot / CTA configuration for A/B (0 = default)
 *   "link_variant": 0 auto, 1 rows gather, 3 row-split carried t-walk, 5 factored two-lane pair walk (FMA mode,
 *                   nine products per site; the FMA default)
 *   "nn_ring_columns": 0 / 1: the ring walks' (NN sweep, checkerboarded dslash) columns schedule: whole t-columns
 *                   for full rounds of blocks, t-chunks for the rest (default 1)
 *   "link_chunk":   t-chunk length of the link walks' work items (0 = auto: the columns schedule)
 *   "dslash_eo_variant": 0 auto, 1 gather kernel, 2 half-lattice ring walk (nx in {32, 64}, even ny, nz)
 *   "dslash_eo_ring_cfg": slot / CTA configuration of that ring walk for A/B (0 = default)
 *   "nn_tma_chunk": t-chunk length of the TMA walk's work items (0 = auto, balances the wave)
 *   "nn_tma_threads": 0 auto, 128 or 256 threads per TMA-walk CTA
 *   "chunk_prologue_x10": relative cost of a work-item prologue, in tenths of a step (chunk picker)
 *   "sweep_zc":     z-planes per visiting chunk of the one-thread-per-site NN sweep and dslash kernels
 *                   (largest divisor of nz <= value; 0 = auto: 8 when a t-slice exceeds half of L2)
 *   "sweep_l2_hints": 1 (default) = the one-thread-per-site NN / dslash kernels load backward
 *                   (last-use) links and v(t-1) evict-first in L2 and store their output streaming
 *   "nn_tma_l2_hints": 1 (default) = the TMA NN kernel gathers U_t evict-first and stores streaming
 *   "dslash_eo_zc", "dslash_eo_hints": the same two knobs for the checkerboarded dslash
 *   "sm_reserve":   SMs the persistent sweep kernels leave free for concurrent kernels
 *                   (NCCL halo exchange of a t-slab sweep); default 0 */
SU3G_API int su3g_set_option(const char *name, int64_t value);

/* ---- per-site routines (8 hot routines x {f32, f64}) ---------------------
 * c = routine(a, b) for every site.                                            */

/* replaces su3bench.simd.mult_su3_mat_vec (simd.py:80-91; scalar.py:49-60) */
SU3G_API int su3g_mult_su3_mat_vec_f32(const float *a, const float *b, float *c, int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_mult_su3_mat_vec_f64(const double *a, const double *b, double *c, int64_t nsites, su3g_stream_t stream);
/* replaces su3bench.simd.mult_adj_su3_mat_vec (simd.py:94-105; scalar.py:63-74) */
SU3G_API int su3g_mult_adj_su3_mat_vec_f32(const float *a, const float *b, float *c, int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_mult_adj_su3_mat_vec_f64(const double *a, const double *b, double *c, int64_t nsites, su3g_stream_t stream);
/* replaces su3bench.simd.mult_su3_nn (simd.py:108-119; scalar.py:77-89) */
SU3G_API int su3g_mult_su3_nn_f32(const float *a, const float *b, float *c, int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_mult_su3_nn_f64(const double *a, const double *b, double *c, int64_t nsites, su3g_stream_t stream);
/* replaces su3bench.simd.mult_su3_na (simd.py:136-149; scalar.py:92-104) */
SU3G_API int su3g_mult_su3_na_f32(const float *a, const float *b, float *c, int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_mult_su3_na_f64(const double *a, const double *b, double *c, int64_t nsites, su3g_stream_t stream);
/* replaces su3bench.simd.mult_su3_an (simd.py:122-133; scalar.py:107-119) */
SU3G_API int su3g_mult_su3_an_f32(const float *a, const float *b, float *c, int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_mult_su3_an_f64(const double *a, const double *b, double *c, int64_t nsites, su3g_stream_t stream);
/* replaces su3bench.simd.mult_adj_su3_mat_vec_4dir (simd.py:172-179; scalar.py:140-146)
 * a4: mat4 per site, b: vec per site, c: vec4 per site */
SU3G_API int su3g_mult_adj_su3_mat_vec_4dir_f32(const float *a4, const float *b, float *c4, int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_mult_adj_su3_mat_vec_4dir_f64(const double *a4, const double *b, double *c4, int64_t nsites, su3g_stream_t stream);
/* replaces su3bench.simd.mult_su3_mat_vec_sum_4dir (simd.py:197-214; scalar.py:168-194)
 * c = sum_d adj(a4[d]) b4[d]  -- the ADJOINT form the reference code implements */
SU3G_API int su3g_mult_su3_mat_vec_sum_4dir_f32(const float *a4, const float *b4, float *c, int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_mult_su3_mat_vec_sum_4dir_f64(const double *a4, const double *b4, double *c, int64_t nsites, su3g_stream_t stream);
/* replaces su3bench.simd.scalar_mult_add_su3_matrix (simd.py:224-230; scalar.py:197-205)
 * c = a + s*b; s_per_site (nsites reals) overrides s when non-NULL (simd.py:217-221) */
SU3G_API int su3g_scalar_mult_add_su3_matrix_f32(const float *a, const float *b, float s, const float *s_per_site, float *c,
                                        int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_scalar_mult_add_su3_matrix_f64(const double *a, const double *b, double s, const double *s_per_site,
                                        double *c, int64_t nsites, su3g_stream_t stream);

/* ---- the other seven Table-1 routines -----------------
 * Same conventions as above: AoS records, device pointers, nsites objects. */
/* replaces su3bench.simd.add_su3_vector (simd.py:71-77; scalar.py:39-46): c = a + b */
SU3G_API int su3g_add_su3_vector_f32(const float *a, const float *b, float *c, int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_add_su3_vector_f64(const double *a, const double *b, double *c, int64_t nsites, su3g_stream_t stream);
/* replaces su3bench.simd.mult_su3_mat_hwvec (simd.py:152-159; scalar.py:122-128)
 * h, c: half-Wilson vectors (2,3,2) per site; c[k] = a h[k] */
SU3G_API int su3g_mult_su3_mat_hwvec_f32(const float *a, const float *h, float *c, int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_mult_su3_mat_hwvec_f64(const double *a, const double *h, double *c, int64_t nsites, su3g_stream_t stream);
/* replaces su3bench.simd.mult_adj_su3_mat_hwvec (simd.py:162-169; scalar.py:131-137): c[k] = adj(a) h[k] */
SU3G_API int su3g_mult_adj_su3_mat_hwvec_f32(const float *a, const float *h, float *c, int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_mult_adj_su3_mat_hwvec_f64(const double *a, const double *h, double *c, int64_t nsites,
                                             su3g_stream_t stream);
/* replaces su3bench.simd.mult_adj_su3_mat_4vec with `outs` (simd.py:182-194; scalar.py:149-165):
 * c_d = adj(a4[d]) b written to four separate (nsites,3,2) destinations c0..c3.
 * (The packed form, outs omitted, is su3g_mult_adj_su3_mat_vec_4dir.) */
SU3G_API int su3g_mult_adj_su3_mat_4vec_f32(const float *a4, const float *b, float *c0, float *c1, float *c2, float *c3,
                                            int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_mult_adj_su3_mat_4vec_f64(const double *a4, const double *b, double *c0, double *c1, double *c2,
                                            double *c3, int64_t nsites, su3g_stream_t stream);
/* replaces su3bench.simd.scalar_mult_add_su3_vector (simd.py:233-239; scalar.py:208-215)
 * c = a + s*b; s_per_site (nsites reals) overrides s when non-NULL */
SU3G_API int su3g_scalar_mult_add_su3_vector_f32(const float *a, const float *b, float s, const float *s_per_site, float *c,
                                                 int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_scalar_mult_add_su3_vector_f64(const double *a, const double *b, double s, const double *s_per_site,
                                                 double *c, int64_t nsites, su3g_stream_t stream);
/* replaces su3bench.simd.su3_projector (simd.py:242-251; scalar.py:218-230): c[i][j] = a[i] conj(b[j]), c a matrix */
SU3G_API int su3g_su3_projector_f32(const float *a, const float *b, float *c, int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_su3_projector_f64(const double *a, const double *b, double *c, int64_t nsites, su3g_stream_t stream);
/* replaces su3bench.simd.sub_four_su3_vecs (simd.py:254-259; scalar.py:233-238)
 * a <- ((((a - b1) - b2) - b3) - b4), IN PLACE on a */
SU3G_API int su3g_sub_four_su3_vecs_f32(float *a, const float *b1, const float *b2, const float *b3, const float *b4,
                                        int64_t nsites, su3g_stream_t stream);
SU3G_API int su3g_sub_four_su3_vecs_f64(double *a, const double *b1, const double *b2, const double *b3,
                                        const double *b4, int64_t nsites, su3g_stream_t stream);

/* ---- seeded fill ---------------------------------------
 * replaces su3bench.lattice.SiteBuffer.randomize (lattice.py:192-197), i.e. numpy
 * Generator.uniform(low, high) on the default PCG64 bit generator, written straight
 * into device memory: out[i] = draw (skip + i) of the stream whose 128-bit state and
 * increment are (state_hi:state_lo, inc_hi:inc_lo) as numpy's
 * bit_generator.state reports them.  Bit-identical to numpy (f32: the float64 draw
 * rounded to nearest, as numpy's assignment into a float32 array). */
SU3G_API int su3g_uniform_fill_f32(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t skip,
                                   double low, double high, float *out, int64_t n, su3g_stream_t stream);
SU3G_API int su3g_uniform_fill_f64(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t skip,
                                   double low, double high, double *out, int64_t n, su3g_stream_t stream);

/* ---- layout transforms ---------------------------------------------------
 * AoS (reference site-major, `reals_per_site` reals per site, sites x-fastest;
 * lattice.py:155-187 SiteBuffer) <-> GPU-internal t-sliced SoA:
 *     soa[(t * reals_per_site + c) * sites_per_slice + s3]
 * where a slice is one fixed-t block of sites_per_slice = nx*ny*nz sites (a
 * t-face is contiguous in the reference numbering, lattice.py:3-6).
 * nslices = 1 gives plain SoA.  reals_per_site in {2, 6, 12, 18, 24, 72}.                        */
SU3G_API int su3g_aos_to_soa_f32(const float *aos, float *soa, int64_t sites_per_slice, int64_t nslices, int32_t reals_per_site,
                        su3g_stream_t stream);
SU3G_API int su3g_aos_to_soa_f64(const double *aos, double *soa, int64_t sites_per_slice, int64_t nslices,
                        int32_t reals_per_site, su3g_stream_t stream);
SU3G_API int su3g_soa_to_aos_f32(const float *soa, float *aos, int64_t sites_per_slice, int64_t nslices, int32_t reals_per_site,
                        su3g_stream_t stream);
SU3G_API int su3g_soa_to_aos_f64(const double *soa, double *aos, int64_t sites_per_slice, int64_t nslices,
                        int32_t reals_per_site, su3g_stream_t stream);

/* ---- periodic nearest-neighbour sweep (BASELINE configs[2], configs[4]) ----
 *   out(x) = sum_mu U_mu(x) v(x+mu) - sum_mu U_mu(x-mu)^dag v(x-mu)
 * in the association of the composed reference oracle:
 *   ((((fw0+fw1)+fw2)+fw3) - bw0 - bw1 - bw2 - bw3), fw = mult_su3_mat_vec,
 *   bw = mult_adj_su3_mat_vec.
 * Fields are t-sliced SoA on a local lattice nx*ny*nz*nt: U has 72 reals per
 * site (mu-major, 18 each), v/out 6.  x, y, z are periodic.  Along t:
 *   v_hi (6*F reals, SoA face) = v on the slice after the last local one, or
 *        NULL -> periodic (slice 0);
 *   w_lo (6*F reals)           = U_t(x)^dag v(x) on the slice before slice 0
 *        (computed by its owner with su3g_nn_halo_w), or NULL -> periodic.
 * Only slices t in [t_begin, t_end) of `out` are written (interior/boundary
 * split for overlapping a halo exchange).
 * mode SU3G_EXACT: reference association, bit-identical to the composed
 * reference; SU3G_FMA: FMA chains in the products (north-star tolerance).
 * Use the same mode for su3g_nn_halo_w so a sharded sweep stays bit-identical
 * to the single-GPU one.                                                    */
SU3G_API int su3g_nn_sweep_f32(const float *U, const float *v, float *out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                      int32_t t_begin, int32_t t_end, const float *v_hi, const float *w_lo, int32_t mode,
                      su3g_stream_t stream);
SU3G_API int su3g_nn_sweep_f64(const double *U, const double *v, double *out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                      int32_t t_begin, int32_t t_end, const double *v_hi, const double *w_lo, int32_t mode,
                      su3g_stream_t stream);
/* w_face = U_t(x)^dag v(x) on the LAST local t-slice (the halo a t-slab sends
 * to its +t neighbour; 6*F reals, SoA face) */
SU3G_API int su3g_nn_halo_w_f32(const float *U, const float *v, float *w_face, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                       int32_t mode, su3g_stream_t stream);
SU3G_API int su3g_nn_halo_w_f64(const double *U, const double *v, double *w_face, int32_t nx, int32_t ny, int32_t nz,
                       int32_t nt, int32_t mode, su3g_stream_t stream);

/* The two boundary slices t = 0 and t = nt-1 of a t-slab application in one launch (same values
 * as su3g_nn_sweep on those slices, with the same v_hi / w_lo halos).  w_next (6*F reals, SoA
 * face, may be NULL) receives U_t^dag out on slice nt-1: the halo the next application sends to
 * rank r+1, identical to su3g_nn_halo_w(U, out) -- the t-slab drivers skip that pack kernel. */
SU3G_API int su3g_nn_sweep_edges_f32(const float *U, const float *v, float *out, int32_t nx, int32_t ny, int32_t nz,
                                     int32_t nt, const float *v_hi, const float *w_lo, float *w_next, int32_t mode,
                                     su3g_stream_t stream);
SU3G_API int su3g_nn_sweep_edges_f64(const double *U, const double *v, double *out, int32_t nx, int32_t ny, int32_t nz,
                                     int32_t nt, const double *v_hi, const double *w_lo, double *w_next, int32_t mode,
                                     su3g_stream_t stream);

/* ---- even/odd dslash -----------------------------------
 * out(x) = sum_mu U_mu(x) v(x+mu) - sum_mu U_mu(x-mu)^dag v(x-mu) for the sites of one
 * parity, (x+y+z+t) % 2 == parity, only; those read v on the other parity only.  Fused:
 * forward mat_vec x4, backward adjoint products of the neighbours (adj_4dir), the
 * add_su3_vector chain and sub_four_su3_vecs, in the NN sweep's association, so the
 * values equal su3g_nn_sweep's on those sites bit for bit (EXACT).  Sites of the other
 * parity in `out` are left untouched.  Every extent must be even; periodic lattice.
 * U: t-sliced SoA, 72 reals/site; v, out: t-sliced SoA, 6 reals/site (full lattice). */
SU3G_API int su3g_dslash_f32(const float *U, const float *v, float *out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                             int32_t parity, int32_t mode, su3g_stream_t stream);
SU3G_API int su3g_dslash_f64(const double *U, const double *v, double *out, int32_t nx, int32_t ny, int32_t nz,
                             int32_t nt, int32_t parity, int32_t mode, su3g_stream_t stream);
/* the same with a caller-provided workspace `scratch` (a full v-sized SoA field, not aliasing v or
 * out): for f32 lattices the TMA t-walk computes the whole sweep into scratch and the parity is
 * copied out -- identical values, faster than the parity kernel at 64^3x16.  NULL scratch, f64 or
 * lattices without a TMA geometry use the one-thread-per-site parity kernel. */
SU3G_API int su3g_dslash_ws_f32(const float *U, const float *v, float *out, float *scratch, int32_t nx, int32_t ny,
                                int32_t nz, int32_t nt, int32_t parity, int32_t mode, su3g_stream_t stream);
SU3G_API int su3g_dslash_ws_f64(const double *U, const double *v, double *out, double *scratch, int32_t nx, int32_t ny,
                                int32_t nz, int32_t nt, int32_t parity, int32_t mode, su3g_stream_t stream);

/* ---- checkerboarded ("eo") fields and the dslash on them ----
 * eo layout: each t-slice keeps the sites of one parity as a contiguous half,
 *     eo[(t*C + c)*F + q*F/2 + h],  q = (x+y+z+t) & 1,  h = (x>>1) + (nx/2)*(y + ny*z),
 * F = nx*ny*nz; every extent even.  su3g_soa_to_eo / su3g_eo_to_soa permute a t-sliced SoA field
 * of C reals per site (src and dst must not alias).  su3g_dslash_eo computes, for the sites of
 * one parity, the same values as su3g_dslash (bitwise in EXACT mode) from eo fields: it reads
 * v's other-parity half and writes out's `parity` half only; whole sectors, no half-used lines. */
SU3G_API int su3g_soa_to_eo_f32(const float *soa, float *eo, int32_t nx, int32_t ny, int32_t nz, int32_t nt, int32_t reals_per_site,
                                su3g_stream_t stream);
SU3G_API int su3g_soa_to_eo_f64(const double *soa, double *eo, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                                int32_t reals_per_site, su3g_stream_t stream);
SU3G_API int su3g_eo_to_soa_f32(const float *eo, float *soa, int32_t nx, int32_t ny, int32_t nz, int32_t nt, int32_t reals_per_site,
                                su3g_stream_t stream);
SU3G_API int su3g_eo_to_soa_f64(const double *eo, double *soa, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                                int32_t reals_per_site, su3g_stream_t stream);
SU3G_API int su3g_dslash_eo_f32(const float *U, const float *v, float *out, int32_t nx, int32_t ny, int32_t nz, int32_t nt,
                                int32_t parity, int32_t mode, su3g_stream_t stream);
SU3G_API int su3g_dslash_eo_f64(const double *U, const double *v, double *out, int32_t nx, int32_t ny, int32_t nz,
                                int32_t nt, int32_t parity, int32_t mode, su3g_stream_t stream);

/* ---- t-slab multi-GPU NN sweep over NCCL (BASELINE configs[4]) ----
 * One process (or thread) per GPU.  Rank r of G holds the t-slices
 * [r*nt_local, (r+1)*nt_local) of the global lattice; U, v, out are its slab in the
 * t-sliced SoA layout of su3g_nn_sweep.  su3g_slab_nn_sweep computes out = D v on the
 * slab, exchanging the two one-site halos with ranks r-1 and r+1 (v on the first local
 * slice, w = U_t^dag v on the last) over NCCL on the communicator's own stream while the
 * interior slices run on `stream`; bit-identical to the unsharded periodic sweep.  A
 * one-rank communicator exchanges with itself (periodic in t).
 * NCCL is loaded at su3g_comm_init (dlopen "libnccl.so.2" or $SU3G_NCCL_LIB).
 * The unique id (SU3G_COMM_ID_BYTES bytes, an ncclUniqueId) is created by one rank with
 * su3g_comm_unique_id and distributed by the host program.  su3g_comm_init is collective
 * and must be called with the rank's device current. */
#define SU3G_COMM_ID_BYTES 128
typedef struct su3g_comm *su3g_comm_t;
SU3G_API int su3g_comm_unique_id(void *id_out);
SU3G_API int su3g_comm_init(int32_t nranks, int32_t rank, const void *id, su3g_comm_t *comm);
SU3G_API int su3g_comm_destroy(su3g_comm_t comm);
SU3G_API int su3g_comm_rank(su3g_comm_t comm, int32_t *rank, int32_t *nranks);
/* Failure detection: waits (host side) for the last enqueued halo exchange, polling NCCL's
 * asynchronous error state (ncclCommGetAsyncError).  On an NCCL error, or when the exchange is
 * still pending after timeout_ms (< 0: no deadline) -- a dead or stalled peer -- the communicator
 * is aborted (ncclCommAbort, so no kernel is left spinning) and SU3G_ENCCL is returned; the
 * handle must then only be destroyed.  su3g_slab_nn_sweep_* also refuses a communicator that is
 * already in an asynchronous error state. */
SU3G_API int su3g_comm_check(su3g_comm_t comm, int64_t timeout_ms);
SU3G_API int su3g_slab_nn_sweep_f32(su3g_comm_t comm, const float *U, const float *v, float *out, int32_t nx,
                                    int32_t ny, int32_t nz, int32_t nt_local, int32_t mode, su3g_stream_t stream);
SU3G_API int su3g_slab_nn_sweep_f64(su3g_comm_t comm, const double *U, const double *v, double *out, int32_t nx,
                                    int32_t ny, int32_t nz, int32_t nt_local, int32_t mode, su3g_stream_t stream);

/* ---- fused compute + halo push over NVLink (t-slab NN sweep) ------------
 * The boundary kernel of application e computes the slab's slices t = 0 and t = nt-1 and
 * stores the NEXT application's halos straight into the neighbours' windows (rank r-1 gets
 * out(t=0) as its v_hi, rank r+1 gets U_t^dag out(nt-1) as its w_lo), then releases a
 * system-scope flag; the interior slices follow on the same stream while the peers' pushes
 * land.  No NCCL kernel, no host round trip, bit-identical to the periodic sweep.
 * Window: one device buffer per rank of su3g_p2p_window_bytes() bytes, zero-initialised
 * (halo faces x 2 parities + flags); every rank maps its neighbours' windows with CUDA IPC
 * (su3g_ipc_get_handle / su3g_ipc_open_handle; with one rank, pass the own window as both
 * peers).  win_lo = window of rank r-1, win_hi = window of rank r+1.
 * Epochs: su3g_p2p_prime(e) pushes the halos of a fresh source v for application e (call it
 * after all ranks' previous launches completed, with e greater than every epoch used so far);
 * su3g_p2p_nn_sweep(e) then computes out = D v for application e and primes e+1 from out, so
 * ping-pong applications e, e+1, e+2, ... need no further priming.  Waits are bounded
 * (~20 s): a timed-out wait sets the error word at su3g_p2p_ctrl_offset() + 20. */
SU3G_API int64_t su3g_p2p_window_bytes(int32_t nx, int32_t ny, int32_t nz, int32_t elem_size);
SU3G_API int64_t su3g_p2p_ctrl_offset(int32_t nx, int32_t ny, int32_t nz, int32_t elem_size);
#define SU3G_IPC_HANDLE_BYTES 64
SU3G_API int su3g_ipc_get_handle(const void *dev_ptr, void *handle_out);
SU3G_API int su3g_ipc_open_handle(const void *handle, void **dev_ptr_out);
SU3G_API int su3g_ipc_close(void *dev_ptr);
SU3G_API int su3g_p2p_prime_f32(const float *U, const float *v, int32_t nx, int32_t ny, int32_t nz, int32_t nt_local,
                                void *win, void *win_lo, void *win_hi, int64_t epoch, int32_t mode, su3g_stream_t stream);
SU3G_API int su3g_p2p_prime_f64(const double *U, const double *v, int32_t nx, int32_t ny, int32_t nz, int32_t nt_local,
                                void *win, void *win_lo, void *win_hi, int64_t epoch, int32_t mode, su3g_stream_t stream);
SU3G_API int su3g_p2p_nn_sweep_f32(const float *U, const float *v, float *out, int32_t nx, int32_t ny, int32_t nz,
                                   int32_t nt_local, void *win, void *win_lo, void *win_hi, int64_t epoch, int32_t mode,
                                   su3g_stream_t stream);
SU3G_API int su3g_p2p_nn_sweep_f64(const double *U, const double *v, double *out, int32_t nx, int32_t ny, int32_t nz,
                                   int32_t nt_local, void *win, void *win_lo, void *win_hi, int64_t epoch, int32_t mode,
                                   su3g_stream_t stream);

/* ---- link-product sweep (BASELINE configs[3]) ------------------------------
 * acc(x) = sum over (mu,nu) in (0,1),(0,2),(0,3),(1,2),(1,3),(2,3) of
 *          s * U_mu(x) U_nu(x+mu) U_mu(x+nu)^dag, accumulated in that order
 *          via mult_su3_nn -> mult_su3_na -> scalar_mult_add_su3_matrix,
 *          starting from acc = 0; periodic lattice.
 * U: t-sliced SoA, 72 reals/site; acc: t-sliced SoA, 18 reals/site.
 * mode SU3G_EXACT = reference association (bitwise), SU3G_FMA = FMA chains.  */
SU3G_API int su3g_link_product_f32(const float *U, float *acc, int32_t nx, int32_t ny, int32_t nz, int32_t nt, float s,
                          int32_t mode, su3g_stream_t stream);
SU3G_API int su3g_link_product_f64(const double *U, double *acc, int32_t nx, int32_t ny, int32_t nz, int32_t nt, double s,
                          int32_t mode, su3g_stream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* SU3G_H */
