/* A plain-C host program against the libsu3g C ABI (include/su3g.h): proves the
 * header is valid C and that the boundary is usable without Python or torch.
 *
 *   cc -std=c11 -I include tests/c/abi_demo.c -L paper_1309_0551_b200/lib -lsu3g \
 *      -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,...
 *   ./abi_demo          # CPU-only checks: ABI version, argument validation, window sizes
 *   ./abi_demo gpu      # + mult_su3_mat_vec on device memory: identity links return v,
 *                         and an NN sweep of a constant field with identity links is 0
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "su3g.h"

static int failures = 0;
#define CHECK(cond)                                                               \
    do {                                                                          \
        if (!(cond)) {                                                            \
            fprintf(stderr, "FAIL %s:%d: %s (%s)\n", __FILE__, __LINE__, #cond,   \
                    su3g_last_error());                                           \
            ++failures;                                                           \
        }                                                                         \
    } while (0)

static void cpu_checks(void) {
    CHECK(su3g_abi_version() == SU3G_ABI_VERSION);
    CHECK(su3g_mult_su3_mat_vec_f32(NULL, NULL, NULL, -1, NULL) == SU3G_EINVAL);
    CHECK(strstr(su3g_last_error(), "negative") != NULL);
    CHECK(su3g_mult_su3_nn_f64(NULL, NULL, NULL, 0, NULL) == SU3G_OK); /* zero sites: no-op */
    CHECK(su3g_nn_sweep_f32(NULL, NULL, NULL, 0, 4, 4, 4, 0, 4, NULL, NULL, SU3G_EXACT, NULL) == SU3G_EINVAL);
    CHECK(su3g_set_option("no_such_option", 1) == SU3G_EINVAL);
    CHECK(su3g_p2p_window_bytes(64, 64, 64, 4) == 4LL * 6 * 64 * 64 * 64 * 4 + 128);
    CHECK(su3g_comm_destroy(NULL) == SU3G_OK);
    char uid[SU3G_COMM_ID_BYTES];
    su3g_comm_t comm = NULL;
    memset(uid, 0, sizeof(uid));
    CHECK(su3g_comm_init(1, 3, uid, &comm) == SU3G_EINVAL && comm == NULL);
}

static void gpu_checks(void) {
    enum { N = 1000 };
    float *hU = malloc(sizeof(float) * N * 18), *hv = malloc(sizeof(float) * N * 6), *hc = malloc(sizeof(float) * N * 6);
    for (int s = 0; s < N; ++s) {
        for (int k = 0; k < 18; ++k) hU[s * 18 + k] = 0.0f;
        for (int i = 0; i < 3; ++i) hU[s * 18 + (3 * i + i) * 2] = 1.0f; /* identity matrix */
        for (int k = 0; k < 6; ++k) hv[s * 6 + k] = (float)(s % 97) - 0.25f * (float)k;
    }
    float *dU, *dv, *dc;
    CHECK(cudaMalloc((void **)&dU, sizeof(float) * N * 18) == cudaSuccess);
    CHECK(cudaMalloc((void **)&dv, sizeof(float) * N * 6) == cudaSuccess);
    CHECK(cudaMalloc((void **)&dc, sizeof(float) * N * 6) == cudaSuccess);
    cudaMemcpy(dU, hU, sizeof(float) * N * 18, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, hv, sizeof(float) * N * 6, cudaMemcpyHostToDevice);
    CHECK(su3g_mult_su3_mat_vec_f32(dU, dv, dc, N, NULL) == SU3G_OK);
    cudaMemcpy(hc, dc, sizeof(float) * N * 6, cudaMemcpyDeviceToHost);
    CHECK(memcmp(hc, hv, sizeof(float) * N * 6) == 0); /* 1*v + 0*... is exact */
    printf("dispatched: %s\n", su3g_last_kernel());

    /* NN sweep on a 4^4 lattice, identity links, constant v: forward sum 4v minus backward 4v = 0 */
    enum { V = 256 };
    float *hL = calloc((size_t)V * 72, sizeof(float)), *hs = malloc(sizeof(float) * V * 6), *ho = malloc(sizeof(float) * V * 6);
    for (int s = 0; s < V; ++s) /* SoA: component c of site s at c*V + s (one t-slice block per t) */
        for (int mu = 0; mu < 4; ++mu)
            for (int i = 0; i < 3; ++i) {
                const int t = s / 64, s3 = s % 64;
                hL[(size_t)(t * 72 + mu * 18 + (3 * i + i) * 2) * 64 + s3] = 1.0f;
            }
    for (int k = 0; k < V * 6; ++k) hs[k] = 0.5f;
    float *dL, *ds, *dout;
    cudaMalloc((void **)&dL, sizeof(float) * V * 72);
    cudaMalloc((void **)&ds, sizeof(float) * V * 6);
    cudaMalloc((void **)&dout, sizeof(float) * V * 6);
    cudaMemcpy(dL, hL, sizeof(float) * V * 72, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, hs, sizeof(float) * V * 6, cudaMemcpyHostToDevice);
    CHECK(su3g_nn_sweep_f32(dL, ds, dout, 4, 4, 4, 4, 0, 4, NULL, NULL, SU3G_EXACT, NULL) == SU3G_OK);
    cudaMemcpy(ho, dout, sizeof(float) * V * 6, cudaMemcpyDeviceToHost);
    for (int k = 0; k < V * 6; ++k) CHECK(ho[k] == 0.0f);

    /* the same operator on checkerboarded fields: permute to eo, dslash both parities, permute back */
    float *dLe, *dse, *doe, *dback;
    cudaMalloc((void **)&dLe, sizeof(float) * V * 72);
    cudaMalloc((void **)&dse, sizeof(float) * V * 6);
    cudaMalloc((void **)&doe, sizeof(float) * V * 6);
    cudaMalloc((void **)&dback, sizeof(float) * V * 6);
    cudaMemset(doe, 0xff, sizeof(float) * V * 6); /* NaN: every site must be written by one parity */
    CHECK(su3g_soa_to_eo_f32(dL, dLe, 4, 4, 4, 4, 72, NULL) == SU3G_OK);
    CHECK(su3g_soa_to_eo_f32(ds, dse, 4, 4, 4, 4, 6, NULL) == SU3G_OK);
    CHECK(su3g_dslash_eo_f32(dLe, dse, doe, 4, 4, 4, 4, 0, SU3G_EXACT, NULL) == SU3G_OK);
    CHECK(su3g_dslash_eo_f32(dLe, dse, doe, 4, 4, 4, 4, 1, SU3G_EXACT, NULL) == SU3G_OK);
    CHECK(su3g_eo_to_soa_f32(doe, dback, 4, 4, 4, 4, 6, NULL) == SU3G_OK);
    cudaMemcpy(ho, dback, sizeof(float) * V * 6, cudaMemcpyDeviceToHost);
    for (int k = 0; k < V * 6; ++k) CHECK(ho[k] == 0.0f);
    /* the t-slab boundary launch on a one-slab lattice with zero halos: slice 0 loses its -t term
     * (4v - 3v = 0.5), slice 3 its +t term (3v - 4v = -0.5) */
    float *dz;
    cudaMalloc((void **)&dz, sizeof(float) * 64 * 6);
    cudaMemset(dz, 0, sizeof(float) * 64 * 6);
    CHECK(su3g_nn_sweep_edges_f32(dL, ds, dout, 4, 4, 4, 4, dz, dz, NULL, SU3G_EXACT, NULL) == SU3G_OK);
    cudaMemcpy(ho, dout, sizeof(float) * V * 6, cudaMemcpyDeviceToHost);
    for (int k = 0; k < 64 * 6; ++k) CHECK(ho[k] == 0.5f && ho[3 * 64 * 6 + k] == -0.5f);
    CHECK(cudaDeviceSynchronize() == cudaSuccess);
    cudaFree(dLe); cudaFree(dse); cudaFree(doe); cudaFree(dback); cudaFree(dz);
    cudaFree(dU); cudaFree(dv); cudaFree(dc); cudaFree(dL); cudaFree(ds); cudaFree(dout);
    free(hU); free(hv); free(hc); free(hL); free(hs); free(ho);
}

int main(int argc, char **argv) {
    cpu_checks();
    if (argc > 1 && strcmp(argv[1], "gpu") == 0) gpu_checks();
    if (failures) {
        fprintf(stderr, "%d check(s) failed\n", failures);
        return 1;
    }
    printf("abi_demo: ok (%s)\n", argc > 1 ? argv[1] : "cpu");
    return 0;
}
