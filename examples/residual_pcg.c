/* A C caller of libebs.so with no Python and no torch: generate the level-L unit-square
 * mesh on the device, assemble A_e = K_e + M_e and b_e (f = 1), build a plan, check the
 * device residual bit for bit against a CPU loop in the reference's order (operators.py:
 * 66-107: per element b_e[j] - sum_k A_e[j][k] x[k], scattered by np.bincount over the
 * flat (j, e) index), then solve the Dirichlet problem with Jacobi-PCG.
 *
 *   gcc -O2 -ffp-contract=off -Iinclude -I/usr/local/cuda/include examples/residual_pcg.c \
 *       -Lpaper_1911_03973_b200 -lebs -L/usr/local/cuda/lib64 -lcudart -lm -o residual_pcg
 *   ./residual_pcg [level]          (exit 0 = all checks passed)
 */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ebs.h"

#define EBS(call)                                                                  \
    do {                                                                           \
        int rc_ = (call);                                                          \
        if (rc_ != EBS_OK) {                                                       \
            char msg_[512];                                                        \
            ebs_last_error(msg_, sizeof msg_);                                     \
            fprintf(stderr, "%s -> %d: %s\n", #call, rc_, msg_);                   \
            return 1;                                                              \
        }                                                                          \
    } while (0)
#define CUDA(call)                                                                 \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) {                                                   \
            fprintf(stderr, "%s -> %s\n", #call, cudaGetErrorString(e_));          \
            return 1;                                                              \
        }                                                                          \
    } while (0)

static void *dev(size_t bytes) {
    void *p = NULL;
    return cudaMalloc(&p, bytes ? bytes : 1) == cudaSuccess ? p : NULL;
}

int main(int argc, char **argv) {
    const int level = argc > 1 ? atoi(argv[1]) : 5;
    const int64_t n = ((int64_t)1 << level) + 1, nn = n * n, ne = 2 * (n - 1) * (n - 1);
    double *nodes = dev(sizeof(double) * 2 * nn), *A = dev(sizeof(double) * 9 * ne);
    double *be = dev(sizeof(double) * 3 * ne), *x = dev(sizeof(double) * nn);
    double *r = dev(sizeof(double) * nn), *x0 = dev(sizeof(double) * nn);
    double *u = dev(sizeof(double) * nn);
    int32_t *conn = dev(sizeof(int32_t) * 3 * ne), *bad = dev(sizeof(int32_t));
    int64_t *degenerate = dev(sizeof(int64_t));
    uint8_t *flags = dev(nn);
    if (!nodes || !A || !be || !x || !r || !x0 || !u || !conn || !bad || !degenerate || !flags) {
        fprintf(stderr, "device allocation failed\n");
        return 1;
    }

    /* mesh + element matrices on the device */
    EBS(ebs_mesh_grid2d(n, nodes, conn, NULL));
    EBS(ebs_assemble_p1(2, ne, nodes, conn, 1.0, NULL, 1.0, NULL, NULL, A, be, degenerate, NULL));
    ebs_plan_t plan = NULL;
    EBS(ebs_plan_create(3, nn, ne, conn, NULL, &plan));
    EBS(ebs_plan_load(plan, A, be, NULL));

    /* x: a fixed pseudo-random vector in [-1, 1) */
    double *hx = malloc(sizeof(double) * nn), *hr = malloc(sizeof(double) * nn);
    double *ref = calloc(nn, sizeof(double)), *hA = malloc(sizeof(double) * 9 * ne);
    double *hbe = malloc(sizeof(double) * 3 * ne);
    int32_t *hc = malloc(sizeof(int32_t) * 3 * ne);
    uint64_t state = 0x9E3779B97F4A7C15ull;
    for (int64_t i = 0; i < nn; ++i) {
        state = state * 6364136223846793005ull + 1442695040888963407ull;
        hx[i] = (double)(state >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    }
    CUDA(cudaMemcpy(x, hx, sizeof(double) * nn, cudaMemcpyHostToDevice));
    EBS(ebs_residual(plan, x, r, EBS_RES_EXACT, 0, bad, NULL));
    CUDA(cudaMemcpy(hr, r, sizeof(double) * nn, cudaMemcpyDeviceToHost));

    /* CPU check in the reference's order: flat index j*ne + e ascending */
    CUDA(cudaMemcpy(hA, A, sizeof(double) * 9 * ne, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(hbe, be, sizeof(double) * 3 * ne, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(hc, conn, sizeof(int32_t) * 3 * ne, cudaMemcpyDeviceToHost));
    for (int j = 0; j < 3; ++j)
        for (int64_t e = 0; e < ne; ++e) {
            const double *row = hA + (e * 3 + j) * 3;
            double loc = row[0] * hx[hc[e]];
            loc = loc + row[1] * hx[hc[ne + e]];
            loc = loc + row[2] * hx[hc[2 * ne + e]];
            ref[hc[j * ne + e]] += hbe[j * ne + e] - loc;
        }
    int64_t mismatches = 0;
    for (int64_t i = 0; i < nn; ++i) mismatches += memcmp(&hr[i], &ref[i], sizeof(double)) != 0;
    printf("level %d: %lld nodes, %lld triangles; residual bitwise mismatches: %lld\n", level,
           (long long)nn, (long long)ne, (long long)mismatches);

    /* the same residual on host buffers, 3 times through the pipelined host entry point
     * (x read from one host row: ldx = 0) -- each row bit-identical to the device call */
    double *hr3 = malloc(sizeof(double) * 3 * nn);
    int32_t hbad[3] = {-1, -1, -1};
    EBS(ebs_residual_many_host(plan, hx, 0, hr3, nn, 3, EBS_RES_EXACT, 0, hbad, NULL));
    int64_t host_mismatches = hbad[0] + hbad[1] + hbad[2];
    for (int64_t i = 0; i < 3 * nn; ++i) host_mismatches += memcmp(&hr3[i], &hr[i % nn], sizeof(double)) != 0;
    printf("host-buffer residuals (3 rows): bitwise mismatches vs the device call: %lld\n",
           (long long)host_mismatches);
    free(hr3);

    /* Dirichlet u = 0 on the boundary, Jacobi-PCG to 1e-10 */
    uint8_t *hf = malloc(nn);
    EBS(ebs_mesh_flags(2, nn, nodes, 0, flags, NULL));
    CUDA(cudaMemcpy(hf, flags, nn, cudaMemcpyDeviceToHost));
    int64_t nd_count = 0;
    int64_t *hnd = malloc(sizeof(int64_t) * nn);
    for (int64_t i = 0; i < nn; ++i)
        if (hf[i]) hnd[nd_count++] = i;
    int64_t *nd = dev(sizeof(int64_t) * nd_count);
    CUDA(cudaMemcpy(nd, hnd, sizeof(int64_t) * nd_count, cudaMemcpyHostToDevice));
    EBS(ebs_plan_set_dirichlet(plan, nd, nd_count, NULL));
    CUDA(cudaMemset(x0, 0, sizeof(double) * nn));
    const int iters = 10000;
    double *norms = malloc(sizeof(double) * (iters + 2));
    int n_norms = 0, diverged = 0;
    ebs_solve_params P;
    memset(&P, 0, sizeof P);
    P.method = EBS_PCG;
    P.iters = iters;
    P.has_tol = 1;
    P.tol = 1e-10;
    P.x0 = x0;
    P.x = u;
    P.norms = norms;
    P.n_norms = &n_norms;
    P.diverged = &diverged;
    EBS(ebs_solve(plan, &P, NULL));
    const double rel = norms[n_norms - 1] / norms[0];
    printf("PCG: %d iterations, ||r||/||r0|| = %.3e, diverged = %d, launches so far %lld\n",
           n_norms - 1, rel, diverged, (long long)ebs_launch_count());

    EBS(ebs_plan_destroy(plan));
    const int ok = mismatches == 0 && !diverged && rel <= 1e-10 && n_norms > 1;
    printf("%s\n", ok ? "OK" : "FAILED");
    return ok ? 0 : 2;
}
