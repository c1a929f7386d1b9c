/* The element-slab multi-GPU path through the C-ABI alone (no Python, no torch, no NCCL):
 * the level-L unit-square mesh cut into P element slabs (the reference's chunk rule,
 * operators.py:100), one plan per slab, the peer-memory halo (ebs_peer_*: windows, sweeps
 * that push the interface partials, flag-waiting combines), damped Jacobi (omega = 0.8,
 * u = 0 on the boundary) -- against the single-GPU ebs_solve on the whole mesh.
 *
 * The P ranks are emulated in this one process on one GPU (every window is a local
 * allocation; each phase is issued for all ranks before the next, so nothing waits).  With
 * one process per GPU, rank p would allocate only its own window with
 * ebs_peer_window_alloc(cap, &win, handle), exchange the 64-byte handles and map the others
 * with ebs_peer_window_open -- the kernels and calls below stay the same.
 *
 *   gcc -O2 -std=c11 -Iinclude -I/usr/local/cuda/include examples/slab_jacobi_peer.c \
 *       -Lpaper_1911_03973_b200 -lebs -L/usr/local/cuda/lib64 -lcudart -lm -o slab_jacobi_peer
 *   ./slab_jacobi_peer [level] [P] [iters]          (exit 0 = all checks passed)
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
            exit(1);                                                               \
        }                                                                          \
    } while (0)
#define CUDA(call)                                                                 \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) {                                                   \
            fprintf(stderr, "%s -> %s\n", #call, cudaGetErrorString(e_));          \
            exit(1);                                                               \
        }                                                                          \
    } while (0)

static void *dev(size_t bytes) {
    void *p = NULL;
    CUDA(cudaMalloc(&p, bytes ? bytes : 1));
    return p;
}
static void *up(const void *h, size_t bytes) {
    void *d = dev(bytes);
    if (bytes) CUDA(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice));
    return d;
}

#define PMAX EBS_PEER_MAX

typedef struct {  /* one element slab = one rank */
    int64_t lo, hi, n;          /* elements [lo, hi), local nodes */
    int64_t *glob;              /* host: global id of local node l (ascending) */
    ebs_peer_t peer;
    ebs_plan_t plan;
    int32_t *chunks;            /* device: chunk list, interface chunks first */
    int64_t n_chunks, n_if_chunks;
    int32_t *old_of_new;        /* host: internal -> local */
    uint8_t *iface, *owned, *free_m;   /* device, internal numbering */
    double *b, *dinv, *xa, *xb, *s, *red3, *norm2;
    void *ws;
    int n_nb;                   /* halo: neighbours, shared-node counts, device index lists */
    int32_t nb[PMAX];
    int64_t lens[PMAX];
    const int64_t *idx[PMAX];
} Rank;

int main(int argc, char **argv) {
    const int level = argc > 1 ? atoi(argv[1]) : 6;
    const int P = argc > 2 ? atoi(argv[2]) : 3;
    const int iters = argc > 3 ? atoi(argv[3]) : 50;
    const double omega = 0.8;
    if (P < 1 || P > PMAX || iters < 1) {
        fprintf(stderr, "1 <= P <= %d, iters >= 1\n", PMAX);
        return 1;
    }
    const int64_t n1 = ((int64_t)1 << level) + 1, nn = n1 * n1, ne = 2 * (n1 - 1) * (n1 - 1);

    /* the global mesh on the device, copied to the host for the partition */
    double *nodes = dev(sizeof(double) * 2 * nn);
    int32_t *conn = dev(sizeof(int32_t) * 3 * ne);
    EBS(ebs_mesh_grid2d(n1, nodes, conn, NULL));
    double *hn = malloc(sizeof(double) * 2 * nn);
    int32_t *hc = malloc(sizeof(int32_t) * 3 * ne);
    CUDA(cudaMemcpy(hn, nodes, sizeof(double) * 2 * nn, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(hc, conn, sizeof(int32_t) * 3 * ne, cudaMemcpyDeviceToHost));

    /* ---- single-GPU reference: ebs_solve(EBS_JACOBI) on the whole mesh ---- */
    double *A = dev(sizeof(double) * 9 * ne), *be = dev(sizeof(double) * 3 * ne);
    int64_t *degenerate = dev(sizeof(int64_t));
    EBS(ebs_assemble_p1(2, ne, nodes, conn, 1.0, NULL, 1.0, NULL, NULL, A, be, degenerate, NULL));
    ebs_plan_t gplan = NULL;
    EBS(ebs_plan_create(3, nn, ne, conn, NULL, &gplan));
    EBS(ebs_plan_load(gplan, A, be, NULL));
    uint8_t *flags = dev(nn), *hf = malloc(nn);
    EBS(ebs_mesh_flags(2, nn, nodes, 0, flags, NULL));
    CUDA(cudaMemcpy(hf, flags, nn, cudaMemcpyDeviceToHost));
    int64_t *hnd = malloc(sizeof(int64_t) * nn), nd_count = 0;
    for (int64_t i = 0; i < nn; ++i)
        if (hf[i]) hnd[nd_count++] = i;
    int64_t *nd = up(hnd, sizeof(int64_t) * nd_count);
    EBS(ebs_plan_set_dirichlet(gplan, nd, nd_count, NULL));
    double *x0 = dev(sizeof(double) * nn), *u1 = dev(sizeof(double) * nn);
    CUDA(cudaMemset(x0, 0, sizeof(double) * nn));
    double *norms1 = malloc(sizeof(double) * (iters + 2));
    int n_norms = 0, diverged = 0;
    ebs_solve_params SP;
    memset(&SP, 0, sizeof SP);
    SP.method = EBS_JACOBI;
    SP.iters = iters;
    SP.omega = omega;
    SP.x0 = x0;
    SP.x = u1;
    SP.norms = norms1;
    SP.n_norms = &n_norms;
    SP.diverged = &diverged;
    EBS(ebs_solve(gplan, &SP, NULL));
    double *hu1 = malloc(sizeof(double) * nn);
    CUDA(cudaMemcpy(hu1, u1, sizeof(double) * nn, cudaMemcpyDeviceToHost));

    /* ---- partition: slabs, local node sets, interfaces, owners ---- */
    Rank R[PMAX];
    int32_t *g2l = malloc(sizeof(int32_t) * nn);
    int8_t *owner = malloc(nn);
    uint8_t *mark = malloc(nn);
    memset(owner, -1, nn);
    for (int p = 0; p < P; ++p) {
        Rank *r = &R[p];
        memset(r, 0, sizeof *r);
        r->lo = (int64_t)((double)p * ne / P);   /* np.linspace(0, n_e, P+1, dtype=int) */
        r->hi = (int64_t)((double)(p + 1) * ne / P);
        memset(mark, 0, nn);
        for (int j = 0; j < 3; ++j)
            for (int64_t e = r->lo; e < r->hi; ++e) mark[hc[j * ne + e]] = 1;
        r->glob = malloc(sizeof(int64_t) * nn);
        for (int64_t g = 0; g < nn; ++g)
            if (mark[g]) {
                r->glob[r->n++] = g;
                if (owner[g] < 0) owner[g] = (int8_t)p;  /* lowest rank touching it */
            }
    }
    int64_t cap = 1;
    int64_t *shared[PMAX][PMAX];   /* shared[p][q]: local ids in p of the nodes shared with q */
    int64_t n_shared[PMAX][PMAX];
    for (int p = 0; p < P; ++p) {
        for (int64_t l = 0; l < R[p].n; ++l) g2l[R[p].glob[l]] = (int32_t)l;
        for (int q = 0; q < P; ++q) {
            n_shared[p][q] = 0;
            shared[p][q] = NULL;
            if (q == p) continue;
            memset(mark, 0, nn);
            for (int64_t l = 0; l < R[q].n; ++l) mark[R[q].glob[l]] = 1;
            shared[p][q] = malloc(sizeof(int64_t) * (R[p].n ? R[p].n : 1));
            for (int64_t l = 0; l < R[p].n; ++l)   /* ascending global id on both sides */
                if (mark[R[p].glob[l]]) shared[p][q][n_shared[p][q]++] = l;
            if (n_shared[p][q] > cap) cap = n_shared[p][q];
        }
    }

    /* ---- per rank: slab mesh, element matrices, plan, Dirichlet set ---- */
    const size_t wsb = ebs_vec_workspace_bytes();
    for (int p = 0; p < P; ++p) {
        Rank *r = &R[p];
        for (int64_t l = 0; l < r->n; ++l) g2l[r->glob[l]] = (int32_t)l;
        const int64_t ne_p = r->hi - r->lo;
        double *hnl = malloc(sizeof(double) * 2 * r->n);
        int32_t *hcl = malloc(sizeof(int32_t) * 3 * ne_p);
        for (int64_t l = 0; l < r->n; ++l) {
            hnl[2 * l] = hn[2 * r->glob[l]];
            hnl[2 * l + 1] = hn[2 * r->glob[l] + 1];
        }
        for (int j = 0; j < 3; ++j)
            for (int64_t e = 0; e < ne_p; ++e) hcl[j * ne_p + e] = g2l[hc[j * ne + r->lo + e]];
        double *nl = up(hnl, sizeof(double) * 2 * r->n);
        int32_t *cl = up(hcl, sizeof(int32_t) * 3 * ne_p);
        double *Al = dev(sizeof(double) * 9 * ne_p), *bel = dev(sizeof(double) * 3 * ne_p);
        EBS(ebs_assemble_p1(2, ne_p, nl, cl, 1.0, NULL, 1.0, NULL, NULL, Al, bel, degenerate, NULL));
        EBS(ebs_plan_create(3, r->n, ne_p, cl, NULL, &r->plan));
        EBS(ebs_plan_load(r->plan, Al, bel, NULL));
        int64_t *hndl = malloc(sizeof(int64_t) * (r->n ? r->n : 1)), ndl = 0;
        for (int64_t l = 0; l < r->n; ++l)
            if (hf[r->glob[l]]) hndl[ndl++] = l;
        int64_t *ndd = up(hndl, sizeof(int64_t) * ndl);
        EBS(ebs_plan_set_dirichlet(r->plan, ndd, ndl, NULL));
        /* internal numbering of the plan: interface / owned flags, chunk lists */
        int32_t *n2o_d = dev(sizeof(int32_t) * r->n), *o2n_d = dev(sizeof(int32_t) * r->n);
        EBS(ebs_plan_node_maps(r->plan, o2n_d, n2o_d, NULL));
        int32_t *new_of_old = malloc(sizeof(int32_t) * r->n);
        r->old_of_new = malloc(sizeof(int32_t) * r->n);
        CUDA(cudaMemcpy(new_of_old, o2n_d, sizeof(int32_t) * r->n, cudaMemcpyDeviceToHost));
        CUDA(cudaMemcpy(r->old_of_new, n2o_d, sizeof(int32_t) * r->n, cudaMemcpyDeviceToHost));
        uint8_t *hif = calloc(r->n, 1), *how = calloc(r->n, 1);
        for (int q = 0; q < P; ++q) {  /* shared nodes per neighbour, internal numbering */
            if (q == p || n_shared[p][q] == 0) continue;
            int64_t *ii = malloc(sizeof(int64_t) * n_shared[p][q]);
            for (int64_t k = 0; k < n_shared[p][q]; ++k) {
                ii[k] = new_of_old[shared[p][q][k]];
                hif[ii[k]] = 1;
            }
            r->nb[r->n_nb] = q;
            r->lens[r->n_nb] = n_shared[p][q];
            r->idx[r->n_nb++] = up(ii, sizeof(int64_t) * n_shared[p][q]);
            free(ii);
        }
        for (int64_t i = 0; i < r->n; ++i) how[i] = owner[r->glob[r->old_of_new[i]]] == p;
        const int64_t nch = (r->n + 31) / 32;
        int32_t *hch = malloc(sizeof(int32_t) * nch);
        uint8_t *chif = calloc(nch, 1);
        for (int64_t i = 0; i < r->n; ++i)
            if (hif[i]) chif[i / 32] = 1;
        for (int64_t c = 0; c < nch; ++c)
            if (chif[c]) hch[r->n_if_chunks++] = (int32_t)c;
        r->n_chunks = r->n_if_chunks;
        for (int64_t c = 0; c < nch; ++c)
            if (!chif[c]) hch[r->n_chunks++] = (int32_t)c;
        r->chunks = up(hch, sizeof(int32_t) * nch);
        r->iface = up(hif, r->n);
        r->owned = up(how, r->n);
        r->free_m = dev(r->n);
        EBS(ebs_plan_free_mask(r->plan, r->free_m, NULL));
        r->b = dev(sizeof(double) * r->n);
        r->dinv = dev(sizeof(double) * r->n);
        r->xa = dev(sizeof(double) * r->n);
        r->xb = dev(sizeof(double) * r->n);
        r->s = dev(sizeof(double) * r->n);
        r->red3 = dev(sizeof(double) * 2);
        r->norm2 = dev(sizeof(double) * (iters + 1));
        r->ws = dev(wsb);
        CUDA(cudaMemset(r->xa, 0, sizeof(double) * r->n));
        CUDA(cudaMemset(r->red3, 0, sizeof(double) * 2));
        CUDA(cudaMemset(r->ws, 0, wsb));
        free(hnl); free(hcl); free(hndl); free(new_of_old); free(hif); free(how);
        free(hch); free(chif);
    }

    /* ---- peer group: one window per rank, every view sees all of them ---- */
    void *wins[PMAX];
    for (int p = 0; p < P; ++p) EBS(ebs_peer_window_alloc(cap, &wins[p], NULL));
    for (int p = 0; p < P; ++p) {
        EBS(ebs_peer_create(p, P, cap, wins, 60.0, &R[p].peer));
        EBS(ebs_peer_set_halo(R[p].peer, R[p].n, R[p].n_nb, R[p].nb, R[p].lens, R[p].idx, NULL));
    }

    /* ---- assembled b and Jacobi 1/diag over the halo: push all ranks, then combine ---- */
    for (int p = 0; p < P; ++p) {
        EBS(ebs_plan_internal_rhs(R[p].plan, R[p].b, NULL));
        EBS(ebs_plan_internal_diag(R[p].plan, R[p].dinv, NULL));
    }
    for (int p = 0; p < P; ++p) EBS(ebs_peer_push(R[p].peer, R[p].b, NULL));
    for (int p = 0; p < P; ++p) EBS(ebs_peer_combine(R[p].peer, R[p].b, R[p].ws, NULL));
    for (int p = 0; p < P; ++p) EBS(ebs_peer_push(R[p].peer, R[p].dinv, NULL));
    for (int p = 0; p < P; ++p) EBS(ebs_peer_combine(R[p].peer, R[p].dinv, R[p].ws, NULL));
    for (int p = 0; p < P; ++p)
        EBS(ebs_vec_dinv(R[p].n, R[p].dinv, R[p].free_m, R[p].dinv, NULL));

    /* ---- damped Jacobi: per iteration every rank's sweep, then every rank's combine ---- */
    for (int k = 0; k <= iters; ++k) {
        const int final = k == iters;
        for (int p = 0; p < P; ++p) {
            Rank *r = &R[p];
            double *src = (k & 1) ? r->xb : r->xa, *dst = (k & 1) ? r->xa : r->xb;
            EBS(ebs_peer_jacobi_sweep(r->plan, r->peer, r->chunks, r->n_chunks, r->n_if_chunks,
                                      omega, src, final ? NULL : dst, r->b, r->dinv, r->iface,
                                      r->s, r->red3, r->ws, NULL));
        }
        for (int p = 0; p < P; ++p) {
            Rank *r = &R[p];
            double *src = (k & 1) ? r->xb : r->xa, *dst = (k & 1) ? r->xa : r->xb;
            EBS(ebs_peer_combine_jacobi(r->peer, r->s, omega, r->b, r->dinv, r->free_m, r->owned,
                                        src, final ? NULL : dst, r->red3, r->norm2 + k, r->ws,
                                        NULL));
        }
    }
    CUDA(cudaDeviceSynchronize());

    /* ---- checks: norm history (owned sums in rank order) and the owned entries of x ---- */
    double *sum = calloc(iters + 1, sizeof(double)), *h2 = malloc(sizeof(double) * (iters + 1));
    double *hx = malloc(sizeof(double) * nn);
    for (int p = 0; p < P; ++p) {
        Rank *r = &R[p];
        EBS(ebs_peer_status(r->peer, NULL));
        CUDA(cudaMemcpy(h2, r->norm2, sizeof(double) * (iters + 1), cudaMemcpyDeviceToHost));
        for (int k = 0; k <= iters; ++k) sum[k] += h2[k];
        double *xf = malloc(sizeof(double) * r->n);
        CUDA(cudaMemcpy(xf, (iters & 1) ? r->xb : r->xa, sizeof(double) * r->n,
                        cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < r->n; ++i) {
            const int64_t g = r->glob[r->old_of_new[i]];
            if (owner[g] == p) hx[g] = xf[i];
        }
        free(xf);
    }
    double worst_norm = 0.0, dx = 0.0, xn = 0.0;
    for (int k = 0; k <= iters && k < n_norms; ++k) {
        const double d = fabs(sqrt(sum[k]) - norms1[k]) / norms1[k];
        if (d > worst_norm) worst_norm = d;
    }
    for (int64_t g = 0; g < nn; ++g) {
        dx += (hx[g] - hu1[g]) * (hx[g] - hu1[g]);
        xn += hu1[g] * hu1[g];
    }
    const double rel_x = sqrt(dx / xn);
    printf("level %d, %d slabs (peer-memory halo), %d Jacobi iterations: max rel norm diff %.2e, "
           "rel x diff %.2e vs single GPU (%d norms), launches %lld\n", level, P, iters,
           worst_norm, rel_x, n_norms, (long long)ebs_launch_count());
    const int ok = n_norms == iters + 1 && !diverged && worst_norm <= 1e-12 && rel_x <= 1e-12;
    for (int p = 0; p < P; ++p) {
        EBS(ebs_peer_destroy(R[p].peer));
        EBS(ebs_plan_destroy(R[p].plan));
        EBS(ebs_peer_window_free(wins[p]));
    }
    EBS(ebs_plan_destroy(gplan));
    printf("%s\n", ok ? "OK" : "FAILED");
    return ok ? 0 : 2;
}
