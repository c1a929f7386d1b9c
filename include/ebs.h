/*
 * ebs.h -- C-ABI of libebs.so, the B200 (sm_100a) element-based P1 solver path.
 *
 * The reference (arXiv 1911.03973, package `ebsolve`, /root/reference/pkg/src/ebsolve)
 * is pure Python/NumPy and has no FFI; its Python functions ARE the operator API
 * (SURVEY.md 8b).  Each entry point below replaces one of those functions (cited
 * as `file.py:line`); the Python package `paper_1911_03973_b200` binds this header
 * with ctypes and maps it back to the reference signatures.
 *
 * Conventions
 *   - Every function returns an int status: EBS_OK (0) or a negative EBS_E* code;
 *     ebs_last_error() returns the message of the calling thread's last failure.
 *     No C++ exception crosses this boundary.
 *   - All array pointers are DEVICE pointers owned by the caller (torch); the library
 *     never frees caller memory.  `stream` is a cudaStream_t (NULL = legacy default).
 *     Calls are asynchronous on `stream` unless stated otherwise.
 *   - A plan may be shared by host threads and streams: calls that use its device
 *     workspace are serialised on the device in call order (a call on a new stream
 *     waits for the previous call's work), as the reference allows concurrent
 *     residual calls on a shared batch.
 *   - Connectivity is int32 structure-of-arrays `conn[j*n_e + e]` (j = local vertex),
 *     i.e. the reference `indt` (mesh.py:151-154) narrowed to int32.
 *   - Element matrices are element-major `A[(e*nb + i)*nb + j]`, the memory behind the
 *     reference's (nb, nb, n_e) views (elements.py:86,93); b_e is SoA `b_e[j*n_e + e]`
 *     (elements.py:112).  nb = dim + 1 (3 triangles, 4 tetrahedra).
 *   - Vectors passed to operators are in the caller's node numbering; the plan keeps its
 *     own locality-ordered internal numbering and converts at the boundary.
 *   - Arithmetic is IEEE fp64 without FMA contraction (the library is compiled with
 *     -fmad=false) so results can be bit-identical to the NumPy reference.
 */
#ifndef EBS_H
#define EBS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EBS_OK 0
#define EBS_EINVAL (-1)      /* invalid argument -> ValueError            */
#define EBS_ENOMEM (-2)      /* device allocation failed -> MemoryError   */
#define EBS_ECUDA (-3)       /* CUDA runtime error -> RuntimeError        */
#define EBS_ENCCL (-4)       /* collective failure -> RuntimeError        */
#define EBS_ENONFINITE (-5)  /* non-finite input -> ValueError            */
#define EBS_EDEGENERATE (-6) /* degenerate element -> ValueError          */
#define EBS_ECALLBACK (-7)   /* user callback asked to stop               */

typedef struct ebs_plan *ebs_plan_t;

/* residual modes (ebs_residual) */
#define EBS_RES_EXACT 0 /* sum_e C_e^T (b_e - A_e x_e), reference order (operators.py:98) */
#define EBS_RES_FAST 1  /* b - sum_e C_e^T A_e x_e with pre-assembled b            */

/* solver methods (ebs_solve) */
#define EBS_RICHARDSON 0 /* solvers.py:163-183                                   */
#define EBS_JACOBI 1     /* damped Jacobi on the solvers.py:117-160 loop (NEW)   */
#define EBS_CG 2         /* conjugate gradients (NEW)                            */
#define EBS_PCG 3        /* Jacobi-preconditioned CG (NEW)                       */
#define EBS_CHEB2 4      /* cyclic two-level Chebyshev, solvers.py:186-213       */
#define EBS_CHEB3 5      /* three-level Chebyshev recurrence, solvers.py:216-261 */

int ebs_version(void);
int ebs_last_error(char *buf, size_t len);
/* number of this library's kernels launched so far (process-wide counter) */
int64_t ebs_launch_count(void);

/* ------------------------------------------------------------------ mesh ---- */
/* mesh.py:104-128 build_grid_mesh: n nodes per side; nodes (n*n, 2) row-major,
 * conn SoA (3, 2(n-1)^2) with per cell lower (ll,ll+1,ll+n+1), upper (ll,ll+n+1,ll+n). */
int ebs_mesh_grid2d(int64_t n, double *nodes, int32_t *conn, void *stream);
/* NEW (no reference): unit cube, N cells/side, 6 Kuhn tets per cube (oracle/ebs_oracle.py
 * kuhn_cube_mesh); nodes ((N+1)^3, 3), conn SoA (4, 6N^3). */
int ebs_mesh_kuhn3d(int64_t N, double *nodes, int32_t *conn, void *stream);
/* mesh.py:145-148 _detect_boundary (which=0: any coordinate within 1e-12 of 0 or 1)
 * or the z=0 face (which=1, BASELINE C3/C5).  flags[n] = 1/0. */
int ebs_mesh_flags(int dim, int64_t n_n, const double *nodes, int which, uint8_t *flags,
                   void *stream);
/* mesh.py:39-52 Mesh.__post_init__ checks: counts[0] = #connectivity entries out of
 * [0, n_n), counts[1] = #elements with signed measure <= 0 (device int64[2], zeroed here). */
int ebs_mesh_check(int dim, int64_t n_n, int64_t n_e, const double *nodes,
                   const int32_t *conn, int64_t *counts, void *stream);
/* signed area (mesh.py:96-101) / volume per element */
int ebs_mesh_measure(int dim, int64_t n_e, const double *nodes, const int32_t *conn,
                     double *measure, void *stream);
/* uniform_refine (mesh.py:157-208): red refinement of a triangle mesh -- 4 children per
 * triangle through the edge midpoints 0.5*(x[lo] + x[hi]), nodes renumbered ascending in
 * (y, x), each child rotated to start at its smallest node (orientation kept), children
 * sorted ascending; a structured level-L mesh becomes build_unit_square_mesh(L+1) bit for bit.
 * coords (n_n, 2) f64, conn (3, n_e) int32 SoA; coords_out needs room for n_n + 3 n_e
 * nodes, conn_out (3, 4 n_e); *n_out (HOST) = the refined node count.  Synchronises
 * `stream` (the node count is data dependent). */
int ebs_refine_tri(int64_t n_n, int64_t n_e, const double *coords, const int32_t *conn,
                   double *coords_out, int32_t *conn_out, int64_t *n_out, void *stream);
/* NEW: relabel nodes, new id of old node i = perm[i] (BASELINE C2/C4 recipe). */
int ebs_mesh_permute(int dim, int64_t n_n, int64_t n_e, const int64_t *perm,
                     const double *nodes, const int32_t *conn, double *nodes_out,
                     int32_t *conn_out, void *stream);
/* elements.py:107 centroids p.mean(axis=1) = ((p0+p1)+p2)/3 [+p3 ../4]; out (n_e, dim). */
int ebs_centroids(int dim, int64_t n_e, const double *nodes, const int32_t *conn,
                  double *out, void *stream);

/* -------------------------------------------------------------- assembly ---- */
/* elements.py:56-137 local_{stiffness,mass,load}_batch + combine_system, fused:
 * K_e = meas * G^T G, M_e = meas * pattern, A_e = K_e + nu*M_e,
 * b_e[j] = (f*meas)/nb with f = f_vals[e] (nullable -> f_const).  Any output may be NULL.
 * n_degenerate (device int64, zeroed here) counts elements with measure <= EPS
 * (elements.py:67-71); the caller raises ValueError when it is non-zero. */
int ebs_assemble_p1(int dim, int64_t n_e, const double *nodes, const int32_t *conn,
                    double nu, const double *f_vals, double f_const, double *K_e,
                    double *M_e, double *A_e, double *b_e, int64_t *n_degenerate,
                    void *stream);
/* elements.py:115-121 combine_system: A = K + nu*M over count doubles. */
int ebs_combine(int64_t count, const double *K_e, const double *M_e, double nu, double *A_e,
                void *stream);

/* ------------------------------------------------------------------ plan ---- */
/* Build the execution plan of a mesh (synchronous on `stream`): node->(j,e) incidence in
 * the bincount order j*n_e+e (operators.py:98), a first-appearance internal node
 * numbering and the SELL-32 slot layout the operator kernels stream.  The plan owns its
 * device workspace; destroy releases it. */
int ebs_plan_create(int nb, int64_t n_nodes, int64_t n_elems, const int32_t *conn,
                    void *stream, ebs_plan_t *out);
int ebs_plan_destroy(ebs_plan_t plan);
/* info[0]=n_nodes info[1]=n_elems info[2]=nb info[3]=n_chunks info[4]=n_rows
 * info[5]=slot bytes resident  info[6]=max valence  info[7]=flags:
 *   1 operator loaded, 2 b_e loaded, 4 packed-delta ids, 8 per-chunk delta tables,
 *   16 two-base 3D rows, 32 one-byte tuple codes, 64 identity numbering (the caller's
 *   numbering is a structured grid and is kept as the internal one) */
int ebs_plan_info(ebs_plan_t plan, int64_t *info);
/* copy the internal numbering maps out (device int32 arrays of n_nodes) */
int ebs_plan_node_maps(ebs_plan_t plan, int32_t *new_of_old, int32_t *old_of_new,
                       void *stream);
/* Load an operator: pack A_e (element-major) rows into the slot stream; when b_e is
 * non-NULL also pack it per slot (exact residual) and pre-assemble b (fast residual). */
int ebs_plan_load(ebs_plan_t plan, const double *A_e, const double *b_e, void *stream);
/* operators.py:29-55 DirichletData.nd (caller numbering, any order): the constrained set
 * used by masked operators and solvers.  n_d = 0 clears it. */
int ebs_plan_set_dirichlet(ebs_plan_t plan, const int64_t *nd, int64_t n_d, void *stream);

/* ------------------------------------------------------------- operators ---- */
/* operators.py:72-111 residual: r = b - A x (mode EBS_RES_EXACT reproduces the reference
 * bit for bit; EBS_RES_FAST uses the pre-assembled b).  masked != 0 also applies
 * mask_dirichlet (operators.py:114-118).  nonfinite (device int32, nullable) is written:
 * 1 when x has a non-finite entry (operators.py:90-91), else 0 (no reset needed). */
int ebs_residual(ebs_plan_t plan, const double *x, double *r, int mode, int masked,
                 int32_t *nonfinite, void *stream);
/* NEW: ebs_residual on k caller-numbered DEVICE vectors (x_i at x + i*ldx, ldx 0 or >=
 * n_nodes; r_i written to r + i*ldr, ldr >= n_nodes; rows must not alias), two residuals
 * in flight: odd i run on a second stream kept by the plan, each stream with its own
 * workspace, forked from and joined back into `stream` (asynchronous; capturable once a
 * first, uncaptured call has created the plan's second stream and workspace).  The
 * permutation / fill of one residual overlaps the other's operator pass.  Each r_i is
 * bit-identical to ebs_residual on x_i.  nonfinite (DEVICE int32[k], nullable): the
 * per-vector flag of ebs_residual. */
int ebs_residual_many(ebs_plan_t plan, const double *x, int64_t ldx, double *r, int64_t ldr,
                      int64_t k, int mode, int masked, int32_t *nonfinite, void *stream);
/* NEW: ebs_residual on k caller-numbered vectors in HOST memory (x_i at x_host + i*ldx,
 * ldx 0 or >= n_nodes; r_i written to r_host + i*ldr, ldr >= n_nodes).  The host->device
 * copy of x_{i+1}, the residual of x_i and the device->host copy of r_{i-1} overlap
 * (copy streams + device buffers kept by the plan); pinned host memory lets the copies
 * run asynchronously.  Each r_i is bit-identical to ebs_residual on x_i.  nonfinite
 * (HOST int32[k], nullable): the per-vector flag of ebs_residual.  Returns once every r_i
 * is in r_host (host-synchronous; not capturable); ordered after prior work on stream. */
int ebs_residual_many_host(ebs_plan_t plan, const double *x_host, int64_t ldx, double *r_host,
                           int64_t ldr, int64_t k, int mode, int masked, int32_t *nonfinite_host,
                           void *stream);
/* spectrum.py:54-61 _apply_masked: y = A x in (j,e) order; masked != 0 zeroes y[nd]. */
int ebs_matvec(ebs_plan_t plan, const double *x, double *y, int masked, void *stream);
/* NEW diag(A) = assemble_rhs(stack_j A_e[j,j,:]), caller numbering. */
int ebs_diagonal(ebs_plan_t plan, double *d, void *stream);
/* spectrum.py:118-120 order: per local vertex j a bincount of A_e[j,j,:], then the
 * per-j sums added j = 0, 1, ... (mass_gershgorin), caller numbering. */
int ebs_diagonal_grouped(ebs_plan_t plan, double *d, void *stream);
/* operators.py:58-63 assemble_rhs: b = bincount(indt, b_e) in (j,e) order; needs only
 * the plan's structure (no load). */
int ebs_assemble_rhs(ebs_plan_t plan, const double *b_e, double *b, void *stream);
/* operators.py:114-118 mask_dirichlet on a caller-numbered vector: out = v, out[nd] = 0. */
int ebs_mask(int64_t n, const double *v, int64_t n_d, const int64_t *nd, double *out,
             void *stream);
/* Internal-numbering access (bench timing, multi-GPU driver).  The plan's internal node
 * order is first appearance over (e, j); vectors in that order are "internal".
 * ebs_to_internal: x_int[m] = x[old_of_new[m]] (+ non-finite flag, nullable);
 * ebs_to_user: v[old_of_new[m]] = v_int[m]. */
int ebs_to_internal(ebs_plan_t plan, const double *x, double *x_int, int32_t *nonfinite,
                    void *stream);
int ebs_to_user(ebs_plan_t plan, const double *v_int, double *v, void *stream);
/* SELL pass (op 0 matvec, 1 fast residual) writing out[out_map[m]] (any int32 map, e.g. a
 * rank's internal -> global ids) and, when s_raw != NULL, the same values in internal
 * order (an element slab's partial sums / partial residuals for the halo). */
int ebs_plan_apply_map(ebs_plan_t plan, int op, const double *x_int, double *out,
                       const int32_t *out_map, double *s_raw, int masked, void *stream);
/* The same pass over a list of SELL chunks only (chunk c = internal nodes 32c .. 32c+31;
 * a rank sweeps its interface chunks, posts the halo exchange, then sweeps the rest).
 * flags: EBS_APPLY_MASKED zeroes constrained rows; EBS_APPLY_ADD adds each value into
 * out[out_map[m]] (out pre-filled with -0.0: bit-identical to storing, and cheaper for a
 * scattered map). */
#define EBS_APPLY_MASKED 1
#define EBS_APPLY_ADD 2
int ebs_plan_apply_map_chunks(ebs_plan_t plan, int op, const int32_t *chunks, int64_t n_list,
                              const double *x_int, double *out, const int32_t *out_map,
                              double *s_raw, int flags, void *stream);
/* One SELL pass on internal vectors: op = 0 matvec, 1 fast residual, 2 exact residual;
 * out_user = 0 writes internal order, 1 the caller's numbering, 2 the caller's numbering
 * by adding into `out`, which the caller has filled with -0.0 (bit-identical to 1 and
 * cheaper: the pre-fill can ride along with an earlier pass over the vector);
 * masked != 0 zeroes constrained rows. */
int ebs_plan_apply(ebs_plan_t plan, int op, const double *x_int, double *out, int out_user,
                   int masked, void *stream);
/* out[0..n) = value (16 B stores); value -0.0 prepares the output of an EBS_APPLY_ADD /
 * out_user = 2 pass. */
int ebs_fill(int64_t n, double value, double *out, void *stream);
/* all-finite check (operators.py:90): *flag (device int32) = 1 if any non-finite. */
int ebs_check_finite(int64_t n, const double *v, int32_t *flag, void *stream);

/* reference.py:25-39 assemble_sparse, on the device (cross-check path, never used by the
 * solvers): CSR of the loaded operator in caller numbering, columns sorted, duplicates
 * summed in (j, e) order.  ebs_csr_nnz fills crow (n+1 entries, int64); ebs_csr_fill
 * writes col (int32) / val.  conn is the plan's connectivity (int32 SoA). */
int ebs_csr_nnz(ebs_plan_t plan, const int32_t *conn, int64_t *crow, void *stream);
int ebs_csr_fill(ebs_plan_t plan, const int32_t *conn, const int64_t *crow, int32_t *col,
                 double *val, void *stream);

/* ----------------------------------------------------------- vector work ---- */
/* deterministic (fixed-order, launch-size independent of the device) reductions */
int ebs_dot(int64_t n, const double *x, const double *y, double *out, void *stream);
int ebs_nrm2(int64_t n, const double *x, double *out, void *stream);
/* y = a*x + b*y */
int ebs_axpby(int64_t n, double a, const double *x, double b, double *y, void *stream);

/* --------------------------------------------------------------- solvers ---- */
/* The solvers.py:117-160 loop (_iterate) run on the device: per iteration one fused
 * element-operator pass plus vector work, norms kept on the device and read once at
 * the end.  Richardson: x += omega*r (solvers.py:179-180), omega = 2/(l1+l2) given by the
 * caller.  Jacobi: x += omega*(dinv*r).  CG / PCG: see oracle/ebs_oracle.py pcg().
 * Iterates, history and divergence semantics follow _iterate (history length
 * n_norms <= iters+1, tol relative to ||r_0||, divergence is a flag, never an error). */
typedef int (*ebs_callback_t)(void *user, int k);

typedef struct {
    int method;              /* EBS_RICHARDSON / EBS_JACOBI / EBS_CG / EBS_PCG           */
    int iters;               /* >= 0                                                     */
    int exact;               /* residual mode for Richardson/Jacobi (1 = EBS_RES_EXACT)  */
    int has_tol;             /* tol is not None                                          */
    double tol;              /* stop when ||r_k|| <= tol*||r_0|| (solvers.py:135)        */
    double omega;            /* Richardson / Jacobi step                                 */
    const double *x0;        /* device, caller numbering (copied, never written)          */
    double *x;               /* device out, caller numbering                             */
    const double *reference; /* device, nullable: error norms ||x_k - reference||         */
    double *norms;           /* HOST out, iters+1 entries                                 */
    double *errors;          /* HOST out, iters+1 entries (when reference != NULL)        */
    int *n_norms;            /* HOST out: recorded history length                         */
    int *diverged;           /* HOST out                                                  */
    ebs_callback_t callback; /* nullable: called as callback(user, k) after x_k and r_k   */
    void *user;              /*   were copied into cb_x / cb_r (device, caller numbering); */
    double *cb_x;            /*   a non-zero return stops the solve with EBS_ECALLBACK     */
    double *cb_r;
    double *r_out;           /* device, nullable: final residual (caller numbering)       */
    const double *coef_a;    /* HOST, iters entries: CHEB2 step 1/alpha_{k mod N};         */
    const double *coef_b;    /*   CHEB3 alpha_k and beta_k (solvers.py:247-258)             */
    int fused;               /* CG / PCG without callback: the whole loop as one cooperative */
                             /*   persistent kernel (grid-wide barriers, no launches per it) */
} ebs_solve_params;

/* synchronous on `stream` (one host read of the history at the end) */
int ebs_solve(ebs_plan_t plan, const ebs_solve_params *params, void *stream);

/* spectrum.py:64-99 power_iteration_lambda_max on the masked operator (loaded Dirichlet
 * set): v = v0 masked and normalised, then v <- A v / ||A v|| until the Rayleigh quotient
 * changes by <= tol*max(1,|lam|) or iters steps; *lam (HOST) receives the estimate, *its
 * (HOST) the steps taken.  Returns EBS_EINVAL when v0 vanishes after masking. */
int ebs_power_iteration(ebs_plan_t plan, const double *v0, int iters, double tol, double *lam,
                        int *its, void *stream);

/* ------------------------------------------------------------ multi-GPU ---- */
/* Element-slab partition helpers.  A rank's plan is built on its element
 * slab with its local node numbering; interface partial sums are exchanged by the host
 * (torch.distributed / NCCL over NVLink) through these pack/unpack kernels.
 * buf[i] = v[idx[i]]                                                          */
int ebs_gather(int64_t n, const int64_t *idx, const double *v, double *buf, void *stream);
/* v[idx[i]] += buf[i]  (idx entries unique)                                   */
int ebs_scatter_add(int64_t n, const int64_t *idx, const double *buf, double *v, void *stream);
/* v[idx[i]] = value;  dst[idx[i]] = src[idx[i]]  (interface combine in rank order)    */
int ebs_index_fill(int64_t n, const int64_t *idx, double value, double *v, void *stream);
int ebs_index_copy(int64_t n, const int64_t *idx, const double *src, double *dst, void *stream);
/* dst[dst_idx[i]] += src[src_idx[i]]  (neighbour partial residuals onto owned entries) */
int ebs_index_add(int64_t n, const int64_t *src_idx, const double *src, const int64_t *dst_idx,
                  double *dst, void *stream);
/* dst[dst_idx[i]] = src[src_idx[i]]  (owned rank results to the caller's numbering)     */
int ebs_index_move(int64_t n, const int64_t *src_idx, const double *src, const int64_t *dst_idx,
                   double *dst, void *stream);
/* Per-rank vector steps on internal-numbered vectors.  `owned` (uint8, 1 = this rank owns
 * the node) restricts every reduction to owned nodes; the host all-reduces `red`.
 * `ws` is a device workspace of ebs_vec_workspace_bytes() bytes (zero-initialised once,
 * one per concurrent stream).  Damped Jacobi / Richardson (dinv NULL) step:
 *   r = free ? b - s : 0;  x_out = x + omega*(dinv*r);  red[0] = sum_owned r^2          */
size_t ebs_vec_workspace_bytes(void);
int ebs_vec_jacobi(int64_t n, double omega, const double *b, const double *s, const double *dinv,
                   const uint8_t *free_m, const uint8_t *owned, const double *x, double *x_out,
                   double *r_out, double *red, int32_t *nonfinite, void *ws, void *stream);
/* CG / PCG steps (oracle/ebs_oracle.py pcg):  q = free ? q : 0, red[0] = sum_owned p.q;
 * update with device scalars rz, pq: alpha = rz/pq, x += alpha p, r -= alpha q,
 * red = [sum_owned r.r, sum_owned r.(dinv r)];  direction: p = dinv r + (rz_new/rz_old) p */
int ebs_vec_pcg_q(int64_t n, const uint8_t *free_m, const uint8_t *owned, const double *p,
                  double *q, double *red, void *ws, void *stream);
int ebs_vec_pcg_update(int64_t n, const double *rz, const double *pq, const uint8_t *owned,
                       const double *dinv, double *x, double *r, const double *p, const double *q,
                       double *red, int32_t *nonfinite, void *ws, void *stream);
int ebs_vec_pcg_direction(int64_t n, const double *rz_old, const double *rz_new,
                          const double *dinv, const double *r, double *p, void *stream);
/* Single-reduction Jacobi-PCG step (Chronopoulos-Gear; one all-reduce per iteration).
 * cur = [gamma_k = r.u, delta_k = w.u, rr_k = r.r, alpha_k (written)] of iteration k, with
 * [0..2] already all-reduced; prev = the same of iteration k-1 (prev[0] == 0: first step,
 * beta = 0).  beta = gamma_k/gamma_{k-1}, alpha = gamma_k/(delta_k - beta gamma_k/alpha_{k-1});
 * p = u + beta p, s = w + beta s, x += alpha p, r -= alpha s, u = dinv r;
 * next[0] = sum_owned r.u, next[2] = sum_owned r.r (next[1] = the matvec's w.u, from
 * ebs_dist_matvec_sweep / ebs_dist_q_iface or ebs_vec_pcg_q with p := u, q := w).
 * ctl (device int32[4], nullable) = [stop, k_stop, k, diverged]: the _iterate loop rules
 * (solvers.py:117-160) on the device -- instead of updating, the launch sets stop (k_stop = k)
 * when sqrt(rr_k) <= tol*sqrt(rr0[0]) (tol >= 0) or rr_k is not finite (diverged = 1);
 * once stop is set every launch is a no-op.  No host synchronisation anywhere. */
int ebs_vec_cg1_update(int64_t n, double *cur, const double *prev, const double *rr0, double tol,
                       int32_t *ctl, const uint8_t *owned, const double *dinv, double *x,
                       double *r, double *u, const double *w, double *p, double *s,
                       double *next, int32_t *nonfinite, void *ws, void *stream);
/* The plan's fused matvec sweeps (ebs_dist_matvec_sweep) become no-ops while *stop != 0
 * (device int32, e.g. ctl[0] above; NULL clears). */
int ebs_dist_set_stop(ebs_plan_t plan, const int32_t *stop);
int ebs_vec_dot_owned(int64_t n, const double *x, const double *y, const uint8_t *owned,
                      double *red, void *ws, void *stream);
/* dinv = free ? (diag ? 1/diag : 1) : 0 */
int ebs_vec_dinv(int64_t n, const double *diag, const uint8_t *free_m, double *dinv,
                 void *stream);
/* Fused slab-rank steps (overlap of the halo exchange with interior work).  The SELL
 * pass sweeps only the `chunks` listed (n_list of them); nodes with iface[m] = 1 (shared
 * with another slab) store their partial sum in s_part / q and are completed after the
 * exchange by the *_iface kernels over the interface node list idx; all other nodes are
 * finished in the pass.  red[0] = sum over the nodes finished (owned) by that launch.
 * Jacobi: r = free ? b - s : 0, x_out = x + omega*(dinv*r) (dinv NULL: Richardson).
 * PCG matvec: q = free ? s : 0, red = p.q. */
int ebs_dist_jacobi_sweep(ebs_plan_t plan, const int32_t *chunks, int64_t n_list, double omega,
                          const double *x, double *x_out, const double *b, const double *dinv,
                          const uint8_t *iface, double *s_part, double *red, void *ws,
                          void *stream);
int ebs_dist_matvec_sweep(ebs_plan_t plan, const int32_t *chunks, int64_t n_list, const double *pv,
                          double *q, const uint8_t *iface, double *red, void *ws, void *stream);
int ebs_dist_jacobi_iface(int64_t n, const int64_t *idx, double omega, const double *b,
                          const double *s, const double *dinv, const uint8_t *free_m,
                          const uint8_t *owned, const double *x, double *x_out,
                          const double *prior, double *red, void *ws, void *stream);
/* Shared-node completion after the halo exchange: v[all_if[i]] = sum over k of
 * srcs[k][pos[i*n_src + k]] (entries with pos < 0 skipped), sources in ascending rank order
 * -- the rank's own partials are the source whose positions are the nodes themselves.
 * srcs is a HOST array of n_src (<= 8) device pointers. */
int ebs_dist_combine(int64_t n_if, const int64_t *all_if, int n_src, const double *const *srcs,
                     const int32_t *pos, double *v, void *stream);
/* The combine and the interface completion fused (one launch less per iteration):
 * s[all_if[i]] = the rank-ordered sum as ebs_dist_combine, then the Jacobi completion of
 * ebs_dist_jacobi_iface on that node (_jacobi), or q = free ? sum : 0 and red[0] = (prior[0]
 * + prior[1]) + sum_owned p.q as ebs_dist_q_iface (_q).  srcs is a HOST array. */
int ebs_dist_combine_jacobi(int64_t n_if, const int64_t *all_if, int n_src,
                            const double *const *srcs, const int32_t *pos, double *s, double omega,
                            const double *b, const double *dinv, const uint8_t *free_m,
                            const uint8_t *owned, const double *x, double *x_out,
                            const double *prior, double *red, void *ws, void *stream);
int ebs_dist_combine_q(int64_t n_if, const int64_t *all_if, int n_src, const double *const *srcs,
                       const int32_t *pos, double *q, const uint8_t *free_m, const uint8_t *owned,
                       const double *pv, const double *prior, double *red, void *ws,
                       void *stream);
/* ... and red[0] = (prior[0] + prior[1]) + the interface nodes' owned p.q (prior, nullable:
 * the interface- and interior-chunk partials of the sweeps): the rank's whole p.q. */
int ebs_dist_q_iface(int64_t n, const int64_t *idx, const uint8_t *free_m, const uint8_t *owned,
                     const double *pv, double *q, const double *prior, double *red, void *ws,
                     void *stream);
/* plan internals in internal numbering: Dirichlet free flags, pre-assembled b, diag(A) */
int ebs_plan_free_mask(ebs_plan_t plan, uint8_t *free_int, void *stream);
int ebs_plan_internal_rhs(ebs_plan_t plan, double *b_int, void *stream);
int ebs_plan_internal_diag(ebs_plan_t plan, double *d_int, void *stream);

/* ------------------------------------------------- element-slab collectives ---- */
/* the NCCL side of the element-slab path inside the library, so a C caller can
 * run the multi-GPU residual / solvers without Python (one process = one GPU = one slab).
 * NCCL is resolved at run time (dlopen libnccl.so.2): the NCCL already loaded in the
 * process (e.g. PyTorch's) or the system one.  Failures return EBS_ENCCL. */
#define EBS_DIST_ID_BYTES 128
/* ncclGetUniqueId on rank 0; the caller broadcasts the EBS_DIST_ID_BYTES bytes. */
int ebs_dist_unique_id(void *id_out);
/* ncclCommInitRank on the current device; the communicator belongs to the plan (freed by
 * ebs_plan_destroy).  Collective over the nranks processes. */
int ebs_dist_init(ebs_plan_t plan, const void *id, int rank, int nranks);
/* Halo exchange: for each of n_peers peers (host arrays peers[], counts[] and device
 * buffer pointers send[] / recv[]), counts[i] doubles go to and come from peers[i], as one
 * NCCL group on `stream` (a peer may be the caller's own rank). */
int ebs_dist_exchange(ebs_plan_t plan, int n_peers, const int32_t *peers, const int64_t *counts,
                      const double *const *send, double *const *recv, void *stream);
/* In-place sum over the ranks of n device doubles (the PCG dots) on `stream`. */
int ebs_dist_allreduce(ebs_plan_t plan, double *buf, int64_t n, void *stream);
/* Failure detection.  ebs_dist_poll: ncclCommGetAsyncError; on an error the communicator is
 * aborted (ncclCommAbort) and EBS_ENCCL returned.  ebs_dist_wait: wait until `stream` is
 * idle while polling; after timeout_s seconds (< 0: never) the communicator is aborted --
 * which also releases NCCL kernels waiting on a lost peer -- and EBS_ENCCL returned.
 * ebs_dist_abort: abort explicitly.  After an abort every collective of the plan returns
 * EBS_ENCCL until ebs_dist_init is called again. */
int ebs_dist_poll(ebs_plan_t plan);
int ebs_dist_wait(ebs_plan_t plan, void *stream, double timeout_s);
int ebs_dist_abort(ebs_plan_t plan);

/* ------------------------------------------------- peer-memory halo (peer.cu) ---- */
/* The element-slab halo and the dot all-reduce without a collective library: every rank of
 * a node (<= EBS_PEER_MAX) owns one device WINDOW that the other ranks map (CUDA IPC; NVLink
 * P2P between GPUs) and write into; epoch flags in the window publish the data.  The fused
 * slab sweeps (ebs_peer_*_sweep) store each interface node's partial sum straight into the
 * neighbours' windows from the SELL epilogue, chunk by chunk, while the same launch sweeps
 * the interior; ebs_peer_combine_* wait for the neighbours' flags, sum the shared nodes in
 * ascending rank order (the values of ebs_dist_combine_*) and complete them.  All ranks must
 * issue the same sequence of peer calls, each rank on one stream (a peer view holds device
 * epoch counters: it is not for concurrent use from several streams).  Waits are bounded by the timeout given to
 * ebs_peer_create; a timed-out wait sets the window's error word (ebs_peer_status ->
 * EBS_ENCCL) instead of hanging.  Replaces the reference's chunk loop + bincount over the
 * whole mesh (operators.py:95-111) across slabs; no reference counterpart for the transport. */
#define EBS_PEER_MAX 8
#define EBS_PEER_HANDLE_BYTES 64
typedef struct ebs_peer_s *ebs_peer_t;
/* Window of a rank whose largest interface has `cap` nodes; zeroed.  handle_out (nullable,
 * EBS_PEER_HANDLE_BYTES) receives its CUDA IPC handle for the other processes. */
size_t ebs_peer_window_bytes(int64_t cap);
int ebs_peer_window_alloc(int64_t cap, void **win, void *handle_out);
int ebs_peer_window_open(const void *handle, void **win); /* another process's window */
int ebs_peer_window_close(void *win);                     /* ... unmapped */
int ebs_peer_window_free(void *win);                      /* own window freed */
/* Peer group view of rank `rank`: wins[q] = rank q's window as mapped in this process
 * (wins[rank] = the own window); every rank uses the same cap.  timeout_s < 0: wait forever. */
int ebs_peer_create(int rank, int world, int64_t cap, void *const *wins, double timeout_s,
                    ebs_peer_t *out);
int ebs_peer_destroy(ebs_peer_t peer);
/* Halo of a slab plan with n_local nodes: neighbours nb_ranks[0..n_nb) (ascending), and per
 * neighbour the nb_len[k] local node ids (device int64, nb_idx[k]) it shares, in the order
 * both sides agree on (ascending global id).  Host arrays of device pointers. */
int ebs_peer_set_halo(ebs_peer_t peer, int64_t n_local, int n_nb, const int32_t *nb_ranks,
                      const int64_t *nb_len, const int64_t *const *nb_idx, void *stream);
/* EBS_ENCCL when a wait of this rank timed out (synchronises `stream`). */
int ebs_peer_status(ebs_peer_t peer, void *stream);
/* In-place sum over the ranks of n device doubles, added in rank order 0..world-1 (identical
 * on every rank).  mode 0: one launch per 256 values; 1 / 2: only the put / only the
 * wait-and-sum phase (n <= 256; for ranks emulated in one process, all puts first). */
int ebs_peer_allreduce(ebs_peer_t peer, double *buf, int64_t n, int mode, void *stream);
/* Generic halo: bufs[k] (nb_len[k] doubles, device) to neighbour k; recv: wait and copy
 * neighbour k's values into out[k].  push: v at the interface nodes to every neighbour;
 * combine: wait, then v[shared] = the rank-ordered sum.  ws: ebs_vec_workspace_bytes(). */
int ebs_peer_send(ebs_peer_t peer, const double *const *bufs, void *stream);
int ebs_peer_recv(ebs_peer_t peer, double *const *out, void *ws, void *stream);
int ebs_peer_push(ebs_peer_t peer, const double *v, void *stream);
int ebs_peer_combine(ebs_peer_t peer, double *v, void *ws, void *stream);
/* Fused slab steps: as ebs_dist_jacobi_sweep / ebs_dist_matvec_sweep over ALL the rank's
 * chunks in one launch, the n_if_chunks chunks holding interface nodes listed first; interface
 * partials go to the neighbours' windows from the epilogue.  Then the combine + completion
 * of ebs_dist_combine_jacobi / ebs_dist_combine_q after waiting for the neighbours. */
int ebs_peer_jacobi_sweep(ebs_plan_t plan, ebs_peer_t peer, const int32_t *chunks, int64_t n_list,
                          int64_t n_if_chunks, double omega, const double *x, double *x_out,
                          const double *b, const double *dinv, const uint8_t *iface,
                          double *s_part, double *red, void *ws, void *stream);
int ebs_peer_matvec_sweep(ebs_plan_t plan, ebs_peer_t peer, const int32_t *chunks, int64_t n_list,
                          int64_t n_if_chunks, const double *pv, double *q, const uint8_t *iface,
                          double *red, void *ws, void *stream);
/* Protocol self-test (synchronises): P peer views of ONE process (emulated ranks, every
 * window in this process) exercised by one cooperative kernel whose block groups act as the
 * ranks, concurrently and skewed -- `iters` rounds of interface pushes / flag waits /
 * rank-ordered sums and of the fused all-reduce, every value checked.  global_ids[r] (device
 * int64) = the global id of each local node of rank r.  *n_errors = the mismatches (0). */
int ebs_peer_selftest(ebs_peer_t const *peers, const int64_t *const *global_ids, int P,
                      int iters, int64_t *n_errors, void *stream);
/* The slab residual in the rank's caller order (its local nodes by ascending global id):
 * out[out_map[m]] = b_p - A_p x for every node (fast mode of ebs_plan_apply_map_chunks;
 * flags EBS_APPLY_ADD: added into a -0.0-filled out instead of stored), interface partials
 * pushed to the neighbours;
 * then the combine adds the neighbours' partials (ascending rank) onto the owned shared
 * entries -- bitwise the NCCL path's ebs_index_add corrections. */
int ebs_peer_residual_sweep(ebs_plan_t plan, ebs_peer_t peer, const int32_t *chunks,
                            int64_t n_list, int64_t n_if_chunks, const double *x_int, double *out,
                            const int32_t *out_map, const uint8_t *iface, int flags,
                            void *stream);
int ebs_peer_residual_combine(ebs_peer_t peer, const uint8_t *owned, const int32_t *out_map,
                              double *out, void *ws, void *stream);
/* One damped-Jacobi iteration k >= 1 in ONE launch, no grid barrier: the first
 * ceil(n_shared/32) warps complete iteration k-1's shared nodes (ebs_peer_combine_jacobi's
 * work: s_part totals, x_cur = x_k there from x_prev = x_{k-1}, red_prev[0] = (prior[0] +
 * prior[1]) + their owned r^2) while the other warps sweep the interior chunks of iteration
 * k from x_cur; the chunk list is [n_if_chunks interface chunks | interior | n_near chunks
 * with a node that shares an element with a shared node], and the interface and near chunks
 * wait for the completion (the interface ones then push their partials, as
 * ebs_peer_jacobi_sweep).  Its partial norm goes to part_out[0] (may alias prior[0]); x_out
 * may alias x_prev (ping-pong buffers). */
int ebs_peer_jacobi_step(ebs_plan_t plan, ebs_peer_t peer, const int32_t *chunks, int64_t n_list,
                         int64_t n_if_chunks, int64_t n_near, double omega, const double *x_prev,
                         double *x_cur, double *x_out, const double *b, const double *dinv,
                         const uint8_t *iface, const uint8_t *owned, double *s_part,
                         const double *prior, double *red_prev, double *part_out, void *ws,
                         void *stream);
int ebs_peer_combine_jacobi(ebs_peer_t peer, double *s, double omega, const double *b,
                            const double *dinv, const uint8_t *free_m, const uint8_t *owned,
                            const double *x, double *x_out, const double *prior, double *red,
                            void *ws, void *stream);
/* stop (device int32, nullable): as ebs_dist_set_stop -- a no-op once *stop != 0 (the matvec
 * sweep sent nothing).  dots (device, nullable; red may point into it): after red[0] is
 * written, dots[0..3) are put as this rank's contribution to the next all-reduce -- the
 * single-reduction PCG's [r.u, w.u, r.r] -- consumed by ebs_peer_cg1_update (or by
 * ebs_peer_allreduce mode 2). */
int ebs_peer_combine_q(ebs_peer_t peer, double *q, const uint8_t *free_m, const uint8_t *owned,
                       const double *pv, const double *prior, double *red, const int32_t *stop,
                       const double *dots, void *ws, void *stream);
/* The two-launch single-reduction PCG iteration: the matvec sweep with delta = the slab's
 * element energies sum_e u_e^T A_e u_e (summed over the ranks: u.mask(A u), u being 0 at
 * constrained nodes) and the put of [dots[0], delta, dots[2]] (dots[1] := delta) by its last
 * block -- no halo wait before the put; w's shared nodes keep their partials (pushed) --
 * then the update kernel that first completes w's shared nodes from the neighbours' pushes
 * (rank-ordered sums, masked; a grid barrier) and reduces the dots (_halo). */
int ebs_peer_matvec_sweep_put(ebs_plan_t plan, ebs_peer_t peer, const int32_t *chunks,
                              int64_t n_list, int64_t n_if_chunks, const double *pv, double *q,
                              const uint8_t *iface, double *dots, void *ws, void *stream);
int ebs_peer_cg1_update_halo(ebs_peer_t peer, int64_t n, double *cur, const double *prev,
                             const double *rr0, double tol, int32_t *ctl, const uint8_t *owned,
                             const uint8_t *free_m, const double *dinv, double *x, double *r,
                             double *u, double *w, double *p, double *s, double *next,
                             int32_t *nonfinite, void *ws, void *stream);
/* ebs_vec_cg1_update whose cur[0..2] are all-reduced on the device: every block waits for the
 * ranks' contributions (put by ebs_peer_combine_q with dots) and adds them in rank order; the
 * sums are stored in cur[0..2] and the reduced r.r once more in cur[4] (cur holds 5 doubles
 * here: [0..2] are later overwritten with partials when the slot is reused); at the first step
 * (ctl[2] == 0) the reduced r.r is also stored in rr0[0] (it is only known there).  No all-reduce launch per iteration. */
int ebs_peer_cg1_update(ebs_peer_t peer, int64_t n, double *cur, const double *prev,
                        const double *rr0, double tol, int32_t *ctl, const uint8_t *owned,
                        const double *dinv, double *x, double *r, double *u, const double *w,
                        double *p, double *s, double *next, int32_t *nonfinite, void *ws,
                        void *stream);

#ifdef __cplusplus
}
#endif
#endif /* EBS_H */
