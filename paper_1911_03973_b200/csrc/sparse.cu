// sparse.cu -- assembled CSR on the device (reference.py:25-39 assemble_sparse).
//
// Cross-check path only: the solver never uses it.  Row n of the
// assembled matrix collects, over the node's (j, e) slots in bincount order, the entries
// A_e[j, i, e] at column conn[i][e]; duplicates (same column) are summed in that order.
// Columns are sorted within a row.  Two passes over the plan's incidence: count the
// distinct columns of each row, then (after a scan) fill.
#include <cub/cub.cuh>

#include "ebs_internal.cuh"

namespace ebs {

constexpr int MAX_ROW_ENTRIES = 256;  // nb * valence; Kuhn 3D interior: 4*24 = 96

// Collect (col, val) of a node's slots, stable-sort by column, merge duplicates.
// Returns the number of distinct columns; writes them when cols/vals are non-null.
__device__ int row_entries(int nb, int64_t n_e, int64_t m, int c_m, int64_t row0, int lane,
                           int rowb, const int32_t *__restrict__ slot_ej,
                           const uint8_t *__restrict__ slot, const int32_t *__restrict__ conn,
                           int32_t *cbuf, double *vbuf, int32_t *cols, double *vals) {
    int cnt = 0;
    for (int k = 0; k < c_m; ++k) {
        const int64_t row = row0 + k;
        const int32_t ej = slot_ej[row * LANES + lane];
        const int64_t e = ej & ID_MASK;
        const double *ap = reinterpret_cast<const double *>(slot + row * rowb) + lane;
        for (int i = 0; i < nb; ++i) {
            if (cnt >= MAX_ROW_ENTRIES) return -1;
            cbuf[cnt] = conn[i * n_e + e];
            vbuf[cnt] = ap[i * LANES];
            ++cnt;
        }
    }
    // stable insertion sort by column
    for (int a = 1; a < cnt; ++a) {
        int32_t c = cbuf[a];
        double v = vbuf[a];
        int b = a - 1;
        while (b >= 0 && cbuf[b] > c) {
            cbuf[b + 1] = cbuf[b];
            vbuf[b + 1] = vbuf[b];
            --b;
        }
        cbuf[b + 1] = c;
        vbuf[b + 1] = v;
    }
    int out = 0;
    for (int a = 0; a < cnt; ++a) {
        if (out > 0 && cbuf[a] == cbuf[out - 1]) {
            vbuf[out - 1] = vbuf[out - 1] + vbuf[a];
        } else {
            cbuf[out] = cbuf[a];
            vbuf[out] = vbuf[a];
            ++out;
        }
    }
    if (cols)
        for (int a = 0; a < out; ++a) {
            cols[a] = cbuf[a];
            vals[a] = vbuf[a];
        }
    return out;
}

__global__ void k_csr_pass(int nb, int64_t n_n, int64_t n_e, int rowb,
                           const int32_t *__restrict__ rowbase, const int32_t *__restrict__ cnt,
                           const int32_t *__restrict__ slot_ej, const uint8_t *__restrict__ slot,
                           const int32_t *__restrict__ conn, const int32_t *__restrict__ old_of_new,
                           int64_t *__restrict__ row_nnz, const int64_t *__restrict__ crow,
                           int32_t *__restrict__ col, double *__restrict__ val, int32_t *bad) {
    int32_t cbuf[MAX_ROW_ENTRIES];
    double vbuf[MAX_ROW_ENTRIES];
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n_n;
         m += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = m / LANES;
        const int lane = (int)(m - c * LANES);
        const int64_t u = old_of_new[m];  // caller row
        int32_t *cols = crow ? col + crow[u] : nullptr;
        double *vals = crow ? val + crow[u] : nullptr;
        int nz = row_entries(nb, n_e, m, cnt[m], rowbase[c], lane, rowb, slot_ej, slot, conn, cbuf,
                             vbuf, cols, vals);
        if (nz < 0) {
            atomicOr(bad, 1);
            nz = 0;
        }
        if (row_nnz) row_nnz[u] = nz;
    }
}

}  // namespace ebs

using namespace ebs;

extern "C" {

int ebs_csr_nnz(ebs_plan_t plan, const int32_t *conn, int64_t *crow, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && conn && crow, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    cudaStream_t s = S(stream);
    const int64_t n = p->n_n;
    CU(cudaMemsetAsync(crow, 0, sizeof(int64_t) * (n + 1), s));
    CU(cudaMemsetAsync(p->flag, 0, sizeof(int32_t), s));
    if (n) {
        k_csr_pass<<<grid_for(n, 128), 128, 0, s>>>(p->nb, n, p->n_e, p->rowb, p->rowbase, p->cnt,
                                                    p->slot_ej, p->slot, conn, p->old_of_new,
                                                    crow + 1, nullptr, nullptr, nullptr, p->flag);
        LAUNCHED();
        // inclusive scan of the row counts into crow[1..n]
        size_t bytes = 0;
        CU(cub::DeviceScan::InclusiveSum(nullptr, bytes, crow + 1, crow + 1, n, s));
        void *tmp = dmalloc<char>(bytes);
        cudaError_t err = cub::DeviceScan::InclusiveSum(tmp, bytes, crow + 1, crow + 1, n, s);
        CU(cudaStreamSynchronize(s));
        cudaFree(tmp);
        CU(err);
        bump_launches(1);
    }
    int32_t bad = 0;
    CU(cudaMemcpyAsync(&bad, p->flag, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    EBS_REQUIRE(bad == 0, "a row has more than %d element entries", MAX_ROW_ENTRIES);
    EBS_CATCH
}

int ebs_csr_fill(ebs_plan_t plan, const int32_t *conn, const int64_t *crow, int32_t *col,
                 double *val, void *stream) {
    EBS_TRY
    EBS_REQUIRE(plan && conn && crow && col && val, "null argument");
    Plan *p = reinterpret_cast<Plan *>(plan);
    EBS_REQUIRE(p->has_A, "no operator loaded (ebs_plan_load)");
    const int64_t n = p->n_n;
    if (n) {
        k_csr_pass<<<grid_for(n, 128), 128, 0, S(stream)>>>(
            p->nb, n, p->n_e, p->rowb, p->rowbase, p->cnt, p->slot_ej, p->slot, conn, p->old_of_new,
            nullptr, crow, col, val, p->flag);
        LAUNCHED();
    }
    EBS_CATCH
}

}  // extern "C"
