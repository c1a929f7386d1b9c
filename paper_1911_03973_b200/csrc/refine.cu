// refine.cu -- uniform_refine (mesh.py:157-208) on the device.
//
// Red refinement of a triangle mesh with the reference's canonical renumbering, so a
// structured level-L mesh becomes build_unit_square_mesh(L + 1) bit for bit:
//   1. one midpoint per geometric edge: the 3 n_e edge slots (ab, bc, ca of every element,
//      slot t*n_e + e) keyed lo*n + hi, radix-sorted; distinct keys in ascending order are
//      the edges of np.unique(axis=0) (lexicographic (lo, hi) == ascending key), midpoint
//      0.5 * (x[lo] + x[hi]) appended after the old nodes;
//   2. nodes renumbered ascending in (y, x): two stable radix sorts (x, then y) of an
//      order-preserving 64-bit image of the coordinates (np.lexsort((x, y)); -0.0 == 0.0
//      as a comparison sort sees them);
//   3. children (a, ab, ca), (ab, b, bc), (ca, bc, c), (ab, bc, ca), child-major like the
//      reference's concatenation, mapped to the new numbering, each rotated to start at
//      its smallest node (orientation kept), rows sorted ascending (stable two-pass
//      radix sort on (c1, c2) then c0 -- np.lexsort((c2, c1, c0))).
// Every step is a coalesced elementwise kernel or a CUB radix sort / scan; no host loop
// over elements.  The node count is data dependent, so the call synchronises once.
#include <cub/cub.cuh>

#include "ebs_internal.cuh"

namespace ebs {

namespace {

__device__ __forceinline__ uint64_t order_key(double v) {
    if (v == 0.0) v = 0.0;  // -0.0 sorts with +0.0
    const uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_edge_keys(int64_t n_e, int64_t n_n, const int32_t *__restrict__ conn,
                            uint64_t *__restrict__ key, int32_t *__restrict__ slot) {
    const int64_t m = 3 * n_e;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / n_e, e = i - t * n_e;
        const int64_t a = conn[t * n_e + e], b = conn[((t + 1) % 3) * n_e + e];
        const int64_t lo = a < b ? a : b, hi = a < b ? b : a;
        key[i] = (uint64_t)(lo * n_n + hi);
        slot[i] = (int32_t)i;
    }
}

__global__ void k_edge_heads(int64_t m, const uint64_t *__restrict__ skey,
                             int32_t *__restrict__ head) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        head[i] = (i == 0 || skey[i] != skey[i - 1]) ? 1 : 0;
}

// edge id of every slot; the first slot of each edge writes its midpoint
__global__ void k_edge_mids(int64_t m, int64_t n_n, const uint64_t *__restrict__ skey,
                            const int32_t *__restrict__ sslot, const int32_t *__restrict__ scan,
                            const double *__restrict__ xy, int32_t *__restrict__ mid_of_slot,
                            double *__restrict__ all_xy) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t id = scan[i] - 1;
        mid_of_slot[sslot[i]] = id;
        if (i == 0 || skey[i] != skey[i - 1]) {
            const int64_t lo = (int64_t)(skey[i] / (uint64_t)n_n);
            const int64_t hi = (int64_t)(skey[i] % (uint64_t)n_n);
            const int64_t o = n_n + id;
            all_xy[2 * o] = 0.5 * (xy[2 * lo] + xy[2 * hi]);          // mesh.py:180
            all_xy[2 * o + 1] = 0.5 * (xy[2 * lo + 1] + xy[2 * hi + 1]);
        }
    }
}

__global__ void k_coord_keys(int64_t n, const double *__restrict__ all_xy,
                             const int32_t *__restrict__ idx, int comp,
                             uint64_t *__restrict__ key, int32_t *__restrict__ ids) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = idx ? idx[i] : i;
        key[i] = order_key(all_xy[2 * j + comp]);
        if (!idx) ids[i] = (int32_t)i;
    }
}

__global__ void k_renumber(int64_t n, const int32_t *__restrict__ order,
                           const double *__restrict__ all_xy, int32_t *__restrict__ rank,
                           double *__restrict__ xy_out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t j = order[i];
        rank[j] = (int32_t)i;
        xy_out[2 * i] = all_xy[2 * j];
        xy_out[2 * i + 1] = all_xy[2 * j + 1];
    }
}

// children in the reference's order (row q*n_e + e), new numbering, rotated to the
// smallest node; sort keys (c1 << 32 | c2) and the rows' c0
__global__ void k_children(int64_t n_e, int64_t n_n, const int32_t *__restrict__ conn,
                           const int32_t *__restrict__ mid, const int32_t *__restrict__ rank,
                           int32_t *__restrict__ c0, uint64_t *__restrict__ k12,
                           uint64_t *__restrict__ k12_sort, int32_t *__restrict__ rows) {
    const int64_t m = 4 * n_e;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = i / n_e, e = i - q * n_e;
        EBS_DCHECK(conn[e] >= 0 && conn[e] < n_n && conn[n_e + e] >= 0 &&
                   conn[n_e + e] < n_n && conn[2 * n_e + e] >= 0 && conn[2 * n_e + e] < n_n);
        EBS_DCHECK(mid[e] >= 0 && mid[n_e + e] >= 0 && mid[2 * n_e + e] >= 0);
        const int32_t a = rank[conn[e]], b = rank[conn[n_e + e]], c = rank[conn[2 * n_e + e]];
        const int32_t ab = rank[n_n + mid[e]], bc = rank[n_n + mid[n_e + e]],
                      ca = rank[n_n + mid[2 * n_e + e]];
        int32_t v0, v1, v2;
        if (q == 0) { v0 = a; v1 = ab; v2 = ca; }        // mesh.py:186-191
        else if (q == 1) { v0 = ab; v1 = b; v2 = bc; }
        else if (q == 2) { v0 = ca; v1 = bc; v2 = c; }
        else { v0 = ab; v1 = bc; v2 = ca; }
        // rotate to the first occurrence of the minimum (np.argmin), keep orientation
        int32_t r0 = v0, r1 = v1, r2 = v2;
        if (v1 < v0 && v1 <= v2) { r0 = v1; r1 = v2; r2 = v0; }
        else if (v2 < v0 && v2 < v1) { r0 = v2; r1 = v0; r2 = v1; }
        c0[i] = r0;
        k12[i] = k12_sort[i] = ((uint64_t)(uint32_t)r1 << 32) | (uint32_t)r2;
        rows[i] = (int32_t)i;
    }
}

__global__ void k_gather_c0(int64_t m, const int32_t *__restrict__ rows,
                            const int32_t *__restrict__ c0, uint32_t *__restrict__ key) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        key[i] = (uint32_t)c0[rows[i]];
}

__global__ void k_write_children(int64_t m, const int32_t *__restrict__ rows,
                                 const int32_t *__restrict__ c0,
                                 const uint64_t *__restrict__ k12, int32_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = rows[i];
        out[i] = c0[r];
        out[m + i] = (int32_t)(k12[r] >> 32);
        out[2 * m + i] = (int32_t)(k12[r] & 0xffffffffu);
    }
}

// device buffer freed on scope exit (every error path of ebs_refine_tri throws)
template <class T>
struct DevBuf {
    T *p = nullptr;
    DevBuf() = default;
    explicit DevBuf(int64_t n) { p = dmalloc<T>((size_t)(n > 0 ? n : 1)); }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// stable radix sort of (key, value) pairs, results back in k / v
template <class K>
void sort_pairs(DevBuf<K> &k, DevBuf<int32_t> &v, int64_t n, int end_bit, cudaStream_t s) {
    DevBuf<K> k2(n);
    DevBuf<int32_t> v2(n);
    size_t bytes = 0;
    CU(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k.p, k2.p, v.p, v2.p, (int)n, 0, end_bit,
                                       s));
    DevBuf<uint8_t> tmp((int64_t)bytes);
    CU(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, k.p, k2.p, v.p, v2.p, (int)n, 0, end_bit,
                                       s));
    CU(cudaStreamSynchronize(s));
    std::swap(k.p, k2.p);
    std::swap(v.p, v2.p);
}

int bits_for(uint64_t max_value) {
    int b = 1;
    while (b < 64 && (max_value >> b)) ++b;
    return b;
}

}  // namespace

}  // namespace ebs

using namespace ebs;

extern "C" {

int ebs_refine_tri(int64_t n_n, int64_t n_e, const double *coords, const int32_t *conn,
                   double *coords_out, int32_t *conn_out, int64_t *n_out, void *stream) {
    EBS_TRY
    EBS_REQUIRE(n_out, "null argument");
    *n_out = 0;
    EBS_REQUIRE(n_n >= 1 && n_e >= 1, "uniform_refine needs at least one node and element");
    EBS_REQUIRE(coords && conn && coords_out && conn_out, "null argument");
    EBS_REQUIRE(n_n + 3 * n_e < (1ll << 30) && 4 * n_e < (1ll << 30),
                "refined mesh too large (2^30 nodes / elements)");
    cudaStream_t s = S(stream);
    const int64_t m = 3 * n_e;
    // 1. edges and midpoints
    DevBuf<double> all_xy(2 * (n_n + m));
    CU(cudaMemcpyAsync(all_xy.p, coords, sizeof(double) * 2 * n_n, cudaMemcpyDeviceToDevice, s));
    DevBuf<uint64_t> ekey(m);
    DevBuf<int32_t> eslot(m);
    k_edge_keys<<<grid_for(m, 256), 256, 0, s>>>(n_e, n_n, conn, ekey.p, eslot.p);
    LAUNCHED();
    sort_pairs(ekey, eslot, m, bits_for((uint64_t)n_n * (uint64_t)n_n), s);
    DevBuf<int32_t> head(m);
    k_edge_heads<<<grid_for(m, 256), 256, 0, s>>>(m, ekey.p, head.p);
    LAUNCHED();
    {
        size_t bytes = 0;
        CU(cub::DeviceScan::InclusiveSum(nullptr, bytes, head.p, head.p, (int)m, s));
        DevBuf<uint8_t> tmp((int64_t)bytes);
        CU(cub::DeviceScan::InclusiveSum(tmp.p, bytes, head.p, head.p, (int)m, s));
        CU(cudaStreamSynchronize(s));
    }
    int32_t n_edges = 0;
    CU(cudaMemcpyAsync(&n_edges, head.p + m - 1, sizeof n_edges, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    DevBuf<int32_t> mid(m);
    k_edge_mids<<<grid_for(m, 256), 256, 0, s>>>(m, n_n, ekey.p, eslot.p, head.p, coords, mid.p,
                                                 all_xy.p);
    LAUNCHED();
    const int64_t N = n_n + n_edges;
    // 2. canonical numbering: stable sort by x, then by y  (np.lexsort((x, y)))
    DevBuf<uint64_t> xkey(N);
    DevBuf<int32_t> ids(N);
    k_coord_keys<<<grid_for(N, 256), 256, 0, s>>>(N, all_xy.p, nullptr, 0, xkey.p, ids.p);
    LAUNCHED();
    sort_pairs(xkey, ids, N, 64, s);
    k_coord_keys<<<grid_for(N, 256), 256, 0, s>>>(N, all_xy.p, ids.p, 1, xkey.p, nullptr);
    LAUNCHED();
    sort_pairs(xkey, ids, N, 64, s);
    DevBuf<int32_t> rank(N);
    k_renumber<<<grid_for(N, 256), 256, 0, s>>>(N, ids.p, all_xy.p, rank.p, coords_out);
    LAUNCHED();
    // 3. children, rotated to their smallest node, rows sorted (np.lexsort((c2, c1, c0)))
    const int64_t mc = 4 * n_e;
    DevBuf<int32_t> c0(mc), rows(mc);
    DevBuf<uint64_t> k12(mc), k12s(mc);  // k12 stays in row order, k12s is sorted
    k_children<<<grid_for(mc, 256), 256, 0, s>>>(n_e, n_n, conn, mid.p, rank.p, c0.p, k12.p,
                                                 k12s.p, rows.p);
    LAUNCHED();
    const int nb = bits_for((uint64_t)N);
    sort_pairs(k12s, rows, mc, 32 + nb, s);
    DevBuf<uint32_t> c0key(mc);
    k_gather_c0<<<grid_for(mc, 256), 256, 0, s>>>(mc, rows.p, c0.p, c0key.p);
    LAUNCHED();
    sort_pairs(c0key, rows, mc, nb, s);
    k_write_children<<<grid_for(mc, 256), 256, 0, s>>>(mc, rows.p, c0.p, k12.p, conn_out);
    LAUNCHED();
    CU(cudaStreamSynchronize(s));
    *n_out = N;
    EBS_CATCH
}

}  // extern "C"
