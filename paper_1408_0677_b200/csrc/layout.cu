// layout.cu -- planarity-preserving layout iteration on B200 (sm_100a), fp64.
//
// One Jacobi step (layout.py:266-286) = kd-tree build (bhtree.py:10-66) +
// Barnes-Hut traversal (_kernels.py:178-230) + one fused per-vertex kernel
// doing spring (layout.py:216-231), node-edge (layout.py:234-256), the
// temperature cap (layout.py:275-278), the limiting-line clamp
// (layout.py:119-184) and the double-buffered update (layout.py:280).
//
// kd-tree: the SHAPE (node ranges, preorder ids, left/right) depends only on
// (n, leaf) and is computed once on the host per plan.  Per step the device
// (1) radix-sorts point ids by x and by y (key = orderable fp64 bits, ties by
// id -- the "mid smallest under (coord, id)" restatement of argpartition),
// (2) walks the levels: every node's bbox is read off the ends of its x- and
// y-sorted runs, its split axis is argmax extent (ties -> x), the primary run
// splits at mid = count // 2 for free and the other run is stably partitioned
// with a scan, (3) sums centroids.  BH is warp-cooperative: a warp owns 32
// consecutive leaf-order points and walks the union of their DFS paths with a
// per-warp (node, lane-mask) stack, right child popped first as in the
// reference, so every lane accumulates its own interactions in the
// reference's order.
#include <utility>
#include <math.h>

#include <cooperative_groups.h>
#include <cub/cub.cuh>
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

#ifndef MDC_BH_SMALL_N
#define MDC_BH_SMALL_N 200000  // meshes up to this size split BH into 2^MDC_BH_CUT_SMALL tasks (else 16)
#endif
#ifndef MDC_BH_CUT_SMALL
#define MDC_BH_CUT_SMALL 6
#endif

namespace mdc {

// ---------------------------------------------------------------------------
// Host-side tree shape.
struct TreeShape {
    int64_t n = 0;
    int leaf = 32;
    std::vector<int32_t> lo, hi, left, right, depth;
    int max_depth = 0;  // depth of the deepest node
    // per level L (0..max_depth-1): frontier segments sorted by lo
    std::vector<int32_t> seg_off;                      // size levels+1
    std::vector<int32_t> seg_lo, seg_hi, seg_node, seg_split;
    // seg_of[L * n + k]: global frontier segment of sorted position k at level
    // L (data-independent: the tree shape depends only on n) -- one coalesced
    // load instead of a binary search per element per phase
    std::vector<int32_t> seg_of;
    // per depth L (0..max_depth): nodes created at that depth
    std::vector<int32_t> nd_off, nd_list;
    // leaves in left-to-right order and each node's contiguous leaf range
    std::vector<int32_t> leaves, leaf_lo, leaf_hi;
    // BH task split: the nodes at depth cut (left to right) each become an
    // independent traversal task; task_path holds their cut ancestors and
    // task_first marks the task that owns an ancestor's monopole.
    int cut = 0, ntask = 1;
    std::vector<int32_t> task_node, task_path, task_first;
};

static int32_t shape_build(TreeShape &t, int32_t lo, int32_t hi, int d) {
    int32_t id = (int32_t)t.lo.size();
    t.lo.push_back(lo);
    t.hi.push_back(hi);
    t.left.push_back(-1);
    t.right.push_back(-1);
    t.depth.push_back(d);
    if (d > t.max_depth) t.max_depth = d;
    if (hi - lo > t.leaf) {
        int32_t mid = (hi - lo) / 2;  // never 0 nor hi-lo when hi-lo > leaf >= 1
        int32_t l = shape_build(t, lo, lo + mid, d + 1);
        int32_t r = shape_build(t, lo + mid, hi, d + 1);
        t.left[id] = l;
        t.right[id] = r;
    }
    return id;
}

static void make_shape(TreeShape &t, int64_t n, int leaf) {
    t = TreeShape();
    t.n = n;
    t.leaf = leaf < 1 ? 1 : leaf;
    if (n <= 0) return;
    shape_build(t, 0, (int32_t)n, 0);
    int nn = (int)t.lo.size();
    // nodes by depth, in left-to-right (lo) order == preorder restricted to a depth
    t.nd_off.assign(t.max_depth + 2, 0);
    for (int i = 0; i < nn; ++i) t.nd_off[t.depth[i] + 1]++;
    for (int L = 0; L <= t.max_depth; ++L) t.nd_off[L + 1] += t.nd_off[L];
    t.nd_list.resize(nn);
    std::vector<int32_t> fill(t.nd_off.begin(), t.nd_off.end() - 1);
    for (int i = 0; i < nn; ++i) t.nd_list[fill[t.depth[i]]++] = i;  // preorder ids ascending == lo ascending per depth
    // leaves by lo; a node's leaves are the contiguous run with lo in [lo, hi)
    for (int i = 0; i < nn; ++i)
        if (t.left[i] < 0) t.leaves.push_back(i);
    std::sort(t.leaves.begin(), t.leaves.end(), [&](int32_t a, int32_t b) { return t.lo[a] < t.lo[b]; });
    t.leaf_lo.resize(nn);
    t.leaf_hi.resize(nn);
    {
        std::vector<int32_t> llo(t.leaves.size());
        for (size_t k = 0; k < t.leaves.size(); ++k) llo[k] = t.lo[t.leaves[k]];
        for (int i = 0; i < nn; ++i) {
            t.leaf_lo[i] = (int32_t)(std::lower_bound(llo.begin(), llo.end(), t.lo[i]) - llo.begin());
            t.leaf_hi[i] = (int32_t)(std::lower_bound(llo.begin(), llo.end(), t.hi[i]) - llo.begin());
        }
    }
    // BH task split at the deepest depth <= 4 above every leaf
    {
        int min_leaf_depth = t.max_depth;
        for (int i = 0; i < nn; ++i)
            if (t.left[i] < 0) min_leaf_depth = std::min(min_leaf_depth, t.depth[i]);
        // more, smaller tasks for small meshes: the walk is latency-bound and
        // ceil(n / 32) point-warps x 16 tasks do not fill the GPU below ~20k points
        const int want = n <= MDC_BH_SMALL_N ? MDC_BH_CUT_SMALL : 4;
        t.cut = std::min(want, min_leaf_depth);
        for (int i = 0; i < nn; ++i)
            if (t.depth[i] == t.cut) t.task_node.push_back(i);
        std::sort(t.task_node.begin(), t.task_node.end(), [&](int32_t a, int32_t b) { return t.lo[a] < t.lo[b]; });
        t.ntask = (int)t.task_node.size();
        std::vector<int32_t> parent(nn, -1);
        for (int i = 0; i < nn; ++i)
            if (t.left[i] >= 0) parent[t.left[i]] = parent[t.right[i]] = i;
        t.task_path.assign((size_t)t.ntask * (t.cut > 0 ? t.cut : 1), -1);
        t.task_first.assign(t.task_path.size(), 0);
        for (int k = 0; k < t.ntask; ++k) {
            int u = t.task_node[k];
            for (int dd = t.cut - 1; dd >= 0; --dd) {
                u = parent[u];
                t.task_path[(size_t)k * t.cut + dd] = u;
                // leftmost depth-cut descendant of u == the task whose node has lo == lo(u)
                t.task_first[(size_t)k * t.cut + dd] = t.lo[t.task_node[k]] == t.lo[u] ? 1 : 0;
            }
        }
    }
    // frontier per level L = nodes with depth == L, plus leaves with depth < L
    t.seg_off.assign(1, 0);
    for (int L = 0; L < t.max_depth; ++L) {
        std::vector<int32_t> segs;
        for (int i = 0; i < nn; ++i)
            if (t.depth[i] == L || (t.depth[i] < L && t.left[i] < 0)) segs.push_back(i);
        std::sort(segs.begin(), segs.end(), [&](int32_t a, int32_t b) { return t.lo[a] < t.lo[b]; });
        for (int32_t s : segs) {
            t.seg_lo.push_back(t.lo[s]);
            t.seg_hi.push_back(t.hi[s]);
            t.seg_node.push_back(s);
            t.seg_split.push_back(t.depth[s] == L && t.left[s] >= 0 ? 1 : 0);
        }
        t.seg_off.push_back((int32_t)t.seg_lo.size());
    }
    t.seg_of.resize((size_t)t.max_depth * (size_t)n);
    for (int L = 0; L < t.max_depth; ++L)
        for (int g = t.seg_off[L]; g < t.seg_off[L + 1]; ++g)
            for (int32_t k = t.seg_lo[g]; k < t.seg_hi[g]; ++k) t.seg_of[(size_t)L * n + k] = g;
}

// ---------------------------------------------------------------------------
// Workspace carving (all offsets 256-byte aligned).
struct Carver {
    char *base;
    size_t off = 0;
    template <typename T>
    T *take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

struct DevTree {
    int32_t *lo, *hi, *left, *right, *axis;
    int32_t *seg_lo, *seg_hi, *seg_node, *seg_split, *nd_list, *seg_of;
    int32_t *leaves, *leaf_lo, *leaf_hi;
    int32_t *seg_off, *nd_off;
    int32_t *task_node, *task_path, *task_first;
    int cut, ntask;
    double *part;       // ntask x n x 2 partial BH forces
    double4 *geo;       // per node: {bmin.x, bmin.y, bmax.x, bmax.y}, {com.x, com.y, size, mass}
    int4 *topo;         // per node: {lo, hi, left, right}
    double *com, *mass, *size, *bmin, *bmax;
    double *leaf_sum;   // 2 per leaf
    double *spts;       // points in leaf (perm) order, n x 2
    int nleaves;
};

struct Buffers {
    DevTree t;
    unsigned long long *kx, *ky, *kx_out, *ky_out;  // kx|ky and kx_out|ky_out are contiguous (2n keys)
    int32_t *ids, *xs[2], *ys[2];                    // ids: 2n sort values; xs[0]|ys[0] contiguous
    int32_t *runflag;                                // 2n, all-zero between steps
    int32_t *rank;                                   // 2n, all-zero between steps (small-n rank sort)
    int32_t *flag, *blocksum;
    double *pos_b, *bh;
    int32_t *ctr;
    void *cub_tmp;
    size_t cub_bytes;
    // bucket rank sort (MDC_SORT_BUCKET): 2B+1 bucket counts (all-zero between
    // steps) and starts, each element's bucket, ids in bucket order, and the
    // per-axis min/max order keys (reset to {~0, 0} between steps)
    int64_t nbucket;  // B per axis
    int32_t *bk_hist, *bk_start, *bk_of, *bk_slot;
    unsigned long long *bk_mm;
    unsigned long long *bk_split;  // sorted sample keys, 1024 per axis
};

constexpr int SCAN_BLOCK = 1024;

static size_t cub_sort_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (unsigned long long *)nullptr,
                                    (unsigned long long *)nullptr, (int32_t *)nullptr,
                                    (int32_t *)nullptr, (int)(2 * n), 0, 32);
    return bytes;
}

#ifndef MDC_SORT_BUCKET
#define MDC_SORT_BUCKET 1  // bucket rank sort (exact (coord, id) order) instead of the radix / count ranks + fixup
#endif
#ifndef MDC_SORT_BUCKET_OCC
#define MDC_SORT_BUCKET_OCC 2  // mean elements per bucket
#endif

// 1024 sample intervals x F linear sub-buckets per axis, ~OCC points per bucket
static int64_t sort_buckets(int64_t n) { return 1024 * std::max<int64_t>(1, n / (1024 * MDC_SORT_BUCKET_OCC)); }

static size_t cub_scan_bytes(int64_t items) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, (int32_t *)nullptr, (int32_t *)nullptr, (int)items);
    return bytes;
}

static size_t carve(Buffers &b, char *base, const TreeShape &s) {
    Carver c{base};
    int64_t n = s.n;
    size_t nn = s.lo.size() ? s.lo.size() : 1;
    size_t ns = s.seg_lo.size() ? s.seg_lo.size() : 1;
    b.t.lo = c.take<int32_t>(nn);
    b.t.hi = c.take<int32_t>(nn);
    b.t.left = c.take<int32_t>(nn);
    b.t.right = c.take<int32_t>(nn);
    b.t.axis = c.take<int32_t>(nn);
    b.t.nd_list = c.take<int32_t>(nn);
    b.t.seg_lo = c.take<int32_t>(ns);
    b.t.seg_hi = c.take<int32_t>(ns);
    b.t.seg_node = c.take<int32_t>(ns);
    b.t.seg_split = c.take<int32_t>(ns);
    b.t.seg_of = c.take<int32_t>(std::max<size_t>(1, (size_t)s.max_depth * (size_t)(n > 0 ? n : 1)));
    size_t nl = s.leaves.size() ? s.leaves.size() : 1;
    b.t.seg_off = c.take<int32_t>(s.seg_off.size() + 1);
    b.t.task_node = c.take<int32_t>(s.task_node.size() + 1);
    b.t.task_path = c.take<int32_t>(s.task_path.size() + 1);
    b.t.task_first = c.take<int32_t>(s.task_first.size() + 1);
    b.t.cut = s.cut;
    b.t.ntask = s.ntask;
    b.t.part = c.take<double>(2 * (size_t)s.ntask * (size_t)(n > 0 ? n : 1));
    b.t.geo = c.take<double4>(2 * nn);
    b.t.topo = c.take<int4>(nn);
    b.t.nd_off = c.take<int32_t>(s.nd_off.size() + 1);
    b.t.leaves = c.take<int32_t>(nl);
    b.t.leaf_lo = c.take<int32_t>(nn);
    b.t.leaf_hi = c.take<int32_t>(nn);
    b.t.leaf_sum = c.take<double>(2 * nl);
    b.t.spts = c.take<double>(2 * (size_t)(n > 0 ? n : 1));
    b.t.nleaves = (int)s.leaves.size();
    b.t.com = c.take<double>(2 * nn);
    b.t.mass = c.take<double>(nn);
    b.t.size = c.take<double>(nn);
    b.t.bmin = c.take<double>(2 * nn);
    b.t.bmax = c.take<double>(2 * nn);
    b.kx = c.take<unsigned long long>(n);
    b.ky = c.take<unsigned long long>(n);
    b.kx_out = c.take<unsigned long long>(n);
    b.ky_out = c.take<unsigned long long>(n);
    b.ids = c.take<int32_t>(2 * n);
    b.xs[0] = c.take<int32_t>(2 * n);
    b.ys[0] = b.xs[0] + n;
    b.xs[1] = c.take<int32_t>(n);
    b.ys[1] = c.take<int32_t>(n);
    b.runflag = c.take<int32_t>(2 * n);
    b.rank = c.take<int32_t>(2 * n);
    b.flag = c.take<int32_t>(n);
    b.blocksum = c.take<int32_t>(std::max<int64_t>((n + SCAN_BLOCK - 1) / SCAN_BLOCK + 1, 1024));
    b.pos_b = c.take<double>(2 * n);
    b.bh = c.take<double>(2 * n);
    b.ctr = c.take<int32_t>(4);
    b.nbucket = sort_buckets(n);
    b.bk_hist = c.take<int32_t>(2 * b.nbucket + 1);
    b.bk_start = c.take<int32_t>(2 * b.nbucket + 1);
    b.bk_of = c.take<int32_t>(2 * n);
    b.bk_slot = c.take<int32_t>(2 * n);
    b.bk_mm = c.take<unsigned long long>(4);
    b.bk_split = c.take<unsigned long long>(2 * 1024);
    b.cub_bytes = std::max(cub_sort_bytes(n), cub_scan_bytes(2 * b.nbucket + 1));
    b.cub_tmp = c.take<char>(b.cub_bytes);
    return c.off + 256;
}

#ifndef MDC_LAYOUT_PDL
#define MDC_LAYOUT_PDL 1  // step kernels launch as programmatic dependents (launch overlaps the predecessor's tail)
#endif
// First statement of every step kernel: under programmatic dependent launch
// the kernel may start before its predecessor finishes and must wait here
// before touching its outputs (a no-op for ordinary launches).
__device__ __forceinline__ void pdl_wait() {
#if MDC_LAYOUT_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

// ---------------------------------------------------------------------------
// Kernels: tree build.

__device__ __forceinline__ unsigned long long order_key(double x) {
    if (x == 0.0) x = 0.0;  // -0.0 ties with +0.0 as in numpy comparisons
    unsigned long long b = (unsigned long long)__double_as_longlong(x);
    return (b & 0x8000000000000000ULL) ? ~b : (b | 0x8000000000000000ULL);
}

// Both axes in ONE radix sort of 2n 32-bit keys {axis bit, top 31
// order-preserving bits of (float)coord}: 4 digit passes instead of 2 x 8
// for fp64 keys.  The
// float rounding is monotone, so the result is already ordered by the exact
// (coord, id) key except inside runs of equal float keys (distinct doubles
// within one float ulp); those runs are detected and re-sorted by the exact
// key below.  Stable sort + ids in input order = ties by id.
__device__ __forceinline__ uint32_t order_key32(double x) {
    float f = (float)x;
    if (f == 0.0f) f = 0.0f;
    uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void keys_kernel(const double *pts, int64_t n, unsigned long long *keys, int32_t *ids) {
    pdl_wait();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 2 * n) return;
    const int axis = i >= n;
    const int64_t j = i - axis * n;
    keys[i] = ((unsigned long long)axis << 31) | (order_key32(pts[2 * j + axis]) >> 1);
    ids[i] = (int32_t)j;
}

// exact order (coord, id) of two ids on one axis
__device__ __forceinline__ bool exact_less(const double *pts, int axis, int32_t a, int32_t b) {
    unsigned long long ka = order_key(pts[2 * a + axis]), kb = order_key(pts[2 * b + axis]);
    return ka < kb || (ka == kb && a < b);
}

// Flag the start of every run of equal float keys that is NOT already in
// exact order (exact-tie runs stay untouched: they are sorted by id).
__global__ void run_mark_kernel(int64_t n, const unsigned long long *keys, const int32_t *ids, const double *pts,
                                int32_t *runflag) {
    pdl_wait();
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (k >= 2 * n || keys[k] != keys[k - 1]) return;
    const int axis = (int)(keys[k] >> 31);
    if (!exact_less(pts, axis, ids[k], ids[k - 1])) return;
    int64_t s0 = k - 1;
    while (s0 > 0 && keys[s0 - 1] == keys[k]) --s0;
    runflag[s0] = 1;
}

// Insertion-sort each flagged run by the exact key (runs are a few elements:
// distinct doubles sharing one float), then clear its flag.
__global__ void run_sort_kernel(int64_t n, const unsigned long long *keys, int32_t *ids, const double *pts,
                                int32_t *runflag) {
    pdl_wait();
    int64_t s0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s0 >= 2 * n || !runflag[s0]) return;
    runflag[s0] = 0;
    const unsigned long long key = keys[s0];
    const int axis = (int)(key >> 31);
    int64_t e = s0 + 1;
    while (e < 2 * n && keys[e] == key) ++e;
    int32_t *r = ids + s0;
    const int64_t len = e - s0;
    if (len <= 64) {
        for (int64_t i = 1; i < len; ++i) {
            const int32_t v = r[i];
            int64_t j = i - 1;
            while (j >= 0 && exact_less(pts, axis, v, r[j])) {
                r[j + 1] = r[j];
                --j;
            }
            r[j + 1] = v;
        }
        return;
    }
    // pathological long run (many distinct doubles inside one float ulp):
    // heap sort keeps it O(L log L)
    auto sift = [&](int64_t root, int64_t end) {
        while (2 * root + 1 < end) {
            int64_t child = 2 * root + 1;
            if (child + 1 < end && exact_less(pts, axis, r[child], r[child + 1])) ++child;
            if (!exact_less(pts, axis, r[root], r[child])) return;
            const int32_t t = r[root];
            r[root] = r[child];
            r[child] = t;
            root = child;
        }
    };
    for (int64_t i = len / 2 - 1; i >= 0; --i) sift(i, len);
    for (int64_t end = len - 1; end > 0; --end) {
        const int32_t t = r[0];
        r[0] = r[end];
        r[end] = t;
        sift(0, end);
    }
}

// Small n: the same 32-bit keys, sorted by counting ranks instead of radix
// passes -- rank(i) = #{j : (k_j, j) < (k_i, i)}, split as k_j <= k_i over
// j < i plus k_j < k_i over j > i (the stable sort's tie order).  grid.z
// splits the j range (partial ranks added atomically: integers, so the
// result is order-independent), then a scatter writes the sorted keys / ids
// exactly as the radix sort would, and the same run fixup follows.
#ifndef MDC_RANK_SORT_MAX
#define MDC_RANK_SORT_MAX 16384  // O(n^2) work: beats the radix passes only for small n
#endif
constexpr int RANK_THREADS = 128;
constexpr int RANK_TILE = 1024;

__device__ __forceinline__ uint32_t axis_key32(const double *pts, int64_t j, int axis) {
    return ((uint32_t)axis << 31) | (order_key32(pts[2 * j + axis]) >> 1);
}

__global__ void __launch_bounds__(RANK_THREADS) rank_count_kernel(const double *pts, int n, int span,
                                                                  int32_t *rank) {
    pdl_wait();
    __shared__ uint32_t tile[RANK_TILE];
    const int axis = blockIdx.y;
    const int i = blockIdx.x * RANK_THREADS + threadIdx.x;
    const uint32_t ki = i < n ? axis_key32(pts, i, axis) : 0u;
    const int j0 = blockIdx.z * span, j1 = min(n, j0 + span);
    int r = 0;
    for (int t0 = j0; t0 < j1; t0 += RANK_TILE) {
        const int cnt = min(RANK_TILE, j1 - t0);
        __syncthreads();
        for (int e = threadIdx.x; e < cnt; e += RANK_THREADS) tile[e] = axis_key32(pts, t0 + e, axis);
        __syncthreads();
        const int m = min(max(i - t0, 0), cnt);  // tile entries with j < i
        for (int e = 0; e < m; ++e) r += tile[e] <= ki;
        for (int e = m; e < cnt; ++e) r += tile[e] < ki;
    }
    // the self comparison (j == i) counted 0: k_i < k_i is false
    if (i < n && r) atomicAdd(rank + (int64_t)axis * n + i, r);
}

__global__ void rank_scatter_kernel(const double *pts, int64_t n, int32_t *rank, unsigned long long *keys_out,
                                    int32_t *ids_out) {
    pdl_wait();
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= 2 * n) return;
    const int axis = k >= n;
    const int64_t i = k - axis * n;
    const int64_t dst = axis * n + rank[k];
    keys_out[dst] = axis_key32(pts, i, axis);
    ids_out[dst] = (int32_t)i;
    rank[k] = 0;  // ready for the next step
}

// Bucket rank sort: the exact (coord, id) order of both axes without radix
// passes or a float-key fixup.  Two-level buckets, non-decreasing in x under
// the exact key: the interval between consecutive keys of a regular sample
// (S = 1024, sorted per axis), then F ~ n / 2S linear sub-buckets inside it
// (correctly rounded monotone operations; the end intervals run to the axis
// min / max).  The sample adapts the coarse level to the data's density, so
// outliers or clusters do not squeeze the bulk into a few buckets, and the
// linear level leaves ~2 points per bucket.  An element's final slot is its
// bucket's start plus its rank among the bucket's members under the exact
// (coord, id) key (a bucket of m points costs m^2 compares: exact ties
// concentrate -- slower, never wrong).
__device__ __forceinline__ double key_to_double(unsigned long long k) {
    return __longlong_as_double((long long)((k & 0x8000000000000000ULL) ? (k & ~0x8000000000000000ULL) : ~k));
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, (unsigned long long)__shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, (unsigned long long)__shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

constexpr int BK_THREADS = 256;

__device__ __forceinline__ void bucket_minmax(const double *pts, int64_t n, unsigned long long *mm, int blk,
                                              int nblk, unsigned long long *s_mm) {
    if (threadIdx.x < 4) s_mm[threadIdx.x] = (threadIdx.x & 1) ? 0ULL : ~0ULL;
    __syncthreads();
    unsigned long long lo[2] = {~0ULL, ~0ULL}, hi[2] = {0ULL, 0ULL};
    for (int64_t i = (int64_t)blk * blockDim.x + threadIdx.x; i < n; i += (int64_t)nblk * blockDim.x) {
        const double2 p = reinterpret_cast<const double2 *>(pts)[i];
        const unsigned long long kx = order_key(p.x), ky = order_key(p.y);
        lo[0] = min(lo[0], kx);
        hi[0] = max(hi[0], kx);
        lo[1] = min(lo[1], ky);
        hi[1] = max(hi[1], ky);
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {
        lo[a] = warp_min_u64(lo[a]);
        hi[a] = warp_max_u64(hi[a]);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&s_mm[0], lo[0]);
        atomicMax(&s_mm[1], hi[0]);
        atomicMin(&s_mm[2], lo[1]);
        atomicMax(&s_mm[3], hi[1]);
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        if (threadIdx.x & 1)
            atomicMax(&mm[threadIdx.x], s_mm[threadIdx.x]);
        else
            atomicMin(&mm[threadIdx.x], s_mm[threadIdx.x]);
    }
}

// Sample splitters (one CTA per axis): S = 1024 order keys at ids s n / S,
// bitonic-sorted (shared memory for partner distances >= 32, shuffles below).
constexpr int BK_SAMPLE = 1024;
__device__ __forceinline__ void bucket_sample(const double *pts, int64_t n, int axis, unsigned long long *spl,
                                              unsigned long long *sk) {
    const int q = threadIdx.x;
    unsigned long long v = order_key(pts[2 * ((int64_t)q * n / BK_SAMPLE) + axis]);
    for (int k = 2; k <= BK_SAMPLE; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            unsigned long long w;
            if (j >= 32) {
                sk[q] = v;
                __syncthreads();
                w = sk[q ^ j];
                __syncthreads();
            } else {
                w = __shfl_xor_sync(0xffffffffu, v, j);
            }
            const bool lower = (q & j) == 0, up = (q & k) == 0;
            v = (lower == up) ? min(v, w) : max(v, w);
        }
    spl[axis * BK_SAMPLE + q] = v;
}

// One launch for both inputs of the bucket map: CTAs 0, 1 sort the x / y
// samples, the rest reduce the per-axis min / max order keys.
// nsample = 0: keep the previous splitters (any sorted splitters give the
// exact order; they only balance the buckets -- within a captured run of
// steps the points move little between resamplings).
__global__ void __launch_bounds__(BK_SAMPLE) bucket_prep_kernel(const double *pts, int64_t n,
                                                                unsigned long long *mm, unsigned long long *spl,
                                                                int nsample) {
    pdl_wait();
    __shared__ unsigned long long sk[BK_SAMPLE];
    if ((int)blockIdx.x < nsample) {
        bucket_sample(pts, n, blockIdx.x, spl, sk);
        return;
    }
    bucket_minmax(pts, n, mm, blockIdx.x - nsample, gridDim.x - nsample, sk);
}

// Bucket = (sample interval c, linear sub-bucket): c = #{j in [1, S) :
// splitter_j <= x}; inside [lo_c, hi_c) (the two end intervals reach the
// axis min / max) F sub-buckets floor(F (x - lo_c)/(hi_c - lo_c)).
constexpr int BK_COUNT_THREADS = 1024;  // the splitter table (16 KB) is staged once per CTA
__global__ void __launch_bounds__(BK_COUNT_THREADS) bucket_count_kernel(const double *pts, int64_t n, int F,
                                                                  const unsigned long long *mm,
                                                                  const unsigned long long *spl, int32_t *hist,
                                                                  int32_t *bk_of) {
    pdl_wait();
    __shared__ unsigned long long s_spl[2 * BK_SAMPLE];
    for (int q = threadIdx.x; q < 2 * BK_SAMPLE; q += BK_COUNT_THREADS) s_spl[q] = spl[q];
    __syncthreads();
    const int64_t e = (int64_t)blockIdx.x * BK_COUNT_THREADS + threadIdx.x;
    if (e >= 2 * n) return;
    const int axis = e >= n;
    const double x = pts[2 * (e - axis * n) + axis];
    const unsigned long long k = order_key(x);
    const unsigned long long *sp = s_spl + axis * BK_SAMPLE;
    int lo = 1, hi = BK_SAMPLE;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (sp[mid] <= k)
            lo = mid + 1;
        else
            hi = mid;
    }
    const int c = lo - 1;
    const double a = key_to_double(c == 0 ? mm[2 * axis] : sp[c]);
    const double b = key_to_double(c == BK_SAMPLE - 1 ? mm[2 * axis + 1] : sp[c + 1]);
    int fine = 0;
    if (b > a) {
        const double t = __dmul_rn(__ddiv_rn(__dsub_rn(x, a), __dsub_rn(b, a)), (double)F);
        fine = (int)fmin(fmax(t, 0.0), (double)(F - 1));
    }
    const int g = (axis * BK_SAMPLE + c) * F + fine;
    bk_of[e] = g;
    atomicAdd(hist + g, 1);
}

// Place every element in its bucket (any order inside it); the atomic
// decrements leave the counts at zero for the next step.
__global__ void __launch_bounds__(BK_THREADS) bucket_scatter_kernel(int64_t n, const int32_t *bk_of,
                                                                    const int32_t *start, int32_t *hist,
                                                                    int32_t *slot, unsigned long long *mm) {
    pdl_wait();
    const int64_t e = (int64_t)blockIdx.x * BK_THREADS + threadIdx.x;
    if (e == 0) {
        mm[0] = mm[2] = ~0ULL;
        mm[1] = mm[3] = 0ULL;
    }
    if (e >= 2 * n) return;
    const int g = bk_of[e];
    const int pos = start[g] + atomicSub(hist + g, 1) - 1;
    slot[pos] = (int32_t)e;  // axis * n + id
}

// Final slot = bucket start + rank under the exact (coord, id) key among the
// bucket's members; ids land in xs0 (x run, then y run) as the sort writes them.
__global__ void __launch_bounds__(BK_THREADS) bucket_rank_kernel(const double *pts, int64_t n,
                                                                 const int32_t *bk_of, const int32_t *start,
                                                                 const int32_t *slot, int32_t *xs0) {
    pdl_wait();
    const int64_t p = (int64_t)blockIdx.x * BK_THREADS + threadIdx.x;
    if (p >= 2 * n) return;
    const int e = slot[p];
    const int axis = e >= n;
    const int id = e - axis * (int)n;
    const int g = bk_of[e];
    const int s0 = start[g], s1 = start[g + 1];
    const unsigned long long k = order_key(pts[2 * id + axis]);
    int r = 0;
    const int off = axis * (int)n;
    auto less = [&](int j) {
        const unsigned long long kj = order_key(pts[2 * j + axis]);
        return (int)((kj < k) || (kj == k && j < id));
    };
    int q = s0;
    // 8 members per round: independent loads in flight (a large bucket is a
    // long latency chain otherwise)
    for (; q + 8 <= s1; q += 8) {
        int j[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) j[u] = slot[q + u] - off;
#pragma unroll
        for (int u = 0; u < 8; ++u) r += less(j[u]);
    }
    for (; q < s1; ++q) r += less(slot[q] - off);
    xs0[s0 + r] = id;
}

// ---------------------------------------------------------------------------
// The whole level walk as ONE cooperative kernel (grid-wide syncs between
// phases) instead of ~6 launches per level: per level
//   phase 1  node stats for this depth; left-flags through each splitting
//            segment's primary run
//   phase 2  per-block counts of the other run's flags        (grid sync)
//   phase 3  global exclusive prefix of those flags           (grid sync)
//   phase 4  stable partition of the other run, copy the rest (grid sync)
// then leaf sums + leaf-order gather, and centroids.
namespace cg = cooperative_groups;
#ifndef MDC_BUILD_THREADS
#define MDC_BUILD_THREADS 1024
#endif
constexpr int BUILD_THREADS = MDC_BUILD_THREADS;  // cooperative (multi-CTA) walk
constexpr int BUILD_SINGLE_THREADS = 1024;
constexpr int64_t BUILD_SINGLE_MAX = 2048;  // one CTA walks the tree up to this n (A/B: slower at 10k)
// Mid-size n: ONE thread-block cluster walks the tree; its per-phase barrier
// is barrier.cluster (hardware, ~sub-microsecond) instead of a grid-wide
// cooperative sync across hundreds of CTAs (~4 us per phase measured).
#ifndef MDC_BUILD_CLUSTER
#define MDC_BUILD_CLUSTER 16
#endif
constexpr int BUILD_CLUSTER = MDC_BUILD_CLUSTER;
constexpr int BUILD_CLUSTER_THREADS = 1024;
#ifndef MDC_BUILD_CLUSTER_MAX
#define MDC_BUILD_CLUSTER_MAX 16384
#endif
constexpr int64_t BUILD_CLUSTER_MAX = MDC_BUILD_CLUSTER_MAX;
#ifndef MDC_BUILD_CLUSTER_SUB
#define MDC_BUILD_CLUSTER_SUB 1  // cluster walk only down to the subtree hand-off level
#endif
enum BuildMode { BUILD_ONE_CTA = 0, BUILD_ONE_CLUSTER = 1, BUILD_GRID = 2 };

struct BuildArgs {
    const double *pts;
    int64_t n;
    DevTree t;
    int max_depth, nnodes;
    int32_t *xs0, *xs1, *ys0, *ys1;
    int32_t *flag, *oflag, *prefix, *blocksum;
    int l_end = 1 << 30;  // walk levels [0, l_end) only (the rest: build_subtree_kernel)
};

// Node stats: bbox from the ends of the node's sorted runs (exact min/max),
// size = hypot(extent) (bhtree.py:47-48), mass = count, split axis
// argmax(extent) with ties -> x (bhtree.py:56).
__device__ __forceinline__ void stats_for(const BuildArgs &a, int node, const int32_t *X, const int32_t *Y) {
    const DevTree &t = a.t;
    int lo = t.lo[node], hi = t.hi[node];
    double xmin = a.pts[2 * X[lo]], xmax = a.pts[2 * X[hi - 1]];
    double ymin = a.pts[2 * Y[lo] + 1], ymax = a.pts[2 * Y[hi - 1] + 1];
    t.bmin[2 * node] = xmin;
    t.bmin[2 * node + 1] = ymin;
    t.bmax[2 * node] = xmax;
    t.bmax[2 * node + 1] = ymax;
    double ex = xmax - xmin, ey = ymax - ymin;
    t.size[node] = hypot(ex, ey);
    t.mass[node] = (double)(hi - lo);
    t.axis[node] = ey > ex ? 1 : 0;
}

// Centroid (ordered sum of the node's leaf sums / count) and the packed node
// records, warp per node over nodes [gw, nnodes) step nw.
__device__ __forceinline__ void node_centroids(const BuildArgs &a, int64_t gw, int64_t nw) {
    const DevTree &t = a.t;
    const int lane = threadIdx.x & 31;
    for (int64_t w = gw; w < a.nnodes; w += nw) {
        int l0 = t.leaf_lo[w], l1 = t.leaf_hi[w];
        double sx = 0.0, sy = 0.0;
        for (int k = l0 + lane; k < l1; k += 32) {
            sx += t.leaf_sum[2 * k];
            sy += t.leaf_sum[2 * k + 1];
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sx += __shfl_xor_sync(0xffffffffu, sx, o);
            sy += __shfl_xor_sync(0xffffffffu, sy, o);
        }
        if (lane == 0) {
            double m = (double)(t.hi[w] - t.lo[w]);
            double cx = sx / m, cy = sy / m;
            t.com[2 * w] = cx;
            t.com[2 * w + 1] = cy;
            t.geo[2 * w] = make_double4(t.bmin[2 * w], t.bmin[2 * w + 1], t.bmax[2 * w], t.bmax[2 * w + 1]);
            t.geo[2 * w + 1] = make_double4(cx, cy, t.size[w], t.mass[w]);
            t.topo[w] = make_int4(t.lo[w], t.hi[w], t.left[w], t.right[w]);
        }
    }
}

// The per-level walk (membership = the reference's argpartition under the
// (coord, id) order): phase 1 node stats + left flags through each splitting
// node's primary run, phase 2/3 flag prefix over the other run, phase 4 stable
// partition.  MODE picks the barrier between phases: one CTA (small n,
// __syncthreads), one thread-block cluster (barrier.cluster), or the whole
// cooperative grid (grid.sync); the code is otherwise identical.
template <int NTH, int MODE>
__device__ __forceinline__ void build_levels_body(const BuildArgs &a) {
    constexpr int BUILD_THREADS = NTH;
    typedef cub::BlockReduce<int, BUILD_THREADS> BR;
    typedef cub::BlockScan<int, BUILD_THREADS> BS;
    struct Sync {
        __device__ void sync() const {
            if constexpr (MODE == BUILD_ONE_CTA) {
                __syncthreads();
            } else if constexpr (MODE == BUILD_ONE_CLUSTER) {
                // release/acquire at cluster scope: global-memory writes of
                // every CTA in the cluster are visible after the barrier
                asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
            } else {
                cg::this_grid().sync();
            }
        }
    } grid;
    __shared__ union {
        typename BR::TempStorage r;
        typename BS::TempStorage s;
    } tmp;
    __shared__ int s_carry;
    const DevTree &t = a.t;
    const int64_t n = a.n;
    // one CTA walks alone even when launched inside a larger grid (the
    // persistent small-mesh step runs it on CTA 0 of its cluster)
    const int G = MODE == BUILD_ONE_CTA ? 1 : (int)gridDim.x, tid = threadIdx.x;
    const int bid = MODE == BUILD_ONE_CTA ? 0 : (int)blockIdx.x;
    const int64_t gtid = (int64_t)bid * BUILD_THREADS + tid, gsz = (int64_t)G * BUILD_THREADS;
    const int64_t chunk = (((n + G - 1) / G) + BUILD_THREADS - 1) / BUILD_THREADS * BUILD_THREADS;
    const int64_t c_lo = min((int64_t)bid * chunk, n), c_hi = min(c_lo + chunk, n);
    int32_t *X = a.xs0, *Y = a.ys0, *Xn = a.xs1, *Yn = a.ys1;
    for (int L = 0; L <= a.max_depth; ++L) {
        if (L >= a.l_end) return;  // deeper levels and the tail run per subtree
        // ---- phase 1
        const int d0 = t.nd_off[L], dn = t.nd_off[L + 1] - d0;
        for (int64_t e = gtid; e < dn; e += gsz) stats_for(a, t.nd_list[d0 + e], X, Y);
        if (L == a.max_depth) break;
        // frontier segments of level L: t.seg_of[L * n + k] (global indices)
        for (int64_t k = gtid; k < n; k += gsz) {
            int s = t.seg_of[(int64_t)L * n + k];
            if (!t.seg_split[s]) continue;
            int lo = t.seg_lo[s], hi = t.seg_hi[s];
            double ex = a.pts[2 * X[hi - 1]] - a.pts[2 * X[lo]];
            double ey = a.pts[2 * Y[hi - 1] + 1] - a.pts[2 * Y[lo] + 1];
            const int32_t *P = ey > ex ? Y : X;
            a.flag[P[k]] = (k - lo) < (hi - lo) / 2 ? 1 : 0;
        }
        grid.sync();
        // ---- phase 2: other-run flags, per-block counts over this block's chunk
        int cnt = 0;
        for (int64_t k = c_lo + tid; k < c_hi; k += BUILD_THREADS) {
            int s = t.seg_of[(int64_t)L * n + k];
            int v = 0;
            if (t.seg_split[s]) {
                const int32_t *O = t.axis[t.seg_node[s]] ? X : Y;
                v = a.flag[O[k]];
            }
            a.oflag[k] = v;
            cnt += v;
        }
        cnt = BR(tmp.r).Sum(cnt);
        if (tid == 0) a.blocksum[bid] = cnt;
        grid.sync();
        // ---- phase 3: global exclusive prefix
        int base = 0;
        for (int b = tid; b < bid; b += BUILD_THREADS) base += a.blocksum[b];
        __syncthreads();
        base = BR(tmp.r).Sum(base);
        if (tid == 0) s_carry = base;
        __syncthreads();
        for (int64_t b0 = c_lo; b0 < c_hi; b0 += BUILD_THREADS) {
            int64_t k = b0 + tid;
            int v = k < c_hi ? a.oflag[k] : 0, ex, agg;
            BS(tmp.s).ExclusiveSum(v, ex, agg);
            if (k < c_hi) a.prefix[k] = s_carry + ex;
            __syncthreads();
            if (tid == 0) s_carry += agg;
            __syncthreads();
        }
        grid.sync();
        // ---- phase 4: stable partition
        for (int64_t k = gtid; k < n; k += gsz) {
            int s = t.seg_of[(int64_t)L * n + k];
            if (!t.seg_split[s]) {
                Xn[k] = X[k];
                Yn[k] = Y[k];
                continue;
            }
            int lo = t.seg_lo[s], hi = t.seg_hi[s];
            int mid = (hi - lo) / 2;
            int ax = t.axis[t.seg_node[s]];
            const int32_t *P = ax ? Y : X;
            const int32_t *O = ax ? X : Y;
            int32_t *Pn = ax ? Yn : Xn;
            int32_t *On = ax ? Xn : Yn;
            Pn[k] = P[k];
            int id = O[k];
            int left_before = a.prefix[k] - a.prefix[lo];
            int dest = a.flag[id] ? lo + left_before : lo + mid + ((int)k - lo - left_before);
            On[dest] = id;
        }
        grid.sync();
        int32_t *tx = X, *ty = Y;
        X = Xn;
        Y = Yn;
        Xn = tx;
        Yn = ty;
    }
    // leaf sums + gather into leaf order (warp per leaf)
    const int lane = tid & 31;
    const int64_t gw = gtid >> 5, nw = gsz >> 5;
    for (int64_t w = gw; w < t.nleaves; w += nw) {
        int node = t.leaves[w];
        int lo = t.lo[node], hi = t.hi[node];
        double sx = 0.0, sy = 0.0;
        for (int k = lo + lane; k < hi; k += 32) {
            double2 p = reinterpret_cast<const double2 *>(a.pts)[X[k]];
            reinterpret_cast<double2 *>(t.spts)[k] = p;
            sx += p.x;
            sy += p.y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sx += __shfl_xor_sync(0xffffffffu, sx, o);
            sy += __shfl_xor_sync(0xffffffffu, sy, o);
        }
        if (lane == 0) {
            t.leaf_sum[2 * w] = sx;
            t.leaf_sum[2 * w + 1] = sy;
        }
    }
    grid.sync();
    node_centroids(a, gw, nw);
}

template <int NTH, int MODE>
__global__ void __launch_bounds__(NTH) build_levels_kernel(BuildArgs a) {
    pdl_wait();
    build_levels_body<NTH, MODE>(a);
}

// Deep levels of the large-n walk: once every frontier segment is small,
// each segment's subtree is independent (its points occupy the same [lo, hi)
// in both axis runs), so one CTA finishes the walk for one segment with block
// barriers, its working set L1-resident -- instead of paying a grid-wide
// barrier and L2 latency per phase for levels with tiny segments.  Same
// phases, same arithmetic, same ping-pong parity as build_levels_kernel.
#ifndef MDC_SUBTREE_THREADS
#define MDC_SUBTREE_THREADS 1024
#endif
constexpr int SUBTREE_THREADS = MDC_SUBTREE_THREADS;
#ifndef MDC_SUBTREE_MAX
#define MDC_SUBTREE_MAX 1024
#endif
constexpr int SUBTREE_MAX = MDC_SUBTREE_MAX;  // largest segment a CTA takes over (0: off)

__device__ __forceinline__ int first_node_at_or_after(const DevTree &t, int L, int lo) {
    int a = t.nd_off[L], b = t.nd_off[L + 1];  // nd_list[a, b): depth-L nodes sorted by lo
    while (a < b) {
        int m = (a + b) >> 1;
        if (t.lo[t.nd_list[m]] < lo)
            a = m + 1;
        else
            b = m;
    }
    return a;
}

__global__ void __launch_bounds__(SUBTREE_THREADS) build_subtree_kernel(BuildArgs a, int L0) {
    pdl_wait();
    typedef cub::BlockScan<int, SUBTREE_THREADS> BS;
    __shared__ typename BS::TempStorage scan_tmp;
    __shared__ int s_carry;
    const DevTree &t = a.t;
    const int64_t n = a.n;
    const int tid = threadIdx.x;
    const int g = t.seg_off[L0] + blockIdx.x;
    const int seg_lo = t.seg_lo[g], seg_hi = t.seg_hi[g];
    int32_t *X = (L0 & 1) ? a.xs1 : a.xs0, *Y = (L0 & 1) ? a.ys1 : a.ys0;
    int32_t *Xn = (L0 & 1) ? a.xs0 : a.xs1, *Yn = (L0 & 1) ? a.ys0 : a.ys1;
    for (int L = L0; L <= a.max_depth; ++L) {
        for (int e = first_node_at_or_after(t, L, seg_lo) + tid; e < t.nd_off[L + 1]; e += SUBTREE_THREADS) {
            const int node = t.nd_list[e];
            if (t.lo[node] >= seg_hi) break;
            stats_for(a, node, X, Y);
        }
        if (L == a.max_depth) break;
        for (int k = seg_lo + tid; k < seg_hi; k += SUBTREE_THREADS) {
            int s = t.seg_of[(int64_t)L * n + k];
            if (!t.seg_split[s]) continue;
            int lo = t.seg_lo[s], hi = t.seg_hi[s];
            double ex = a.pts[2 * X[hi - 1]] - a.pts[2 * X[lo]];
            double ey = a.pts[2 * Y[hi - 1] + 1] - a.pts[2 * Y[lo] + 1];
            const int32_t *P = ey > ex ? Y : X;
            a.flag[P[k]] = (k - lo) < (hi - lo) / 2 ? 1 : 0;
        }
        if (tid == 0) s_carry = 0;
        __syncthreads();
        // other-run flags and their exclusive prefix over [seg_lo, seg_hi)
        for (int b0 = seg_lo; b0 < seg_hi; b0 += SUBTREE_THREADS) {
            const int k = b0 + tid;
            int v = 0;
            if (k < seg_hi) {
                int s = t.seg_of[(int64_t)L * n + k];
                if (t.seg_split[s]) {
                    const int32_t *O = t.axis[t.seg_node[s]] ? X : Y;
                    v = a.flag[O[k]];
                }
            }
            int ex, agg;
            BS(scan_tmp).ExclusiveSum(v, ex, agg);
            if (k < seg_hi) a.prefix[k] = s_carry + ex;
            __syncthreads();
            if (tid == 0) s_carry += agg;
            __syncthreads();
        }
        for (int k = seg_lo + tid; k < seg_hi; k += SUBTREE_THREADS) {
            int s = t.seg_of[(int64_t)L * n + k];
            if (!t.seg_split[s]) {
                Xn[k] = X[k];
                Yn[k] = Y[k];
                continue;
            }
            int lo = t.seg_lo[s], hi = t.seg_hi[s];
            int mid = (hi - lo) / 2;
            int ax = t.axis[t.seg_node[s]];
            const int32_t *P = ax ? Y : X;
            const int32_t *O = ax ? X : Y;
            int32_t *Pn = ax ? Yn : Xn;
            int32_t *On = ax ? Xn : Yn;
            Pn[k] = P[k];
            int id = O[k];
            int left_before = a.prefix[k] - a.prefix[lo];
            int dest = a.flag[id] ? lo + left_before : lo + mid + (k - lo - left_before);
            On[dest] = id;
        }
        __syncthreads();
        int32_t *tx = X, *ty = Y;
        X = Xn;
        Y = Yn;
        Xn = tx;
        Yn = ty;
    }
    __syncthreads();
    // leaf sums + gather into leaf order for this subtree's leaves (warp per leaf)
    const int lane = tid & 31, wid = tid >> 5;
    const int root = t.seg_node[g];
    for (int w = t.leaf_lo[root] + wid; w < t.leaf_hi[root]; w += SUBTREE_THREADS / 32) {
        int node = t.leaves[w];
        int lo = t.lo[node], hi = t.hi[node];
        double sx = 0.0, sy = 0.0;
        for (int k = lo + lane; k < hi; k += 32) {
            double2 p = reinterpret_cast<const double2 *>(a.pts)[X[k]];
            reinterpret_cast<double2 *>(t.spts)[k] = p;
            sx += p.x;
            sy += p.y;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sx += __shfl_xor_sync(0xffffffffu, sx, o);
            sy += __shfl_xor_sync(0xffffffffu, sy, o);
        }
        if (lane == 0) {
            t.leaf_sum[2 * w] = sx;
            t.leaf_sum[2 * w + 1] = sy;
        }
    }
}

__global__ void centroid_kernel(BuildArgs a) {
    pdl_wait();
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    node_centroids(a, gtid >> 5, ((int64_t)gridDim.x * blockDim.x) >> 5);
}

// ---------------------------------------------------------------------------
// Barnes-Hut traversal (warp-cooperative union DFS).
#ifndef MDC_BH_WARPS
#define MDC_BH_WARPS 4
#endif
constexpr int BH_WARPS = MDC_BH_WARPS;
constexpr int BH_STACK = 64;

// fp64 reciprocal / reciprocal square root: MUFU seed + one third-order
// correction each (seed error e ~ 2^-22 -> O(e^3) ~ 2^-66, i.e. ~1 ulp after
// rounding).  The reference's IEEE division/sqrt agree to ~1e-16, far inside
// the 1e-12 per-step contract.  The opening criterion keeps the IEEE sqrt so
// every far/near decision matches the reference bit for bit.
#ifndef MDC_BH_NEWTON
#define MDC_BH_NEWTON 2  // order of the correction after the MUFU rcp/rsqrt approximations
#endif
__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);      // r = (1 - e)/x
#if MDC_BH_NEWTON == 1
    return fma(r, e, r);             // r (1 + e): relative error ~ e^2
#else
    return fma(r, fma(e, e, e), r);  // r (1 + e + e^2)
#endif
}
__device__ __forceinline__ double rsqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x * y, y, 1.0);                 // y = (1 - e)^(1/2) / sqrt(x)
#if MDC_BH_NEWTON == 1
    return fma(y, 0.5 * e, y);                      // y (1 + e/2): relative error ~ 3e^2/8
#else
    return fma(y * e, fma(0.375, e, 0.5), y);       // y (1 + e/2 + 3e^2/8)
#endif
}

// r = sqrt(x) from the same MUFU seed y0 ~ 1/sqrt(x): r = x y0 (1 + e/2 + 3e^2/8)
// with e = 1 - x y0^2 -- the rsqrt_nr series applied to r0 = x y0 directly,
// one multiply fewer than x * rsqrt_nr(x).
#ifndef MDC_BH_SQRT_NR
#define MDC_BH_SQRT_NR 1
#endif
__device__ __forceinline__ double sqrt_nr(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double r0 = x * y;
    const double e = fma(-r0, y, 1.0);
    return fma(r0, e * fma(0.375, e, 0.5), r0);
}

#ifndef MDC_BH_F32TEST
#define MDC_BH_F32TEST 1  // fp32 pre-test of the opening criterion (exact fp64 only inside its band)
#endif
__device__ __forceinline__ bool far_node(const double4 g0, double size, double xi, double yi, double theta) {
    double gx = g0.x - xi;
    if (gx < 0.0) gx = xi - g0.z;
    if (gx < 0.0) gx = 0.0;
    double gy = g0.y - yi;
    if (gy < 0.0) gy = yi - g0.w;
    if (gy < 0.0) gy = 0.0;
#if MDC_BH_F32TEST
    {
        // fp32 pre-test: gx, gy are exact fp64 differences rounded once to
        // fp32 (relative 2^-24), so d2 and size^2 carry < 1e-6 relative
        // error; outside a 1e-4 band the fp32 decision equals the fp64 one.
        const float gxf = (float)gx, gyf = (float)gy, sf = (float)size, tf = (float)theta;
        const float d2f = __fmaf_rn(gxf, gxf, gyf * gyf), lf = sf * sf, rf = (tf * tf) * d2f;
        if (lf < rf * (1.0f - 1e-4f)) return true;
        if (lf > rf * (1.0f + 1e-4f)) return false;
    }
#endif
    const double d2 = __dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy));
    // The reference decides size < theta * sqrt(d2) with both roundings.
    // Squared comparison with a 2^-40 relative guard band settles every case
    // outside the band identically (rounding moves either side by < 2^-51);
    // only cases inside the band take the exact IEEE-sqrt path.
    const double lhs = __dmul_rn(size, size), rhs = __dmul_rn(__dmul_rn(theta, theta), d2);
    if (lhs < rhs * (1.0 - 0x1p-40)) return true;
    if (lhs > rhs * (1.0 + 0x1p-40)) return false;
    return size < __dmul_rn(theta, __dsqrt_rn(d2));
}

// Accumulates mass * (x_i - com) / (r^3 + eta); the caller scales by c once.
__device__ __forceinline__ void monopole(const double4 g1, double xi, double yi, double eta, double &fx,
                                         double &fy) {
    double dx = xi - g1.x, dy = yi - g1.y;
    double r2 = dx * dx + dy * dy;
#if MDC_BH_SQRT_NR
    double coef = g1.w * rcp_nr(fma(r2, sqrt_nr(r2), eta));
#else
    double r = r2 * rsqrt_nr(r2);
    double coef = g1.w * rcp_nr(r * r * r + eta);
#endif
    fx = fma(coef, dx, fx);
    fy = fma(coef, dy, fy);
}

// grid.x: groups of BH_WARPS warps (32 leaf-order points each); grid.y: task.
// A task re-checks its cut ancestors per lane (an accepted ancestor's
// monopole is added by exactly one task), then walks its subtree.  The set of
// interactions per point is exactly the reference's; partial sums per task
// are combined in task order by the consumer.
// COUNT (profiling only, mdc_layout_profile): also tally leaf-pair and
// monopole interactions and node opening tests into cnt[0..2].
// One warp's work item: point-warp `pw` (32 leaf-order points from k0) x task.
// s_node / s_mask / s_leaf: this warp's BH_STACK / BH_STACK / 32 entries.
template <bool COUNT>
__device__ __forceinline__ void bh_body(int64_t n, int64_t k0, int64_t k1, const DevTree &t, double c, double eta,
                                        double theta, unsigned long long *cnt, int64_t pw, int task, int *s_node_w,
                                        unsigned *s_mask_w, double2 *s_leaf_w) {
    unsigned long long n_leaf = 0, n_mono = 0, n_test = 0, n_slot = 0;
    const int lane = threadIdx.x & 31;
    const int64_t k = k0 + pw * 32 + lane;
    const bool valid = k < k1;
    double xi = 0.0, yi = 0.0;
    if (valid) {
        double2 p = reinterpret_cast<const double2 *>(t.spts)[k];
        xi = p.x;
        yi = p.y;
    }
    double fx = 0.0, fy = 0.0;
    bool act = valid;
    for (int dd = 0; dd < t.cut; ++dd) {
        int a = t.task_path[task * t.cut + dd];
        double4 g0 = t.geo[2 * a], g1 = t.geo[2 * a + 1];
        if (COUNT && act) ++n_test;
        if (act && far_node(g0, g1.z, xi, yi, theta)) {
            act = false;
            if (t.task_first[task * t.cut + dd]) {
                monopole(g1, xi, yi, eta, fx, fy);
                if (COUNT) ++n_mono;
            }
        }
    }
    unsigned m0 = __ballot_sync(0xffffffffu, act);
    if (m0) {
        if (lane == 0) {
            s_node_w[0] = t.task_node[task];
            s_mask_w[0] = m0;
        }
        int sp = 1;
        __syncwarp();
        const double2 *sp2 = reinterpret_cast<const double2 *>(t.spts);
        while (sp > 0) {
            --sp;
            int node = s_node_w[sp];
            unsigned mask = s_mask_w[sp];
            __syncwarp();
            bool on = (mask >> lane) & 1u;
            int4 tp = t.topo[node];
            // the node's geometry loads issue with its topology: one L1/L2
            // round trip per visit instead of two (unused for leaves)
            const double4 g0 = t.geo[2 * node], g1 = t.geo[2 * node + 1];
            if (COUNT && lane == 0) n_slot += tp.z < 0 ? 32ull * (unsigned long long)(tp.y - tp.x) : 32ull;
            if (tp.z < 0) {
                // Leaf: pairwise sum over its points (_kernels.py:194-205).  The
                // self term is exactly +0 (dx = dy = 0; + 1e-300 keeps r2 > 0 and
                // the weight finite, absorbed exactly by any r2 > ~1e-284), so no
                // j != i test is needed -- coincident distinct points also
                // contribute 0 in the reference.
                // The warp stages the leaf's points in shared memory (one
                // coalesced load per 32 points), then every active lane sums its
                // pairs from shared broadcasts in point order, in two
                // accumulation chains (even / odd points) for fp64 ILP.
                if (COUNT && on) n_leaf += (unsigned long long)(tp.y - tp.x);
                for (int base = tp.x; base < tp.y; base += 32) {
                    const int cnt = min(32, tp.y - base);
                    if (lane < cnt) s_leaf_w[lane] = __ldg(sp2 + base + lane);
                    __syncwarp();
                    if (on) {
                        auto pair = [&](int q, double &ax, double &ay) {
                            const double2 pj = s_leaf_w[q];
                            double dx = xi - pj.x, dy = yi - pj.y;
                            double r2 = fma(dx, dx, fma(dy, dy, 1e-300));
#if MDC_BH_SQRT_NR
                            double w = rcp_nr(fma(r2, sqrt_nr(r2), eta));
#else
                            double y = rsqrt_nr(r2);
                            double w = rcp_nr(r2 * (r2 * y) + eta);
#endif
                            ax = fma(w, dx, ax);
                            ay = fma(w, dy, ay);
                        };
                        double gx = 0.0, gy = 0.0;
                        int q = 0;
#pragma unroll 4
                        for (; q + 1 < cnt; q += 2) {
                            pair(q, fx, fy);
                            pair(q + 1, gx, gy);
                        }
                        if (q < cnt) pair(q, fx, fy);
                        fx += gx;
                        fy += gy;
                    }
                    __syncwarp();
                }
                continue;
            }
            bool open = false;
            if (on) {
                if (COUNT) ++n_test;
                if (far_node(g0, g1.z, xi, yi, theta)) {
                    monopole(g1, xi, yi, eta, fx, fy);
                    if (COUNT) ++n_mono;
                } else {
                    open = true;
                }
            }
            unsigned om = __ballot_sync(0xffffffffu, open);
            if (om) {
                if (lane == 0) {
                    s_node_w[sp] = tp.z;
                    s_mask_w[sp] = om;
                    s_node_w[sp + 1] = tp.w;
                    s_mask_w[sp + 1] = om;
                }
                sp += 2;
                __syncwarp();
            }
        }
    }
    if (valid) reinterpret_cast<double2 *>(t.part)[(size_t)task * n + k] = make_double2(c * fx, c * fy);
    if (COUNT && valid) {
        atomicAdd(cnt + 0, n_leaf);
        atomicAdd(cnt + 1, n_mono);
        atomicAdd(cnt + 2, n_test);
        if (lane == 0) atomicAdd(cnt + 3, n_slot);
    }
}

template <bool COUNT>
#ifndef MDC_BH_MINB
#define MDC_BH_MINB 0  // 0: no occupancy target (the register count caps BH at 8 CTAs = 50 % occupancy)
#endif
__global__ void __launch_bounds__(BH_WARPS * 32, MDC_BH_MINB) bh_kernel(int64_t n, int64_t k0, int64_t k1, DevTree t,
                                                           double c, double eta, double theta,
                                                           unsigned long long *cnt) {
    pdl_wait();
    __shared__ int s_node[BH_WARPS][BH_STACK];
    __shared__ unsigned s_mask[BH_WARPS][BH_STACK];
    __shared__ double2 s_leaf[BH_WARPS][32];  // the leaf being summed
    const int wib = threadIdx.x >> 5;
    bh_body<COUNT>(n, k0, k1, t, c, eta, theta, cnt, (int64_t)blockIdx.x * BH_WARPS + wib, blockIdx.y, s_node[wib],
                   s_mask[wib], s_leaf[wib]);
}

// Combine the task partials (task order) into out[i] by point id.
__device__ __forceinline__ double2 bh_total(const DevTree &t, int64_t n, int64_t k) {
    double fx = 0.0, fy = 0.0;
    for (int task = 0; task < t.ntask; ++task) {
        double2 v = reinterpret_cast<const double2 *>(t.part)[(size_t)task * n + k];
        fx += v.x;
        fy += v.y;
    }
    return make_double2(fx, fy);
}

__global__ void bh_combine_kernel(int64_t n, int64_t k0, int64_t k1, DevTree t, const int32_t *perm, double *out) {
    pdl_wait();
    int64_t k = k0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= k1) return;
    reinterpret_cast<double2 *>(out)[perm[k]] = bh_total(t, n, k);
}

// ---------------------------------------------------------------------------
// Fused per-vertex step.  Written with explicit _rn intrinsics so every
// operation is one IEEE rounding in the reference's order (numpy never fuses).
constexpr int MDC_MAX_PEERS = 8;

struct LocalArgs {
    int64_t n;
    const double *pos;
    double *pos_out;
    const double *bh;
    const int32_t *csr_off, *csr_tgt, *tris, *inc_off, *inc;
    double spring, dlen, eta, c;
    const double *temps;
    const int32_t *ctr;
    double *dbg_bh, *dbg_force, *dbg_scale;
    const int32_t *perm;  // partitioned step: vertex = perm[k0 + idx]
    int64_t k0, k1;
    // peer-memory exchange: the new position goes to every rank's
    // next-parity buffer (NVLink stores) instead of pos_out
    int npeer;
    double *peer_out[MDC_MAX_PEERS];
    // all-gather exchange: the owned slice's new positions, packed in leaf
    // order (send[idx] for vertex perm[k0 + idx]), instead of pos_out
    double *send;
};

__device__ __forceinline__ double2 ld2(const double *p, int i) {
    return reinterpret_cast<const double2 *>(p)[i];
}

// Per-node clamp factor (layout.py:160-184 clamp_factors, one node): the
// largest s in [0, 1] keeping the node eta clear of the three mid-segment
// limiting lines of every incident triangle inc[b0, b1) under displacement f.
// Smallest factor over incident triangles inc[b0, b1) step `stride` (INFINITY: none binds).
__device__ __forceinline__ double clamp_factor_raw(const double *pos, const int32_t *tris, const int32_t *inc, int b0,
                                                   int b1, int stride, double2 pi, double2 f, double eta) {
    double smin = INFINITY;
    for (int e = b0; e < b1; e += stride) {
        int tt = inc[e] >> 2;
        int4 tr = reinterpret_cast<const int4 *>(tris)[tt];
        double2 A = ld2(pos, tr.x), B = ld2(pos, tr.y), C = ld2(pos, tr.z);
        double mabx = dmul(0.5, dadd(A.x, B.x)), maby = dmul(0.5, dadd(A.y, B.y));
        double mbcx = dmul(0.5, dadd(B.x, C.x)), mbcy = dmul(0.5, dadd(B.y, C.y));
        double mcax = dmul(0.5, dadd(C.x, A.x)), mcay = dmul(0.5, dadd(C.y, A.y));
        const double ptx[3] = {mabx, mabx, mbcx}, pty[3] = {maby, maby, mbcy};
        const double drx[3] = {dsub(mcax, mabx), dsub(mbcx, mabx), dsub(mcax, mbcx)};
        const double dry[3] = {dsub(mcay, maby), dsub(mbcy, maby), dsub(mcay, mbcy)};
#pragma unroll
        for (int l = 0; l < 3; ++l) {
            double nx = -dry[l], ny = drx[l];
            double ln = hypot(nx, ny);
            if (ln == 0.0) ln = 1.0;
            nx = __ddiv_rn(nx, ln);
            ny = __ddiv_rn(ny, ln);
            double relx = dsub(pi.x, ptx[l]), rely = dsub(pi.y, pty[l]);
            double sg = dadd(dmul(relx, nx), dmul(rely, ny));
            double side = sg >= 0.0 ? 1.0 : -1.0;
            double dist = fabs(sg);
            double allowed = fmax(0.0, dsub(dist, eta));
            double toward = dmul(-side, dadd(dmul(f.x, nx), dmul(f.y, ny)));
            if (toward > allowed) {
                double fac = __ddiv_rn(allowed, toward);
                if (fac < smin) smin = fac;
            }
        }
    }
    return smin;
}

__device__ __forceinline__ double clamp_factor(const double *pos, const int32_t *tris, const int32_t *inc, int b0,
                                               int b1, double2 pi, double2 f, double eta) {
    const double smin = clamp_factor_raw(pos, tris, inc, b0, b1, 1, pi, f, eta);
    return smin == INFINITY ? 1.0 : fmin(fmax(smin, 0.0), 1.0);
}

__global__ void clamp_factors_kernel(int64_t n, const double *pos, const double *disp, const int32_t *tris,
                                     const int32_t *inc_off, const int32_t *inc, double eta, double *s_out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    s_out[i] = clamp_factor(pos, tris, inc, inc_off[i], inc_off[i + 1], ld2(pos, (int)i), ld2(disp, (int)i), eta);
}

__global__ void local_kernel(LocalArgs a) {
    pdl_wait();
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t idx = i;
    if (a.perm) {
        if (a.k0 + i >= a.k1) return;
        i = a.perm[a.k0 + i];
    } else if (i >= a.n) {
        return;
    }
    const double T = a.temps[*a.ctr];
    const double2 pi = ld2(a.pos, (int)i);
    double2 f = ld2(a.bh, (int)i);
    if (a.dbg_bh) reinterpret_cast<double2 *>(a.dbg_bh)[i] = f;
    // spring (layout.py:216-231): coef = -s*log((r+eta)/D); bincount in edge order
    {
        double sx = 0.0, sy = 0.0;
        const double ns = -a.spring;
        for (int e = a.csr_off[i]; e < a.csr_off[i + 1]; ++e) {
            double2 pj = ld2(a.pos, a.csr_tgt[e]);
            double dx = dsub(pi.x, pj.x), dy = dsub(pi.y, pj.y);
            double r = hypot(dx, dy);
            double coef = dmul(ns, log(__ddiv_rn(dadd(r, a.eta), a.dlen)));
            sx = dadd(sx, dmul(coef, dx));
            sy = dadd(sy, dmul(coef, dy));
        }
        f.x = dadd(f.x, sx);
        f.y = dadd(f.y, sy);
    }
    // node-edge (layout.py:234-256): per corner k a bincount sum in triangle
    // order, subtracted k = 0, 1, 2.  inc is sorted by (corner, triangle).
    const int b0 = a.inc_off[i], b1 = a.inc_off[i + 1];
    {
        double nex = 0.0, ney = 0.0;  // running forces array (starts at zeros)
        int e = b0;
        for (int k = 0; k < 3; ++k) {
            double px = 0.0, py = 0.0;
            for (; e < b1 && (a.inc[e] & 3) == k; ++e) {
                int tt = a.inc[e] >> 2;
                int4 tr = reinterpret_cast<const int4 *>(a.tris)[tt];
                int tv[3] = {tr.x, tr.y, tr.z};
                double2 av = ld2(a.pos, tv[(k + 1) % 3]);
                double2 bv = ld2(a.pos, tv[(k + 2) % 3]);
                double ex = dsub(bv.x, av.x), ey = dsub(bv.y, av.y);
                double ee = dadd(dmul(ex, ex), dmul(ey, ey));
                if (ee == 0.0) ee = 1.0;
                double t = __ddiv_rn(dadd(dmul(dsub(pi.x, av.x), ex), dmul(dsub(pi.y, av.y), ey)), ee);
                double rx = dsub(dadd(av.x, dmul(t, ex)), pi.x);
                double ry = dsub(dadd(av.y, dmul(t, ey)), pi.y);
                double nr = hypot(rx, ry);
                double coef = nr >= 1e-12 ? __ddiv_rn(__ddiv_rn(a.c, dadd(dmul(nr, nr), a.eta)), nr) : 0.0;
                px = dadd(px, dmul(coef, rx));
                py = dadd(py, dmul(coef, ry));
            }
            nex = dsub(nex, px);
            ney = dsub(ney, py);
        }
        f.x = dadd(f.x, nex);
        f.y = dadd(f.y, ney);
    }
    if (a.dbg_force) reinterpret_cast<double2 *>(a.dbg_force)[i] = f;
    // temperature cap (layout.py:275-278)
    double mag = hypot(f.x, f.y);
    if (mag > T) {
        double k = __ddiv_rn(T, mag);
        f.x = dmul(f.x, k);
        f.y = dmul(f.y, k);
    }
    // limiting-line clamp (layout.py:119-184): 3 rows per incident triangle
    const double s = clamp_factor(a.pos, a.tris, a.inc, b0, b1, pi, f, a.eta);
    if (a.dbg_scale) a.dbg_scale[i] = s;
    const double2 np = make_double2(dadd(pi.x, dmul(s, f.x)), dadd(pi.y, dmul(s, f.y)));
    if (a.send) {
        reinterpret_cast<double2 *>(a.send)[idx] = np;
    } else if (a.npeer) {
        for (int r = 0; r < a.npeer; ++r) reinterpret_cast<double2 *>(a.peer_out[r])[i] = np;
        __threadfence_system();  // visible to the peers once the step is over
    } else {
        reinterpret_cast<double2 *>(a.pos_out)[i] = np;
    }
}

// Lane-group variant: LG lanes per vertex evaluate the spring, node-edge and
// limiting-line terms of that vertex in parallel; the group leader adds the
// spring and node-edge terms in exactly the serial kernel's order (terms are
// gathered by shuffles), the clamp is a min (order-free).  Same values bit
// for bit as local_kernel, LG times the threads for the gather latency.
// A/B: 10k vertices 37 -> 20 us (LG 4; one thread per vertex leaves the
// GPU latency-bound), 100k no gain (51 -> 55 us), so small meshes only.
#ifndef MDC_LOCAL_LG
#define MDC_LOCAL_LG 4  // lanes per vertex for n <= MDC_LOCAL_LG_MAXN (0: never)
#endif
#ifndef MDC_LOCAL_LG_MAXN
#define MDC_LOCAL_LG_MAXN 32768
#endif
constexpr int LOCAL_SL = 4;  // terms per lane per gather round

// gthread: this thread's global index over the n x LG lanes (all 32 lanes of
// a warp must call together: the group reductions are warp collectives).
template <int LG>
__device__ __forceinline__ void local_group_body(const LocalArgs &a, int64_t gthread) {
    const unsigned FULL = 0xffffffffu;
    const int sub = threadIdx.x & (LG - 1);
    const int64_t idx = gthread / LG;
    bool live;
    int64_t i;
    if (a.perm) {
        live = a.k0 + idx < a.k1;
        i = live ? a.perm[a.k0 + idx] : a.perm[a.k0];
    } else {
        live = idx < a.n;
        i = live ? idx : 0;
    }
    const bool lead = sub == 0;
    const double T = a.temps[*a.ctr];
    const double2 pi = ld2(a.pos, (int)i);
    double2 f = ld2(a.bh, (int)i);
    if (a.dbg_bh && live && lead) reinterpret_cast<double2 *>(a.dbg_bh)[i] = f;
    constexpr int RW = LG * LOCAL_SL;  // entries per round
    // spring (layout.py:216-231), terms in edge order
    {
        const int e0 = a.csr_off[i], e1 = a.csr_off[i + 1];
        const int rounds = __reduce_max_sync(FULL, (e1 - e0 + RW - 1) / RW);
        const double ns = -a.spring;
        double sx = 0.0, sy = 0.0;
        for (int r = 0; r < rounds; ++r) {
            double tx[LOCAL_SL], ty[LOCAL_SL];
#pragma unroll
            for (int q = 0; q < LOCAL_SL; ++q) {
                const int e = e0 + r * RW + q * LG + sub;
                tx[q] = ty[q] = 0.0;
                if (e < e1) {
                    double2 pj = ld2(a.pos, a.csr_tgt[e]);
                    double dx = dsub(pi.x, pj.x), dy = dsub(pi.y, pj.y);
                    double rr = hypot(dx, dy);
                    double coef = dmul(ns, log(__ddiv_rn(dadd(rr, a.eta), a.dlen)));
                    tx[q] = dmul(coef, dx);
                    ty[q] = dmul(coef, dy);
                }
            }
#pragma unroll
            for (int q = 0; q < LOCAL_SL; ++q)
#pragma unroll
                for (int l = 0; l < LG; ++l) {
                    const double vx = __shfl_sync(FULL, tx[q], l, LG), vy = __shfl_sync(FULL, ty[q], l, LG);
                    if (e0 + r * RW + q * LG + l < e1) {
                        sx = dadd(sx, vx);
                        sy = dadd(sy, vy);
                    }
                }
        }
        f.x = dadd(f.x, sx);
        f.y = dadd(f.y, sy);
    }
    // node-edge (layout.py:234-256): inc is sorted by (corner, triangle); the
    // per-corner sums are subtracted corner by corner, as in local_kernel
    const int b0 = a.inc_off[i], b1 = a.inc_off[i + 1];
    {
        const int rounds = __reduce_max_sync(FULL, (b1 - b0 + RW - 1) / RW);
        double nex = 0.0, ney = 0.0, px = 0.0, py = 0.0;
        int cur = 0;
        for (int r = 0; r < rounds; ++r) {
            double tx[LOCAL_SL], ty[LOCAL_SL];
#pragma unroll
            for (int q = 0; q < LOCAL_SL; ++q) {
                const int e = b0 + r * RW + q * LG + sub;
                tx[q] = ty[q] = 0.0;
                if (e < b1) {
                    const int code = a.inc[e];
                    const int k = code & 3, tt = code >> 2;
                    int4 tr = reinterpret_cast<const int4 *>(a.tris)[tt];
                    int tv[3] = {tr.x, tr.y, tr.z};
                    double2 av = ld2(a.pos, tv[(k + 1) % 3]);
                    double2 bv = ld2(a.pos, tv[(k + 2) % 3]);
                    double ex = dsub(bv.x, av.x), ey = dsub(bv.y, av.y);
                    double ee = dadd(dmul(ex, ex), dmul(ey, ey));
                    if (ee == 0.0) ee = 1.0;
                    double t = __ddiv_rn(dadd(dmul(dsub(pi.x, av.x), ex), dmul(dsub(pi.y, av.y), ey)), ee);
                    double rx = dsub(dadd(av.x, dmul(t, ex)), pi.x);
                    double ry = dsub(dadd(av.y, dmul(t, ey)), pi.y);
                    double nr = hypot(rx, ry);
                    double coef = nr >= 1e-12 ? __ddiv_rn(__ddiv_rn(a.c, dadd(dmul(nr, nr), a.eta)), nr) : 0.0;
                    tx[q] = dmul(coef, rx);
                    ty[q] = dmul(coef, ry);
                }
            }
#pragma unroll
            for (int q = 0; q < LOCAL_SL; ++q)
#pragma unroll
                for (int l = 0; l < LG; ++l) {
                    const double vx = __shfl_sync(FULL, tx[q], l, LG), vy = __shfl_sync(FULL, ty[q], l, LG);
                    const int e = b0 + r * RW + q * LG + l;
                    if (lead && e < b1) {
                        const int k = a.inc[e] & 3;
                        for (; cur < k; ++cur) {
                            nex = dsub(nex, px);
                            ney = dsub(ney, py);
                            px = py = 0.0;
                        }
                        px = dadd(px, vx);
                        py = dadd(py, vy);
                    }
                }
        }
        for (; cur < 3; ++cur) {
            nex = dsub(nex, px);
            ney = dsub(ney, py);
            px = py = 0.0;
        }
        f.x = dadd(f.x, nex);
        f.y = dadd(f.y, ney);
    }
    f.x = __shfl_sync(FULL, f.x, 0, LG);
    f.y = __shfl_sync(FULL, f.y, 0, LG);
    if (a.dbg_force && live && lead) reinterpret_cast<double2 *>(a.dbg_force)[i] = f;
    double mag = hypot(f.x, f.y);
    if (mag > T) {
        double k = __ddiv_rn(T, mag);
        f.x = dmul(f.x, k);
        f.y = dmul(f.y, k);
    }
    // limiting-line clamp: each lane takes every LG-th incident triangle, min over the group
    double smin = INFINITY;
    {
        double sl = clamp_factor_raw(a.pos, a.tris, a.inc, b0 + sub, b1, LG, pi, f, a.eta);
#pragma unroll
        for (int o = LG / 2; o > 0; o >>= 1) sl = fmin(sl, __shfl_xor_sync(FULL, sl, o, LG));
        smin = sl;
    }
    const double s = smin == INFINITY ? 1.0 : fmin(fmax(smin, 0.0), 1.0);
    if (!live || !lead) return;
    if (a.dbg_scale) a.dbg_scale[i] = s;
    const double2 np = make_double2(dadd(pi.x, dmul(s, f.x)), dadd(pi.y, dmul(s, f.y)));
    if (a.send) {
        reinterpret_cast<double2 *>(a.send)[idx] = np;
    } else if (a.npeer) {
        for (int r = 0; r < a.npeer; ++r) reinterpret_cast<double2 *>(a.peer_out[r])[i] = np;
        __threadfence_system();
    } else {
        reinterpret_cast<double2 *>(a.pos_out)[i] = np;
    }
}

template <int LG>
__global__ void __launch_bounds__(128) local_group_kernel(LocalArgs a) {
    pdl_wait();
    local_group_body<LG>(a, (int64_t)blockIdx.x * blockDim.x + threadIdx.x);
}

__global__ void incr_kernel(int32_t *ctr) {
    pdl_wait();
    ctr[0] += 1;
}

// ---------------------------------------------------------------------------
// Small meshes (n <= MDC_LAYOUT_SMALL_MAX, one GPU): the whole step -- exact
// (coord, id) ranks on both axes, the one-CTA level walk, Barnes-Hut over
// (point-warp, task) items, the task-ordered combine and the local update --
// in ONE persistent CTA, for all k steps of the call, with block barriers
// between phases instead of ~9 kernel launches per step (config 1: 150
// points, where launch latency, not work, set the step time).  Same device
// code and summation orders as the multi-kernel step: bit-identical.
#ifndef MDC_LAYOUT_SMALL_MAX
#define MDC_LAYOUT_SMALL_MAX 512  // one CTA only pays off for tiny meshes (n = 2000: 1.9 ms vs ~0.1 ms per step)
#endif
#ifndef MDC_SMALL_THREADS
#define MDC_SMALL_THREADS 256  // per CTA of the cluster (A/B at config 1: 128 29.5, 256 27.0, 512 28.2 us/step)
#endif
constexpr int SMALL_THREADS = MDC_SMALL_THREADS;
#ifndef MDC_SMALL_LG
#define MDC_SMALL_LG MDC_LOCAL_LG  // lanes per vertex in the persistent step's local update
#endif
constexpr int SMALL_LG = MDC_SMALL_LG;

struct SmallArgs {
    BuildArgs ba;  // ba.pts is set per step
    LocalArgs la;  // pos / pos_out / ctr are set per step
    double *bufs[2];
    int k;
    double c, eta, theta;
    int32_t *ctr;
    // shared-memory staging: mesh topology (CSR neighbours, incidences,
    // triangles) and, on CTA 0, the tree shape and walk scratch
    int nE, nI, ntri, nn, ns, nl;
};

// Per-CTA shared-memory carve of the persistent small step (16-byte aligned
// pieces); the host computes the same size.
struct SmallSmem {
    double *pos, *bh;
    int4 *tris;
    int32_t *csr_off, *csr_tgt, *inc_off, *inc;
    int32_t *xs0, *xs1, *ys1, *flag, *oflag, *prefix, *blocksum;
    int32_t *lo, *hi, *left, *right, *nd_off, *nd_list, *seg_off, *seg_lo, *seg_hi, *seg_node, *seg_split, *seg_of,
        *leaves, *leaf_lo, *leaf_hi;
};
__host__ __device__ inline size_t small_carve(SmallSmem &m, unsigned char *base, int64_t n, int nE, int nI, int ntri,
                                              int nn, int ns, int nl, int md) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        unsigned char *p = base + off;
        off += (bytes + 15) & ~(size_t)15;
        return p;
    };
    m.pos = (double *)take(16 * (size_t)n);
    m.bh = (double *)take(16 * (size_t)n);
    m.tris = (int4 *)take(16 * (size_t)ntri);
    m.csr_off = (int32_t *)take(4 * (size_t)(n + 1));
    m.csr_tgt = (int32_t *)take(4 * (size_t)nE);
    m.inc_off = (int32_t *)take(4 * (size_t)(n + 1));
    m.inc = (int32_t *)take(4 * (size_t)nI);
    m.xs0 = (int32_t *)take(8 * (size_t)n);
    m.xs1 = (int32_t *)take(4 * (size_t)n);
    m.ys1 = (int32_t *)take(4 * (size_t)n);
    m.flag = (int32_t *)take(4 * (size_t)n);
    m.oflag = (int32_t *)take(4 * (size_t)n);
    m.prefix = (int32_t *)take(4 * (size_t)n);
    m.blocksum = (int32_t *)take(4 * 32);
    m.lo = (int32_t *)take(4 * (size_t)nn);
    m.hi = (int32_t *)take(4 * (size_t)nn);
    m.left = (int32_t *)take(4 * (size_t)nn);
    m.right = (int32_t *)take(4 * (size_t)nn);
    m.nd_off = (int32_t *)take(4 * (size_t)(md + 2));
    m.nd_list = (int32_t *)take(4 * (size_t)nn);
    m.seg_off = (int32_t *)take(4 * (size_t)(md + 1));
    m.seg_lo = (int32_t *)take(4 * (size_t)ns);
    m.seg_hi = (int32_t *)take(4 * (size_t)ns);
    m.seg_node = (int32_t *)take(4 * (size_t)ns);
    m.seg_split = (int32_t *)take(4 * (size_t)ns);
    m.seg_of = (int32_t *)take(4 * (size_t)md * (size_t)n);
    m.leaves = (int32_t *)take(4 * (size_t)nl);
    m.leaf_lo = (int32_t *)take(4 * (size_t)nn);
    m.leaf_hi = (int32_t *)take(4 * (size_t)nn);
    return off;
}

__device__ __forceinline__ void copy_i32(int32_t *dst, const int32_t *src, int64_t count) {
    for (int64_t i = threadIdx.x; i < count; i += blockDim.x) dst[i] = src[i];
}

#ifndef MDC_SMALL_CLUSTER
#define MDC_SMALL_CLUSTER 8  // CTAs (one thread-block cluster) sharing the persistent small-mesh step
#endif
constexpr int SMALL_CLUSTER = MDC_SMALL_CLUSTER;

// barrier over the whole cluster with release/acquire at cluster scope: the
// CTAs' global-memory writes before it are visible to all of them after it
__device__ __forceinline__ void small_sync() {
    if (SMALL_CLUSTER > 1)
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    else
        __syncthreads();
}

// The step's phases spread over a cluster of SMALL_CLUSTER CTAs: the BH items
// and the local lanes are split across the cluster (one SM's FP64 pipe
// bounded the local update), the ranks and the tree walk run on CTA 0.  The
// mesh topology is staged in each CTA's shared memory once per launch, the
// tree shape and the walk's scratch in CTA 0's, and every step's positions
// and combined BH forces in each CTA's -- the local update and the walk then
// read shared memory instead of L2.  Same device code and summation orders:
// bit-identical to the multi-kernel step.
__global__ void __launch_bounds__(SMALL_THREADS, 1) layout_small_kernel(SmallArgs sa) {
    constexpr int W = SMALL_THREADS / 32;
    __shared__ int s_node[W][BH_STACK];
    __shared__ unsigned s_mask[W][BH_STACK];
    __shared__ double2 s_leaf[W][32];
    __shared__ int32_t s_step;
    __shared__ unsigned long long s_key[2 * MDC_LAYOUT_SMALL_MAX];
    extern __shared__ __align__(16) unsigned char s_dyn[];
    const int tid = threadIdx.x, wib = tid >> 5;
    const int cta = blockIdx.x, C = gridDim.x;  // the grid is one cluster
    const int64_t n = sa.ba.n;
    const DevTree &t = sa.ba.t;  // global tree: BH, combine
    const int md = sa.ba.max_depth;
    SmallSmem m;
    small_carve(m, s_dyn, n, sa.nE, sa.nI, sa.ntri, sa.nn, sa.ns, sa.nl, md);
    // mesh topology (every CTA), tree shape (CTA 0)
    copy_i32(m.csr_off, sa.la.csr_off, n + 1);
    copy_i32(m.csr_tgt, sa.la.csr_tgt, sa.nE);
    copy_i32(m.inc_off, sa.la.inc_off, n + 1);
    copy_i32(m.inc, sa.la.inc, sa.nI);
    copy_i32(reinterpret_cast<int32_t *>(m.tris), sa.la.tris, 4 * (int64_t)sa.ntri);
    BuildArgs ba = sa.ba;  // CTA 0's walk: shape + scratch in shared memory, outputs global
    if (cta == 0) {
        copy_i32(m.lo, t.lo, sa.nn);
        copy_i32(m.hi, t.hi, sa.nn);
        copy_i32(m.left, t.left, sa.nn);
        copy_i32(m.right, t.right, sa.nn);
        copy_i32(m.nd_off, t.nd_off, md + 2);
        copy_i32(m.nd_list, t.nd_list, sa.nn);
        copy_i32(m.seg_off, t.seg_off, md + 1);
        copy_i32(m.seg_lo, t.seg_lo, sa.ns);
        copy_i32(m.seg_hi, t.seg_hi, sa.ns);
        copy_i32(m.seg_node, t.seg_node, sa.ns);
        copy_i32(m.seg_split, t.seg_split, sa.ns);
        copy_i32(m.seg_of, t.seg_of, (int64_t)md * n);
        copy_i32(m.leaves, t.leaves, sa.nl);
        copy_i32(m.leaf_lo, t.leaf_lo, sa.nn);
        copy_i32(m.leaf_hi, t.leaf_hi, sa.nn);
        DevTree &u = ba.t;
        u.lo = m.lo, u.hi = m.hi, u.left = m.left, u.right = m.right;
        u.nd_off = m.nd_off, u.nd_list = m.nd_list, u.seg_off = m.seg_off;
        u.seg_lo = m.seg_lo, u.seg_hi = m.seg_hi, u.seg_node = m.seg_node, u.seg_split = m.seg_split;
        u.seg_of = m.seg_of, u.leaves = m.leaves, u.leaf_lo = m.leaf_lo, u.leaf_hi = m.leaf_hi;
        ba.xs0 = m.xs0, ba.ys0 = m.xs0 + n, ba.xs1 = m.xs1, ba.ys1 = m.ys1;
        ba.flag = m.flag, ba.oflag = m.oflag, ba.prefix = m.prefix, ba.blocksum = m.blocksum;
        ba.pts = m.pos;
    }
    const int32_t *sperm = (md & 1) ? m.xs1 : m.xs0;                  // CTA 0: leaf order after the walk
    int32_t *gperm = (md & 1) ? sa.ba.xs1 : sa.ba.xs0;                 // the same, published for the cluster
    LocalArgs la = sa.la;
    la.pos = m.pos;
    la.bh = m.bh;
    la.csr_off = m.csr_off, la.csr_tgt = m.csr_tgt, la.inc_off = m.inc_off, la.inc = m.inc;
    la.tris = reinterpret_cast<const int32_t *>(m.tris);
    la.ctr = &s_step;
    __syncthreads();
#if MDC_SMALL_PROF  // experiments: per-phase clock totals, printed once
    long long ph[6] = {0, 0, 0, 0, 0, 0}, t0 = clock64();
#define MDC_PH(i) do { if (tid == 0) { long long t1 = clock64(); ph[i] += t1 - t0; t0 = t1; } } while (0)
#else
#define MDC_PH(i) do {} while (0)
#endif
    for (int step = 0; step < sa.k; ++step) {
        const double *pin = sa.bufs[step & 1];
        double *pout = sa.bufs[(step & 1) ^ 1];
        for (int64_t e = tid; e < 2 * n; e += SMALL_THREADS) m.pos[e] = pin[e];
        __syncthreads();
        if (cta == 0) {
            // exact ranks -> ids in (coord, id) order, x run then y run (the
            // order the device sort produces)
            for (int64_t e = tid; e < 2 * n; e += SMALL_THREADS) {
                const int axis = e >= n;
                s_key[e] = order_key(m.pos[2 * (e - axis * n) + axis]);
            }
            __syncthreads();
            for (int64_t e = tid; e < 2 * n; e += SMALL_THREADS) {
                const int axis = e >= n;
                const int64_t i = e - axis * n;
                const unsigned long long ki = s_key[e];
                const unsigned long long *kk = s_key + axis * n;
                int r = 0;
#pragma unroll 8
                for (int j = 0; j < (int)n; ++j) {
                    const unsigned long long kj = kk[j];
                    r += (kj < ki) || (kj == ki && j < i);
                }
                m.xs0[axis * n + r] = (int32_t)i;
            }
            __syncthreads();
            MDC_PH(0);
            build_levels_body<SMALL_THREADS, BUILD_ONE_CTA>(ba);
            __syncthreads();
            for (int64_t k = tid; k < n; k += SMALL_THREADS) gperm[k] = sperm[k];
        }
        small_sync();
        MDC_PH(1);
        const int64_t npw = (n + 31) / 32;
        for (int64_t it = (int64_t)cta * W + wib; it < npw * t.ntask; it += (int64_t)C * W)
            bh_body<false>(n, 0, n, t, sa.c, sa.eta, sa.theta, nullptr, it % npw, (int)(it / npw), s_node[wib],
                           s_mask[wib], s_leaf[wib]);
        small_sync();
        MDC_PH(2);
        // every CTA combines all points into its own shared copy
        for (int64_t k = tid; k < n; k += SMALL_THREADS)
            reinterpret_cast<double2 *>(m.bh)[gperm[k]] = bh_total(t, n, k);
        if (tid == 0) s_step = step;
        __syncthreads();
        MDC_PH(3);
        la.pos_out = pout;
        {
            // lane groups split evenly over the cluster in whole warps (a warp
            // calls the body together: its reductions are warp collectives)
            const int64_t lanes = n * SMALL_LG;
            const int64_t chunk = ((lanes + C - 1) / C + 31) / 32 * 32;
            const int64_t lo = (int64_t)cta * chunk, hi = min(lanes, lo + chunk);
            for (int64_t base = lo; base < hi; base += SMALL_THREADS)
                if (base + (tid & ~31) < hi) local_group_body<SMALL_LG>(la, base + tid);
        }
        small_sync();
        MDC_PH(4);
    }
#if MDC_SMALL_PROF
    if (tid == 0 && cta == 0)
        printf("small-step cycles/step: ranks %lld build %lld bh %lld combine %lld local %lld (n=%lld k=%d)\n",
               ph[0] / sa.k, ph[1] / sa.k, ph[2] / sa.k, ph[3] / sa.k, ph[4] / sa.k, (long long)n, sa.k);
#endif
#undef MDC_PH
    if (tid == 0 && cta == 0) *sa.ctr = sa.k;
}

// All-gather exchange, receive side: recv holds every rank's packed slice
// (rank r at r * chunk, n*r/w .. n*(r+1)/w in leaf order); scatter them to
// vertex order through the step's tree permutation.
__global__ void gather_scatter_kernel(int64_t n, int world, int64_t chunk, const int32_t *perm,
                                      const double *recv, double *pos) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // leaf-order index
    if (k >= n) return;
    // owner rank of leaf slot k: the largest r with n*r/w <= k
    int r = (int)((k * world) / n);
    while (r + 1 < world && n * (r + 1) / world <= k) ++r;
    while (r > 0 && n * r / world > k) --r;
    const int64_t idx = k - n * r / world;
    reinterpret_cast<double2 *>(pos)[perm[k]] = reinterpret_cast<const double2 *>(recv)[r * chunk + idx];
}

}  // namespace mdc

using namespace mdc;

struct MdcLayoutPlan {
    MdcLayoutArgs a;
    TreeShape shape;
    Buffers b;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    cudaGraphExec_t graph_multi = nullptr;  // MDC_LAYOUT_MULTI consecutive steps in one graph
    cudaStream_t cap_stream = nullptr;
    const double *graph_temps = nullptr;
    int build_blocks = 0;
    int sms = 148;
    // profiling (mdc_layout_profile): events recorded between step phases
    bool cluster_ok = false;  // the device can co-schedule one BUILD_CLUSTER cluster
    int small_nE = 0, small_nI = 0;  // CSR neighbour / incidence counts (persistent small-mesh step)
    bool small_ok = false;           // the device co-schedules the small step's cluster (else: multi-kernel step)
    int subtree_l0 = -1;      // grid walk: first level handed to build_subtree_kernel (-1: none)
    int subtree_nseg = 0;
    cudaEvent_t ev[8] = {};
    int nev = 0;
    // peer-memory exchange (mdc_layout_set_peers)
    int npeer = 0;
    double *peers[2][MDC_MAX_PEERS] = {};
    // all-gather exchange (mdc_layout_set_gather): packed send buffer, and the
    // leaf permutation of the last enqueued step (fixed pointer per plan)
    double *gather_send = nullptr;
    const int32_t *last_perm = nullptr;
    bool timing = false;
    unsigned long long *count = nullptr;  // non-null: instrumented BH launch
    void mark(cudaStream_t s) {
        if (timing && nev < 8) cudaEventRecord(ev[nev++], s);
    }
};

namespace mdc {

// Launch as a programmatic dependent of the stream's previous kernel
// (MDC_LAYOUT_PDL): its CTAs may be scheduled while the predecessor drains;
// the kernel's pdl_wait() orders its reads.  Captured into the step graph as
// programmatic edges.
template <typename... KT, typename... AT>
static cudaError_t launch_pdl(void (*kern)(KT...), dim3 grid, dim3 block, cudaStream_t s, AT &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = MDC_LAYOUT_PDL ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<AT>(args)...);
}

// Builds the tree for pts into b.t; returns the final perm (leaf order).
static int build_tree(MdcLayoutPlan *p, const double *pts, cudaStream_t s, const int32_t **perm_out,
                      bool sample = true) {
    const TreeShape &sh = p->shape;
    Buffers &b = p->b;
    int64_t n = sh.n;
    // one 32-bit key radix sort for both axes + exact-order fixup of equal-key
    // runs (a one-CTA 64-bit block sort was tried for small n: 143 us at any n
    // up to 12k vs ~25 us for this path)
    const int nb2 = (int)((2 * n + 255) / 256);
    if (MDC_SORT_BUCKET) {
        const int64_t B = b.nbucket;
        const int nmm = (int)std::min<int64_t>((n + BK_SAMPLE - 1) / BK_SAMPLE, (int64_t)p->sms);
        const int nsample = sample ? 2 : 0;
        MDC_CHECK_CUDA(launch_pdl(bucket_prep_kernel, dim3(nmm + nsample), dim3(BK_SAMPLE), s, pts, n, b.bk_mm,
                                  b.bk_split, nsample));
        MDC_CHECK_CUDA(launch_pdl(bucket_count_kernel, dim3((unsigned)((2 * n + BK_COUNT_THREADS - 1) / BK_COUNT_THREADS)),
                                  dim3(BK_COUNT_THREADS), s, pts, n, (int)(B / BK_SAMPLE),
                                  (const unsigned long long *)b.bk_mm, (const unsigned long long *)b.bk_split,
                                  b.bk_hist, b.bk_of));
        size_t bytes = b.cub_bytes;
        MDC_CHECK_CUDA(cub::DeviceScan::ExclusiveSum(b.cub_tmp, bytes, b.bk_hist, b.bk_start, (int)(2 * B + 1), s));
        MDC_CHECK_CUDA(launch_pdl(bucket_scatter_kernel, dim3(nb2), dim3(BK_THREADS), s, n,
                                  (const int32_t *)b.bk_of, (const int32_t *)b.bk_start, b.bk_hist, b.bk_slot,
                                  b.bk_mm));
        MDC_CHECK_CUDA(launch_pdl(bucket_rank_kernel, dim3(nb2), dim3(BK_THREADS), s, pts, n,
                                  (const int32_t *)b.bk_of, (const int32_t *)b.bk_start, (const int32_t *)b.bk_slot,
                                  b.xs[0]));
        MDC_CHECK_LAUNCH();
    } else if (n <= MDC_RANK_SORT_MAX) {
        // b.rank (2n) is all-zero between steps: the scatter clears it
        const int bx = (int)((n + RANK_THREADS - 1) / RANK_THREADS);
        int chunks = (4 * p->sms + 2 * bx - 1) / (2 * bx);
        chunks = std::max(1, std::min(chunks, (int)((n + RANK_TILE - 1) / RANK_TILE) * 8));
        const int span = (int)((n + chunks - 1) / chunks);
        chunks = (int)((n + span - 1) / span);
        MDC_CHECK_CUDA(launch_pdl(rank_count_kernel, dim3(bx, 2, chunks), dim3(RANK_THREADS), s, pts, (int)n, span,
                                  b.rank));
        MDC_CHECK_CUDA(launch_pdl(rank_scatter_kernel, dim3(nb2), dim3(256), s, pts, n, b.rank, b.kx_out, b.xs[0]));
        MDC_CHECK_LAUNCH();
    } else {
        MDC_CHECK_CUDA(launch_pdl(keys_kernel, dim3(nb2), dim3(256), s, pts, n, b.kx, b.ids));
        MDC_CHECK_LAUNCH();
        size_t bytes = b.cub_bytes;
        MDC_CHECK_CUDA(cub::DeviceRadixSort::SortPairs(b.cub_tmp, bytes, b.kx, b.kx_out, b.ids, b.xs[0],
                                                       (int)(2 * n), 0, 32, s));
    }
    if (!MDC_SORT_BUCKET) {
        MDC_CHECK_CUDA(launch_pdl(run_mark_kernel, dim3(nb2), dim3(256), s, n,
                                  (const unsigned long long *)b.kx_out, (const int32_t *)b.xs[0], pts, b.runflag));
        MDC_CHECK_CUDA(launch_pdl(run_sort_kernel, dim3(nb2), dim3(256), s, n,
                                  (const unsigned long long *)b.kx_out, b.xs[0], pts, b.runflag));
        MDC_CHECK_LAUNCH();
    }
    p->mark(s);  // sorts done
    BuildArgs ba;
    ba.pts = pts;
    ba.n = n;
    ba.t = b.t;
    ba.max_depth = sh.max_depth;
    ba.nnodes = (int)sh.lo.size();
    ba.xs0 = b.xs[0];
    ba.xs1 = b.xs[1];
    ba.ys0 = b.ys[0];
    ba.ys1 = b.ys[1];
    ba.flag = b.flag;
    ba.oflag = reinterpret_cast<int32_t *>(b.kx_out);  // free after the sorts
    ba.prefix = reinterpret_cast<int32_t *>(b.kx);
    ba.blocksum = b.blocksum;
    if (n <= BUILD_SINGLE_MAX) {
        MDC_CHECK_CUDA(launch_pdl(build_levels_kernel<BUILD_SINGLE_THREADS, BUILD_ONE_CTA>, dim3(1),
                                  dim3(BUILD_SINGLE_THREADS), s, ba));
        MDC_CHECK_LAUNCH();
    } else if (n <= BUILD_CLUSTER_MAX && p->cluster_ok) {
        const bool sub = MDC_BUILD_CLUSTER_SUB && p->subtree_l0 >= 0;
        if (sub) ba.l_end = p->subtree_l0;  // the cluster walks the top levels, one CTA per subtree the rest
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(BUILD_CLUSTER);
        cfg.blockDim = dim3(BUILD_CLUSTER_THREADS);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = BUILD_CLUSTER;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        MDC_CHECK_CUDA(cudaLaunchKernelEx(&cfg, build_levels_kernel<BUILD_CLUSTER_THREADS, BUILD_ONE_CLUSTER>, ba));
        if (sub) {
            MDC_CHECK_CUDA(launch_pdl(build_subtree_kernel, dim3(p->subtree_nseg), dim3(SUBTREE_THREADS), s, ba,
                                      p->subtree_l0));
            MDC_CHECK_CUDA(launch_pdl(centroid_kernel, dim3((unsigned)(((int64_t)ba.nnodes * 32 + 255) / 256)),
                                      dim3(256), s, ba));
            MDC_CHECK_LAUNCH();
        }
    } else {
        if (p->subtree_l0 >= 0) ba.l_end = p->subtree_l0;
        void *kargs[] = {&ba};
        MDC_CHECK_CUDA(cudaLaunchCooperativeKernel((const void *)build_levels_kernel<BUILD_THREADS, BUILD_GRID>,
                                                   dim3(p->build_blocks), dim3(BUILD_THREADS), kargs, 0, s));
        if (p->subtree_l0 >= 0) {
            MDC_CHECK_CUDA(launch_pdl(build_subtree_kernel, dim3(p->subtree_nseg), dim3(SUBTREE_THREADS), s, ba,
                                      p->subtree_l0));
            MDC_CHECK_CUDA(launch_pdl(centroid_kernel, dim3((unsigned)(((int64_t)ba.nnodes * 32 + 255) / 256)),
                                      dim3(256), s, ba));
            MDC_CHECK_LAUNCH();
        }
    }
    p->mark(s);  // tree levels + centroids done
    int cur = sh.max_depth & 1;
    *perm_out = b.xs[cur];
    return MDC_OK;
}

static void part_range(const MdcLayoutPlan *p, int64_t &k0, int64_t &k1) {
    int64_t n = p->shape.n;
    int w = p->a.part_world > 1 ? p->a.part_world : 1;
    int r = p->a.part_world > 1 ? p->a.part_rank : 0;
    k0 = n * r / w;
    k1 = n * (r + 1) / w;
}

static int run_bh(MdcLayoutPlan *p, const double *pts, double *out, cudaStream_t s,
                  const int32_t **perm_out = nullptr, bool sample = true) {
    const int32_t *perm = nullptr;
    int rc = build_tree(p, pts, s, &perm, sample);
    if (rc) return rc;
    int64_t n = p->shape.n, k0, k1;
    part_range(p, k0, k1);
    int64_t warps = (k1 - k0 + 31) / 32;
    if (warps > 0) {
        dim3 grid((unsigned)((warps + BH_WARPS - 1) / BH_WARPS), (unsigned)p->shape.ntask);
        if (p->count)
            bh_kernel<true><<<grid, BH_WARPS * 32, 0, s>>>(n, k0, k1, p->b.t, p->a.c, p->a.eta, p->a.theta, p->count);
        else
            MDC_CHECK_CUDA(launch_pdl(bh_kernel<false>, grid, dim3(BH_WARPS * 32), s, n, k0, k1, p->b.t, p->a.c,
                                      p->a.eta, p->a.theta, (unsigned long long *)nullptr));
        p->mark(s);  // traversal done
        MDC_CHECK_CUDA(launch_pdl(bh_combine_kernel, dim3((unsigned)((k1 - k0 + 255) / 256)), dim3(256), s, n, k0,
                                  k1, p->b.t, perm, out));
        p->mark(s);  // combine done
    }
    MDC_CHECK_LAUNCH();
    if (perm_out) *perm_out = perm;
    return MDC_OK;
}

static int enqueue_step(MdcLayoutPlan *p, const double *pin, double *pout, const double *temps,
                        cudaStream_t s, bool sample = true) {
    int64_t n = p->shape.n;
    const int32_t *perm = nullptr;
    p->mark(s);  // step start
    if (n >= 2) {
        int rc = run_bh(p, pin, p->b.bh, s, &perm, sample);
        if (rc) return rc;
    } else {
        MDC_CHECK_CUDA(cudaMemsetAsync(p->b.bh, 0, sizeof(double) * 2 * (size_t)n, s));
    }
    LocalArgs la;
    la.n = n;
    la.pos = pin;
    la.pos_out = pout;
    la.bh = p->b.bh;
    la.csr_off = p->a.csr_off;
    la.csr_tgt = p->a.csr_tgt;
    la.tris = p->a.tris;
    la.inc_off = p->a.inc_off;
    la.inc = p->a.inc;
    la.spring = p->a.spring;
    la.dlen = p->a.dlen;
    la.eta = p->a.eta;
    la.c = p->a.c;
    la.temps = temps;
    la.ctr = p->b.ctr;
    la.dbg_bh = p->a.dbg_bh;
    la.dbg_force = p->a.dbg_force;
    la.dbg_scale = p->a.dbg_scale;
    la.perm = nullptr;
    la.k0 = 0;
    la.k1 = n;
    la.npeer = 0;
    la.send = nullptr;
    p->last_perm = perm;
    if (p->a.part_world > 1 && perm) {
        part_range(p, la.k0, la.k1);
        la.perm = perm;
        if (p->gather_send) {
            la.send = p->gather_send;  // every slot of pos_out is rewritten by the scatter
        } else if (p->npeer) {
            const int par_out = pout == p->a.pos ? 0 : 1;  // which parity buffer the step writes
            la.npeer = p->npeer;
            for (int r = 0; r < p->npeer; ++r) la.peer_out[r] = p->peers[par_out][r];
        } else {
            MDC_CHECK_CUDA(cudaMemsetAsync(pout, 0, sizeof(double) * 2 * (size_t)n, s));
        }
    }
#if MDC_LOCAL_LG
    if (la.k1 > la.k0 && la.k1 - la.k0 <= MDC_LOCAL_LG_MAXN)
        MDC_CHECK_CUDA(launch_pdl(local_group_kernel<MDC_LOCAL_LG>,
                                  dim3((unsigned)(((la.k1 - la.k0) * MDC_LOCAL_LG + 127) / 128)), dim3(128), s, la));
    else
#endif
        if (la.k1 > la.k0)
            MDC_CHECK_CUDA(launch_pdl(local_kernel, dim3((unsigned)((la.k1 - la.k0 + 127) / 128)), dim3(128), s, la));
    p->mark(s);  // local forces + update done
    MDC_CHECK_CUDA(launch_pdl(incr_kernel, dim3(1), dim3(1), s, p->b.ctr));
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}

}  // namespace mdc

extern "C" size_t mdc_layout_workspace_bytes(int64_t n, int32_t leaf) {
    TreeShape sh;
    make_shape(sh, n, leaf);
    Buffers b;
    return carve(b, nullptr, sh);
}

extern "C" int mdc_layout_plan_create(const MdcLayoutArgs *a, MdcLayoutPlan **plan, void *stream) {
    MDC_REQUIRE(a && plan, "null pointer");
    MDC_REQUIRE(a->n >= 1 && a->n < (1LL << 31), "n out of range");
    MDC_REQUIRE(a->leaf >= 1, "leaf must be >= 1");
    MDC_REQUIRE(a->pos && a->csr_off && a->csr_tgt && a->inc_off && (a->ntri == 0 || (a->tris && a->inc)),
                "null topology pointer");
    MdcLayoutPlan *p = new MdcLayoutPlan();
    p->a = *a;
    make_shape(p->shape, a->n, a->leaf);
    size_t need = carve(p->b, reinterpret_cast<char *>(a->workspace), p->shape);
    if (a->workspace == nullptr || a->workspace_bytes < need) {
        delete p;
        set_error("layout workspace too small: need " + std::to_string(need) + " bytes");
        return MDC_EINVAL;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const TreeShape &sh = p->shape;
    size_t nn = sh.lo.size();
    auto up = [&](int32_t *dst, const std::vector<int32_t> &v) -> int {
        if (!v.empty())
            MDC_CHECK_CUDA(cudaMemcpyAsync(dst, v.data(), v.size() * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        return MDC_OK;
    };
    int rc = 0;
    rc |= up(p->b.t.lo, sh.lo);
    rc |= up(p->b.t.hi, sh.hi);
    rc |= up(p->b.t.left, sh.left);
    rc |= up(p->b.t.right, sh.right);
    rc |= up(p->b.t.nd_list, sh.nd_list);
    rc |= up(p->b.t.seg_lo, sh.seg_lo);
    rc |= up(p->b.t.seg_hi, sh.seg_hi);
    rc |= up(p->b.t.seg_node, sh.seg_node);
    rc |= up(p->b.t.seg_split, sh.seg_split);
    rc |= up(p->b.t.seg_of, sh.seg_of);
    rc |= up(p->b.t.leaves, sh.leaves);
    rc |= up(p->b.t.seg_off, sh.seg_off);
    rc |= up(p->b.t.task_node, sh.task_node);
    rc |= up(p->b.t.task_path, sh.task_path);
    rc |= up(p->b.t.task_first, sh.task_first);
    rc |= up(p->b.t.nd_off, sh.nd_off);
    rc |= up(p->b.t.leaf_lo, sh.leaf_lo);
    rc |= up(p->b.t.leaf_hi, sh.leaf_hi);
    (void)nn;
    if (rc) {
        delete p;
        return MDC_ECUDA;
    }
    {
        int dev = 0, sms = 0, per_sm = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms > 0) p->sms = sms;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, build_levels_kernel<BUILD_THREADS, BUILD_GRID>,
                                                      BUILD_THREADS, 0);
        int want = (int)((p->shape.n + BUILD_THREADS - 1) / BUILD_THREADS);
        p->build_blocks = std::max(1, std::min(std::max(1, per_sm) * sms, want));
        if (p->build_blocks > 1024) p->build_blocks = 1024;  // blocksum capacity below
        // first level whose frontier segments all fit one subtree CTA
        const TreeShape &sh2 = p->shape;
        for (int L = 0; L < sh2.max_depth && SUBTREE_MAX > 0; ++L) {
            int mx = 0;
            for (int g = sh2.seg_off[L]; g < sh2.seg_off[L + 1]; ++g) mx = std::max(mx, sh2.seg_hi[g] - sh2.seg_lo[g]);
            if (mx <= SUBTREE_MAX) {
                p->subtree_l0 = L;
                p->subtree_nseg = sh2.seg_off[L + 1] - sh2.seg_off[L];
                break;
            }
        }
        if (SMALL_CLUSTER > 8)
            cudaFuncSetAttribute(layout_small_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        auto ck = build_levels_kernel<BUILD_CLUSTER_THREADS, BUILD_ONE_CLUSTER>;
        if (BUILD_CLUSTER > 8)
            cudaFuncSetAttribute(ck, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(BUILD_CLUSTER);
        cfg.blockDim = dim3(BUILD_CLUSTER_THREADS);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = BUILD_CLUSTER;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        p->cluster_ok = cudaOccupancyMaxActiveClusters(&nclusters, ck, &cfg) == cudaSuccess && nclusters >= 1;
        cudaGetLastError();  // a refused query leaves the cooperative path in charge
        if (p->shape.n <= MDC_LAYOUT_SMALL_MAX) {
            // the small step's cluster at its largest shared-memory carve (n = SMALL_MAX-sized bound)
            cudaFuncSetAttribute(layout_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
            cudaLaunchConfig_t sc = {};
            sc.gridDim = dim3(SMALL_CLUSTER);
            sc.blockDim = dim3(SMALL_THREADS);
            sc.dynamicSmemBytes = 160 * 1024;
            cudaLaunchAttribute sat[1];
            sat[0].id = cudaLaunchAttributeClusterDimension;
            sat[0].val.clusterDim.x = SMALL_CLUSTER;
            sat[0].val.clusterDim.y = 1;
            sat[0].val.clusterDim.z = 1;
            sc.attrs = sat;
            sc.numAttrs = SMALL_CLUSTER > 1 ? 1 : 0;
            int nsc = 0;
            p->small_ok = SMALL_CLUSTER <= 1 ||
                          (cudaOccupancyMaxActiveClusters(&nsc, layout_small_kernel, &sc) == cudaSuccess && nsc >= 1);
            cudaGetLastError();
        }
    }
    if (p->shape.n <= MDC_LAYOUT_SMALL_MAX) {  // staged topology sizes of the persistent small step
        cudaMemcpyAsync(&p->small_nE, a->csr_off + p->shape.n, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(&p->small_nI, a->inc_off + p->shape.n, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    }
    cudaMemsetAsync(p->b.runflag, 0, sizeof(int32_t) * 2 * (size_t)p->shape.n, s);
    cudaMemsetAsync(p->b.rank, 0, sizeof(int32_t) * 2 * (size_t)p->shape.n, s);
    cudaMemsetAsync(p->b.bk_hist, 0, sizeof(int32_t) * (2 * (size_t)p->b.nbucket + 1), s);
    cudaMemsetAsync(p->b.bk_mm, 0xFF, 4 * sizeof(unsigned long long), s);
    cudaMemsetAsync(p->b.bk_mm + 1, 0, sizeof(unsigned long long), s);
    cudaMemsetAsync(p->b.bk_mm + 3, 0, sizeof(unsigned long long), s);
    // host vectors must outlive the async copies
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        delete p;
        set_error(std::string("plan upload: ") + cudaGetErrorString(e));
        return MDC_ECUDA;
    }
    *plan = p;
    return MDC_OK;
}

extern "C" int mdc_layout_plan_destroy(MdcLayoutPlan *p) {
    if (p)
        for (int i = 0; i < 8; ++i)
            if (p->ev[i]) cudaEventDestroy(p->ev[i]);
    if (!p) return MDC_OK;
    for (auto &g : p->graph)
        if (g) cudaGraphExecDestroy(g);
    if (p->graph_multi) cudaGraphExecDestroy(p->graph_multi);
    if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
    delete p;
    return MDC_OK;
}

#ifndef MDC_LAYOUT_MULTI
#define MDC_LAYOUT_MULTI 32  // steps per multi-step graph (even: the buffer parity returns to 0)
#endif
static_assert(MDC_LAYOUT_MULTI % 2 == 0, "a multi-step graph must span an even number of steps");

extern "C" int mdc_layout_steps(MdcLayoutPlan *p, int32_t k, const double *temps, int32_t use_graph,
                                void *stream) {
    MDC_REQUIRE(p && temps, "null pointer");
    MDC_REQUIRE(k >= 0, "k must be >= 0");
    if (k == 0) return MDC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    MDC_CHECK_CUDA(cudaMemsetAsync(p->b.ctr, 0, sizeof(int32_t), s));
    double *bufs[2] = {p->a.pos, p->b.pos_b};
    bool dbg = p->a.dbg_bh || p->a.dbg_force || p->a.dbg_scale;
    const int64_t n = p->shape.n;
    if (use_graph && !dbg && MDC_LOCAL_LG && p->small_ok && n >= 2 && n <= MDC_LAYOUT_SMALL_MAX && n <= BUILD_SINGLE_MAX &&
        p->a.part_world <= 1) {
        // small mesh: every step of the call in one persistent CTA
        SmallArgs sa;
        BuildArgs &ba = sa.ba;
        ba.pts = nullptr;
        ba.n = n;
        ba.t = p->b.t;
        ba.max_depth = p->shape.max_depth;
        ba.nnodes = (int)p->shape.lo.size();
        ba.xs0 = p->b.xs[0];
        ba.xs1 = p->b.xs[1];
        ba.ys0 = p->b.ys[0];
        ba.ys1 = p->b.ys[1];
        ba.flag = p->b.flag;
        ba.oflag = reinterpret_cast<int32_t *>(p->b.kx_out);
        ba.prefix = reinterpret_cast<int32_t *>(p->b.kx);
        ba.blocksum = p->b.blocksum;
        LocalArgs &la = sa.la;
        la = LocalArgs{};
        la.n = n;
        la.bh = p->b.bh;
        la.csr_off = p->a.csr_off;
        la.csr_tgt = p->a.csr_tgt;
        la.tris = p->a.tris;
        la.inc_off = p->a.inc_off;
        la.inc = p->a.inc;
        la.spring = p->a.spring;
        la.dlen = p->a.dlen;
        la.eta = p->a.eta;
        la.c = p->a.c;
        la.temps = temps;
        la.k0 = 0;
        la.k1 = n;
        sa.bufs[0] = bufs[0];
        sa.bufs[1] = bufs[1];
        sa.k = k;
        sa.c = p->a.c;
        sa.eta = p->a.eta;
        sa.theta = p->a.theta;
        sa.ctr = p->b.ctr;
        sa.nE = p->small_nE;
        sa.nI = p->small_nI;
        sa.ntri = (int)p->a.ntri;
        sa.nn = (int)p->shape.lo.size();
        sa.ns = (int)p->shape.seg_lo.size();
        sa.nl = (int)p->shape.leaves.size();
        {
            SmallSmem mm;
            const size_t smem = small_carve(mm, nullptr, n, sa.nE, sa.nI, sa.ntri, sa.nn, sa.ns, sa.nl,
                                            p->shape.max_depth);
            MDC_CHECK_CUDA(cudaFuncSetAttribute(layout_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)smem));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(SMALL_CLUSTER);
            cfg.blockDim = dim3(SMALL_THREADS);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = SMALL_CLUSTER;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = SMALL_CLUSTER > 1 ? 1 : 0;
            MDC_CHECK_CUDA(cudaLaunchKernelEx(&cfg, layout_small_kernel, sa));
        }
        MDC_CHECK_LAUNCH();
        if (k & 1)
            MDC_CHECK_CUDA(cudaMemcpyAsync(p->a.pos, p->b.pos_b, sizeof(double) * 2 * (size_t)n,
                                           cudaMemcpyDeviceToDevice, s));
        return MDC_OK;
    }
    if (use_graph && !dbg) {
        for (int par = 0; par < 2; ++par) {
            if (p->graph[par]) continue;
            if (!p->cap_stream) MDC_CHECK_CUDA(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
            MDC_CHECK_CUDA(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
            int rc = enqueue_step(p, bufs[par], bufs[par ^ 1], temps, p->cap_stream);
            cudaGraph_t g;
            cudaError_t e = cudaStreamEndCapture(p->cap_stream, &g);
            if (rc) return rc;
            MDC_CHECK_CUDA(e);
            e = cudaGraphInstantiate(&p->graph[par], g, 0);
            cudaGraphDestroy(g);
            MDC_CHECK_CUDA(e);
            p->graph_temps = temps;
        }
        MDC_REQUIRE(p->graph_temps == temps, "temps pointer changed after graph capture");
        int it = 0;
        if (MDC_LAYOUT_MULTI > 1 && k >= MDC_LAYOUT_MULTI) {
            // runs of MDC_LAYOUT_MULTI (even) steps as ONE graph launch: no
            // per-step launch gap, which dominates small meshes (config 1:
            // ~10 tiny kernels per step)
            if (!p->graph_multi) {
                MDC_CHECK_CUDA(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
                int rc = 0;
                for (int j = 0; j < MDC_LAYOUT_MULTI && !rc; ++j)  // sort splitters resampled every 8 steps
                    rc = enqueue_step(p, bufs[j & 1], bufs[(j & 1) ^ 1], temps, p->cap_stream, j % 8 == 0);
                cudaGraph_t g;
                cudaError_t e = cudaStreamEndCapture(p->cap_stream, &g);
                if (rc) return rc;
                MDC_CHECK_CUDA(e);
                e = cudaGraphInstantiate(&p->graph_multi, g, 0);
                cudaGraphDestroy(g);
                MDC_CHECK_CUDA(e);
            }
            for (; it + MDC_LAYOUT_MULTI <= k; it += MDC_LAYOUT_MULTI)
                MDC_CHECK_CUDA(cudaGraphLaunch(p->graph_multi, s));
        }
        for (; it < k; ++it) MDC_CHECK_CUDA(cudaGraphLaunch(p->graph[it & 1], s));
    } else {
        for (int it = 0; it < k; ++it) {
            int rc = enqueue_step(p, bufs[it & 1], bufs[(it & 1) ^ 1], temps, s);
            if (rc) return rc;
        }
    }
    if (k & 1)
        MDC_CHECK_CUDA(cudaMemcpyAsync(p->a.pos, p->b.pos_b, sizeof(double) * 2 * (size_t)p->shape.n,
                                       cudaMemcpyDeviceToDevice, s));
    return MDC_OK;
}

extern "C" int mdc_layout_profile(MdcLayoutPlan *p, const double *temps, float *ms_out, int64_t *counts_out,
                                  void *stream) {
    MDC_REQUIRE(p && temps && ms_out, "null pointer");
    MDC_REQUIRE(p->shape.n >= 2, "profiling needs n >= 2");
    cudaStream_t s = (cudaStream_t)stream;
    int64_t n = p->shape.n;
    // instrumented traversal first (its own launch, outside the timing)
    if (counts_out) {
        unsigned long long *cnt = nullptr;
        MDC_CHECK_CUDA(cudaMallocAsync((void **)&cnt, 4 * sizeof(unsigned long long), s));
        MDC_CHECK_CUDA(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), s));
        p->count = cnt;
        int rc = run_bh(p, p->a.pos, p->b.bh, s);
        p->count = nullptr;
        if (rc) return rc;
        unsigned long long h[4];
        MDC_CHECK_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
        MDC_CHECK_CUDA(cudaStreamSynchronize(s));
        MDC_CHECK_CUDA(cudaFreeAsync(cnt, s));
        for (int i = 0; i < 4; ++i) counts_out[i] = (int64_t)h[i];
    }
    for (int i = 0; i < 8; ++i)
        if (!p->ev[i]) MDC_CHECK_CUDA(cudaEventCreate(&p->ev[i]));
    MDC_CHECK_CUDA(cudaMemsetAsync(p->b.ctr, 0, sizeof(int32_t), s));
    p->nev = 0;
    p->timing = true;
    int rc = enqueue_step(p, p->a.pos, p->b.pos_b, temps, s);
    p->timing = false;
    if (rc) return rc;
    MDC_CHECK_CUDA(cudaMemcpyAsync(p->a.pos, p->b.pos_b, sizeof(double) * 2 * (size_t)n, cudaMemcpyDeviceToDevice, s));
    MDC_CHECK_CUDA(cudaStreamSynchronize(s));
    MDC_REQUIRE(p->nev == 6, "unexpected phase count");
    for (int i = 0; i < 5; ++i) MDC_CHECK_CUDA(cudaEventElapsedTime(&ms_out[i], p->ev[i], p->ev[i + 1]));
    return MDC_OK;
}

extern "C" int mdc_layout_set_peers(MdcLayoutPlan *p, int32_t world, double *const *peers0, double *const *peers1) {
    MDC_REQUIRE(p && peers0 && peers1, "null pointer");
    MDC_REQUIRE(world == p->a.part_world && world >= 2 && world <= MDC_MAX_PEERS,
                "world must equal the plan's part_world (2..8)");
    MDC_REQUIRE(peers0[p->a.part_rank] == p->a.pos, "peers0[rank] must be this plan's position buffer");
    for (int r = 0; r < world; ++r) MDC_REQUIRE(peers0[r] && peers1[r], "null peer buffer");
    for (auto &g : p->graph)
        if (g) {
            cudaGraphExecDestroy(g);
            g = nullptr;
        }
    p->npeer = world;
    for (int r = 0; r < world; ++r) {
        p->peers[0][r] = peers0[r];
        p->peers[1][r] = peers1[r];
    }
    p->b.pos_b = peers1[p->a.part_rank];  // the second parity buffer is this rank's shared one
    return MDC_OK;
}

extern "C" int mdc_layout_step_parity(MdcLayoutPlan *p, int32_t parity, const double *temps, int32_t use_graph,
                                      void *stream) {
    MDC_REQUIRE(p && temps && (parity == 0 || parity == 1), "bad arguments");
    cudaStream_t s = (cudaStream_t)stream;
    double *bufs[2] = {p->a.pos, p->b.pos_b};
    if (!use_graph) return enqueue_step(p, bufs[parity], bufs[parity ^ 1], temps, s);
    if (!p->graph[parity]) {
        if (!p->cap_stream) MDC_CHECK_CUDA(cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking));
        MDC_CHECK_CUDA(cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal));
        int rc = enqueue_step(p, bufs[parity], bufs[parity ^ 1], temps, p->cap_stream);
        cudaGraph_t g;
        cudaError_t e = cudaStreamEndCapture(p->cap_stream, &g);
        if (rc) return rc;
        MDC_CHECK_CUDA(e);
        e = cudaGraphInstantiate(&p->graph[parity], g, 0);
        cudaGraphDestroy(g);
        MDC_CHECK_CUDA(e);
        p->graph_temps = temps;
    }
    MDC_REQUIRE(p->graph_temps == temps, "temps pointer changed after graph capture");
    MDC_CHECK_CUDA(cudaGraphLaunch(p->graph[parity], s));
    return MDC_OK;
}

extern "C" int mdc_layout_set_gather(MdcLayoutPlan *p, double *send) {
    MDC_REQUIRE(p, "null pointer");
    MDC_REQUIRE(p->a.part_world > 1, "the all-gather exchange needs a partitioned plan (part_world > 1)");
    MDC_REQUIRE(!p->graph[0] && !p->graph[1] && !p->graph_multi,
                "set the gather buffer before the first captured step");
    p->gather_send = send;
    return MDC_OK;
}

extern "C" int mdc_layout_scatter(MdcLayoutPlan *p, const double *recv, int64_t chunk, void *stream) {
    MDC_REQUIRE(p && recv, "null pointer");
    MDC_REQUIRE(p->gather_send && p->last_perm, "no partitioned all-gather step has been enqueued");
    const int64_t n = p->shape.n;
    const int w = p->a.part_world;
    MDC_REQUIRE(chunk >= (n + w - 1) / w, "chunk must hold the largest slice, ceil(n / world)");
    if (n == 0) return MDC_OK;
    gather_scatter_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n, w, chunk, p->last_perm,
                                                                                         recv, p->a.pos);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}

extern "C" int mdc_layout_reset_counter(MdcLayoutPlan *p, void *stream) {
    MDC_REQUIRE(p, "null pointer");
    MDC_CHECK_CUDA(cudaMemsetAsync(p->b.ctr, 0, sizeof(int32_t), (cudaStream_t)stream));
    return MDC_OK;
}

extern "C" int mdc_ipc_alloc(size_t bytes, void **ptr, void *handle) {
    MDC_REQUIRE(ptr && handle && bytes > 0, "bad arguments");
    MDC_CHECK_CUDA(cudaMalloc(ptr, bytes));
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, *ptr);
    if (e != cudaSuccess) {
        cudaFree(*ptr);
        *ptr = nullptr;
        MDC_CHECK_CUDA(e);
    }
    memcpy(handle, &h, sizeof(h));
    return MDC_OK;
}

extern "C" int mdc_ipc_open(const void *handle, void **ptr) {
    MDC_REQUIRE(ptr && handle, "bad arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    MDC_CHECK_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return MDC_OK;
}

extern "C" int mdc_ipc_close(void *ptr) {
    MDC_CHECK_CUDA(cudaIpcCloseMemHandle(ptr));
    return MDC_OK;
}

extern "C" int mdc_ipc_free(void *ptr) {
    MDC_CHECK_CUDA(cudaFree(ptr));
    return MDC_OK;
}

extern "C" int mdc_layout_clamp_factors(int64_t n, const double *pos, const double *disp, const int32_t *tris,
                                        const int32_t *inc_off, const int32_t *inc, double eta, double *s_out,
                                        void *stream) {
    MDC_REQUIRE(n >= 0 && pos && disp && inc_off && s_out, "null pointer");
    if (n == 0) return MDC_OK;
    clamp_factors_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(n, pos, disp, tris, inc_off,
                                                                                       inc, eta, s_out);
    MDC_CHECK_LAUNCH();
    return MDC_OK;
}

extern "C" int mdc_layout_repulsion(MdcLayoutPlan *p, const double *pts, double *out, void *stream) {
    MDC_REQUIRE(p && pts && out, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    if (p->shape.n < 2) {
        MDC_CHECK_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * 2 * (size_t)p->shape.n, s));
        return MDC_OK;
    }
    return run_bh(p, pts, out, s);
}

extern "C" int64_t mdc_layout_node_count(const MdcLayoutPlan *p) { return p ? (int64_t)p->shape.lo.size() : 0; }

extern "C" int mdc_layout_kdtree(MdcLayoutPlan *p, const double *pts, int32_t *perm, int32_t *lo,
                                 int32_t *hi, int32_t *left, int32_t *right, double *com,
                                 double *mass, double *size, double *bmin, double *bmax,
                                 void *stream) {
    MDC_REQUIRE(p && pts, "null pointer");
    cudaStream_t s = (cudaStream_t)stream;
    const int32_t *pm = nullptr;
    int rc = build_tree(p, pts, s, &pm);
    if (rc) return rc;
    size_t nn = p->shape.lo.size();
    int64_t n = p->shape.n;
    auto cp = [&](void *dst, const void *src, size_t bytes) -> int {
        if (dst) MDC_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, s));
        return MDC_OK;
    };
    rc |= cp(perm, pm, n * 4);
    rc |= cp(lo, p->b.t.lo, nn * 4);
    rc |= cp(hi, p->b.t.hi, nn * 4);
    rc |= cp(left, p->b.t.left, nn * 4);
    rc |= cp(right, p->b.t.right, nn * 4);
    rc |= cp(com, p->b.t.com, nn * 16);
    rc |= cp(mass, p->b.t.mass, nn * 8);
    rc |= cp(size, p->b.t.size, nn * 8);
    rc |= cp(bmin, p->b.t.bmin, nn * 16);
    rc |= cp(bmax, p->b.t.bmax, nn * 16);
    return rc ? MDC_ECUDA : MDC_OK;
}
