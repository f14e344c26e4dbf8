// tree.cu -- the canonical reduction of per-chunk partials (PAPER.md P:202-206:
// partial sums "stored in an array before the final summation", App. A permanent step 4).
//
// Every walk writes one double-double partial per chunk.  They are combined by ONE fixed binary tree over
// the chunks' absolute indices: node (L+1, k) = node (L, 2k) + node (L, 2k+1) (dd add, left first).  A span
// of chunks [a0, a0+count) -- what one launch, one step or one GPU walked -- reduces to its maximal complete
// nodes: at most two per level, exported sorted by position.  Nodes of disjoint spans then merge on the host
// (perm_c128_tree_combine) into exactly the value a single launch over the union gives, so per(A) is
// bit-identical for any number of GPUs, any slicing of the chunk range into steps, and any grid.
//
// Device side: passes of 8 levels, one 256-thread block per group of 256 nodes; a node is complete when
// all its leaves lie in the span; complete nodes whose parent is not complete are exported.  A finishing
// single-block kernel sorts the exports, writes the fixed-size node array (for the all-gather) and their
// left-to-right sum.
#include "internal.h"

namespace perm {

namespace {

constexpr int kGroup = 256;   // nodes per block and pass (8 levels)

struct TreeWs {
    unsigned count;           // exports so far
    unsigned pad[3];
    TreeNode exp[kTreeMaxNodes];
};

__device__ __forceinline__ void export_node(TreeWs* w, uint32_t level, uint64_t index, const ddc& v) {
    const unsigned k = atomicAdd(&w->count, 1u);
    PERM_DCHECK(k < (unsigned)kTreeMaxNodes);
    if (k < (unsigned)kTreeMaxNodes) {
        w->exp[k].level = level;
        w->exp[k].reserved = 0;
        w->exp[k].index = index;
        w->exp[k].v = v;
    }
}

// in[i] = node (level, a0 + i), i < cnt.  Block b takes group g = (a0 >> 8) + b: its children
// [g*256, g*256 + 256) at `level`, the present ones [lo, hi) relative to the group.
__global__ void __launch_bounds__(kGroup) tree_pass_kernel(const ddc* __restrict__ in, uint64_t a0, uint64_t cnt,
                                                           uint32_t level, ddc* __restrict__ out, uint64_t out_a0,
                                                           TreeWs* w) {
    __shared__ ddc s[kGroup];
    const uint64_t g = (a0 >> 8) + blockIdx.x;
    const uint64_t gb = g << 8;
    const uint64_t end = a0 + cnt;
    const int lo = a0 > gb ? (int)(a0 - gb) : 0;
    const int hi = end < gb + kGroup ? (int)(end - gb) : kGroup;
    const int t = threadIdx.x;
    PERM_DCHECK(lo >= 0 && lo < hi && hi <= kGroup && gb + (uint64_t)hi - a0 <= cnt);
    if (t >= lo && t < hi) s[t] = in[gb + t - a0];
    __syncthreads();
#pragma unroll 1
    for (int sl = 1; sl <= 8; sl++) {
        const int nn = kGroup >> sl;
        bool comp = false;
        ddc v;
        if (t < nn) {
            comp = (t << sl) >= lo && ((t + 1) << sl) <= hi;
            if (comp) {
                v = ddc_add(s[2 * t], s[2 * t + 1]);
            } else {
#pragma unroll
                for (int c = 2 * t; c <= 2 * t + 1; c++)
                    if ((c << (sl - 1)) >= lo && ((c + 1) << (sl - 1)) <= hi)
                        export_node(w, level + sl - 1, (g << (9 - sl)) + (uint64_t)c, s[c]);
            }
        }
        __syncthreads();
        if (comp) s[t] = v;
        __syncthreads();
    }
    PERM_DCHECK(!(t == 0 && lo == 0 && hi == kGroup) || g >= out_a0);
    if (t == 0 && lo == 0 && hi == kGroup) out[g - out_a0] = s[0];
}

// Sort the exports by position, write the node array and the left-to-right sum.
__global__ void tree_finish_kernel(TreeWs* w, TreeNode* __restrict__ nodes, ddc* __restrict__ raw,
                                   ddc* __restrict__ out_dd, double2* __restrict__ out_c, double f) {
    if (threadIdx.x != 0) return;
    unsigned m = w->count;
    PERM_DCHECK(m <= (unsigned)kTreeMaxNodes);
    if (m > (unsigned)kTreeMaxNodes) m = kTreeMaxNodes;   // cannot happen: <= 2 per level
    TreeNode* e = w->exp;
    for (unsigned i = 1; i < m; i++) {                    // insertion sort by first leaf
        TreeNode x = e[i];
        const uint64_t px = x.index << x.level;
        unsigned j = i;
        while (j > 0 && (e[j - 1].index << e[j - 1].level) > px) {
            e[j] = e[j - 1];
            j--;
        }
        e[j] = x;
    }
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    for (unsigned i = 0; i < m; i++) acc = i == 0 ? e[0].v : ddc_add(acc, e[i].v);
    if (nodes) {
        for (unsigned i = 0; i < (unsigned)kTreeMaxNodes; i++) {
            if (i < m) {
                nodes[i] = e[i];
            } else {
                nodes[i].level = kTreeUnused;
                nodes[i].reserved = 0;
                nodes[i].index = 0;
                nodes[i].v.re.hi = nodes[i].v.re.lo = nodes[i].v.im.hi = nodes[i].v.im.lo = 0.0;
            }
        }
    }
    if (raw) *raw = acc;
    if (out_dd || out_c) {
        ddc r = acc;                                      // f = 2(-1)^n: exact in dd
        r.re.hi *= f; r.re.lo *= f; r.im.hi *= f; r.im.lo *= f;
        if (out_dd) *out_dd = r;
        if (out_c) *out_c = make_double2(r.re.hi + r.re.lo, r.im.hi + r.im.lo);
    }
    w->count = 0;                                         // ready for the next use of this workspace
}

size_t round256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace

size_t tree_workspace_bytes(uint64_t count) {
    // level arrays of the passes: ceil-ish count/256 + count/256^2 + ... + a few per pass
    size_t lv = 0;
    for (uint64_t c = count; c > 0; c >>= 8) lv += (c >> 8) + 2;
    return round256(sizeof(TreeWs)) + round256(lv * sizeof(ddc));
}

cudaError_t tree_launch(const ddc* leaves, uint64_t a0, uint64_t count, void* ws, TreeNode* nodes_dev, ddc* raw_dev,
                        ddc* out_dd, double2* out_c, double f, cudaStream_t s, int* launches) {
    TreeWs* w = (TreeWs*)ws;
    ddc* lvbuf = (ddc*)((char*)ws + round256(sizeof(TreeWs)));
    int nl = 0;
    cudaError_t e = cudaMemsetAsync(w, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    const ddc* in = leaves;
    uint64_t a = a0, n = count;
    uint32_t level = 0;
    while (n > 0) {
        const uint64_t g0 = a >> 8, g1 = (a + n - 1) >> 8;
        const uint64_t oa = (a + 255) >> 8, oe = (a + n) >> 8;
        const uint64_t on = oe > oa ? oe - oa : 0;
        const uint64_t ng = g1 - g0 + 1;
        if (ng > 0x7fffffffull) return cudaErrorInvalidValue;
        tree_pass_kernel<<<(unsigned)ng, kGroup, 0, s>>>(in, a, n, level, lvbuf, oa, w);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        nl++;
        in = lvbuf;
        lvbuf += on;
        a = oa;
        n = on;
        level += 8;
    }
    tree_finish_kernel<<<1, 32, 0, s>>>(w, nodes_dev, raw_dev, out_dd, out_c, f);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    nl++;
    if (launches) *launches = nl;
    return cudaSuccess;
}

}  // namespace perm
