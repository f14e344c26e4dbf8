// abi.cu -- the extern "C" boundary of libperm.so (include/perm.h): argument validation, launch
// planning (partition of the Gray-rank range into aligned chunks), workspace
// layout, stream handling and status codes.  All arithmetic of the method runs in the kernels.
#include <cmath>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>

#include "../../include/perm.h"
#include "internal.h"

namespace perm {

cudaError_t malloc_async(void** p, size_t bytes, cudaStream_t s) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    static std::once_flag once[64];
    if (dev >= 0 && dev < 64) {
        std::call_once(once[dev], [](int d) {
            cudaMemPool_t pool;
            if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
                uint64_t thr = UINT64_MAX;
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
            cudaGetLastError();
        }, dev);
    }
    return cudaMallocAsync(p, bytes, s);
}

}  // namespace perm

namespace {

using perm::ddc;
using perm::Segment;

thread_local char g_err[512] = "";
thread_local uint32_t g_launches = 0;

perm_status_t cuda_fail(cudaError_t e, const char* what) {
    snprintf(g_err, sizeof(g_err), "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    return PERM_E_CUDA;
}

#define PERM_CUDA(call, what)                              \
    do {                                                   \
        cudaError_t e_ = (call);                           \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

bool is_device_ptr(const void* p) {
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();   // clear: plain host pointers may report an error on old runtimes
        return false;
    }
    return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

struct WalkPlan {
    int grid = 1;        // blocks of the main launch
    int grid_edge = 0;   // blocks of the edge launch (constant-bank path with unaligned pieces)
    int threads = 0;
    int b = 0;
    int nseg = 0;
    int use_const = 0;
    int body = 0;
    Segment seg[perm::kMaxSegments];
    uint64_t items = 0;
};

int floor_log2(uint64_t x) { return x ? 63 - __builtin_clzll(x) : -1; }

// Chunk length 2^b of the range API for a span of `total` ranks and T resident threads: at least ~128
// chunks per thread so the static round-robin leaves < 1% tail, at least the unrolled block 2^U, at most
// the whole-permanent chunk length walk_chunk_log2(n).
int choose_b(int n, uint64_t total, uint64_t T) {
    const int U = perm::walk_inner_bits(n);
    int b = floor_log2(total / (T * 128ull > 0 ? T * 128ull : 1));
    if (b < U) b = U;
    if (b > perm::walk_chunk_log2(n)) b = perm::walk_chunk_log2(n);
    if (b < U) b = U;
    if (b > n - 1) b = n - 1;
    if (b < 0) b = 0;
    // development override (profiling a sub-range at the full run's chunk length)
    if (const char* f = getenv("PERM_FORCE_CHUNK_LOG2")) {
        const int fb = atoi(f);
        if (fb >= U && fb <= n - 1 && fb <= 30) b = fb;
    }
    return b;
}

// Cut [k0, k1) into maximal aligned pieces of 2^e ranks, e <= b; pieces with 0 < e < U become single
// ranks (e = 0).  Consecutive equal-e pieces merge into one Segment.
bool decompose(int n, uint64_t k0, uint64_t k1, int b, WalkPlan& p) {
    const int U = perm::walk_inner_bits(n);
    p.nseg = 0;
    p.items = 0;
    uint64_t r = k0;
    auto emit = [&](uint64_t c0, uint64_t count, int e) -> bool {
        if (p.nseg > 0) {
            Segment& s = p.seg[p.nseg - 1];
            if (s.e == e && s.c0 + s.count == c0) {
                s.count += count;
                p.items += count;
                return true;
            }
        }
        if (p.nseg >= perm::kMaxSegments) return false;
        p.seg[p.nseg].c0 = c0;
        p.seg[p.nseg].count = count;
        p.seg[p.nseg].e = e;
        p.nseg++;
        p.items += count;
        return true;
    };
    while (r < k1) {
        int e = (r == 0) ? 63 : __builtin_ctzll(r);
        if (e > b) e = b;
        while (e > 0 && (k1 - r) < (1ull << e)) e--;
        if (e < U) e = 0;
        if (e == b && e > 0) {
            const uint64_t cnt = (k1 - r) >> b;          // run of whole 2^b chunks
            if (!emit(r >> b, cnt, b)) return false;
            r += cnt << b;
        } else {
            if (!emit(r >> e, 1, e)) return false;
            r += 1ull << e;
        }
    }
    return true;
}

// Per-(device, n) launch geometry, computed once: resident blocks of the walk kernel, chunk walkers
// (lane groups) per block, resident blocks of the constant-bank kernel (0 if that path does not exist
// for n).  The first query also sets the walk kernel's dynamic shared-memory attribute on that device.
// Read-only after initialisation (std::call_once), so concurrent calls stay safe.
constexpr int kMaxDevices = 64;
struct Geometry {
    std::once_flag once;
    cudaError_t err = cudaSuccess;
    int max_grid = 0, nt = 0, max_grid_c = 0;
};
Geometry g_geom[kMaxDevices][perm::kMaxN + 1];

perm_status_t device_threads(int n, int* max_grid, int* nt, int* max_grid_c = nullptr) {
    int dev = 0;
    PERM_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    if (dev < 0 || dev >= kMaxDevices) return cuda_fail(cudaErrorInvalidDevice, "device index");
    Geometry& G = g_geom[dev][n];
    std::call_once(G.once, [&] {
        int sms = 0, bps = 0, bc = 0;
        G.err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (G.err == cudaSuccess) G.err = perm::walk_occupancy_n(n, &bps, &G.nt);
        if (G.err == cudaSuccess) G.err = perm::walk_occupancy_c_n(n, &bc);
        if (bps < 1) bps = 1;
        G.max_grid = sms * bps;
        G.max_grid_c = sms * bc;
    });
    if (G.err != cudaSuccess) return cuda_fail(G.err, "walk geometry");
    *max_grid = G.max_grid;
    *nt = G.nt;
    if (max_grid_c) *max_grid_c = G.max_grid_c;
    return PERM_OK;
}

// b_req >= 0: walk chunks of exactly 2^b_req ranks (whole permanent, chunk API); else choose_b.
perm_status_t plan_walk(int n, uint64_t k0, uint64_t k1, int b_req, WalkPlan& p) {
    int max_grid = 0, nt = 0, max_grid_c = 0;
    perm_status_t st = device_threads(n, &max_grid, &nt, &max_grid_c);
    if (st != PERM_OK) return st;
    p.threads = nt;
    const uint64_t T = (uint64_t)(max_grid_c > 0 ? max_grid_c * perm::walk_body_walkers(n) : max_grid * nt);
    p.b = b_req >= 0 ? b_req : choose_b(n, k1 - k0, T);
    if (!decompose(n, k0, k1, p.b, p)) {
        snprintf(g_err, sizeof(g_err), "range decomposition exceeded %d segments", perm::kMaxSegments);
        return PERM_E_ARG;
    }
    // constant-bank path for the biggest walked segment (the aligned body)
    p.use_const = 0;
    if (max_grid_c > 0) {
        int best = -1;
        for (int s = 0; s < p.nseg; s++)
            if (p.seg[s].e > perm::walk_inner_bits(n) && (best < 0 || p.seg[s].count > p.seg[best].count)) best = s;
        if (best >= 0) {
            p.use_const = 1;
            p.body = best;
            const uint64_t body = p.seg[best].count;
            const uint64_t wc = perm::walk_body_walkers(n);
            uint64_t need = (body + wc - 1) / wc;
            p.grid = (int)(need < (uint64_t)max_grid_c ? need : (uint64_t)max_grid_c);
            if (p.grid < 1) p.grid = 1;
            const uint64_t rest = p.items - body;
            need = (rest + nt - 1) / nt;
            p.grid_edge = rest == 0 ? 0 : (int)(need < (uint64_t)max_grid ? need : (uint64_t)max_grid);
            return PERM_OK;
        }
    }
    uint64_t need = (p.items + nt - 1) / nt;
    p.grid = (int)(need < (uint64_t)max_grid ? need : (uint64_t)max_grid);
    if (p.grid < 1) p.grid = 1;
    p.grid_edge = 0;
    return PERM_OK;
}

// The results block at the end of the workspace: what a host-output call copies back in one D2H.
struct ResBlock {
    ddc raw;          // left-to-right sum of the maximal tree nodes (raw partial, no 2(-1)^n)
    ddc out_dd;       // raw * 2(-1)^n (whole permanent)
    double2 out_c;    // out_dd rounded
};

struct WsLayout {
    size_t a_off, items_off, tree_off, nodes_off, res_off, total;
};

WsLayout ws_layout(int n, uint64_t items) {
    WsLayout L;
    L.a_off = 0;
    L.items_off = align256((size_t)n * n * sizeof(double2));
    L.tree_off = align256(L.items_off + (size_t)items * sizeof(ddc));
    L.nodes_off = align256(L.tree_off + perm::tree_workspace_bytes(items));
    L.res_off = align256(L.nodes_off + (size_t)perm::kTreeMaxNodes * sizeof(perm::TreeNode));
    L.total = align256(L.res_off + sizeof(ResBlock));
    return L;
}

perm_status_t check_order(int n) { return (n < 1 || n > perm::kMaxN) ? PERM_E_ORDER : PERM_OK; }

bool all_finite(const perm_c128_t* h, size_t cnt) {
    for (size_t k = 0; k < cnt; k++)
        if (!std::isfinite(h[k].re) || !std::isfinite(h[k].im)) return false;
    return true;
}

// Host copy of A when the launch needs it on the host (constant-bank path: the inner columns ride in the
// kernel parameters; the chunk walk and the sparse planner always) or A is host memory; entries are then
// checked here.  A device matrix on the other paths is not copied back: a non-finite entry always makes
// the result non-finite (every Glynn row sum carries each a_ij with coefficient +-1/2), and a host-output
// call checks A only then (nonfinite_status).
perm_status_t host_matrix(const perm_c128_t* A, int n, bool a_dev, bool need_host, cudaStream_t s,
                          std::vector<perm_c128_t>& host, const perm_c128_t** h) {
    const size_t cnt = (size_t)n * n;
    *h = a_dev ? nullptr : A;
    if (a_dev && need_host) {
        host.resize(cnt);
        PERM_CUDA(cudaMemcpyAsync(host.data(), A, cnt * sizeof(perm_c128_t), cudaMemcpyDeviceToHost, s),
                  "cudaMemcpyAsync(A D2H)");
        PERM_CUDA(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        *h = host.data();
    }
    if (*h && !all_finite(*h, cnt)) return PERM_E_NONFINITE;
    return PERM_OK;
}

// A non-finite result of a host-output call: PERM_E_NONFINITE if A has a non-finite entry, else PERM_OK
// (a genuine overflow of the binary64 products, C13).
perm_status_t nonfinite_status(const perm_c128_t* A, int n, cudaStream_t s) {
    std::vector<perm_c128_t> host;
    const perm_c128_t* h = nullptr;
    return host_matrix(A, n, is_device_ptr(A), true, s, host, &h);
}

// Unit-column normalisation (internal.h walk_unit0): A'_ij = a_ij / a_i0 with column 0 set to exactly
// 1, and scale = prod_i a_i0 in double-double (per(A) = scale * per(A') term by term).  false (walk A as is) when the
// order does not use it or a row's column-0 entry is zero or so far from the row's other entries that A' could
// overflow.
bool unit0_normalize(const perm_c128_t* h, int n, std::vector<perm_c128_t>& out, perm::ddc& scale) {
    if (n < 2 || !perm::walk_unit0(n)) return false;
    static const bool enabled = !(getenv("PERM_UNIT0") && atoi(getenv("PERM_UNIT0")) == 0);   // (development)
    if (!enabled) return false;
    out.resize((size_t)n * n);
    scale.re = perm::dd{1.0, 0.0};
    scale.im = perm::dd{0.0, 0.0};
    for (int i = 0; i < n; i++) {
        const double ar = h[(size_t)i * n].re, ai = h[(size_t)i * n].im;
        const double m = std::fabs(ar) > std::fabs(ai) ? std::fabs(ar) : std::fabs(ai);
        if (!(m > 0.0)) return false;
        double rmax = 0.0;
        for (int j = 1; j < n; j++) {
            const double v = std::fabs(h[(size_t)i * n + j].re) + std::fabs(h[(size_t)i * n + j].im);
            rmax = v > rmax ? v : rmax;
        }
        if (rmax / m > 1e100) return false;               // keep |a'_ij| far from overflow
        // 1 / a_i0 = conj(a_i0) / |a_i0|^2, scaled by m to avoid underflow of |a_i0|^2
        const double sr = ar / m, si = ai / m, d = sr * sr + si * si;
        const double ir = sr / (d * m), ii = -si / (d * m);
        out[(size_t)i * n] = perm_c128_t{1.0, 0.0};
        for (int j = 1; j < n; j++) {
            const perm_c128_t a = h[(size_t)i * n + j];
            out[(size_t)i * n + j] = perm_c128_t{a.re * ir - a.im * ii, a.re * ii + a.im * ir};
        }
        perm::ddc f;
        f.re = perm::dd{ar, 0.0};
        f.im = perm::dd{ai, 0.0};
        scale = perm::ddc_mul(scale, f);
    }
    return std::isfinite(scale.re.hi) && std::isfinite(scale.im.hi);
}

// The walk of plan p over A into items (device, p.items entries).  ws_a: device scratch for A if A is host.
perm_status_t launch_walk(const perm_c128_t* A, int n, const WalkPlan& p, ddc* items, char* ws_a, cudaStream_t s,
                          perm_stats_t* stats, uint32_t* launches) {
    const bool a_dev = is_device_ptr(A);
    std::vector<perm_c128_t> host;
    const perm_c128_t* h = nullptr;
    perm_status_t st = host_matrix(A, n, a_dev, p.use_const != 0, s, host, &h);
    if (st != PERM_OK) return st;
    const double2* A_dev = (const double2*)A;
    // unit-column walk (internal.h walk_unit0): A' = D^{-1} A with column 0 all ones, scale = prod_i a_i0
    std::vector<perm_c128_t> unit;
    perm::ddc scale{};
    const bool use_unit = p.use_const && h != nullptr && ws_a != nullptr && unit0_normalize(h, n, unit, scale);
    if (use_unit) {
        PERM_CUDA(cudaMemcpyAsync(ws_a, unit.data(), (size_t)n * n * sizeof(double2), cudaMemcpyHostToDevice, s),
                  "cudaMemcpyAsync(A' H2D)");
        A_dev = (const double2*)ws_a;
        h = unit.data();
    } else if (!a_dev) {
        PERM_CUDA(cudaMemcpyAsync(ws_a, A, (size_t)n * n * sizeof(double2), cudaMemcpyHostToDevice, s),
                  "cudaMemcpyAsync(A H2D)");
        A_dev = (const double2*)ws_a;
    }
    perm::WalkLaunch WL;
    WL.A_dev = A_dev;
    WL.A_host = (const double2*)h;
    WL.unit0 = use_unit ? 1 : 0;
    WL.scaled = use_unit ? 1 : 0;
    WL.scale = scale;
    WL.n = n;
    WL.nseg = p.nseg;
    for (int i = 0; i < p.nseg; i++) WL.seg[i] = p.seg[i];
    WL.items = items;
    WL.nitems = p.items;
    WL.grid = p.grid;
    WL.use_const = p.use_const;
    WL.body = p.body;
    WL.grid_edge = p.grid_edge;
    WL.stream = s;
    if (stats && stats->ev_walk_begin)
        PERM_CUDA(cudaEventRecord((cudaEvent_t)stats->ev_walk_begin, s), "cudaEventRecord");
    if (p.items > 0) PERM_CUDA(perm::walk_launch_n(n, WL), "walk kernel launch");
    if (stats && stats->ev_walk_end)
        PERM_CUDA(cudaEventRecord((cudaEvent_t)stats->ev_walk_end, s), "cudaEventRecord");
    *launches += p.items > 0 ? 1u + (p.grid_edge > 0 ? 1u : 0u) : 0u;
    if (stats) {
        stats->terms = 0;
        for (int i = 0; i < p.nseg; i++) stats->terms += p.seg[i].count << p.seg[i].e;
        stats->chunk_log2 = (uint32_t)p.b;
        stats->blocks = (uint32_t)(p.grid + p.grid_edge);
        stats->threads = (uint32_t)((p.grid + p.grid_edge) * perm::walk_block_threads(n));
        stats->const_path = (uint32_t)p.use_const;
        stats->items = p.items;
    }
    return PERM_OK;
}

// Shared body of perm_c128 (n_final = n, b_req = walk_chunk_log2(n)) and perm_c128_range (n_final = 0):
// walk -> one dd partial per item -> canonical tree over the item index -> left-to-right sum of the
// maximal nodes (for a whole permanent: the root) -> (x 2(-1)^n).  A small whole permanent (n <= 16) is
// one cluster launch that does all of it (walk_small_kernel, same chunks and tree, same bits).
perm_status_t run_walk(const perm_c128_t* A, int n, uint64_t k0, uint64_t k1, int n_final, int b_req, void* out_c,
                       void* out_dd, void* workspace, size_t workspace_bytes, void* stream, perm_stats_t* stats) {
    g_launches = 0;
    cudaStream_t s = (cudaStream_t)stream;
    WalkPlan p;
    perm_status_t st = plan_walk(n, k0, k1, b_req, p);
    if (st != PERM_OK) return st;
    static const bool small_enabled = !(getenv("PERM_SMALL_PATH") && atoi(getenv("PERM_SMALL_PATH")) == 0);
    const bool small = small_enabled && n_final > 0 && n <= perm::kSmallMaxN && p.items <= perm::kSmallMaxChunks &&
                       p.nseg == 1 && k0 == 0 && (p.items & (p.items - 1)) == 0;   // (PERM_SMALL_PATH=0: development)
    const WsLayout L = ws_layout(n, small ? 0 : p.items);
    char* ws = (char*)workspace;
    bool own_ws = false;
    if (ws == nullptr) {
        PERM_CUDA(perm::malloc_async((void**)&ws, L.total, s), "cudaMallocAsync(workspace)");
        own_ws = true;
    } else if (workspace_bytes < L.total) {
        return PERM_E_WORKSPACE;
    }
    perm_status_t result = PERM_OK;
    uint32_t launches = 0;
    ResBlock* res = (ResBlock*)(ws + L.res_off);
    double2* small_c = nullptr;                           // device outputs the small kernel writes directly
    ddc* small_dd = nullptr;
    do {
        cudaError_t e = cudaSuccess;
        if (small) {
            std::vector<perm_c128_t> host;
            const perm_c128_t* h = nullptr;
            const bool a_dev = is_device_ptr(A);
            result = host_matrix(A, n, a_dev, false, s, host, &h);
            if (result != PERM_OK) break;
            const double2* A_dev = (const double2*)A;
            if (!a_dev) {
                e = cudaMemcpyAsync(ws + L.a_off, A, (size_t)n * n * sizeof(double2), cudaMemcpyHostToDevice, s);
                if (e != cudaSuccess) { result = cuda_fail(e, "cudaMemcpyAsync(A H2D)"); break; }
                A_dev = (const double2*)(ws + L.a_off);
            }
            // device outputs are written by the kernel itself (no extra copy node on the latency path)
            if (out_c && is_device_ptr(out_c)) { small_c = (double2*)out_c; }
            if (out_dd && is_device_ptr(out_dd)) { small_dd = (ddc*)out_dd; }
            if (stats && stats->ev_walk_begin) cudaEventRecord((cudaEvent_t)stats->ev_walk_begin, s);
            e = perm::walk_small_launch_n(n, A_dev, p.seg[0].e, p.items, &res->raw, small_dd ? small_dd : &res->out_dd,
                                          small_c ? small_c : &res->out_c, s);
            if (e != cudaSuccess) { result = cuda_fail(e, "small walk launch"); break; }
            if (stats && stats->ev_walk_end) cudaEventRecord((cudaEvent_t)stats->ev_walk_end, s);
            launches = 1;
            if (stats) {
                stats->terms = k1 - k0;
                stats->chunk_log2 = (uint32_t)p.b;
                stats->items = p.items;
                stats->const_path = 0;
                stats->blocks = (uint32_t)(p.items >= 64 ? (p.items / 64 > 16 ? 16 : p.items / 64) : 1);
                stats->threads = (uint32_t)p.items;
            }
        } else {
            result = launch_walk(A, n, p, (ddc*)(ws + L.items_off), ws + L.a_off, s, stats, &launches);
            if (result != PERM_OK) break;
            int tl = 0;
            const double f = n_final > 0 ? ((n_final & 1) ? -2.0 : 2.0) : 0.0;
            e = perm::tree_launch((const ddc*)(ws + L.items_off), 0, p.items, ws + L.tree_off, nullptr, &res->raw,
                                  &res->out_dd, &res->out_c, f, s, &tl);
            if (e != cudaSuccess) { result = cuda_fail(e, "tree kernel launch"); break; }
            launches += (uint32_t)tl;
        }
        const void* src_c = &res->out_c;
        const void* src_dd = n_final > 0 ? (const void*)&res->out_dd : (const void*)&res->raw;
        const bool c_dev = small_c != nullptr || (out_c && is_device_ptr(out_c));
        const bool dd_dev = small_dd != nullptr || (out_dd && is_device_ptr(out_dd));
        if (c_dev && !small_c) {
            e = cudaMemcpyAsync(out_c, src_c, sizeof(double2), cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) { result = cuda_fail(e, "cudaMemcpyAsync(result)"); break; }
        }
        if (dd_dev && !small_dd) {
            e = cudaMemcpyAsync(out_dd, src_dd, sizeof(ddc), cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) { result = cuda_fail(e, "cudaMemcpyAsync(result dd)"); break; }
        }
        const bool host_out = (out_c && !c_dev) || (out_dd && !dd_dev);
        ResBlock hr;
        if (host_out) {
            e = cudaMemcpyAsync(&hr, res, sizeof(ResBlock), cudaMemcpyDeviceToHost, s);
            if (e != cudaSuccess) { result = cuda_fail(e, "cudaMemcpyAsync(result D2H)"); break; }
        }
        if (own_ws) {
            e = cudaFreeAsync(ws, s);
            own_ws = false;
            if (e != cudaSuccess) { result = cuda_fail(e, "cudaFreeAsync(workspace)"); break; }
        }
        if (host_out) {
            e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) { result = cuda_fail(e, "cudaStreamSynchronize"); break; }
            const ddc& v = n_final > 0 ? hr.out_dd : hr.raw;
            if (!(std::isfinite(v.re.hi) && std::isfinite(v.im.hi))) {
                result = nonfinite_status(A, n, s);
                if (result != PERM_OK) break;
            }
            if (out_c && !c_dev) memcpy(out_c, &hr.out_c, sizeof(double2));
            if (out_dd && !dd_dev) memcpy(out_dd, n_final > 0 ? &hr.out_dd : &hr.raw, sizeof(ddc));
        }
    } while (0);
    if (own_ws) cudaFreeAsync(ws, s);
    if (result == PERM_OK) {
        g_launches = launches;
        if (stats) stats->launches = launches;
    }
    return result;
}

// Host merge of tree nodes (tree.cu): siblings (L, 2k), (L, 2k+1) -> (L+1, k) = left + right until none are
// left, then the remaining nodes are summed left to right.  Returns false if nodes overlap.
bool tree_merge(std::vector<perm::TreeNode>& v) {
    auto pos = [](const perm::TreeNode& x) { return x.index << x.level; };
    std::sort(v.begin(), v.end(), [&](const perm::TreeNode& a, const perm::TreeNode& b) { return pos(a) < pos(b); });
    for (size_t i = 1; i < v.size(); i++) {
        const perm::TreeNode& a = v[i - 1];
        const uint64_t end_a = a.level >= 64 ? ~0ull : (a.index + 1) << a.level;
        if (pos(v[i]) < end_a) return false;
    }
    bool merged = true;
    while (merged) {                       // one left-to-right sweep per round; <= 64 rounds
        merged = false;
        std::vector<perm::TreeNode> w;
        w.reserve(v.size());
        for (size_t i = 0; i < v.size(); i++) {
            if (i + 1 < v.size() && v[i].level == v[i + 1].level && (v[i].index & 1ull) == 0 &&
                v[i + 1].index == v[i].index + 1) {
                perm::TreeNode p = v[i];
                p.v = perm::ddc_add(v[i].v, v[i + 1].v);
                p.level += 1;
                p.index >>= 1;
                w.push_back(p);
                i++;
                merged = true;
            } else {
                w.push_back(v[i]);
            }
        }
        v.swap(w);
    }
    return true;
}

}  // namespace

extern "C" {

int perm_version(void) { return 1; }

uint32_t perm_last_launches(void) { return g_launches; }

const char* perm_last_error(void) { return g_err; }

const char* perm_status_string(perm_status_t s) {
    switch (s) {
        case PERM_OK: return "ok";
        case PERM_E_ARG: return "invalid argument";
        case PERM_E_ORDER: return "matrix order out of range";
        case PERM_E_NONFINITE: return "non-finite matrix entry";
        case PERM_E_NOT01: return "entry other than 0 or 1";
        case PERM_E_CUDA: return "CUDA error";
        case PERM_E_WORKSPACE: return "workspace too small";
        case PERM_E_CHECK: return "integer self-check failed (sum not divisible by 2^(n-1))";
    }
    return "unknown status";
}

perm_status_t perm_workspace_bytes(int n, uint64_t k_begin, uint64_t k_end, size_t* bytes) {
    if (!bytes) return PERM_E_ARG;
    perm_status_t st = check_order(n);
    if (st != PERM_OK) return st;
    if (k_begin > k_end) return PERM_E_ARG;
    if (n < 64 && k_end > (1ull << (n - 1))) return PERM_E_ORDER;
    WalkPlan p;
    st = plan_walk(n, k_begin, k_end, -1, p);              // perm_c128_range's plan
    if (st != PERM_OK) return st;
    size_t need = ws_layout(n, p.items).total;
    const int b = perm::walk_chunk_log2(n);                // perm_c128's plan (whole range)
    if (k_begin == 0 && n < 64 && k_end == (1ull << (n - 1))) {
        const size_t full = ws_layout(n, k_end >> b).total;
        if (full > need) need = full;
    }
    *bytes = need;
    return PERM_OK;
}

int perm_chunk_log2(int n) { return (n < 1 || n > perm::kMaxN) ? -1 : perm::walk_chunk_log2(n); }

perm_status_t perm_chunk_walkers(int n, int chunk_log2, uint64_t* walkers) {
    if (!walkers) return PERM_E_ARG;
    perm_status_t st = check_order(n);
    if (st != PERM_OK) return st;
    int max_grid = 0, nt = 0, max_grid_c = 0;
    st = device_threads(n, &max_grid, &nt, &max_grid_c);
    if (st != PERM_OK) return st;
    const bool cbank = max_grid_c > 0 && chunk_log2 > perm::walk_inner_bits(n);
    *walkers = cbank ? (uint64_t)max_grid_c * (uint64_t)perm::walk_body_walkers(n)
                     : (uint64_t)max_grid * (uint64_t)nt;
    return PERM_OK;
}

perm_status_t perm_c128(const perm_c128_t* A, int n, perm_c128_t* out, perm_dd_c128_t* out_dd, void* workspace,
                        size_t workspace_bytes, void* stream, perm_stats_t* stats) {
    if (!A || !out) return PERM_E_ARG;
    perm_status_t st = check_order(n);
    if (st != PERM_OK) return st;
    const uint64_t total = 1ull << (n - 1);
    return run_walk(A, n, 0, total, n, perm::walk_chunk_log2(n), out, out_dd, workspace, workspace_bytes, stream,
                    stats);
}

perm_status_t perm_c128_chunks(const perm_c128_t* A, int n, int chunk_log2, uint64_t c_begin, uint64_t c_end,
                               perm_dd_c128_t* partials_dev, void* workspace, size_t workspace_bytes, void* stream,
                               perm_stats_t* stats) {
    g_launches = 0;
    if (!A || (!partials_dev && c_end > c_begin) || c_begin > c_end) return PERM_E_ARG;
    perm_status_t st = check_order(n);
    if (st != PERM_OK) return st;
    const int U = perm::walk_inner_bits(n);
    const int b = chunk_log2;
    if (b < 0 || b > n - 1 || b > 30 || (b > 0 && b < U)) return PERM_E_ARG;
    if (c_end > (1ull << (n - 1 - b))) return PERM_E_ORDER;
    if (c_begin == c_end) return PERM_OK;                   // empty span: nothing to walk
    if (!is_device_ptr(partials_dev)) return PERM_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    WalkPlan p;
    st = plan_walk(n, c_begin << b, c_end << b, b, p);
    if (st != PERM_OK) return st;
    if (p.items != c_end - c_begin) return PERM_E_ARG;     // cannot happen for b = 0 or b >= U
    const bool a_dev = is_device_ptr(A);
    const size_t a_bytes = (size_t)n * n * sizeof(double2);
    char* ws = (char*)workspace;
    bool own = false;
    if (!ws) {
        // (a device matrix needs scratch only for the unit-column walk's normalised copy)
        PERM_CUDA(perm::malloc_async((void**)&ws, a_bytes, s), "cudaMallocAsync(A)");
        own = true;
    } else if (workspace_bytes < a_bytes) {
        if (!a_dev) return PERM_E_WORKSPACE;
        ws = nullptr;                                       // device A, scratch too small: walk A as given
    }
    uint32_t launches = 0;
    // the chunk walk always checks A on the host (a device matrix is copied back once): it has no
    // result block to carry the staging flag
    std::vector<perm_c128_t> host;
    const perm_c128_t* h = nullptr;
    st = host_matrix(A, n, a_dev, true, s, host, &h);
    if (st == PERM_OK) st = launch_walk(A, n, p, (ddc*)partials_dev, ws, s, stats, &launches);
    if (own) cudaFreeAsync(ws, s);
    if (st != PERM_OK) return st;
    g_launches = launches;
    if (stats) stats->launches = launches;
    return PERM_OK;
}

perm_status_t perm_tree_workspace_bytes(uint64_t count, size_t* bytes) {
    if (!bytes) return PERM_E_ARG;
    *bytes = align256(perm::tree_workspace_bytes(count)) +
             align256((size_t)perm::kTreeMaxNodes * sizeof(perm::TreeNode)) + align256(sizeof(ddc));
    return PERM_OK;
}

perm_status_t perm_c128_tree(const perm_dd_c128_t* partials_dev, uint64_t c_begin, uint64_t c_end,
                             perm_tree_node_t* nodes, perm_dd_c128_t* raw, void* workspace, size_t workspace_bytes,
                             void* stream) {
    g_launches = 0;
    static_assert(sizeof(perm_tree_node_t) == sizeof(perm::TreeNode), "perm_tree_node_t layout");
    static_assert(PERM_TREE_MAX_NODES == perm::kTreeMaxNodes, "PERM_TREE_MAX_NODES");
    if (c_begin > c_end || (c_end > c_begin && !partials_dev) || (!nodes && !raw)) return PERM_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    size_t need = 0;
    perm_tree_workspace_bytes(c_end - c_begin, &need);
    char* ws = (char*)workspace;
    bool own = false;
    if (!ws) {
        PERM_CUDA(perm::malloc_async((void**)&ws, need, s), "cudaMallocAsync(tree workspace)");
        own = true;
    } else if (workspace_bytes < need) {
        return PERM_E_WORKSPACE;
    }
    const size_t nodes_off = align256(perm::tree_workspace_bytes(c_end - c_begin));
    const size_t raw_off = nodes_off + align256((size_t)perm::kTreeMaxNodes * sizeof(perm::TreeNode));
    const bool nodes_dev = nodes && is_device_ptr(nodes);
    const bool raw_dev = raw && is_device_ptr(raw);
    perm::TreeNode* dn = nodes_dev ? (perm::TreeNode*)nodes : (perm::TreeNode*)(ws + nodes_off);
    ddc* dr = raw_dev ? (ddc*)raw : (ddc*)(ws + raw_off);
    perm_status_t result = PERM_OK;
    int tl = 0;
    do {
        cudaError_t e = perm::tree_launch((const ddc*)partials_dev, c_begin, c_end - c_begin, ws, dn, dr, nullptr,
                                          nullptr, 0.0, s, &tl);
        if (e != cudaSuccess) { result = cuda_fail(e, "tree kernel launch"); break; }
        bool sync = false;
        if (nodes && !nodes_dev) {
            e = cudaMemcpyAsync(nodes, dn, (size_t)perm::kTreeMaxNodes * sizeof(perm::TreeNode),
                                cudaMemcpyDeviceToHost, s);
            if (e != cudaSuccess) { result = cuda_fail(e, "cudaMemcpyAsync(nodes)"); break; }
            sync = true;
        }
        if (raw && !raw_dev) {
            e = cudaMemcpyAsync(raw, dr, sizeof(ddc), cudaMemcpyDeviceToHost, s);
            if (e != cudaSuccess) { result = cuda_fail(e, "cudaMemcpyAsync(raw)"); break; }
            sync = true;
        }
        if (own) {
            own = false;
            e = cudaFreeAsync(ws, s);
            if (e != cudaSuccess) { result = cuda_fail(e, "cudaFreeAsync"); break; }
        }
        if (sync) {
            e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) { result = cuda_fail(e, "cudaStreamSynchronize"); break; }
        }
    } while (0);
    if (own) cudaFreeAsync(ws, s);
    if (result == PERM_OK) g_launches = (uint32_t)tl;
    return result;
}

perm_status_t perm_c128_tree_combine(const perm_tree_node_t* nodes, int count, perm_dd_c128_t* raw, int* root_level) {
    if (count < 0 || (count > 0 && !nodes) || !raw) return PERM_E_ARG;
    std::vector<perm::TreeNode> v;
    for (int k = 0; k < count; k++) {
        if (nodes[k].level == perm::kTreeUnused) continue;
        if (nodes[k].level >= 64 || (nodes[k].level > 0 && (nodes[k].index >> (64 - nodes[k].level)) != 0))
            return PERM_E_ARG;
        perm::TreeNode t;
        memcpy(&t, &nodes[k], sizeof(t));
        v.push_back(t);
    }
    if (!tree_merge(v)) return PERM_E_ARG;
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    for (size_t i = 0; i < v.size(); i++) acc = i == 0 ? v[0].v : perm::ddc_add(acc, v[i].v);
    raw->hi_re = acc.re.hi;
    raw->lo_re = acc.re.lo;
    raw->hi_im = acc.im.hi;
    raw->lo_im = acc.im.lo;
    if (root_level) *root_level = (v.size() == 1 && v[0].index == 0) ? (int)v[0].level : -1;
    return PERM_OK;
}

perm_status_t perm_c128_range(const perm_c128_t* A, int n, uint64_t k_begin, uint64_t k_end,
                              perm_dd_c128_t* partial, void* workspace, size_t workspace_bytes, void* stream,
                              perm_stats_t* stats) {
    if (!A || !partial) return PERM_E_ARG;
    perm_status_t st = check_order(n);
    if (st != PERM_OK) return st;
    if (k_begin > k_end) return PERM_E_ARG;
    if (k_end > (1ull << (n - 1))) return PERM_E_ORDER;
    return run_walk(A, n, k_begin, k_end, 0, -1, nullptr, partial, workspace, workspace_bytes, stream, stats);
}

perm_status_t perm_c128_finalize(const perm_dd_c128_t* partials, int count, int n, perm_c128_t* out,
                                 perm_dd_c128_t* out_dd) {
    if (!out || count < 0 || (count > 0 && !partials)) return PERM_E_ARG;
    perm_status_t st = check_order(n);
    if (st != PERM_OK) return st;
    ddc acc;
    acc.re.hi = acc.re.lo = acc.im.hi = acc.im.lo = 0.0;
    for (int k = 0; k < count; k++) {
        ddc v;
        v.re.hi = partials[k].hi_re;
        v.re.lo = partials[k].lo_re;
        v.im.hi = partials[k].hi_im;
        v.im.lo = partials[k].lo_im;
        acc = perm::ddc_add(acc, v);
    }
    const double f = (n & 1) ? -2.0 : 2.0;
    acc.re.hi *= f; acc.re.lo *= f; acc.im.hi *= f; acc.im.lo *= f;
    out->re = acc.re.hi + acc.re.lo;
    out->im = acc.im.hi + acc.im.lo;
    if (out_dd) {
        out_dd->hi_re = acc.re.hi;
        out_dd->lo_re = acc.re.lo;
        out_dd->hi_im = acc.im.hi;
        out_dd->lo_im = acc.im.lo;
    }
    return PERM_OK;
}

perm_status_t perm_c128_batched_x(const perm_c128_t* A_dev, int n, int64_t B, perm_c128_t* per_dev, double* abs2_dev,
                                  double* x_dev, void* stream) {
    g_launches = 0;
    if (B < 0) return PERM_E_ARG;
    if (n < 1 || n > perm::kMaxBatchedN) return PERM_E_ORDER;
    if (B == 0) return PERM_OK;
    if (!A_dev || (!per_dev && !abs2_dev && !x_dev)) return PERM_E_ARG;
    int launches = 0;
    cudaError_t e = perm::batched_launch((const double2*)A_dev, n, B, (double2*)per_dev, abs2_dev, x_dev,
                                         (cudaStream_t)stream, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "batched kernel launch");
    g_launches = (uint32_t)launches;
    return PERM_OK;
}

perm_status_t perm_c128_batched(const perm_c128_t* A_dev, int n, int64_t B, perm_c128_t* per_dev,
                                double* abs2_dev, void* stream) {
    return perm_c128_batched_x(A_dev, n, B, per_dev, abs2_dev, nullptr, stream);
}

// greedypartition (App. B) on the host, as a single scan: the paper repeatedly takes the
// remaining row of least out-degree (lowest index on ties) and discards every row whose support meets the
// taken one.  Visiting the rows once in (degree, index) order and taking a row iff its support is disjoint
// from the union of the supports taken so far selects the same rows in the same order (a skipped row meets
// the union, which only grows; a taken row is the least remaining one).  Returns false if A has a zero
// row or column (per = 0).
static bool sparse_partition(const perm_c128_t* A, int n, perm_sparse_info_t& I) {
    struct Row { int deg, idx; uint64_t supp; };
    std::vector<Row> rows((size_t)n);
    uint64_t cols = 0;
    bool empty_row = false;
    for (int r = 0; r < n; r++) {
        uint64_t m = 0;
        for (int c = 0; c < n; c++) {
            const perm_c128_t z = A[(size_t)r * n + c];
            if (z.re != 0.0 || z.im != 0.0) m |= 1ull << c;
        }
        rows[(size_t)r] = Row{__builtin_popcountll(m), r, m};
        cols |= m;
        empty_row |= (m == 0);
    }
    std::stable_sort(rows.begin(), rows.end(), [](const Row& x, const Row& y) { return x.deg < y.deg; });
    const uint64_t full = n == 64 ? ~0ull : ((1ull << n) - 1ull);
    uint64_t taken = 0;
    I.d = 0;
    for (const Row& r : rows) {
        if (r.supp & taken) continue;          // (a zero row is taken, with S = {}, as in the paper)
        I.smask[I.d++] = r.supp;
        taken |= r.supp;
    }
    I.tmask = full & ~taken;
    I.nt = (uint32_t)__builtin_popcountll(I.tmask);
    const bool zero = empty_row || cols != full;
    double sets = std::ldexp(1.0, (int)I.nt);
    for (uint32_t l = 0; l < I.d; l++) sets *= std::ldexp(1.0, __builtin_popcountll(I.smask[l])) - 1.0;
    I.sets = zero ? 0.0 : sets;
    I.chunk_log2 = -1;
    return !zero;
}

perm_status_t perm_sparse_plan(const perm_c128_t* A_host, int n, perm_sparse_info_t* info) {
    if (!A_host || !info) return PERM_E_ARG;
    if (n < 1 || n > 64) return PERM_E_ORDER;
    for (size_t k = 0; k < (size_t)n * n; k++)
        if (!std::isfinite(A_host[k].re) || !std::isfinite(A_host[k].im)) return PERM_E_NONFINITE;
    memset(info, 0, sizeof(*info));
    sparse_partition(A_host, n, *info);
    return PERM_OK;
}

perm_status_t perm_c128_sparse(const perm_c128_t* A, int n, perm_c128_t* out_host, perm_sparse_info_t* info,
                               void* stream) {
    g_launches = 0;
    if (!A || !out_host) return PERM_E_ARG;
    if (n < 1 || n > perm::kMaxSparseN) return PERM_E_ORDER;
    cudaStream_t s = (cudaStream_t)stream;
    const bool a_dev = is_device_ptr(A);
    std::vector<perm_c128_t> host;
    const perm_c128_t* Ah = nullptr;
    perm_status_t st = host_matrix(A, n, a_dev, true, s, host, &Ah);   // the partition is planned on the host
    if (st != PERM_OK) return st;
    perm_sparse_info_t I;
    memset(&I, 0, sizeof(I));
    if (!sparse_partition(Ah, n, I)) {                    // a zero row or column: per = 0
        out_host->re = 0.0;
        out_host->im = 0.0;
        if (info) *info = I;
        return PERM_OK;
    }
    perm::SparseLaunch L;
    memset(&L, 0, sizeof(L));
    L.n = n;
    L.d = (int)I.d;
    L.nt = (int)I.nt;
    L.A_host = (const double2*)Ah;
    int slot = 0;
    for (int j = 0; j < n; j++)
        if ((I.tmask >> j) & 1ull) L.col[slot++] = j;
    uint64_t outer = 1;
    for (int l = 0; l < L.d; l++) {
        L.soff[l] = slot;
        L.ssz[l] = __builtin_popcountll(I.smask[l]);
        for (int j = 0; j < n; j++)
            if ((I.smask[l] >> j) & 1ull) L.col[slot++] = j;
        outer *= (1ull << L.ssz[l]) - 1ull;
    }
    L.outer = outer;
    for (int i = 0; i < n; i++) L.row[i] = i;
    L.group = 0;
    int dev = 0, sms = 0, bps = 0;
    PERM_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    PERM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "cudaDeviceGetAttribute");
    PERM_CUDA(perm::sparse_occupancy(n, &bps), "sparse occupancy");
    if (bps < 1) bps = 1;
    const uint64_t threads = (uint64_t)sms * bps * perm::walk_block_threads(n);
    // T-walk chunk length: at least ~128 items per thread, at least the unrolled block, at most |T|
    const int U = perm::walk_inner_bits(n);
    int e = 0;
    if (L.nt >= U && U >= 1) {
        const double per_thread = I.sets / ((double)threads * 128.0);
        e = per_thread >= 2.0 ? (int)std::floor(std::log2(per_thread)) : 0;
        if (e > L.nt) e = L.nt;
        if (e > 30) e = 30;
        if (e < U) e = U;
        if (const char* f = getenv("PERM_FORCE_CHUNK_LOG2")) {   // test / profiling override, as in choose_b
            const int fe = atoi(f);
            if (fe >= U && fe <= L.nt && fe <= 30) e = fe;
        }
    }
    L.e = e;
    L.chunks = 1ull << (L.nt - e);
    // shared-rows group walk (sparse.cuh walk_seeded_group), on the constant-bank path (e > U): greedily take the
    // T columns that add the fewest new nonzero rows while their union stays within kSparseGroupRows rows (up to
    // kSparseGroupMaxG columns, G < e); they become T slots 0..G-1 -- the walk's lowest Gray bits; any order of the
    // T columns enumerates the same sets -- and the rows are ordered so that the union's rows come last
    // (per(PA) = per(A)).  PERM_SPARSE_GROUP=g caps G (0: the plain T walk).
    {
        int gmax = perm::kSparseGroupMaxG;
        if (const char* ev = getenv("PERM_SPARSE_GROUP")) gmax = std::min(gmax, std::max(0, atoi(ev)));
        gmax = std::min(gmax, std::min(e - 1, L.nt));
        if (perm::sparse_group_path(n) && e > U && gmax >= 1) {
            std::vector<uint64_t> rows_of((size_t)L.nt, 0);
            for (int q = 0; q < L.nt; q++)
                for (int r = 0; r < n; r++) {
                    const perm_c128_t z = Ah[(size_t)r * n + L.col[q]];
                    if (z.re != 0.0 || z.im != 0.0) rows_of[(size_t)q] |= 1ull << r;
                }
            uint64_t R = 0;
            int G = 0;
            while (G < gmax) {
                int best = -1, bcnt = 65;
                for (int q = G; q < L.nt; q++) {          // slots < G hold the columns taken so far
                    const int cnt = __builtin_popcountll(R | rows_of[(size_t)q]);
                    if (cnt < bcnt) { bcnt = cnt; best = q; }
                }
                if (best < 0 || bcnt > perm::kSparseGroupRows) break;
                std::swap(L.col[G], L.col[best]);
                std::swap(rows_of[(size_t)G], rows_of[(size_t)best]);
                R |= rows_of[(size_t)G];
                G++;
            }
            if (G >= 1) {
                // positions n-M .. n-1: the union's rows, then rows outside it to fill (the thin columns are zero
                // there, so they give every term of a block the same factor)
                int lo = 0, hi = n - perm::kSparseGroupRows;
                for (int r = 0; r < n; r++)
                    if ((R >> r) & 1ull) L.row[hi++] = r;
                for (int r = 0; r < n; r++)
                    if (!((R >> r) & 1ull)) {
                        if (lo < n - perm::kSparseGroupRows) L.row[lo++] = r;
                        else L.row[hi++] = r;
                    }
                L.group = G;
            }
        }
    }
    I.group_cols = L.group;
    const uint64_t items = L.outer * L.chunks;
    const uint64_t bthreads = (uint64_t)perm::walk_block_threads(n);
    uint64_t grid = (items + bthreads - 1) / bthreads;
    if (grid > (uint64_t)sms * bps) grid = (uint64_t)sms * bps;
    L.grid = (int)grid;
    L.stream = s;
    I.chunk_log2 = e;
    char* ws = nullptr;
    const size_t part_bytes = (size_t)L.grid * sizeof(ddc);
    const size_t total = part_bytes + sizeof(ddc) + (a_dev ? 0 : (size_t)n * n * sizeof(double2));
    PERM_CUDA(perm::malloc_async((void**)&ws, total, s), "cudaMallocAsync(sparse workspace)");
    perm_status_t result = PERM_OK;
    do {
        const double2* A_dev = (const double2*)A;
        if (!a_dev) {
            A_dev = (const double2*)(ws + part_bytes + sizeof(ddc));
            cudaError_t e2 = cudaMemcpyAsync((void*)A_dev, A, (size_t)n * n * sizeof(double2), cudaMemcpyHostToDevice, s);
            if (e2 != cudaSuccess) { result = cuda_fail(e2, "cudaMemcpyAsync(A H2D)"); break; }
        }
        L.A_dev = A_dev;
        L.partials = (ddc*)ws;
        cudaError_t e2 = perm::sparse_launch(L);
        if (e2 != cudaSuccess) { result = cuda_fail(e2, "sparse kernel launch"); break; }
        ddc* res = (ddc*)(ws + part_bytes);
        e2 = perm::reduce_launch(L.partials, L.grid, 0, res, nullptr, s);
        if (e2 != cudaSuccess) { result = cuda_fail(e2, "reduce kernel launch"); break; }
        ddc r;
        e2 = cudaMemcpyAsync(&r, res, sizeof(ddc), cudaMemcpyDeviceToHost, s);
        if (e2 == cudaSuccess) e2 = cudaFreeAsync(ws, s);
        ws = nullptr;
        if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(s);
        if (e2 != cudaSuccess) { result = cuda_fail(e2, "sparse result"); break; }
        const double f = (n & 1) ? -1.0 : 1.0;             // (-1)^n
        out_host->re = (r.re.hi + r.re.lo) * f;
        out_host->im = (r.im.hi + r.im.lo) * f;
        g_launches = 2;
    } while (0);
    if (ws) cudaFreeAsync(ws, s);
    if (info) *info = I;
    return result;
}

perm_status_t perm_c128_band_batched(const perm_c128_t* A_dev, int n, int k, int64_t B, perm_c128_t* per_dev,
                                     double* abs2_dev, void* stream) {
    g_launches = 0;
    if (B < 0 || k < 0 || k > perm::kMaxBandK || (n >= 1 && k > n - 1)) return PERM_E_ARG;
    if (n < 1 || n > (1 << 20)) return PERM_E_ORDER;
    if (B == 0) return PERM_OK;
    if (!A_dev || (!per_dev && !abs2_dev)) return PERM_E_ARG;
    int launches = 0;
    cudaError_t e = perm::band_launch((const double2*)A_dev, n, k, B, (double2*)per_dev, abs2_dev,
                                      (cudaStream_t)stream, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "band kernel launch");
    g_launches = (uint32_t)launches;
    return PERM_OK;
}

perm_status_t perm_c128_weighted_batched(const perm_c128_t* C_dev, const int32_t* mult_dev, int n, int R,
                                         int64_t B, perm_c128_t* per_dev, double* abs2_dev, void* stream) {
    g_launches = 0;
    if (B < 0 || R < 1 || R > perm::kMaxWeightedR) return PERM_E_ARG;
    if (n < 1 || n > perm::kMaxBatchedN) return PERM_E_ORDER;
    if (B == 0) return PERM_OK;
    if (!C_dev || !mult_dev || (!per_dev && !abs2_dev)) return PERM_E_ARG;
    int launches = 0;
    cudaError_t e = perm::weighted_launch((const double2*)C_dev, mult_dev, n, R, B, (double2*)per_dev, abs2_dev,
                                          (cudaStream_t)stream, &launches);
    if (e != cudaSuccess) return cuda_fail(e, "weighted kernel launch");
    g_launches = (uint32_t)launches;
    return PERM_OK;
}

perm_status_t perm_int01_workspace_bytes(int n, int64_t B, size_t* bytes) {
    if (!bytes || B < 0) return PERM_E_ARG;
    if (n < 1 || n > perm::kMaxInt01N) return PERM_E_ORDER;
    const int64_t chunk = B < 65535 ? B : 65535;
    *bytes = perm::int01_workspace_bytes(n, chunk > 0 ? chunk : 1);
    return PERM_OK;
}

static perm_status_t run_int(const uint8_t* A_dev, bool pm1, int n, int64_t B, perm_i128_t* out_dev, void* workspace,
                             size_t workspace_bytes, void* stream) {
    g_launches = 0;
    if (B < 0) return PERM_E_ARG;
    if (n < 1 || n > perm::kMaxInt01N) return PERM_E_ORDER;
    if (B == 0) return PERM_OK;
    if (!A_dev || !out_dev) return PERM_E_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t step = 65535;
    const size_t need = perm::int01_workspace_bytes(n, B < step ? B : step);
    char* ws = (char*)workspace;
    bool own = false;
    if (!ws) {
        PERM_CUDA(perm::malloc_async((void**)&ws, need, s), "cudaMallocAsync(workspace)");
        own = true;
    } else if (workspace_bytes < need) {
        return PERM_E_WORKSPACE;
    }
    perm_status_t result = PERM_OK;
    uint32_t launches = 0;
    for (int64_t b0 = 0; b0 < B && result == PERM_OK; b0 += step) {
        const int64_t nb = (B - b0) < step ? (B - b0) : step;
        int flag = 0, l = 0;
        cudaError_t e = perm::int01_launch(A_dev + b0 * n * n, n, nb, pm1, out_dev + b0, ws, need, s, &flag, &l);
        launches += (uint32_t)l;
        if (e != cudaSuccess) result = cuda_fail(e, "int01 kernel");
        else if (flag & 1) result = PERM_E_NOT01;
        else if (flag & 2) result = PERM_E_CHECK;
    }
    if (own) cudaFreeAsync(ws, s);
    if (result == PERM_OK) g_launches = launches;
    return result;
}

perm_status_t perm_int01(const uint8_t* A_dev, int n, int64_t B, perm_i128_t* out_dev, void* workspace,
                         size_t workspace_bytes, void* stream) {
    return run_int(A_dev, false, n, B, out_dev, workspace, workspace_bytes, stream);
}

perm_status_t perm_pm1(const int8_t* A_dev, int n, int64_t B, perm_i128_t* out_dev, void* workspace,
                       size_t workspace_bytes, void* stream) {
    return run_int((const uint8_t*)A_dev, true, n, B, out_dev, workspace, workspace_bytes, stream);
}

perm_status_t perm_int01_range(const uint8_t* A_dev, int n, uint64_t k_begin, uint64_t k_end, perm_i128_t* partial,
                               void* stream) {
    g_launches = 0;
    if (!A_dev || !partial || k_begin > k_end) return PERM_E_ARG;
    if (n < 1 || n > perm::kMaxInt01N) return PERM_E_ORDER;
    const int bits = n > perm::kMaxGlynnInt01N ? n : n - 1;     // rank space of the walk
    if (k_end > (1ull << bits)) return PERM_E_ORDER;
    partial->lo = 0;
    partial->hi = 0;
    if (k_begin == k_end) return PERM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    char* ws = nullptr;
    PERM_CUDA(perm::malloc_async((void**)&ws, perm::int01_range_workspace_bytes(), s), "cudaMallocAsync(workspace)");
    unsigned long long raw[2] = {0, 0};
    int flag = 0, l = 0;
    const cudaError_t e = perm::int01_range_launch(A_dev, n, k_begin, k_end, ws, s, raw, &flag, &l);
    cudaFreeAsync(ws, s);
    if (e != cudaSuccess) return cuda_fail(e, "int01 range kernel");
    if (flag & 1) return PERM_E_NOT01;
    partial->lo = raw[0];
    partial->hi = (int64_t)raw[1];
    g_launches = (uint32_t)l;
    return PERM_OK;
}

perm_status_t perm_int01_finalize(const perm_i128_t* partials, int count, int n, perm_i128_t* out) {
    if (!out || count < 0 || (count > 0 && !partials)) return PERM_E_ARG;
    if (n < 1 || n > perm::kMaxInt01N) return PERM_E_ORDER;
    unsigned __int128 sum = 0;                                  // mod 2^128: exact, order-free
    for (int k = 0; k < count; k++)
        sum += ((unsigned __int128)(uint64_t)partials[k].hi << 64) | (unsigned __int128)partials[k].lo;
    __int128 v;
    if (n > perm::kMaxGlynnInt01N) {                            // full-range Ryser: per = (-1)^{n+1} Sum
        v = (__int128)sum;
        if (!(n & 1)) v = -v;
    } else {
        const unsigned __int128 mask = (((unsigned __int128)1) << (n - 1)) - 1;
        if (sum & mask) return PERM_E_CHECK;
        v = (__int128)sum >> (n - 1);                           // Sum / 2^{n-1}
        if (n & 1) v = -v;                                      // per = (-1)^n Sum / 2^{n-1}
    }
    out->lo = (uint64_t)v;
    out->hi = (int64_t)((unsigned __int128)v >> 64);
    return PERM_OK;
}

perm_status_t perm_c128_seed(const perm_c128_t* A, int n, const uint64_t* ranks, int count, perm_c128_t* w_out,
                             void* stream) {
    g_launches = 0;
    if (!A || !ranks || !w_out || count < 0) return PERM_E_ARG;
    perm_status_t st = check_order(n);
    if (st != PERM_OK) return st;
    for (int k = 0; k < count; k++)
        if (n < 64 && ranks[k] >= (1ull << (n - 1))) return PERM_E_ORDER;
    if (count == 0) return PERM_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const size_t a_bytes = (size_t)n * n * sizeof(double2);
    const size_t r_bytes = (size_t)count * sizeof(uint64_t);
    const size_t w_bytes = (size_t)count * n * sizeof(double2);
    char* ws = nullptr;
    PERM_CUDA(perm::malloc_async((void**)&ws, align256(a_bytes) + align256(r_bytes) + w_bytes, s), "cudaMallocAsync");
    char* a_d = ws;
    char* r_d = ws + align256(a_bytes);
    char* w_d = r_d + align256(r_bytes);
    perm_status_t result = PERM_OK;
    do {
        const bool a_dev = is_device_ptr(A);
        cudaError_t e = cudaMemcpyAsync(a_d, A, a_bytes, a_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(r_d, ranks, r_bytes, cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) { result = cuda_fail(e, "cudaMemcpyAsync"); break; }
        const bool w_dev = is_device_ptr(w_out);
        e = perm::walk_seed_launch_n(n, (const double2*)a_d, (const uint64_t*)r_d, count,
                                     w_dev ? (double2*)w_out : (double2*)w_d, s);
        if (e != cudaSuccess) { result = cuda_fail(e, "seed kernel launch"); break; }
        if (!w_dev) {
            e = cudaMemcpyAsync(w_out, w_d, w_bytes, cudaMemcpyDeviceToHost, s);
            if (e == cudaSuccess) e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) { result = cuda_fail(e, "cudaMemcpyAsync(w)"); break; }
        }
        g_launches = 1;
    } while (0);
    cudaFreeAsync(ws, s);
    return result;
}

perm_status_t perm_fp64_probe(int blocks, int threads, int iters, double* sink_dev, void* stream) {
    if (blocks < 1 || threads < 1 || threads > 1024 || iters < 0 || !sink_dev) return PERM_E_ARG;
    cudaError_t e = perm::fp64_probe_launch(blocks, threads, iters, sink_dev, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "fp64 probe launch");
    g_launches = 1;
    return PERM_OK;
}

}  // extern "C"
