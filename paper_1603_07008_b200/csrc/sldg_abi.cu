// sldg_abi.cu -- host side of the C ABI declared in include/sldg.h.
//
// Owns device memory (two coefficient arrays for ping-pong, weight tables, staging), the
// CUDA stream, the optional NCCL communicator, and the sweep sequencing:
//   validate -> upload field -> build weights (a1, a2) -> [halo exchange] -> sweep (a3-a7)
//   -> swap buffers.
#include <cuda_runtime.h>
#include <float.h>
#include <math.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <string>
#include <vector>

#include "sldg_internal.h"
#include "../../include/sldg_testing.h"

using namespace sldg;

namespace {

thread_local std::string g_last_error;

sldg_status fail(sldg_status st, const std::string& msg)
{
    g_last_error = msg;
    return st;
}

#define CU(call)                                                                                   \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            return fail(e_ == cudaErrorMemoryAllocation ? SLDG_ENOMEM : SLDG_ECUDA,                \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                       \
    } while (0)

#define NC(call)                                                                                   \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess) return fail(SLDG_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

// Balanced block split of n layers over world ranks.
void split(int64_t n, int world, int rank, int64_t* first, int64_t* count)
{
    int64_t base = n / world, extra = n % world;
    *count = base + (rank < extra ? 1 : 0);
    *first = rank * base + std::min<int64_t>(rank, extra);
}

int owner_of(int64_t n, int world, int64_t layer, int64_t* local)
{
    for (int r = 0; r < world; ++r) {
        int64_t f, c;
        split(n, world, r, &f, &c);
        if (layer >= f && layer < f + c) {
            if (local) *local = layer - f;
            return r;
        }
    }
    return -1;
}

// 8 nd + 4 (K - nd) bytes per stored cell (S:163-169 generalised; the paper's (o, d))
size_t bytes_per_cell(const Layout& L) { return (size_t)8 * L.nd + (size_t)4 * (L.K - L.nd); }

// One array: nd fp64 planes per layer, then (K - nd) fp32 planes per layer (sldg_internal.h)
Arrays arrays_of(const Layout& L, void* base)
{
    Arrays a;
    const size_t rows = (size_t)(L.layers + 2 * L.pad) * (size_t)L.L;
    a.mass = (double*)base;
    if (L.prec == SLDG_FP64) a.s64 = a.mass;
    size_t off = ((rows * 8 * (size_t)L.nd + 255) / 256) * 256;
    a.pl = (L.nd < L.K) ? (float*)((char*)base + off) : nullptr;
    return a;
}

size_t array_alloc_bytes(const Layout& L)
{
    const size_t rows = (size_t)(L.layers + 2 * L.pad) * (size_t)L.L;
    return ((rows * 8 * (size_t)L.nd + 255) / 256) * 256 + rows * 4 * (size_t)(L.K - L.nd);
}

sldg_status ensure_weights(sldg_grid g, int64_t n_entries, Weights* wp = nullptr)
{
    Weights& w = wp ? *wp : g->w;
    if (w.cap >= n_entries) return SLDG_OK;
    if (g->capturing)
        return fail(SLDG_EINVAL, "the weight table grows on the first sweep with this many field entries: run the "
                                 "sequence once before capturing it");
    if (&w == &g->w) g->w_const = false;
    cudaFree(w.shift);
    cudaFree(w.smod);
    cudaFree(w.copy);
    cudaFree(w.ab);
    cudaFree(w.rec);
    w = Weights{};
    int64_t cap = std::max<int64_t>(n_entries, 64);
    const int k = g->lay.k;
    CU(cudaMalloc(&w.shift, cap * sizeof(int64_t)));
    CU(cudaMalloc(&w.smod, cap * sizeof(int64_t)));
    CU(cudaMalloc(&w.copy, cap * sizeof(int)));
    CU(cudaMalloc(&w.ab, cap * 2 * k * k * sizeof(double)));
    CU(cudaMalloc(&w.rec, cap * (2 * k * k + 2) * sizeof(double)));
    w.cap = cap;
    return SLDG_OK;
}

sldg_status ensure_field(sldg_grid g, int64_t n)
{
    if (g->field_cap >= n) return SLDG_OK;
    if (g->capturing) return fail(SLDG_EINVAL, "the field buffer grows on first use: run the sequence once before capturing it");
    cudaFree(g->d_field);
    g->d_field = nullptr;
    g->field_cap = 0;
    int64_t cap = std::max<int64_t>(n, 64);
    CU(cudaMalloc(&g->d_field, cap * sizeof(double)));
    g->field_cap = cap;
    return SLDG_OK;
}

// Host shift field -> g->d_field, asynchronously, without retaining the caller's pointer: the
// entries are copied into a pinned staging slot (a ring of kFieldStages; a slot is reused once
// the event after its upload has completed) and uploaded from there on the grid's stream.
static sldg_status upload_host_field(sldg_grid g, const double* field, int64_t n)
{
    sldg_status st = ensure_field(g, n);
    if (st != SLDG_OK) return st;
    constexpr int NS = sldg_grid_s::kFieldStages;
    if (g->fstage_cap < n) {
        for (int s = 0; s < NS; ++s) {
            if (g->fstage_busy[s]) CU(cudaEventSynchronize(g->fstage_ev[s]));
            g->fstage_busy[s] = false;
            if (g->h_fstage[s]) cudaFreeHost(g->h_fstage[s]);
            g->h_fstage[s] = nullptr;
        }
        g->fstage_cap = 0;
        const int64_t cap = std::max<int64_t>(n, 64);
        for (int s = 0; s < NS; ++s) {
            CU(cudaHostAlloc((void**)&g->h_fstage[s], cap * sizeof(double), cudaHostAllocDefault));
            if (!g->fstage_ev[s]) CU(cudaEventCreateWithFlags(&g->fstage_ev[s], cudaEventDisableTiming));
        }
        g->fstage_cap = cap;
    }
    const int s = g->fstage_next;
    g->fstage_next = (s + 1) % NS;
    if (g->fstage_busy[s]) CU(cudaEventSynchronize(g->fstage_ev[s]));
    memcpy(g->h_fstage[s], field, (size_t)n * sizeof(double));
    CU(cudaMemcpyAsync(g->d_field, g->h_fstage[s], (size_t)n * sizeof(double), cudaMemcpyHostToDevice, g->stream));
    CU(cudaEventRecord(g->fstage_ev[s], g->stream));
    g->fstage_busy[s] = true;
    return SLDG_OK;
}

sldg_status ensure_stage(sldg_grid g)
{
    if (g->d_stage) return SLDG_OK;
    const size_t elems = (size_t)1 << 23;  // 64 MiB of fp64 per chunk
    CU(cudaMalloc(&g->d_stage, elems * sizeof(double)));
    CU(cudaMallocHost(&g->h_stage, elems * sizeof(double)));
    g->stage_elems = elems;
    return SLDG_OK;
}

sldg_status check_device_error(sldg_grid g)
{
    int err = 0;
    CU(cudaMemcpyAsync(&err, g->d_err, sizeof(int), cudaMemcpyDeviceToHost, g->stream));
    CU(cudaStreamSynchronize(g->stream));
    if (err) {
        CU(cudaMemsetAsync(g->d_err, 0, sizeof(int), g->stream));
        return fail(SLDG_EINVAL, "a device-resident shift field held a non-finite or |nu| >= 2^62 entry; "
                                 "its lines were left unchanged");
    }
    return SLDG_OK;
}

cudaEvent_t pool_event(sldg_grid g)
{
    if (!g->ev_pool.empty()) {
        cudaEvent_t e = g->ev_pool.back();
        g->ev_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// Launch one sweep kernel over local layers [lb, le) with optional profiling events.
constexpr size_t kTimelineMax = 4096;  // profiled intervals kept for sldg_timeline

sldg_status run_sweep(sldg_grid g, const Sweep& sw, const Arrays& src, const Arrays& dst, int64_t lb, int64_t le,
                      const Layout* lay = nullptr)
{
    const Layout& LY = lay ? *lay : g->lay;
    if (le <= lb) return SLDG_OK;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaEvent_t t0 = nullptr, t1 = nullptr;  // timeline copies (sldg_timeline owns them)
    if (g->profile) {
        e0 = pool_event(g);
        e1 = pool_event(g);
        t0 = pool_event(g);
        t1 = pool_event(g);
        CU(cudaEventRecord(t0, g->stream));
        CU(cudaEventRecord(e0, g->stream));
    }
    int nl = 0;
    CU(launch_sweep(LY, sw, src, dst, lb, le, g->stream, &nl));
    g->launches += nl;
    if (g->profile) {
        CU(cudaEventRecord(e1, g->stream));
        CU(cudaEventRecord(t1, g->stream));
        g->ev_pairs.push_back({e0, e1});
        g->ev_bytes.push_back(2.0 * (double)bytes_per_cell(LY) * (double)((le - lb) * LY.L));
        g->ev_dim.push_back(sw.dim);
        if (g->tl_ev.size() < kTimelineMax) {  // bounded: a long profiled run keeps its first entries
            g->tl_ev.push_back({t0, t1});
            g->tl_kind.push_back(sw.dim);
        } else {
            g->ev_pool.push_back(t0);
            g->ev_pool.push_back(t1);
        }
    }
    return SLDG_OK;
}

// Halo plan for a sweep along the sharded layer dim.  This rank's halo slots are the padded
// local layers [pad-left, pad) (global layers first-left..first-1) and [pad+layers,
// pad+layers+right) (global first+layers..), all mod n.  Entries, in an order both sides of
// every peer pair agree on (the receiver's halo-slot order):
//   kind 0: receive into padded slot `slot` from rank `peer`
//   kind 1: send my padded layer `slot` to rank `peer`
//   kind 2: copy my own padded layer `src` into slot `slot` (wrap-around onto this rank)
struct Xfer {
    int kind;
    int peer;
    int64_t slot;
    int64_t src;
};

std::vector<Xfer> halo_plan(int64_t n, int world, int rank, int64_t pad, int64_t left, int64_t right)
{
    std::vector<Xfer> xs;
    int64_t first, layers;
    split(n, world, rank, &first, &layers);
    for (int64_t j = 0; j < left + right; ++j) {
        int64_t gl = (j < left) ? first - left + j : first + layers + (j - left);
        int64_t slot = (j < left) ? pad - left + j : pad + layers + (j - left);
        gl = ((gl % n) + n) % n;
        int64_t loc = 0;
        int own = owner_of(n, world, gl, &loc);
        if (own == rank) xs.push_back({2, rank, slot, pad + loc});
        else xs.push_back({0, own, slot, 0});
    }
    for (int p = 0; p < world; ++p) {
        if (p == rank) continue;
        int64_t pf, pc;
        split(n, world, p, &pf, &pc);
        for (int64_t j = 0; j < left + right; ++j) {
            int64_t gl = (j < left) ? pf - left + j : pf + pc + (j - left);
            gl = ((gl % n) + n) % n;
            int64_t loc = 0;
            if (owner_of(n, world, gl, &loc) == rank) xs.push_back({1, p, pad + loc, 0});
        }
    }
    return xs;
}

// Halo exchange along the sharded layer dim: this rank receives global layers
// [first-left, first) and [first+layers, first+layers+right) (mod n) into its pad region of
// `a`, and sends whatever other ranks need from its own layers.  Grouped NCCL send/recv on
// the comm stream (two adjacent source cells => halo of ceil|nu| layers).
sldg_status halo_exchange(sldg_grid g, const Arrays& a, int64_t left, int64_t right)
{
    const Layout& L = g->lay;
    const int64_t n = L.n[L.D - 1];
    ncclComm_t comm = (ncclComm_t)g->comm;
    const size_t mass_elems = (size_t)L.L;
    const size_t pl_elems = (size_t)L.L * (size_t)(L.K - 1);
    const size_t s64_elems = (size_t)L.L * (size_t)L.K;
    (void)mass_elems;
    (void)s64_elems;
    (void)pl_elems;
    // one layer of all slots: nd fp64 planes (one chunk) + (K - nd) fp32 planes (one chunk)
    auto layer_ptrs = [&](int64_t lp, void** p0, size_t* c0, void** p1, size_t* c1) {
        const size_t dn = (size_t)L.L * (size_t)L.nd, fn = (size_t)L.L * (size_t)(L.K - L.nd);
        *p0 = a.mass + (size_t)lp * dn;
        *c0 = dn;
        *p1 = fn ? (void*)(a.pl + (size_t)lp * fn) : nullptr;
        *c1 = fn;
    };
    std::vector<Xfer> xs = halo_plan(n, g->world, g->rank, L.pad, left, right);
    for (const Xfer& x : xs) {  // layers this rank owns itself (wrap-around): device copies
        if (x.kind != 2 || g->nccl_self) continue;
        void *d0, *d1, *s0, *s1;
        size_t c0, c1;
        layer_ptrs(x.slot, &d0, &c0, &d1, &c1);
        layer_ptrs(x.src, &s0, &c0, &s1, &c1);
        CU(cudaMemcpyAsync(d0, s0, c0 * 8, cudaMemcpyDeviceToDevice, g->comm_stream));
        if (d1) CU(cudaMemcpyAsync(d1, s1, c1 * 4, cudaMemcpyDeviceToDevice, g->comm_stream));
    }
    bool any = false;
    for (const Xfer& x : xs) any |= (x.kind != 2 || g->nccl_self);
    if (!any) return SLDG_OK;
    NC(ncclGroupStart());
    for (const Xfer& x : xs) {
        if (x.kind == 2) {
            if (!g->nccl_self) continue;
            // SLDG_DIST_NCCL_SELF: the wrap-around copy as a send/recv pair to this rank
            void *d0, *d1, *s0, *s1;
            size_t c0, c1;
            layer_ptrs(x.slot, &d0, &c0, &d1, &c1);
            layer_ptrs(x.src, &s0, &c0, &s1, &c1);
            NC(ncclSend(s0, c0, ncclFloat64, g->rank, comm, g->comm_stream));
            if (s1) NC(ncclSend(s1, c1, ncclFloat32, g->rank, comm, g->comm_stream));
            NC(ncclRecv(d0, c0, ncclFloat64, g->rank, comm, g->comm_stream));
            if (d1) NC(ncclRecv(d1, c1, ncclFloat32, g->rank, comm, g->comm_stream));
            continue;
        }
        void *p0, *p1;
        size_t c0, c1;
        layer_ptrs(x.slot, &p0, &c0, &p1, &c1);
        if (x.kind == 1) {
            NC(ncclSend(p0, c0, ncclFloat64, x.peer, comm, g->comm_stream));
            if (p1) NC(ncclSend(p1, c1, ncclFloat32, x.peer, comm, g->comm_stream));
        } else {
            NC(ncclRecv(p0, c0, ncclFloat64, x.peer, comm, g->comm_stream));
            if (p1) NC(ncclRecv(p1, c1, ncclFloat32, x.peer, comm, g->comm_stream));
        }
    }
    NC(ncclGroupEnd());
    return SLDG_OK;
}

// ---- transpose path of a sweep along the sharded dim (SURVEY 8(e) "When to transpose") ------
// Used when the halo would not fit the pad layers or would move more than the transpose
// (left + right > 2 n_local (P-1)/P).  The slab dim e = D-2 is block-split over the ranks like
// the layer dim: rank r receives, from every rank p, p's layers restricted to r's slab
// [a_r, a_r + s_r) of dim e -- a contiguous inner range of every plane -- so it holds whole lines
// along D-1 for its slab, sweeps them locally (periodic, no halo), and sends them back.
struct TrPart {
    int64_t send_layer_first, send_layer_count, send_slab_first, send_slab_count;
    int64_t recv_layer_first, recv_layer_count, recv_slab_first, recv_slab_count;
};

std::vector<TrPart> transpose_plan(int64_t n_outer, int64_t n_slab, int world, int rank)
{
    std::vector<TrPart> ps(world);
    int64_t f_r, c_r, a_r, s_r;
    split(n_outer, world, rank, &f_r, &c_r);
    split(n_slab, world, rank, &a_r, &s_r);
    for (int p = 0; p < world; ++p) {
        int64_t f_p, c_p, a_p, s_p;
        split(n_outer, world, p, &f_p, &c_p);
        split(n_slab, world, p, &a_p, &s_p);
        ps[p] = {f_r, c_r, a_p, s_p, f_p, c_p, a_r, s_r};
    }
    return ps;
}

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

sldg_status transpose_sweep(sldg_grid g, Sweep sw, const double* dfield, double shift, int64_t n_entries,
                            const Arrays& src, const Arrays& dst)
{
    const Layout& L = g->lay;
    const int D = L.D, e = D - 2, P = g->world, r = g->rank;
    const int64_t Mp = L.S[e];
    const std::vector<TrPart> plan = transpose_plan(L.n[D - 1], L.n[e], P, r);
    const int64_t nl = L.layers, nd = L.nd, nf = L.K - L.nd;
    // slab layout: this rank's slab of dim e, all layers, no pad
    Layout T = L;
    T.n[e] = plan[r].recv_slab_count;
    T.L = Mp * T.n[e];
    T.layers = L.n[D - 1];
    T.first_layer = 0;
    T.pad = 0;
    T.cells = T.layers * T.L;
    const size_t tb = align256(array_alloc_bytes(T));
    // message blocks (this rank's layers x slab p), per peer: fp64 part then fp32 part
    std::vector<size_t> boff(P + 1, 0);
    for (int p = 0; p < P; ++p) {
        const int64_t len = plan[p].send_slab_count * Mp;
        boff[p + 1] = boff[p] + align256((size_t)(nl * nd * len) * 8) + align256((size_t)(nl * nf * len) * 4);
    }
    const size_t need = 2 * tb + boff[P];
    if (g->t_bytes < need && g->capturing)
        return fail(SLDG_EINVAL, "the transpose path's buffers grow on its first use: run the sequence once "
                                 "before capturing it");
    if (g->t_bytes < need) {
        CU(cudaStreamSynchronize(g->stream));
        tmap_cache_forget(g->t_alloc, g->t_bytes);
        cudaFree(g->t_alloc);
        g->t_alloc = nullptr;
        g->t_bytes = 0;
        CU(cudaMalloc(&g->t_alloc, need));
        g->t_bytes = need;
    }
    char* tbase = (char*)g->t_alloc;
    const Arrays Tin = arrays_of(T, tbase), Tout = arrays_of(T, tbase + tb);
    char* stage_inv = tbase + 2 * tb;
    // forward staging: the dst array's memory (overwritten by the unpack at the end) when the
    // padded blocks fit in it; small shards whose 256-byte-aligned blocks do not fit share the
    // inverse staging instead (the forward sends complete, stream-ordered, before the inverse
    // receives land there)
    char* stage_fwd = (boff[P] <= g->alloc_bytes) ? (char*)g->alloc[1 - g->cur] : stage_inv;
    auto bm = [&](char* base, int p) { return (double*)(base + boff[p]); };
    auto bf = [&](char* base, int p) {
        return (float*)(base + boff[p] + align256((size_t)(nl * nd * plan[p].send_slab_count * Mp) * 8));
    };
    const int64_t lenr = plan[r].recv_slab_count * Mp;
    ncclComm_t comm = (ncclComm_t)g->comm;
    cudaStream_t st = g->stream;
    // forward: pack, exchange, self copy
    for (int p = 0; p < P; ++p) {
        CU(launch_tr_block(L, src, nl, plan[p].send_slab_first * Mp, plan[p].send_slab_count * Mp, bm(stage_fwd, p),
                           bf(stage_fwd, p), true, st));
        g->launches += 1;
    }
    const bool via_nccl_self = g->nccl_self;  // SLDG_DIST_NCCL_SELF: own block through NCCL too
    if (P > 1 || via_nccl_self) {
        NC(ncclGroupStart());
        for (int p = 0; p < P; ++p) {
            if (p == r && !via_nccl_self) continue;
            const int64_t len = plan[p].send_slab_count * Mp;
            if (nl * nd * len) NC(ncclSend(bm(stage_fwd, p), (size_t)(nl * nd * len), ncclFloat64, p, comm, st));
            if (nl * nf * len) NC(ncclSend(bf(stage_fwd, p), (size_t)(nl * nf * len), ncclFloat32, p, comm, st));
            const int64_t rf = plan[p].recv_layer_first, rc = plan[p].recv_layer_count;
            if (rc * nd * lenr) NC(ncclRecv(Tin.mass + rf * nd * lenr, (size_t)(rc * nd * lenr), ncclFloat64, p, comm, st));
            if (rc * nf * lenr) NC(ncclRecv(Tin.pl + rf * nf * lenr, (size_t)(rc * nf * lenr), ncclFloat32, p, comm, st));
        }
        NC(ncclGroupEnd());
    }
    if (!via_nccl_self) {
        const int64_t rf = plan[r].recv_layer_first;
        if (nl * nd * lenr)
            CU(cudaMemcpyAsync(Tin.mass + rf * nd * lenr, bm(stage_fwd, r), (size_t)(nl * nd * lenr) * 8,
                               cudaMemcpyDeviceToDevice, st));
        if (nl * nf * lenr)
            CU(cudaMemcpyAsync(Tin.pl + rf * nf * lenr, bf(stage_fwd, r), (size_t)(nl * nf * lenr) * 4,
                               cudaMemcpyDeviceToDevice, st));
    }
    // local sweep of whole lines along D-1 on the slab (periodic, no halo)
    if (T.cells > 0) {
        Sweep swT = sw;
        swT.wrap = 1;
        int64_t n_T = 1;
        for (int d = 0; d < kMaxDim; ++d) {
            swT.fstride[d] = 0;
            if (d < D && (sw.fmask >> d & 1u)) {
                swT.fstride[d] = n_T;
                n_T *= T.n[d];
            }
        }
        const double* fT = nullptr;
        if (dfield) {
            if (g->tfield_cap < n_T && g->capturing)
                return fail(SLDG_EINVAL, "the transpose path's field buffer grows on its first use: run the "
                                         "sequence once before capturing it");
            if (g->tfield_cap < n_T) {
                CU(cudaStreamSynchronize(st));
                cudaFree(g->d_tfield);
                g->d_tfield = nullptr;
                g->tfield_cap = 0;
                CU(cudaMalloc(&g->d_tfield, (size_t)std::max<int64_t>(n_T, 1) * sizeof(double)));
                g->tfield_cap = n_T;
            }
            CU(launch_field_slab(dfield, n_T, sw.fmask, T, L, e, plan[r].recv_slab_first, g->d_tfield, st));
            g->launches += 1;
            fT = g->d_tfield;
        }
        (void)n_entries;
        CU(launch_weights(T, T.n[D - 1], fT, shift, n_T, g->w, g->d_err, st));
        g->launches += 1;
        g->w_const = false;
        swT.shift = g->w.shift;
        swT.smod = g->w.smod;
        swT.copy = g->w.copy;
        swT.ab = g->w.ab;
        swT.rec = g->w.rec;
        sldg_status s2 = run_sweep(g, swT, Tin, Tout, 0, T.layers, &T);
        if (s2 != SLDG_OK) return s2;
    }
    // inverse: exchange back, self copy, unpack into dst
    if (P > 1 || via_nccl_self) {
        NC(ncclGroupStart());
        for (int p = 0; p < P; ++p) {
            if (p == r && !via_nccl_self) continue;
            const int64_t rf = plan[p].recv_layer_first, rc = plan[p].recv_layer_count;
            if (rc * nd * lenr) NC(ncclSend(Tout.mass + rf * nd * lenr, (size_t)(rc * nd * lenr), ncclFloat64, p, comm, st));
            if (rc * nf * lenr) NC(ncclSend(Tout.pl + rf * nf * lenr, (size_t)(rc * nf * lenr), ncclFloat32, p, comm, st));
            const int64_t len = plan[p].send_slab_count * Mp;
            if (nl * nd * len) NC(ncclRecv(bm(stage_inv, p), (size_t)(nl * nd * len), ncclFloat64, p, comm, st));
            if (nl * nf * len) NC(ncclRecv(bf(stage_inv, p), (size_t)(nl * nf * len), ncclFloat32, p, comm, st));
        }
        NC(ncclGroupEnd());
    }
    if (!via_nccl_self) {
        const int64_t rf = plan[r].recv_layer_first;
        if (nl * nd * lenr)
            CU(cudaMemcpyAsync(bm(stage_inv, r), Tout.mass + rf * nd * lenr, (size_t)(nl * nd * lenr) * 8,
                               cudaMemcpyDeviceToDevice, st));
        if (nl * nf * lenr)
            CU(cudaMemcpyAsync(bf(stage_inv, r), Tout.pl + rf * nf * lenr, (size_t)(nl * nf * lenr) * 4,
                               cudaMemcpyDeviceToDevice, st));
    }
    for (int p = 0; p < P; ++p) {
        CU(launch_tr_block(L, dst, nl, plan[p].send_slab_first * Mp, plan[p].send_slab_count * Mp, bm(stage_inv, p),
                           bf(stage_inv, p), false, st));
        g->launches += 1;
    }
    g->transposes += 1;
    return SLDG_OK;
}

// bounded: the caller guarantees every field entry lies in [nu_lo, nu_hi] (sldg_advect_device_bounded);
// the halo plan is sized from that bound instead of a device -> host read of the field's range
sldg_status advect_impl(sldg_grid g, int dim, double shift, const double* field, bool field_on_device,
                        uint32_t mask, bool bounded = false, double nu_lo = 0.0, double nu_hi = 0.0)
{
    const Layout& L = g->lay;
    if (dim < 0 || dim >= L.D) return fail(SLDG_EINVAL, "dim out of range");
    if (mask >> L.D) return fail(SLDG_EINVAL, "field_mask has bits >= ndim");
    if (field && (mask & (1u << dim))) return fail(SLDG_EINVAL, "field_mask contains the advected dim");
    if (!field && mask) return fail(SLDG_EINVAL, "field_mask given without a field");
    int64_t n_entries = 1;
    Sweep sw{};
    sw.dim = dim;
    sw.nd = L.n[dim];
    sw.fmask = field ? mask : 0;
    {
        int64_t st = 1;
        for (int e = 0; e < kMaxDim; ++e) {
            sw.fstride[e] = 0;
            if (e < L.D && (sw.fmask >> e & 1u)) {
                sw.fstride[e] = st;
                st *= L.n[e];
            }
        }
        n_entries = st;
    }
    const bool sharded_sweep = (g->halo_mode && dim == L.D - 1);
    int64_t imin = 0, imax = 0;
    int64_t ilo = INT64_MIN, ihi = INT64_MAX;  // device-checked bound of the field's i*
    auto int_part = [](double nu) {
        const double fl = floor(nu);
        return (int64_t)fl + ((nu - fl >= 1.0) ? 1 : 0);
    };
    if (bounded) {
        if (!field) return fail(SLDG_EINVAL, "a shift bound needs a field");
        if (!(fabs(nu_lo) < 4.611686018427387904e18) || !(fabs(nu_hi) < 4.611686018427387904e18) || nu_lo > nu_hi)
            return fail(SLDG_EINVAL, "shift bound must be finite with nu_min <= nu_max");
        ilo = imin = int_part(nu_lo);
        ihi = imax = int_part(nu_hi);
    }
    if (sharded_sweep && field && field_on_device && !bounded && g->capturing)
        return fail(SLDG_EINVAL, "a device-field sweep along the sharded dim inside a graph capture needs a shift "
                                 "bound (sldg_advect_device_bounded): its halo is sized on the host");
    if (bounded) {
    } else if (!field) {
        if (!(fabs(shift) < 4.611686018427387904e18)) return fail(SLDG_EINVAL, "non-finite or huge shift");
        double fl = floor(shift);
        imin = imax = (int64_t)fl + ((shift - fl >= 1.0) ? 1 : 0);
    } else if (!field_on_device) {
        imin = INT64_MAX;
        imax = INT64_MIN;
        for (int64_t e = 0; e < n_entries; ++e) {
            double nu = field[e];
            if (!(fabs(nu) < 4.611686018427387904e18))
                return fail(SLDG_EINVAL, "non-finite or |nu| >= 2^62 entry in shift field");
            double fl = floor(nu);
            int64_t is = (int64_t)fl + ((nu - fl >= 1.0) ? 1 : 0);
            imin = std::min(imin, is);
            imax = std::max(imax, is);
        }
    }
    sldg_status st = ensure_weights(g, n_entries);
    if (st != SLDG_OK) return st;
    const double* dfield = nullptr;
    if (field) {
        if (field_on_device) {
            dfield = field;
        } else {
            st = upload_host_field(g, field, n_entries);
            if (st != SLDG_OK) return st;
            dfield = g->d_field;
        }
    }
    if (sharded_sweep && field && field_on_device && !bounded) {
        CU(launch_field_range(dfield, n_entries, shift, g->d_range, g->stream));
        int64_t r[2];
        CU(cudaMemcpyAsync(r, g->d_range, sizeof(r), cudaMemcpyDeviceToHost, g->stream));
        CU(cudaStreamSynchronize(g->stream));
        imin = r[0];
        imax = r[1];
        if (imin > imax) imin = imax = 0;  // all entries invalid: lines are copied (error sticky)
    }
    if (field || !g->w_const || g->w_shift != shift || g->w_n != sw.nd) {
        CU(launch_weights(L, sw.nd, dfield, shift, n_entries, g->w, g->d_err, g->stream, ilo, ihi));
        g->launches += 1;
        g->w_const = !field;
        g->w_shift = shift;
        g->w_n = sw.nd;
    }
    sw.shift = g->w.shift;
    sw.smod = g->w.smod;
    sw.copy = g->w.copy;
    sw.ab = g->w.ab;
    sw.rec = g->w.rec;

    const Arrays& src = g->buf[g->cur];
    const Arrays& dst = g->buf[1 - g->cur];
    if (!sharded_sweep) {
        sw.wrap = 1;
        st = run_sweep(g, sw, src, dst, 0, L.layers);
        if (st != SLDG_OK) return st;
    } else {
        int64_t left = std::max<int64_t>(0, imax + 1), right = std::max<int64_t>(0, -imin);
        const int P = g->world;
        if (g->peer_halo && !g->force_transpose && left <= L.pad && right <= L.pad) {
            // the pads ARE the neighbours' edge layers: one launch over all local layers, its pad
            // boxes read the neighbours' memory directly; fences order it against their sweeps
            sw.wrap = 0;
            CU(peer_fence(g));
            st = run_sweep(g, sw, src, dst, 0, L.layers);
            if (st != SLDG_OK) return st;
            CU(peer_fence(g));
            g->cur = 1 - g->cur;
            return SLDG_OK;
        }
        if (g->force_transpose || left > L.pad || right > L.pad ||
            (P > 1 && (left + right) * P > 2 * L.layers * (P - 1))) {
            st = transpose_sweep(g, sw, dfield, shift, n_entries, src, dst);
            if (st != SLDG_OK) return st;
            g->cur = 1 - g->cur;
            return SLDG_OK;
        }
        sw.wrap = 0;
        CU(cudaEventRecord(g->ev_ready, g->stream));
        CU(cudaStreamWaitEvent(g->comm_stream, g->ev_ready, 0));
        cudaEvent_t h0 = nullptr, h1 = nullptr;
        if (g->profile) {
            h0 = pool_event(g);
            h1 = pool_event(g);
            CU(cudaEventRecord(h0, g->comm_stream));
        }
        st = halo_exchange(g, src, left, right);
        if (st != SLDG_OK) return st;
        if (g->profile) {
            CU(cudaEventRecord(h1, g->comm_stream));
            if (g->tl_ev.size() < kTimelineMax) {
                g->tl_ev.push_back({h0, h1});
                g->tl_kind.push_back(-1);
            } else {
                g->ev_pool.push_back(h0);
                g->ev_pool.push_back(h1);
            }
        }
        CU(cudaEventRecord(g->ev_halo, g->comm_stream));
        // interior layers need no halo: overlap them with the exchange, leaving comm_sms SMs to
        // the NCCL kernel (a persistent sweep CTA and an NCCL CTA do not fit one SM together)
        int64_t ib = std::min(left, L.layers), ie = std::max(ib, L.layers - right);
        const bool exchange = (P > 1 || g->nccl_self) && (left + right) > 0;
        Sweep swi = sw;
        swi.sm_reserve = exchange ? g->comm_sms : 0;
        st = run_sweep(g, swi, src, dst, ib, ie);
        if (st != SLDG_OK) return st;
        CU(cudaStreamWaitEvent(g->stream, g->ev_halo, 0));
        st = run_sweep(g, sw, src, dst, 0, ib);
        if (st != SLDG_OK) return st;
        st = run_sweep(g, sw, src, dst, ie, L.layers);
        if (st != SLDG_OK) return st;
    }
    g->cur = 1 - g->cur;
    return SLDG_OK;
}

// sldg_advect_pair: the dim-0 sweep then the dim-1 sweep, in one pass when fused_plan accepts
// the shapes and fields (sldg_fused.cu), else as the two sweeps.
sldg_status advect_pair_impl(sldg_grid g, double shift0, const double* f0, uint32_t m0, double shift1,
                             const double* f1, uint32_t m1, bool on_device)
{
    const Layout& L = g->lay;
    if (L.D < 2) return fail(SLDG_EINVAL, "a sweep pair needs dims 0 and 1");
    auto make_sweep = [&](int dim, const double* f, uint32_t mask, int64_t* n_entries) -> sldg_status {
        if (mask >> L.D) return fail(SLDG_EINVAL, "field_mask has bits >= ndim");
        if (f && (mask & (1u << dim))) return fail(SLDG_EINVAL, "field_mask contains the advected dim");
        if (!f && mask) return fail(SLDG_EINVAL, "field_mask given without a field");
        *n_entries = 1;
        for (int e = 0; e < L.D; ++e)
            if (f && (mask >> e & 1u)) *n_entries *= L.n[e];
        return SLDG_OK;
    };
    int64_t ne0 = 1, ne1 = 1;
    sldg_status st = make_sweep(0, f0, m0, &ne0);
    if (st != SLDG_OK) return st;
    st = make_sweep(1, f1, m1, &ne1);
    if (st != SLDG_OK) return st;
    auto sweep_of = [&](int dim, const double* f, uint32_t mask) {
        Sweep sw{};
        sw.dim = dim;
        sw.nd = L.n[dim];
        sw.fmask = f ? mask : 0;
        sw.wrap = 1;
        int64_t stv = 1;
        for (int e = 0; e < kMaxDim; ++e) {
            sw.fstride[e] = 0;
            if (e < L.D && (sw.fmask >> e & 1u)) {
                sw.fstride[e] = stv;
                stv *= L.n[e];
            }
        }
        return sw;
    };
    if (!on_device && g->capturing && (f0 || f1))
        return fail(SLDG_EINVAL, "a host shift field cannot be captured in a graph: use sldg_advect_pair_device");
    Sweep s0 = sweep_of(0, f0, m0), s1 = sweep_of(1, f1, m1);
    FusedPlan fp;
    // dim 1 must not be the sharded layer dim (D >= 3); both fields constant over dims 0, 1
    const bool fuse = L.D >= 3 && fused_plan(L, s0, s1, &fp);
    if (!fuse) {
        st = advect_impl(g, 0, shift0, f0, on_device, m0);
        if (st != SLDG_OK) return st;
        return advect_impl(g, 1, shift1, f1, on_device, m1);
    }
    if (!on_device) {
        for (int pass = 0; pass < 2; ++pass) {
            const double* f = pass ? f1 : f0;
            const int64_t n = pass ? ne1 : ne0;
            const double sh = pass ? shift1 : shift0;
            if (!f) {
                if (!(fabs(sh) < 4.611686018427387904e18)) return fail(SLDG_EINVAL, "non-finite or huge shift");
                continue;
            }
            for (int64_t e = 0; e < n; ++e)
                if (!(fabs(f[e]) < 4.611686018427387904e18))
                    return fail(SLDG_EINVAL, "non-finite or |nu| >= 2^62 entry in shift field");
        }
    }
    st = ensure_weights(g, ne0);
    if (st != SLDG_OK) return st;
    st = ensure_weights(g, ne1, &g->w2);
    if (st != SLDG_OK) return st;
    // weights of each sweep (a host field goes through the pinned staging ring, stream-ordered
    // before its weight build)
    const double* d0 = f0;
    if (f0 && !on_device) {
        st = upload_host_field(g, f0, ne0);
        if (st != SLDG_OK) return st;
        d0 = g->d_field;
    }
    CU(launch_weights(L, L.n[0], d0, shift0, ne0, g->w, g->d_err, g->stream));
    g->launches += 1;
    g->w_const = false;
    const double* d1 = f1;
    if (f1 && !on_device) {
        st = upload_host_field(g, f1, ne1);
        if (st != SLDG_OK) return st;
        d1 = g->d_field;
    }
    CU(launch_weights(L, L.n[1], d1, shift1, ne1, g->w2, g->d_err, g->stream));
    g->launches += 1;
    s0.shift = g->w.shift;
    s0.smod = g->w.smod;
    s0.copy = g->w.copy;
    s0.ab = g->w.ab;
    s0.rec = g->w.rec;
    s1.shift = g->w2.shift;
    s1.smod = g->w2.smod;
    s1.copy = g->w2.copy;
    s1.ab = g->w2.ab;
    s1.rec = g->w2.rec;
    cudaEvent_t e0 = nullptr, e1 = nullptr, t0 = nullptr, t1 = nullptr;
    if (g->profile) {
        e0 = pool_event(g);
        e1 = pool_event(g);
        t0 = pool_event(g);
        t1 = pool_event(g);
        CU(cudaEventRecord(t0, g->stream));
        CU(cudaEventRecord(e0, g->stream));
    }
    CU(launch_fused01(L, s0, s1, g->buf[g->cur], g->buf[1 - g->cur], fp, g->stream));
    g->launches += 1;
    if (g->profile) {
        CU(cudaEventRecord(e1, g->stream));
        CU(cudaEventRecord(t1, g->stream));
        g->ev_pairs.push_back({e0, e1});
        g->ev_bytes.push_back(2.0 * (double)bytes_per_cell(L) * (double)L.cells);  // ONE read + write: two sweeps
        g->ev_dim.push_back(kMaxDim);
        if (g->tl_ev.size() < kTimelineMax) {
            g->tl_ev.push_back({t0, t1});
            g->tl_kind.push_back(-2);
        } else {
            g->ev_pool.push_back(t0);
            g->ev_pool.push_back(t1);
        }
    }
    g->cur = 1 - g->cur;
    return SLDG_OK;
}

sldg_status advect_vnodes_impl(sldg_grid g, int dim, int vdim, const double* nodal, bool on_device)
{
    const Layout& L = g->lay;
    if (dim < 0 || dim >= L.D || vdim < 0 || vdim >= L.D || dim == vdim)
        return fail(SLDG_EINVAL, "dim and vdim must be distinct dims of the grid");
    if (!nodal) return fail(SLDG_EINVAL, "null nodal field");
    if (L.k > 4) return fail(SLDG_ENOTSUP, "the Gauss-node sweep supports k <= 4");
    if (g->halo_mode && dim == L.D - 1) return fail(SLDG_ENOTSUP, "Gauss-node sweep along the sharded dim");
    const int64_t nv = L.n[vdim], n_entries = nv * L.k;
    const double* dn = nodal;
    if (!on_device) {
        for (int64_t i = 0; i < n_entries; ++i)
            if (!(fabs(nodal[i]) < 4.611686018427387904e18))
                return fail(SLDG_EINVAL, "non-finite or |nu| >= 2^62 entry in the nodal field");
        sldg_status st = upload_host_field(g, nodal, n_entries);  // copied before return (pinned ring)
        if (st != SLDG_OK) return st;
        dn = g->d_field;
    }
    const int64_t words = vnode_rec_words(L.k) * nv;
    if (g->vnrec_cap < words) {
        CU(cudaStreamSynchronize(g->stream));
        cudaFree(g->d_vnrec);
        g->d_vnrec = nullptr;
        g->vnrec_cap = 0;
        CU(cudaMalloc(&g->d_vnrec, words * sizeof(double)));
        g->vnrec_cap = words;
    }
    CU(launch_vnode_weights(L.k, dn, nv, g->d_vnrec, g->d_err, g->stream));
    g->launches += 1;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (g->profile) {
        e0 = pool_event(g);
        e1 = pool_event(g);
        CU(cudaEventRecord(e0, g->stream));
    }
    CU(launch_vnode_sweep(L, dim, vdim, g->d_vnrec, g->buf[g->cur], g->buf[1 - g->cur], g->stream));
    g->launches += 1;
    if (g->profile) {
        CU(cudaEventRecord(e1, g->stream));
        g->ev_pairs.push_back({e0, e1});
        g->ev_bytes.push_back(2.0 * (double)bytes_per_cell(L) * (double)L.cells);
        g->ev_dim.push_back(dim);
    }
    g->cur = 1 - g->cur;
    return SLDG_OK;
}

}  // namespace

sldg_status sldg::set_error(sldg_status st, const std::string& msg) { return fail(st, msg); }

extern "C" {

const char* sldg_last_error(void) { return g_last_error.c_str(); }

sldg_status sldg_nccl_unique_id(void* out128)
{
    if (!out128) return fail(SLDG_EINVAL, "null output");
    ncclUniqueId id;
    NC(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(out128, &id, 128);
    return SLDG_OK;
}

sldg_status sldg_halo_widths(int64_t imin, int64_t imax, int64_t* left, int64_t* right)
{
    if (!left || !right || imin > imax) return fail(SLDG_EINVAL, "bad arguments");
    *left = std::max<int64_t>(0, imax + 1);
    *right = std::max<int64_t>(0, -imin);
    return SLDG_OK;
}

sldg_status sldg_halo_plan(int64_t n, int world, int rank, int64_t pad, int64_t left, int64_t right,
                           int64_t* out, int64_t max_entries, int64_t* n_entries)
{
    if (n < 1 || world < 1 || world > n || rank < 0 || rank >= world || left < 0 || right < 0 || !n_entries)
        return fail(SLDG_EINVAL, "bad arguments");
    std::vector<Xfer> xs = halo_plan(n, world, rank, pad, left, right);
    *n_entries = (int64_t)xs.size();
    if (!out) return SLDG_OK;
    if ((int64_t)xs.size() > max_entries) return fail(SLDG_EINVAL, "output too small");
    for (size_t i = 0; i < xs.size(); ++i) {
        out[4 * i + 0] = xs[i].kind;
        out[4 * i + 1] = xs[i].peer;
        out[4 * i + 2] = xs[i].slot;
        out[4 * i + 3] = xs[i].src;
    }
    return SLDG_OK;
}

sldg_status sldg_layer_owner(int64_t n, int world, int64_t layer, int* owner, int64_t* local)
{
    if (n < 1 || world < 1 || world > n || layer < 0 || layer >= n || !owner)
        return fail(SLDG_EINVAL, "bad arguments");
    *owner = owner_of(n, world, layer, local);
    return SLDG_OK;
}

sldg_status sldg_transpose_plan(int64_t n_outer, int64_t n_slab, int world, int rank, int64_t* out)
{
    if (n_outer < 1 || n_slab < 1 || world < 1 || world > n_outer || rank < 0 || rank >= world || !out)
        return fail(SLDG_EINVAL, "bad arguments");
    const std::vector<TrPart> ps = transpose_plan(n_outer, n_slab, world, rank);
    for (int p = 0; p < world; ++p) {
        const TrPart& t = ps[p];
        const int64_t v[8] = {t.send_layer_first, t.send_layer_count, t.send_slab_first, t.send_slab_count,
                              t.recv_layer_first, t.recv_layer_count, t.recv_slab_first, t.recv_slab_count};
        for (int i = 0; i < 8; ++i) out[8 * p + i] = v[i];
    }
    return SLDG_OK;
}

sldg_status sldg_advect_vnodes(sldg_grid g, int dim, int vdim, const double* nodal_nu)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    // a captured graph would bake in one slot of the pinned staging ring (later host-field calls
    // overwrite it) and a captured event that upload_host_field later synchronises on
    if (g->capturing) return fail(SLDG_EINVAL, "host nodal field during graph capture: use sldg_advect_vnodes_device");
    return advect_vnodes_impl(g, dim, vdim, nodal_nu, false);
}

sldg_status sldg_advect_vnodes_device(sldg_grid g, int dim, int vdim, const double* d_nodal_nu)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    return advect_vnodes_impl(g, dim, vdim, d_nodal_nu, true);
}

sldg_status sldg_peer_halo_check(const sldg_grid_desc* grid, int k, sldg_precision prec, int world, int pad,
                                 int64_t gran)
{
    if (!grid || grid->ndim < 1 || grid->ndim > SLDG_MAX_DIM || k < 1 || k > SLDG_MAX_K || world < 1 || pad < 0 ||
        gran < 1 || (prec != SLDG_MIXED && prec != SLDG_FP64))
        return fail(SLDG_EINVAL, "bad arguments");
    Layout L{};
    L.D = grid->ndim;
    L.k = k;
    int64_t K = 1, cells_per_layer = 1;
    for (int d = 0; d < L.D; ++d) {
        if (grid->cells[d] < 1) return fail(SLDG_EINVAL, "cells must be >= 1");
        K *= k;
        L.n[d] = grid->cells[d];
        if (d < L.D - 1) cells_per_layer *= grid->cells[d];
    }
    if (L.D >= 2 && grid->cells[L.D - 1] < world) return fail(SLDG_EINVAL, "sharded extent smaller than world");
    L.K = (int)K;
    L.nd = (prec == SLDG_MIXED && K > 1) ? 1 : (int)K;
    L.L = cells_per_layer;
    L.pad = pad;
    std::string why = peer_halo_check(L, world, (size_t)gran);
    return why.empty() ? SLDG_OK : fail(SLDG_ENOTSUP, why);
}

sldg_status sldg_transpose_count(sldg_grid g, int64_t* n)
{
    if (!g || !n) return fail(SLDG_EINVAL, "null argument");
    *n = g->transposes;
    return SLDG_OK;
}

static sldg_status create_impl(const sldg_grid_desc* grid, int k, const sldg_domain* dom, int prec, int nd_req,
                               const sldg_dist* dist, sldg_grid* out);

sldg_status sldg_create(const sldg_grid_desc* grid, int k, const sldg_domain* dom, sldg_precision prec,
                        const sldg_dist* dist, sldg_grid* out)
{
    if (prec != SLDG_MIXED && prec != SLDG_FP64) return fail(SLDG_EINVAL, "bad precision");
    return create_impl(grid, k, dom, prec, -1, dist, out);
}

sldg_status sldg_create_ex(const sldg_grid_desc* grid, int k, const sldg_domain* dom, int n_double,
                           const sldg_dist* dist, sldg_grid* out)
{
    if (!grid || grid->ndim < 1 || grid->ndim > SLDG_MAX_DIM || k < 1 || k > SLDG_MAX_K)
        return fail(SLDG_EINVAL, "bad grid or k");
    int64_t K = 1;
    for (int d = 0; d < grid->ndim; ++d) K *= k;
    if (n_double < 0 || n_double > K) return fail(SLDG_EINVAL, "n_double must be in 0..k^D");
    if (n_double == 1) return create_impl(grid, k, dom, SLDG_MIXED, 1, dist, out);
    if (n_double == K) return create_impl(grid, k, dom, SLDG_FP64, (int)K, dist, out);
    if (grid->ndim != 1)
        return fail(SLDG_ENOTSUP, "n_double other than 1 or k^D is supported for 1D grids (the paper's tables)");
    return create_impl(grid, k, dom, SLDG_GENERAL, n_double, dist, out);
}

static sldg_status create_impl(const sldg_grid_desc* grid, int k, const sldg_domain* dom, int prec, int nd_req,
                               const sldg_dist* dist, sldg_grid* out)
{
    if (!grid || !dom || !out) return fail(SLDG_EINVAL, "null argument");
    *out = nullptr;
    if (grid->ndim < 1 || grid->ndim > SLDG_MAX_DIM) return fail(SLDG_EINVAL, "ndim must be in 1..6");
    if (k < 1 || k > SLDG_MAX_K) return fail(SLDG_EINVAL, "k must be in 1..8");
    const int D = grid->ndim;
    int64_t K = 1;
    for (int d = 0; d < D; ++d) {
        if (grid->cells[d] < 1) return fail(SLDG_EINVAL, "cells must be >= 1");
        if (!(dom->hi[d] > dom->lo[d]) || !isfinite(dom->lo[d]) || !isfinite(dom->hi[d]))
            return fail(SLDG_EINVAL, "domain must have lo < hi (finite)");
        K *= k;
    }
    if (K > (1 << 20)) return fail(SLDG_EINVAL, "k^D too large");
    // k^D == 1: the only coefficient is the mass, stored fp64 either way -- the mixed layout is
    // the fp64 layout (one fp64 plane, no fp32 planes), and the kernels treat it as such
    if (K == 1 && prec == SLDG_MIXED) prec = SLDG_FP64;
    int rank = 0, world = 1;
    if (dist) {
        rank = dist->rank;
        world = dist->world;
        if (world < 1 || rank < 0 || rank >= world) return fail(SLDG_EINVAL, "bad rank/world");
        if (world > 1 && D < 2) return fail(SLDG_EINVAL, "a 1D grid cannot be sharded");
        if (world > 1 && grid->cells[D - 1] < world)
            return fail(SLDG_EINVAL, "sharded extent smaller than world");
        if (world > 1 && !dist->nccl_unique_id && !dist->nccl_comm)
            return fail(SLDG_EINVAL, "distributed grid needs an ncclUniqueId or ncclComm");
    }
    sldg_grid g = new (std::nothrow) sldg_grid_s();
    if (!g) return fail(SLDG_ENOMEM, "host allocation failed");
    Layout& L = g->lay;
    L.D = D;
    L.k = k;
    L.K = (int)K;
    L.prec = prec;
    L.nd = (prec == SLDG_MIXED) ? 1 : (prec == SLDG_FP64) ? (int)K : nd_req;
    int64_t S = 1;
    for (int d = 0; d < kMaxDim; ++d) {
        L.n[d] = d < D ? grid->cells[d] : 1;
        L.S[d] = S;
        if (d < D) {
            g->lo[d] = dom->lo[d];
            g->hi[d] = dom->hi[d];
            g->h[d] = (dom->hi[d] - dom->lo[d]) / (double)grid->cells[d];
            S *= grid->cells[d];
        } else {
            g->lo[d] = 0.0;
            g->hi[d] = 1.0;
            g->h[d] = 1.0;
        }
    }
    if (D == 1) {
        L.L = L.n[0];
        L.layers = 1;
        L.first_layer = 0;
    } else {
        L.L = 1;
        for (int d = 0; d < D - 1; ++d) L.L *= L.n[d];
        split(L.n[D - 1], world, rank, &L.first_layer, &L.layers);
    }
    g->halo_mode = (world > 1) || (dist && (dist->flags & (SLDG_DIST_FORCE_HALO | SLDG_DIST_FORCE_TRANSPOSE)) && D >= 2);
    g->force_transpose = dist && (dist->flags & SLDG_DIST_FORCE_TRANSPOSE) && D >= 2;
    g->nccl_self = dist && (dist->flags & SLDG_DIST_NCCL_SELF) && world == 1;
    g->peer_halo = g->halo_mode && (dist->flags & SLDG_DIST_PEER_HALO);
    L.pad = g->halo_mode ? ((dist->max_halo > 0) ? dist->max_halo : 2) : 0;
    L.cells = L.layers * L.L;
    g->rank = rank;
    g->world = world;

    auto bail = [&](sldg_status st) {
        sldg_destroy(g);
        return st;
    };
    if (cudaGetDevice(&g->device) != cudaSuccess) return bail(fail(SLDG_ECUDA, "no CUDA device"));
    if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess)
        return bail(fail(SLDG_ECUDA, "stream create failed"));
    g->own_stream = true;
    if (cudaStreamCreateWithFlags(&g->comm_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->ev_halo, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(SLDG_ECUDA, "stream/event create failed"));
    if (const char* e = getenv("SLDG_COMM_SMS")) g->comm_sms = std::max(0, atoi(e));  // tuning override
    {  // the minimum weight table (constant shifts): such sweeps never allocate, also inside a capture
        sldg_status ws = ensure_weights(g, 1);
        if (ws != SLDG_OK) return bail(ws);
    }
    if (cudaMalloc(&g->d_partials, kMassBlocks * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&g->d_scalar, 64 * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&g->d_err, sizeof(int)) != cudaSuccess ||
        cudaMalloc(&g->d_range, 2 * sizeof(int64_t)) != cudaSuccess)
        return bail(fail(SLDG_ENOMEM, "device allocation failed"));
    if (cudaMemsetAsync(g->d_err, 0, sizeof(int), g->stream) != cudaSuccess)
        return bail(fail(SLDG_ECUDA, "memset failed"));
    if (g->nccl_self) {  // a one-rank communicator: self transfers go through NCCL (testing)
        ncclUniqueId id;
        ncclComm_t c;
        ncclResult_t r = ncclGetUniqueId(&id);
        if (r == ncclSuccess) r = ncclCommInitRank(&c, 1, id, 0);
        if (r != ncclSuccess) return bail(fail(SLDG_ENCCL, std::string("ncclCommInitRank(1): ") + ncclGetErrorString(r)));
        g->comm = c;
        g->own_comm = true;
    }
    if (world > 1) {
        if (dist->nccl_comm) {
            g->comm = dist->nccl_comm;
            g->own_comm = false;
        } else {
            ncclUniqueId id;
            memcpy(&id, dist->nccl_unique_id, sizeof(id));
            ncclComm_t c;
            ncclResult_t r = ncclCommInitRank(&c, world, id, rank);
            if (r != ncclSuccess) return bail(fail(SLDG_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r)));
            g->comm = c;
            g->own_comm = true;
        }
    }
    g->alloc_bytes = array_alloc_bytes(L);
    if (g->peer_halo) {  // pads mapped onto the neighbours' edge layers (sldg_peer.cu); collective
        std::string why = peer_alloc(g, (dist->flags & SLDG_DIST_PEER_VIA_FD) != 0);
        if (!why.empty()) return bail(fail(SLDG_ENOTSUP, "SLDG_DIST_PEER_HALO: " + why));
        for (int b = 0; b < 2; ++b) g->buf[b] = arrays_of(L, g->alloc[b]);
    }
    for (int b = 0; b < 2 && !g->peer_halo; ++b) {
        cudaError_t e = cudaMalloc(&g->alloc[b], g->alloc_bytes);
        if (e != cudaSuccess)
            return bail(fail(SLDG_ENOMEM, "device allocation of " + std::to_string(g->alloc_bytes) +
                                              " bytes failed: " + cudaGetErrorString(e)));
        if (cudaMemsetAsync(g->alloc[b], 0, g->alloc_bytes, g->stream) != cudaSuccess)
            return bail(fail(SLDG_ECUDA, "memset failed"));
        g->buf[b] = arrays_of(L, g->alloc[b]);
    }
    if (cudaStreamSynchronize(g->stream) != cudaSuccess) return bail(fail(SLDG_ECUDA, "sync failed"));
    *out = g;
    return SLDG_OK;
}

sldg_status sldg_destroy(sldg_grid g)
{
    if (!g) return SLDG_OK;
    if (g->stream) cudaStreamSynchronize(g->stream);
    if (g->comm_stream) cudaStreamSynchronize(g->comm_stream);
    if (g->own_comm && g->comm) ncclCommDestroy((ncclComm_t)g->comm);
    for (int b = 0; b < 2; ++b) {
        tmap_cache_forget(g->alloc[b], g->alloc_bytes);
        fused_cache_forget(g->alloc[b], g->alloc_bytes);
        if (!g->peer) cudaFree(g->alloc[b]);
    }
    peer_free(g);
    tmap_cache_forget(g->t_alloc, g->t_bytes);
    cudaFree(g->w2.shift);
    cudaFree(g->w2.smod);
    cudaFree(g->w2.copy);
    cudaFree(g->w2.ab);
    cudaFree(g->w2.rec);
    cudaFree(g->w.shift);
    cudaFree(g->w.smod);
    cudaFree(g->w.copy);
    cudaFree(g->w.ab);
    cudaFree(g->w.rec);
    cudaFree(g->d_field);
    for (int s = 0; s < sldg_grid_s::kFieldStages; ++s) {
        if (g->h_fstage[s]) cudaFreeHost(g->h_fstage[s]);
        if (g->fstage_ev[s]) cudaEventDestroy(g->fstage_ev[s]);
    }
    cudaFree(g->d_partials);
    cudaFree(g->d_scalar);
    cudaFree(g->d_err);
    cudaFree(g->d_range);
    cudaFree(g->t_alloc);
    cudaFree(g->d_tfield);
    cudaFree(g->d_vnrec);
    cudaFree(g->d_stage);
    if (g->h_stage) cudaFreeHost(g->h_stage);
    for (auto& p : g->ev_pairs) {
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    for (auto& p : g->tl_ev) {
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
    }
    for (auto e : g->ev_pool) cudaEventDestroy(e);
    if (g->ev_ready) cudaEventDestroy(g->ev_ready);
    if (g->ev_halo) cudaEventDestroy(g->ev_halo);
    if (g->comm_stream) cudaStreamDestroy(g->comm_stream);
    if (g->own_stream && g->stream) cudaStreamDestroy(g->stream);
    delete g;
    return SLDG_OK;
}

sldg_status sldg_set_coeffs(sldg_grid g, const double* src, int64_t first_cell, int64_t n_cells)
{
    if (!g || (!src && n_cells > 0)) return fail(SLDG_EINVAL, "null argument");
    const Layout& L = g->lay;
    if (first_cell < 0 || n_cells < 0 || first_cell + n_cells > L.cells)
        return fail(SLDG_EINVAL, "cell range outside the local shard");
    const int64_t n = n_cells * L.K;
    for (int64_t e = 0; e < n; ++e) {  // all-or-nothing validation
        double v = src[e];
        if (!isfinite(v)) return fail(SLDG_EINVAL, "non-finite coefficient at element " + std::to_string(e));
        if ((e % L.K) >= L.nd && fabs(v) > (double)FLT_MAX)
            return fail(SLDG_EINVAL, "value beyond FLT_MAX in an fp32 slot at element " + std::to_string(e));
    }
    sldg_status st = ensure_stage(g);
    if (st != SLDG_OK) return st;
    const int64_t chunk_cells = (int64_t)g->stage_elems / L.K;
    for (int64_t c0 = 0; c0 < n_cells; c0 += chunk_cells) {
        int64_t nc = std::min(chunk_cells, n_cells - c0);
        memcpy(g->h_stage, src + c0 * L.K, (size_t)nc * L.K * sizeof(double));
        CU(cudaMemcpyAsync(g->d_stage, g->h_stage, (size_t)nc * L.K * sizeof(double), cudaMemcpyHostToDevice, g->stream));
        CU(launch_set(L, g->buf[g->cur], g->d_stage, first_cell + c0, nc, g->stream));
        g->launches += 1;
        CU(cudaStreamSynchronize(g->stream));
    }
    return SLDG_OK;
}

sldg_status sldg_get_coeffs(sldg_grid g, double* dst, int64_t first_cell, int64_t n_cells)
{
    if (!g || (!dst && n_cells > 0)) return fail(SLDG_EINVAL, "null argument");
    const Layout& L = g->lay;
    if (first_cell < 0 || n_cells < 0 || first_cell + n_cells > L.cells)
        return fail(SLDG_EINVAL, "cell range outside the local shard");
    sldg_status st = ensure_stage(g);
    if (st != SLDG_OK) return st;
    const int64_t chunk_cells = (int64_t)g->stage_elems / L.K;
    for (int64_t c0 = 0; c0 < n_cells; c0 += chunk_cells) {
        int64_t nc = std::min(chunk_cells, n_cells - c0);
        CU(launch_get(L, g->buf[g->cur], g->d_stage, first_cell + c0, nc, g->stream));
        g->launches += 1;
        CU(cudaMemcpyAsync(g->h_stage, g->d_stage, (size_t)nc * L.K * sizeof(double), cudaMemcpyDeviceToHost, g->stream));
        CU(cudaStreamSynchronize(g->stream));
        memcpy(dst + c0 * L.K, g->h_stage, (size_t)nc * L.K * sizeof(double));
    }
    return check_device_error(g);
}

sldg_status sldg_advect(sldg_grid g, int dim, double shift, const double* field, uint32_t field_mask)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    if (field && g->capturing)
        return fail(SLDG_EINVAL, "a host shift field cannot be captured in a graph: use sldg_advect_device");
    return advect_impl(g, dim, shift, field, false, field_mask);
}

// ---- CUDA graphs of asynchronous call sequences (launch-bound small grids) ------------------
struct sldg_graph_s {
    sldg_grid g = nullptr;
    cudaGraphExec_t exec = nullptr;
    int cur_begin = 0, cur_end = 0;
    int64_t launches = 0;
};

sldg_status sldg_graph_begin(sldg_grid g)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    if (g->capturing) return fail(SLDG_EINVAL, "a capture is already open");
    CU(cudaStreamBeginCapture(g->stream, cudaStreamCaptureModeThreadLocal));
    g->capturing = true;
    g->cap_cur = g->cur;
    g->cap_launches = g->launches;
    g->cap_profile = g->profile;
    g->profile = false;  // per-sweep events are bookkept on the host: not inside a graph
    g->w_const = false;  // the captured sequence builds its own weights
    return SLDG_OK;
}

sldg_status sldg_graph_end(sldg_grid g, sldg_graph* out)
{
    if (!g || !out) return fail(SLDG_EINVAL, "null argument");
    if (!g->capturing) return fail(SLDG_EINVAL, "no capture is open");
    *out = nullptr;
    cudaGraph_t graph = nullptr;
    cudaError_t e = cudaStreamEndCapture(g->stream, &graph);
    g->capturing = false;
    g->profile = g->cap_profile;
    g->w_const = false;
    const int cur_end = g->cur;
    const int64_t nl = g->launches - g->cap_launches;
    g->cur = g->cap_cur;  // nothing ran: the captured sweeps run at sldg_graph_launch
    g->launches = g->cap_launches;
    if (e != cudaSuccess) return fail(SLDG_ECUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e));
    sldg_graph gr = new (std::nothrow) sldg_graph_s;
    if (!gr) {
        cudaGraphDestroy(graph);
        return fail(SLDG_ENOMEM, "host allocation");
    }
    e = cudaGraphInstantiate(&gr->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
        delete gr;
        return fail(SLDG_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
    }
    gr->g = g;
    gr->cur_begin = g->cap_cur;
    gr->cur_end = cur_end;
    gr->launches = nl;
    *out = gr;
    return SLDG_OK;
}

sldg_status sldg_graph_launch(sldg_graph gr)
{
    if (!gr) return fail(SLDG_EINVAL, "null graph");
    sldg_grid g = gr->g;
    if (g->cur != gr->cur_begin)
        return fail(SLDG_EINVAL, "the grid's current buffer differs from the one the graph was captured on "
                                 "(an odd number of sweeps: capture two steps)");
    CU(cudaGraphLaunch(gr->exec, g->stream));
    g->cur = gr->cur_end;
    g->launches += gr->launches;
    g->w_const = false;
    return SLDG_OK;
}

sldg_status sldg_graph_destroy(sldg_graph gr)
{
    if (!gr) return SLDG_OK;
    if (gr->g) cudaStreamSynchronize(gr->g->stream);
    if (gr->exec) cudaGraphExecDestroy(gr->exec);
    delete gr;
    return SLDG_OK;
}

sldg_status sldg_advect_device_bounded(sldg_grid g, int dim, double shift, const double* d_field,
                                       uint32_t field_mask, double nu_min, double nu_max)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    if (!d_field) return fail(SLDG_EINVAL, "null device field");
    return advect_impl(g, dim, shift, d_field, true, field_mask, true, nu_min, nu_max);
}

sldg_status sldg_advect_pair(sldg_grid g, double shift0, const double* field0, uint32_t mask0, double shift1,
                             const double* field1, uint32_t mask1)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    return advect_pair_impl(g, shift0, field0, mask0, shift1, field1, mask1, false);
}

sldg_status sldg_advect_pair_device(sldg_grid g, double shift0, const double* d_field0, uint32_t mask0, double shift1,
                                    const double* d_field1, uint32_t mask1)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    return advect_pair_impl(g, shift0, d_field0, mask0, shift1, d_field1, mask1, true);
}

sldg_status sldg_timeline(sldg_grid g, double* t_ms, int* kinds, int max_entries, int* n_out, int reset)
{
    if (!g || !n_out || (max_entries > 0 && (!t_ms || !kinds))) return fail(SLDG_EINVAL, "null argument");
    CU(cudaStreamSynchronize(g->stream));
    CU(cudaStreamSynchronize(g->comm_stream));
    const int n = (int)g->tl_ev.size();
    *n_out = n;
    if (n == 0) return SLDG_OK;
    cudaEvent_t origin = g->tl_ev[0].first;  // the first recorded interval starts at 0
    for (int i = 0; i < n && i < max_entries; ++i) {
        float a = 0.f, b = 0.f;
        CU(cudaEventElapsedTime(&a, origin, g->tl_ev[i].first));
        CU(cudaEventElapsedTime(&b, origin, g->tl_ev[i].second));
        t_ms[2 * i] = a;
        t_ms[2 * i + 1] = b;
        kinds[i] = g->tl_kind[i];
    }
    if (reset) {
        for (auto& pr : g->tl_ev) {
            g->ev_pool.push_back(pr.first);
            g->ev_pool.push_back(pr.second);
        }
        g->tl_ev.clear();
        g->tl_kind.clear();
    }
    return SLDG_OK;
}

sldg_status sldg_advect_device(sldg_grid g, int dim, double shift, const double* d_field, uint32_t field_mask)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    return advect_impl(g, dim, shift, d_field, true, field_mask);
}

sldg_status sldg_mass(sldg_grid g, double* mass_out)
{
    if (!g || !mass_out) return fail(SLDG_EINVAL, "null argument");
    const Layout& L = g->lay;
    CU(launch_mass_partials(L, g->buf[g->cur], g->d_partials, g->d_scalar, g->stream));
    g->launches += 2;
    double vol = 1.0;
    for (int d = 0; d < L.D; ++d) vol *= g->h[d];
    std::vector<double> parts((size_t)g->world, 0.0);
    if (g->world > 1) {
        NC(ncclAllGather(g->d_scalar, g->d_scalar + 1, 1, ncclFloat64, (ncclComm_t)g->comm, g->stream));
        CU(cudaMemcpyAsync(parts.data(), g->d_scalar + 1, g->world * sizeof(double), cudaMemcpyDeviceToHost, g->stream));
    } else {
        CU(cudaMemcpyAsync(parts.data(), g->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, g->stream));
    }
    CU(cudaStreamSynchronize(g->stream));
    double s = 0.0;
    for (int r = 0; r < g->world; ++r) s += parts[r];  // rank-ordered
    *mass_out = vol * s;
    return check_device_error(g);
}

sldg_status sldg_shard_info(sldg_grid g, int64_t* first_layer, int64_t* n_layers)
{
    if (!g || !first_layer || !n_layers) return fail(SLDG_EINVAL, "null argument");
    *first_layer = g->lay.first_layer;
    *n_layers = g->lay.layers;
    return SLDG_OK;
}

sldg_status sldg_sync(sldg_grid g)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    CU(cudaStreamSynchronize(g->stream));
    CU(cudaStreamSynchronize(g->comm_stream));
    return check_device_error(g);
}

sldg_status sldg_set_stream(sldg_grid g, void* cuda_stream)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    CU(cudaStreamSynchronize(g->stream));
    if (g->own_stream) cudaStreamDestroy(g->stream);
    if (cuda_stream) {
        g->stream = (cudaStream_t)cuda_stream;
        g->own_stream = false;
    } else {
        CU(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
        g->own_stream = true;
    }
    return SLDG_OK;
}

sldg_status sldg_get_stream(sldg_grid g, void** cuda_stream)
{
    if (!g || !cuda_stream) return fail(SLDG_EINVAL, "null argument");
    *cuda_stream = (void*)g->stream;
    return SLDG_OK;
}

size_t sldg_memory_bytes(sldg_grid g)
{
    if (!g) return 0;
    return (size_t)g->lay.cells * bytes_per_cell(g->lay);
}

sldg_status sldg_fill_random(sldg_grid g, uint64_t seed)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    CU(launch_fill_random(g->lay, g->buf[g->cur], seed, g->stream));
    g->launches += 1;
    return SLDG_OK;
}

sldg_status sldg_fill_separable(sldg_grid g, int n_terms, const double* tables)
{
    if (!g || !tables || n_terms < 1) return fail(SLDG_EINVAL, "bad arguments");
    const Layout& L = g->lay;
    int64_t per_term = 0;
    for (int d = 0; d < L.D; ++d) per_term += L.n[d] * L.k;
    const size_t bytes = (size_t)per_term * n_terms * sizeof(double);
    for (size_t e = 0; e < (size_t)per_term * n_terms; ++e)
        if (!isfinite(tables[e])) return fail(SLDG_EINVAL, "non-finite table entry");
    double* d_tab = nullptr;
    CU(cudaMallocAsync((void**)&d_tab, bytes, g->stream));
    CU(cudaMemcpyAsync(d_tab, tables, bytes, cudaMemcpyHostToDevice, g->stream));
    CU(launch_fill_separable(L, g->buf[g->cur], n_terms, d_tab, g->stream));
    g->launches += 1;
    CU(cudaFreeAsync(d_tab, g->stream));
    CU(cudaStreamSynchronize(g->stream));
    return SLDG_OK;
}

sldg_status sldg_profile(sldg_grid g, int enable)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    g->profile = enable != 0;
    return SLDG_OK;
}

sldg_status sldg_kernel_time(sldg_grid g, int dim, double* ms, int64_t* launches, double* bytes, int reset)
{
    if (!g) return fail(SLDG_EINVAL, "null grid");
    if (dim < -2 || dim >= g->lay.D) return fail(SLDG_EINVAL, "dim out of range");
    CU(cudaStreamSynchronize(g->stream));
    for (size_t i = 0; i < g->ev_pairs.size(); ++i) {
        float t = 0.f;
        CU(cudaEventElapsedTime(&t, g->ev_pairs[i].first, g->ev_pairs[i].second));
        const int d = g->ev_dim[i];
        g->prof_ms[d] += t;
        g->prof_bytes[d] += g->ev_bytes[i];
        g->prof_launches[d] += 1;
        g->ev_pool.push_back(g->ev_pairs[i].first);
        g->ev_pool.push_back(g->ev_pairs[i].second);
    }
    g->ev_pairs.clear();
    g->ev_bytes.clear();
    g->ev_dim.clear();
    double m = 0.0, b = 0.0;
    int64_t n = 0;
    for (int d = 0; d <= kMaxDim; ++d) {
        if (d >= g->lay.D && d != kMaxDim) continue;
        if (dim >= 0 && d != dim) continue;
        if (dim == -2 && d != kMaxDim) continue;  // -2: fused sweep pairs only
        m += g->prof_ms[d];
        b += g->prof_bytes[d];
        n += g->prof_launches[d];
    }
    if (ms) *ms = m;
    if (launches) *launches = n;
    if (bytes) *bytes = b;
    if (reset) {
        for (int d = 0; d <= kMaxDim; ++d) {
            g->prof_ms[d] = 0.0;
            g->prof_bytes[d] = 0.0;
            g->prof_launches[d] = 0;
        }
    }
    return SLDG_OK;
}

int64_t sldg_launch_count(sldg_grid g) { return g ? g->launches : 0; }

const char* sldg_sweep_kernel(sldg_grid g, int dim)
{
    if (!g || dim < 0 || dim >= g->lay.D) return "";
    Sweep sw{};
    sw.dim = dim;
    sw.nd = g->lay.n[dim];
    return sweep_kernel_name(g->lay, sw);
}

}  // extern "C"
