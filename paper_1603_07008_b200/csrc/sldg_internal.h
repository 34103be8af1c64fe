// sldg_internal.h -- internal types of the B200 SLDG library (not part of the ABI).
//
// Device layout of one coefficient array:
//   The outermost dim D-1 (D >= 2) is the LAYER dim (sharded across ranks); a layer holds
//   L = prod_{d<D-1} n_d cells.  For D == 1 there is one virtual layer with L = n_0.
//   mixed : mass[(pad + layer) * L + inner]                        (fp64, slot q = 0)
//           pl  [((pad + layer) * (K-1) + (q-1)) * L + inner]       (fp32, slots q >= 1)
//   fp64  : s64 [((pad + layer) * K + q) * L + inner]                (fp64, all slots)
//   inner = sum_{d<D-1} i_d S_d.  One layer of all slots is contiguous per array, so a halo
//   layer is two contiguous chunks (mixed) or one (fp64).  `pad` layers on each side hold
//   halos when the layer dim is sharded.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/sldg.h"

namespace sldg {

constexpr int kMaxDim = SLDG_MAX_DIM;
constexpr int kMaxK = SLDG_MAX_K;

// One coefficient array (a ping-pong buffer).  General addressing (any nd):
//   slot q <  nd: mass[((pad + layer) * nd + q) * L + inner]            (fp64)
//   slot q >= nd: pl  [((pad + layer) * (K - nd) + (q - nd)) * L + inner] (fp32)
// which is the mixed layout for nd = 1 and the fp64 layout (s64 == mass) for nd = K.
struct Arrays {
    double* mass = nullptr;  // fp64 slots (mixed: slot 0; fp64 variant: all, == s64)
    float* pl = nullptr;     // fp32 slots
    double* s64 = nullptr;   // fp64 variant: all slots
};

constexpr int SLDG_GENERAL = 2;  // internal precision tag: 1D grid with an arbitrary nd

__host__ __device__ __forceinline__ double* dslot(const Arrays& a, int64_t layerp, int nd, int q, int64_t L,
                                                  int64_t inner)
{
    return a.mass + (layerp * nd + q) * L + inner;
}
__host__ __device__ __forceinline__ float* fslot(const Arrays& a, int64_t layerp, int K, int nd, int q, int64_t L,
                                                 int64_t inner)
{
    return a.pl + (layerp * (K - nd) + (q - nd)) * L + inner;
}

// Per-sweep weight table: one entry per field entry (or a single one for a constant shift).
struct Weights {
    int64_t* shift = nullptr;  // i* (raw) per entry
    int64_t* smod = nullptr;   // i* mod n_d in [0, n_d) per entry
    int* copy = nullptr;       // 1 if alpha == 0 (exact rotation)
    double* ab = nullptr;      // [entry][2][k][k]: A then B, row-major
    double* rec = nullptr;     // [entry][2k^2 + 2]: A, B, i* mod n (int64 bits), copy (int64 bits)
    int64_t cap = 0;
};

// Layout + sweep description passed by value to the kernels.
struct Layout {
    int D;
    int k;
    int K;            // k^D
    int prec;         // SLDG_MIXED (nd = 1) / SLDG_FP64 (nd = K) / SLDG_GENERAL (1D, any nd)
    int nd;           // number of leading slots q < nd stored in fp64 (the paper's "# double")
    int64_t n[kMaxDim];   // GLOBAL extents
    int64_t S[kMaxDim];   // inner strides S_d (d < D-1); S_{D-1} unused
    int64_t L;            // cells per layer
    int64_t layers;       // local layers
    int64_t first_layer;  // global index of local layer 0
    int64_t pad;          // halo layers per side
    int64_t cells;        // local cells = layers * L
};

struct Sweep {
    int dim;
    int64_t nd;                // extent along dim (global)
    uint32_t fmask;
    int64_t fstride[kMaxDim];  // field index stride per dim (0 if not masked)
    int wrap;                  // 1: periodic modulo indexing; 0: read halos (layer dim sharded)
    const int64_t* shift;  // raw i*
    const int64_t* smod;   // i* mod nd
    const int* copy;
    const double* ab;
    const double* rec;     // packed line records (see Weights::rec)
    int sm_reserve = 0;    // persistent TMA kernels: leave this many SMs free (a concurrent halo
                           // exchange's NCCL kernel cannot co-reside with a ~200 KB-smem CTA)
};

struct Grid {
    Layout lay;
    double h[kMaxDim];
    double lo[kMaxDim], hi[kMaxDim];
    Arrays buf[2];
    int cur = 0;
    void* alloc[2] = {nullptr, nullptr};
    size_t alloc_bytes = 0;
    Weights w;
    Weights w2;  // the second sweep's table of a fused pair (sldg_advect_pair)
    // the weight table holds the constant shift w_shift along an extent of w_n (no field):
    // a repeated constant-shift sweep reuses it instead of relaunching the build kernel
    bool w_const = false;
    double w_shift = 0.0;
    int64_t w_n = 0;
    double* d_field = nullptr;
    int64_t field_cap = 0;
    // pinned staging ring for host shift fields: the caller's buffer is copied on the host before
    // sldg_advect returns (never read later by a DMA), then uploaded asynchronously
    static constexpr int kFieldStages = 4;
    double* h_fstage[kFieldStages] = {};
    cudaEvent_t fstage_ev[kFieldStages] = {};
    bool fstage_busy[kFieldStages] = {};
    int64_t fstage_cap = 0;
    int fstage_next = 0;
    double* d_partials = nullptr;  // mass partial sums
    double* d_scalar = nullptr;    // misc device scalars
    int* d_err = nullptr;          // sticky device error flag
    double* d_stage = nullptr;     // set/get staging (device)
    double* h_stage = nullptr;     // set/get staging (pinned host)
    size_t stage_elems = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int device = 0;
    // distribution
    int rank = 0, world = 1;
    void* comm = nullptr;  // ncclComm_t
    bool own_comm = false;
    // instrumentation
    bool profile = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pairs;
    std::vector<double> ev_bytes;
    std::vector<int> ev_dim;
    std::vector<cudaEvent_t> ev_pool;
    double prof_ms[kMaxDim + 1] = {}, prof_bytes[kMaxDim + 1] = {};  // [kMaxDim]: fused pairs
    int64_t prof_launches[kMaxDim + 1] = {};
    int64_t launches = 0;
};

// records msg as sldg_last_error() and returns st (sldg_abi.cu)
sldg_status set_error(sldg_status st, const std::string& msg);

// k-point Gauss-Legendre nodes (ascending) and weights on [-1, 1], computed once per k on the
// host (Newton on P_k) and passed to the weight kernels by value (kernel-parameter bank).
struct GaussTab {
    double x[kMaxK];
    double w[kMaxK];
};
const GaussTab& gauss_table(int k);

// ---- kernel launchers (sldg_kernels.cu) -------------------------------------------------
// [ilo, ihi]: integer-shift bound of the field (sldg_advect_device_bounded); an entry outside
// it (or non-finite) leaves its lines unchanged and raises the sticky device error
cudaError_t launch_weights(const Layout& lay, int64_t nd, const double* d_field, double shift,
                           int64_t n_entries, Weights& w, int* d_err, cudaStream_t s,
                           int64_t ilo = INT64_MIN, int64_t ihi = INT64_MAX);
cudaError_t launch_sweep(const Layout& lay, const Sweep& sw, const Arrays& src, const Arrays& dst,
                         int64_t layer_begin, int64_t layer_end, cudaStream_t s, int* n_launched);
cudaError_t launch_mass_partials(const Layout& lay, const Arrays& a, double* d_partials,
                                 double* d_out, cudaStream_t s);
cudaError_t launch_set(const Layout& lay, const Arrays& a, const double* d_src, int64_t first_cell,
                       int64_t n_cells, cudaStream_t s);
cudaError_t launch_get(const Layout& lay, const Arrays& a, double* d_dst, int64_t first_cell,
                       int64_t n_cells, cudaStream_t s);
cudaError_t launch_fill_random(const Layout& lay, const Arrays& a, uint64_t seed, cudaStream_t s);
cudaError_t launch_fill_separable(const Layout& lay, const Arrays& a, int n_terms,
                                  const double* d_tables, cudaStream_t s);
cudaError_t launch_field_range(const double* d_field, int64_t n, double shift, int64_t* d_out2,
                               cudaStream_t s);
// Gauss-node velocity sweep (sldg_vnodes.cu, NEXT-3)
constexpr int kVnMaxOfs = 6;  // source offsets per v-cell (nodes' integer parts may differ)
int64_t vnode_rec_words(int k);
cudaError_t launch_vnode_weights(int k, const double* d_nodal, int64_t nv, double* d_rec, int* d_err, cudaStream_t s);
cudaError_t launch_vnode_sweep(const Layout& lay, int d, int e, const double* d_rec, const Arrays& src,
                               const Arrays& dst, cudaStream_t s);
// transpose path (sldg_abi.cu transpose_sweep): one (layer range, inner range) message block
cudaError_t launch_tr_block(const Layout& lay, const Arrays& a, int64_t nl, int64_t first, int64_t len, double* bm,
                            float* bf, bool pack, cudaStream_t s);
cudaError_t launch_field_slab(const double* in, int64_t n_out, uint32_t mask, const Layout& nT, const Layout& nF,
                              int sd, int64_t off, double* out, cudaStream_t s);

constexpr int kMassBlocks = 592;  // 4 x 148 SMs; fixed => deterministic reduction order

// ---- TMA-staged sweeps (sldg_sweep_tma.cu) ------------------------------------------------
constexpr int kTmaConsumerWarps = 8;
constexpr int kTmaThreads = (kTmaConsumerWarps + 1) * 32;  // + 1 producer warp
struct TmaPlan {
    int W = 0;      // strided: i_0 columns per tile
    int T = 0;      // strided: targets along d per tile
    int Tsub = 0;   // strided: nominal targets per stage (rows = Rmax = Tsub + 4)
    int Rmax = 0;   // strided: source rows per slot per stage
    int R = 0;      // d0: whole lines per stage
    int GC = 0;     // d0: coupled groups per stage
    int rec1 = 0;   // d0: the tile's R lines share one field entry (one record per tile)
    int pspan = 0;  // strided: the producer warp computes the tile shift spans (sldg_sweep_tma.cu)
    int stage_bytes = 0;
    int stages = 0;
    int ctas = 1;   // CTAs per SM (shared-memory budget and register bound of the instance)
};
bool tma_plan(const Layout& lay, const Sweep& sw, TmaPlan* pl);
// cudaFuncAttributeMaxDynamicSharedMemorySize = the opt-in maximum for `func` on the CURRENT device
// (set once per (device, function); the attribute is per device context)
void ensure_max_smem(const void* func);
// fused dim-0 + dim-1 sweeps (sldg_fused.cu, NEXT-4 multi-sweep fusion)
struct FusedPlan {
    int NS = 0;          // slabs ("lanes") per tile = 256 / n0
    int Tsub = 0;        // target rows per stage (the line's first stage loads one more row)
    int rows_alloc = 0;  // Tsub + 1
    int lane_bytes = 0;  // one lane's region of a stage
    int stage_bytes = 0;
    int stages = 0;
    int64_t nslab = 0;   // local slabs (cells of dims >= 2)
    int64_t M_mid = 0;   // prod_{2 <= d < D-1} n_d
};
bool fused_plan(const Layout& lay, const Sweep& s0, const Sweep& s1, FusedPlan* fp);
cudaError_t launch_fused01(const Layout& lay, const Sweep& s0, const Sweep& s1, const Arrays& src, const Arrays& dst,
                           const FusedPlan& fp, cudaStream_t s);
void fused_cache_forget(const void* base, size_t bytes);
const char* sweep_kernel_name(const Layout& lay, const Sweep& sw);
// 1D sweeps, any precision layout (sldg_line.cu)
cudaError_t launch_line(const Layout& lay, const Sweep& sw, const Arrays& src, const Arrays& dst, cudaStream_t s,
                        const char** name);
const char* line_kernel_name(const Layout& lay);
cudaError_t launch_sweep_tma(const Layout& lay, const Sweep& sw, const Arrays& src, const Arrays& dst,
                             int64_t layer_begin, int64_t layer_end, const TmaPlan& pl, cudaStream_t s);
// drop cached tensor maps of buffers inside [base, base + bytes) (before that memory is freed)
void tmap_cache_forget(const void* base, size_t bytes);

}  // namespace sldg

// The opaque ABI handle: the grid plus the distributed-sweep state (sldg_abi.cu).
struct sldg_grid_s : public sldg::Grid {
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_halo = nullptr;
    int64_t* d_range = nullptr;
    bool halo_mode = false;  // sweeps along the layer dim read halo layers (sharded, or forced)
    bool force_transpose = false;  // every sweep along the layer dim takes the transpose path
    bool nccl_self = false;        // world == 1 with a one-rank NCCL communicator: self transfers via NCCL
    void* t_alloc = nullptr;       // transpose path: two slab arrays + receive staging
    size_t t_bytes = 0;
    double* d_tfield = nullptr;    // transpose path: the field restricted to this rank's slab
    int64_t tfield_cap = 0;
    int64_t transposes = 0;        // sweeps that took the transpose path
    int comm_sms = 8;              // SMs the interior sweep leaves to the concurrent halo exchange
    // profile mode: device intervals of halo exchanges (comm stream) and of every profiled sweep
    // launch, for the overlap timeline (sldg_timeline)
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tl_ev;
    std::vector<int> tl_kind;      // sweep dim, or -1 for a halo exchange
    // SLDG_DIST_PEER_HALO: the pad layers are mappings of the neighbours' edge layers (sldg_peer.cu)
    bool peer_halo = false;
    struct sldg_peer_s* peer = nullptr;
    double* d_vnrec = nullptr;     // Gauss-node sweep: per-v-cell operator records
    int64_t vnrec_cap = 0;
    // graph capture (sldg_graph_begin/end)
    bool capturing = false, cap_profile = false;
    int cap_cur = 0;
    int64_t cap_launches = 0;
};

// peer-mapped halo layers (sldg_peer.cu)
namespace sldg {
// "" if the layout can back its pads with the neighbours' edge chunks at allocation granularity
// `gran` on every rank of `world`, else the reason
std::string peer_halo_check(const Layout& L, int world, size_t gran);
size_t peer_granularity(int device);  // 0 if the virtual-memory API is unavailable
std::string peer_alloc(sldg_grid g, bool via_fd);  // sets g->alloc[0..1] and g->peer; "" or the reason
void peer_free(sldg_grid g);
cudaError_t peer_fence(sldg_grid g);  // world > 1: NCCL fence with both ring neighbours
}  // namespace sldg
