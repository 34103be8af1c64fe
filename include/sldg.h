/*
 * sldg.h -- C ABI of the B200-native mixed-precision semi-Lagrangian discontinuous Galerkin
 * (SLDG) translate-and-project step of Einkemmer, "A mixed precision semi-Lagrangian
 * algorithm and its performance on accelerators" (arXiv:1603.07008).
 *
 * Citation keys: P:NNN = /root/reference/PAPER.md line NNN (section in parentheses),
 * S:NNN = SPEC.md line NNN (interface shapes only), SURVEY = /root/repo/SURVEY.md,
 * R<n> = reading n in /root/repo/DESIGN.md.
 *
 * What the library computes (SS II-A):
 *   Each cell of a periodic tensor-product grid (D = 1..6 dims, n_d cells along dim d,
 *   width h_d = (hi_d - lo_d)/n_d) holds a modal Legendre expansion with k coefficients per
 *   dim (k^D per cell, "u(x) ~ sum_j c_j P_j(2x/h)").  One advection sweep along
 *   dim d translates the function exactly by nu*h_d (nu = CFL number in CELLS, per line)
 *   and L2-projects it back:
 *       c'_{i,j} = sum_l A_jl(alpha) c_{(i-i*-1) mod n, l} + sum_l B_jl(alpha) c_{(i-i*) mod n, l}
 *   with i* = floor(nu), alpha = nu - i* (readings R1-R2), A and B the k x k
 *   shift matrices, applied to the coefficient index along d while the
 *   other indices are spectators (dimension splitting).  alpha = 0 is an exact
 *   rotation (R4).
 *
 * Storage (R5): SLDG_MIXED keeps the all-zero multi-index coefficient (c_0, the
 * cell mass) in fp64 and every other coefficient in fp32, rounded to nearest-even on every
 * store; arithmetic is fp64 (R6).  SLDG_FP64 keeps all coefficients in fp64 (the baseline the
 * paper compares against, Tables III-VI).
 *
 * Host coefficient layout used by set/get (fp64, all-or-nothing):
 *   buf[c * K + q], K = k^D, c = local linear cell index = sum_d i_d * S_d with S_0 = 1,
 *   S_d = prod_{e<d} n_e (dim 0 fastest; for a sharded grid i_{D-1} is the LOCAL layer index,
 *   see sldg_shard_info), q = sum_d m_d k^d (m_0 fastest).
 *
 * Errors: every function returns sldg_status; no C++ exception crosses the ABI.
 * sldg_last_error() returns a thread-local message for the last failure on this thread.
 * EINVAL failures leave the grid unchanged.  Ownership: the handle owns all device memory
 * it allocates (and the NCCL communicator if it created one); the caller owns all host
 * buffers, which are never retained after a call returns (a host shift field is copied into
 * the handle's pinned staging ring before sldg_advect returns, pinned caller memory included).
 * Threading: a handle is not thread-safe; distinct handles are independent.  When the grid
 * is distributed (world > 1) every call except sldg_last_error / sldg_memory_bytes /
 * sldg_shard_info is collective and must be made in the same order on all ranks.
 * Streams: all device work is ordered on the handle's stream (its own non-blocking stream,
 * or the one given to sldg_set_stream).  advect and fill_* are asynchronous; set_coeffs,
 * get_coeffs, mass, sync and kernel_time block the host.
 */
#ifndef SLDG_H
#define SLDG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SLDG_MAX_DIM 6
#define SLDG_MAX_K 8

typedef struct sldg_grid_s* sldg_grid; /* opaque handle */

typedef enum {
    SLDG_OK = 0,
    SLDG_EINVAL = 1,  /* invalid argument; no state changed                            */
    SLDG_ENOMEM = 2,  /* device or pinned-host allocation failed               */
    SLDG_ECUDA = 3,   /* CUDA runtime error; message in sldg_last_error()              */
    SLDG_ENCCL = 4,   /* NCCL error; message in sldg_last_error()                      */
    SLDG_ENOTSUP = 5  /* valid request this build does not support (e.g. halo > pad)   */
} sldg_status;

typedef enum {
    SLDG_MIXED = 0, /* c_{0..0} fp64, all other coefficients fp32          */
    SLDG_FP64 = 1   /* all coefficients fp64 (the paper's "double precision" baseline)  */
} sldg_precision;

typedef struct {
    int ndim;                      /* D in 1..SLDG_MAX_DIM                                 */
    int64_t cells[SLDG_MAX_DIM];   /* n_d >= 1 (GLOBAL extents); cells[0] is contiguous    */
} sldg_grid_desc;

typedef struct {
    double lo[SLDG_MAX_DIM], hi[SLDG_MAX_DIM]; /* periodic box, h_d = (hi-lo)/n_d > 0      */
} sldg_domain;

/* Distribution over `world` GPUs (one process per GPU).  The outermost dim D-1 (D >= 2) is
 * block-sharded: rank r owns global layers [r*n/world + min(r, n%world) ...) (balanced).
 * Sweeps along dims < D-1 are communication-free; a sweep along D-1 exchanges halo layers
 * with NCCL send/recv over NVLink.  Exactly one of nccl_unique_id / nccl_comm is non-NULL. */
typedef struct {
    int rank, world;
    const void* nccl_unique_id; /* 128-byte ncclUniqueId, identical on all ranks, or NULL  */
    void* nccl_comm;            /* caller-owned ncclComm_t (rank/world must match), or NULL */
    int max_halo;               /* halo layers allocated per side; <= 0 selects 2          */
    int flags;                  /* SLDG_DIST_* bits                                        */
} sldg_dist;
/* Test-only bits of `flags` (one-GPU stand-ins for the multi-GPU paths) are in
 * include/sldg_testing.h. */
/* Peer-mapped halos: the pad layers of both coefficient arrays are CUDA
 * virtual-memory mappings of the ring neighbours' edge layers (left pad = the left neighbour's
 * last `max_halo` layers, right pad = the right neighbour's first ones; with world == 1 and
 * SLDG_DIST_FORCE_HALO (sldg_testing.h), this rank's own).  A sweep along the sharded dim whose halo fits the
 * pads is then ONE launch over all local layers whose boundary tiles read the neighbours' HBM
 * directly (NVLink for another GPU): no exchange step.  world > 1: an NCCL fence with both
 * neighbours before and after such a sweep (device-side, capturable); the chunks are shared
 * between processes as POSIX file descriptors over abstract unix sockets (SCM_RIGHTS; no ptrace
 * rights needed).  Creation is collective and fails
 * with ENOTSUP unless sldg_peer_halo_check accepts the layout at the device's allocation
 * granularity. */
#define SLDG_DIST_PEER_HALO 8

/* Create a grid (zero-filled).  k in 1..SLDG_MAX_K coefficients per dim (the paper's order
 * o = p+1).  dist may be NULL (single GPU).  The device is the caller's current
 * CUDA device.  Errors: EINVAL (ndim, k, n_d < 1, lo >= hi, world/rank, sharded extent
 * < world), ENOMEM, ECUDA, ENCCL. */
sldg_status sldg_create(const sldg_grid_desc* grid, int k, const sldg_domain* dom,
                        sldg_precision prec, const sldg_dist* dist, sldg_grid* out);
/* General precision layout (the paper's "# double", SS III-A, Tables II-VI): coefficient slots
 * q < n_double (linear index of the host layout) are stored in fp64, the others in fp32
 * (RNE); arithmetic is fp64 either way.  n_double = 1 is SLDG_MIXED, n_double = k^D is
 * SLDG_FP64, n_double = 0 is pure fp32 storage (mass no longer conserved to fp64).
 * Values other than 1 and k^D: 1D grids only (ENOTSUP otherwise). */
sldg_status sldg_create_ex(const sldg_grid_desc* grid, int k, const sldg_domain* dom, int n_double,
                           const sldg_dist* dist, sldg_grid* out);
sldg_status sldg_destroy(sldg_grid g);

/* Copy n_cells cells starting at local cell first_cell from host fp64 (layout above) into
 * the grid; fp32 slots are rounded to nearest-even.  Validation before any
 * write (all-or-nothing): range inside the local shard; every value finite; every fp32
 * slot |v| <= FLT_MAX.  Blocks until the copy is complete. */
sldg_status sldg_set_coeffs(sldg_grid g, const double* src, int64_t first_cell, int64_t n_cells);
/* Copy cells out to host fp64 (fp32 slots promoted exactly).  Blocks. */
sldg_status sldg_get_coeffs(sldg_grid g, double* dst, int64_t first_cell, int64_t n_cells);

/* One SLDG sweep along dim.  shift/field are CFL numbers in cells (R2).
 * field == NULL: every line uses nu = shift.  Otherwise `field` (HOST memory) holds one nu
 * per combination of the dims set in field_mask, indexed sum_{e in mask, ascending}
 * i_e * prod_{e' in mask, e' < e} n_e' over GLOBAL indices; unmasked perpendicular dims
 * broadcast (per-line variable CFL).  Errors (EINVAL, no state change): dim out
 * of range, bit `dim` set in field_mask, mask bits >= D, non-finite or |nu| >= 2^62 entry
 * (S:211).  A sharded sweep whose halo exceeds max_halo (or would move more data than a
 * re-shard) takes the transpose path (sldg_transpose_plan).  Asynchronous. */
sldg_status sldg_advect(sldg_grid g, int dim, double shift, const double* field, uint32_t field_mask);
/* Same, with the field already resident in DEVICE memory (d_field, fp64, same indexing).
 * Entries are validated on the device: a non-finite entry leaves its lines unchanged and
 * makes the next blocking call return EINVAL (sticky device error). */
sldg_status sldg_advect_device(sldg_grid g, int dim, double shift, const double* d_field,
                               uint32_t field_mask);
/* Same, with a caller-supplied bound: every entry of d_field lies in [nu_min, nu_max] (host
 * doubles, finite, nu_min <= nu_max).  A sweep along the sharded dim then sizes its halo (and
 * chooses halo or transpose) from the bound's integer parts floor(nu_min),
 * floor(nu_max) instead of reading the field's range back to the host, so it never blocks and
 * can be captured in a CUDA graph.  Entries outside the bound are found on the device: their
 * lines are left unchanged and the next blocking call returns EINVAL (sticky device error),
 * as for non-finite entries.  Errors: EINVAL (null field, bad bound, as sldg_advect_device).
 * Asynchronous. */
sldg_status sldg_advect_device_bounded(sldg_grid g, int dim, double shift, const double* d_field,
                                       uint32_t field_mask, double nu_min, double nu_max);

/* Two sweeps of a split step: along dim 0 with (shift0, field0, mask0), then along dim 1 with
 * (shift1, field1, mask1) -- exactly sldg_advect(g, 0, ...) followed by sldg_advect(g, 1, ...)
 * (P:144-149 dimension splitting, each sweep P:259-272), including the intermediate rounded to
 * the storage precision.  When both fields are constant over dims 0 and 1 (they depend only on
 * dims >= 2, as the x1 / x2 CFL numbers v1, v2 of the 4D Vlasov workload) and D >= 3,
 * 32 <= n_0 <= 256 with 256 % n_0 == 0, k <= 3, the pair runs as ONE pass over HBM (one read
 * and one write of every stored coefficient for both sweeps), with results bit
 * for bit those of the two sweeps; otherwise as the two sweeps.  Fields: HOST memory
 * (sldg_advect_pair; copied before return) or DEVICE memory (_device; validated on the device as
 * in sldg_advect_device).  Errors: EINVAL as sldg_advect.  Asynchronous. */
sldg_status sldg_advect_pair(sldg_grid g, double shift0, const double* field0, uint32_t mask0, double shift1,
                             const double* field1, uint32_t mask1);
sldg_status sldg_advect_pair_device(sldg_grid g, double shift0, const double* d_field0, uint32_t mask0,
                                    double shift1, const double* d_field1, uint32_t mask1);

/* Gauss-node velocity treatment of an x-sweep (NEXT-3, reading V7): a sweep along
 * `dim` whose CFL number varies with the velocity coordinate of dim `vdim` INSIDE each v-cell.
 * Per v-cell j: modal -> nodal in vdim at the k Gauss-Legendre nodes, one SLDG line
 * update per node with its own CFL number, nodal -> modal by Gauss quadrature
 * (S:303).  nodal_nu[j * k + n] = nu at node n (ascending xi_n) of v-cell j (GLOBAL j),
 * HOST memory (sldg_advect_vnodes) or DEVICE memory (_device; non-finite entries leave their
 * v-cell unchanged and make the next blocking call return EINVAL).  fp64 arithmetic, RNE
 * stores; no exact-copy path (the nodal transform pair is the identity only up to rounding).
 * Errors: EINVAL (dims equal / out of range, null or non-finite field), ENOTSUP (k > 4; dim
 * is the sharded layer dim); the nodes of one v-cell spanning more than 5 integer parts make
 * that cell's lines unchanged with the sticky EINVAL).  Asynchronous. */
sldg_status sldg_advect_vnodes(sldg_grid g, int dim, int vdim, const double* nodal_nu);
sldg_status sldg_advect_vnodes_device(sldg_grid g, int dim, int vdim, const double* d_nodal_nu);
/* Total mass M = (prod_d h_d) * sum_cells c_{cell,0}, a deterministic
 * fixed-order fp64 reduction; collective over ranks (rank-ordered sum).  Blocks. */
sldg_status sldg_mass(sldg_grid g, double* mass_out);

/* Local shard: first global layer along dim D-1 and number of local layers (1D: 0, 1). */
sldg_status sldg_shard_info(sldg_grid g, int64_t* first_layer, int64_t* n_layers);
sldg_status sldg_sync(sldg_grid g);
/* Use an external CUDA stream (cudaStream_t) for all subsequent work (NULL = own stream). */
sldg_status sldg_set_stream(sldg_grid g, void* cuda_stream);
sldg_status sldg_get_stream(sldg_grid g, void** cuda_stream);
/* Bytes of one coefficient array of the local shard: cells*(8+4(K-1)) mixed, cells*8K fp64
 * (S:163-169); the library holds two (ping-pong) plus halo layers. */
size_t sldg_memory_bytes(sldg_grid g);
const char* sldg_last_error(void);

/* ---- synthetic inputs; not part of the method ----------------------------- */
/* Counter-based parity generator, bit-identical to sldg_inputs.random_coeffs:
 * u = (splitmix64(seed*2^40 + g*K + q) >> 11) * 2^-53, r = 2u-1, c_0 = 1 + r/2,
 * c_m = r / n_0^{|m|_1}; g = GLOBAL cell index.  Asynchronous. */
sldg_status sldg_fill_random(sldg_grid g, uint64_t seed);
/* c[cell,q] = sum_t prod_d T[t][d][i_d][m_d]; `tables` is HOST fp64, concatenated over
 * t (n_terms) then d then [n_d global][k].  Used for Landau-type initial values. */
sldg_status sldg_fill_separable(sldg_grid g, int n_terms, const double* tables);

/* ---- instrumentation (for the bench harness) ------------------------------------------- */
/* When enabled, CUDA events bracket every sweep kernel on the handle's stream. */
sldg_status sldg_profile(sldg_grid g, int enable);
/* Sum of sweep-kernel durations (ms) since the last reset for sweeps along `dim` (-1: all
 * dims and fused pairs, -2: fused sweep pairs only), their launch count, and the algorithmic
 * bytes those launches moved (one load + one store per stored coefficient; a fused
 * pair counts its single pass).  Blocks.  reset != 0 clears all accumulators. */
sldg_status sldg_kernel_time(sldg_grid g, int dim, double* ms, int64_t* launches, double* bytes, int reset);
/* Profile mode: the device intervals (ms from the first recorded one) of every sweep launch
 * (kinds[i] = its dim; -2 for a fused sweep pair) and every halo exchange on the comm stream
 * (kinds[i] = -1), in the order
 * they were enqueued: 2 doubles per entry in t_ms.  Shows whether the interior sweep of a
 * sharded sweep overlaps its halo exchange.  *n_out = number of recorded entries (the first 4096
 * after a reset are kept; up to max_entries are written); reset != 0 clears them.  Blocks. */
sldg_status sldg_timeline(sldg_grid g, double* t_ms, int* kinds, int max_entries, int* n_out, int reset);
/* Number of kernels this handle has launched (all kinds). */
int64_t sldg_launch_count(sldg_grid g);
/* Name of the sweep kernel a sweep along `dim` uses on this grid (static string; "" on bad
 * arguments): the TMA-staged kernels when their shape constraints hold, else the register
 * kernels. */
const char* sldg_sweep_kernel(sldg_grid g, int dim);

/* ---- CUDA graphs ------------------------------------------------------------------------ */
/* Capture a sequence of ASYNCHRONOUS calls on this grid (sldg_advect with field == NULL,
 * sldg_advect_device, sldg_advect_vnodes_device, sldg_fill_*) into a CUDA graph and replay
 * it with one launch: for small grids whose sweeps are shorter than the host's per-call cost.
 * Nothing runs during the capture.  A replay must start on the buffer the capture started on
 * (an odd number of sweeps flips the ping-pong buffer: capture two steps).  Device shift
 * fields must stay valid and are read at replay time.  Sharded grids: a device-field sweep
 * along the sharded dim must use sldg_advect_device_bounded (its halo exchange, NCCL on the
 * grid's comm stream, is captured with it), and a transpose-path sweep must have run once
 * before (its buffers are allocated on first use).  Errors: EINVAL (capture already open /
 * not open, host field during capture, unbounded device field along the sharded dim, wrong
 * current buffer at launch), ECUDA (a blocking call was made inside the capture; the capture
 * is then invalid). */
typedef struct sldg_graph_s* sldg_graph;
sldg_status sldg_graph_begin(sldg_grid g);
sldg_status sldg_graph_end(sldg_grid g, sldg_graph* out);
sldg_status sldg_graph_launch(sldg_graph gr);
sldg_status sldg_graph_destroy(sldg_graph gr);

/* ---- distributed helpers ---------------------------------------------------------------- */
/* Write a fresh 128-byte ncclUniqueId into out128 (call on rank 0, broadcast it). */
sldg_status sldg_nccl_unique_id(void* out128);
/* Host-only halo planner for a sweep along the sharded dim (no device, no NCCL):
 * given global extent n, world, rank and the integer-shift range [imin, imax] of the
 * sweep's lines (i* = floor(nu)), returns the halo widths this rank needs on the left
 * (layers below its first layer) and right.  Lines with integer part i* read layers
 * i - i* - 1 and i - i*, so left = max(0, imax + 1), right = max(0, -imin). */
sldg_status sldg_halo_widths(int64_t imin, int64_t imax, int64_t* left, int64_t* right);
/* Host-only halo transfer plan of `rank` for a sharded sweep with halo widths (left, right)
 * and `pad` halo layers per side: 4 int64 per entry {kind, peer, slot, src} where kind 0 =
 * receive into padded local layer `slot` from `peer`, 1 = send padded local layer `slot` to
 * `peer`, 2 = copy own padded layer `src` into `slot`.  Entries to/from one peer appear in
 * the receiver's halo-slot order on both sides (the order NCCL pairs them in).  out == NULL
 * returns only *n_entries.  This is exactly the plan sldg_advect executes with NCCL. */
sldg_status sldg_halo_plan(int64_t n, int world, int rank, int64_t pad, int64_t left, int64_t right,
                           int64_t* out, int64_t max_entries, int64_t* n_entries);
/* Owner rank and local index of global layer `layer` in a balanced block split of n over
 * world ranks. */
sldg_status sldg_layer_owner(int64_t n, int world, int64_t layer, int* owner, int64_t* local);
/* Host-only plan of the TRANSPOSE path of a sweep along the sharded dim D-1:
 * taken when the halo exceeds max_halo, or when the halo would move more than the transpose
 * (left + right > 2 n_local (P-1)/P).  The slab dim D-2 (extent n_slab) is block-split over
 * the ranks like the layer dim (extent n_outer); rank r sends to every rank p its own layers
 * restricted to p's slab, receives from p p's layers restricted to r's slab (whole lines along
 * D-1 for its slab), sweeps them locally with periodic wrap, and returns them the same way.
 * out[8 p + 0..3] = {send layer first, send layer count, send slab first, send slab count},
 * out[8 p + 4..7] = {recv layer first, recv layer count, recv slab first, recv slab count}
 * for p = 0..world-1 (out holds 8 * world int64).  The forward and inverse messages of
 * sldg_advect follow exactly this plan (inverse = the same pairs reversed). */
sldg_status sldg_transpose_plan(int64_t n_outer, int64_t n_slab, int world, int rank, int64_t* out);
/* Host-only check of SLDG_DIST_PEER_HALO for a grid (`prec` SLDG_MIXED or SLDG_FP64, k, the
 * global extents), `world` ranks, `pad` halo layers per side and allocation granularity `gran`
 * bytes (the device's minimum; 2 MiB on B200): every rank must hold >= 2 pad layers, and pad
 * and every rank's layer count times the per-layer bytes of each precision section (fp64
 * planes, fp32 planes) must be multiples of gran.  SLDG_OK, else ENOTSUP with the reason in
 * sldg_last_error(); EINVAL for bad arguments. */
sldg_status sldg_peer_halo_check(const sldg_grid_desc* grid, int k, sldg_precision prec, int world, int pad,
                                 int64_t gran);
/* Number of sweeps of this handle that took the transpose path. */
sldg_status sldg_transpose_count(sldg_grid g, int64_t* n);

/* ---- Vlasov-Poisson driver around the sweep (NEXT-2, readings V1-V6) -------
 * The model is the paper's: d_t f + v.grad_x f + E(x).grad_v f = 0, reduced by
 * Cheng-Knorr splitting to 1D advections whose CFL number depends on the field
 * (P:269-272).  The paper does not state the field solver; the one here follows S:267-334
 * (V2-V3) and a spectral reading for two space dims (V4).
 * Grid: D = 2 dx dims ordered [x_1..x_dx, v_1..v_dx] (dx = 1, 2 or 3); x_c pairs with v_c.
 * Density rho[i_x * k^dx + m_x] (i_x = sum_c i_xc S_c over the x dims, m_x likewise):
 *   rho = (prod_c h_vc) sum_{i_v} c_{(i_x, i_v), (m_x, m_v = 0)}                        (V2)
 * Field, dx = 1: d_x E = rho - mean(rho), periodic, zero mean, exact antiderivative of the
 *   DG density per cell (E of degree k per cell; coefficients e[i * (k+1) + n])          (V3)
 * Field, dx = 2, 3: -Lap phi = rho - mean, E = -grad phi, spectral on the cell means
 *   (Nyquist modes of the derivative zeroed), sampled at cell centres                     (V4)
 * E at x-cell centres: e_out[c * N_x + i_x].  Energy: 1/2 int |E|^2 (exact for dx = 1,
 *   cell-centre rule for dx >= 2).
 * CFL fields (R7, V5): x_c sweeps nu = v_c(cell centre) tau / h_xc over the v_c dim; v_c
 *   sweeps nu = E_c(x-cell centre) tau / h_vc over the x dims.
 * Strang step (V6): x sweeps dt/2; density; field; v sweeps dt; x sweeps dt/2 --
 *   every step on the grid's stream, no host round trip (except the halo range check of a
 *   sharded v sweep).  Distributed grids: the density is summed over ranks in rank order
 *   (ncclAllGather of the partial sums); calls are collective.
 * Errors: EINVAL for a grid that is not [x.., v..] with dx in {1, 2, 3} or for null handles.
 * Ownership: the driver holds device buffers; the grid must outlive it. */
typedef struct sldg_vp_s* sldg_vp;
sldg_status sldg_vp_create(sldg_grid g, int dx, sldg_vp* out);
sldg_status sldg_vp_destroy(sldg_vp vp);
/* Density of the grid's current f (V2).  rho_out: HOST, N_x * k^dx doubles, or NULL (device
 * only).  Blocks when rho_out != NULL. */
sldg_status sldg_vp_density(sldg_vp vp, double* rho_out);
/* Field from a given HOST density rho (N_x * k^dx) -- or, rho == NULL, from the grid's current
 * f -- into the optional HOST outputs: e_out (dx * N_x centre values), e_coef (dx = 1 only:
 * N_x * (k+1) Legendre coefficients of E per cell), energy.  Blocks when any output is given. */
sldg_status sldg_vp_field(sldg_vp vp, const double* rho, double* e_out, double* e_coef, double* energy);
/* on != 0: the x sweeps of sldg_vp_step use the Gauss-node velocity treatment (V7,
 * sldg_advect_vnodes: nu at the k Gauss nodes of every v-cell) instead of the cell-centre
 * velocity (V5).  ENOTSUP for k > 4. */
sldg_status sldg_vp_set_nodal(sldg_vp vp, int on);
/* One Strang step of length dt (V6).  energy_out (HOST or NULL): electric energy of the
 * mid-step field (blocks when given).  Asynchronous otherwise. */
sldg_status sldg_vp_step(sldg_vp vp, double dt, double* energy_out);

#ifdef __cplusplus
}
#endif
#endif /* SLDG_H */
