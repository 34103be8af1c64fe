/* sldg_testing.h -- test-only bits of sldg_dist.flags (include/sldg.h).  Each runs a multi-GPU
 * code path on ONE GPU, with the rank as its own ring neighbour, so the single-GPU tests and
 * benches exercise the exact addressing, message plans and NCCL calls of sharded runs.  Not for
 * production use: they change no results, only which path computes them. */
#ifndef SLDG_TESTING_H
#define SLDG_TESTING_H

#include "sldg.h"

/* Run sweeps along the sharded dim through the halo path even when world == 1 (the ring
 * neighbour is the rank itself: halo layers are device copies).  Exercises the exact halo
 * addressing of multi-GPU runs on one GPU; no NCCL communicator is needed. */
#define SLDG_DIST_FORCE_HALO 1
/* Every sweep along the layer dim takes the transpose path (testing on one GPU; see
 * sldg_transpose_plan).  Implies the halo layout. */
#define SLDG_DIST_FORCE_TRANSPOSE 2
/* world == 1 only: create a one-rank NCCL communicator and send this rank's own halo layers,
 * transpose blocks and density partials through ncclSend/ncclRecv/ncclAllGather instead of
 * device copies -- the multi-GPU NCCL code paths (message pointers, counts, pairing order)
 * exercised on one GPU. */
#define SLDG_DIST_NCCL_SELF 4
/* Testing (with SLDG_DIST_PEER_HALO, world == 1): the rank's own edge chunks are exported as
 * POSIX file descriptors, passed back over the rank's own unix socket and imported -- the descriptor path of
 * world > 1 exercised in one process. */
#define SLDG_DIST_PEER_VIA_FD 16

#endif /* SLDG_TESTING_H */
