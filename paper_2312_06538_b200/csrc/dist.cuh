// dist.cuh — the multi-GPU data plane of the library (SURVEY §8(a) a14,
// §8(b) crsh_dist_init, §8(e)): an NCCL communicator per scene, a symmetric
// NCCL window holding the packed per-slot result of a frame, and the two
// merges of the per-rank results.
//
//  * PEER (default): the fused variant of §8(e). The epilogue kernels of every
//    rank store the packed result of each ray it owns -- and the empty
//    sentinel into every ray-less slot -- straight into EVERY rank's window
//    through the NVLink load/store (LSA) pointers of the window
//    (ncclGetLsaPointer, resolved once per window on the device). Each slot
//    of each window is therefore written with its final value by exactly one
//    rank (the empty sentinel by all, identically), so after an LSA barrier
//    every rank holds the merged frame without a reduction; k_unpack_packed
//    turns it into hit_tri / t. A second LSA barrier at the start of the next
//    frame keeps a fast rank from overwriting a window a peer still reads.
//  * NCCL: the plain variant of §8(e): every rank writes its packed frame
//    (owned slots; UINT64-MAX-like sentinels elsewhere) into its own window
//    buffer, then ncclAllReduce(ncclMin, ncclUint64) merges it in place.
//
// Both run inside the frame's CUDA graph (NCCL collectives are capturable).
// The per-rank traversal counters are summed with ncclAllReduce(ncclSum) in
// both modes. The mode is agreed by all ranks at crsh_dist_init (an
// all-reduce MIN of each rank's capability), so no rank can wait in a merge
// its peers do not run. Any NCCL failure surfaces as CRSH_ENCCL.
#pragma once
#include <nccl.h>
#include <nccl_device.h>

#include "common.cuh"

namespace crsh {

enum { MERGE_NONE = 0, MERGE_NCCL = 1, MERGE_PEER = 2 };

struct Dist {
  ncclComm_t comm = nullptr;
  ncclDevComm dev{};
  bool dev_ok = false;
  int rank = 0, world = 1;
  int mode = MERGE_NCCL;
  ncclWindow_t win = nullptr;       // symmetric window over wbuf
  void* wbuf = nullptr;             // ncclMemAlloc'd packed frame ([slots] u64)
  size_t wcap = 0;                  // bytes
  PeerOut peers{};                  // LSA pointers of every rank's window (PEER mode)
  unsigned long long* d_ptrs = nullptr;   // scratch for k_window_peers
};

// LSA barrier over all ranks (one CTA). The release/acquire of the barrier
// orders the peer stores of the preceding kernels (stream order makes them
// visible to this kernel; the system-scope fence publishes them) before any
// rank's following kernels.
__global__ void k_lsa_barrier(ncclDevComm comm) {
  __threadfence_system();
  ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamTagLsa(), 0);
  bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

// device addresses of the window on every LSA peer (rank order)
__global__ void k_window_peers(ncclWindow_t w, int n, unsigned long long* out) {
  const int p = threadIdx.x;
  if (p < n) out[p] = (unsigned long long)ncclGetLsaPointer(w, 0, p);
}

}  // namespace crsh
