// common.cuh — shared device primitives of the CRSH library: single-pass
// decoupled look-back prefix (Merrill & Garland) used by the trim, chunk,
// decompression-scan and plan kernels, warp helpers, and launch constants.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define CRSH_FULL 0xFFFFFFFFu

namespace crsh {

// Checked build (-DCRSH_CHECKED=1, tools/build_ab.sh checked -DCRSH_CHECKED=1):
// device-side bounds checks of every indexed write of the hot kernels; the
// first failing check's id is kept in g_crsh_check and reported by crsh_stats
// as CRSH_ECUDA. The stand-in for compute-sanitizer memcheck, which is closed
// on this GPU pool (B200_PROFILING.md); compiled out otherwise.
#ifndef CRSH_CHECKED
#define CRSH_CHECKED 0
#endif
__device__ unsigned int g_crsh_check = 0u;
#define CRSH_CHECK(cond, id)                                                     \
  do {                                                                           \
    if (CRSH_CHECKED && !(cond)) atomicCAS(&::crsh::g_crsh_check, 0u, (unsigned)(id)); \
  } while (0)

constexpr int MAX_SEG = 3;
constexpr int MAX_LEVELS = 8;

// ---------------------------------------------------------------- frame descriptor
// Per-frame counts that only the GPU knows (rays after trimming, chunks, the
// padded segment layout, level sizes, work items). Written by k_raygen /
// k_frame_plan / k_rle / k_chunk_plan / k_plan and read by every later kernel,
// so the host never waits for them: all grids are sized from static upper
// bounds and surplus blocks exit, and the whole frame is one CUDA graph.
struct FrameDesc {
  uint32_t N;                          // non-empty rays (all segments)
  uint32_t seg_comp_start[MAX_SEG + 1];// compacted start of each segment; [n_seg] = N
  uint32_t seg_n[MAX_SEG];
  uint32_t seg_pad_base[MAX_SEG + 1];  // padded sorted-ray base (multiple of the group span); [n_seg] = Np
  uint32_t Np, G;                      // padded rays, traversal groups
  uint32_t C;                          // chunks
  uint32_t seg_chunk_start[MAX_SEG + 1];
  uint32_t seg_C[MAX_SEG];
  uint32_t sort_tile_start[MAX_SEG + 1];
  uint32_t n_items;                    // traversal work items
  uint32_t g_lo, g_hi;                 // this rank's traversal groups [g_lo, g_hi) (work-balanced cut, k_cut)
  uint32_t level_n[MAX_LEVELS + 1];    // padded nodes at level k
};

// Fused multi-GPU epilogue (crsh_trace_secondary_peer): destination packed
// buffers (this rank's and its peers', e.g. NVLink peer pointers); n = 0 off.
constexpr int MAX_PEERS = 8;
struct PeerOut {
  unsigned long long* p[MAX_PEERS];
  int32_t n;
  __device__ __forceinline__ void store(size_t slot, unsigned long long v) const {
    for (int d = 0; d < n; ++d) p[d][slot] = v;
  }
};

// k_frame_plan: padded layout from the segment counts (one warp).
__global__ void k_frame_plan(FrameDesc* fd, int n_seg, uint32_t GR, uint32_t B0, uint32_t B, int Lv) {
  if (threadIdx.x != 0) return;
  uint32_t base = 0;
  for (int s = 0; s < n_seg; ++s) {
    const uint32_t n = fd->seg_comp_start[s + 1] - fd->seg_comp_start[s];
    fd->seg_n[s] = n;
    fd->seg_pad_base[s] = base;
    base += (n + GR - 1) / GR * GR;
  }
  fd->seg_pad_base[n_seg] = base;
  fd->N = fd->seg_comp_start[n_seg];
  fd->Np = base;
  fd->G = base / GR;
  uint32_t per = B0;
  for (int k = 1; k <= Lv; ++k) { fd->level_n[k] = base / per; per *= B; }
}

// ---------------------------------------------------------------- scan tiles
// 256 threads x 8 items, striped (item i of thread t = tile_base + i*256 + t):
// coalesced loads, and the (item, warp) lexicographic order equals slot order.
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Look-back status word: high 32 bits = flag (0 none, 1 aggregate, 2 inclusive
// prefix), low 32 bits = value. One 64-bit store publishes flag and value
// together, so readers never see a flag without its value.
__device__ __forceinline__ void lb_store(unsigned long long* p, uint32_t flag, uint32_t v) {
  const unsigned long long w = ((unsigned long long)flag << 32) | v;
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long lb_load(const unsigned long long* p) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}

// Single-pass scan tile (Merrill & Garland decoupled look-back), called by
// EVERY thread of the block (it contains barriers): warp 0 scans the 64
// (item, warp) counts of s_cnt (flattened item-major) into s_excl and
// publishes the tile aggregate; then all threads look back together, thread i at
// predecessor tile - 1 - i, so one round trip covers blockDim.x predecessors
// (a warp-only look-back covers 32): with many tiles resident at once, tile
// k waits ~k / (2 window) round trips for the inclusive frontier. Measured
// against the warp-only look-back: cfg2 generate+trim 31.9 -> 28.6 us,
// compress 18.9 -> 16.2 us; neutral at cfg4, where the tiles are bound by
// their own work (k_raygen: ~370 instructions per slot of IEEE div/sqrt and
// the hash polynomial).
// NE = (item, warp) entries of s_cnt (SCAN_ITEMS * 8 by default; a multiple of 32).
template <int NE = SCAN_ITEMS * 8>
__device__ __forceinline__ uint32_t tile_scan_lookback_block(const uint32_t* s_cnt, uint32_t* s_excl, uint32_t* s_prefix,
                                                             unsigned long long* status, int tile) {
  __shared__ uint32_t s_lb_total, s_lb_stop, s_lb_red[32];
  const int tid = (int)threadIdx.x, lane = (int)lane_id(), warp = tid >> 5, nw = (int)(blockDim.x >> 5);
  if (warp == 0) {
    constexpr int PER = NE / 32;
    uint32_t x[PER], sum = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) { x[q] = s_cnt[PER * lane + q]; sum += x[q]; }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(CRSH_FULL, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t run = incl - sum;
#pragma unroll
    for (int q = 0; q < PER; ++q) { s_excl[PER * lane + q] = run; run += x[q]; }
    const uint32_t total = __shfl_sync(CRSH_FULL, incl, 31);
    if (lane == 0) {
      s_lb_total = total;
      lb_store(&status[tile], tile == 0 ? 2u : 1u, total);
    }
  }
  __syncthreads();
  const uint32_t total = s_lb_total;
  uint32_t excl = 0;
  if (tile > 0) {   // block-uniform
    int p = tile - 1;
    for (;;) {
      const int idx = p - tid;
      unsigned long long w = idx >= 0 ? lb_load(&status[idx]) : (2ull << 32);
      while ((w >> 32) == 0ull) w = lb_load(&status[idx]);   // predecessors were dispatched earlier: they publish
      if (tid == 0) s_lb_stop = 0xFFFFFFFFu;
      __syncthreads();
      if ((w >> 32) == 2ull) atomicMin(&s_lb_stop, (uint32_t)tid);   // nearest inclusive prefix in the window
      __syncthreads();
      const uint32_t stop = s_lb_stop;
      const uint32_t v = __reduce_add_sync(CRSH_FULL, (uint32_t)tid <= stop ? (uint32_t)w : 0u);
      if (lane == 0) s_lb_red[warp] = v;
      __syncthreads();
      uint32_t sum = 0;
      for (int q = 0; q < nw; ++q) sum += s_lb_red[q];
      excl += sum;
      if (stop != 0xFFFFFFFFu) break;
      p -= (int)blockDim.x;
      __syncthreads();   // s_lb_stop / s_lb_red are reused
    }
    if (tid == 0) lb_store(&status[tile], 2u, excl + total);
  }
  if (tid == 0) *s_prefix = excl;
  return total;
}

// Per-segment counter add from a whole warp: lane values are summed per
// segment with one warp reduction each and added by lane 0 -- one 64-bit
// shared atomic per (warp, segment) instead of one contended CAS loop per
// thread (64-bit shared atomics are CAS loops). Call with all 32 lanes.
__device__ __forceinline__ void warp_seg_add(unsigned long long* base, int stride, int n_seg, int seg, uint32_t v) {
  for (int q = 0; q < n_seg; ++q) {
    const uint32_t sq = __reduce_add_sync(CRSH_FULL, seg == q ? v : 0u);
    if (sq && (threadIdx.x & 31) == 0) atomicAdd(base + q * stride, (unsigned long long)sq);
  }
}

// Block-wide exclusive scan of one uint32 per thread (blockDim.x == 32 NW).
template <int NW>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp /*NW*/, uint32_t* total);

// Block-wide exclusive scan of one uint32 per thread (blockDim.x == 256).
__device__ __forceinline__ uint32_t block_excl_scan_256(uint32_t v, uint32_t* s_warp /*8*/, uint32_t* total) {
  return block_excl_scan<8>(v, s_warp, total);
}

template <int NW>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp /*NW*/, uint32_t* total) {
  const int lane = (int)lane_id(), warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(CRSH_FULL, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const uint32_t x = s_warp[w];
    wpre += (w < warp) ? x : 0u;
    tot += x;
  }
  __syncthreads();
  if (total) *total = tot;
  return wpre + incl - v;
}

}  // namespace crsh
