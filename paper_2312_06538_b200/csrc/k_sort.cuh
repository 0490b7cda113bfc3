// k_sort.cuh — K2 compression into chunks (Fig 5), K3 LSD radix
// sort of the chunks by key (P:107-109 [MG10]; onesweep-style), K4
// decompression (Fig 6: skeleton of sorted sizes, exclusive scan,
// fill). Together: a stable sort of the (key, slot) pairs of every segment
// (SURVEY F7), with bit-exact keys and permutation.
#pragma once
#include "common.cuh"

namespace crsh {

// ============================================================== K2: compression
struct RleArgs {
  FrameDesc* fd;                        // in: N, seg_comp_start; out: seg_chunk_start, C
  const uint32_t* keys;                 // compacted keys [N]
  int32_t n_seg;
  uint32_t* ckey;                       // [C]
  uint32_t* cbase;                      // [C + 1], global compacted index of each chunk head
  uint32_t* hist;                       // optional [3][4][256]: digit histograms of the chunk keys (zeroed)
  unsigned long long* status;
  uint32_t* ticket;
};
constexpr int RLE_HIST_WORDS = MAX_SEG * 4 * 256;

// Head flag: 1 where the key differs from the previous pair; also at
// every segment start so chunks never straddle two hierarchies (R5).
// RLE_ITEMS keys per thread (32 for large frames: a quarter of the tiles, so
// a quarter of the look-back chain). With `hist` (all segments' digit
// histograms of the chunk keys, the radix sort's first step) the tile also
// counts its chunk keys' digits in shared memory and adds them to the global
// histograms -- the separate histogram pass over the chunk keys is gone.
template <int RLE_ITEMS>
__global__ void __launch_bounds__(SCAN_THREADS) k_rle(const RleArgs a) {
  constexpr int NE = RLE_ITEMS * 8;
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ uint32_t s_cnt[NE], s_excl[NE];
  __shared__ uint32_t s_hist[RLE_HIST_WORDS];
  if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1u);
  if (a.hist)
    for (int i = threadIdx.x; i < RLE_HIST_WORDS; i += SCAN_THREADS) s_hist[i] = 0u;
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t N = a.fd->N;
  constexpr uint32_t TILE = (uint32_t)SCAN_THREADS * RLE_ITEMS;
  const uint32_t n_tiles = (N + TILE - 1) / TILE;
  if (tile >= n_tiles) return;   // surplus block (grid sized from the slot bound)
  // segment starts in registers: every loop over them is unrolled to MAX_SEG
  // with a bound check (a runtime-indexed array would live in local memory)
  uint32_t segst[MAX_SEG + 1];
#pragma unroll
  for (int s = 0; s <= MAX_SEG; ++s) segst[s] = s <= a.n_seg ? a.fd->seg_comp_start[s] : 0xFFFFFFFFu;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t key[RLE_ITEMS], ballot[RLE_ITEMS];
#pragma unroll
  for (int it = 0; it < RLE_ITEMS; ++it) {
    const uint32_t i = tile * TILE + it * SCAN_THREADS + threadIdx.x;
    bool head = false;
    uint32_t k = 0;
    if (i < N) {
      k = __ldg(a.keys + i);
      head = (i == 0) || (k != __ldg(a.keys + i - 1));
#pragma unroll
      for (int s = 0; s < MAX_SEG; ++s) head |= (s < a.n_seg) & (i == segst[s]);
    }
    key[it] = k;
    ballot[it] = __ballot_sync(CRSH_FULL, head);
    if (lane == 0) s_cnt[it * 8 + warp] = __popc(ballot[it]);
  }
  __syncthreads();
  tile_scan_lookback_block<NE>(s_cnt, s_excl, &s_prefix, a.status, (int)tile);
  __syncthreads();
  const uint32_t prefix = s_prefix, lt = lanemask_lt();
#pragma unroll
  for (int it = 0; it < RLE_ITEMS; ++it) {
    const uint32_t i = tile * TILE + it * SCAN_THREADS + threadIdx.x;
    if ((ballot[it] >> lane) & 1u) {
      const uint32_t c = prefix + s_excl[it * 8 + warp] + __popc(ballot[it] & lt);
      CRSH_CHECK(c < N, 201);
      a.ckey[c] = key[it];
      a.cbase[c] = i;
      int sg = 0;
#pragma unroll
      for (int s = 0; s < MAX_SEG; ++s) {
        if (s < a.n_seg && i == segst[s]) a.fd->seg_chunk_start[s] = c;
        sg = (s < a.n_seg && i >= segst[s]) ? s : sg;
      }
      if (a.hist) {
        const uint32_t k = key[it];
#pragma unroll
        for (int p = 0; p < 4; ++p) atomicAdd(&s_hist[(sg * 4 + p) * 256 + ((k >> (8 * p)) & 255u)], 1u);
      }
    }
  }
  if (tile == n_tiles - 1 && threadIdx.x == 0) {
    uint32_t t = 0;
    for (int q = 0; q < NE; ++q) t += s_cnt[q];
    const uint32_t C = prefix + t;
    a.cbase[C] = N;
    a.fd->seg_chunk_start[a.n_seg] = C;
    a.fd->C = C;
#pragma unroll
    for (int s = 0; s < MAX_SEG; ++s)
      if (s < a.n_seg && segst[s] >= N) a.fd->seg_chunk_start[s] = C;   // empty trailing segment
  }
  if (a.hist) {
    __syncthreads();
    for (int i = threadIdx.x; i < a.n_seg * 4 * 256; i += SCAN_THREADS)
      if (s_hist[i]) atomicAdd(a.hist + i, s_hist[i]);
  }
}

// per-segment chunk counts and sort-tile offsets (one thread)
__global__ void k_chunk_plan(FrameDesc* fd, int n_seg, uint32_t sort_tile) {
  if (threadIdx.x != 0) return;
  uint32_t tiles = 0;
  for (int s = 0; s < n_seg; ++s) {
    const uint32_t c = fd->seg_n[s] ? fd->seg_chunk_start[s + 1] - fd->seg_chunk_start[s] : 0u;
    fd->seg_C[s] = c;
    fd->sort_tile_start[s] = tiles;
    tiles += (c + sort_tile - 1) / sort_tile;
  }
  fd->sort_tile_start[n_seg] = tiles;
}

// ============================================================== K3: radix sort
constexpr int RADIX_BITS = 8;
constexpr int RADIX_BINS = 256;
constexpr int SORT_THREADS = 256;
constexpr int SORT_WARPS = SORT_THREADS / 32;
#ifndef CRSH_SORT_ITEMS
#define CRSH_SORT_ITEMS 16
#endif
constexpr int SORT_ITEMS = CRSH_SORT_ITEMS;   // 4096-key tiles: half the tiles (and look-back hops) of 2048 (A/B: sort 0.47 -> 0.44 ms at cfg4)
constexpr int SORT_TILE = SORT_THREADS * SORT_ITEMS;
constexpr int SORT_PASSES = 32 / RADIX_BITS;
// k_onesweep at 3 CTAs per SM (80 registers, no spills; 141 registers and 2
// CTAs per SM without the bound): A/B at cfg4 sort 0.44 -> 0.41 ms; 4 CTAs
// (64 registers) spill and are slower, as are 16/32-word look-back batches
#ifndef CRSH_SORT_MATCH
#define CRSH_SORT_MATCH 0   // 1: rank with __match_any_sync (round 1); 0: ballot-based peer masks
#endif
#ifndef CRSH_SORT_MINB
#define CRSH_SORT_MINB 3
#endif

struct SegChunks {   // per-segment chunk ranges, loaded from the FrameDesc
  int32_t n_seg;
  uint32_t start[MAX_SEG + 1];     // global chunk index of each segment's first chunk
  uint32_t count[MAX_SEG];
  uint32_t tile_start[MAX_SEG + 1];
  __device__ void load(const FrameDesc* fd, int ns) {
    n_seg = ns;
#pragma unroll
    for (int s = 0; s <= MAX_SEG; ++s) {
      start[s] = s <= ns ? fd->seg_chunk_start[s] : 0xFFFFFFFFu;
      tile_start[s] = s <= ns ? fd->sort_tile_start[s] : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int s = 0; s < MAX_SEG; ++s) count[s] = s < ns ? fd->seg_C[s] : 0u;
  }
};

// Segment lookups over register arrays: loops unrolled to MAX_SEG with a
// bound check and selects instead of a runtime index, so the per-segment
// arrays stay in registers (a runtime-indexed array lives in local memory).
__device__ __forceinline__ int seg_of(const uint32_t* starts, int n, uint32_t i) {
  int s = 0;
#pragma unroll
  for (int q = 1; q < MAX_SEG; ++q) s = (q < n && i >= starts[q]) ? q : s;
  return s;
}
__device__ __forceinline__ uint32_t seg_sel(const uint32_t* arr, int s) {
  uint32_t r = arr[0];
#pragma unroll
  for (int q = 1; q <= MAX_SEG; ++q) r = (q == s) ? arr[q] : r;
  return r;
}

// Per-segment digit histograms of all passes in one read of the keys.
__global__ void __launch_bounds__(256) k_radix_hist(const FrameDesc* fd, int n_seg, const uint32_t* __restrict__ keys,
                                                    uint32_t* __restrict__ hist /*[3][4][256]*/) {
  __shared__ uint32_t h[MAX_SEG * SORT_PASSES * RADIX_BINS];
  SegChunks sc;
  sc.load(fd, n_seg);
  const uint32_t C = fd->C;
  for (int i = threadIdx.x; i < MAX_SEG * SORT_PASSES * RADIX_BINS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < C; i += gridDim.x * blockDim.x) {
    const uint32_t k = __ldg(keys + i);
    const int s = seg_of(sc.start, sc.n_seg, i);
#pragma unroll
    for (int p = 0; p < SORT_PASSES; ++p) atomicAdd(&h[(s * SORT_PASSES + p) * RADIX_BINS + ((k >> (8 * p)) & 255u)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < MAX_SEG * SORT_PASSES * RADIX_BINS; i += blockDim.x)
    if (h[i]) atomicAdd(hist + i, h[i]);
}

struct SortPassArgs {
  const FrameDesc* fd;
  int32_t n_seg;
  int32_t pass;
  const uint32_t* keys_in;
  const uint32_t* vals_in;   // nullptr on the first pass: values = global chunk index
  uint32_t* keys_out;
  uint32_t* vals_out;
  const uint32_t* hist;      // [3][4][256]
  uint32_t* status;          // [tiles][256]: bits 31..30 flag, 29..0 count
  uint32_t* ticket;
};

__device__ __forceinline__ uint32_t st_load32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_store32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// One digit pass over all segments: stable local ranking with warp
// match.any, per-warp shared-memory histograms, decoupled look-back per digit
// across the segment's tiles, and a shared-memory reorder so the global
// writes are contiguous within each digit run.
__global__ void __launch_bounds__(SORT_THREADS, CRSH_SORT_MINB) k_onesweep(const SortPassArgs a) {
  extern __shared__ uint32_t sm[];
  uint32_t* s_keys = sm;                            // SORT_TILE
  uint32_t* s_vals = sm + SORT_TILE;                // SORT_TILE
  uint32_t* s_whist = sm + 2 * SORT_TILE;           // SORT_WARPS * 256
  __shared__ uint32_t s_bin_excl[RADIX_BINS], s_base[RADIX_BINS], s_warp[8];
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1u);
  for (int i = threadIdx.x; i < SORT_WARPS * RADIX_BINS; i += SORT_THREADS) s_whist[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  SegChunks sc;
  sc.load(a.fd, a.n_seg);
  if (tile >= seg_sel(sc.tile_start, sc.n_seg)) return;   // surplus block
  const int seg = seg_of(sc.tile_start, sc.n_seg, tile);
  const uint32_t t_local = tile - seg_sel(sc.tile_start, seg);
  uint32_t n = sc.count[0];
#pragma unroll
  for (int q = 1; q < MAX_SEG; ++q) n = (q == seg) ? sc.count[q] : n;
  const uint32_t seg0 = seg_sel(sc.start, seg);
  const int shift = RADIX_BITS * a.pass;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, lt = lanemask_lt();

  uint32_t k[SORT_ITEMS], v[SORT_ITEMS], rank[SORT_ITEMS];
  const uint32_t wbase = t_local * SORT_TILE + warp * (32 * SORT_ITEMS);
#pragma unroll
  for (int it = 0; it < SORT_ITEMS; ++it) {
    const uint32_t idx = wbase + it * 32 + lane;
    const bool ok = idx < n;
    k[it] = ok ? __ldg(a.keys_in + seg0 + idx) : 0xFFFFFFFFu;
    v[it] = ok ? (a.vals_in ? __ldg(a.vals_in + seg0 + idx) : seg0 + idx) : 0u;
  }
#pragma unroll
  for (int it = 0; it < SORT_ITEMS; ++it) {
    const uint32_t idx = wbase + it * 32 + lane;
    const bool ok = idx < n;
#if CRSH_SORT_MATCH
    const uint32_t d = ok ? ((k[it] >> shift) & 255u) : 0x100u + lane;   // invalid lanes never match
    const uint32_t peers = __match_any_sync(CRSH_FULL, d);
#else
    // lanes with the same digit from RADIX_BITS ballots (short-latency votes;
    // MATCH.ANY's latency was the stall of the ranking loop, ncu r2: sort at
    // cfg4 0.409 -> 0.359 ms, cfg2 59.4 -> 56.0 us); invalid lanes (tile
    // tail) are masked out of every valid lane's peers
    const uint32_t d = (k[it] >> shift) & 255u;
    uint32_t peers = __ballot_sync(CRSH_FULL, ok);
#pragma unroll
    for (int bit = 0; bit < RADIX_BITS; ++bit) {
      const bool on = (d >> bit) & 1u;
      const uint32_t bb = __ballot_sync(CRSH_FULL, on);
      peers &= on ? bb : ~bb;
    }
#endif
    const uint32_t leader = __ffs(peers) - 1;
    uint32_t base = 0;
    if (ok && lane == leader) {
      base = s_whist[warp * RADIX_BINS + d];
      s_whist[warp * RADIX_BINS + d] = base + __popc(peers);
    }
    base = __shfl_sync(CRSH_FULL, base, leader);
    rank[it] = base + __popc(peers & lt);
    __syncwarp();
  }
  __syncthreads();
  // per-bin tile count, and per-warp exclusive offsets within the bin
  const uint32_t b = threadIdx.x;
  uint32_t cnt = 0;
#pragma unroll
  for (int w = 0; w < SORT_WARPS; ++w) {
    const uint32_t c = s_whist[w * RADIX_BINS + b];
    s_whist[w * RADIX_BINS + b] = cnt;
    cnt += c;
  }
  // decoupled look-back over the tiles of this segment, one bin per thread
  uint32_t* st = a.status + (size_t)tile * RADIX_BINS + b;
  uint32_t excl = 0;
  if (t_local == 0) {
    st_store32(st, (2u << 30) | cnt);
  } else {
    st_store32(st, (1u << 30) | cnt);
    // batched look-back: 8 predecessors' words are requested at once, so a
    // one-wave sort (every tile looking back at aggregates) costs ~1/8 of the
    // round trips of a one-by-one walk; the segment's first tile is inclusive
    const int first = (int)seg_sel(sc.tile_start, seg);
    int p = (int)tile - 1;
    bool done = false;
    while (!done) {
      uint32_t w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = (p - i >= first) ? st_load32(a.status + (size_t)(p - i) * RADIX_BINS + b) : 0u;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (done || p - i < first) continue;
        while ((w[i] >> 30) == 0u) w[i] = st_load32(a.status + (size_t)(p - i) * RADIX_BINS + b);
        excl += w[i] & 0x3FFFFFFFu;
        done = (w[i] >> 30) == 2u;
      }
      p -= 8;
    }
    st_store32(st, (2u << 30) | (excl + cnt));
  }
  // digit base of the segment (exclusive scan of its global histogram)
  const uint32_t hcount = __ldg(a.hist + ((size_t)seg * SORT_PASSES + a.pass) * RADIX_BINS + b);
  const uint32_t hexcl = block_excl_scan_256(hcount, s_warp, nullptr);
  const uint32_t texcl = block_excl_scan_256(cnt, s_warp, nullptr);
  s_base[b] = hexcl + excl;
  s_bin_excl[b] = texcl;
  __syncthreads();
#pragma unroll
  for (int it = 0; it < SORT_ITEMS; ++it) {
    const uint32_t idx = wbase + it * 32 + lane;
    if (idx < n) {
      const uint32_t d = (k[it] >> shift) & 255u;
      const uint32_t pos = s_bin_excl[d] + s_whist[warp * RADIX_BINS + d] + rank[it];
      CRSH_CHECK(pos < (uint32_t)SORT_TILE, 302);
      s_keys[pos] = k[it];
      s_vals[pos] = v[it];
    }
  }
  __syncthreads();
  const uint32_t t_n = min((uint32_t)SORT_TILE, n - t_local * SORT_TILE);
  for (uint32_t j = threadIdx.x; j < t_n; j += SORT_THREADS) {
    const uint32_t key = s_keys[j];
    const uint32_t d = (key >> shift) & 255u;
    const uint32_t out = seg0 + s_base[d] + (j - s_bin_excl[d]);
    CRSH_CHECK(out < seg0 + n && j >= s_bin_excl[d], 301);
    a.keys_out[out] = key;
    a.vals_out[out] = s_vals[j];
  }
}

// ============================================================== K4: decompression
constexpr int EXP_TILE = 2048;

struct ScanSizeArgs {
  const FrameDesc* fd;                // C, N
  const uint32_t* sorted_cidx;   // chunk index of each sorted chunk
  const uint32_t* cbase;         // [C + 1]
  uint32_t* pos;                 // out [C + 1]: exclusive scan of the skeleton
  uint32_t* first_chunk;         // out [ceil(N / EXP_TILE)]
  unsigned long long* status;
  uint32_t* ticket;
};

// The skeleton array (sorted chunk sizes) and its exclusive scan.
template <int SS_ITEMS>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_sizes(const ScanSizeArgs a) {
  constexpr int NE = SS_ITEMS * 8;
  constexpr uint32_t TILE = (uint32_t)SCAN_THREADS * SS_ITEMS;
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ uint32_t s_cnt[NE], s_excl[NE];
  if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t C = a.fd->C, N = a.fd->N;
  const uint32_t n_tiles = (C + TILE - 1) / TILE;
  if (tile >= n_tiles) return;   // surplus block
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t size[SS_ITEMS], wex[SS_ITEMS];
#pragma unroll
  for (int it = 0; it < SS_ITEMS; ++it) {
    const uint32_t c = tile * TILE + it * SCAN_THREADS + threadIdx.x;
    uint32_t sz = 0;
    if (c < C) {
      const uint32_t ci = __ldg(a.sorted_cidx + c);
      sz = __ldg(a.cbase + ci + 1) - __ldg(a.cbase + ci);
    }
    uint32_t incl = sz;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(CRSH_FULL, incl, o);
      if ((int)lane >= o) incl += y;
    }
    size[it] = sz;
    wex[it] = incl - sz;
    if (lane == 31) s_cnt[it * 8 + warp] = incl;
  }
  __syncthreads();
  tile_scan_lookback_block<NE>(s_cnt, s_excl, &s_prefix, a.status, (int)tile);
  __syncthreads();
  const uint32_t prefix = s_prefix;
#pragma unroll
  for (int it = 0; it < SS_ITEMS; ++it) {
    const uint32_t c = tile * TILE + it * SCAN_THREADS + threadIdx.x;
    if (c < C) {
      const uint32_t p = prefix + s_excl[it * 8 + warp] + wex[it];
      a.pos[c] = p;
      // the chunk covering each output tile start k*EXP_TILE in [p, p + size)
      for (uint32_t kk = (p + EXP_TILE - 1) / EXP_TILE; kk * EXP_TILE < p + size[it]; ++kk) a.first_chunk[kk] = c;
    }
  }
  if (tile == n_tiles - 1 && threadIdx.x == 0) a.pos[C] = N;
}

struct ExpandArgs {
  const FrameDesc* fd;      // N, C, seg_comp_start, seg_pad_base
  const uint32_t* pos;
  const uint32_t* first_chunk;
  const uint32_t* skey;
  const uint32_t* scidx;
  const uint32_t* cbase;
  const uint32_t* vals_c;
  int32_t n_seg;
  uint32_t* sorted_key;     // padded layout
  uint32_t* sorted_slot;
};

// Fill: every output position finds its chunk by a binary search over
// the tile's slice of the scan (load-balanced: long runs are split across
// tiles), then gathers the slot id of the run element.
__global__ void __launch_bounds__(256) k_expand(const ExpandArgs a) {
  __shared__ uint32_t s_pos[EXP_TILE + 2];
  const uint32_t N = a.fd->N, C = a.fd->C;
  const uint32_t nb = (N + EXP_TILE - 1) / EXP_TILE;
  if (blockIdx.x >= nb) return;   // surplus block
  uint32_t segc[MAX_SEG + 1], segp[MAX_SEG + 1];
#pragma unroll
  for (int s = 0; s <= MAX_SEG; ++s) {
    segc[s] = s <= a.n_seg ? a.fd->seg_comp_start[s] : 0xFFFFFFFFu;
    segp[s] = s <= a.n_seg ? a.fd->seg_pad_base[s] : 0xFFFFFFFFu;
  }
  const uint32_t o0 = blockIdx.x * EXP_TILE;
  const uint32_t o1 = min(o0 + EXP_TILE, N);
  const uint32_t c_lo = __ldg(a.first_chunk + blockIdx.x);
  const uint32_t c_hi = (blockIdx.x + 1 < nb) ? __ldg(a.first_chunk + blockIdx.x + 1) : C - 1;
  const uint32_t nc = c_hi - c_lo + 1;
  for (uint32_t j = threadIdx.x; j <= nc; j += blockDim.x) s_pos[j] = __ldg(a.pos + c_lo + j);
  __syncthreads();
  for (uint32_t o = o0 + threadIdx.x; o < o1; o += blockDim.x) {
    uint32_t lo = 0, hi = nc;   // largest j in [0, nc) with s_pos[j] <= o
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_pos[mid] <= o) lo = mid; else hi = mid;
    }
    const uint32_t c = c_lo + lo;
    const uint32_t src = __ldg(a.cbase + __ldg(a.scidx + c)) + (o - s_pos[lo]);
    const int s = seg_of(segc, a.n_seg, o);
    const uint32_t dst = seg_sel(segp, s) + (o - seg_sel(segc, s));
    CRSH_CHECK(dst < a.fd->Np && src < N && c < C, 401);
    a.sorted_key[dst] = __ldg(a.skey + c);
    a.sorted_slot[dst] = __ldg(a.vals_c + src);
  }
}

// RAH (CRSH_F_SORT off): rays stay in generation order.
__global__ void k_copy_unsorted(const ExpandArgs a) {
  const uint32_t N = a.fd->N;
  uint32_t segc[MAX_SEG + 1], segp[MAX_SEG + 1];
#pragma unroll
  for (int s = 0; s <= MAX_SEG; ++s) {
    segc[s] = s <= a.n_seg ? a.fd->seg_comp_start[s] : 0xFFFFFFFFu;
    segp[s] = s <= a.n_seg ? a.fd->seg_pad_base[s] : 0xFFFFFFFFu;
  }
  for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < N; o += gridDim.x * blockDim.x) {
    const int s = seg_of(segc, a.n_seg, o);
    const uint32_t dst = seg_sel(segp, s) + (o - seg_sel(segc, s));
    a.sorted_key[dst] = __ldg(a.skey + o);
    a.sorted_slot[dst] = __ldg(a.vals_c + o);
  }
}

}  // namespace crsh
