// k_traverse.cuh — top-down traversal of the ray-space hierarchy (P:169-187,
// §3.3.7-3.3.8):
//   K7  k_mesh_cull  Eq 9 of every top node against every mesh sphere
//                    (whole-mesh culling at the top level);
//                    one bit per (top node, mesh).
//   K7b k_plan       per group of K consecutive top nodes: triangles of the
//                    meshes any of them kept, cut into work items.
//   K8  k_traverse   persistent CTAs over the work items. Per item: the
//                    surviving meshes' triangles are streamed in tiles of
//                    bounding spheres through shared memory; the dense
//                    (top node x triangle) Eq 9 tests run from registers and
//                    shared memory; survivors go to a per-level shared-memory
//                    queue (warp-aggregated appends) and are expanded level by
//                    level down to the bundles ("triangles rejected at
//                    the top levels will not be tested again"); each surviving
//                    (bundle, triangle) pair runs Moller-Trumbore against the
//                    bundle's rays, and the closest hit is kept by a
//                    64-bit atomicMin on (float_bits(t) << 32 | tri) -- in
//                    shared memory when the group's rays fit, then global.
//   K9  k_unpack     per sorted ray -> per-slot (hit_tri, t) or packed u64.
// Counters follow the paper's convention: a test is
// counted per (node, triangle) pair actually tested; misses + hits = tests.
#pragma once
#include "common.cuh"
#include "numspec.cuh"

namespace crsh {

// counters layout (uint64): per segment CTR_STRIDE words
constexpr int CTR_TESTS = 0;         // + level (1..8)
constexpr int CTR_HITS = 9;          // + level
constexpr int CTR_MESH_TESTS = 18;
constexpr int CTR_MESH_HITS = 19;
constexpr int CTR_FINAL_TESTS = 20;
constexpr int CTR_FINAL_HITS = 21;
constexpr int CTR_RAYS_HIT = 22;
constexpr int CTR_CL_TESTS = 23;     // object sphere-tree (CRSH_F_OBJTREE): node vs cluster sphere
constexpr int CTR_CL_HITS = 24;
constexpr int CTR_CH_SKIP = 25;      // counted Eq 9 tests K8 did not evaluate (prefilter, cull_pf)
constexpr int CTR_PF_TESTS = 26;     // child-prefilter tests evaluated
constexpr int CTR_STRIDE = 32;
constexpr uint32_t CLUSTER_TRIS = 32;   // triangles per object-tree cluster (reading O1): one warp slice

constexpr unsigned long long BEST_NONE = 0xFFFFFFFFFFFFFFFFull;
constexpr unsigned long long PACK_MISS = 0x7F800000FFFFFFFFull;
constexpr unsigned long long PACK_EMPTY = 0x7FFFFFFFFFFFFFFFull;

__device__ __forceinline__ unsigned long long pack_hit(float t, uint32_t tri) {
  return ((unsigned long long)__float_as_uint(t) << 32) | tri;
}

// ============================================================== K7
// Eq 9 of every top node against every mesh sphere, over ALL groups (every
// rank runs this cheap pre-pass on the whole frame: the work-balanced cut
// below needs the work of every group); the mesh tests/hits of
// this rank's groups are counted in k_plan.
struct CullArgs {
  const FrameDesc* fd;         // G
  int32_t K;
  int32_t W;                   // mask words per node = ceil(n_meshes / 32)
  const float4* trav_top;      // level Lv, traversal layout
  int32_t n_meshes;
  const float4* mesh_sph;
  const uint32_t* mesh_count;
  int32_t cull_on;
  uint32_t* masks;             // [n_top_padded][W]
};

__global__ void __launch_bounds__(256) k_mesh_cull(const CullArgs a) {
  const uint32_t n_top = a.fd->G * (uint32_t)a.K;
  const uint64_t gid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (gid >= (uint64_t)n_top * a.W) return;
  const uint32_t n = (uint32_t)(gid / a.W);
  const int w = (int)(gid % a.W);
  const float4 p0 = __ldg(a.trav_top + 3 * (size_t)n), p1 = __ldg(a.trav_top + 3 * (size_t)n + 1),
               p2 = __ldg(a.trav_top + 3 * (size_t)n + 2);
  uint32_t bits = 0;
  if (p0.w >= 0.0f) {   // existing node
    const f3 C = mk3(p0.x, p0.y, p0.z), A = mk3(p1.x, p1.y, p1.z);
    for (int b = 0; b < 32; ++b) {
      const int m = w * 32 + b;
      if (m >= a.n_meshes) break;
      if (__ldg(a.mesh_count + m) == 0) continue;
      if (!a.cull_on || cull_ns(C, p0.w, A, p1.w, p2.x, __ldg(a.mesh_sph + m))) bits |= 1u << b;
    }
  }
  a.masks[(size_t)n * a.W + w] = bits;
}

// ============================================================== K7a
// Work-balanced sharding: the work of group g is its number of
// top-level tests, sum over its K top nodes of the triangles of the meshes
// the node kept; rank r takes the contiguous groups whose work prefix falls
// in [total r / world, total (r+1) / world). Every rank derives the same cut
// from the same data, so the ranks partition the groups with no exchange.
struct WorkArgs {
  const FrameDesc* fd;
  int32_t K, W, n_meshes;
  const uint32_t* masks;
  const uint32_t* mesh_count;
  const float4* trav_top;      // node existence (radius >= 0)
  int32_t cull_on, n_nonempty;
  int32_t objtree;             // CRSH_F_OBJTREE or K8-PF: a mesh's triangles count in whole clusters (slices)
  unsigned long long* work;    // [G] top-level tests of the group (the cut's work)
  uint4* gstat;                // [G] {triangles of the meshes any node kept, mesh tests, mesh passes, 0}
};

// one warp per group, lane j = top node j (K <= 32): the per-node masks are
// combined with warp votes/reductions, so no thread walks a group serially
__global__ void __launch_bounds__(256) k_group_work(const WorkArgs a) {
  const uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = lane_id();
  if (g >= a.fd->G) return;   // warp-uniform
  const bool in = (int)lane < a.K;
  unsigned long long work = 0;
  uint32_t T = 0, mh = 0;
  for (int w = 0; w < a.W; ++w) {
    const uint32_t mj = in ? __ldg(a.masks + ((size_t)g * a.K + lane) * a.W + w) : 0u;
    mh += __popc(mj);
    const uint32_t u = __reduce_or_sync(CRSH_FULL, mj);   // meshes any node kept
    uint32_t nb = 0;                                     // lane b: nodes that kept mesh w*32+b
#pragma unroll 4
    for (int b = 0; b < 32; ++b) {
      const uint32_t c = __popc(__ballot_sync(CRSH_FULL, (mj >> b) & 1u));
      nb = ((int)lane == b) ? c : nb;
    }
    const int m = w * 32 + (int)lane;
    const uint32_t real = (m < a.n_meshes) ? __ldg(a.mesh_count + m) : 0u;
    // cluster-aligned virtual range (items); the cut's work stays the
    // group's top-level test count (real triangles only)
    const uint32_t cnt = a.objtree ? (real + CLUSTER_TRIS - 1) / CLUSTER_TRIS * CLUSTER_TRIS : real;
    T += ((u >> lane) & 1u) ? cnt : 0u;
    work += (unsigned long long)nb * real;
  }
  const uint32_t ex = (in && __ldg(&a.trav_top[3 * ((size_t)g * a.K + lane)].w) >= 0.0f) ? 1u : 0u;
  T = __reduce_add_sync(CRSH_FULL, T);
  mh = __reduce_add_sync(CRSH_FULL, mh);
  const uint32_t n_ex = __reduce_add_sync(CRSH_FULL, ex);
  // 64-bit work: two 32-bit halves reduced separately
  const uint32_t lo = __reduce_add_sync(CRSH_FULL, (uint32_t)(work & 0xFFFFu)),
                 hi = __reduce_add_sync(CRSH_FULL, (uint32_t)(work >> 16));
  if (lane == 0) {
    a.work[g] = ((unsigned long long)hi << 16) + lo;
    a.gstat[g] = make_uint4(T, a.cull_on ? n_ex * (uint32_t)a.n_nonempty : 0u, a.cull_on ? mh : 0u, 0u);
  }
}

constexpr int CUT_THREADS = 1024;
// one CTA: prefix of the group work, cut points of ranks rank and rank+1
__global__ void __launch_bounds__(CUT_THREADS) k_cut(FrameDesc* fd, const unsigned long long* work, int rank, int world) {
  const uint32_t G = fd->G;
  if (world <= 1) {
    if (threadIdx.x == 0) { fd->g_lo = 0u; fd->g_hi = G; }
    return;
  }
  __shared__ unsigned long long s_sum[CUT_THREADS];
  __shared__ uint32_t s_cut[2];
  const uint32_t per = (G + CUT_THREADS - 1) / CUT_THREADS;
  const uint32_t lo = min(G, threadIdx.x * per), hi = min(G, lo + per);
  unsigned long long t = 0;
  for (uint32_t g = lo; g < hi; ++g) t += work[g];
  s_sum[threadIdx.x] = t;
  if (threadIdx.x < 2) s_cut[threadIdx.x] = (rank + (int)threadIdx.x >= world) ? G : 0u;
  __syncthreads();
  for (int o = 1; o < CUT_THREADS; o <<= 1) {   // inclusive scan (Hillis-Steele)
    const unsigned long long y = threadIdx.x >= (unsigned)o ? s_sum[threadIdx.x - o] : 0ull;
    __syncthreads();
    s_sum[threadIdx.x] += y;
    __syncthreads();
  }
  const unsigned long long total = s_sum[CUT_THREADS - 1];
  unsigned long long pre = threadIdx.x ? s_sum[threadIdx.x - 1] : 0ull;   // work before group lo
  // cut(q) = min{g : P(g) >= ceil(total q / world)}, P(g) = work of groups
  // [0, g); cut(0) = 0, cut(world) = G. The group that crosses the boundary
  // (P(g) < target <= P(g + 1)) is owned by exactly one thread's range.
  for (int c = 0; c < 2; ++c) {
    const int qr = rank + c;
    if (qr <= 0 || qr >= world) continue;
    const unsigned long long target = (total * (unsigned long long)qr + (unsigned long long)world - 1) / (unsigned long long)world;
    unsigned long long p = pre;
    for (uint32_t g = lo; g < hi; ++g) {
      const unsigned long long w = work[g];
      if (p < target && p + w >= target) { s_cut[c] = g + 1; break; }
      p += w;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t c0 = s_cut[0], c1 = s_cut[1];
    if (total == 0ull) {   // no work anywhere: split by group count
      c0 = (uint32_t)((uint64_t)G * rank / world);
      c1 = (uint32_t)((uint64_t)G * (rank + 1) / world);
    }
    fd->g_lo = c0;
    fd->g_hi = max(c0, c1);
  }
}

// ============================================================== K7b
struct PlanArgs {
  FrameDesc* fd;               // g_lo, g_hi: this rank's group range; out: n_items
  uint32_t group_rays;
  int32_t n_seg;
  const uint4* gstat;          // k_group_work: {triangles, mesh tests, mesh passes, 0} per group
  unsigned long long* counters;
  uint32_t item_tris;
  uint32_t items_cap;          // capacity of items (checked builds)
  uint4* items;                // (group, v_begin, v_end, 0)
  unsigned long long* status;
  uint32_t* ticket;
};

__global__ void __launch_bounds__(SCAN_THREADS) k_plan(const PlanArgs a) {
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ uint32_t s_cnt[SCAN_ITEMS * 8], s_excl[SCAN_ITEMS * 8];
  if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t g_lo = a.fd->g_lo, g_hi = a.fd->g_hi;
  const uint32_t n_tiles = (g_hi - g_lo + SCAN_TILE - 1) / SCAN_TILE;
  if (tile >= n_tiles) {   // surplus block; the first one reports "no items" for an empty range
    if (tile == 0 && threadIdx.x == 0) a.fd->n_items = 0u;
    return;
  }
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  __shared__ unsigned long long s_mesh[MAX_SEG][2];
  if (threadIdx.x < MAX_SEG * 2) (&s_mesh[0][0])[threadIdx.x] = 0ull;
  uint32_t seg_group_start[MAX_SEG];   // registers: every loop below is unrolled to MAX_SEG
#pragma unroll
  for (int q = 0; q < MAX_SEG; ++q) seg_group_start[q] = q < a.n_seg ? a.fd->seg_pad_base[q] / a.group_rays : 0xFFFFFFFFu;
  __syncthreads();
  uint32_t ntri[SCAN_ITEMS], nit[SCAN_ITEMS], wex[SCAN_ITEMS];
  uint32_t mt[MAX_SEG] = {0u, 0u, 0u}, mh[MAX_SEG] = {0u, 0u, 0u};
#pragma unroll
  for (int it = 0; it < SCAN_ITEMS; ++it) {
    const uint32_t g = g_lo + tile * SCAN_TILE + it * SCAN_THREADS + threadIdx.x;
    uint32_t T = 0;
    if (g < g_hi) {
      const uint4 st = __ldg(a.gstat + g);   // whole-mesh tests / passes of the group's top nodes
      T = st.x;
      int sg = 0;
#pragma unroll
      for (int q = 1; q < MAX_SEG; ++q) sg = (g >= seg_group_start[q]) ? q : sg;
#pragma unroll
      for (int q = 0; q < MAX_SEG; ++q) {
        mt[q] += (sg == q) ? st.y : 0u;
        mh[q] += (sg == q) ? st.z : 0u;
      }
    }
    const uint32_t ni = (T + a.item_tris - 1) / a.item_tris;
    uint32_t incl = ni;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(CRSH_FULL, incl, o);
      if ((int)lane >= o) incl += y;
    }
    ntri[it] = T;
    nit[it] = ni;
    wex[it] = incl - ni;
    if (lane == 31) s_cnt[it * 8 + warp] = incl;
  }
#pragma unroll
  for (int q = 0; q < MAX_SEG; ++q) {
    if (q >= a.n_seg) break;
    warp_seg_add(&s_mesh[0][0], 2, a.n_seg, q, mt[q]);
    warp_seg_add(&s_mesh[0][1], 2, a.n_seg, q, mh[q]);
  }
  __syncthreads();
  tile_scan_lookback_block(s_cnt, s_excl, &s_prefix, a.status, (int)tile);
  __syncthreads();
  const uint32_t prefix = s_prefix;
#pragma unroll
  for (int it = 0; it < SCAN_ITEMS; ++it) {
    const uint32_t g = g_lo + tile * SCAN_TILE + it * SCAN_THREADS + threadIdx.x;
    const uint32_t off = prefix + s_excl[it * 8 + warp] + wex[it];
    for (uint32_t q = 0; q < nit[it]; ++q) {
      CRSH_CHECK(off + q < a.items_cap, 701);
      a.items[off + q] = make_uint4(g, q * a.item_tris, min(ntri[it], (q + 1) * a.item_tris), 0u);
    }
  }
  if (tile == n_tiles - 1 && threadIdx.x == 0) {
    uint32_t t = 0;
    for (int q = 0; q < SCAN_ITEMS * 8; ++q) t += s_cnt[q];
    a.fd->n_items = prefix + t;
  }
  if (threadIdx.x < MAX_SEG * 2) {
    const unsigned long long v = (&s_mesh[0][0])[threadIdx.x];
    if (v) atomicAdd(a.counters + (threadIdx.x / 2) * CTR_STRIDE + CTR_MESH_TESTS + (threadIdx.x & 1), v);
  }
}

// ============================================================== K8
// Warp-synchronous traversal. Each warp streams 32-triangle slices of the
// item's virtual triangle range; lane i owns triangle i of the slice.
//  * top level: K top nodes x 32 triangles (Eq 9), node data broadcast from
//    shared memory;
//  * level Lv-1: every (top node j, triangle) that passed is tested at once
//    against the B children of j (all lanes iterate the same j and child, so
//    the node reads are broadcasts; B = 8 is fully unrolled);
//  * child survivors go to the warp's queue; deeper levels (Lv >= 3) are
//    expanded by 32-lane steps, and each 32-lane step of the bundle level runs
//    Moller-Trumbore for B0 rays of 32/B0 (bundle, triangle) entries. A step
//    is taken from the LOWEST level that has a full step, so the queues stay
//    bounded and persist across slices; the rest is drained at the item end.
// No block barrier is executed inside the hot loop.
#ifndef CRSH_TRAV_THREADS
#define CRSH_TRAV_THREADS 256
#endif
constexpr int TRAV_THREADS = CRSH_TRAV_THREADS;
constexpr int TRAV_WARPS = TRAV_THREADS / 32;
constexpr uint32_t SMALL_GROUP_RAYS = 512;   // groups up to this size live in shared memory
constexpr int LOWQ = 64;                     // capacity of a warp queue below level Lv-1
// Consecutive work items per ticket: the items of a group are consecutive, so
// a chunk shares the group setup (rays, nodes, mesh list into shared memory)
// across its items; chunks cost load balance at the end of the kernel, so
// the chunk grows with the items per CTA: min(ITEM_CHUNK_MAX, n_items /
// (CTAs x ITEM_CHUNK_DIV)), at least 1 (A/B, fixed chunks of 1 / 2 / 4: cfg2
// R6 103.4 / 100.7 / 93.6 Mrays/s, 46 items per CTA; cfg3 R6 53.2 / - / 55.6;
// adaptive: cfg2 unchanged, cfg3 R6 53.2 -> 55.0, cfg3 Z-order 510 -> 550)
#ifndef CRSH_LDS32
#define CRSH_LDS32 1   // child records through 32-bit shared addresses (A/B cfg4 R6 18.78 -> 18.85)
#endif
#ifndef CRSH_TOP_UNIFORM
#define CRSH_TOP_UNIFORM 1   // top-level pair skips on a uniform mask, records through 32-bit shared addresses
#endif
#ifndef CRSH_SEL_BITS
#define CRSH_SEL_BITS 1   // Eq 9 pair decisions as mask bits (chained setp + one select per test)
#endif
#ifndef CRSH_DYN_SLICE
#define CRSH_DYN_SLICE 1   // plain instantiation: slices of an item handed out by a shared counter
#endif
#ifndef CRSH_OBJ_TWOPHASE
#define CRSH_OBJ_TWOPHASE 1   // object tree: cluster tests into a CTA list, then one passing cluster per claim
#endif
#ifndef CRSH_OBJ_LIST
#define CRSH_OBJ_LIST 512     // entries of that list (8 bytes each)
#endif
#ifndef CRSH_PF_NODES
#define CRSH_PF_NODES 1   // K8-PF: nodes without a child pair past the prefilter are not iterated
#endif
#ifndef CRSH_APPEND_BITS
#define CRSH_APPEND_BITS 1   // K8-PF: child survivors appended child by child (ballot ranks)
#endif
#ifndef CRSH_PF_BULK
#define CRSH_PF_BULK 1   // K8-PF: skipped nodes' child tests counted with one warp sum when the group is full
#endif
#ifndef CRSH_TRAV_PREFETCH
#define CRSH_TRAV_PREFETCH 0
#endif
#ifndef CRSH_ITEM_CHUNK_MAX
#define CRSH_ITEM_CHUNK_MAX 4
#endif
#ifndef CRSH_ITEM_CHUNK_DIV
#define CRSH_ITEM_CHUNK_DIV 64
#endif
// The group's rays as paired records (rays 2i, 2i+1; mt2_ns) in four planes
// of float4 (plane k = float4 #k of every record): record pp sits at index
// ray_rix(pp) = pp + pp / 8 of each plane. The skew of one slot per 8 records
// (two bundles of B0 = 8) puts the k-th load of 32 lanes at 8 different
// bundles on 8 different 16-byte bank groups, and the bundle's records are
// contiguous, so one base index per (bundle, triangle) entry addresses all
// its loads with compile-time offsets (RAY_PLANE is fixed for the largest
// shared-memory group). Replaces an XOR swizzle of 64-byte records (A/B:
// cfg2 R6 83.5 -> 89.1 Mrays/s, Z-order 497 -> 520: the swizzle's per-load
// address arithmetic and its remaining bank conflicts).
__host__ __device__ __forceinline__ constexpr uint32_t ray_rix(uint32_t pp) { return pp + (pp >> 3); }
constexpr uint32_t RAY_PLANE = ray_rix(SMALL_GROUP_RAYS / 2u) + 1u;   // float4 per ray plane (289)

struct TravArgs {
  int32_t Lv, B0, B, K, logB0, logB;
  uint32_t group_rays;
  const float4* trav[MAX_LEVELS + 1]; // level k (1..Lv), traversal layout
  uint32_t per_group[MAX_LEVELS + 1]; // nodes per group at level k
  const float4* sorted_rays;          // !SMALL groups: rays in sorted (padded) order
  const uint32_t* sorted_slot;        // SMALL groups: the group's rays are gathered by slot
  const float4* rays;                 //   from the generation order ([slots][2])
  const float4* tri_e;
  const float4* tri_sph;
  const uint32_t* masks;
  int32_t W, n_meshes;
  const uint32_t* mesh_first;
  const uint32_t* mesh_count;
  // CRSH_F_OBJTREE (null otherwise): triangle ids in cluster order, the
  // triangle spheres in that order, first cluster of each mesh, cluster spheres
  const int32_t* tri_order;
  const float4* tri_sph_ord;
  const uint32_t* mesh_cluster_first;
  const float4* cluster_sph;
  const float4* cluster_pf;           // PF: per cluster, a sphere containing its triangle spheres (k_cluster_pf)
  const uint4* items;
  uint32_t M;                         // triangles (checked builds)
  uint32_t obj_list_cap;              // object tree: entries of the cluster list used (<= CRSH_OBJ_LIST, >= CPB x warps)
  const FrameDesc* fd;                // n_items, seg_pad_base (group starts)
  uint32_t* ticket;
  unsigned long long* best;           // [Np]
  unsigned long long* counters;
  int32_t n_seg;
};

// dynamic shared-memory layout (bytes), shared by host and device
struct TravSmem {
  uint32_t off_top, off_tpairs, off_exm, off_act_nmask, off_act_prefix, off_act_first, off_act_cnt, off_act_cfirst, off_q,
      off_best, off_nodes, off_rays,
      off_pairs, node_off[MAX_LEVELS + 1], q_off[MAX_LEVELS + 1], q_warp, total;
  __host__ __device__ static TravSmem make(int K, int B, int n_meshes, int Lv, bool small, const uint32_t* per_group,
                                           uint32_t group_rays) {
    TravSmem s;
    uint32_t o = 0;
    auto take = [&](uint32_t bytes) { const uint32_t r = o; o += (bytes + 15u) & ~15u; return r; };
    s.off_top = take(K * 48u);
    s.off_tpairs = take(80u * ((K + 1) / 2));   // top nodes as paired records (cull2_ns); odd K: zero partner
    s.off_exm = take(4u * K);   // existing-children mask of each top node
    s.off_act_nmask = take(4u * n_meshes);
    s.off_act_prefix = take(4u * (n_meshes + 1));
    s.off_act_first = take(4u * n_meshes);
    s.off_act_cnt = take(4u * n_meshes);
    s.off_act_cfirst = take(4u * n_meshes);
    // per-warp queues of uint2 (node_local, triangle): Lv == 1: the top (=
    // bundle) level holds one slice (32 K) plus a partial step; Lv >= 2:
    // level Lv-1 receives the dense child tests of one top node (32 B) plus
    // a partial step; deeper levels LOWQ (they receive <= 32 per step)
    uint32_t qw = 0;
    for (int k = 0; k <= MAX_LEVELS; ++k) { s.q_off[k] = 0; s.node_off[k] = 0; }
    for (int k = 1; k <= Lv; ++k) {
      s.q_off[k] = qw;
      if (Lv == 1) qw += 32u * K + 32u;
      else if (k == Lv - 1) qw += 32u * B + 32u;
      else if (k < Lv - 1) qw += (uint32_t)LOWQ;
    }
    s.q_warp = qw;
    s.off_q = take(8u * qw * TRAV_WARPS);
    s.off_best = s.off_nodes = s.off_rays = s.off_pairs = 0;
    if (small) {
      uint32_t n4 = 0;   // float4 slots of the group's nodes below the top level
      for (int k = 1; k < Lv; ++k) { s.node_off[k] = n4; n4 += 3u * per_group[k]; }
      s.off_nodes = take(16u * (n4 ? n4 : 1u));
      s.off_rays = take(64u * RAY_PLANE);
      s.off_best = take(8u * group_rays);
      // level Lv-1 nodes as paired records for the packed child tests (cull2_ns)
      s.off_pairs = take(Lv >= 2 ? 80u * (per_group[Lv - 1] / 2u) : 16u);
    }
    s.total = o;
    return s;
  }
};

// Conservative child prefilter (NOT the paper's arithmetic, and not part of
// NUMSPEC: it only decides which Eq 9 evaluations can be skipped). Node
// n0 = {C, d}, n1 = {a, tan}, sc = sec; S = a sphere containing the slice's
// triangle spheres (k_cluster_pf). Eq 9 is monotone in the target sphere: if
// (P, R) passes, so does every (P', R') with |P - P'| + R <= R' (the halfspace
// term moves by at most the shift; the cone term by at most
// |u_perp| + |u_par| tan <= |u| sec, Cauchy-Schwarz). The test is evaluated
// with S's radius grown by 2^-12 of the magnitudes involved, ~200x the
// float32 decision error of either evaluation (a few ulps of |v|, d, R: the
// cone side is only near the boundary when rhs <= |w| <= |v|), so a false
// here implies false for every triangle of the slice in cull2_ns.
// Wide nodes (tan = sec = 1e30) always pass, as in Eq 9.
__device__ __forceinline__ bool cull_pf(float4 n0, float4 n1, float sc, float4 S) {
  const float vx = S.x - n0.x, vy = S.y - n0.y, vz = S.z - n0.z;
  const float mag = fabsf(vx) + fabsf(vy) + fabsf(vz) + fabsf(n0.w) + S.w;
  const float dr = n0.w + S.w + mag * 0x1p-12f;
  const float s = vx * n1.x + vy * n1.y + vz * n1.z;
  if (s < -dr) return false;
  const float wx = vx - s * n1.x, wy = vy - s * n1.y, wz = vz - s * n1.z;
  const float w2 = wx * wx + wy * wy + wz * wz;
  const float rhs = fmaxf(s, 0.0f) * n1.w + dr * sc;
  return w2 <= rhs * rhs;
}

// cull_pf for the two children of a paired child record (cull2_ns layout:
// {Cx0,Cx1,Cy0,Cy1} {Cz0,Cz1,d0,d1} {ax0,ax1,ay0,ay1} {az0,az1,tan0,tan1}
// {sec0,sec1,-,-}) in packed f32x2 arithmetic: the same bound and margin as
// cull_pf (the FMA forms only round less). Returns bit 0 / bit 1: child 0 / 1
// may pass.
__device__ __forceinline__ uint32_t cull2_pf_s(uint32_t rec, float4 S) {
  const float4 A = lds128(rec), Bv = lds128(rec + 16u), Cc = lds128(rec + 32u), D = lds128(rec + 48u),
               E = lds128(rec + 64u);
  const f2 vx = sub2(pk2(S.x, S.x), pk2(A.x, A.y)), vy = sub2(pk2(S.y, S.y), pk2(A.z, A.w)),
           vz = sub2(pk2(S.z, S.z), pk2(Bv.x, Bv.y));
  float x0, x1, y0, y1, z0, z1;
  up2(vx, x0, x1);
  up2(vy, y0, y1);
  up2(vz, z0, z1);
  const f2 mag = pk2(fabsf(x0) + fabsf(y0) + fabsf(z0) + fabsf(Bv.z) + S.w,
                     fabsf(x1) + fabsf(y1) + fabsf(z1) + fabsf(Bv.w) + S.w);
  const f2 dr = fma2(mag, pk2(0x1p-12f, 0x1p-12f), add2(pk2(Bv.z, Bv.w), pk2(S.w, S.w)));
  const f2 s = fma2(vx, pk2(Cc.x, Cc.y), fma2(vy, pk2(Cc.z, Cc.w), mul2(vz, pk2(D.x, D.y))));
  const f2 wx = fma2(s, pk2(-Cc.x, -Cc.y), vx), wy = fma2(s, pk2(-Cc.z, -Cc.w), vy), wz = fma2(s, pk2(-D.x, -D.y), vz);
  const f2 w2 = fma2(wx, wx, fma2(wy, wy, mul2(wz, wz)));
  float s0, s1;
  up2(s, s0, s1);
  const f2 rhs = fma2(pk2(fmaxf(s0, 0.0f), fmaxf(s1, 0.0f)), pk2(D.z, D.w), mul2(dr, pk2(E.x, E.y)));
  const f2 rr = mul2(rhs, rhs);
  float w0, w1, r0, r1, d0, d1;
  up2(w2, w0, w1);
  up2(rr, r0, r1);
  up2(dr, d0, d1);
  return ((s0 >= -d0) & (w0 <= r0) ? 1u : 0u) | ((s1 >= -d1) & (w1 <= r1) ? 2u : 0u);
}

// BT / B0T / LVT: compile-time branching factor / bundle size / levels (0 =
// runtime a.B / a.B0 / a.Lv); with LVT the length of the bundle-level queue
// Q[1] lives in a (warp-uniform) register instead of shared memory
// Occupancy: the compile-time Lv = 2 shape runs 4 CTAs (32 warps) per SM at
// 64 registers (A/B: +3.4 % at cfg2, +3.8 % at cfg3 over 3 CTAs at 80
// registers, despite ~100 bytes of spills); the runtime shapes keep 3.
#ifndef CRSH_TRAV_MINB
#define CRSH_TRAV_MINB 3
#endif
#ifndef CRSH_TRAV_MINB_LV2
#define CRSH_TRAV_MINB_LV2 4
#endif
// OBJ: the object sphere-tree path (CRSH_F_OBJTREE) as its own instantiation,
// so the plain path keeps its single slice loop (register allocation)
template <bool SMALL, int BT, int B0T, int LVT, bool OBJ, int PF = 0>
__global__ void __launch_bounds__(TRAV_THREADS, LVT == 2 ? CRSH_TRAV_MINB_LV2 : CRSH_TRAV_MINB)
    k_traverse(const TravArgs a, const TravSmem L) {
  extern __shared__ __align__(16) unsigned char smraw[];
  float4* s_top = reinterpret_cast<float4*>(smraw + L.off_top);
  uint32_t* s_act_nmask = reinterpret_cast<uint32_t*>(smraw + L.off_act_nmask);
  uint32_t* s_act_prefix = reinterpret_cast<uint32_t*>(smraw + L.off_act_prefix);
  uint32_t* s_act_first = reinterpret_cast<uint32_t*>(smraw + L.off_act_first);
  uint32_t* s_act_cnt = reinterpret_cast<uint32_t*>(smraw + L.off_act_cnt);
  uint32_t* s_act_cfirst = reinterpret_cast<uint32_t*>(smraw + L.off_act_cfirst);
  // cluster-aligned slices: the object tree, or the prefilter's clusters
  // (PF >= 1: the plain traversal over the same cluster order; PF = 1 child
  // prefilter, PF = 2 child and top-level prefilter)
  constexpr bool objtree = OBJ || PF > 0;
  const float4* tsph = objtree ? a.tri_sph_ord : a.tri_sph;
  unsigned long long* s_best = reinterpret_cast<unsigned long long*>(smraw + L.off_best);
  const float4* s_nodes = reinterpret_cast<const float4*>(smraw + L.off_nodes);
  const float4* s_rays = reinterpret_cast<const float4*>(smraw + L.off_rays);
  uint32_t* s_exm = reinterpret_cast<uint32_t*>(smraw + L.off_exm);
  float4* s_pairs = reinterpret_cast<float4*>(smraw + L.off_pairs);
  float4* s_tpairs = reinterpret_cast<float4*>(smraw + L.off_tpairs);
  const uint32_t pairs_s = (uint32_t)__cvta_generic_to_shared(s_pairs);   // 32-bit shared address (CRSH_LDS32)
  const uint32_t tpairs_s = (uint32_t)__cvta_generic_to_shared(s_tpairs);
  __shared__ uint32_t s_item, s_cur_g, s_n_act, s_carry, s_carry_c, s_blk;
  __shared__ uint32_t s_exm_full;   // every top node of the group has all B children
#if CRSH_OBJ_TWOPHASE
  __shared__ uint32_t s_lcnt, s_lclaim, s_lexh;          // object tree: cluster list fill / claim, blocks exhausted
  __shared__ uint2 s_list[OBJ ? CRSH_OBJ_LIST : 1];      // object tree: (cluster, node mask) of passing clusters
#endif
  __shared__ uint32_t s_warp[TRAV_WARPS];
  __shared__ unsigned long long s_ctr[MAX_SEG * CTR_STRIDE];
  __shared__ uint32_t s_qlen[TRAV_WARPS][MAX_LEVELS + 1];
  // per-level tables copied out of the kernel parameters: a runtime index into
  // a parameter array compiles to a select chain, into shared memory to one LDS
  __shared__ uint32_t s_qoff[MAX_LEVELS + 1], s_noff[MAX_LEVELS + 1], s_pg[MAX_LEVELS + 1];
  __shared__ const float4* s_trav[MAX_LEVELS + 1];
  if (threadIdx.x <= MAX_LEVELS) {
    s_qoff[threadIdx.x] = L.q_off[threadIdx.x];
    s_noff[threadIdx.x] = L.node_off[threadIdx.x];
    s_pg[threadIdx.x] = a.per_group[threadIdx.x];
    s_trav[threadIdx.x] = a.trav[threadIdx.x];
  }

  // K (top nodes per group, host: min(32, 512 / span)) is compile-time when the shape is
  constexpr int SPAN_T = (LVT && BT && B0T) ? B0T * (LVT >= 2 ? BT : 1) * (LVT >= 3 ? BT : 1) : 0;
  constexpr int KT = (LVT && LVT <= 3 && SPAN_T) ? (SPAN_T >= 512 ? 1 : (512 / SPAN_T < 32 ? 512 / SPAN_T : 32)) : 0;
  const int Lv = LVT ? LVT : a.Lv, K = KT ? KT : a.K, logB0 = a.logB0;
  const int B = BT ? BT : a.B;
  const int logB = BT ? __builtin_ctz(BT) : a.logB;
  const uint32_t Bm = (uint32_t)B - 1u;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
  const uint32_t lt = lanemask_lt();
  uint2* q = reinterpret_cast<uint2*>(smraw + L.off_q) + warp * L.q_warp;
  uint32_t* qlen = s_qlen[warp];
  constexpr bool QREG = LVT != 0;
  // queue capacity of level k per warp (TravSmem: levels packed in order, q_warp in all)
  auto qcap = [&](int k) -> uint32_t { return (k < Lv ? s_qoff[k + 1] : L.q_warp) - s_qoff[k]; };
  uint32_t q1n = 0;   // QREG: length of Q[1]
  auto qget = [&](int k) -> uint32_t { return (QREG && k == 1) ? q1n : qlen[k]; };
  auto qset = [&](int k, uint32_t v) {   // all 32 lanes, between __syncwarp()s
    if (QREG && k == 1) q1n = v;
    else if (lane == 0) qlen[k] = v;
  };
  const uint32_t step_exp = (32u >> logB) ? (32u >> logB) : 1u;   // entries per expansion step
  const uint32_t step_mt = 32u;                                   // entries per final-test step (one per lane)
  for (uint32_t i = tid; i < MAX_SEG * CTR_STRIDE; i += TRAV_THREADS) s_ctr[i] = 0ull;
  if (lane <= MAX_LEVELS) qlen[lane] = 0u;
  if (tid == 0) s_cur_g = 0xFFFFFFFFu;
  const uint32_t n_items = a.fd->n_items;
  // real rays of segment s end at seg_real_end[s]; registers (loops unrolled to MAX_SEG)
  uint32_t seg_group_start[MAX_SEG], seg_real_end[MAX_SEG];
#pragma unroll
  for (int q = 0; q < MAX_SEG; ++q) {
    seg_group_start[q] = q < a.n_seg ? a.fd->seg_pad_base[q] / a.group_rays : 0xFFFFFFFFu;
    seg_real_end[q] = q < a.n_seg ? a.fd->seg_pad_base[q] + a.fd->seg_n[q] : 0u;
  }

  const uint32_t chunk =
      max(1u, min((uint32_t)CRSH_ITEM_CHUNK_MAX, n_items / (gridDim.x * (uint32_t)CRSH_ITEM_CHUNK_DIV)));
  uint32_t ch_next = 0, ch_end = 0;   // CTA-uniform: the rest of the current ticket's chunk of items
  unsigned long long acc_tt = 0, acc_th = 0, acc_ct = 0, acc_ch = 0, acc_mt = 0, acc_mh = 0, acc_clt = 0, acc_clh = 0;
  int acc_seg = -1;
  auto flush_acc = [&]() {
    if (acc_seg >= 0 && lane == 0) {
      unsigned long long* c = s_ctr + acc_seg * CTR_STRIDE;
      // (PF reuses the cluster counters for its prefilter tests / skipped child tests)
      if (acc_clt) atomicAdd(&c[PF > 0 ? CTR_PF_TESTS : CTR_CL_TESTS], acc_clt);
      if (acc_clh) atomicAdd(&c[PF > 0 ? CTR_CH_SKIP : CTR_CL_HITS], acc_clh);
      if (acc_tt) atomicAdd(&c[CTR_TESTS + Lv], acc_tt);
      if (acc_th) atomicAdd(&c[CTR_HITS + Lv], acc_th);
      if (Lv >= 2 && acc_ct) atomicAdd(&c[CTR_TESTS + Lv - 1], acc_ct);
      if (Lv >= 2 && acc_ch) atomicAdd(&c[CTR_HITS + Lv - 1], acc_ch);
      if (acc_mt) atomicAdd(&c[CTR_FINAL_TESTS], acc_mt);
      if (acc_mh) atomicAdd(&c[CTR_FINAL_HITS], acc_mh);
    }
    acc_tt = acc_th = acc_ct = acc_ch = acc_mt = acc_mh = acc_clt = acc_clh = 0;
  };
  // Block barriers sit at chunk boundaries (the ticket) and group changes
  // (shared group data, the group's smem closest hits) only; consecutive items
  // of one group run back to back per warp (queues are warp-private). The
  // object-tree instantiation keeps a barrier per item (its per-item block
  // counter). The group's s_best is flushed to global at the group change.
  uint32_t cur_g = 0xFFFFFFFFu, n_act = 0;   // CTA-uniform copies of the current group
  auto group_end = [&]() {   // all warps: the current group's closest hits to global
    __syncthreads();
    if (SMALL && cur_g != 0xFFFFFFFFu) {
      const size_t rb = (size_t)cur_g * a.group_rays;
      for (uint32_t r = tid; r < a.group_rays; r += TRAV_THREADS) {
        const unsigned long long b = s_best[r];
        if (b != BEST_NONE) atomicMin(a.best + rb + r, b);
      }
    }
    __syncthreads();
  };
  // per-item barrier and slice counter: the object-tree instantiation (its
  // cluster blocks) and, with CRSH_DYN_SLICE, the plain one (its slices)
  constexpr bool PER_ITEM = OBJ || CRSH_DYN_SLICE;
  for (;;) {
    if (PER_ITEM || ch_next >= ch_end) {
      __syncthreads();
      if (ch_next >= ch_end && tid == 0) s_item = atomicAdd(a.ticket, 1u) * chunk;
      __syncthreads();
      if (ch_next >= ch_end) {
        ch_next = s_item;
        ch_end = min(ch_next + chunk, n_items);
      }
    }
    const uint32_t it = ch_next++;
    if (it >= n_items) break;
    const uint4 item = __ldg(a.items + it);
    const uint32_t g = item.x;
    int seg = 0;
#pragma unroll
    for (int qq = 1; qq < MAX_SEG; ++qq) seg = (g >= seg_group_start[qq]) ? qq : seg;
    unsigned long long* ctr = s_ctr + seg * CTR_STRIDE;
    if (seg != acc_seg) {   // uniform: the warp's running counters belong to one segment
      flush_acc();
      acc_seg = seg;
    }
    // rays [0, g_real) of the group are real, the rest padding (segments are
    // padded at their end): ray validity without loading the ray
    uint32_t g_real = 0;
    {
      uint32_t se = 0;
#pragma unroll
      for (int qq = 0; qq < MAX_SEG; ++qq) se = (qq == seg) ? seg_real_end[qq] : se;
      const uint32_t g0 = g * a.group_rays;
      g_real = se > g0 ? min(se - g0, a.group_rays) : 0u;
    }

    const bool new_group = g != cur_g;   // uniform
    if (new_group) {   // group setup (top nodes, surviving meshes, group data)
      group_end();     // every warp is done with the previous group
      for (int j = tid; j < 3 * K; j += TRAV_THREADS) s_top[j] = __ldg(s_trav[Lv] + (size_t)g * K * 3 + j);
      if (SMALL) {
        float4* sn = reinterpret_cast<float4*>(smraw + L.off_nodes);
        for (int k = 1; k < Lv; ++k) {
          const uint32_t n4 = 3u * s_pg[k];
          const float4* src = s_trav[k] + (size_t)g * n4;
          for (uint32_t j = tid; j < n4; j += TRAV_THREADS) sn[s_noff[k] + j] = __ldg(src + j);
        }
        // the group's rays as paired records (rays 2i, 2i+1) for mt2_ns, in
        // ray planes (ray_rix above), gathered from the generation order by
        // the sort permutation (K5 does not write a sorted copy for these
        // groups); padding rays (past the group's real rays) are tmin = tmax = -1
        float4* sr = reinterpret_cast<float4*>(smraw + L.off_rays);
        const uint32_t* ss = a.sorted_slot + (size_t)g * a.group_rays;
        for (uint32_t pp = tid; pp < a.group_rays / 2u; pp += TRAV_THREADS) {
          float4 a0 = make_float4(0.f, 0.f, 0.f, -1.0f), a1 = make_float4(0.f, 0.f, 1.f, -1.0f), b0 = a0, b1 = a1;
          const uint32_t r = 2u * pp;
          const uint32_t sl0 = r < g_real ? __ldg(ss + r) : 0u, sl1 = r + 1u < g_real ? __ldg(ss + r + 1) : 0u;
          if (r < g_real) { a0 = __ldg(a.rays + 2 * (size_t)sl0); a1 = __ldg(a.rays + 2 * (size_t)sl0 + 1); }
          if (r + 1u < g_real) { b0 = __ldg(a.rays + 2 * (size_t)sl1); b1 = __ldg(a.rays + 2 * (size_t)sl1 + 1); }
          float4* rp = sr + ray_rix(pp);
          rp[0] = make_float4(a0.x, b0.x, a0.y, b0.y);
          rp[RAY_PLANE] = make_float4(a0.z, b0.z, a0.w, b0.w);
          rp[2 * RAY_PLANE] = make_float4(a1.x, b1.x, a1.y, b1.y);
          rp[3 * RAY_PLANE] = make_float4(a1.z, b1.z, a1.w, b1.w);
        }
      }
      if (tid == 0) { s_carry = 0u; s_carry_c = 0u; s_exm_full = 1u; }
      __syncthreads();
      for (int jp = tid; jp < (K + 1) / 2; jp += TRAV_THREADS) {
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 a0 = s_top[6 * jp], a1 = s_top[6 * jp + 1], a2 = s_top[6 * jp + 2];
        const bool has1 = 2 * jp + 1 < K;
        const float4 b0 = has1 ? s_top[6 * jp + 3] : z, b1 = has1 ? s_top[6 * jp + 4] : z, b2 = has1 ? s_top[6 * jp + 5] : z;
        float4* rec = s_tpairs + 5 * jp;
        rec[0] = make_float4(a0.x, b0.x, a0.y, b0.y);
        rec[1] = make_float4(a0.z, b0.z, a0.w, b0.w);
        rec[2] = make_float4(a1.x, b1.x, a1.y, b1.y);
        rec[3] = make_float4(a1.z, b1.z, a1.w, b1.w);
        rec[4] = make_float4(a2.x, b2.x, 0.f, 0.f);
      }
      if (Lv >= 2) {   // existing-children masks and (SMALL) paired child records
        const int k1 = Lv - 1;
        for (int j = tid; j < K; j += TRAV_THREADS) {
          uint32_t m = 0;
          for (int c = 0; c < B; ++c) {
            const uint32_t child = ((uint32_t)j << logB) | (uint32_t)c;
            const float r = SMALL ? s_nodes[s_noff[k1] + 3 * child].w
                                  : __ldg(&s_trav[k1][3 * ((size_t)g * s_pg[k1] + child)].w);
            m |= (r >= 0.0f ? 1u : 0u) << c;
          }
          s_exm[j] = m;
          if (m != (B == 32 ? 0xFFFFFFFFu : ((1u << B) - 1u))) s_exm_full = 0u;   // benign race: all write 0
        }
        if (SMALL) {
          const uint32_t n_pairs = s_pg[k1] / 2u;
          for (uint32_t pp = tid; pp < n_pairs; pp += TRAV_THREADS) {
            const float4* n0 = s_nodes + s_noff[k1] + 3 * (2 * pp);
            const float4 a0 = n0[0], a1 = n0[1], a2 = n0[2], b0 = n0[3], b1 = n0[4], b2 = n0[5];
            float4* rec = s_pairs + 5 * pp;
            rec[0] = make_float4(a0.x, b0.x, a0.y, b0.y);
            rec[1] = make_float4(a0.z, b0.z, a0.w, b0.w);
            rec[2] = make_float4(a1.x, b1.x, a1.y, b1.y);
            rec[3] = make_float4(a1.z, b1.z, a1.w, b1.w);
            rec[4] = make_float4(a2.x, b2.x, 0.f, 0.f);
          }
        }
      }
      // compact the meshes any of the K nodes kept, in mesh order, with the
      // exclusive prefix of their triangle counts (the group's virtual
      // triangle index space, cut into work items by k_plan)
      for (int m0 = 0; m0 < a.n_meshes; m0 += TRAV_THREADS) {
        const int m = m0 + (int)tid;
        uint32_t nm = 0, cnt = 0;
        if (m < a.n_meshes) {
          const int w = m >> 5, b = m & 31;
          for (int j = 0; j < K; ++j) nm |= ((__ldg(a.masks + ((size_t)g * K + j) * a.W + w) >> b) & 1u) << j;
          cnt = nm ? __ldg(a.mesh_count + m) : 0u;
        }
        const uint32_t real_cnt = cnt;
        if (objtree) cnt = (cnt + CLUSTER_TRIS - 1) / CLUSTER_TRIS * CLUSTER_TRIS;   // whole clusters (slices)
        const uint32_t act = nm ? 1u : 0u;
        uint32_t tot_a, tot_c;
        const uint32_t ea = block_excl_scan<TRAV_WARPS>(act, s_warp, &tot_a);
        const uint32_t ec = block_excl_scan<TRAV_WARPS>(cnt, s_warp, &tot_c);
        const uint32_t base_a = s_carry, base_c = s_carry_c;
        if (act) {
          s_act_nmask[base_a + ea] = nm;
          s_act_prefix[base_a + ea] = base_c + ec;
          s_act_first[base_a + ea] = __ldg(a.mesh_first + m);
          s_act_cnt[base_a + ea] = real_cnt;
          if (objtree) s_act_cfirst[base_a + ea] = __ldg(a.mesh_cluster_first + m);
        }
        __syncthreads();
        if (tid == 0) { s_carry = base_a + tot_a; s_carry_c = base_c + tot_c; }
        __syncthreads();
      }
      if (tid == 0) s_act_prefix[s_carry] = s_carry_c;
      if (tid == 0) { s_n_act = s_carry; s_cur_g = g; }
      if (SMALL) {
        for (uint32_t r = tid; r < a.group_rays; r += TRAV_THREADS) s_best[r] = BEST_NONE;
      }
      cur_g = g;
    }
    if (PER_ITEM && tid == 0) s_blk = 0u;
#if CRSH_OBJ_TWOPHASE
    if (OBJ && tid == 0) { s_lcnt = 0u; s_lclaim = 0u; s_lexh = 0u; }
#endif
    if (PER_ITEM || new_group) {
      __syncthreads();
      n_act = s_n_act;
    }
    const size_t rbase = (size_t)g * a.group_rays;
    uint32_t c_top_t = 0, c_top_h = 0, c_ch_t = 0, c_ch_h = 0, c_mt_t = 0, c_mt_h = 0;   // item counters (all but c_ch_t per lane)
    uint32_t c_cl_t = 0, c_cl_h = 0;   // object-tree cluster tests / passes (lane 0 of each slice)

    // final tests: one step = up to 32 (bundle, triangle) entries
    // from the end of Q[1], one per lane; the lane loads its triangle once
    // and runs Moller-Trumbore against the bundle's B0 rays
    const uint2* q1base = q + s_qoff[1];
    const int B0 = B0T ? B0T : a.B0;
    auto step_mt_fn = [&]() {
      const uint32_t qk = qget(1);
      const uint32_t n = min(qk, step_mt);
      if (lane < n) {
        const uint2 e = q1base[qk - n + lane];
        const float4* te = a.tri_e + 3 * (size_t)e.y;
        const float4 tv0 = __ldg(te), te1 = __ldg(te + 1), te2 = __ldg(te + 2);
        const f3 v0 = mk3(tv0.x, tv0.y, tv0.z), e1 = mk3(te1.x, te1.y, te1.z), e2 = mk3(te2.x, te2.y, te2.z);
        const uint32_t rl0 = B0T ? e.x * (uint32_t)B0T : e.x << logB0;   // first ray of the bundle (B0 even)
        // ray-plane base of the bundle: its records are ray_rix(rl0/2) + i
        // while they stay inside one block of 8 (compile-time B0 <= 16)
        constexpr bool RB_CONST = B0T >= 2 && B0T <= 16;
        const float4* rb = s_rays + ray_rix(rl0 >> 1);
        auto ray_rec = [&](uint32_t rl, int r, int k) -> float4 {
          if (RB_CONST) return rb[(uint32_t)k * RAY_PLANE + (uint32_t)(r >> 1)];
          return s_rays[(uint32_t)k * RAY_PLANE + ray_rix(rl >> 1)];
        };
        const uint32_t nr = min((uint32_t)B0, g_real - rl0);   // real rays of the bundle (>= 1: the bundle exists)
        CRSH_CHECK(rl0 < g_real && rl0 + (uint32_t)B0 <= a.group_rays && e.y < a.M, 804);
        c_mt_t += nr;   // every real ray of the bundle is tested against the triangle
        // a padding ray (odd nr: the partner of the last real ray) has
        // tmin = tmax = -1 (k_leaves), so no t passes tmin < t < tmax: it
        // never hits and needs no mask
        // the bundle's leaf record: {c, d}, {a, tan}, {sec, shared-origin flag} (k_leaves)
        const float4* lf = Lv == 1 ? s_top + 3 * e.x
                                   : (SMALL ? s_nodes + s_noff[1] + 3 * e.x : s_trav[1] + 3 * ((size_t)g * s_pg[1] + e.x));
        const bool shared_o = SMALL ? lf[2].y != 0.0f : __ldg(&lf[2].y) != 0.0f;
        if (shared_o && SMALL) {   // all rays start at the leaf centre: per-(bundle, triangle) terms once
          const float4 c0 = lf[0];
          const f3 tv = mk3(c0.x, c0.y, c0.z) - v0;
          const f3 qv = cross3(tv, e1);
          const float tq = dot3(e2, qv);
#pragma unroll
          for (int r = 0; r < (B0T ? B0T : 64); r += 2) {
            if (!B0T && r >= B0) break;
            if ((uint32_t)r >= nr) break;
            const uint32_t rl = rl0 + (uint32_t)r;
            const float4 Bq = ray_rec(rl, r, 1), Cq = ray_rec(rl, r, 2), Dq = ray_rec(rl, r, 3);
            float t0, t1;
            const uint32_t hm = mt2o_ns(Bq, Cq, Dq, e1, e2, tv, qv, tq, t0, t1);   // bit i: ray rl+i hit
            if (hm) {
              c_mt_h += __popc(hm);
              if (hm & 1u) atomicMin(s_best + rl, pack_hit(t0, e.y));
              if (hm & 2u) atomicMin(s_best + rl + 1, pack_hit(t1, e.y));
            }
          }
        } else
#pragma unroll
        for (int r = 0; r < (B0T ? B0T : 64); r += 2) {
          if (!B0T && r >= B0) break;
          if ((uint32_t)r >= nr) break;
          const uint32_t rl = rl0 + (uint32_t)r;
          float4 A, Bq, Cq, Dq;
          if (SMALL) {
            A = ray_rec(rl, r, 0); Bq = ray_rec(rl, r, 1); Cq = ray_rec(rl, r, 2); Dq = ray_rec(rl, r, 3);
          } else {
            const float4* rs = a.sorted_rays + 2 * (rbase + rl);
            const float4 a0 = __ldg(rs), a1 = __ldg(rs + 1), b0 = __ldg(rs + 2), b1 = __ldg(rs + 3);
            A = make_float4(a0.x, b0.x, a0.y, b0.y); Bq = make_float4(a0.z, b0.z, a0.w, b0.w);
            Cq = make_float4(a1.x, b1.x, a1.y, b1.y); Dq = make_float4(a1.z, b1.z, a1.w, b1.w);
          }
          float t0, t1;
          const uint32_t hm = mt2_ns(A, Bq, Cq, Dq, v0, e1, e2, t0, t1);   // bit i: ray rl+i hit
          if (hm) {
            c_mt_h += __popc(hm);
            if (hm & 1u) {
              const unsigned long long pk = pack_hit(t0, e.y);
              if (SMALL) atomicMin(s_best + rl, pk); else atomicMin(a.best + rbase + rl, pk);
            }
            if (hm & 2u) {
              const unsigned long long pk = pack_hit(t1, e.y);
              if (SMALL) atomicMin(s_best + rl + 1, pk); else atomicMin(a.best + rbase + rl + 1, pk);
            }
          }
        }
      }
      __syncwarp();
      qset(1, qk - n);
      if (!QREG) __syncwarp();
    };
    // expansion step at level k >= 2 (only when Lv >= 3 reaches below Lv-1)
    auto step_exp_fn = [&](int k) {
      const uint32_t qk = qget(k);
      const uint32_t n = min(qk, step_exp);
      const uint2* qin = q + s_qoff[k] + (qk - n);
      const uint32_t e_i = lane >> logB;
      bool test = false, pass = false;
      uint2 out = make_uint2(0u, 0u);
      if (e_i < n) {
        const uint2 e = qin[e_i];
        const uint32_t child = (e.x << logB) | (lane & Bm);
        const float4* nd = SMALL ? s_nodes + s_noff[k - 1] + 3 * child
                                 : s_trav[k - 1] + 3 * ((size_t)g * s_pg[k - 1] + child);
        const float4 c0 = SMALL ? nd[0] : __ldg(nd);
        if (c0.w >= 0.0f) {   // existing child
          const float4 c1 = SMALL ? nd[1] : __ldg(nd + 1);
          const float c2 = SMALL ? nd[2].x : __ldg(&nd[2].x);
          test = true;
          pass = cull_ns(mk3(c0.x, c0.y, c0.z), c0.w, mk3(c1.x, c1.y, c1.z), c1.w, c2, __ldg(a.tri_sph + e.y));
          out = make_uint2(child, e.y);
        }
      }
      const uint32_t bt = __ballot_sync(CRSH_FULL, test);
      const uint32_t b = __ballot_sync(CRSH_FULL, pass);
      const uint32_t q1 = qget(k - 1);
      CRSH_CHECK(!pass || q1 + __popc(b & lt) < qcap(k - 1), 801);
      if (pass) q[s_qoff[k - 1] + q1 + __popc(b & lt)] = out;
      __syncwarp();
      qset(k - 1, q1 + __popc(b));
      qset(k, qk - n);
      if (lane == 0) {
        atomicAdd(&ctr[CTR_TESTS + (k - 1)], (unsigned long long)__popc(bt));
        atomicAdd(&ctr[CTR_HITS + (k - 1)], (unsigned long long)__popc(b));
      }
      __syncwarp();
    };
    // take steps from the lowest level with a full step; when `all`, finish
    // with partial steps
    auto drain = [&](bool all) {
      for (;;) {
        if (qget(1) >= step_mt) { step_mt_fn(); continue; }
        int pick = 0;
        for (int k = 2; k < Lv - (Lv >= 2 ? 0 : 0); ++k)   // levels 2 .. Lv-1 (Lv >= 3 only)
          if (qget(k) >= step_exp) { pick = k; break; }
        if (!pick && all) {
          if (qget(1)) { step_mt_fn(); continue; }
          for (int k = 2; k < Lv; ++k)
            if (qget(k)) { pick = k; break; }
        }
        if (!pick) return;
        step_exp_fn(pick);
      }
    };

    uint32_t mlo = 0xFFFFFFFFu;   // the lane's active-mesh index in its previous lookup (v only grows)
    // active mesh of virtual triangle index v: largest p with prefix[p] <= v
    // (binary search for the first lookup of the item, then forward walks)
    auto mesh_of = [&](uint32_t v) -> uint32_t {
      uint32_t lo = 0;
      if (mlo == 0xFFFFFFFFu) {
        uint32_t hi = n_act;
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (s_act_prefix[mid] <= v) lo = mid; else hi = mid;
        }
      } else {
        lo = mlo;
        while (lo + 1 < n_act && s_act_prefix[lo + 1] <= v) ++lo;
      }
      mlo = lo;
      return lo;
    };
    // one 32-triangle slice, lane = triangle (tri, sph), nm = the lane's top
    // nodes to test: the top-level tests, the dense child tests, the queues
    auto slice_body = [&](uint32_t tri, float4 sph, uint32_t nm, float4 pfs) {
      const f2 Px = pk2(sph.x, sph.x), Py = pk2(sph.y, sph.y), Pz = pk2(sph.z, sph.z), Pr = pk2(sph.w, sph.w);
      // top level, all K nodes first: nodes (j, j+1) per packed test (paired
      // records); a lane tests node j only if its triangle's mesh survived
      // j's mesh cull. pm = the lane's passing top nodes.
      uint32_t pm = 0;
#if CRSH_TOP_UNIFORM
      // the nodes some lane's mesh kept, as one uniform mask: the pair skips
      // are uniform branches, and the lane's own mesh mask is applied once
      uint32_t nmu = __reduce_or_sync(CRSH_FULL, nm);
      uint32_t pa = 0xFFFFFFFFu;   // PF: child pairs that may pass (lane-l bit: node l/4, pair l%4)
      bool pa_done = false;
      if constexpr (PF == 2 && KT > 0 && KT <= 32) {
        // top-level prefilter (PF = 2): the K top nodes against the slice's
        // prefilter sphere, lanes 0..K-1; a node pair neither of which passes
        // is not evaluated (its counted tests are reported as skipped)
        {
          bool pp = false;
          if (lane < (uint32_t)KT) {
            const float4* t = s_top + 3 * lane;
            pp = cull_pf(t[0], t[1], t[2].x, pfs);
          }
          const uint32_t tp = __ballot_sync(CRSH_FULL, pp);
          const uint32_t ev = (tp | (tp >> 1)) & 0x55555555u;   // pairs evaluated (bit 2p)
          const uint32_t keep = ev | (ev << 1);
          c_cl_t += lane == 0 ? (uint32_t)__popc(nmu) : 0u;   // prefilter tests: nodes some lane's mesh kept
          c_cl_h += __popc(nm & ~keep);                        // this lane's counted top tests not evaluated
          nmu &= keep;
        }
      }
#pragma unroll
      for (int j = 0; j < K; j += 2) {
        if (((nmu >> j) & 3u) == 0u) continue;   // no lane's mesh kept node j or j+1 (or the prefilter rejected both)
#if CRSH_SEL_BITS
        pm |= cull2_bits_s(tpairs_s + 80u * (uint32_t)(j >> 1), Px, Py, Pz, Pr, 1u << j, 2u << j);
#else
        bool p0, p1;
        cull2_ns_s(tpairs_s + 80u * (uint32_t)(j >> 1), Px, Py, Pz, Pr, p0, p1);
        pm |= (p0 ? 1u << j : 0u) | (p1 ? 2u << j : 0u);
#endif
      }
      pm &= nm;
#else
#pragma unroll
      for (int j = 0; j < K; j += 2) {
        const bool n0 = (nm >> j) & 1u, n1 = (nm >> (j + 1)) & 1u;
        if (__ballot_sync(CRSH_FULL, n0 | n1) == 0u) continue;   // no lane's mesh kept node j or j+1
        bool p0, p1;
        cull2_ns(s_tpairs + 5 * (j >> 1), Px, Py, Pz, Pr, p0, p1);
        p0 &= n0;
        p1 &= n1;
        pm |= ((uint32_t)p0 << j) | ((uint32_t)p1 << (j + 1));
      }
#endif
      c_top_t += __popc(nm);   // every (node, triangle) with a surviving mesh was tested (skipped pairs have none)
      c_top_h += __popc(pm);
      // then each top node that passed for some lane
      uint32_t jm0 = __reduce_or_sync(CRSH_FULL, pm);
#if CRSH_PF_NODES
      if constexpr (PF > 0 && SMALL && BT == 8 && KT == 8) {
        if (jm0 != 0u && Lv >= 2) {
          // the slice's child prefilter now (all 64 children, one packed test
          // per lane), then only the nodes with a child pair that may pass
          // are iterated; the others' child tests are counted (and reported
          // as not evaluated) here
          pa = __ballot_sync(CRSH_FULL, cull2_pf_s(pairs_s + 80u * lane, pfs) != 0u);
          pa_done = true;
          if (PF == 1 || lane == 0) c_cl_t += (uint32_t)(KT * BT);
          uint32_t t = pa | (pa >> 1);
          t = (t | (t >> 2)) & 0x11111111u;   // bit 4j: node j has a pair that may pass
          t = (t | (t >> 3)) & 0x03030303u;
          t = (t | (t >> 6)) & 0x000F000Fu;
          t = (t | (t >> 12)) & 0xFFu;        // bit j
          const uint32_t skn = jm0 & ~t;
          if (skn != 0u) {
            if (CRSH_PF_BULK && s_exm_full) {   // uniform: every skipped node has B children -- one warp sum
              const uint32_t nt = (uint32_t)BT * __reduce_add_sync(CRSH_FULL, (uint32_t)__popc(pm & skn));
              c_ch_t += nt;
              if (PF == 1 || lane == 0) c_cl_h += nt;
            } else {
              for (uint32_t sk = skn; sk; sk &= sk - 1) {
                const int j = __ffs(sk) - 1;
                const uint32_t bj = __ballot_sync(CRSH_FULL, (pm >> j) & 1u);
                const uint32_t nt = __popc(bj) * __popc(s_exm[j]);
                c_ch_t += nt;
                if (PF == 1 || lane == 0) c_cl_h += nt;
              }
            }
          }
          jm0 &= t;
        }
      }
#endif
      for (uint32_t jm = jm0; jm; jm &= jm - 1) {
        const int j = __ffs(jm) - 1;
        const bool pass = (pm >> j) & 1u;
        const uint32_t b = __ballot_sync(CRSH_FULL, pass);
        if (Lv == 1) {   // the top level is the bundle level: queue for the final tests
          const uint32_t ql = qget(1);
          CRSH_CHECK(!pass || ql + __popc(b & lt) < qcap(1), 802);
          if (pass) q[s_qoff[1] + ql + __popc(b & lt)] = make_uint2((uint32_t)j, tri);
          __syncwarp();
          qset(1, ql + __popc(b));
          if (!QREG) __syncwarp();
          drain(false);   // keeps the queue below one top node's passes plus a partial step
          continue;
        }
        // dense children of node j (level Lv-1), two per packed f32x2 test;
        // per-lane survivor mask, appended once per top node with a warp scan
        const int k1 = Lv - 1;
        const uint32_t cbase = (uint32_t)j << logB;
        const uint32_t exm = s_exm[j];
        // PF: the child pairs of node j that may pass for some triangle of
        // the slice (all K x B children were tested once per slice against
        // its prefilter sphere, below); a pair neither of whose children
        // passes is not evaluated for any lane
        uint32_t pfm = 0xFFFFFFFFu;   // bit 2p: child pair p may pass
        if constexpr (PF > 0 && SMALL && BT == 8 && KT == 8) {
          if (!pa_done) {   // uniform: the slice's first child iteration
            pa = __ballot_sync(CRSH_FULL, cull2_pf_s(pairs_s + 80u * lane, pfs) != 0u);   // lane l: node l/4, pair l%4
            pa_done = true;
            if (PF == 1 || lane == 0) c_cl_t += (uint32_t)(KT * BT);   // prefilter tests evaluated
          }
          uint32_t x = (pa >> (4u * (uint32_t)j)) & 0xFu;   // pairs 0..3 of node j
          x = (x | (x << 2)) & 0x33u;
          x = (x | (x << 1)) & 0x55u;                       // pair p -> bit 2p
          pfm = x;
          // PF = 1: warp-uniform sums (lane 0's copy is flushed); PF = 2: sums
          // over the lanes (the top-level skips are per lane), lane 0 adds here
          if (PF == 1 || lane == 0) c_cl_h += __popc(b) * __popc(exm & ~(x | (x << 1)));   // counted, not evaluated
          if (x == 0u) {   // uniform: no child pair of node j can pass -- counted, nothing evaluated
            c_ch_t += __popc(b) * __popc(exm);
            continue;
          }
        }
        uint32_t m = 0;
#pragma unroll
        for (int c = 0; c < (BT ? BT : 32); c += 2) {
          if (!BT && c >= B) break;
          if constexpr (PF > 0) {
            if (((pfm >> c) & 1u) == 0u) continue;   // uniform
          }
          bool p0, p1;
          if (SMALL) {
#if CRSH_SEL_BITS && CRSH_LDS32
            m |= cull2_bits_s(pairs_s + 80u * ((cbase >> 1) + (uint32_t)(c >> 1)), Px, Py, Pz, Pr, 1u << c, 2u << c);
            continue;
#elif CRSH_LDS32
            cull2_ns_s(pairs_s + 80u * ((cbase >> 1) + (uint32_t)(c >> 1)), Px, Py, Pz, Pr, p0, p1);
#else
            cull2_ns(s_pairs + 5 * ((cbase >> 1) + (uint32_t)(c >> 1)), Px, Py, Pz, Pr, p0, p1);
#endif
          } else {
            const float4* nd = s_trav[k1] + 3 * ((size_t)g * s_pg[k1] + cbase + (uint32_t)c);
            const float4 a0 = __ldg(nd), a1 = __ldg(nd + 1), a2 = __ldg(nd + 2), b0 = __ldg(nd + 3),
                         b1 = __ldg(nd + 4), b2 = __ldg(nd + 5);
            const float4 rec[5] = {make_float4(a0.x, b0.x, a0.y, b0.y), make_float4(a0.z, b0.z, a0.w, b0.w),
                                   make_float4(a1.x, b1.x, a1.y, b1.y), make_float4(a1.z, b1.z, a1.w, b1.w),
                                   make_float4(a2.x, b2.x, 0.f, 0.f)};
            cull2_ns(rec, Px, Py, Pz, Pr, p0, p1);
          }
          m |= ((p0 ? 1u : 0u) << c) | ((p1 ? 1u : 0u) << (c + 1));
        }
        m = pass ? (m & exm) : 0u;
        c_ch_t += __popc(b) * __popc(exm);
        const uint32_t cnt = __popc(m);
        c_ch_h += cnt;
#if CRSH_APPEND_BITS
        if constexpr (PF == 1) {   // (measured on R6; the Z-order instantiation keeps the scan)
          // few children survive past the prefilter: append child by child
          // (a ballot per child some lane kept, entries at popc ranks) instead
          // of a warp scan of the per-lane counts
          uint32_t om = __reduce_or_sync(CRSH_FULL, m);
          if (om == 0u) continue;   // the common case: no child survived
          uint32_t ql = qget(k1);
          uint2* qb = q + s_qoff[k1];
          for (; om; om &= om - 1) {
            const uint32_t c = __ffs(om) - 1;
            const bool has = (m >> c) & 1u;
            const uint32_t bc = __ballot_sync(CRSH_FULL, has);
            CRSH_CHECK(ql + __popc(bc) <= qcap(k1), 803);
            if (has) qb[ql + __popc(bc & lt)] = make_uint2(cbase | c, tri);
            ql += __popc(bc);
          }
          __syncwarp();
          qset(k1, ql);
          if (!QREG || k1 != 1) __syncwarp();
          drain(false);
          continue;
        }
#endif
        if (__ballot_sync(CRSH_FULL, m != 0u) == 0u) continue;   // the common case: no child survived
        uint32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(CRSH_FULL, incl, o);
          if ((int)lane >= o) incl += y;
        }
        const uint32_t tot = __shfl_sync(CRSH_FULL, incl, 31);
        const uint32_t ql0 = qget(k1);
        CRSH_CHECK(ql0 + tot <= qcap(k1), 803);
        uint2* qd = q + s_qoff[k1] + ql0 + (incl - cnt);
        while (m) {
          const uint32_t c = __ffs(m) - 1;
          m &= m - 1;
          *qd++ = make_uint2(cbase | c, tri);
        }
        __syncwarp();
        qset(k1, ql0 + tot);
        if (!QREG || k1 != 1) __syncwarp();
        drain(false);
      }
    };
    if constexpr (PF > 0) {
      // child prefilter (the bench shape's plain traversal): slices are the
      // clusters of the kept meshes (each mesh padded to whole clusters),
      // handed out by a shared counter; lanes = the cluster's triangles in
      // cluster order; the cluster's prefilter sphere rides along
      for (;;) {
        uint32_t si = 0;
        if (lane == 0) si = atomicAdd(&s_blk, 1u);
        const uint32_t s0 = item.y + __shfl_sync(CRSH_FULL, si, 0) * 32u;
        if (s0 >= item.z) break;
        const uint32_t lo = mesh_of(s0);   // a cluster-aligned slice lies in one mesh
        const uint32_t rel = s0 - s_act_prefix[lo];
        const uint32_t loc = rel + lane;
        uint32_t tri = 0, nm = 0;
        float4 sph = make_float4(0.f, 0.f, 0.f, 0.f);
        if (loc < s_act_cnt[lo]) {   // else a padding lane of the mesh's last cluster
          const uint32_t pidx = s_act_first[lo] + loc;
          tri = (uint32_t)__ldg(a.tri_order + pidx);
          sph = __ldg(a.tri_sph_ord + pidx);
          nm = s_act_nmask[lo];
        }
        const float4 pfs = __ldg(a.cluster_pf + s_act_cfirst[lo] + rel / CLUSTER_TRIS);
        slice_body(tri, sph, nm, pfs);
      }
    } else if constexpr (!OBJ) {
#if CRSH_TRAV_PREFETCH
      // software-pipelined slices: the next slice's mesh lookup and triangle
      // sphere load are issued before the current slice's tests, so the L2
      // latency of the sphere load overlaps them (ncu cfg4 Z-order: the first
      // use of the sphere was a top stall)
      auto fetch = [&](uint32_t s0, uint32_t& tri, float4& sph, uint32_t& nm) {
        const uint32_t v = s0 + lane;
        nm = 0; tri = 0;
        sph = make_float4(0.f, 0.f, 0.f, 0.f);
        if (v < item.z) {
          const uint32_t lo = mesh_of(v);
          tri = s_act_first[lo] + (v - s_act_prefix[lo]);
          sph = __ldg(a.tri_sph + tri);
          nm = s_act_nmask[lo];
        }
      };
      uint32_t s0 = item.y + warp * 32u;
      uint32_t tri_n = 0, nm_n = 0;
      float4 sph_n;
      if (s0 < item.z) fetch(s0, tri_n, sph_n, nm_n);
      for (; s0 < item.z; s0 += TRAV_THREADS) {
        const uint32_t tri = tri_n, nm = nm_n;
        const float4 sph = sph_n;
        if (s0 + TRAV_THREADS < item.z) fetch(s0 + TRAV_THREADS, tri_n, sph_n, nm_n);
        slice_body(tri, sph, nm, make_float4(0.f, 0.f, 0.f, 0.f));
      }
#elif CRSH_DYN_SLICE
      // slices handed out dynamically (a shared counter per item): the
      // warps of an item finish within one slice of each other (static
      // striding left them waiting at the chunk barrier, ncu cfg4 Z-order);
      // each warp's slices still come in increasing order (mesh_of walks
      // forward)
      for (;;) {
        uint32_t si = 0;
        if (lane == 0) si = atomicAdd(&s_blk, 1u);
        const uint32_t s0 = item.y + __shfl_sync(CRSH_FULL, si, 0) * 32u;
        if (s0 >= item.z) break;
        const uint32_t v = s0 + lane;
        uint32_t nm = 0, tri = 0;
        float4 sph = make_float4(0.f, 0.f, 0.f, 0.f);
        if (v < item.z) {
          const uint32_t lo = mesh_of(v);
          tri = s_act_first[lo] + (v - s_act_prefix[lo]);
          sph = __ldg(a.tri_sph + tri);
          nm = s_act_nmask[lo];
        }
        slice_body(tri, sph, nm, make_float4(0.f, 0.f, 0.f, 0.f));
      }
#else
      for (uint32_t s0 = item.y + warp * 32u; s0 < item.z; s0 += TRAV_THREADS) {
        const uint32_t v = s0 + lane;
        uint32_t nm = 0, tri = 0;
        float4 sph = make_float4(0.f, 0.f, 0.f, 0.f);
        if (v < item.z) {
          const uint32_t lo = mesh_of(v);
          tri = s_act_first[lo] + (v - s_act_prefix[lo]);
          sph = __ldg(a.tri_sph + tri);
          nm = s_act_nmask[lo];
        }
        slice_body(tri, sph, nm, make_float4(0.f, 0.f, 0.f, 0.f));
      }
#endif
    } else {
      // object sphere-tree (NEXT-4, reading O1): the item's virtual range is
      // cluster-aligned (each kept mesh padded to whole clusters), so cluster
      // c is the slice [32 c, 32 c + 32). A warp takes blocks of CPB = 32 / K
      // consecutive clusters and tests every (cluster, top node) pair of the
      // block at once, lane = (cluster lane / K, node lane % K): Eq 9 of the
      // cluster sphere against the node if the node kept the cluster's mesh.
      // Then only the clusters that passed some node are streamed as slices,
      // each lane testing its triangle against the nodes its cluster passed.
      const uint32_t cy = item.y / CLUSTER_TRIS, cz = (item.z + CLUSTER_TRIS - 1) / CLUSTER_TRIS;
      const uint32_t CPB = 32u / (uint32_t)K;   // K <= 32
      const uint32_t ci = lane / (uint32_t)K, jn = lane - ci * (uint32_t)K;
      const uint32_t kmask = K == 32 ? 0xFFFFFFFFu : ((1u << K) - 1u);
#if CRSH_OBJ_TWOPHASE
      // two phases per round: (A) blocks of clusters handed out dynamically,
      // the cluster tests of a block at once, each cluster that passed some
      // node appended to a CTA list (cluster, node mask); (B) the list's
      // clusters handed out one per claim and streamed as slices. The heavy
      // per-cluster work is then balanced to one slice (with whole blocks
      // per claim, warps waited at the item barrier behind a few heavy
      // blocks, ncu cfg4 Z-order + tree: 22 % of the stall samples). A round
      // ends when the list could overflow; rounds repeat until the blocks
      // are exhausted.
      for (;;) {
        mlo = 0xFFFFFFFFu;   // phase A claims increase per warp: a fresh forward walk
        for (;;) {
          if (*(volatile uint32_t*)&s_lcnt > a.obj_list_cap - CPB * TRAV_WARPS) break;   // list nearly full
          uint32_t bi = 0;
          if (lane == 0) bi = atomicAdd(&s_blk, 1u);
          const uint32_t b0 = cy + __shfl_sync(CRSH_FULL, bi, 0) * CPB;
          if (b0 >= cz) {
            if (lane == 0) s_lexh = 1u;
            break;
          }
          const uint32_t c = b0 + ci;
          uint32_t lo = 0;
          bool tst = false, pass = false;
          if (ci < CPB && c < cz) {
            lo = mesh_of(c * CLUSTER_TRIS);
            tst = (s_act_nmask[lo] >> jn) & 1u;
            if (tst) {
              const float4 cs = __ldg(a.cluster_sph + s_act_cfirst[lo] + (c * CLUSTER_TRIS - s_act_prefix[lo]) / CLUSTER_TRIS);
              const float4 t0 = s_top[3 * jn], t1 = s_top[3 * jn + 1], t2 = s_top[3 * jn + 2];
              pass = cull_ns(mk3(t0.x, t0.y, t0.z), t0.w, mk3(t1.x, t1.y, t1.z), t1.w, t2.x, cs);
            }
          }
          const uint32_t bt = __ballot_sync(CRSH_FULL, tst), bp = __ballot_sync(CRSH_FULL, pass);
          if (lane == 0) { c_cl_t += __popc(bt); c_cl_h += __popc(bp); }
          const uint32_t cmk_l = lane < CPB ? (bp >> (lane * (uint32_t)K)) & kmask : 0u;   // lane q: cluster b0+q
          const uint32_t qm = __ballot_sync(CRSH_FULL, cmk_l != 0u);
          if (qm) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&s_lcnt, (uint32_t)__popc(qm));
            base = __shfl_sync(CRSH_FULL, base, 0);
            CRSH_CHECK(base + __popc(qm) <= a.obj_list_cap, 807);
            if (cmk_l) s_list[base + __popc(qm & lt)] = make_uint2(b0 + lane, cmk_l);
          }
        }
        __syncthreads();
        const uint32_t n_list = s_lcnt;
        for (;;) {
          uint32_t ei = 0;
          if (lane == 0) ei = atomicAdd(&s_lclaim, 1u);
          ei = __shfl_sync(CRSH_FULL, ei, 0);
          if (ei >= n_list) break;
          const uint2 en = s_list[ei];
          mlo = 0xFFFFFFFFu;   // list order is not monotone per warp: binary search
          const uint32_t lok = mesh_of(en.x * CLUSTER_TRIS);
          const uint32_t loc = en.x * CLUSTER_TRIS + lane - s_act_prefix[lok];
          uint32_t tri = 0, nm = 0;
          float4 sph = make_float4(0.f, 0.f, 0.f, 0.f);
          if (loc < s_act_cnt[lok]) {   // else a padding lane of the mesh's last cluster
            const uint32_t pidx = s_act_first[lok] + loc;
            tri = (uint32_t)__ldg(a.tri_order + pidx);
            sph = __ldg(tsph + pidx);
            nm = en.y;
          }
          slice_body(tri, sph, nm, make_float4(0.f, 0.f, 0.f, 0.f));
        }
        __syncthreads();
        const bool exhausted = s_lexh != 0u;
        __syncthreads();
        if (exhausted) break;
        if (tid == 0) { s_lcnt = 0u; s_lclaim = 0u; }
        __syncthreads();
      }
#else
      // blocks are handed out dynamically (a shared counter per item): the
      // clusters that pass are unevenly spread, and static striding left
      // warps waiting at the item barrier (ncu cfg4: barrier stalls)
      for (;;) {
        uint32_t bi = 0;
        if (lane == 0) bi = atomicAdd(&s_blk, 1u);
        const uint32_t b0 = cy + __shfl_sync(CRSH_FULL, bi, 0) * CPB;
        if (b0 >= cz) break;
        const uint32_t c = b0 + ci;
        uint32_t lo = 0;
        bool tst = false, pass = false;
        if (ci < CPB && c < cz) {
          lo = mesh_of(c * CLUSTER_TRIS);
          tst = (s_act_nmask[lo] >> jn) & 1u;
          if (tst) {
            const float4 cs = __ldg(a.cluster_sph + s_act_cfirst[lo] + (c * CLUSTER_TRIS - s_act_prefix[lo]) / CLUSTER_TRIS);
            const float4 t0 = s_top[3 * jn], t1 = s_top[3 * jn + 1], t2 = s_top[3 * jn + 2];
            pass = cull_ns(mk3(t0.x, t0.y, t0.z), t0.w, mk3(t1.x, t1.y, t1.z), t1.w, t2.x, cs);
          }
        }
        const uint32_t bt = __ballot_sync(CRSH_FULL, tst), bp = __ballot_sync(CRSH_FULL, pass);
        if (lane == 0) { c_cl_t += __popc(bt); c_cl_h += __popc(bp); }
        for (uint32_t q = 0; q < CPB; ++q) {
          const uint32_t cmk = (bp >> (q * (uint32_t)K)) & kmask;
          if (!cmk) continue;   // uniform: this cluster passed no node
          const uint32_t lok = __shfl_sync(CRSH_FULL, lo, q * (uint32_t)K);
          const uint32_t loc = (b0 + q) * CLUSTER_TRIS + lane - s_act_prefix[lok];
          uint32_t tri = 0, nm = 0;
          float4 sph = make_float4(0.f, 0.f, 0.f, 0.f);
          if (loc < s_act_cnt[lok]) {   // else a padding lane of the mesh's last cluster
            const uint32_t pidx = s_act_first[lok] + loc;
            tri = (uint32_t)__ldg(a.tri_order + pidx);
            sph = __ldg(tsph + pidx);
            nm = cmk;
          }
          slice_body(tri, sph, nm, make_float4(0.f, 0.f, 0.f, 0.f));
        }
      }
#endif
    }
    drain(true);
    // item counters -> the warp's running 64-bit counters (flushed to the CTA
    // counters when the segment changes and at the end: per-item 64-bit
    // shared atomics are CAS loops that the 8 warps contended on, ncu cfg4)
    // (A/B: +0.8 % at cfg4 R6; the object-tree instantiation, whose items
    // are short, measured 3 % slower with them -- its extra live registers
    // spill -- and keeps the per-item flush)
    acc_tt += __reduce_add_sync(CRSH_FULL, c_top_t);
    acc_th += __reduce_add_sync(CRSH_FULL, c_top_h);
    acc_mt += __reduce_add_sync(CRSH_FULL, c_mt_t);
    acc_mh += __reduce_add_sync(CRSH_FULL, c_mt_h);
    acc_ch += __reduce_add_sync(CRSH_FULL, c_ch_h);
    acc_ct += c_ch_t;      // warp-uniform already
    if constexpr (PF == 2) {   // per-lane sums
      acc_clt += __reduce_add_sync(CRSH_FULL, c_cl_t);
      acc_clh += __reduce_add_sync(CRSH_FULL, c_cl_h);
    } else {
      acc_clt += c_cl_t;     // lane 0 only (lane 0 flushes)
      acc_clh += c_cl_h;
    }
    if constexpr (OBJ) flush_acc();
  }
  group_end();
  flush_acc();
  __syncthreads();
  for (uint32_t i = tid; i < MAX_SEG * CTR_STRIDE; i += TRAV_THREADS)
    if (s_ctr[i]) atomicAdd(a.counters + i, s_ctr[i]);
}

// ============================================================== brute force (N x M)
struct BruteArgs {
  const FrameDesc* fd;          // N, seg_comp_start
  const uint32_t* vals_c;       // compacted slot ids
  const float4* rays;           // [slots][2]
  const float4* tri_e;
  int64_t M;
  int32_t n_seg;
  int32_t* out_hit;
  float* out_t;
  unsigned long long* out_packed;
  PeerOut peer;
  unsigned long long* counters;
};

// Naive ray tracing: one thread per ray, every triangle, staged 256 at
// a time through shared memory (broadcast reads); closest hit with the same
// (t, tri) order as the hierarchy path.
__global__ void __launch_bounds__(256) k_brute(const BruteArgs a) {
  __shared__ float4 s_tri[3 * 256];
  __shared__ unsigned long long s_hit[MAX_SEG], s_tests[MAX_SEG];
  if (threadIdx.x < MAX_SEG) { s_hit[threadIdx.x] = 0ull; s_tests[threadIdx.x] = 0ull; }
  const uint32_t i = blockIdx.x * 256u + threadIdx.x;
  const uint32_t N = a.fd->N;
  if (blockIdx.x * 256u >= N) return;   // surplus block (uniform)
  const bool ok = i < N;
  uint32_t slot = 0;
  float4 r0 = make_float4(0.f, 0.f, 0.f, 1.f), r1 = make_float4(0.f, 0.f, 1.f, -1.f);
  if (ok) {
    slot = __ldg(a.vals_c + i);
    r0 = __ldg(a.rays + 2 * (size_t)slot);
    r1 = __ldg(a.rays + 2 * (size_t)slot + 1);
  }
  const f3 o = mk3(r0.x, r0.y, r0.z), d = mk3(r1.x, r1.y, r1.z);
  unsigned long long best = BEST_NONE;
  int seg = 0;
  uint32_t hv = 0;
  for (int64_t t0 = 0; t0 < a.M; t0 += 256) {
    __syncthreads();
    const int nt = (int)((a.M - t0) < 256 ? (a.M - t0) : 256);
    for (int j = threadIdx.x; j < 3 * nt; j += 256) s_tri[j] = __ldg(a.tri_e + 3 * t0 + j);
    __syncthreads();
    if (ok) {
      for (int k = 0; k < nt; ++k) {
        const float4 v0 = s_tri[3 * k], e1 = s_tri[3 * k + 1], e2 = s_tri[3 * k + 2];
        float th;
        if (mt_ns(o, d, r0.w, r1.w, mk3(v0.x, v0.y, v0.z), mk3(e1.x, e1.y, e1.z), mk3(e2.x, e2.y, e2.z), &th)) {
          const unsigned long long pk = pack_hit(th, (uint32_t)(t0 + k));
          best = pk < best ? pk : best;
        }
      }
    }
  }
  if (ok) {
    int s = 0;
    for (int q = 1; q < a.n_seg; ++q) s = (i >= a.fd->seg_comp_start[q]) ? q : s;
    const bool hit = best != BEST_NONE;
    if (a.peer.n) {
      a.peer.store(slot, hit ? best : PACK_MISS);
    } else if (a.out_packed) {
      a.out_packed[slot] = hit ? best : PACK_MISS;
    } else {
      a.out_hit[slot] = hit ? (int32_t)(uint32_t)(best & 0xFFFFFFFFull) : -1;
      a.out_t[slot] = hit ? __uint_as_float((uint32_t)(best >> 32)) : __int_as_float(0x7f800000);
    }
    seg = s;
    hv = hit ? 1u : 0u;
  }
  warp_seg_add(s_hit, 1, a.n_seg, seg, hv);
  warp_seg_add(s_tests, 1, a.n_seg, seg, ok ? 1u : 0u);   // rays x M below
  __syncthreads();
  if (threadIdx.x < MAX_SEG) {
    if (s_hit[threadIdx.x]) atomicAdd(a.counters + threadIdx.x * CTR_STRIDE + CTR_RAYS_HIT, s_hit[threadIdx.x]);
    if (s_tests[threadIdx.x])
      atomicAdd(a.counters + threadIdx.x * CTR_STRIDE + CTR_FINAL_TESTS, s_tests[threadIdx.x] * (unsigned long long)a.M);
  }
}

// ============================================================== K9
struct UnpackArgs {
  const FrameDesc* fd;          // g_lo, g_hi, seg_pad_base, seg_n -> this rank's sorted-ray range
  uint32_t group_rays;
  int32_t n_seg;
  const uint32_t* sorted_slot;
  const unsigned long long* best;
  int32_t* out_hit;
  float* out_t;
  unsigned long long* out_packed;
  PeerOut peer;                 // fused multi-GPU epilogue: store owned results into every destination
  unsigned long long* counters;
  uint32_t n_slots;             // checked builds
};

__global__ void __launch_bounds__(256) k_unpack(const UnpackArgs a) {
  __shared__ unsigned long long s_hit[MAX_SEG];
  if (threadIdx.x < MAX_SEG) s_hit[threadIdx.x] = 0ull;
  __syncthreads();
  const uint32_t r_lo = a.fd->g_lo * a.group_rays, r_hi = a.fd->g_hi * a.group_rays;
  const uint32_t i = r_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (r_lo + blockIdx.x * blockDim.x >= r_hi) return;   // surplus block (uniform)
  int s = 0;
  uint32_t hv = 0;
  if (i < r_hi) {
    for (int q = 1; q < a.n_seg; ++q) s = (i >= a.fd->seg_pad_base[q]) ? q : s;
    if (i - a.fd->seg_pad_base[s] < a.fd->seg_n[s]) {
      const uint32_t slot = __ldg(a.sorted_slot + i);
      CRSH_CHECK(slot < a.n_slots, 901);
      const unsigned long long b = __ldg(a.best + i);
      const bool hit = b != BEST_NONE;
      if (a.peer.n) {
        a.peer.store(slot, hit ? b : PACK_MISS);
      } else if (a.out_packed) {
        a.out_packed[slot] = hit ? b : PACK_MISS;
      } else {
        a.out_hit[slot] = hit ? (int32_t)(uint32_t)(b & 0xFFFFFFFFull) : -1;
        a.out_t[slot] = hit ? __uint_as_float((uint32_t)(b >> 32)) : __int_as_float(0x7f800000);
      }
      hv = hit ? 1u : 0u;
    }
  }
  warp_seg_add(s_hit, 1, a.n_seg, s, hv);
  __syncthreads();
  if (threadIdx.x < MAX_SEG && s_hit[threadIdx.x]) atomicAdd(a.counters + threadIdx.x * CTR_STRIDE + CTR_RAYS_HIT, s_hit[threadIdx.x]);
}

// packed (min-reduced across ranks) -> hit_tri / t
__global__ void k_unpack_packed(const unsigned long long* packed, uint64_t n, int32_t* hit, float* t) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = packed[i];
    if (v >= PACK_EMPTY) { hit[i] = -2; t[i] = __int_as_float(0x7f800000); }
    else if ((v >> 32) == 0x7F800000ull) { hit[i] = -1; t[i] = __int_as_float(0x7f800000); }
    else { hit[i] = (int32_t)(uint32_t)(v & 0xFFFFFFFFull); t[i] = __uint_as_float((uint32_t)(v >> 32)); }
  }
}

}  // namespace crsh
