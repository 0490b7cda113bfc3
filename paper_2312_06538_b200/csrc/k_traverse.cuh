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
constexpr int CTR_STRIDE = 32;

constexpr unsigned long long BEST_NONE = 0xFFFFFFFFFFFFFFFFull;
constexpr unsigned long long PACK_MISS = 0x7F800000FFFFFFFFull;
constexpr unsigned long long PACK_EMPTY = 0x7FFFFFFFFFFFFFFFull;

__device__ __forceinline__ unsigned long long pack_hit(float t, uint32_t tri) {
  return ((unsigned long long)__float_as_uint(t) << 32) | tri;
}

// ============================================================== K7
struct CullArgs {
  uint32_t top_lo, top_hi;     // padded top-node range of this shard
  int32_t W;                   // mask words per node = ceil(n_meshes / 32)
  const float4* trav_top;      // level Lv, traversal layout
  int32_t n_meshes;
  const float4* mesh_sph;
  const uint32_t* mesh_count;
  int32_t cull_on;
  uint32_t* masks;             // [n_top_padded][W]
  unsigned long long* counters;
  int32_t n_seg;
  uint32_t seg_top_start[MAX_SEG + 1];
};

__global__ void __launch_bounds__(256) k_mesh_cull(const CullArgs a) {
  __shared__ unsigned long long s_ctr[MAX_SEG][2];
  if (threadIdx.x < MAX_SEG * 2) (&s_ctr[0][0])[threadIdx.x] = 0ull;
  __syncthreads();
  const uint64_t gid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t total = (uint64_t)(a.top_hi - a.top_lo) * a.W;
  if (gid < total) {
    const uint32_t n = a.top_lo + (uint32_t)(gid / a.W);
    const int w = (int)(gid % a.W);
    const float4 p0 = __ldg(a.trav_top + 3 * (size_t)n), p1 = __ldg(a.trav_top + 3 * (size_t)n + 1),
                 p2 = __ldg(a.trav_top + 3 * (size_t)n + 2);
    uint32_t bits = 0, tests = 0, hits = 0;
    if (p0.w >= 0.0f) {
      const f3 C = mk3(p0.x, p0.y, p0.z), A = mk3(p1.x, p1.y, p1.z);
      for (int b = 0; b < 32; ++b) {
        const int m = w * 32 + b;
        if (m >= a.n_meshes) break;
        if (__ldg(a.mesh_count + m) == 0) continue;
        if (a.cull_on) {
          ++tests;
          if (cull_ns(C, p0.w, A, p1.w, p2.x, __ldg(a.mesh_sph + m))) { bits |= 1u << b; ++hits; }
        } else {
          bits |= 1u << b;
        }
      }
    }
    a.masks[(size_t)n * a.W + w] = bits;
    if (tests) {
      int s = 0;
      for (int q = 1; q < a.n_seg; ++q) s = (n >= a.seg_top_start[q]) ? q : s;
      atomicAdd(&s_ctr[s][0], (unsigned long long)tests);
      atomicAdd(&s_ctr[s][1], (unsigned long long)hits);
    }
  }
  __syncthreads();
  if (threadIdx.x < MAX_SEG * 2) {
    const unsigned long long v = (&s_ctr[0][0])[threadIdx.x];
    if (v) atomicAdd(a.counters + (threadIdx.x / 2) * CTR_STRIDE + CTR_MESH_TESTS + (threadIdx.x & 1), v);
  }
}

// ============================================================== K7b
struct PlanArgs {
  uint32_t g_lo, g_hi;         // group range of this shard
  int32_t K, W;
  const uint32_t* masks;
  int32_t n_meshes;
  const uint32_t* mesh_count;
  uint32_t item_tris;
  uint4* items;                // (group, v_begin, v_end, 0)
  uint32_t* n_items;
  unsigned long long* status;
  uint32_t* ticket;
};

__global__ void __launch_bounds__(SCAN_THREADS) k_plan(const PlanArgs a) {
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ uint32_t s_cnt[SCAN_ITEMS * 8], s_excl[SCAN_ITEMS * 8];
  if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t ntri[SCAN_ITEMS], nit[SCAN_ITEMS], wex[SCAN_ITEMS];
#pragma unroll
  for (int it = 0; it < SCAN_ITEMS; ++it) {
    const uint32_t g = a.g_lo + tile * SCAN_TILE + it * SCAN_THREADS + threadIdx.x;
    uint32_t T = 0;
    if (g < a.g_hi) {
      for (int w = 0; w < a.W; ++w) {
        uint32_t m = 0;
        for (int j = 0; j < a.K; ++j) m |= __ldg(a.masks + ((size_t)g * a.K + j) * a.W + w);
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          T += __ldg(a.mesh_count + w * 32 + b);
        }
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
  __syncthreads();
  if (warp == 0) tile_scan_lookback(s_cnt, s_excl, &s_prefix, a.status, (int)tile);
  __syncthreads();
  const uint32_t prefix = s_prefix;
#pragma unroll
  for (int it = 0; it < SCAN_ITEMS; ++it) {
    const uint32_t g = a.g_lo + tile * SCAN_TILE + it * SCAN_THREADS + threadIdx.x;
    const uint32_t off = prefix + s_excl[it * 8 + warp] + wex[it];
    for (uint32_t q = 0; q < nit[it]; ++q)
      a.items[off + q] = make_uint4(g, q * a.item_tris, min(ntri[it], (q + 1) * a.item_tris), 0u);
  }
  const uint32_t n_tiles = (a.g_hi - a.g_lo + SCAN_TILE - 1) / SCAN_TILE;
  if (tile == n_tiles - 1 && threadIdx.x == 0) {
    uint32_t t = 0;
    for (int q = 0; q < SCAN_ITEMS * 8; ++q) t += s_cnt[q];
    *a.n_items = prefix + t;
  }
}

// ============================================================== K8
constexpr int TRAV_THREADS = 256;
constexpr int TRI_BITS = 9;           // tile-local triangle index bits in queue entries
constexpr int MAX_TILE = 1 << TRI_BITS;

struct TravArgs {
  int32_t Lv, B0, B, K;
  uint32_t group_rays;
  int32_t tile;                       // triangles per tile (<= 512)
  int32_t qcap;                       // capacity of the lower-level queues
  int32_t qtop_cap;                   // K * tile
  const float4* trav[MAX_LEVELS + 1]; // level k (1..Lv), traversal layout
  uint32_t per_group[MAX_LEVELS + 1]; // nodes per group at level k
  const float4* sorted_rays;
  const float4* tri_e;
  const float4* tri_sph;
  const uint32_t* masks;
  int32_t W, n_meshes;
  const uint32_t* mesh_first;
  const uint32_t* mesh_count;
  const uint4* items;
  const uint32_t* n_items;
  uint32_t* ticket;
  unsigned long long* best;           // [Np]
  unsigned long long* counters;
  int32_t n_seg;
  uint32_t seg_group_start[MAX_SEG + 1];
};

// dynamic shared-memory layout (bytes), shared by host and device
struct TravSmem {
  uint32_t off_top, off_act_mesh, off_act_nmask, off_act_prefix, off_act_first, off_tri_sph, off_tri_id,
      off_tri_nmask, off_q[MAX_LEVELS + 1], off_best, total;
  __host__ __device__ static TravSmem make(int K, int n_meshes, int tile, int Lv, int qcap, bool smem_best) {
    TravSmem s;
    uint32_t o = 0;
    auto take = [&](uint32_t bytes) { const uint32_t r = o; o += (bytes + 15u) & ~15u; return r; };
    s.off_top = take(K * 48u);
    s.off_act_mesh = take(4u * n_meshes);
    s.off_act_nmask = take(4u * n_meshes);
    s.off_act_prefix = take(4u * (n_meshes + 1));
    s.off_act_first = take(4u * n_meshes);
    s.off_tri_sph = take(16u * tile);
    s.off_tri_id = take(4u * tile);
    s.off_tri_nmask = take(4u * tile);
    for (int k = 0; k <= MAX_LEVELS; ++k) s.off_q[k] = 0;
    for (int k = 1; k <= Lv; ++k) s.off_q[k] = take(4u * (k == Lv ? (uint32_t)(K * tile) : (uint32_t)qcap));
    s.off_best = smem_best ? take(8u * 512u) : 0u;
    s.total = o;
    return s;
  }
};

// warp-aggregated append of `val` where pred; every lane of the warp calls.
__device__ __forceinline__ void push_warp(bool pred, uint32_t val, uint32_t* q, uint32_t* qlen) {
  const uint32_t b = __ballot_sync(CRSH_FULL, pred);
  if (b == 0u) return;
  const uint32_t lane = lane_id();
  const int leader = __ffs(b) - 1;
  uint32_t base = 0;
  if ((int)lane == leader) base = atomicAdd(qlen, (uint32_t)__popc(b));
  base = __shfl_sync(CRSH_FULL, base, leader);
  if (pred) q[base + __popc(b & lanemask_lt())] = val;
}

__device__ __forceinline__ void warp_count(unsigned long long* dst, uint32_t v) {
  const uint32_t s = __reduce_add_sync(CRSH_FULL, v);
  if (lane_id() == 0 && s) atomicAdd(dst, (unsigned long long)s);
}

template <bool SMEM_BEST>
__global__ void __launch_bounds__(TRAV_THREADS) k_traverse(const TravArgs a, const TravSmem L) {
  extern __shared__ __align__(16) unsigned char smraw[];
  float4* s_top = reinterpret_cast<float4*>(smraw + L.off_top);
  uint32_t* s_act_mesh = reinterpret_cast<uint32_t*>(smraw + L.off_act_mesh);
  uint32_t* s_act_nmask = reinterpret_cast<uint32_t*>(smraw + L.off_act_nmask);
  uint32_t* s_act_prefix = reinterpret_cast<uint32_t*>(smraw + L.off_act_prefix);
  uint32_t* s_act_first = reinterpret_cast<uint32_t*>(smraw + L.off_act_first);
  float4* s_tri_sph = reinterpret_cast<float4*>(smraw + L.off_tri_sph);
  uint32_t* s_tri_id = reinterpret_cast<uint32_t*>(smraw + L.off_tri_id);
  uint32_t* s_tri_nmask = reinterpret_cast<uint32_t*>(smraw + L.off_tri_nmask);
  unsigned long long* s_best = reinterpret_cast<unsigned long long*>(smraw + L.off_best);
  __shared__ uint32_t s_qlen[MAX_LEVELS + 1];
  __shared__ uint32_t s_item, s_cur_g, s_n_act, s_carry, s_carry_c;
  __shared__ uint32_t s_warp[8];
  __shared__ unsigned long long s_ctr[MAX_SEG * CTR_STRIDE];

  const int Lv = a.Lv, B = a.B, B0 = a.B0, K = a.K;
  const uint32_t tid = threadIdx.x, lane = lane_id();
  for (uint32_t i = tid; i < MAX_SEG * CTR_STRIDE; i += TRAV_THREADS) s_ctr[i] = 0ull;
  if (tid == 0) s_cur_g = 0xFFFFFFFFu;
  if (tid <= MAX_LEVELS) s_qlen[tid] = 0u;
  const uint32_t n_items = *a.n_items;

  for (;;) {
    __syncthreads();
    if (tid == 0) s_item = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const uint32_t it = s_item;
    if (it >= n_items) break;
    const uint4 item = __ldg(a.items + it);
    const uint32_t g = item.x;
    int seg = 0;
    for (int q = 1; q < a.n_seg; ++q) seg = (g >= a.seg_group_start[q]) ? q : seg;
    unsigned long long* ctr = s_ctr + seg * CTR_STRIDE;

    if (g != s_cur_g) {   // uniform: group setup (top nodes, surviving meshes)
      for (int j = tid; j < 3 * K; j += TRAV_THREADS) s_top[j] = __ldg(a.trav[Lv] + (size_t)g * K * 3 + j);
      if (tid == 0) { s_carry = 0u; s_carry_c = 0u; }
      __syncthreads();
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
        const uint32_t act = nm ? 1u : 0u;
        uint32_t tot_a, tot_c;
        const uint32_t ea = block_excl_scan_256(act, s_warp, &tot_a);
        const uint32_t ec = block_excl_scan_256(cnt, s_warp, &tot_c);
        const uint32_t base_a = s_carry, base_c = s_carry_c;
        if (act) {
          s_act_mesh[base_a + ea] = (uint32_t)m;
          s_act_nmask[base_a + ea] = nm;
          s_act_prefix[base_a + ea] = base_c + ec;
          s_act_first[base_a + ea] = __ldg(a.mesh_first + m);
        }
        __syncthreads();
        if (tid == 0) { s_carry = base_a + tot_a; s_carry_c = base_c + tot_c; }
        __syncthreads();
      }
      if (tid == 0) s_act_prefix[s_carry] = s_carry_c;
      if (tid == 0) { s_n_act = s_carry; s_cur_g = g; }
      __syncthreads();
    }
    const uint32_t n_act = s_n_act;
    if (SMEM_BEST) {
      for (uint32_t r = tid; r < a.group_rays; r += TRAV_THREADS) s_best[r] = BEST_NONE;
    }
    __syncthreads();

    for (uint32_t tb = item.y; tb < item.z; tb += a.tile) {
      const uint32_t n_t = min((uint32_t)a.tile, item.z - tb);
      // ---- stage the tile's triangle spheres (contiguous per mesh, coalesced)
      for (uint32_t i = tid; i < (uint32_t)a.tile; i += TRAV_THREADS) {
        uint32_t nm = 0;
        if (i < n_t) {
          const uint32_t v = tb + i;
          uint32_t lo = 0, hi = n_act;   // largest q with prefix[q] <= v
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (s_act_prefix[mid] <= v) lo = mid; else hi = mid;
          }
          const uint32_t tri = s_act_first[lo] + (v - s_act_prefix[lo]);
          s_tri_sph[i] = __ldg(a.tri_sph + tri);
          s_tri_id[i] = tri;
          nm = s_act_nmask[lo];
        }
        s_tri_nmask[i] = nm;
      }
      __syncthreads();
      // ---- top level: dense (top node x triangle) Eq 9 tests
      {
        uint32_t* q = reinterpret_cast<uint32_t*>(smraw + L.off_q[Lv]);
        uint32_t tests = 0, hits = 0;
        for (uint32_t i0 = 0; i0 < (uint32_t)a.tile; i0 += TRAV_THREADS) {
          const uint32_t i = i0 + tid;
          const bool in = i < n_t;
          const float4 tgt = in ? s_tri_sph[i] : make_float4(0.f, 0.f, 0.f, 0.f);
          const uint32_t nm = in ? s_tri_nmask[i] : 0u;
          for (int j = 0; j < K; ++j) {
            const bool need = (nm >> j) & 1u;
            bool pass = false;
            if (need) {
              const float4 n0 = s_top[3 * j], n1 = s_top[3 * j + 1], n2 = s_top[3 * j + 2];
              pass = cull_ns(mk3(n0.x, n0.y, n0.z), n0.w, mk3(n1.x, n1.y, n1.z), n1.w, n2.x, tgt);
              ++tests;
              hits += pass;
            }
            push_warp(pass, ((uint32_t)j << TRI_BITS) | i, q, &s_qlen[Lv]);
          }
        }
        warp_count(ctr + CTR_TESTS + Lv, tests);
        warp_count(ctr + CTR_HITS + Lv, hits);
      }
      __syncthreads();
      // ---- drain: expand survivors level by level, then final tests
      for (;;) {
        for (int k = Lv; k >= 2; --k) {
          const uint32_t qk = s_qlen[k], qk1 = s_qlen[k - 1];
          const uint32_t cap = (k - 1 == Lv) ? (uint32_t)a.qtop_cap : (uint32_t)a.qcap;
          const uint32_t n_take = min(qk, (cap - qk1) / (uint32_t)B);
          if (n_take == 0) continue;
          const uint32_t* qin = reinterpret_cast<const uint32_t*>(smraw + L.off_q[k]) + (qk - n_take);
          uint32_t* qout = reinterpret_cast<uint32_t*>(smraw + L.off_q[k - 1]);
          const float4* tv = a.trav[k - 1];
          const size_t gbase = (size_t)g * a.per_group[k - 1];
          uint32_t tests = 0, hits = 0;
          const uint32_t n_work = n_take * (uint32_t)B;
          for (uint32_t w0 = 0; w0 < n_work; w0 += TRAV_THREADS) {
            const uint32_t w = w0 + tid;
            bool pass = false;
            uint32_t val = 0;
            if (w < n_work) {
              const uint32_t e = qin[w / B];
              const uint32_t child = (e >> TRI_BITS) * B + (w % B);
              const uint32_t tl = e & (MAX_TILE - 1);
              const float4 c0 = __ldg(tv + 3 * (gbase + child));
              if (c0.w >= 0.0f) {   // existing child
                const float4 c1 = __ldg(tv + 3 * (gbase + child) + 1), c2 = __ldg(tv + 3 * (gbase + child) + 2);
                pass = cull_ns(mk3(c0.x, c0.y, c0.z), c0.w, mk3(c1.x, c1.y, c1.z), c1.w, c2.x, s_tri_sph[tl]);
                ++tests;
                hits += pass;
                val = (child << TRI_BITS) | tl;
              }
            }
            push_warp(pass, val, qout, &s_qlen[k - 1]);
          }
          warp_count(ctr + CTR_TESTS + (k - 1), tests);
          warp_count(ctr + CTR_HITS + (k - 1), hits);
          __syncthreads();
          if (tid == 0) s_qlen[k] = qk - n_take;
          __syncthreads();
        }
        // final intersection tests of the bundle survivors
        const uint32_t q1 = s_qlen[1];
        {
          const uint32_t* qin = reinterpret_cast<const uint32_t*>(smraw + L.off_q[1]);
          const uint32_t n_work = q1 * (uint32_t)B0;
          const size_t rbase = (size_t)g * a.group_rays;
          uint32_t tests = 0, hits = 0;
          for (uint32_t w = tid; w < n_work; w += TRAV_THREADS) {
            const uint32_t e = qin[w / B0];
            const uint32_t rl = (e >> TRI_BITS) * B0 + (w % B0);
            const float4 r0 = __ldg(a.sorted_rays + 2 * (rbase + rl));
            if (r0.w < 0.0f) continue;   // padding ray
            const float4 r1 = __ldg(a.sorted_rays + 2 * (rbase + rl) + 1);
            const uint32_t tri = s_tri_id[e & (MAX_TILE - 1)];
            const float4 v0 = __ldg(a.tri_e + 3 * (size_t)tri), e1 = __ldg(a.tri_e + 3 * (size_t)tri + 1),
                         e2 = __ldg(a.tri_e + 3 * (size_t)tri + 2);
            ++tests;
            float th;
            if (mt_ns(mk3(r0.x, r0.y, r0.z), mk3(r1.x, r1.y, r1.z), r0.w, r1.w, mk3(v0.x, v0.y, v0.z),
                      mk3(e1.x, e1.y, e1.z), mk3(e2.x, e2.y, e2.z), &th)) {
              ++hits;
              const unsigned long long pk = pack_hit(th, tri);
              if (SMEM_BEST) atomicMin(s_best + rl, pk);
              else atomicMin(a.best + rbase + rl, pk);
            }
          }
          warp_count(ctr + CTR_FINAL_TESTS, tests);
          warp_count(ctr + CTR_FINAL_HITS, hits);
        }
        __syncthreads();
        if (tid == 0) s_qlen[1] = 0u;
        __syncthreads();
        bool more = false;
        for (int k = 2; k <= Lv; ++k) more |= s_qlen[k] != 0u;
        if (!more) break;
      }
      __syncthreads();
    }
    if (SMEM_BEST) {
      const size_t rbase = (size_t)g * a.group_rays;
      for (uint32_t r = tid; r < a.group_rays; r += TRAV_THREADS) {
        const unsigned long long b = s_best[r];
        if (b != BEST_NONE) atomicMin(a.best + rbase + r, b);
      }
    }
  }
  __syncthreads();
  for (uint32_t i = tid; i < MAX_SEG * CTR_STRIDE; i += TRAV_THREADS)
    if (s_ctr[i]) atomicAdd(a.counters + i, s_ctr[i]);
}

// ============================================================== K9
struct UnpackArgs {
  uint32_t r_lo, r_hi;          // padded sorted-ray range of this shard
  int32_t n_seg;
  uint32_t seg_pad_base[MAX_SEG + 1];
  uint32_t seg_n[MAX_SEG];
  const uint32_t* sorted_slot;
  const unsigned long long* best;
  int32_t* out_hit;
  float* out_t;
  unsigned long long* out_packed;
  unsigned long long* counters;
};

__global__ void __launch_bounds__(256) k_unpack(const UnpackArgs a) {
  __shared__ unsigned long long s_hit[MAX_SEG];
  if (threadIdx.x < MAX_SEG) s_hit[threadIdx.x] = 0ull;
  __syncthreads();
  const uint32_t i = a.r_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < a.r_hi) {
    int s = 0;
    for (int q = 1; q < a.n_seg; ++q) s = (i >= a.seg_pad_base[q]) ? q : s;
    if (i - a.seg_pad_base[s] < a.seg_n[s]) {
      const uint32_t slot = __ldg(a.sorted_slot + i);
      const unsigned long long b = __ldg(a.best + i);
      const bool hit = b != BEST_NONE;
      if (a.out_packed) {
        a.out_packed[slot] = hit ? b : PACK_MISS;
      } else {
        a.out_hit[slot] = hit ? (int32_t)(uint32_t)(b & 0xFFFFFFFFull) : -1;
        a.out_t[slot] = hit ? __uint_as_float((uint32_t)(b >> 32)) : __int_as_float(0x7f800000);
      }
      if (hit) atomicAdd(&s_hit[s], 1ull);
    }
  }
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
