// k_raygen.cuh — K1: secondary ray generation + type-specific hash + trimming
// in one pass (§3.3.2, Figs 2-4).
//
// One thread per (slot, item): the slot is decoded to (type, light, pixel)
// (canonical slot order, crsh.h), the ray is generated from the G-buffer and
// written as a 32-byte record (o.xyz, tmin | d.xyz, tmax) at rays[slot], its
// 32-bit key computed (R6 layout or Z-order), and the non-empty slots are
// compacted in slot order. The paper's head-flag array + inclusive scan +
// shift (Fig 4) is realised as a single-pass decoupled look-back scan: the
// flags never touch HBM, and the compaction order is exactly slot order
// (deterministic), which the stable sort downstream relies on.
#pragma once
#include "common.cuh"
#include "numspec.cuh"

namespace crsh {

struct RaygenArgs {
  int32_t P;
  const float* pos;
  const float* nrm;
  const int32_t* mat;
  const float* materials;
  int32_t n_mat;
  float eye[3];
  const float* dir;                   // optional [3][P] incident directions (Whitted bounce > 0)
  const float4* in_rays;              // ray-batch mode (crsh_trace_rays): slot i = {o, tmin}, {d, tmax}
  float lights[16 * 3];
  int32_t n_lights;
  int32_t zorder;
  float box_min[3], box_ext[3];
  float eps_t;
  uint32_t n_slots;
  int32_t n_seg;
  int32_t seg_type[MAX_SEG];          // 0 = SH, 1 = RE, 2 = RR
  uint32_t seg_slot_start[MAX_SEG + 1];
  float4* rays;                       // [n_slots][2]
  uint32_t* keys_c;                   // compacted keys
  uint32_t* vals_c;                   // compacted slot ids
  int32_t* out_hit;                   // optional: -2 / +inf for empty slots
  float* out_t;
  unsigned long long* out_packed;     // optional: sentinel for every slot
  PeerOut peer;                       // optional (n > 0): sentinel for every EMPTY slot, in every destination
  unsigned long long* status;         // look-back, one word per tile
  uint32_t* ticket;
  FrameDesc* fd;                      // out: seg_comp_start[0..n_seg]
};

// One G-buffer pixel: material and position, loaded once per pixel.
struct Pix {
  int m;
  f3 x;
};
__device__ __forceinline__ bool load_pix(const RaygenArgs& a, uint32_t p, Pix& px) {
  px.m = __ldg(a.mat + p);
  if (px.m < 0 || px.m >= a.n_mat) return false;
  const size_t P = (size_t)a.P;
  px.x = mk3(__ldg(a.pos + p), __ldg(a.pos + P + p), __ldg(a.pos + 2 * P + p));
  return true;
}
// shadow ray of light l, origin inverted to the light
__device__ __forceinline__ void gen_sh(const RaygenArgs& a, const Pix& px, uint32_t l, float4& r0, float4& r1,
                                       uint32_t& key) {
  const f3 L = mk3(a.lights[3 * l], a.lights[3 * l + 1], a.lights[3 * l + 2]);
  const f3 v = px.x - L;
  const float len = len3(v);
  const f3 d = len > 0.0f ? v * (1.0f / len) : mk3(0.0f, 0.0f, 1.0f);
  r0 = make_float4(L.x, L.y, L.z, a.eps_t);
  r1 = make_float4(d.x, d.y, d.z, len - a.eps_t);
  key = hash_shadow_ns(l, d, a.zorder != 0);
}
// reflection (type 1) / refraction (type 2) ray of pixel p; false if the
// material emits none (or total internal reflection). VALID_ONLY: the same
// decision without the ray (the pixel-major generator's counting pass).
template <bool VALID_ONLY>
__device__ __forceinline__ bool gen_bounce(const RaygenArgs& a, const Pix& px, uint32_t p, int type, float4& r0,
                                           float4& r1, uint32_t& key) {
  const int m = px.m;
  const size_t P = (size_t)a.P;
  const float refl = __ldg(a.materials + 3 * m), trans = __ldg(a.materials + 3 * m + 1);
  if (type == 1 && !(refl > 0.0f)) return false;     // reflection iff reflectivity > 0
  if (type == 2 && !(trans > 0.0f)) return false;    // refraction iff transmissivity > 0 (and no TIR)
  if (VALID_ONLY && type == 1) return true;
  const f3 i = a.dir ? mk3(__ldg(a.dir + p), __ldg(a.dir + P + p), __ldg(a.dir + 2 * P + p))
                     : norm3(px.x - mk3(a.eye[0], a.eye[1], a.eye[2]));
  f3 n = mk3(__ldg(a.nrm + p), __ldg(a.nrm + P + p), __ldg(a.nrm + 2 * P + p));
  f3 d;
  if (type == 1) {
    if (dot3(i, n) > 0.0f) n = neg3(n);
    const float k2 = 2.0f * dot3(i, n);
    d = norm3(mk3(__fmaf_rn(-k2, n.x, i.x), __fmaf_rn(-k2, n.y, i.y), __fmaf_rn(-k2, n.z, i.z)));
  } else {   // Snell
    const float ior = __ldg(a.materials + 3 * m + 2);
    float c = -dot3(i, n), eta;
    if (c < 0.0f) { n = neg3(n); c = -c; eta = ior; } else { eta = 1.0f / ior; }
    const float k = 1.0f - (eta * eta) * (1.0f - c * c);
    if (k < 0.0f) return false;
    if (VALID_ONLY) return true;
    const float t1 = eta * c - sqrtf(k);
    d = norm3(mk3(__fmaf_rn(eta, i.x, t1 * n.x), __fmaf_rn(eta, i.y, t1 * n.y), __fmaf_rn(eta, i.z, t1 * n.z)));
  }
  r0 = make_float4(px.x.x, px.x.y, px.x.z, a.eps_t);
  r1 = make_float4(d.x, d.y, d.z, __int_as_float(0x7f800000));
  key = hash_bounce_ns(px.x, d, a.box_min, a.box_ext, a.zorder != 0);
  return true;
}

__device__ __forceinline__ bool gen_ray(const RaygenArgs& a, uint32_t slot, float4& r0, float4& r1, uint32_t& key) {
  if (a.in_rays) {   // given rays (primary pass, external batches): bounce-type hash, empty iff !(tmax > tmin)
    r0 = __ldg(a.in_rays + 2 * (size_t)slot);
    r1 = __ldg(a.in_rays + 2 * (size_t)slot + 1);
    if (!(r1.w > r0.w)) return false;
    key = hash_bounce_ns(mk3(r0.x, r0.y, r0.z), mk3(r1.x, r1.y, r1.z), a.box_min, a.box_ext, a.zorder != 0);
    return true;
  }
  int s = 0;
  while (s + 1 < a.n_seg && slot >= a.seg_slot_start[s + 1]) ++s;
  const uint32_t local = slot - a.seg_slot_start[s];
  const int type = a.seg_type[s];
  uint32_t p = local, l = 0;
  if (type == 0) {
    l = local / (uint32_t)a.P;
    p = local - l * (uint32_t)a.P;
  }
  Pix px;
  if (!load_pix(a, p, px)) return false;
  if (type == 0) {
    gen_sh(a, px, l, r0, r1, key);
    return true;
  }
  return gen_bounce<false>(a, px, p, type, r0, r1, key);
}

__global__ void __launch_bounds__(SCAN_THREADS) k_raygen(const RaygenArgs a) {
  __shared__ uint32_t s_tile, s_prefix;
  __shared__ uint32_t s_cnt[SCAN_ITEMS * 8], s_excl[SCAN_ITEMS * 8];
  if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  uint32_t key[SCAN_ITEMS], ballot[SCAN_ITEMS];
#pragma unroll
  for (int it = 0; it < SCAN_ITEMS; ++it) {
    const uint32_t slot = tile * SCAN_TILE + it * SCAN_THREADS + threadIdx.x;
    bool ok = false;
    uint32_t k = 0;
    if (slot < a.n_slots) {
      float4 r0, r1;
      ok = gen_ray(a, slot, r0, r1, k);
      if (ok) {
        a.rays[2 * (size_t)slot] = r0;
        a.rays[2 * (size_t)slot + 1] = r1;
      } else if (a.out_hit) {
        a.out_hit[slot] = -2;
        a.out_t[slot] = __int_as_float(0x7f800000);
      }
      if (a.out_packed) a.out_packed[slot] = 0x7FFFFFFFFFFFFFFFull;
      if (a.peer.n && !ok) a.peer.store(slot, 0x7FFFFFFFFFFFFFFFull);   // rayed slots: written by their owner only
    }
    key[it] = k;
    ballot[it] = __ballot_sync(CRSH_FULL, ok);
    if (lane == 0) s_cnt[it * 8 + warp] = __popc(ballot[it]);
  }
  __syncthreads();
  tile_scan_lookback_block(s_cnt, s_excl, &s_prefix, a.status, (int)tile);
  __syncthreads();
  const uint32_t prefix = s_prefix;
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int it = 0; it < SCAN_ITEMS; ++it) {
    const uint32_t slot = tile * SCAN_TILE + it * SCAN_THREADS + threadIdx.x;
    const uint32_t pos = prefix + s_excl[it * 8 + warp] + __popc(ballot[it] & lt);
    if ((ballot[it] >> lane) & 1u) {
      CRSH_CHECK(pos < a.n_slots, 101);
      a.keys_c[pos] = key[it];
      a.vals_c[pos] = slot;
    }
    for (int s = 0; s < a.n_seg; ++s)
      if (slot == a.seg_slot_start[s] && slot < a.n_slots) a.fd->seg_comp_start[s] = pos;
  }
  const uint32_t n_tiles = (a.n_slots + SCAN_TILE - 1) / SCAN_TILE;
  if (tile == n_tiles - 1 && threadIdx.x == 0) {
    const uint32_t total = prefix + [&] {
      uint32_t t = 0;
      for (int q = 0; q < SCAN_ITEMS * 8; ++q) t += s_cnt[q];
      return t;
    }();
    a.fd->seg_comp_start[a.n_seg] = total;
  }
}

}  // namespace crsh

namespace crsh {

// ============================================================== K1, pixel-major (G-buffer frames)
// The same rays, keys and compaction as k_raygen, computed per PIXEL instead
// of per slot: a pixel's G-buffer entry is read once for its L shadow rays
// and its reflection / refraction rays (the slot-major kernel decoded every
// slot -- an integer division -- and re-read the pixel L + 2 times). The
// compacted position of a ray is known without a look-back: in slot order a
// shadow ray of light l of pixel p sits at l * V_sh + rank_sh(p) (a pixel
// emits a shadow ray for every light or none, R4), a reflection ray at the
// segment start + rank_re(p), a refraction ray at its segment start +
// rank_rr(p), where V are the frame's counts and rank the count of emitting
// pixels before p. K1a counts per tile, K1b sums the preceding tiles' counts
// (ranks) and generates. Compaction order = slot order, exactly as k_raygen.
// PX_ITEMS pixels per thread: 8 (2048-pixel tiles) for large frames, 2
// (512-pixel tiles) below 2^20 pixels, where 2048-pixel tiles are fewer than
// one wave of CTAs (cfg2: 128 tiles on 148 SMs)
constexpr uint32_t PX_SMALL_FRAME = 1u << 20;
__host__ __device__ constexpr uint32_t px_tile(int items) { return SCAN_THREADS * (uint32_t)items; }

struct PxArgs {
  RaygenArgs rg;
  int32_t seg_of_type[3];        // segment index of SH / RE / RR, -1 if absent
  uint32_t* tile_cnt;            // [3][n_tiles]: emitting pixels per tile and type
  uint32_t* total;               // [3]: emitting pixels per type (zeroed per frame)
};

__device__ __forceinline__ void px_flags(const PxArgs& a, uint32_t p, bool& sh, bool& re, bool& rr) {
  Pix px;
  sh = re = rr = false;
  if (!load_pix(a.rg, p, px)) return;
  float4 r0, r1;
  uint32_t key;
  sh = a.seg_of_type[0] >= 0 && a.rg.n_lights > 0;
  re = a.seg_of_type[1] >= 0 && gen_bounce<true>(a.rg, px, p, 1, r0, r1, key);
  rr = a.seg_of_type[2] >= 0 && gen_bounce<true>(a.rg, px, p, 2, r0, r1, key);
}

// K1a: emitting pixels per tile and type
template <int PX_ITEMS>
__global__ void __launch_bounds__(SCAN_THREADS) k_raygen_count(const PxArgs a) {
  constexpr uint32_t PX_TILE = px_tile(PX_ITEMS);
  __shared__ uint32_t s_c[3];
  if (threadIdx.x < 3) s_c[threadIdx.x] = 0u;
  __syncthreads();
  uint32_t c[3] = {0u, 0u, 0u};
  for (int it = 0; it < PX_ITEMS; ++it) {
    const uint32_t p = blockIdx.x * PX_TILE + it * SCAN_THREADS + threadIdx.x;
    bool f[3] = {false, false, false};
    if (p < (uint32_t)a.rg.P) px_flags(a, p, f[0], f[1], f[2]);
    for (int t = 0; t < 3; ++t) c[t] += __popc(__ballot_sync(CRSH_FULL, f[t]));
  }
  if (lane_id() == 0)
    for (int t = 0; t < 3; ++t) atomicAdd(&s_c[t], c[t]);
  __syncthreads();
  if (threadIdx.x < 3) {
    a.tile_cnt[threadIdx.x * gridDim.x + blockIdx.x] = s_c[threadIdx.x];
    atomicAdd(a.total + threadIdx.x, s_c[threadIdx.x]);
  }
}

// K1b: ranks from the preceding tiles' counts, then every ray of the tile's pixels
template <int PX_ITEMS>
__global__ void __launch_bounds__(SCAN_THREADS) k_raygen_px(const PxArgs a) {
  constexpr uint32_t PX_TILE = px_tile(PX_ITEMS);
  __shared__ uint32_t s_cnt[3][PX_ITEMS * 8], s_excl[3][PX_ITEMS * 8];
  __shared__ uint32_t s_red[3][SCAN_THREADS / 32];
  const RaygenArgs& g = a.rg;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, lt = lanemask_lt();
  const uint32_t P = (uint32_t)g.P, tile = blockIdx.x;
  // frame counts and segment starts (slot order: SH of all lights, RE, RR)
  const uint32_t L = (uint32_t)g.n_lights;
  const uint32_t vt[3] = {__ldcg(a.total), __ldcg(a.total + 1), __ldcg(a.total + 2)};
  uint32_t seg_start[3] = {0u, 0u, 0u};
  {
    uint32_t acc = 0;
    for (int s = 0; s < g.n_seg; ++s) {
      const int t = g.seg_type[s];
      for (int q = 0; q < 3; ++q) seg_start[q] = (q == t) ? acc : seg_start[q];
      acc += (t == 0) ? L * vt[0] : vt[t];
      if (tile == 0 && threadIdx.x == 0) g.fd->seg_comp_start[s + 1] = acc;
    }
    if (tile == 0 && threadIdx.x == 0) g.fd->seg_comp_start[0] = 0u;
  }
  // emitting pixels of the preceding tiles, per type
  uint32_t pre[3] = {0u, 0u, 0u};
  for (uint32_t q = threadIdx.x; q < tile; q += SCAN_THREADS)
    for (int t = 0; t < 3; ++t) pre[t] += __ldcg(a.tile_cnt + t * gridDim.x + q);
  for (int t = 0; t < 3; ++t) {
    const uint32_t v = __reduce_add_sync(CRSH_FULL, pre[t]);
    if (lane == 0) s_red[t][warp] = v;
  }
  // this tile's flags (bit 3 it + t of `fl`) and their per-warp ballots
  // (shared memory: the generation loop below is not unrolled, and
  // runtime-indexed register arrays would live in local memory)
  __shared__ uint32_t s_bal[3][PX_ITEMS][SCAN_THREADS / 32];
  uint32_t fl = 0;
#pragma unroll
  for (int it = 0; it < PX_ITEMS; ++it) {
    const uint32_t p = tile * PX_TILE + it * SCAN_THREADS + threadIdx.x;
    bool f0 = false, f1 = false, f2 = false;
    if (p < P) px_flags(a, p, f0, f1, f2);
    fl |= (f0 ? 1u : 0u) << (3 * it) | (f1 ? 2u : 0u) << (3 * it) | (f2 ? 4u : 0u) << (3 * it);
    const uint32_t b0 = __ballot_sync(CRSH_FULL, f0), b1 = __ballot_sync(CRSH_FULL, f1), b2 = __ballot_sync(CRSH_FULL, f2);
    if (lane == 0) {
      s_bal[0][it][warp] = b0; s_bal[1][it][warp] = b1; s_bal[2][it][warp] = b2;
      s_cnt[0][it * 8 + warp] = __popc(b0); s_cnt[1][it * 8 + warp] = __popc(b1); s_cnt[2][it * 8 + warp] = __popc(b2);
    }
  }
  __syncthreads();
  if (warp < 3) {   // exclusive scan of the PX_ITEMS * 8 (item, warp) counts of type `warp`
    constexpr int PER = PX_ITEMS * 8 / 32 > 0 ? PX_ITEMS * 8 / 32 : 1;   // entries per lane (2 or 1 with 4 unused lanes)
    uint32_t x[PER], sum = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = (int)lane * PER + q;
      x[q] = e < PX_ITEMS * 8 ? s_cnt[warp][e] : 0u;
      sum += x[q];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(CRSH_FULL, incl, o);
      if ((int)lane >= o) incl += y;
    }
    uint32_t run = incl - sum;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = (int)lane * PER + q;
      if (e < PX_ITEMS * 8) s_excl[warp][e] = run;
      run += x[q];
    }
  }
  __syncthreads();
  uint32_t base[3];
  for (int t = 0; t < 3; ++t) {
    uint32_t b = 0;
    for (int w = 0; w < SCAN_THREADS / 32; ++w) b += s_red[t][w];
    base[t] = b;
  }
  // generate: shadow rays of every light, then the bounce rays
#pragma unroll 1
  for (int it = 0; it < PX_ITEMS; ++it) {
    const uint32_t p = tile * PX_TILE + it * SCAN_THREADS + threadIdx.x;
    if (p >= P) break;
    Pix px;
    if (!load_pix(g, p, px)) px.m = -1;   // no primary hit: every slot of the pixel is empty
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      const int s = a.seg_of_type[t];
      if (s < 0) continue;
      const bool emits = (fl >> (3 * it + t)) & 1u;
      const uint32_t rank = base[t] + s_excl[t][it * 8 + warp] + __popc(s_bal[t][it][warp] & lt);
      const uint32_t n_r = (t == 0) ? L : 1u;
      for (uint32_t l = 0; l < n_r; ++l) {
        const uint32_t slot = g.seg_slot_start[s] + l * P + p;
        float4 r0, r1;
        uint32_t key = 0;
        bool ok = false;
        if (emits) {
          if (t == 0) { gen_sh(g, px, l, r0, r1, key); ok = true; }
          else ok = gen_bounce<false>(g, px, p, t, r0, r1, key);
          CRSH_CHECK(ok, 103);   // the counting pass decided with the same code
        }
        if (ok) {
          g.rays[2 * (size_t)slot] = r0;
          g.rays[2 * (size_t)slot + 1] = r1;
          const uint32_t pos = seg_start[t] + ((t == 0) ? l * vt[0] : 0u) + rank;
          CRSH_CHECK(pos < g.n_slots, 102);
          g.keys_c[pos] = key;
          g.vals_c[pos] = slot;
        } else if (g.out_hit) {
          g.out_hit[slot] = -2;
          g.out_t[slot] = __int_as_float(0x7f800000);
        }
        if (g.out_packed) g.out_packed[slot] = 0x7FFFFFFFFFFFFFFFull;
        if (g.peer.n && !ok) g.peer.store(slot, 0x7FFFFFFFFFFFFFFFull);
      }
    }
  }
}

}  // namespace crsh
