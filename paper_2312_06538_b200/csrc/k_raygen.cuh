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
  const int m = __ldg(a.mat + p);
  if (m < 0 || m >= a.n_mat) return false;
  const size_t P = (size_t)a.P;
  const f3 x = mk3(__ldg(a.pos + p), __ldg(a.pos + P + p), __ldg(a.pos + 2 * P + p));
  if (type == 0) {   // shadow ray, origin inverted to the light
    const f3 L = mk3(a.lights[3 * l], a.lights[3 * l + 1], a.lights[3 * l + 2]);
    const f3 v = x - L;
    const float len = len3(v);
    const f3 d = len > 0.0f ? v * (1.0f / len) : mk3(0.0f, 0.0f, 1.0f);
    r0 = make_float4(L.x, L.y, L.z, a.eps_t);
    r1 = make_float4(d.x, d.y, d.z, len - a.eps_t);
    key = hash_shadow_ns(l, d, a.zorder != 0);
    return true;
  }
  const float refl = __ldg(a.materials + 3 * m), trans = __ldg(a.materials + 3 * m + 1);
  const f3 i = a.dir ? mk3(__ldg(a.dir + p), __ldg(a.dir + P + p), __ldg(a.dir + 2 * P + p))
                     : norm3(x - mk3(a.eye[0], a.eye[1], a.eye[2]));
  f3 n = mk3(__ldg(a.nrm + p), __ldg(a.nrm + P + p), __ldg(a.nrm + 2 * P + p));
  f3 d;
  if (type == 1) {   // reflection, iff reflectivity > 0
    if (!(refl > 0.0f)) return false;
    if (dot3(i, n) > 0.0f) n = neg3(n);
    const float k2 = 2.0f * dot3(i, n);
    d = norm3(mk3(__fmaf_rn(-k2, n.x, i.x), __fmaf_rn(-k2, n.y, i.y), __fmaf_rn(-k2, n.z, i.z)));
  } else {           // refraction (Snell), iff transmissivity > 0 and no TIR
    if (!(trans > 0.0f)) return false;
    const float ior = __ldg(a.materials + 3 * m + 2);
    float c = -dot3(i, n), eta;
    if (c < 0.0f) { n = neg3(n); c = -c; eta = ior; } else { eta = 1.0f / ior; }
    const float k = 1.0f - (eta * eta) * (1.0f - c * c);
    if (k < 0.0f) return false;
    const float t1 = eta * c - sqrtf(k);
    d = norm3(mk3(__fmaf_rn(eta, i.x, t1 * n.x), __fmaf_rn(eta, i.y, t1 * n.y), __fmaf_rn(eta, i.z, t1 * n.z)));
  }
  r0 = make_float4(x.x, x.y, x.z, a.eps_t);
  r1 = make_float4(d.x, d.y, d.z, __int_as_float(0x7f800000));
  key = hash_bounce_ns(x, d, a.box_min, a.box_ext, a.zorder != 0);
  return true;
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
