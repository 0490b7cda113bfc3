// k_build.cuh — scene preparation (triangle data + padded minimal spheres,
// P:173, R1, R2) and the bottom-up hierarchy build (§3.3.6):
// K5 gathers the sorted rays into a contiguous array and builds the first
// level (sphere: Eqs 7-8 in balanced pairwise order, R9; cone: Eqs 1-4
// sequentially in sorted order), K6 builds one upper level (Eqs 5-8).
//
// Sorted rays live in a padded layout: every segment starts at a multiple of
// the traversal group span, so node j of level k covers rays
// [j*B0*B^(k-1), (j+1)*B0*B^(k-1)) uniformly; padding rays have tmin = -1 and
// padding nodes r = -1 ("empty"), and neither is tested nor counted.
#pragma once
#include "common.cuh"
#include "numspec.cuh"

namespace crsh {

// ------------------------------------------------------------ scene prep
__device__ __forceinline__ void dfinalize(double cx, double cy, double cz, const double* px, const double* py,
                                          const double* pz, float pad, float4* out) {
  const float fx = (float)cx, fy = (float)cy, fz = (float)cz;
  double r2 = 0.0;
  for (int i = 0; i < 3; ++i) {
    const double dx = px[i] - (double)fx, dy = py[i] - (double)fy, dz = pz[i] - (double)fz;
    r2 = fmax(r2, dx * dx + dy * dy + dz * dz);
  }
  const double r = sqrt(r2);
  float rf = (float)r;
  if ((double)rf < r) rf = nextafterf(rf, __int_as_float(0x7f800000));
  *out = make_float4(fx, fy, fz, rf + pad);
}

// Per triangle: v0, e1 = v1 - v0, e2 = v2 - v0 (3 float4) and the minimal
// sphere of its vertices (longest-edge midpoint when right/obtuse, else the
// circumcentre), centre rounded to float, radius = max distance from that
// centre rounded up, plus pad.
__global__ void k_tri_prep(const float* __restrict__ tris, int64_t M, float pad, float4* __restrict__ tri_e,
                           float4* __restrict__ tri_sph) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M; t += (int64_t)gridDim.x * blockDim.x) {
    const float* v = tris + 9 * t;
    float f[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) f[i] = v[i];
    tri_e[3 * t] = make_float4(f[0], f[1], f[2], 0.f);
    tri_e[3 * t + 1] = make_float4(f[3] - f[0], f[4] - f[1], f[5] - f[2], 0.f);
    tri_e[3 * t + 2] = make_float4(f[6] - f[0], f[7] - f[1], f[8] - f[2], 0.f);
    const double ax = f[0], ay = f[1], az = f[2], bx = f[3], by = f[4], bz = f[5], cx = f[6], cy = f[7], cz = f[8];
    const double abx = bx - ax, aby = by - ay, abz = bz - az;
    const double acx = cx - ax, acy = cy - ay, acz = cz - az;
    const double bcx = cx - bx, bcy = cy - by, bcz = cz - bz;
    double ox, oy, oz;
    if (abx * acx + aby * acy + abz * acz <= 0.0) {                 // angle at a >= 90
      ox = (bx + cx) * 0.5; oy = (by + cy) * 0.5; oz = (bz + cz) * 0.5;
    } else if ((-abx) * bcx + (-aby) * bcy + (-abz) * bcz <= 0.0) { // at b
      ox = (ax + cx) * 0.5; oy = (ay + cy) * 0.5; oz = (az + cz) * 0.5;
    } else if (acx * bcx + acy * bcy + acz * bcz <= 0.0) {          // at c
      ox = (ax + bx) * 0.5; oy = (ay + by) * 0.5; oz = (az + bz) * 0.5;
    } else {                                                        // circumcentre
      const double nx = aby * acz - abz * acy, ny = abz * acx - abx * acz, nz = abx * acy - aby * acx;
      const double den = 2.0 * (nx * nx + ny * ny + nz * nz);
      const double ac2 = acx * acx + acy * acy + acz * acz, ab2 = abx * abx + aby * aby + abz * abz;
      // (n x ab) * |ac|^2 + (ac x n) * |ab|^2
      const double qx = (ny * abz - nz * aby) * ac2 + (acy * nz - acz * ny) * ab2;
      const double qy = (nz * abx - nx * abz) * ac2 + (acz * nx - acx * nz) * ab2;
      const double qz = (nx * aby - ny * abx) * ac2 + (acx * ny - acy * nx) * ab2;
      const double inv = 1.0 / den;
      ox = ax + qx * inv; oy = ay + qy * inv; oz = az + qz * inv;
    }
    const double px[3] = {ax, bx, cx}, py[3] = {ay, by, cy}, pz[3] = {az, bz, cz};
    dfinalize(ox, oy, oz, px, py, pz, pad, &tri_sph[t]);
  }
}

// Object sphere-tree clusters (CRSH_F_OBJTREE, NEXT-4, reading O1): cluster i
// covers positions [rng.x, rng.y) of the cluster order; its sphere is centred
// at the midpoint of its vertices' bounding box (double, rounded to float),
// radius = the largest distance from that float centre (double, rounded up),
// plus pad. Also the triangle spheres permuted into cluster order.
__global__ void k_cluster_prep(const float* __restrict__ tris, const int32_t* __restrict__ order,
                               const uint2* __restrict__ rng, int64_t n_clusters, float pad, float4* __restrict__ cl_sph) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_clusters; c += (int64_t)gridDim.x * blockDim.x) {
    const uint2 r = rng[c];
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (uint32_t i = r.x; i < r.y; ++i) {
      const float* v = tris + 9 * (size_t)order[i];
      for (int k = 0; k < 9; ++k) {
        const double q = (double)v[k];
        lo[k % 3] = fmin(lo[k % 3], q);
        hi[k % 3] = fmax(hi[k % 3], q);
      }
    }
    const float fx = (float)((lo[0] + hi[0]) * 0.5), fy = (float)((lo[1] + hi[1]) * 0.5), fz = (float)((lo[2] + hi[2]) * 0.5);
    double r2 = 0.0;
    for (uint32_t i = r.x; i < r.y; ++i) {
      const float* v = tris + 9 * (size_t)order[i];
      for (int k = 0; k < 3; ++k) {
        const double dx = (double)v[3 * k] - (double)fx, dy = (double)v[3 * k + 1] - (double)fy,
                     dz = (double)v[3 * k + 2] - (double)fz;
        r2 = fmax(r2, dx * dx + dy * dy + dz * dz);
      }
    }
    const double rd = sqrt(r2);
    float rf = (float)rd;
    if ((double)rf < rd) rf = nextafterf(rf, __int_as_float(0x7f800000));
    cl_sph[c] = make_float4(fx, fy, fz, rf + pad);
  }
}
__global__ void k_permute_sph(const float4* __restrict__ tri_sph, const int32_t* __restrict__ order, int64_t M,
                              float4* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = tri_sph[order[i]];
}
// K8's child prefilter spheres (not the paper's arithmetic; k_traverse.cuh
// cull_pf): per cluster, the cluster sphere's centre and a radius that
// contains every triangle sphere of the cluster, |P_i - C| + R_i in double,
// rounded up to float. Runs after k_permute_sph (tri_sph_ord).
__global__ void k_cluster_pf(const float4* __restrict__ cl_sph, const float4* __restrict__ tri_sph_ord,
                             const uint2* __restrict__ rng, int64_t n_clusters, float4* __restrict__ cl_pf) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n_clusters; c += (int64_t)gridDim.x * blockDim.x) {
    const float4 C = cl_sph[c];
    const uint2 r = rng[c];
    double R = 0.0;
    for (uint32_t i = r.x; i < r.y; ++i) {
      const float4 t = tri_sph_ord[i];
      const double dx = (double)t.x - (double)C.x, dy = (double)t.y - (double)C.y, dz = (double)t.z - (double)C.z;
      R = fmax(R, sqrt(dx * dx + dy * dy + dz * dz) + (double)t.w);
    }
    float rf = (float)R;
    if ((double)rf < R) rf = nextafterf(rf, __int_as_float(0x7f800000));
    cl_pf[c] = make_float4(C.x, C.y, C.z, rf);
  }
}

// ------------------------------------------------------------ nodes
// so: (leaves) every ray of the bundle starts at the node centre, bit for bit
__device__ __forceinline__ void store_node(float4* nodes, float4* trav, size_t j, const NodeV& n, bool so = false) {
  nodes[2 * j] = make_float4(n.c.x, n.c.y, n.c.z, n.r);
  nodes[2 * j + 1] = make_float4(n.a.x, n.a.y, n.a.z, n.alpha);
  // traversal layout: {c, d}, {a, tan(alpha)}, {sec(alpha), 0, 0, 0};
  // wide cones (alpha >= pi/2): a = 0, tan = sec = 1e30 (pass-all, numspec.cuh)
  float tn = 0.f, sc = 0.f;
  f3 a = n.a;
  if (n.r >= 0.0f) {
    tansec_ns(n.alpha, &tn, &sc);
    if (n.alpha >= CRSH_PI2_F) a = mk3(0.f, 0.f, 0.f);
  }
  trav[3 * j] = make_float4(n.c.x, n.c.y, n.c.z, n.r);
  trav[3 * j + 1] = make_float4(a.x, a.y, a.z, tn);
  trav[3 * j + 2] = make_float4(sc, so ? 1.0f : 0.0f, 0.f, 0.f);
}
__device__ __forceinline__ NodeV load_node(const float4* nodes, size_t j) {
  const float4 p = nodes[2 * j], q = nodes[2 * j + 1];
  NodeV n;
  n.c = mk3(p.x, p.y, p.z); n.r = p.w; n.a = mk3(q.x, q.y, q.z); n.alpha = q.w;
  return n;
}

struct LeafArgs {
  const FrameDesc* fd;                    // level_n[1], seg_pad_base, seg_n
  int32_t n_seg;
  const uint32_t* sorted_slot;
  const float4* rays;                     // [slots][2]
  float4* sorted_rays;                    // [Np][2]; written only if write_sorted
  int32_t write_sorted;                   // 0: K8 gathers its groups' rays by sorted_slot itself (groups in smem)
  float4* nodes;                          // level 1, paper layout [2 per node]
  float4* trav;                           // level 1, traversal layout [3 per node]
};

// K5: one thread per bundle (leaf). The sphere is the balanced pairwise tree
// ((0,1),(2,3)),((4,5),(6,7)) of radius-0 origin spheres (R9), evaluated with
// compile-time indices (registers); missing rays pass through (r = -1).
#ifndef CRSH_LEAVES_PREFETCH
#define CRSH_LEAVES_PREFETCH 1
#endif
template <int B0>
__global__ void __launch_bounds__(128) k_leaves(const LeafArgs a) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.fd->level_n[1]) return;
  const uint32_t p0 = j * B0;
  int s = 0;
  for (int q = 1; q < a.n_seg; ++q) s = (p0 >= a.fd->seg_pad_base[q]) ? q : s;
  const uint32_t local = p0 - a.fd->seg_pad_base[s];
  const uint32_t ns = a.fd->seg_n[s];
  const int real = (int)min((uint32_t)B0, ns > local ? ns - local : 0u);
  f3 sc[B0];
  float sr[B0];
  f3 x = mk3(0.f, 0.f, 1.f);
  float phi = 0.0f;
  bool same = true;   // all real rays share the first ray's origin, bit for bit
  f3 o0 = mk3(0.f, 0.f, 0.f);
#if CRSH_LEAVES_PREFETCH
  // every gather of the bundle is issued before the first store (B0 <= 16:
  // the bundle's rays in registers), so the 2 B0 ray loads are in flight
  // together instead of one load-store round trip per ray (A/B: build stage
  // cfg2 24.6 -> 22.5 us, cfg4 224 -> 218 us)
  constexpr int PF = B0 <= 16 ? B0 : 1;
  float4 pr0[PF], pr1[PF];
  if (B0 <= 16) {
    uint32_t slot[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) slot[i] = i < real ? __ldg(a.sorted_slot + p0 + i) : 0u;
#pragma unroll
    for (int i = 0; i < PF; ++i) {
      if (i < real) {
        pr0[i] = __ldg(a.rays + 2 * (size_t)slot[i]);
        pr1[i] = __ldg(a.rays + 2 * (size_t)slot[i] + 1);
      }
    }
  }
#endif
#pragma unroll
  for (int i = 0; i < B0; ++i) {
    float4 r0, r1;
    if (i < real) {
#if CRSH_LEAVES_PREFETCH
      if (B0 <= 16) {
        r0 = pr0[i < PF ? i : 0];
        r1 = pr1[i < PF ? i : 0];
      } else
#endif
      {
        const uint32_t slot = __ldg(a.sorted_slot + p0 + i);
        r0 = __ldg(a.rays + 2 * (size_t)slot);
        r1 = __ldg(a.rays + 2 * (size_t)slot + 1);
      }
    } else {
      r0 = make_float4(0.f, 0.f, 0.f, -1.0f);   // padding ray: tmin = -1
      r1 = make_float4(0.f, 0.f, 1.f, -1.0f);
    }
    if (a.write_sorted) {
      a.sorted_rays[2 * (size_t)(p0 + i)] = r0;
      a.sorted_rays[2 * (size_t)(p0 + i) + 1] = r1;
    }
    sc[i] = mk3(r0.x, r0.y, r0.z);
    sr[i] = (i < real) ? 0.0f : -1.0f;
    if (i == 0) o0 = sc[0];
    if (i > 0 && i < real)
      same = same && __float_as_uint(r0.x) == __float_as_uint(sc[0].x) && __float_as_uint(r0.y) == __float_as_uint(sc[0].y) &&
             __float_as_uint(r0.z) == __float_as_uint(sc[0].z);
    if (i < real) {
      const f3 d = mk3(r1.x, r1.y, r1.z);
      if (i == 0) { x = d; phi = 0.0f; }     // leaves start as radius 0 / angle 0
      else cone_grow_ns(&x, &phi, d);        // Eqs 1-4 in sorted order
    }
  }
#pragma unroll
  for (int w = 1; w < B0; w *= 2) {
#pragma unroll
    for (int i = 0; i < B0; i += 2 * w) {
      f3 c2;
      float r2;
      sphere_union_ns(sc[i], sr[i], sc[i + w], sr[i + w], &c2, &r2);   // Eqs 7-8
      sc[i] = c2; sr[i] = r2;
    }
  }
  NodeV n;
  if (real == 0) {
    n = empty_node();
  } else {
    n.c = sc[0]; n.r = sr[0]; n.a = x; n.alpha = phi;
  }
  // shared-origin flag for the final tests: the centre then equals that origin
  const bool so = real > 0 && same && __float_as_uint(n.c.x) == __float_as_uint(o0.x) &&
                  __float_as_uint(n.c.y) == __float_as_uint(o0.y) && __float_as_uint(n.c.z) == __float_as_uint(o0.z);
  store_node(a.nodes, a.trav, j, n, so);
}

// sorted rays of a segment for the CRSH_TAP_SORTED_RAYS tap when K5 did not
// write them: padded position i <- rays[sorted_slot[i]]
__global__ void k_gather_sorted(const uint32_t* __restrict__ sorted_slot, const float4* __restrict__ rays, uint32_t n,
                                float4* __restrict__ out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t slot = sorted_slot[i];
    out[2 * (size_t)i] = rays[2 * (size_t)slot];
    out[2 * (size_t)i + 1] = rays[2 * (size_t)slot + 1];
  }
}

struct UpperArgs {
  const FrameDesc* fd;
  int32_t level;             // padded nodes of this level: fd->level_n[level]
  const float4* child_nodes; // paper layout of level k-1
  float4* nodes;
  float4* trav;
};

// K6: node j = balanced pairwise union (Eqs 5-8, R9, R11) of children
// [j*B, (j+1)*B); empty children pass through. Two forms, bit-identical:
// thread per parent (default), and a segmented warp reduction (BASELINE
// north_star: "sphere-cone merge done as segmented warp reductions per
// level"; -DCRSH_UPPER_WARP=1): lane = child (coalesced child loads), 32 / B
// parents per warp; step w exchanges with lane ^ w and both lanes form
// union(lower, upper), so after log2 B steps every lane of the segment holds
// the union in exactly the balanced order ((0,1),(2,3)),((4,5),(6,7)) of R9.
// Measured at cfg4: 57 us for the warp form vs 19 us thread-per-parent (every
// lane forms each union: 3.5x the union work, each two atan2 + a division).
// (The leaf level, K5, is thread-per-bundle either way: its cone is a
// SEQUENTIAL fold of Eqs 1-4 over the bundle's rays, not a reduction.)
__device__ __forceinline__ NodeV shfl_xor_node(const NodeV& n, int w) {
  NodeV o;
  o.c = mk3(__shfl_xor_sync(CRSH_FULL, n.c.x, w), __shfl_xor_sync(CRSH_FULL, n.c.y, w), __shfl_xor_sync(CRSH_FULL, n.c.z, w));
  o.r = __shfl_xor_sync(CRSH_FULL, n.r, w);
  o.a = mk3(__shfl_xor_sync(CRSH_FULL, n.a.x, w), __shfl_xor_sync(CRSH_FULL, n.a.y, w), __shfl_xor_sync(CRSH_FULL, n.a.z, w));
  o.alpha = __shfl_xor_sync(CRSH_FULL, n.alpha, w);
  return o;
}
#ifndef CRSH_UPPER_WARP
#define CRSH_UPPER_WARP 0   // 1: segmented warp reduction (A/B at cfg4: k_upper 19 -> 57 us, every lane forms each union)
#endif
#if !CRSH_UPPER_WARP
template <int B>
__global__ void __launch_bounds__(128) k_upper(const UpperArgs a) {   // thread per parent (A/B)
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.fd->level_n[a.level]) return;
  NodeV st[B];
#pragma unroll
  for (int i = 0; i < B; ++i) st[i] = load_node(a.child_nodes, (size_t)j * B + i);
#pragma unroll
  for (int w = 1; w < B; w *= 2) {
#pragma unroll
    for (int i = 0; i < B; i += 2 * w) st[i] = node_union_ns(st[i], st[i + w]);
  }
  store_node(a.nodes, a.trav, j, st[0]);
}
#else
template <int B>
__global__ void __launch_bounds__(128) k_upper(const UpperArgs a) {
  const uint32_t gl = blockIdx.x * blockDim.x + threadIdx.x;   // global lane = child index
  const uint32_t n_par = a.fd->level_n[a.level];
  if ((gl & ~31u) >= n_par * (uint32_t)B) return;   // warp-uniform: the whole warp is past the level
  const uint32_t lane = gl & 31u;
  NodeV v = gl < n_par * (uint32_t)B ? load_node(a.child_nodes, gl) : empty_node();
#pragma unroll
  for (int w = 1; w < B; w *= 2) {
    const NodeV o = shfl_xor_node(v, w);
    v = (lane & (uint32_t)w) ? node_union_ns(o, v) : node_union_ns(v, o);   // union(lower lane, upper lane)
  }
  if ((lane & (uint32_t)(B - 1)) == 0u && gl < n_par * (uint32_t)B) store_node(a.nodes, a.trav, gl / B, v);
}
#endif

// ---------------------------------------------------------------- dynamic scenes
// (§3.3.1): creation-time vertices -> per-mesh
// affine transform [A | b] (row-major 3x4), per axis
// fma(a0, x, fma(a1, y, fma(a2, z, b))); AABB of the result.
__global__ void k_transform(const float* __restrict__ tris0, const int32_t* __restrict__ mesh_ids, int64_t M,
                            const float* __restrict__ xf, float* __restrict__ tris, float* __restrict__ box /*6*/) {
  float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < M; t += (int64_t)gridDim.x * blockDim.x) {
    const float* a = xf + 12 * __ldg(mesh_ids + t);
    for (int v = 0; v < 3; ++v) {
      const float x = tris0[9 * t + 3 * v], y = tris0[9 * t + 3 * v + 1], z = tris0[9 * t + 3 * v + 2];
      for (int r = 0; r < 3; ++r) {
        const float o = __fmaf_rn(a[4 * r], x, __fmaf_rn(a[4 * r + 1], y, __fmaf_rn(a[4 * r + 2], z, a[4 * r + 3])));
        tris[9 * t + 3 * v + r] = o;
        mn[r] = fminf(mn[r], o);
        mx[r] = fmaxf(mx[r], o);
      }
    }
  }
  // min / max are exact and order-free: warp reduce, then one atomic per warp
  // on the float bits ordered as integers (monotone map of IEEE floats)
  for (int r = 0; r < 3; ++r) {
    float lo = mn[r], hi = mx[r];
    for (int o = 16; o > 0; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(CRSH_FULL, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(CRSH_FULL, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
      auto key = [](float f) {   // order-preserving float -> int
        const int i = __float_as_int(f);
        return i >= 0 ? i : (int)(i ^ 0x7FFFFFFF);
      };
      atomicMin(reinterpret_cast<int*>(box) + r, key(lo));
      atomicMax(reinterpret_cast<int*>(box) + 3 + r, key(hi));
    }
  }
}

}  // namespace crsh
