// numspec.cuh — device float32 arithmetic of the CRSH path, in the frozen
// evaluation order of DESIGN.md §4 ("NUMSPEC"). This file is the GPU side's
// own implementation; it shares no code with oracle/. The translation unit is
// compiled with --fmad=false, so the only fused multiply-adds are the explicit
// __fmaf_rn calls below; divisions and square roots are IEEE round-to-nearest.
// That makes keys, nodes and test decisions bit-identical to any other
// implementation of NUMSPEC (the oracle), which the parity tests check.
#pragma once
#include <stdint.h>

namespace crsh {

struct f3 { float x, y, z; };
__device__ __forceinline__ f3 mk3(float x, float y, float z) { f3 r; r.x = x; r.y = y; r.z = z; return r; }
__device__ __forceinline__ f3 operator-(f3 a, f3 b) { return mk3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ f3 operator+(f3 a, f3 b) { return mk3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ f3 operator*(f3 a, float s) { return mk3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ f3 neg3(f3 a) { return mk3(-a.x, -a.y, -a.z); }
// dot = fma(ax,bx, fma(ay,by, az*bz))
__device__ __forceinline__ float dot3(f3 a, f3 b) { return __fmaf_rn(a.x, b.x, __fmaf_rn(a.y, b.y, a.z * b.z)); }
// cross = (fma(ay,bz,-(az*by)), fma(az,bx,-(ax*bz)), fma(ax,by,-(ay*bx)))
__device__ __forceinline__ f3 cross3(f3 a, f3 b) {
  return mk3(__fmaf_rn(a.y, b.z, -(a.z * b.y)), __fmaf_rn(a.z, b.x, -(a.x * b.z)), __fmaf_rn(a.x, b.y, -(a.y * b.x)));
}
__device__ __forceinline__ float len3(f3 a) { return sqrtf(dot3(a, a)); }
__device__ __forceinline__ f3 norm3(f3 a) { return a * (1.0f / sqrtf(dot3(a, a))); }

#define CRSH_PI_F 0x1.921fb6p+1f
#define CRSH_PI2_F 0x1.921fb6p+0f
#define CRSH_PI4_F 0x1.921fb6p-1f
#define CRSH_PI34_F 0x1.2d97c8p+1f
#define CRSH_PI_LO (-0x1.777a5cp-24f)
#define CRSH_PI2_LO (-0x1.777a5cp-25f)
#define CRSH_WIDE 1e30f   // tan/sec stand-in for alpha >= pi/2 (pass-all)

// atan2 by a degree-15 odd polynomial on [0,1] + octant reconstruction (R7).
__device__ __forceinline__ float atan2_ns(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float hi = fmaxf(ax, ay), lo = fminf(ax, ay);
  if (hi == 0.0f) return 0.0f;
  const float a = lo / hi;
  const float s = a * a;
  float p = -0x1.099aap-8f;
  p = __fmaf_rn(p, s, 0x1.66138cp-6f);
  p = __fmaf_rn(p, s, -0x1.c9ec26p-5f);
  p = __fmaf_rn(p, s, 0x1.8ae4c6p-4f);
  p = __fmaf_rn(p, s, -0x1.1cd608p-3f);
  p = __fmaf_rn(p, s, 0x1.988098p-3f);
  p = __fmaf_rn(p, s, -0x1.554c2ep-2f);
  p = __fmaf_rn(p, s, 0x1.ffffeap-1f);
  float r = a * p;
  if (ay > ax) r = CRSH_PI2_F - r;
  if (x < 0.0f) r = CRSH_PI_F - r;
  if (y < 0.0f) r = -r;
  return r;
}

// Taylor sin / cos on |y| <= pi/4, Horner in y^2.
__device__ __forceinline__ float sin_ns(float y) {
  const float s = y * y;
  float p = -0x1.ae7f3ep-41f;
  p = __fmaf_rn(p, s, 0x1.612462p-33f);
  p = __fmaf_rn(p, s, -0x1.ae6456p-26f);
  p = __fmaf_rn(p, s, 0x1.71de3ap-19f);
  p = __fmaf_rn(p, s, -0x1.a01a02p-13f);
  p = __fmaf_rn(p, s, 0x1.111112p-7f);
  p = __fmaf_rn(p, s, -0x1.555556p-3f);
  return __fmaf_rn(y * s, p, y);
}
__device__ __forceinline__ float cos_ns(float y) {
  const float s = y * y;
  float p = 0x1.ae7f3ep-45f;
  p = __fmaf_rn(p, s, -0x1.93974ap-37f);
  p = __fmaf_rn(p, s, 0x1.1eed8ep-29f);
  p = __fmaf_rn(p, s, -0x1.27e4fcp-22f);
  p = __fmaf_rn(p, s, 0x1.a01a02p-16f);
  p = __fmaf_rn(p, s, -0x1.6c16c2p-10f);
  p = __fmaf_rn(p, s, 0x1.555556p-5f);
  p = __fmaf_rn(p, s, -0.5f);
  return __fmaf_rn(s, p, 1.0f);
}
// cos, sin of phi in [0, pi]
__device__ __forceinline__ void sincos_ns(float phi, float* c, float* s) {
  if (phi <= CRSH_PI4_F) { *c = cos_ns(phi); *s = sin_ns(phi); return; }
  if (phi <= CRSH_PI34_F) { const float y = (CRSH_PI2_F - phi) + CRSH_PI2_LO; *c = sin_ns(y); *s = cos_ns(y); return; }
  const float y = (CRSH_PI_F - phi) + CRSH_PI_LO;
  *c = -cos_ns(y);
  *s = sin_ns(y);
}
// angle between unit vectors: atan2(|u x v|, u.v) (R10/R11)
__device__ __forceinline__ float angle_ns(f3 u, f3 v) { return atan2_ns(len3(cross3(u, v)), dot3(u, v)); }

// (tan alpha, sec alpha) for the Eq 9 test; alpha >= pi/2 -> pass-all stand-in.
__device__ __forceinline__ void tansec_ns(float alpha, float* tn, float* sc) {
  if (alpha >= CRSH_PI2_F) { *tn = CRSH_WIDE; *sc = CRSH_WIDE; return; }
  float c, s;
  sincos_ns(alpha, &c, &s);
  *tn = s / c;
  *sc = 1.0f / c;
}

// ---------------------------------------------------------------- hashes (R6)
__device__ __forceinline__ uint32_t quant_ns(float u, int bits) {
  const uint32_t top = (1u << bits) - 1u;
  const uint32_t v = (uint32_t)floorf(fmaxf(u, 0.0f) * (float)top);
  return v < top ? v : top;
}
__device__ __forceinline__ uint32_t quant_origin_ns(float o, float mn, float ext) {
  if (!(ext > 0.0f)) return 0u;
  const uint32_t v = (uint32_t)floorf(fmaxf((o - mn) / ext, 0.0f) * 32.0f);
  return v < 31u ? v : 31u;
}
// spread the low `bits` bits of v to every 2nd / 3rd position (Z-order)
__device__ __forceinline__ uint32_t spread2_ns(uint32_t v) {
  v &= 0xFFFFu;
  v = (v | (v << 8)) & 0x00FF00FFu;
  v = (v | (v << 4)) & 0x0F0F0F0Fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}
__device__ __forceinline__ uint32_t spread3_ns(uint32_t v) {
  v &= 0x3FFu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
__device__ __forceinline__ void spherical_ns(f3 d, float* th, float* ph) {
  *th = atan2_ns(sqrtf(__fmaf_rn(d.x, d.x, d.y * d.y)), d.z);
  *ph = atan2_ns(d.y, d.x);
}
__device__ __forceinline__ uint32_t hash_shadow_ns(uint32_t light, f3 d, bool zorder) {
  float th, ph;
  spherical_ns(d, &th, &ph);
  const uint32_t qt = quant_ns(th / CRSH_PI_F, 14), qp = quant_ns((ph + CRSH_PI_F) / (2.0f * CRSH_PI_F), 14);
  if (zorder) return (light << 28) | (spread2_ns(qt) << 1) | spread2_ns(qp);
  return (light << 28) | (qt << 14) | qp;
}
__device__ __forceinline__ uint32_t hash_bounce_ns(f3 o, f3 d, const float* bmin, const float* bext, bool zorder) {
  float th, ph;
  spherical_ns(d, &th, &ph);
  const uint32_t qt = quant_ns(th / CRSH_PI_F, 8), qp = quant_ns((ph + CRSH_PI_F) / (2.0f * CRSH_PI_F), 9);
  const uint32_t qx = quant_origin_ns(o.x, bmin[0], bext[0]);
  const uint32_t qy = quant_origin_ns(o.y, bmin[1], bext[1]);
  const uint32_t qz = quant_origin_ns(o.z, bmin[2], bext[2]);
  if (zorder)
    return (((spread3_ns(qx) << 2) | (spread3_ns(qy) << 1) | spread3_ns(qz)) << 17) | ((qp >> 8) << 16) |
           (spread2_ns(qt) << 1) | spread2_ns(qp & 0xFFu);
  return (qx << 27) | (qy << 22) | (qz << 17) | (qt << 9) | qp;
}

// ---------------------------------------------------------------- sphere-cone nodes
struct NodeV { f3 c; float r; f3 a; float alpha; };   // r < 0: empty (no rays)

__device__ __forceinline__ NodeV empty_node() {
  NodeV n; n.c = mk3(0.f, 0.f, 0.f); n.r = -1.0f; n.a = mk3(0.f, 0.f, 0.f); n.alpha = 0.0f; return n;
}

// Eqs 7-8
__device__ __forceinline__ void sphere_union_ns(f3 c1, float r1, f3 c2, float r2, f3* c, float* r) {
  if (r1 < 0.0f) { *c = c2; *r = r2; return; }
  if (r2 < 0.0f) { *c = c1; *r = r1; return; }
  *c = (c1 + c2) * 0.5f;
  *r = len3(c2 - c1) * 0.5f + fmaxf(r1, r2);
}
// Eqs 5-6 (R11, containment-exact evaluation)
__device__ __forceinline__ void cone_union_ns(f3 x1, float p1, f3 x2, float p2, f3* x, float* p) {
  if (p1 >= CRSH_PI_F || p2 >= CRSH_PI_F) { *x = x1; *p = CRSH_PI_F; return; }
  const f3 s = x1 + x2;
  const float L = len3(s);
  if (L < 1e-6f) { *x = x1; *p = CRSH_PI_F; return; }
  const f3 xn = s * (1.0f / L);
  const float ph = fmaxf(angle_ns(xn, x1) + p1, angle_ns(xn, x2) + p2);
  *x = xn;
  *p = ph < CRSH_PI_F ? ph : CRSH_PI_F;
}
// Eqs 1-4 (R10, containment-exact evaluation)
__device__ __forceinline__ void cone_grow_ns(f3* x, float* phi, f3 r) {
  const float p0 = *phi;
  if (p0 >= CRSH_PI_F) return;
  const f3 x0 = *x;
  const float gamma = angle_ns(x0, r);
  if (gamma <= p0) return;
  if (p0 + gamma >= CRSH_PI_F) { *phi = CRSH_PI_F; return; }
  const float c = dot3(x0, r);
  const f3 w = mk3(__fmaf_rn(-c, x0.x, r.x), __fmaf_rn(-c, x0.y, r.y), __fmaf_rn(-c, x0.z, r.z));
  if (!(dot3(w, w) > 0.0f)) { *phi = CRSH_PI_F; return; }
  const f3 q = norm3(w);
  float cp, sp;
  sincos_ns(p0, &cp, &sp);
  const f3 e = mk3(__fmaf_rn(q.x, sp, -(x0.x * cp)), __fmaf_rn(q.y, sp, -(x0.y * cp)), __fmaf_rn(q.z, sp, -(x0.z * cp)));
  const f3 xn = norm3(r - e);
  const float pn = fmaxf(angle_ns(xn, r), angle_ns(xn, x0) + p0);
  *x = xn;
  *phi = pn < CRSH_PI_F ? pn : CRSH_PI_F;
}
__device__ __forceinline__ NodeV node_union_ns(const NodeV& A, const NodeV& B) {
  if (A.r < 0.0f) return B;
  if (B.r < 0.0f) return A;
  NodeV n;
  sphere_union_ns(A.c, A.r, B.c, B.r, &n.c, &n.r);
  cone_union_ns(A.a, A.alpha, B.a, B.alpha, &n.a, &n.alpha);
  return n;
}

// Eq 9 (R12, R13). Node given as (C, d, a, tan, sec). Wide cones
// (alpha >= pi/2) are stored in the traversal layout as a = 0, tan = sec =
// 1e30: then s = 0 passes the behind-apex check and rhs overflows to +inf,
// i.e. pass-all, exactly where the oracle's explicit alpha >= pi/2 branch
// passes.
__device__ __forceinline__ bool cull_ns(f3 C, float d, f3 a, float tn, float sc, float4 tgt) {
  const f3 v = mk3(tgt.x - C.x, tgt.y - C.y, tgt.z - C.z);
  const float s = dot3(v, a);
  const f3 w = mk3(__fmaf_rn(-s, a.x, v.x), __fmaf_rn(-s, a.y, v.y), __fmaf_rn(-s, a.z, v.z));
  const float w2 = dot3(w, w);
  const float dr = d + tgt.w;
  const float rhs = __fmaf_rn(fmaxf(s, 0.0f), tn, dr * sc);
  return (s >= -dr) & (w2 <= rhs * rhs);
}

// Moller-Trumbore (R15), two-sided, division-free decision order:
// barycentric numerators against |det|; one reciprocal for t of a candidate.
__device__ __forceinline__ bool mt_ns(f3 o, f3 d, float tmin, float tmax, f3 v0, f3 e1, f3 e2, float* tout) {
  const f3 p = cross3(d, e2);
  const float det = dot3(e1, p);
  if (det == 0.0f) return false;
  const float sg = det > 0.0f ? 1.0f : -1.0f;
  const float adet = det * sg;
  const f3 tv = o - v0;
  const float un = dot3(tv, p) * sg;
  if (un < 0.0f || un > adet) return false;
  const f3 q = cross3(tv, e1);
  const float vn = dot3(d, q) * sg;
  if (vn < 0.0f || un + vn > adet) return false;
  const float t = dot3(e2, q) * (1.0f / det);
  if (!(t > tmin && t < tmax)) return false;
  *tout = t;
  return true;
}

}  // namespace crsh

// ---------------------------------------------------------------- packed f32x2 (sm_100a FFMA2 & co)
// Two independent IEEE round-to-nearest float32 operations per instruction:
// each half is bit-identical to the scalar operation, so cull2_ns gives the
// same decisions as two cull_ns calls.
namespace crsh {
typedef float2 f2;
// the sm_100 f32x2 builtins (fma/add/mul .rn.f32x2): the compiler sees them as
// arithmetic on register pairs, so packed operands stay in aligned pairs
__device__ __forceinline__ f2 pk2(float lo, float hi) { return make_float2(lo, hi); }
__device__ __forceinline__ void up2(f2 v, float& lo, float& hi) { lo = v.x; hi = v.y; }
__device__ __forceinline__ f2 add2(f2 a, f2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ f2 sub2(f2 a, f2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }   // negation is exact
__device__ __forceinline__ f2 mul2(f2 a, f2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { return __ffma2_rn(a, b, c); }

// Paired node record (two children c, c+1), 5 x float4 in shared memory:
// {Cx0,Cx1,Cy0,Cy1}, {Cz0,Cz1,d0,d1}, {ax0,ax1,ay0,ay1}, {az0,az1,tan0,tan1}, {sec0,sec1,-,-}
// Eq 9 for both children against one target sphere (px,py,pz,r); same
// operation order as cull_ns.
__device__ __forceinline__ void cull2_terms(const float4* rec, f2 Px, f2 Py, f2 Pz, f2 R, f2& s, f2& dr, f2& w2,
                                            f2& rr) {
  const float4 A = rec[0], Bv = rec[1], Cc = rec[2], D = rec[3], E = rec[4];
  const f2 cx = pk2(A.x, A.y), cy = pk2(A.z, A.w), cz = pk2(Bv.x, Bv.y), dd = pk2(Bv.z, Bv.w);
  const f2 ax = pk2(Cc.x, Cc.y), ay = pk2(Cc.z, Cc.w), az = pk2(D.x, D.y), tn = pk2(D.z, D.w), sc = pk2(E.x, E.y);
  const f2 vx = sub2(Px, cx), vy = sub2(Py, cy), vz = sub2(Pz, cz);
  s = fma2(vx, ax, fma2(vy, ay, mul2(vz, az)));
  // w = v + s * (-a) = fma(-s, a, v) exactly (negation is exact)
  const f2 wx = fma2(s, pk2(-Cc.x, -Cc.y), vx), wy = fma2(s, pk2(-Cc.z, -Cc.w), vy), wz = fma2(s, pk2(-D.x, -D.y), vz);
  w2 = fma2(wx, wx, fma2(wy, wy, mul2(wz, wz)));
  dr = add2(dd, R);
  float s0, s1;
  up2(s, s0, s1);
  const f2 rhs = fma2(pk2(fmaxf(s0, 0.0f), fmaxf(s1, 0.0f)), tn, mul2(dr, sc));
  rr = mul2(rhs, rhs);
}
__device__ __forceinline__ void cull2_ns(const float4* rec, f2 Px, f2 Py, f2 Pz, f2 R, bool& p0, bool& p1) {
  f2 s, dr, w2, rr;
  cull2_terms(rec, Px, Py, Pz, R, s, dr, w2, rr);
  float s0, s1, w0, w1, r0, r1, d0, d1;
  up2(s, s0, s1);
  up2(w2, w0, w1);
  up2(rr, r0, r1);
  up2(dr, d0, d1);
  p0 = (s0 >= -d0) & (w0 <= r0);
  p1 = (s1 >= -d1) & (w1 <= r1);
}
// the same two decisions as mask bits, (p0 ? bit0 : 0) | (p1 ? bit1 : 0): the
// two compares of each test chained in one predicate (setp ... .and) and one
// select per test, instead of the compiler's per-compare selects
__device__ __forceinline__ uint32_t cull2_bits(const float4* rec, f2 Px, f2 Py, f2 Pz, f2 R, uint32_t bit0,
                                               uint32_t bit1) {
  f2 s, dr, w2, rr;
  cull2_terms(rec, Px, Py, Pz, R, s, dr, w2, rr);
  float s0, s1, w0, w1, r0, r1, d0, d1;
  up2(s, s0, s1);
  up2(w2, w0, w1);
  up2(rr, r0, r1);
  up2(dr, d0, d1);
  uint32_t m;
  asm("{\n\t.reg .pred q0, q1;\n\t.reg .f32 n0, n1;\n\t.reg .b32 t0, t1;\n\t"
      "neg.f32 n0, %3;\n\tneg.f32 n1, %4;\n\t"
      "setp.ge.f32 q0, %1, n0;\n\tsetp.le.and.f32 q0, %5, %7, q0;\n\t"
      "setp.ge.f32 q1, %2, n1;\n\tsetp.le.and.f32 q1, %6, %8, q1;\n\t"
      "selp.b32 t0, %9, 0, q0;\n\tselp.b32 t1, %10, 0, q1;\n\tor.b32 %0, t0, t1;\n\t}"
      : "=r"(m)
      : "f"(s0), "f"(s1), "f"(d0), "f"(d1), "f"(w0), "f"(w1), "f"(r0), "f"(r1), "r"(bit0), "r"(bit1));
  return m;
}
// cull2_ns with the paired record read through a 32-bit shared-memory address
// (ld.shared: no generic-to-shared window computation per record; the same
// values, so the same decisions). Volatile with a memory clobber: the
// compiler must not hoist these loads across the group setup that writes the
// records (an address that does not change between groups would otherwise
// look loop-invariant); the SASS of the K8 instantiations is unchanged.
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void cull2_ns_s(uint32_t rec, f2 Px, f2 Py, f2 Pz, f2 R, bool& p0, bool& p1) {
  const float4 r4[5] = {lds128(rec), lds128(rec + 16u), lds128(rec + 32u), lds128(rec + 48u), lds128(rec + 64u)};
  cull2_ns(r4, Px, Py, Pz, R, p0, p1);
}
__device__ __forceinline__ uint32_t cull2_bits_s(uint32_t rec, f2 Px, f2 Py, f2 Pz, f2 R, uint32_t bit0,
                                                 uint32_t bit1) {
  const float4 r4[5] = {lds128(rec), lds128(rec + 16u), lds128(rec + 32u), lds128(rec + 48u), lds128(rec + 64u)};
  return cull2_bits(r4, Px, Py, Pz, R, bit0, bit1);
}
}  // namespace crsh

namespace crsh {
// Moller-Trumbore (mt_ns, same per-half operation order) for two rays given
// as a paired record {ox0,ox1,oy0,oy1} {oz0,oz1,tmin0,tmin1}
// {dx0,dx1,dy0,dy1} {dz0,dz1,tmax0,tmax1} against one triangle; the
// triangle's scalars enter the packed instructions as broadcast operands.
// Returns a hit mask (bit i: ray i hits in (tmin, tmax)) with t0 / t1; a
// mask rather than two bools keeps the hit test in predicates and one
// register (bools set on several return paths were materialised as bytes).
// EARLY: leave as soon as both rays failed a barycentric test (a warp of 32
// lanes almost never takes that exit together, so the branch-free form, which
// lets independent ray pairs interleave, is the default in the traversal).
template <bool EARLY = true>
__device__ __forceinline__ uint32_t mt2_ns(float4 A, float4 Bq, float4 Cq, float4 Dq, f3 v0, f3 e1, f3 e2, float& t0,
                                           float& t1) {
  const f2 ox = pk2(A.x, A.y), oy = pk2(A.z, A.w), oz = pk2(Bq.x, Bq.y);
  const f2 dx = pk2(Cq.x, Cq.y), dy = pk2(Cq.z, Cq.w), dz = pk2(Dq.x, Dq.y);
  const f2 px = fma2(dy, pk2(e2.z, e2.z), mul2(dz, pk2(-e2.y, -e2.y)));
  const f2 py = fma2(dz, pk2(e2.x, e2.x), mul2(dx, pk2(-e2.z, -e2.z)));
  const f2 pz = fma2(dx, pk2(e2.y, e2.y), mul2(dy, pk2(-e2.x, -e2.x)));
  const f2 det = fma2(pk2(e1.x, e1.x), px, fma2(pk2(e1.y, e1.y), py, mul2(pk2(e1.z, e1.z), pz)));
  float d0, d1;
  up2(det, d0, d1);
  const f2 sg = pk2(d0 > 0.0f ? 1.0f : -1.0f, d1 > 0.0f ? 1.0f : -1.0f);
  const f2 adet = mul2(det, sg);
  const f2 tx = sub2(ox, pk2(v0.x, v0.x)), ty = sub2(oy, pk2(v0.y, v0.y)), tz = sub2(oz, pk2(v0.z, v0.z));
  const f2 un = mul2(fma2(tx, px, fma2(ty, py, mul2(tz, pz))), sg);
  float u0, u1, a0v, a1v;
  up2(un, u0, u1);
  up2(adet, a0v, a1v);
  bool k0 = (d0 != 0.0f) & (u0 >= 0.0f) & (u0 <= a0v);
  bool k1 = (d1 != 0.0f) & (u1 >= 0.0f) & (u1 <= a1v);
  if (EARLY && !(k0 | k1)) return 0u;
  const f2 qx = fma2(ty, pk2(e1.z, e1.z), mul2(tz, pk2(-e1.y, -e1.y)));
  const f2 qy = fma2(tz, pk2(e1.x, e1.x), mul2(tx, pk2(-e1.z, -e1.z)));
  const f2 qz = fma2(tx, pk2(e1.y, e1.y), mul2(ty, pk2(-e1.x, -e1.x)));
  const f2 vn = mul2(fma2(dx, qx, fma2(dy, qy, mul2(dz, qz))), sg);
  const f2 s = add2(un, vn);
  float v0f, v1f, s0, s1;
  up2(vn, v0f, v1f);
  up2(s, s0, s1);
  k0 &= (v0f >= 0.0f) & (s0 <= a0v);
  k1 &= (v1f >= 0.0f) & (s1 <= a1v);
  if (EARLY && !(k0 | k1)) return 0u;
  const f2 tt = mul2(fma2(pk2(e2.x, e2.x), qx, fma2(pk2(e2.y, e2.y), qy, mul2(pk2(e2.z, e2.z), qz))),
                     pk2(1.0f / d0, 1.0f / d1));
  up2(tt, t0, t1);
  return ((k0 & (t0 > Bq.z) & (t0 < Dq.z)) ? 1u : 0u) | ((k1 & (t1 > Bq.w) & (t1 < Dq.w)) ? 2u : 0u);
}

// mt2_ns for two rays that share their origin o (bit for bit): tv = o - v0,
// q = cross(tv, e1) and tq = dot(e2, q) are passed in, computed once for the
// bundle -- exactly the values mt2_ns computes per ray, so the decisions and
// t are bit-identical. Ray record halves: Bq = {-, -, tmin0, tmin1},
// Cq = {dx0, dx1, dy0, dy1}, Dq = {dz0, dz1, tmax0, tmax1}.
__device__ __forceinline__ uint32_t mt2o_ns(float4 Bq, float4 Cq, float4 Dq, f3 e1, f3 e2, f3 tv, f3 q, float tq, float& t0,
                                            float& t1) {
  const f2 dx = pk2(Cq.x, Cq.y), dy = pk2(Cq.z, Cq.w), dz = pk2(Dq.x, Dq.y);
  const f2 px = fma2(dy, pk2(e2.z, e2.z), mul2(dz, pk2(-e2.y, -e2.y)));
  const f2 py = fma2(dz, pk2(e2.x, e2.x), mul2(dx, pk2(-e2.z, -e2.z)));
  const f2 pz = fma2(dx, pk2(e2.y, e2.y), mul2(dy, pk2(-e2.x, -e2.x)));
  const f2 det = fma2(pk2(e1.x, e1.x), px, fma2(pk2(e1.y, e1.y), py, mul2(pk2(e1.z, e1.z), pz)));
  float d0, d1;
  up2(det, d0, d1);
  const f2 sg = pk2(d0 > 0.0f ? 1.0f : -1.0f, d1 > 0.0f ? 1.0f : -1.0f);
  const f2 adet = mul2(det, sg);
  const f2 un = mul2(fma2(pk2(tv.x, tv.x), px, fma2(pk2(tv.y, tv.y), py, mul2(pk2(tv.z, tv.z), pz))), sg);
  float u0, u1, a0v, a1v;
  up2(un, u0, u1);
  up2(adet, a0v, a1v);
  bool k0 = (d0 != 0.0f) & (u0 >= 0.0f) & (u0 <= a0v);
  bool k1 = (d1 != 0.0f) & (u1 >= 0.0f) & (u1 <= a1v);
  if (!(k0 | k1)) return 0u;
  const f2 vn = mul2(fma2(dx, pk2(q.x, q.x), fma2(dy, pk2(q.y, q.y), mul2(dz, pk2(q.z, q.z)))), sg);
  const f2 s = add2(un, vn);
  float v0f, v1f, s0, s1;
  up2(vn, v0f, v1f);
  up2(s, s0, s1);
  k0 &= (v0f >= 0.0f) & (s0 <= a0v);
  k1 &= (v1f >= 0.0f) & (s1 <= a1v);
  if (!(k0 | k1)) return 0u;
  const f2 tt = mul2(pk2(tq, tq), pk2(1.0f / d0, 1.0f / d1));
  up2(tt, t0, t1);
  return ((k0 & (t0 > Bq.z) & (t0 < Dq.z)) ? 1u : 0u) | ((k1 & (t1 > Bq.w) & (t1 < Dq.w)) ? 2u : 0u);
}
}  // namespace crsh
