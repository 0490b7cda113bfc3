/* oracle/oracle.cpp — CPU oracle for the Coherent Ray-Space Hierarchy (CRSH)
 * secondary-ray path of Reis, Costa & Pereira, arXiv 2312.06538.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_2312_06538_b200/) never includes, links or calls anything here, and
 * this file shares no code with it.
 *
 * Citations: "P:n" = line n of the paper text, "S:n" = line n of
 * SPEC.md, "R#" = a reading listed in DESIGN.md §3 (where the paper is silent,
 * garbled or inconsistent). "NUMSPEC" = the frozen float32 evaluation order in
 * DESIGN.md §4, which the CUDA path implements independently; both follow it so
 * that hash keys, nodes and test counts can be compared bit for bit.
 *
 * Precision: float32 (the paper stores the G-buffer as "four 32 bit floats"
 * P:71 and a node as "eight floats" P:131). Built with -ffp-contract=off; the
 * only fused multiply-adds are the explicit fmaf() calls NUMSPEC names (fmaf is
 * correctly rounded, so it is deterministic across CPU and GPU).
 *
 * Parity pins: every function is pinned in tests/test_oracle_*.py against
 * closed forms, SPEC worked examples, invariants or brute force (see the
 * docstring of each test). Node values beyond containment are "parity
 * unpinned" except through those invariants.
 */
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <thread>
#include <vector>

#define EXPORT extern "C" __attribute__((visibility("default")))

namespace {

// ---------------------------------------------------------------------------
// NUMSPEC float32 vector arithmetic
struct V3 { float x, y, z; };
inline V3 v3(float x, float y, float z) { return V3{x, y, z}; }
inline V3 sub(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
inline V3 add(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
inline V3 scale(V3 a, float s) { return v3(a.x * s, a.y * s, a.z * s); }
inline V3 neg(V3 a) { return v3(-a.x, -a.y, -a.z); }
inline float dot3(V3 a, V3 b) { return fmaf(a.x, b.x, fmaf(a.y, b.y, a.z * b.z)); }
inline V3 cross3(V3 a, V3 b) {
  return v3(fmaf(a.y, b.z, -(a.z * b.y)), fmaf(a.z, b.x, -(a.x * b.z)), fmaf(a.x, b.y, -(a.y * b.x)));
}
inline float len3(V3 a) { return sqrtf(dot3(a, a)); }
inline V3 norm3(V3 a) { return scale(a, 1.0f / sqrtf(dot3(a, a))); }

const float PI_F = 0x1.921fb6p+1f;       // (float)pi
const float PI2_F = 0x1.921fb6p+0f;      // (float)(pi/2)
const float PI4_F = 0x1.921fb6p-1f;      // (float)(pi/4)
const float PI34_F = 0x1.2d97c8p+1f;     // (float)(3pi/4)
const float PI_LO = -0x1.777a5cp-24f;    // pi - PI_F
const float PI2_LO = -0x1.777a5cp-25f;   // pi/2 - PI2_F

// atan2 replacement, R7: degree-15 odd polynomial for atan on [0,1],
// then octant reconstruction. Only IEEE basic ops -> identical on CPU and GPU.
float atan2p(float y, float x) {
  float ax = fabsf(x), ay = fabsf(y);
  float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  if (mx == 0.0f) return 0.0f;
  float a = mn / mx;
  float s = a * a;
  float p = -0x1.099aap-8f;
  p = fmaf(p, s, 0x1.66138cp-6f);
  p = fmaf(p, s, -0x1.c9ec26p-5f);
  p = fmaf(p, s, 0x1.8ae4c6p-4f);
  p = fmaf(p, s, -0x1.1cd608p-3f);
  p = fmaf(p, s, 0x1.988098p-3f);
  p = fmaf(p, s, -0x1.554c2ep-2f);
  p = fmaf(p, s, 0x1.ffffeap-1f);
  float r = a * p;
  if (ay > ax) r = PI2_F - r;
  if (x < 0.0f) r = PI_F - r;
  if (y < 0.0f) r = -r;
  return r;
}

// Taylor polynomials for |y| <= pi/4 (NUMSPEC).
float sin_p(float y) {
  float s = y * y;
  float p = -0x1.ae7f3ep-41f;
  p = fmaf(p, s, 0x1.612462p-33f);
  p = fmaf(p, s, -0x1.ae6456p-26f);
  p = fmaf(p, s, 0x1.71de3ap-19f);
  p = fmaf(p, s, -0x1.a01a02p-13f);
  p = fmaf(p, s, 0x1.111112p-7f);
  p = fmaf(p, s, -0x1.555556p-3f);
  return fmaf(y * s, p, y);
}
float cos_p(float y) {
  float s = y * y;
  float p = 0x1.ae7f3ep-45f;
  p = fmaf(p, s, -0x1.93974ap-37f);
  p = fmaf(p, s, 0x1.1eed8ep-29f);
  p = fmaf(p, s, -0x1.27e4fcp-22f);
  p = fmaf(p, s, 0x1.a01a02p-16f);
  p = fmaf(p, s, -0x1.6c16c2p-10f);
  p = fmaf(p, s, 0x1.555556p-5f);
  p = fmaf(p, s, -0.5f);
  return fmaf(s, p, 1.0f);
}
// cos and sin of phi in [0, pi] by reduction to |y| <= pi/4 (NUMSPEC).
void sincos_p(float phi, float* c, float* s) {
  if (phi <= PI4_F) { *c = cos_p(phi); *s = sin_p(phi); return; }
  if (phi <= PI34_F) { float y = (PI2_F - phi) + PI2_LO; *c = sin_p(y); *s = cos_p(y); return; }
  float y = (PI_F - phi) + PI_LO;
  *c = -cos_p(y);
  *s = sin_p(y);
}
// angle between unit vectors, R10/R11: the paper's arccos(u.v) (Eq 6, and the
// angle of Eq 4) evaluated in the stable form atan2(|u x v|, u.v).
float angle_between(V3 u, V3 v) { return atan2p(len3(cross3(u, v)), dot3(u, v)); }

// ---------------------------------------------------------------------------
// Hashes (Fig 2; Fig 3; bit layouts S:308/S:375, R6)
uint32_t quant(float u, int bits) {   // floor(u * (2^b - 1)), clamped
  uint32_t top = (1u << bits) - 1u;
  float q = floorf(fmaxf(u, 0.0f) * (float)top);
  uint32_t v = (uint32_t)q;
  return v < top ? v : top;
}
void spherical(V3 d, float* theta, float* phi) {  // theta from +z, phi from +x toward +y
  *theta = atan2p(sqrtf(fmaf(d.x, d.x, d.y * d.y)), d.z);
  *phi = atan2p(d.y, d.x);
}
// Z-order variant (flag CRSH_F_ZORDER; SURVEY §8(f) NEXT-4 "improved hash
// functions"): the same quantised fields, bits interleaved
// (theta bit i -> 2i+1, phi bit i -> 2i; origin x,y,z bit i -> 3i+2,3i+1,3i).
uint32_t spread2(uint32_t v, int bits) {
  uint32_t out = 0;
  for (int i = 0; i < bits; ++i) out |= ((v >> i) & 1u) << (2 * i);
  return out;
}
uint32_t spread3(uint32_t v, int bits) {
  uint32_t out = 0;
  for (int i = 0; i < bits; ++i) out |= ((v >> i) & 1u) << (3 * i);
  return out;
}
uint32_t hash_shadow(uint32_t light, V3 d, bool zorder) {
  float th, ph;
  spherical(d, &th, &ph);
  uint32_t qt = quant(th / PI_F, 14), qp = quant((ph + PI_F) / (2.0f * PI_F), 14);
  if (zorder) return (light << 28) | (spread2(qt, 14) << 1) | spread2(qp, 14);
  return (light << 28) | (qt << 14) | qp;
}
uint32_t quant_origin(float o, float mn, float ext) {
  if (!(ext > 0.0f)) return 0u;
  float q = floorf(fmaxf((o - mn) / ext, 0.0f) * 32.0f);
  uint32_t v = (uint32_t)q;
  return v < 31u ? v : 31u;
}
uint32_t hash_bounce(V3 o, V3 d, const float* box_min, const float* box_ext, bool zorder) {
  float th, ph;
  spherical(d, &th, &ph);
  uint32_t qt = quant(th / PI_F, 8), qp = quant((ph + PI_F) / (2.0f * PI_F), 9);
  uint32_t qx = quant_origin(o.x, box_min[0], box_ext[0]);
  uint32_t qy = quant_origin(o.y, box_min[1], box_ext[1]);
  uint32_t qz = quant_origin(o.z, box_min[2], box_ext[2]);
  if (zorder)
    return ((spread3(qx, 5) << 2 | spread3(qy, 5) << 1 | spread3(qz, 5)) << 17) | ((qp >> 8) << 16) |
           (spread2(qt, 8) << 1) | spread2(qp & 0xFFu, 8);
  return (qx << 27) | (qy << 22) | (qz << 17) | (qt << 9) | qp;
}

// ---------------------------------------------------------------------------
// Sphere-cone node: c, r (sphere of origins), a, alpha (cone of
// directions). Empty node (no rays; padding): r = -1.
struct Node { V3 c; float r; V3 a; float alpha; };
const Node EMPTY_NODE = {{0, 0, 0}, -1.0f, {0, 0, 0}, 0.0f};

// Eqs 7-8. "Missing children pass through" (R9).
void sphere_union(V3 c1, float r1, V3 c2, float r2, V3* c, float* r) {
  if (r1 < 0.0f) { *c = c2; *r = r2; return; }
  if (r2 < 0.0f) { *c = c1; *r = r1; return; }
  *c = scale(add(c1, c2), 0.5f);                          // Eq 7
  *r = len3(sub(c2, c1)) * 0.5f + fmaxf(r1, r2);           // Eq 8
}

// Eqs 5-6, R11: phi = arccos(x1.x2)/2 + max(phi1, phi2), clamped to pi.
void cone_union(V3 x1, float p1, V3 x2, float p2, V3* x, float* p) {
  if (p1 >= PI_F || p2 >= PI_F) { *x = x1; *p = PI_F; return; }
  V3 s = add(x1, x2);
  float L = len3(s);
  if (L < 1e-6f) { *x = x1; *p = PI_F; return; }   // antiparallel axes: full cone
  V3 xn = scale(s, 1.0f / L);                        // Eq 5
  // Eq 6, R11: arccos(x1.x2)/2 + max(phi1, phi2) is, in exact arithmetic, the
  // larger of angle(x, x_i) + phi_i; evaluated in that form it contains both
  // children even when the computed bisector x is off (nearly antiparallel x_i).
  float phi = fmaxf(angle_between(xn, x1) + p1, angle_between(xn, x2) + p2);
  *x = xn;
  *p = phi < PI_F ? phi : PI_F;
}

// Eqs 1-4, R10: grow cone (x, phi) to contain unit direction r.
void cone_grow(V3 x, float phi, V3 r, V3* xo, float* po) {
  if (phi >= PI_F) { *xo = x; *po = PI_F; return; }
  float gamma = angle_between(x, r);
  if (gamma <= phi) { *xo = x; *po = phi; return; }            // already inside
  if (phi + gamma >= PI_F) { *xo = x; *po = PI_F; return; }    // would wrap: full cone
  float c = dot3(x, r);
  V3 w = v3(fmaf(-c, x.x, r.x), fmaf(-c, x.y, r.y), fmaf(-c, x.z, r.z));
  float wl = dot3(w, w);
  if (!(wl > 0.0f)) { *xo = x; *po = PI_F; return; }
  V3 q = norm3(w);                                           // Eq 1
  float cphi, sphi;
  sincos_p(phi, &cphi, &sphi);
  V3 e = v3(fmaf(q.x, sphi, -(x.x * cphi)), fmaf(q.y, sphi, -(x.y * cphi)),
            fmaf(q.z, sphi, -(x.z * cphi)));                  // Eq 2: e = -x cos(phi) + q sin(phi)
  V3 xn = norm3(sub(r, e));                                  // Eq 3: (-e + r)/|-e + r|
  // Eq 4, R10: cos(phi_new) = x_new . r, i.e. phi_new = angle(x_new, r); in
  // exact arithmetic it also equals angle(x_new, x) + phi = (phi + gamma)/2.
  // Taking the larger of the two keeps r AND the old cone inside even when
  // the computed x_new is off (phi + gamma near pi).
  float pn = fmaxf(angle_between(xn, r), angle_between(xn, x) + phi);
  *xo = xn;
  *po = pn < PI_F ? pn : PI_F;
}

Node node_union(const Node& A, const Node& B) {
  if (A.r < 0.0f) return B;
  if (B.r < 0.0f) return A;
  Node n;
  sphere_union(A.c, A.r, B.c, B.r, &n.c, &n.r);
  cone_union(A.a, A.alpha, B.a, B.alpha, &n.a, &n.alpha);
  return n;
}

// Eq 9, R12/R13: node (sphere C,d + cone a,alpha) vs target sphere (P, r).
bool cull_test(const Node& n, V3 P, float r) {
  if (n.alpha >= PI2_F) return true;                 // tan diverges; pass
  float ca, sa;
  sincos_p(n.alpha, &ca, &sa);
  float tana = sa / ca, seca = 1.0f / ca;
  V3 v = sub(P, n.c);
  float s = dot3(v, n.a);                            // signed distance of H along the axis
  if (s < -(n.r + r)) return false;                  // R13: wholly behind the apex
  V3 w = v3(fmaf(-s, n.a.x, v.x), fmaf(-s, n.a.y, v.y), fmaf(-s, n.a.z, v.z));   // P - H
  float w2 = dot3(w, w);
  float sp = fmaxf(s, 0.0f);                         // R13: clamp behind the apex
  float rhs = fmaf(sp, tana, (n.r + r) * seca);      // |C-H| tan(a) + (d+r)/cos(a)
  return w2 <= rhs * rhs;                            // >= |P-H|
}

// Moller-Trumbore ray-triangle test (P:185 [Mol97]; R15), two-sided, in the
// original paper's division-free decision order: the barycentric numerators
// are compared against |det| (sign folded in exactly), and the single
// reciprocal of det is only taken for t of a candidate hit.
bool moller_trumbore(V3 o, V3 d, float tmin, float tmax, V3 v0, V3 e1, V3 e2, float* t_out) {
  V3 p = cross3(d, e2);
  float det = dot3(e1, p);
  if (det == 0.0f) return false;
  float sg = det > 0.0f ? 1.0f : -1.0f;
  float adet = det * sg;                 // |det|
  V3 tv = sub(o, v0);
  float un = dot3(tv, p) * sg;           // u * |det|
  if (un < 0.0f || un > adet) return false;
  V3 q = cross3(tv, e1);
  float vn = dot3(d, q) * sg;            // v * |det|
  if (vn < 0.0f || un + vn > adet) return false;
  float t = dot3(e2, q) * (1.0f / det);
  if (!(t > tmin && t < tmax)) return false;
  *t_out = t;
  return true;
}

inline uint64_t pack_hit(float t, uint32_t tri) {  // closest hit, ties -> smaller tri
  uint32_t tb;
  std::memcpy(&tb, &t, 4);
  return ((uint64_t)tb << 32) | tri;
}

// ---------------------------------------------------------------------------
// double-precision bounding spheres (scene prep, untimed, R1, R2)
struct D3 { double x, y, z; };
inline D3 dsub(D3 a, D3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline D3 dadd(D3 a, D3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline D3 dscale(D3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double ddot(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline D3 dcross(D3 a, D3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }

// Round a double centre to float and take the radius as the max distance from
// that float centre to the points, rounded up (containment is exact).
void finalize_sphere(D3 c, const D3* pts, size_t n, float* out) {
  float cf[3] = {(float)c.x, (float)c.y, (float)c.z};
  D3 cd = {cf[0], cf[1], cf[2]};
  double r2 = 0.0;
  for (size_t i = 0; i < n; ++i) r2 = std::max(r2, ddot(dsub(pts[i], cd), dsub(pts[i], cd)));
  double r = std::sqrt(r2);
  float rf = (float)r;
  if ((double)rf < r) rf = nextafterf(rf, INFINITY);
  out[0] = cf[0]; out[1] = cf[1]; out[2] = cf[2]; out[3] = rf;
}

// Minimal sphere of a triangle: longest-edge midpoint if right/obtuse,
// else the circumcentre.
D3 tri_sphere_center(D3 a, D3 b, D3 c) {
  D3 ab = dsub(b, a), ac = dsub(c, a), bc = dsub(c, b);
  if (ddot(ab, ac) <= 0.0) return dscale(dadd(b, c), 0.5);          // angle at a >= 90
  if (ddot(dscale(ab, -1.0), bc) <= 0.0) return dscale(dadd(a, c), 0.5);  // at b
  if (ddot(ac, bc) <= 0.0) return dscale(dadd(a, b), 0.5);          // at c
  D3 n = dcross(ab, ac);
  double den = 2.0 * ddot(n, n);
  D3 num = dadd(dscale(dcross(n, ab), ddot(ac, ac)), dscale(dcross(ac, n), ddot(ab, ab)));
  return dadd(a, dscale(num, 1.0 / den));
}

// Welzl / Gartner move-to-front miniball [Gar99] in double.
struct Ball { D3 c; double r2; };
Ball ball_support(const D3* R, int k) {
  if (k == 0) return {{0, 0, 0}, -1.0};
  if (k == 1) return {R[0], 0.0};
  if (k == 2) { D3 c = dscale(dadd(R[0], R[1]), 0.5); return {c, ddot(dsub(R[0], c), dsub(R[0], c))}; }
  if (k == 3) {
    D3 ab = dsub(R[1], R[0]), ac = dsub(R[2], R[0]);
    D3 n = dcross(ab, ac);
    double den = 2.0 * ddot(n, n);
    if (den == 0.0) {   // collinear: diameter ball of the farthest pair
      Ball best = ball_support(R, 2);
      D3 p2[2] = {R[0], R[2]}; Ball b2 = ball_support(p2, 2); if (b2.r2 > best.r2) best = b2;
      D3 p3[2] = {R[1], R[2]}; Ball b3 = ball_support(p3, 2); if (b3.r2 > best.r2) best = b3;
      return best;
    }
    D3 num = dadd(dscale(dcross(n, ab), ddot(ac, ac)), dscale(dcross(ac, n), ddot(ab, ab)));
    D3 c = dadd(R[0], dscale(num, 1.0 / den));
    return {c, ddot(dsub(R[0], c), dsub(R[0], c))};
  }
  D3 ab = dsub(R[1], R[0]), ac = dsub(R[2], R[0]), ad = dsub(R[3], R[0]);
  double det = ddot(ab, dcross(ac, ad));
  if (det == 0.0) {   // coplanar: largest of the 3-point balls
    Ball best = {{0, 0, 0}, -1.0};
    for (int skip = 0; skip < 4; ++skip) {
      D3 q[3]; int m = 0;
      for (int i = 0; i < 4; ++i) if (i != skip) q[m++] = R[i];
      Ball b = ball_support(q, 3);
      if (b.r2 > best.r2) best = b;
    }
    return best;
  }
  double bb = 0.5 * ddot(ab, ab), cc = 0.5 * ddot(ac, ac), dd = 0.5 * ddot(ad, ad);
  // solve [ab; ac; ad] x = [bb, cc, dd] by Cramer's rule
  D3 x = dscale(dadd(dadd(dscale(dcross(ac, ad), bb), dscale(dcross(ad, ab), cc)), dscale(dcross(ab, ac), dd)),
                1.0 / det);
  return {dadd(R[0], x), ddot(x, x)};
}
Ball mtf_mb(std::vector<D3>& L, size_t end, D3* R, int k) {
  Ball b = ball_support(R, k);
  if (k == 4) return b;
  for (size_t i = 0; i < end; ++i) {
    D3 d = dsub(L[i], b.c);
    if (b.r2 < 0.0 || ddot(d, d) > b.r2 * (1.0 + 1e-13)) {
      R[k] = L[i];
      b = mtf_mb(L, i, R, k + 1);
      D3 p = L[i];
      std::memmove(&L[1], &L[0], i * sizeof(D3));
      L[0] = p;
    }
  }
  return b;
}

struct Counters {   // per (segment) traversal counters, §4.1, Tables 1-3
  uint64_t tests[9] = {0}, hits[9] = {0};
  uint64_t mesh_tests = 0, mesh_hits = 0, final_tests = 0, final_hits = 0;
  uint64_t cluster_tests = 0, cluster_hits = 0;   // object sphere-tree level (NEXT-4)
  void add(const Counters& o) {
    for (int k = 0; k < 9; ++k) { tests[k] += o.tests[k]; hits[k] += o.hits[k]; }
    mesh_tests += o.mesh_tests; mesh_hits += o.mesh_hits;
    final_tests += o.final_tests; final_hits += o.final_hits;
    cluster_tests += o.cluster_tests; cluster_hits += o.cluster_hits;
  }
};

inline Node load_node(const float* p) {
  return Node{v3(p[0], p[1], p[2]), p[3], v3(p[4], p[5], p[6]), p[7]};
}
inline void store_node(float* p, const Node& n) {
  p[0] = n.c.x; p[1] = n.c.y; p[2] = n.c.z; p[3] = n.r;
  p[4] = n.a.x; p[5] = n.a.y; p[6] = n.a.z; p[7] = n.alpha;
}

}  // namespace

// ===========================================================================
// exported building blocks (each pinned in tests/test_oracle_*.py)

EXPORT float or_atan2p(float y, float x) { return atan2p(y, x); }
EXPORT void or_sincos(float phi, float* c, float* s) { sincos_p(phi, c, s); }
EXPORT uint32_t or_hash_shadow(uint32_t light, const float* d, int zorder) {
  return hash_shadow(light, v3(d[0], d[1], d[2]), zorder != 0);
}
EXPORT uint32_t or_hash_bounce(const float* o, const float* d, const float* bmin, const float* bext, int zorder) {
  return hash_bounce(v3(o[0], o[1], o[2]), v3(d[0], d[1], d[2]), bmin, bext, zorder != 0);
}
EXPORT void or_cone_grow(const float* x, float phi, const float* r, float* xo, float* po) {
  V3 X;
  cone_grow(v3(x[0], x[1], x[2]), phi, v3(r[0], r[1], r[2]), &X, po);
  xo[0] = X.x; xo[1] = X.y; xo[2] = X.z;
}
EXPORT void or_cone_union(const float* x1, float p1, const float* x2, float p2, float* xo, float* po) {
  V3 X;
  cone_union(v3(x1[0], x1[1], x1[2]), p1, v3(x2[0], x2[1], x2[2]), p2, &X, po);
  xo[0] = X.x; xo[1] = X.y; xo[2] = X.z;
}
EXPORT void or_sphere_union(const float* s1, const float* s2, float* so) {
  V3 c;
  sphere_union(v3(s1[0], s1[1], s1[2]), s1[3], v3(s2[0], s2[1], s2[2]), s2[3], &c, &so[3]);
  so[0] = c.x; so[1] = c.y; so[2] = c.z;
}
EXPORT int or_cull(const float* node8, const float* sphere4) {
  return cull_test(load_node(node8), v3(sphere4[0], sphere4[1], sphere4[2]), sphere4[3]) ? 1 : 0;
}
/* ray8 = o, tmin, d, tmax; tri9 = v0, e1, e2. Returns 1 and *t on a hit. */
EXPORT int or_mt(const float* ray8, const float* tri9, float* t) {
  return moller_trumbore(v3(ray8[0], ray8[1], ray8[2]), v3(ray8[4], ray8[5], ray8[6]), ray8[3], ray8[7],
                         v3(tri9[0], tri9[1], tri9[2]), v3(tri9[3], tri9[4], tri9[5]),
                         v3(tri9[6], tri9[7], tri9[8]), t) ? 1 : 0;
}
EXPORT void or_tri_sphere(const float* tri9v, float* out4) {   // tri9v = v0, v1, v2 (vertices)
  D3 p[3];
  for (int k = 0; k < 3; ++k) p[k] = {tri9v[3 * k], tri9v[3 * k + 1], tri9v[3 * k + 2]};
  finalize_sphere(tri_sphere_center(p[0], p[1], p[2]), p, 3, out4);
}
EXPORT int or_miniball(const float* pts, int64_t n, float* out4) {
  if (n <= 0) return 2;   // "no points"
  std::vector<D3> L(n);
  for (int64_t i = 0; i < n; ++i) L[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
  std::vector<D3> keep(L);
  D3 R[4];
  Ball b = mtf_mb(L, L.size(), R, 0);
  finalize_sphere(b.c, keep.data(), keep.size(), out4);
  return 0;
}

/* Scene preparation (untimed): per-triangle v0/e1/e2 and padded
 * minimal spheres, per-mesh padded miniballs, AABB, pad and eps_t (R2, R3).
 * mesh_ids must be non-decreasing and dense from 0. consts out:
 * [min.xyz, max.xyz, pad, eps_t]. */
EXPORT int or_scene_prep(const float* tris, const int32_t* mesh_ids, int64_t M, int32_t n_meshes,
                         float* tri_e /*M*9*/, float* tri_sph /*M*4*/, float* mesh_sph /*n*4*/,
                         int64_t* mesh_range /*n*2*/, float* consts /*8*/, float pad_in, float eps_in,
                         const float* mesh_sph_in) {
  float mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t t = 0; t < M; ++t)
    for (int v = 0; v < 3; ++v)
      for (int k = 0; k < 3; ++k) {
        mn[k] = fminf(mn[k], tris[9 * t + 3 * v + k]);
        mx[k] = fmaxf(mx[k], tris[9 * t + 3 * v + k]);
      }
  double diag = 0.0;
  for (int k = 0; k < 3; ++k) { double e = (double)mx[k] - (double)mn[k]; diag += e * e; }
  diag = std::sqrt(diag);
  // a transformed scene keeps the creation-time pad and eps_t (pad_in >= 0)
  const float pad = pad_in >= 0.0f ? pad_in : (float)(1e-5 * diag), eps_t = pad_in >= 0.0f ? eps_in : (float)(1e-4 * diag);
  for (int k = 0; k < 3; ++k) { consts[k] = mn[k]; consts[3 + k] = mx[k]; }
  consts[6] = pad; consts[7] = eps_t;
  for (int64_t t = 0; t < M; ++t) {
    const float* v = tris + 9 * t;
    V3 v0 = v3(v[0], v[1], v[2]), v1 = v3(v[3], v[4], v[5]), v2 = v3(v[6], v[7], v[8]);
    V3 e1 = sub(v1, v0), e2 = sub(v2, v0);
    float* o = tri_e + 9 * t;
    o[0] = v0.x; o[1] = v0.y; o[2] = v0.z; o[3] = e1.x; o[4] = e1.y; o[5] = e1.z; o[6] = e2.x; o[7] = e2.y; o[8] = e2.z;
    or_tri_sphere(v, tri_sph + 4 * t);
    tri_sph[4 * t + 3] += pad;
  }
  for (int32_t m = 0; m < n_meshes; ++m) { mesh_range[2 * m] = 0; mesh_range[2 * m + 1] = 0; }
  for (int64_t t = 0; t < M; ++t) {
    if (t > 0 && mesh_ids[t] < mesh_ids[t - 1]) return 2;
    if (mesh_ids[t] < 0 || mesh_ids[t] >= n_meshes) return 2;
  }
  int64_t t0 = 0;
  for (int32_t m = 0; m < n_meshes; ++m) {
    int64_t t1 = t0;
    while (t1 < M && mesh_ids[t1] == m) ++t1;
    mesh_range[2 * m] = t0; mesh_range[2 * m + 1] = t1;
    if (mesh_sph_in) {   // bounding-volume update result: no recomputation
      for (int k = 0; k < 4; ++k) mesh_sph[4 * m + k] = mesh_sph_in[4 * m + k];
    } else if (t1 > t0) {
      or_miniball(tris + 9 * t0, 3 * (t1 - t0), mesh_sph + 4 * m);
      mesh_sph[4 * m + 3] += pad;
    } else {
      mesh_sph[4 * m] = mesh_sph[4 * m + 1] = mesh_sph[4 * m + 2] = 0.0f;
      mesh_sph[4 * m + 3] = -1.0f;
    }
    t0 = t1;
  }
  return 0;
}

/* Secondary ray generation + hashing (§3.3.2; R4, R5), one slot per
 * (type, light, pixel) in canonical slot order: SH light 0 pixels 0..P-1, SH
 * light 1, ..., then RE pixels, then RR pixels (only requested types).
 * Outputs per slot: ray8 (o, tmin, d, tmax), key, empty flag (1 = no ray:
 * P:91 "a 0 or a 1, indicating if there is a ray or not, respectively"). */
EXPORT int64_t or_generate(int32_t P, const float* pos, const float* nrm, const int32_t* mat,
                           const float* materials, int32_t n_mat, const float* eye, const float* dir,
                           const float* lights, int32_t n_lights, uint32_t types, const float* box_min,
                           const float* box_ext, float eps_t, uint32_t flags, float* rays, uint32_t* keys,
                           uint32_t* empty) {
  const bool zorder = (flags & 4u) != 0;   // CRSH_F_ZORDER
  int64_t slot = 0;
  auto fragment = [&](int32_t p) { return v3(pos[p], pos[P + p], pos[2 * (int64_t)P + p]); };
  auto normal = [&](int32_t p) { return v3(nrm[p], nrm[P + p], nrm[2 * (int64_t)P + p]); };
  auto put = [&](int64_t s, V3 o, float tmin, V3 d, float tmax) {
    float* r = rays + 8 * s;
    r[0] = o.x; r[1] = o.y; r[2] = o.z; r[3] = tmin; r[4] = d.x; r[5] = d.y; r[6] = d.z; r[7] = tmax;
  };
  if (types & 1u) {   // shadow rays: origin inverted to the light
    for (int32_t l = 0; l < n_lights; ++l) {
      V3 L = v3(lights[3 * l], lights[3 * l + 1], lights[3 * l + 2]);
      for (int32_t p = 0; p < P; ++p, ++slot) {
        if (mat[p] < 0 || mat[p] >= n_mat) { empty[slot] = 1; keys[slot] = 0; continue; }
        V3 v = sub(fragment(p), L);
        float len = len3(v);
        V3 d = len > 0.0f ? scale(v, 1.0f / len) : v3(0.0f, 0.0f, 1.0f);
        put(slot, L, eps_t, d, len - eps_t);
        keys[slot] = hash_shadow((uint32_t)l, d, zorder);
        empty[slot] = 0;
      }
    }
  }
  for (int type = 2; type <= 4; type *= 2) {
    if (!(types & (uint32_t)type)) continue;
    for (int32_t p = 0; p < P; ++p, ++slot) {
      empty[slot] = 1; keys[slot] = 0;
      if (mat[p] < 0 || mat[p] >= n_mat) continue;
      const float* mt = materials + 3 * mat[p];
      V3 x = fragment(p);
      // view vector: from the camera (primary G-buffer), or the given incident
      // direction of a later Whitted bounce
      V3 i = dir ? v3(dir[p], dir[P + p], dir[2 * (int64_t)P + p]) : norm3(sub(x, v3(eye[0], eye[1], eye[2])));
      V3 n = normal(p);
      V3 d;
      if (type == 2) {   // reflection (mirror), emitted iff reflectivity > 0
        if (!(mt[0] > 0.0f)) continue;
        if (dot3(i, n) > 0.0f) n = neg(n);
        float k2 = 2.0f * dot3(i, n);
        d = norm3(v3(fmaf(-k2, n.x, i.x), fmaf(-k2, n.y, i.y), fmaf(-k2, n.z, i.z)));
      } else {           // refraction (Snell), emitted iff transmissivity > 0 and no TIR
        if (!(mt[1] > 0.0f)) continue;
        float c = -dot3(i, n), eta;
        if (c < 0.0f) { n = neg(n); c = -c; eta = mt[2]; } else { eta = 1.0f / mt[2]; }
        float k = 1.0f - (eta * eta) * (1.0f - c * c);
        if (k < 0.0f) continue;
        float t1 = eta * c - sqrtf(k);
        d = norm3(v3(fmaf(eta, i.x, t1 * n.x), fmaf(eta, i.y, t1 * n.y), fmaf(eta, i.z, t1 * n.z)));
      }
      put(slot, x, eps_t, d, INFINITY);
      keys[slot] = hash_bounce(x, d, box_min, box_ext, zorder);
      empty[slot] = 0;
    }
  }
  return slot;
}

/* Trimming (Fig 4): inclusive scan of the head flags (1 = empty)
 * gives each pair its left shift. Returns the number of kept pairs. */
EXPORT int64_t or_trim(int64_t n, const uint32_t* empty, const uint32_t* keys, const uint32_t* vals,
                       uint32_t* keys_out, uint32_t* vals_out) {
  std::vector<uint64_t> scan(n);
  uint64_t acc = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (empty[i] > 1u) return -1;   // S:169 flag value other than 0/1
    acc += empty[i];
    scan[i] = acc;                  // inclusive scan [MG09]
  }
  int64_t kept = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (empty[i]) continue;
    keys_out[i - scan[i]] = keys[i];
    vals_out[i - scan[i]] = vals[i];
    ++kept;
  }
  return kept;
}

/* Compression into chunks (Fig 5): head flag 1 where the key
 * differs from the previous pair, inclusive scan, chunk key/base/size. */
EXPORT int64_t or_compress(int64_t n, const uint32_t* keys, uint32_t* ckey, uint32_t* cbase, uint32_t* csize) {
  if (n == 0) return 0;
  std::vector<uint32_t> head(n), scan(n);
  for (int64_t i = 0; i < n; ++i) head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
  uint32_t acc = 0;
  for (int64_t i = 0; i < n; ++i) { acc += head[i]; scan[i] = acc; }
  const int64_t C = acc;
  for (int64_t i = 0; i < n; ++i) {
    uint32_t c = scan[i] - 1;
    if (head[i]) { ckey[c] = keys[i]; cbase[c] = (uint32_t)i; csize[c] = 0; }
    csize[c] += 1;
  }
  return C;
}

/* Sorting (§3.3.4: radix sort of the chunks by key; a stable sort
 * of the chunk indices by key -- LSD radix sort is stable) and decompression
 * (Fig 6: skeleton of sorted sizes, exclusive scan, fill). */
EXPORT void or_sort_decompress(int64_t C, const uint32_t* ckey, const uint32_t* cbase, const uint32_t* csize,
                               const uint32_t* vals, uint32_t* skeys, uint32_t* svals, uint32_t* sorted_chunk) {
  std::vector<uint32_t> order(C);
  for (int64_t c = 0; c < C; ++c) order[c] = (uint32_t)c;
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return ckey[a] < ckey[b]; });
  std::vector<uint64_t> skel(C), start(C);
  for (int64_t c = 0; c < C; ++c) skel[c] = csize[order[c]];
  uint64_t acc = 0;
  for (int64_t c = 0; c < C; ++c) { start[c] = acc; acc += skel[c]; }   // exclusive scan
  for (int64_t c = 0; c < C; ++c) {
    if (sorted_chunk) sorted_chunk[c] = order[c];
    for (uint64_t j = 0; j < skel[c]; ++j) {
      skeys[start[c] + j] = ckey[order[c]];
      svals[start[c] + j] = vals[cbase[order[c]] + j];
    }
  }
}

namespace {
// balanced pairwise union over the aligned power-of-two range [lo, lo+size) of
// `count` present items (R9); items beyond `count` are missing (pass through).
template <class Get>
Node balanced(int64_t lo, int64_t size, int64_t count, const Get& get) {
  if (lo >= count) return EMPTY_NODE;
  if (size == 1) return get(lo);
  int64_t h = size / 2;
  return node_union(balanced(lo, h, count, get), balanced(lo + h, h, count, get));
}
}  // namespace

/* First level of the hierarchy: node j holds sorted rays
 * [j*B0, min((j+1)*B0, n)); sphere = balanced Eqs 7-8 over radius-0 origin
 * spheres (R9), cone = sequential Eqs 1-4 from (d_first, 0) in sorted order. */
EXPORT int64_t or_build_leaves(int64_t n, const float* rays, int32_t B0, float* nodes) {
  int64_t nl = (n + B0 - 1) / B0;
  for (int64_t j = 0; j < nl; ++j) {
    int64_t lo = j * B0, cnt = std::min<int64_t>(B0, n - lo);
    Node s = balanced(0, B0, cnt, [&](int64_t i) {
      const float* r = rays + 8 * (lo + i);
      return Node{v3(r[0], r[1], r[2]), 0.0f, v3(0, 0, 1), 0.0f};
    });
    const float* r0 = rays + 8 * lo;
    V3 x = v3(r0[4], r0[5], r0[6]);
    float phi = 0.0f;   // leaves: "a cone with spread angle equal to 0"
    for (int64_t i = 1; i < cnt; ++i) {
      const float* r = rays + 8 * (lo + i);
      cone_grow(x, phi, v3(r[4], r[5], r[6]), &x, &phi);
    }
    Node nd = {s.c, s.r, x, phi};
    store_node(nodes + 8 * j, nd);
  }
  return nl;
}

/* Upper level: node j = balanced union (Eqs 5-8) of children
 * [j*B, min((j+1)*B, n_children)). */
EXPORT int64_t or_build_upper(int64_t n_children, const float* children, int32_t B, float* nodes) {
  int64_t np = (n_children + B - 1) / B;
  for (int64_t j = 0; j < np; ++j) {
    int64_t lo = j * B, cnt = std::min<int64_t>(B, n_children - lo);
    Node u = balanced(0, B, cnt, [&](int64_t i) { return load_node(children + 8 * (lo + i)); });
    store_node(nodes + 8 * j, u);
  }
  return np;
}

/* Top-down traversal with mesh culling and final closest-hit tests
 * (§3.3.7-3.3.8), counting per the paper's convention (
 * SURVEY F1, R14). level_nodes[k-1] / level_count[k-1] = level k (1 = leaves,
 * Lv = top). best[n_rays] is initialised to UINT64_MAX by the caller and
 * receives min over packed (t, tri). counters out (uint64):
 * [tests[1..8], hits[1..8], mesh_tests, mesh_hits, final_tests, final_hits]
 * -> tests[k] at out[k-1], hits[k] at out[8+k-1], then 16..19. */
/* Object sphere-tree ("combine our coherent ray
 * hierarchy with a deeper object hierarchy"), reading O1: below
 * each mesh sphere, the mesh's triangles are ordered by the 30-bit Morton code
 * of their centroid (((v0 + v1) + v2) / 3 in double) quantised to 1024 cells
 * per axis of the mesh's vertex bounding box (q = floor(((c - lo) / (hi - lo))
 * * 1024) clamped to [0, 1023], 0 on a flat axis), ties by triangle index, and
 * cut into clusters of CL consecutive triangles of that order (the last one of
 * a mesh may be shorter). A cluster is bounded by the sphere centred at the
 * midpoint of its vertices' bounding box (double, rounded to float) with
 * radius = the largest distance from that float centre to a vertex (double,
 * rounded up) + pad -- the triangle spheres' finalisation. order_in (nullable):
 * a given order (a moved scene keeps its creation-time order, reading G2);
 * out_order [M]: the order (triangle ids, mesh by mesh); out_sph [clusters][4];
 * mesh_cluster_first [n_meshes + 1]. Returns the number of clusters. */
EXPORT int64_t or_cluster_spheres(const float* tris, const int64_t* mesh_range, int32_t n_meshes, int32_t CL, float pad,
                                  const int32_t* order_in, int32_t* out_order, float* out_sph,
                                  int64_t* mesh_cluster_first) {
  auto spread3 = [](uint64_t v) {   // 10 bits -> every third bit
    uint64_t r = 0;
    for (int b = 0; b < 10; ++b) r |= ((v >> b) & 1ull) << (3 * b);
    return r;
  };
  int64_t nc = 0;
  for (int32_t m = 0; m < n_meshes; ++m) {
    mesh_cluster_first[m] = nc;
    const int64_t t0 = mesh_range[2 * m], t1 = mesh_range[2 * m + 1];
    if (order_in) {
      for (int64_t t = t0; t < t1; ++t) out_order[t] = order_in[t];
    } else {
      double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int64_t i = 9 * t0; i < 9 * t1; ++i) {
        lo[i % 3] = std::min(lo[i % 3], (double)tris[i]);
        hi[i % 3] = std::max(hi[i % 3], (double)tris[i]);
      }
      std::vector<std::pair<uint64_t, int64_t>> key;
      for (int64_t t = t0; t < t1; ++t) {
        uint64_t code = 0;
        for (int k = 0; k < 3; ++k) {
          const float* v = tris + 9 * t;
          const double c = (((double)v[k] + (double)v[3 + k]) + (double)v[6 + k]) / 3.0;
          uint64_t q = 0;
          if (hi[k] > lo[k]) {
            const double u = std::floor(((c - lo[k]) / (hi[k] - lo[k])) * 1024.0);
            q = u <= 0.0 ? 0 : (u >= 1023.0 ? 1023 : (uint64_t)u);
          }
          code |= spread3(q) << (2 - k);   // x highest
        }
        key.push_back({code, t});
      }
      std::sort(key.begin(), key.end());   // (code, index): ties by triangle index
      for (int64_t i = 0; i < (int64_t)key.size(); ++i) out_order[t0 + i] = (int32_t)key[i].second;
    }
    for (int64_t c0 = t0; c0 < t1; c0 += CL) {
      const int64_t c1 = std::min<int64_t>(c0 + CL, t1);
      std::vector<D3> pts;
      double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int64_t i = c0; i < c1; ++i)
        for (int v = 0; v < 3; ++v) {
          const float* p = tris + 9 * (int64_t)out_order[i] + 3 * v;
          pts.push_back(D3{p[0], p[1], p[2]});
          const double q[3] = {p[0], p[1], p[2]};
          for (int k = 0; k < 3; ++k) { lo[k] = std::min(lo[k], q[k]); hi[k] = std::max(hi[k], q[k]); }
        }
      const D3 c = {(lo[0] + hi[0]) * 0.5, (lo[1] + hi[1]) * 0.5, (lo[2] + hi[2]) * 0.5};
      finalize_sphere(c, pts.data(), pts.size(), out_sph + 4 * nc);
      out_sph[4 * nc + 3] += pad;
      ++nc;
    }
  }
  mesh_cluster_first[n_meshes] = nc;
  return nc;
}

EXPORT void or_traverse(int32_t Lv, int32_t B0, int32_t B, const float* const* level_nodes,
                        const int64_t* level_count, int64_t n_rays, const float* rays, const float* tri_e,
                        const float* tri_sph, int32_t n_meshes, const float* mesh_sph,
                        const int64_t* mesh_range, uint32_t flags, int32_t n_threads, uint64_t* best,
                        uint64_t* counters_out, const float* cluster_sph, const int64_t* mesh_cluster_first,
                        int32_t CL, const int32_t* cluster_order) {
  const bool mesh_cull = (flags & 2u) != 0;
  const bool objtree = (flags & 64u) != 0 && cluster_sph && cluster_order && CL > 0;   // CRSH_F_OBJTREE
  const int64_t n_top = level_count[Lv - 1];
  std::atomic<int64_t> next{0};
  std::vector<Counters> per_thread(std::max(1, n_threads));

  auto worker = [&](int tid) {
    Counters& C = per_thread[tid];
    // descend(k, node, tri): the pair (node at level k, tri) passed; test children.
    std::function<void(int, int64_t, int64_t)> descend = [&](int k, int64_t n, int64_t t) {
      if (k == 1) {   // final intersection tests against every ray of the bundle
        const float* te = tri_e + 9 * t;
        for (int64_t r = n * B0; r < std::min<int64_t>((n + 1) * B0, n_rays); ++r) {
          const float* ry = rays + 8 * r;
          C.final_tests++;
          float th;
          if (moller_trumbore(v3(ry[0], ry[1], ry[2]), v3(ry[4], ry[5], ry[6]), ry[3], ry[7],
                              v3(te[0], te[1], te[2]), v3(te[3], te[4], te[5]), v3(te[6], te[7], te[8]), &th)) {
            C.final_hits++;
            best[r] = std::min(best[r], pack_hit(th, (uint32_t)t));
          }
        }
        return;
      }
      const float* sp = tri_sph + 4 * t;
      for (int64_t c = n * B; c < std::min<int64_t>((n + 1) * B, level_count[k - 2]); ++c) {
        C.tests[k - 2]++;
        if (cull_test(load_node(level_nodes[k - 2] + 8 * c), v3(sp[0], sp[1], sp[2]), sp[3])) {
          C.hits[k - 2]++;
          descend(k - 1, c, t);
        }
      }
    };
    for (;;) {
      int64_t n = next.fetch_add(1);
      if (n >= n_top) break;
      Node top = load_node(level_nodes[Lv - 1] + 8 * n);
      for (int32_t m = 0; m < n_meshes; ++m) {
        if (mesh_range[2 * m + 1] <= mesh_range[2 * m]) continue;
        if (mesh_cull) {   // whole-mesh culling at the top level
          C.mesh_tests++;
          const float* ms = mesh_sph + 4 * m;
          if (!cull_test(top, v3(ms[0], ms[1], ms[2]), ms[3])) continue;
          C.mesh_hits++;
        }
        // top-level tests of the triangles at [ta, tb) of the mesh's index order
        // (objtree: of its cluster order)
        auto triangles = [&](int64_t ta, int64_t tb) {
          for (int64_t i = ta; i < tb; ++i) {
            const int64_t t = objtree ? (int64_t)cluster_order[i] : i;
            const float* sp = tri_sph + 4 * t;
            C.tests[Lv - 1]++;
            if (cull_test(top, v3(sp[0], sp[1], sp[2]), sp[3])) {
              C.hits[Lv - 1]++;
              descend(Lv, n, t);
            }
          }
        };
        if (!objtree) {
          triangles(mesh_range[2 * m], mesh_range[2 * m + 1]);
          continue;
        }
        // the object sphere-tree level: Eq 9 against each cluster sphere of the mesh
        for (int64_t c = mesh_cluster_first[m]; c < mesh_cluster_first[m + 1]; ++c) {
          C.cluster_tests++;
          const float* cs = cluster_sph + 4 * c;
          if (!cull_test(top, v3(cs[0], cs[1], cs[2]), cs[3])) continue;
          C.cluster_hits++;
          const int64_t ta = mesh_range[2 * m] + (c - mesh_cluster_first[m]) * CL;
          triangles(ta, std::min<int64_t>(ta + CL, mesh_range[2 * m + 1]));
        }
      }
    }
  };
  std::vector<std::thread> th;
  for (int i = 1; i < n_threads; ++i) th.emplace_back(worker, i);
  worker(0);
  for (auto& t : th) t.join();
  Counters tot;
  for (auto& c : per_thread) tot.add(c);
  for (int k = 0; k < 8; ++k) { counters_out[k] = tot.tests[k]; counters_out[8 + k] = tot.hits[k]; }
  counters_out[16] = tot.mesh_tests; counters_out[17] = tot.mesh_hits;
  counters_out[18] = tot.final_tests; counters_out[19] = tot.final_hits;
  counters_out[20] = tot.cluster_tests; counters_out[21] = tot.cluster_hits;
}

/* Whole-mesh culling alone, the first step of
 * or_traverse's top-node loop without the descent: for every top node and every
 * non-empty mesh one Eq 9 test against the mesh sphere; out3 = {mesh tests,
 * mesh passes, triangles of the passing meshes}. The third number is what
 * or_traverse counts as the top-level tests (tests[Lv], one per triangle of a
 * kept mesh), so it checks that count at sizes where the full traversal is too
 * slow for the oracle. */
EXPORT void or_mesh_cull(int64_t n_top, const float* top_nodes, int32_t n_meshes, const float* mesh_sph,
                         const int64_t* mesh_range, uint64_t* out3) {
  uint64_t tests = 0, hits = 0, kept = 0;
  for (int64_t n = 0; n < n_top; ++n) {
    Node top = load_node(top_nodes + 8 * n);
    for (int32_t m = 0; m < n_meshes; ++m) {
      if (mesh_range[2 * m + 1] <= mesh_range[2 * m]) continue;
      tests++;
      const float* ms = mesh_sph + 4 * m;
      if (!cull_test(top, v3(ms[0], ms[1], ms[2]), ms[3])) continue;
      hits++;
      kept += (uint64_t)(mesh_range[2 * m + 1] - mesh_range[2 * m]);
    }
  }
  out3[0] = tests; out3[1] = hits; out3[2] = kept;
}

/* Naive N x M ray tracing: closest hit of every ray over all triangles,
 * the plain definition the conservative CRSH path must reproduce (A1). */
EXPORT void or_brute(int64_t n_rays, const float* rays, int64_t M, const float* tri_e, int32_t n_threads,
                     uint64_t* best) {
  std::atomic<int64_t> next{0};
  auto worker = [&]() {
    for (;;) {
      int64_t r0 = next.fetch_add(64);
      if (r0 >= n_rays) break;
      for (int64_t r = r0; r < std::min<int64_t>(r0 + 64, n_rays); ++r) {
        const float* ry = rays + 8 * r;
        uint64_t b = UINT64_MAX;
        for (int64_t t = 0; t < M; ++t) {
          const float* te = tri_e + 9 * t;
          float th;
          if (moller_trumbore(v3(ry[0], ry[1], ry[2]), v3(ry[4], ry[5], ry[6]), ry[3], ry[7],
                              v3(te[0], te[1], te[2]), v3(te[3], te[4], te[5]), v3(te[6], te[7], te[8]), &th))
            b = std::min(b, pack_hit(th, (uint32_t)t));
        }
        best[r] = b;
      }
    }
  };
  std::vector<std::thread> th;
  for (int i = 1; i < n_threads; ++i) th.emplace_back(worker);
  worker();
  for (auto& t : th) t.join();
}

/* ---------------------------------------------------------------------------
 * Multi-bounce Whitted loop ("accumulate
 * shading ... output another set of secondary rays onto the ray array ... and
 * continue"; SPEC S:514-522 shade_and_spawn, [Whi80]). A bounce is a set of
 * VERTICES laid out like a G-buffer (pos, winding normal, material, incident
 * direction); tracing it with crsh's secondary pass gives the shadow-ray
 * visibility of every light and the closest hits of the reflection and
 * refraction rays, which become the next bounce's vertices. Radiance is then
 * assembled bottom-up:  L(v) = direct(v) + refl(v) L(re child) + trans(v) L(rr child).
 * Readings (W1-W4): white lights of intensity 1/n_lights;
 * diffuse weight kd = max(0, 1 - refl - trans); Lambert with the normal turned
 * toward the incoming ray; background (miss) radiance 0.
 * ------------------------------------------------------------------------- */

/* direct term per vertex from the shadow rays of this bounce (slots l*P + v):
 * a light counts iff its shadow ray found no occluder (hit_tri == -1). */
EXPORT void or_shade(int32_t P, const float* pos, const float* nrm, const int32_t* mat, const float* materials,
                     int32_t n_mat, const float* eye, const float* dir, const float* lights, int32_t n_lights,
                     const int32_t* hit_tri, float* direct) {
  for (int32_t v = 0; v < P; ++v) {
    direct[v] = 0.0f;
    if (mat[v] < 0 || mat[v] >= n_mat || n_lights <= 0) continue;
    const float* mt = materials + 3 * mat[v];
    const float kd = fmaxf(0.0f, (1.0f - mt[0]) - mt[1]);
    V3 x = v3(pos[v], pos[P + v], pos[2 * (int64_t)P + v]);
    V3 n = v3(nrm[v], nrm[P + v], nrm[2 * (int64_t)P + v]);
    V3 i = dir ? v3(dir[v], dir[P + v], dir[2 * (int64_t)P + v]) : norm3(sub(x, v3(eye[0], eye[1], eye[2])));
    if (dot3(i, n) > 0.0f) n = neg(n);   // face the incoming side
    float acc = 0.0f;
    for (int32_t l = 0; l < n_lights; ++l) {
      if (hit_tri[(int64_t)l * P + v] != -1) continue;   // occluded
      V3 lv = sub(v3(lights[3 * l], lights[3 * l + 1], lights[3 * l + 2]), x);
      const float len = len3(lv);
      const float c = dot3(n, lv);
      if (c > 0.0f && len > 0.0f) acc = acc + c / len;
    }
    direct[v] = (kd * acc) * (1.0f / (float)n_lights);
  }
}

/* next bounce's vertices from this bounce's RE / RR closest hits, in vertex
 * order (RE child before RR child): pos = o + t d (fma per axis), normal =
 * norm(e1 x e2) of the hit triangle, material of the triangle, incident
 * direction d. c_re / c_rr: child index or -1. Returns the vertex count. */
EXPORT int64_t or_spawn(int32_t P, int32_t n_lights, uint32_t types, const float* rays, const int32_t* hit_tri,
                        const float* t, const float* tri_e, const int32_t* tri_mat, int64_t cap, float* npos,
                        float* nnrm, int32_t* nmat, float* ndir, int32_t* c_re, int32_t* c_rr) {
  const int64_t sh = (types & 1u) ? (int64_t)n_lights * P : 0;
  const int64_t re0 = sh, rr0 = sh + ((types & 2u) ? P : 0);
  int64_t k = 0;
  std::vector<int64_t> src;   // slot of each child
  for (int32_t v = 0; v < P; ++v) {
    c_re[v] = c_rr[v] = -1;
    if ((types & 2u) && hit_tri[re0 + v] >= 0) { c_re[v] = (int32_t)k++; src.push_back(re0 + v); }
    if ((types & 4u) && hit_tri[rr0 + v] >= 0) { c_rr[v] = (int32_t)k++; src.push_back(rr0 + v); }
  }
  if (k > cap) return -1;
  for (int64_t c = 0; c < k; ++c) {
    const int64_t s = src[c];
    const float* r = rays + 8 * s;
    const float th = t[s];
    const int32_t tri = hit_tri[s];
    const float* te = tri_e + 9 * (int64_t)tri;
    V3 nn = norm3(cross3(v3(te[3], te[4], te[5]), v3(te[6], te[7], te[8])));
    npos[c] = fmaf(th, r[4], r[0]); npos[k + c] = fmaf(th, r[5], r[1]); npos[2 * k + c] = fmaf(th, r[6], r[2]);
    nnrm[c] = nn.x; nnrm[k + c] = nn.y; nnrm[2 * k + c] = nn.z;
    ndir[c] = r[4]; ndir[k + c] = r[5]; ndir[2 * k + c] = r[6];
    nmat[c] = tri_mat[tri];
  }
  return k;
}

/* L(v) = direct(v), then + refl L(re child), then + trans L(rr child) (fma). */
EXPORT void or_backprop(int32_t P, const int32_t* mat, const float* materials, int32_t n_mat, const float* direct,
                        const int32_t* c_re, const int32_t* c_rr, const float* L_next, float* L) {
  for (int32_t v = 0; v < P; ++v) {
    float r = direct[v];
    if (mat[v] >= 0 && mat[v] < n_mat) {
      const float* mt = materials + 3 * mat[v];
      if (c_re && c_re[v] >= 0) r = fmaf(mt[0], L_next[c_re[v]], r);
      if (c_rr && c_rr[v] >= 0) r = fmaf(mt[1], L_next[c_rr[v]], r);
    }
    L[v] = r;
  }
}

/* ---------------------------------------------------------------------------
 * GPU primary pass mirror. cam = eye[3],
 * right[3], up[3], fwd[3], tan_half_vfov (13 floats); pixel (i, j), j = 0 at
 * the top, ray through the pixel centre.
 * ------------------------------------------------------------------------- */
EXPORT void or_camera_rays(const float* cam, int32_t W, int32_t H, float* rays) {
  const float ax = cam[12] * ((float)W / (float)H);
  for (int32_t j = 0; j < H; ++j)
    for (int32_t i = 0; i < W; ++i) {
      const float u = ((float)(2 * i + 1) / (float)W - 1.0f) * ax;
      const float v = (1.0f - (float)(2 * j + 1) / (float)H) * cam[12];
      V3 dd = v3(fmaf(u, cam[3], fmaf(v, cam[6], cam[9])), fmaf(u, cam[4], fmaf(v, cam[7], cam[10])),
                 fmaf(u, cam[5], fmaf(v, cam[8], cam[11])));
      V3 d = norm3(dd);
      float* r = rays + 8 * ((int64_t)j * W + i);
      r[0] = cam[0]; r[1] = cam[1]; r[2] = cam[2]; r[3] = 0.0f;
      r[4] = d.x; r[5] = d.y; r[6] = d.z; r[7] = INFINITY;
    }
}

/* keys / empty flags of a given ray batch: the bounce-ray hash of (o, d);
 * a ray with !(tmax > tmin) is an empty slot. */
EXPORT void or_keys_given(int64_t n, const float* rays, const float* box_min, const float* box_ext, uint32_t flags,
                          uint32_t* keys, uint32_t* empty) {
  const bool zorder = (flags & 4u) != 0;
  for (int64_t s = 0; s < n; ++s) {
    const float* r = rays + 8 * s;
    if (!(r[7] > r[3])) { empty[s] = 1; keys[s] = 0; continue; }
    keys[s] = hash_bounce(v3(r[0], r[1], r[2]), v3(r[4], r[5], r[6]), box_min, box_ext, zorder);
    empty[s] = 0;
  }
}

/* G-buffer from the primary hits: pos = fma(t, d, o), n = norm(e1 x e2)
 * turned toward the camera, material of the triangle; miss -> 0, 0, -1. */
EXPORT void or_gbuffer(int64_t P, const float* rays, const int32_t* hit_tri, const float* t, const float* tri_e,
                       const int32_t* tri_mat, float* pos, float* nrm, int32_t* mat) {
  for (int64_t p = 0; p < P; ++p) {
    const int32_t h = hit_tri[p];
    if (h < 0) {
      pos[p] = pos[P + p] = pos[2 * P + p] = 0.0f;
      nrm[p] = nrm[P + p] = nrm[2 * P + p] = 0.0f;
      mat[p] = -1;
      continue;
    }
    const float* r = rays + 8 * p;
    const float* te = tri_e + 9 * (int64_t)h;
    V3 n = norm3(cross3(v3(te[3], te[4], te[5]), v3(te[6], te[7], te[8])));
    V3 d = v3(r[4], r[5], r[6]);
    if (dot3(d, n) > 0.0f) n = neg(n);
    pos[p] = fmaf(t[p], r[4], r[0]); pos[P + p] = fmaf(t[p], r[5], r[1]); pos[2 * P + p] = fmaf(t[p], r[6], r[2]);
    nrm[p] = n.x; nrm[P + p] = n.y; nrm[2 * P + p] = n.z;
    mat[p] = tri_mat[h];
  }
}

/* ---------------------------------------------------------------------------
 * Dynamic scenes (§3.3.1 Bounding Volume Update, P:75-77;
 * S:226-234): per-mesh affine transforms xf = [A | b] (3x4 row-major) applied
 * to the creation-time vertices; the mesh spheres are UPDATED, not recomputed
 * ("we only update the center and the radius"): c' = A c + b, r' = r sigma_max(A)
 * (largest singular value, conservative), rounded up.
 * ------------------------------------------------------------------------- */
static inline float xf_axis(const float* xf, int row, float x, float y, float z) {
  return fmaf(xf[4 * row], x, fmaf(xf[4 * row + 1], y, fmaf(xf[4 * row + 2], z, xf[4 * row + 3])));
}

EXPORT void or_transform(const float* tris, const int32_t* mesh_ids, int64_t M, const float* xf, float* out) {
  for (int64_t t = 0; t < M; ++t) {
    const float* a = xf + 12 * mesh_ids[t];
    for (int v = 0; v < 3; ++v) {
      const float* p = tris + 9 * t + 3 * v;
      for (int r = 0; r < 3; ++r) out[9 * t + 3 * v + r] = xf_axis(a, r, p[0], p[1], p[2]);
    }
  }
}

/* sigma_max(A) = sqrt(largest eigenvalue of A^T A), closed form for the
 * symmetric 3x3 (trigonometric method), double precision. */
EXPORT double or_sigma_max(const float* xf) {
  double A[3][3], S[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) A[r][c] = (double)xf[4 * r + c];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) S[i][j] = A[0][i] * A[0][j] + A[1][i] * A[1][j] + A[2][i] * A[2][j];
  const double p1 = S[0][1] * S[0][1] + S[0][2] * S[0][2] + S[1][2] * S[1][2];
  double lam;
  if (p1 == 0.0) {
    lam = std::max(S[0][0], std::max(S[1][1], S[2][2]));
  } else {
    const double q = (S[0][0] + S[1][1] + S[2][2]) / 3.0;
    const double p2 = (S[0][0] - q) * (S[0][0] - q) + (S[1][1] - q) * (S[1][1] - q) + (S[2][2] - q) * (S[2][2] - q) + 2.0 * p1;
    const double p = std::sqrt(p2 / 6.0);
    double B[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) B[i][j] = (S[i][j] - (i == j ? q : 0.0)) / p;
    const double det = B[0][0] * (B[1][1] * B[2][2] - B[1][2] * B[2][1]) - B[0][1] * (B[1][0] * B[2][2] - B[1][2] * B[2][0]) +
                       B[0][2] * (B[1][0] * B[2][1] - B[1][1] * B[2][0]);
    const double r = det / 2.0;
    const double phi = r <= -1.0 ? M_PI / 3.0 : (r >= 1.0 ? 0.0 : std::acos(r) / 3.0);
    lam = q + 2.0 * p * std::cos(phi);
  }
  return std::sqrt(std::max(lam, 0.0));
}

EXPORT void or_update_sphere(const float* sph, const float* xf, float* out) {
  if (sph[3] < 0.0f) { for (int k = 0; k < 4; ++k) out[k] = sph[k]; return; }   // empty mesh
  for (int r = 0; r < 3; ++r) out[r] = xf_axis(xf, r, sph[0], sph[1], sph[2]);
  const double want = (double)sph[3] * or_sigma_max(xf);
  float rf = (float)want;
  if ((double)rf < want) rf = std::nextafter(rf, INFINITY);
  out[3] = rf;
}
