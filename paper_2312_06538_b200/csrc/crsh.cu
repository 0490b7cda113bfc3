// crsh.cu — host runtime and C ABI of the CRSH library (include/crsh.h):
// scene preparation, a grow-only device arena, the per-frame launch sequence
// K1..K9 on the caller's stream, counters, debug taps. All compute runs in
// the kernels of k_*.cuh; there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/crsh.h"
#include "common.cuh"
#include "k_build.cuh"
#include "k_raygen.cuh"
#include "k_sort.cuh"
#include "k_traverse.cuh"
#include "k_whitted.cuh"
#include "k_primary.cuh"
#include "dist.cuh"

using namespace crsh;

namespace {

thread_local std::string g_err;

crsh_status fail(crsh_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define NCK(call)                                                                                    \
  do {                                                                                               \
    ncclResult_t n_ = (call);                                                                        \
    if (n_ != ncclSuccess) return fail(CRSH_ENCCL, "%s: %s (%s:%d)", #call, ncclGetErrorString(n_),   \
                                       __FILE__, __LINE__);                                          \
  } while (0)

#define CK(call)                                                                                     \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) return fail(e_ == cudaErrorMemoryAllocation ? CRSH_ENOMEM : CRSH_ECUDA,  \
                                       "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

cudaError_t ensure(Buf& b, size_t bytes) {
  if (bytes <= b.cap && b.p) return cudaSuccess;
  b.release();
  size_t want = std::max<size_t>(bytes + bytes / 8, 256);
  cudaError_t e = cudaMalloc(&b.p, want);
  if (e == cudaSuccess) b.cap = want;
  return e;
}

inline uint32_t cdiv(uint64_t a, uint64_t b) { return (uint32_t)((a + b - 1) / b); }
inline uint64_t roundup(uint64_t a, uint64_t b) { return (a + b - 1) / b * b; }

// -------------------------------------------------------------- host miniball (scene prep, P:79 [Gar99])
// Move-to-front Welzl in double: the smallest ball with support set R
// (|R| <= 4) on its boundary, grown point by point.
struct HBall { double c[3]; double r2; };

HBall ball_of(const double (*R)[3], int k) {
  HBall b{{0, 0, 0}, -1.0};
  if (k == 0) return b;
  if (k == 1) { for (int i = 0; i < 3; ++i) b.c[i] = R[0][i]; b.r2 = 0; return b; }
  double a[3], u[3], v[3], w[3];
  for (int i = 0; i < 3; ++i) a[i] = R[0][i];
  auto d2 = [](const double* p, const double* q) {
    return (p[0] - q[0]) * (p[0] - q[0]) + (p[1] - q[1]) * (p[1] - q[1]) + (p[2] - q[2]) * (p[2] - q[2]);
  };
  auto cross = [](const double* p, const double* q, double* o) {
    o[0] = p[1] * q[2] - p[2] * q[1]; o[1] = p[2] * q[0] - p[0] * q[2]; o[2] = p[0] * q[1] - p[1] * q[0];
  };
  auto dot = [](const double* p, const double* q) { return p[0] * q[0] + p[1] * q[1] + p[2] * q[2]; };
  if (k == 2) {
    for (int i = 0; i < 3; ++i) b.c[i] = (R[0][i] + R[1][i]) * 0.5;
    b.r2 = d2(R[0], b.c);
    return b;
  }
  for (int i = 0; i < 3; ++i) { u[i] = R[1][i] - a[i]; v[i] = R[2][i] - a[i]; }
  if (k == 3) {
    double n[3];
    cross(u, v, n);
    const double den = 2.0 * dot(n, n);
    if (den == 0.0) {   // collinear: widest pair
      HBall best = b;
      const int pr[3][2] = {{0, 1}, {0, 2}, {1, 2}};
      for (auto& q : pr) {
        const double P2[2][3] = {{R[q[0]][0], R[q[0]][1], R[q[0]][2]}, {R[q[1]][0], R[q[1]][1], R[q[1]][2]}};
        HBall c = ball_of(P2, 2);
        if (c.r2 > best.r2) best = c;
      }
      return best;
    }
    double nu[3], vn[3];
    cross(n, u, nu);
    cross(v, n, vn);
    const double uu = dot(u, u), vv = dot(v, v);
    for (int i = 0; i < 3; ++i) b.c[i] = a[i] + (nu[i] * vv + vn[i] * uu) / den;
    b.r2 = d2(R[0], b.c);
    return b;
  }
  for (int i = 0; i < 3; ++i) w[i] = R[3][i] - a[i];
  double vw[3], wu[3], uv[3];
  cross(v, w, vw);
  cross(w, u, wu);
  cross(u, v, uv);
  const double det = dot(u, vw);
  if (det == 0.0) {   // coplanar: largest 3-point ball
    HBall best = b;
    for (int skip = 0; skip < 4; ++skip) {
      double P3[3][3];
      int m = 0;
      for (int i = 0; i < 4; ++i) if (i != skip) { for (int c = 0; c < 3; ++c) P3[m][c] = R[i][c]; ++m; }
      HBall c = ball_of(P3, 3);
      if (c.r2 > best.r2) best = c;
    }
    return best;
  }
  const double hu = 0.5 * dot(u, u), hv = 0.5 * dot(v, v), hw = 0.5 * dot(w, w);
  double x[3];
  for (int i = 0; i < 3; ++i) x[i] = (vw[i] * hu + wu[i] * hv + uv[i] * hw) / det;
  for (int i = 0; i < 3; ++i) b.c[i] = a[i] + x[i];
  b.r2 = dot(x, x);
  return b;
}

HBall mtf(std::vector<std::array<double, 3>>& L, size_t n, double (*R)[3], int k) {
  HBall b = ball_of(R, k);
  if (k == 4) return b;
  for (size_t i = 0; i < n; ++i) {
    const double* p = L[i].data();
    const double dd = (p[0] - b.c[0]) * (p[0] - b.c[0]) + (p[1] - b.c[1]) * (p[1] - b.c[1]) +
                      (p[2] - b.c[2]) * (p[2] - b.c[2]);
    if (b.r2 < 0.0 || dd > b.r2 * (1.0 + 1e-13)) {
      for (int c = 0; c < 3; ++c) R[k][c] = p[c];
      b = mtf(L, i, R, k + 1);
      std::rotate(L.begin(), L.begin() + i, L.begin() + i + 1);
    }
  }
  return b;
}

// float centre, radius = max distance from it (rounded up), + pad
void mesh_sphere(const float* tris, int64_t t0, int64_t t1, float pad, float out[4]) {
  std::vector<std::array<double, 3>> L;
  L.reserve(3 * (t1 - t0));
  for (int64_t t = t0; t < t1; ++t)
    for (int v = 0; v < 3; ++v) L.push_back({tris[9 * t + 3 * v], tris[9 * t + 3 * v + 1], tris[9 * t + 3 * v + 2]});
  std::vector<std::array<double, 3>> pts(L);
  double R[4][3];
  HBall b = mtf(L, L.size(), R, 0);
  const float cf[3] = {(float)b.c[0], (float)b.c[1], (float)b.c[2]};
  double r2 = 0.0;
  for (auto& p : pts) {
    const double dx = p[0] - (double)cf[0], dy = p[1] - (double)cf[1], dz = p[2] - (double)cf[2];
    r2 = std::max(r2, dx * dx + dy * dy + dz * dz);
  }
  const double r = std::sqrt(r2);
  float rf = (float)r;
  if ((double)rf < r) rf = std::nextafter(rf, INFINITY);
  out[0] = cf[0]; out[1] = cf[1]; out[2] = cf[2]; out[3] = rf + pad;
}

// Object sphere-tree order (reading O1): per mesh, triangles sorted by the
// 30-bit Morton code of their centroid (((v0 + v1) + v2) / 3, double) in 1024
// cells per axis of the mesh's vertex box (x most significant), ties by
// index; clusters of 32 consecutive triangles of that order.
void cluster_order(const float* tris, const std::vector<uint32_t>& first, const std::vector<uint32_t>& count,
                   std::vector<int32_t>& order, std::vector<uint32_t>& cl_first, std::vector<uint32_t>& cl_range) {
  const size_t nm = first.size();
  size_t M = 0;
  for (size_t m = 0; m < nm; ++m) M += count[m];
  order.assign(M, 0);
  cl_first.assign(nm + 1, 0);
  cl_range.clear();
  auto spread = [](uint64_t v) {
    uint64_t r = 0;
    for (int b = 0; b < 10; ++b) r |= ((v >> b) & 1ull) << (3 * b);
    return r;
  };
  uint32_t nc = 0;
  for (size_t m = 0; m < nm; ++m) {
    cl_first[m] = nc;
    const uint32_t t0 = first[m], n = count[m];
    if (!n) continue;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (size_t i = 9 * (size_t)t0; i < 9 * (size_t)(t0 + n); ++i) {
      lo[i % 3] = std::min(lo[i % 3], (double)tris[i]);
      hi[i % 3] = std::max(hi[i % 3], (double)tris[i]);
    }
    std::vector<std::pair<uint64_t, uint32_t>> key(n);
    for (uint32_t j = 0; j < n; ++j) {
      const float* v = tris + 9 * (size_t)(t0 + j);
      uint64_t code = 0;
      for (int k = 0; k < 3; ++k) {
        uint64_t q = 0;
        if (hi[k] > lo[k]) {
          const double c = (((double)v[k] + (double)v[3 + k]) + (double)v[6 + k]) / 3.0;
          const double u = std::floor(((c - lo[k]) / (hi[k] - lo[k])) * 1024.0);
          q = u <= 0.0 ? 0 : (u >= 1023.0 ? 1023 : (uint64_t)u);
        }
        code |= spread(q) << (2 - k);
      }
      key[j] = {code, t0 + j};
    }
    std::sort(key.begin(), key.end());
    for (uint32_t j = 0; j < n; ++j) order[t0 + j] = (int32_t)key[j].second;
    for (uint32_t c0 = 0; c0 < n; c0 += 32) {
      cl_range.push_back(t0 + c0);
      cl_range.push_back(t0 + std::min(c0 + 32, n));
      ++nc;
    }
  }
  cl_first[nm] = nc;
}

}  // namespace

// ============================================================== scene
// Static (host-known) plan of a frame: slot layout, hierarchy shape and the
// upper bounds every grid and buffer is sized from. The data-dependent counts
// live in the device FrameDesc; `fd` below is its host copy after the frame.
struct FrameInfo {
  bool valid = false;
  int n_seg = 0;
  int seg_type[MAX_SEG] = {0, 0, 0};
  uint64_t S = 0;
  uint32_t seg_slot_start[MAX_SEG + 1] = {0};
  int Lv = 0, B0 = 0, B = 0, K = 0;
  uint32_t span = 0, GR = 0;
  uint64_t Np_max = 0, G_max = 0;
  size_t level_off[MAX_LEVELS + 1] = {0};   // node offset of level k in the node arrays (from the bounds)
  uint64_t level_max[MAX_LEVELS + 1] = {0};
  uint32_t flags = 0;
  uint32_t item_tris = 2048;                // triangles per traversal work item (item_tris_for)
  uint32_t obj_list = CRSH_OBJ_LIST;        // object tree: cluster-list entries used per round (obj_list_for)
  int32_t prefilter = 1;                    // K8 child prefilter (CRSH_NO_PREFILTER=1: off)
  int32_t top_prefilter = 0;                // K8 top-level prefilter (plan_frame; CRSH_TOP_PREFILTER=0|1)
  bool big_tiles = false;                   // k_rle / k_scan_sizes with 8192-entry tiles (large frames)
  bool rle_hist = true;                     // k_rle builds the radix digit histograms (no k_radix_hist pass)
  int rank = 0, world = 1;
  bool sorted = false, timed = false, ktimed = false, brute = false;
  const float4* in_rays = nullptr;          // ray-batch mode (crsh_trace_rays)
  FrameDesc fd{};                           // host copy of the device counts (refreshed lazily)
  bool fd_fresh = false;
};

struct crsh_scene {
  int device = 0;
  int64_t M = 0;
  int32_t n_meshes = 0, n_nonempty = 0;    // meshes / meshes with at least one triangle
  float box_min[3], box_max[3], box_ext[3], pad = 0, eps_t = 0;
  Buf tri_e, tri_sph, mesh_sph, mesh_first, mesh_count;
  std::vector<float> h_mesh_sph;
  // per-frame arena (grow-only; `gen` counts reallocations, which invalidate the graph)
  Buf rays, keys_c, vals_c, ckey, cbase, k1, v1, k2, v2, pos, first_chunk, sorted_key, sorted_slot, sorted_rays, px_tiles,
      nodes, trav, masks, gwork, gstat, items, best, zero, stage_in, stage_out;
  uint64_t gen = 0;
  unsigned long long* h_counters = nullptr;   // pinned
  FrameDesc* h_fd = nullptr;                   // pinned
  FrameInfo fi;
  int64_t launches = 0;
  cudaStream_t last_stream = nullptr;
  cudaStream_t gstream = nullptr;              // non-blocking stream the frame graph runs on
  cudaEvent_t ev[10] = {nullptr};
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  cudaGraphExec_t gexec = nullptr;
  std::vector<unsigned char> gkey;
  int64_t graph_launches = 0;                  // kernels inside the cached graph
  int sm_count = 148;
  // multi-bounce Whitted loop (crsh_render_whitted): per-bounce vertex sets and terms
  std::vector<std::array<Buf, 8>> wb;   // pos, nrm, dir, mat, direct, c_re, c_rr, L
  Buf w_hit, w_t, w_zero;
  Buf prim_rays;                        // crsh_primary_gbuffer camera rays
  // dynamic scenes (crsh_scene_transform): creation-time geometry and spheres
  Buf tris0, mesh_ids, tris_cur, xf, boxk;
  std::vector<float> h_mesh_sph0;
  Dist* dist = nullptr;                 // crsh_dist_init: NCCL communicator, window, merge mode
  // object sphere-tree (CRSH_F_OBJTREE, reading O1): cluster order, ranges, spheres
  Buf cl_order, cl_range, cl_first, cl_sph, tri_sph_ord, cl_pf;   // cl_pf: K8 child-prefilter spheres (k_cluster_pf)
  int64_t n_clusters = 0;
};

namespace {

cudaError_t grow(crsh_scene* sc, Buf& b, size_t bytes) {
  if (bytes <= b.cap && b.p) return cudaSuccess;
  ++sc->gen;
  return ensure(b, bytes);
}

// zero region layout (bytes), sized by the slot bound; reset at every frame
struct ZeroLayout {
  size_t fd, counters, tickets, hist, st_rg, st_rle, st_scan, st_plan, st_radix, radix_tiles_cap, px_total, total;
  static ZeroLayout make(uint64_t S, uint64_t G_max) {
    ZeroLayout z;
    size_t o = 0;
    auto take = [&](size_t b) { size_t r = o; o += (b + 255) & ~size_t(255); return r; };
    const uint64_t scan_tiles = cdiv(std::max<uint64_t>(S, 1), SCAN_TILE) + 1;
    const uint64_t plan_tiles = cdiv(std::max<uint64_t>(G_max, 1), SCAN_TILE) + 1;
    z.radix_tiles_cap = cdiv(std::max<uint64_t>(S, 1), SORT_TILE) + MAX_SEG + 1;
    z.fd = take(sizeof(FrameDesc));
    z.counters = take(8 * MAX_SEG * CTR_STRIDE);
    z.tickets = take(4 * 32);
    z.hist = take(4 * MAX_SEG * SORT_PASSES * RADIX_BINS);
    z.st_rg = take(8 * scan_tiles);
    z.st_rle = take(8 * scan_tiles);
    z.st_scan = take(8 * scan_tiles);
    z.st_plan = take(8 * plan_tiles);
    z.st_radix = take(4 * SORT_PASSES * z.radix_tiles_cap * RADIX_BINS);
    z.px_total = take(4 * 4);
    z.total = o;
    return z;
  }
};

enum { T_RG = 0, T_RLE = 1, T_SCAN = 2, T_PLAN = 3, T_TRAV = 4, T_RADIX = 8 };

bool is_pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }

template <class F>
cudaError_t dispatch_b0(int B0, F&& f) {
  switch (B0) {
    case 2: return f(std::integral_constant<int, 2>());
    case 4: return f(std::integral_constant<int, 4>());
    case 8: return f(std::integral_constant<int, 8>());
    case 16: return f(std::integral_constant<int, 16>());
    case 32: return f(std::integral_constant<int, 32>());
    case 64: return f(std::integral_constant<int, 64>());
  }
  return cudaErrorInvalidValue;
}
template <class F>
cudaError_t dispatch_b(int B, F&& f) {
  switch (B) {
    case 2: return f(std::integral_constant<int, 2>());
    case 4: return f(std::integral_constant<int, 4>());
    case 8: return f(std::integral_constant<int, 8>());
    case 16: return f(std::integral_constant<int, 16>());
    case 32: return f(std::integral_constant<int, 32>());
  }
  return cudaErrorInvalidValue;
}

#ifndef CRSH_ITEM_TRIS
#define CRSH_ITEM_TRIS 0   // 0: chosen per frame by item_tris_for(); else fixed (A/B builds)
#endif
// Triangles per traversal work item (load balance). Small frames (about one
// group per traversal CTA, cfg2) need 2048-triangle items to spread the work;
// frames with many groups per CTA (cfg3, cfg4) lose less to per-item setup
// with larger items (measured on B200, Mrays/s at 2048 / 4096 / 8192 /
// 16384 / 32768 / 65536 / one item per group:
//   cfg3 R6      60.0 / 62.1 / 62.8 / 63.3 / 62.8 / 63.2 / 55.0
//   cfg3 Z-order  587 /  636 /  666 /  697 /  698 /  661 /  424
//   cfg4 R6      17.2 / 18.0 / 18.4 / 18.6 / 18.7 / 18.7 / 18.3
//   cfg4 Z-order  234 /  261 /  275 /  284 /  289 /  292 /  219;
// cfg2 R6 at 2048 / 3072 / 4096: 109.6 / 109.1 / 107.1).
constexpr uint64_t ITEM_BIG_GROUPS_PER_SM = 16;   // G_max at or above 16 groups per SM -> ITEM_TRIS_BIG
#ifndef CRSH_ITEM_TRIS_SMALL_OBJ
#define CRSH_ITEM_TRIS_SMALL_OBJ 2048u
#endif
#ifndef CRSH_ITEM_TRIS_BIG
#define CRSH_ITEM_TRIS_BIG 16384
#endif
// The decision uses this rank's share of the groups (G_max / world): with
// hash-range sharding a rank traverses about G_max / world groups, and a small
// share needs the small items to balance. CRSH_ITEM_TRIS=<n> (environment,
// read per call) forces n triangles per item -- a test hook that runs the
// large-item path on small frames.
// With the object sphere-tree (CRSH_F_OBJTREE) most of an item's clusters are
// culled by one lane-parallel test each, so an item costs less and large
// frames take twice the triangles per item (A/B, Z-order + tree, 16384 /
// 32768 / 65536: cfg3 984 / 1020 / 892, cfg4 547 / 577 / 593 Mrays/s).
inline uint32_t item_tris_for(uint64_t G_max, int world, int sm_count, bool objtree = false) {
  if (CRSH_ITEM_TRIS) return CRSH_ITEM_TRIS;
  if (const char* e = std::getenv("CRSH_ITEM_TRIS")) {
    const long v = std::strtol(e, nullptr, 10);
    if (v >= 32 && v <= (1l << 24) && (v % 32) == 0) return (uint32_t)v;
  }
  const uint64_t share = G_max / (uint64_t)std::max(world, 1);
  const bool big = share >= ITEM_BIG_GROUPS_PER_SM * (uint64_t)std::max(sm_count, 1);
  // very large frames (>= 64 groups per SM, cfg4 ~160): twice that again
  const uint32_t huge = share >= 4 * ITEM_BIG_GROUPS_PER_SM * (uint64_t)std::max(sm_count, 1) ? 2u : 1u;
  if (objtree) return big ? 2u * huge * (uint32_t)CRSH_ITEM_TRIS_BIG : CRSH_ITEM_TRIS_SMALL_OBJ;
  // plain path, since its slices are handed out dynamically within an item
  // (A/B, Mrays/s at 16384 / 32768 / 65536 triangles: cfg3 R6 69.3 / 69.8 /
  // 69.2, Z-order 787 / 795 / 752; cfg4 R6 20.59 / 20.66 / 20.64, Z-order
  // 336 / 340 / 341): 32768 for every large frame
  return big ? 2u * (uint32_t)CRSH_ITEM_TRIS_BIG : 2048u;
}

// Entries of K8's object-tree cluster list used per round: the compiled size,
// or CRSH_OBJ_LIST_CAP (tests: a small list forces many rounds per item),
// never below one block per warp (32 / K clusters each), the fill bound
inline uint32_t obj_list_for(int K) {
  const uint32_t lo = (32u / (uint32_t)std::max(K, 1)) * (uint32_t)TRAV_WARPS;
  uint32_t v = CRSH_OBJ_LIST;
  if (const char* e = std::getenv("CRSH_OBJ_LIST_CAP")) v = (uint32_t)std::max(0l, std::strtol(e, nullptr, 10));
  return std::min<uint32_t>(std::max(v, lo), CRSH_OBJ_LIST);
}

// Everything a frame's launch sequence depends on: if the key of a call equals
// the cached one, the cached CUDA graph is replayed.
struct CallKey {
  const void *pos, *nrm, *mat, *materials, *dir, *out_hit, *out_t, *out_packed;
  PeerOut peer;
  int32_t W, H, n_mat, n_lights;
  float eye[3], lights[48];
  uint32_t types;
  crsh_opts o;
  uint64_t gen;
  uint32_t item_tris;
  uint32_t tiles;
  uint32_t obj_list;
  int32_t prefilter, top_prefilter;
};

// The ray-definition part of K1's arguments (G-buffer, lights, slot layout);
// also used by the Whitted loop to regenerate a traced ray bit for bit.
RaygenArgs raygen_def(const crsh_scene* sc, const FrameInfo& fi, const crsh_primary_hits* h, const float* lights,
                      int32_t n_lights) {
  RaygenArgs a{};
  a.P = h->width * h->height; a.pos = h->pos; a.nrm = h->nrm; a.mat = h->mat; a.materials = h->materials;
  a.n_mat = h->n_mat;
  for (int i = 0; i < 3; ++i) a.eye[i] = h->eye[i];
  a.dir = h->dir;
  a.in_rays = fi.in_rays;
  for (int i = 0; i < 3 * n_lights; ++i) a.lights[i] = lights[i];
  a.n_lights = n_lights; a.zorder = (fi.flags & CRSH_F_ZORDER) ? 1 : 0;
  for (int i = 0; i < 3; ++i) { a.box_min[i] = sc->box_min[i]; a.box_ext[i] = sc->box_ext[i]; }
  a.eps_t = sc->eps_t; a.n_slots = (uint32_t)fi.S; a.n_seg = fi.n_seg;
  for (int s = 0; s < fi.n_seg; ++s) a.seg_type[s] = fi.seg_type[s];
  for (int s = 0; s <= fi.n_seg; ++s) a.seg_slot_start[s] = fi.seg_slot_start[s];
  return a;
}

// Enqueue one frame on `st` (directly or under graph capture). Returns the
// number of kernels launched.
crsh_status enqueue_frame(crsh_scene* sc, const FrameInfo& fi, const crsh_primary_hits* h, const float* lights,
                          int32_t n_lights, int32_t* out_hit, float* out_t, unsigned long long* out_packed,
                          const PeerOut& peer, cudaStream_t st, int64_t* n_launch, const Dist* dist = nullptr) {
  const uint64_t S = fi.S;
  const int Lv = fi.Lv, B0 = fi.B0, B = fi.B;
  const ZeroLayout Z = ZeroLayout::make(S, fi.G_max);
  char* zb = sc->zero.as<char>();
  FrameDesc* fd = reinterpret_cast<FrameDesc*>(zb + Z.fd);
  unsigned long long* counters = reinterpret_cast<unsigned long long*>(zb + Z.counters);
  uint32_t* tickets = reinterpret_cast<uint32_t*>(zb + Z.tickets);
  int64_t nl = 0;
  // stage marks (all with CRSH_F_STAGE_TIMING, only around k_traverse with
  // CRSH_F_KERNEL_TIMING); under capture they must be external record nodes
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(st, &cap));
  auto mark = [&](int i) -> cudaError_t {
    if (!(fi.timed || (fi.ktimed && (i == 6 || i == 7)))) return cudaSuccess;
    return cap == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(sc->ev[i], st, cudaEventRecordExternal)
                                                : cudaEventRecord(sc->ev[i], st);
  };
  CK(cudaMemsetAsync(sc->zero.p, 0, Z.total, st));
  if (dist && dist->mode == MERGE_PEER) {
    // every rank has finished reading its window (previous frame's unpack)
    // before any rank stores this frame's results into it
    k_lsa_barrier<<<1, 128, 0, st>>>(dist->dev);
    CK(cudaGetLastError());
    ++nl;
  }
  CK(mark(0));

  // ---------------------------------------------------------------- K1: generate + hash + trim
  {
    RaygenArgs a = raygen_def(sc, fi, h, lights, n_lights);
    a.rays = sc->rays.as<float4>(); a.keys_c = sc->keys_c.as<uint32_t>(); a.vals_c = sc->vals_c.as<uint32_t>();
    a.out_hit = out_packed ? nullptr : out_hit; a.out_t = out_packed ? nullptr : out_t; a.out_packed = out_packed;
    a.peer = peer;
    a.status = reinterpret_cast<unsigned long long*>(zb + Z.st_rg); a.ticket = tickets + T_RG;
    a.fd = fd;
    if (fi.in_rays || std::getenv("CRSH_SLOT_MAJOR")) {   // given ray batches: slot-major with look-back
      k_raygen<<<cdiv(S, SCAN_TILE), SCAN_THREADS, 0, st>>>(a);
      CK(cudaGetLastError());
      ++nl;
    } else {   // G-buffer frames: pixel-major (count, then rank + generate)
      PxArgs px{};
      px.rg = a;
      for (int t = 0; t < 3; ++t) px.seg_of_type[t] = -1;
      for (int s = 0; s < fi.n_seg; ++s) px.seg_of_type[fi.seg_type[s]] = s;
      px.tile_cnt = sc->px_tiles.as<uint32_t>();
      px.total = reinterpret_cast<uint32_t*>(zb + Z.px_total);
      const uint64_t P = (uint64_t)h->width * h->height;
      if (P >= PX_SMALL_FRAME) {
        const uint32_t tiles = cdiv(P, px_tile(8));
        k_raygen_count<8><<<tiles, SCAN_THREADS, 0, st>>>(px);
        CK(cudaGetLastError());
        k_raygen_px<8><<<tiles, SCAN_THREADS, 0, st>>>(px);
      } else {
        const uint32_t tiles = cdiv(P, px_tile(2));
        k_raygen_count<2><<<tiles, SCAN_THREADS, 0, st>>>(px);
        CK(cudaGetLastError());
        k_raygen_px<2><<<tiles, SCAN_THREADS, 0, st>>>(px);
      }
      CK(cudaGetLastError());
      nl += 2;
    }
    k_frame_plan<<<1, 32, 0, st>>>(fd, fi.n_seg, fi.GR, (uint32_t)B0, (uint32_t)B, Lv);
    CK(cudaGetLastError());
    ++nl;
  }
  CK(mark(1));

  if (fi.brute) {   // N x M baseline (NEXT-1): no hierarchy
    for (int i = 2; i <= 7; ++i) CK(mark(i));
    if (fi.rank == 0) {
      BruteArgs b{};
      b.fd = fd; b.vals_c = sc->vals_c.as<uint32_t>(); b.rays = sc->rays.as<float4>(); b.tri_e = sc->tri_e.as<float4>();
      b.M = sc->M; b.n_seg = fi.n_seg;
      b.out_hit = out_hit; b.out_t = out_t; b.out_packed = out_packed; b.peer = peer; b.counters = counters;
      k_brute<<<cdiv(S, 256), 256, 0, st>>>(b);
      CK(cudaGetLastError());
      ++nl;
    }
  } else {
    // ---------------------------------------------------------------- K2-K4: compress, sort, decompress
    if (fi.sorted) {
      {
        RleArgs a{};
        a.fd = fd; a.keys = sc->keys_c.as<uint32_t>(); a.n_seg = fi.n_seg;
        a.ckey = sc->ckey.as<uint32_t>(); a.cbase = sc->cbase.as<uint32_t>();
        a.hist = fi.rle_hist ? reinterpret_cast<uint32_t*>(zb + Z.hist) : nullptr;
        a.status = reinterpret_cast<unsigned long long*>(zb + Z.st_rle); a.ticket = tickets + T_RLE;
        // 2048-key tiles (A/B at cfg4: 8192-key tiles 83 -> 107 us; they do pay
        // for the decompression scan below)
        k_rle<SCAN_ITEMS><<<cdiv(S, SCAN_TILE), SCAN_THREADS, 0, st>>>(a);
        CK(cudaGetLastError());
        k_chunk_plan<<<1, 32, 0, st>>>(fd, fi.n_seg, (uint32_t)SORT_TILE);
        CK(cudaGetLastError());
        nl += 2;
      }
      CK(mark(2));
      uint32_t* hist = reinterpret_cast<uint32_t*>(zb + Z.hist);
      if (!fi.rle_hist) {
        k_radix_hist<<<std::min<uint32_t>(cdiv(S, 256 * 8), 4 * sc->sm_count), 256, 0, st>>>(fd, fi.n_seg,
                                                                                             sc->ckey.as<uint32_t>(), hist);
        CK(cudaGetLastError());
        ++nl;
      }
      const size_t sm_bytes = (2 * SORT_TILE + SORT_WARPS * RADIX_BINS) * 4;
      if (sm_bytes > 48 * 1024) CK(cudaFuncSetAttribute(k_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_bytes));
      const uint32_t* kin = sc->ckey.as<uint32_t>();
      const uint32_t* vin = nullptr;
      for (int p = 0; p < SORT_PASSES; ++p) {
        SortPassArgs a{};
        a.fd = fd; a.n_seg = fi.n_seg; a.pass = p; a.keys_in = kin; a.vals_in = vin;
        a.keys_out = (p & 1) ? sc->k2.as<uint32_t>() : sc->k1.as<uint32_t>();
        a.vals_out = (p & 1) ? sc->v2.as<uint32_t>() : sc->v1.as<uint32_t>();
        a.hist = hist;
        a.status = reinterpret_cast<uint32_t*>(zb + Z.st_radix) + (size_t)p * Z.radix_tiles_cap * RADIX_BINS;
        a.ticket = tickets + T_RADIX + p;
        k_onesweep<<<(uint32_t)Z.radix_tiles_cap, SORT_THREADS, sm_bytes, st>>>(a);
        CK(cudaGetLastError());
        ++nl;
        kin = a.keys_out; vin = a.vals_out;
      }
      CK(mark(3));
      {
        ScanSizeArgs a{};
        a.fd = fd; a.sorted_cidx = sc->v2.as<uint32_t>(); a.cbase = sc->cbase.as<uint32_t>();
        a.pos = sc->pos.as<uint32_t>(); a.first_chunk = sc->first_chunk.as<uint32_t>();
        a.status = reinterpret_cast<unsigned long long*>(zb + Z.st_scan); a.ticket = tickets + T_SCAN;
        if (fi.big_tiles) k_scan_sizes<32><<<cdiv(S, SCAN_THREADS * 32), SCAN_THREADS, 0, st>>>(a);
        else k_scan_sizes<SCAN_ITEMS><<<cdiv(S, SCAN_TILE), SCAN_THREADS, 0, st>>>(a);
        CK(cudaGetLastError());
        ++nl;
      }
      {
        ExpandArgs a{};
        a.fd = fd; a.pos = sc->pos.as<uint32_t>(); a.first_chunk = sc->first_chunk.as<uint32_t>();
        a.skey = sc->k2.as<uint32_t>(); a.scidx = sc->v2.as<uint32_t>(); a.cbase = sc->cbase.as<uint32_t>();
        a.vals_c = sc->vals_c.as<uint32_t>(); a.n_seg = fi.n_seg;
        a.sorted_key = sc->sorted_key.as<uint32_t>(); a.sorted_slot = sc->sorted_slot.as<uint32_t>();
        k_expand<<<cdiv(S, EXP_TILE), 256, 0, st>>>(a);
        CK(cudaGetLastError());
        ++nl;
      }
    } else {
      CK(mark(2));
      CK(mark(3));
      ExpandArgs a{};
      a.fd = fd; a.skey = sc->keys_c.as<uint32_t>(); a.vals_c = sc->vals_c.as<uint32_t>(); a.n_seg = fi.n_seg;
      a.sorted_key = sc->sorted_key.as<uint32_t>(); a.sorted_slot = sc->sorted_slot.as<uint32_t>();
      k_copy_unsorted<<<std::min<uint32_t>(cdiv(S, 256), 8 * sc->sm_count), 256, 0, st>>>(a);
      CK(cudaGetLastError());
      ++nl;
    }
    CK(mark(4));

    // ---------------------------------------------------------------- K5-K6: hierarchy build
    float4* nodes = sc->nodes.as<float4>();
    float4* trav = sc->trav.as<float4>();
    {
      LeafArgs a{};
      a.fd = fd; a.n_seg = fi.n_seg;
      a.sorted_slot = sc->sorted_slot.as<uint32_t>(); a.rays = sc->rays.as<float4>();
      a.sorted_rays = sc->sorted_rays.as<float4>(); a.nodes = nodes; a.trav = trav;
      a.write_sorted = fi.GR <= SMALL_GROUP_RAYS ? 0 : 1;   // smem groups gather their rays in K8
      const uint32_t grid = cdiv(std::max<uint64_t>(fi.level_max[1], 1), 128);
      CK(dispatch_b0(B0, [&](auto b0) {
        k_leaves<decltype(b0)::value><<<grid, 128, 0, st>>>(a);
        return cudaGetLastError();
      }));
      ++nl;
    }
    for (int k = 2; k <= Lv; ++k) {
      UpperArgs a{};
      a.fd = fd; a.level = k;
      a.child_nodes = nodes + 2 * fi.level_off[k - 1];
      a.nodes = nodes + 2 * fi.level_off[k];
      a.trav = trav + 3 * fi.level_off[k];
      const uint32_t grid = cdiv(std::max<uint64_t>(fi.level_max[k] * (CRSH_UPPER_WARP ? (uint64_t)B : 1u), 1), 128);
      CK(dispatch_b(B, [&](auto b) {
        k_upper<decltype(b)::value><<<grid, 128, 0, st>>>(a);
        return cudaGetLastError();
      }));
      ++nl;
    }
    CK(mark(5));

    // ---------------------------------------------------------------- K7-K9: traversal
    const int W = (sc->n_meshes + 31) / 32;
    // K8's child prefilter (the bench shape's plain instantiation): slices are
    // the object-tree clusters (whole clusters per kept mesh, as with
    // CRSH_F_OBJTREE), each with its prefilter sphere (k_cluster_pf)
    const bool objt = (fi.flags & CRSH_F_OBJTREE) != 0;
    const bool pf = fi.prefilter && !objt && sc->n_clusters > 0 && fi.GR <= SMALL_GROUP_RAYS && B == 8 && B0 == 8 &&
                    Lv == 2 && fi.K == 8;
    CK(cudaMemsetAsync(sc->best.p, 0xFF, 8 * (size_t)fi.Np_max, st));
    {
      CullArgs a{};
      a.fd = fd; a.K = fi.K; a.W = W;
      a.trav_top = trav + 3 * fi.level_off[Lv];
      a.n_meshes = sc->n_meshes; a.mesh_sph = sc->mesh_sph.as<float4>(); a.mesh_count = sc->mesh_count.as<uint32_t>();
      a.cull_on = (fi.flags & CRSH_F_MESH_CULL) ? 1 : 0;
      a.masks = sc->masks.as<uint32_t>();
      k_mesh_cull<<<cdiv(std::max<uint64_t>(fi.G_max * fi.K * W, 1), 256), 256, 0, st>>>(a);
      CK(cudaGetLastError());
      ++nl;
      {   // per-group triangles / mesh counters / work (one warp per group)
        WorkArgs w{};
        w.fd = fd; w.K = fi.K; w.W = W; w.n_meshes = sc->n_meshes;
        w.masks = sc->masks.as<uint32_t>(); w.mesh_count = sc->mesh_count.as<uint32_t>();
        w.trav_top = trav + 3 * fi.level_off[Lv]; w.cull_on = a.cull_on; w.n_nonempty = sc->n_nonempty;
        w.objtree = (objt || pf) ? 1 : 0;   // cluster-aligned virtual ranges
        w.work = sc->gwork.as<unsigned long long>(); w.gstat = sc->gstat.as<uint4>();
        k_group_work<<<cdiv(std::max<uint64_t>(fi.G_max, 1), 8), 256, 0, st>>>(w);
        CK(cudaGetLastError());
        ++nl;
      }
      if (fi.world > 1) {   // work-balanced cut of the groups over the ranks
        k_cut<<<1, CUT_THREADS, 0, st>>>(fd, sc->gwork.as<unsigned long long>(), fi.rank, fi.world);
      } else {
        k_cut<<<1, 32, 0, st>>>(fd, nullptr, 0, 1);
      }
      CK(cudaGetLastError());
      ++nl;
      PlanArgs p{};
      p.fd = fd; p.group_rays = fi.GR; p.n_seg = fi.n_seg; p.gstat = sc->gstat.as<uint4>(); p.counters = counters;
      p.item_tris = fi.item_tris;
      p.items_cap = (uint32_t)std::min<uint64_t>(sc->items.cap / 16, 0xFFFFFFFFull);
      p.items = sc->items.as<uint4>();
      p.status = reinterpret_cast<unsigned long long*>(zb + Z.st_plan); p.ticket = tickets + T_PLAN;
      k_plan<<<cdiv(std::max<uint64_t>(fi.G_max, 1), SCAN_TILE), SCAN_THREADS, 0, st>>>(p);
      CK(cudaGetLastError());
      ++nl;
    }
    CK(mark(6));
    {
      TravArgs t{};
      t.Lv = Lv; t.B0 = B0; t.B = B; t.K = fi.K; t.group_rays = fi.GR;
      t.logB0 = __builtin_ctz((unsigned)B0); t.logB = __builtin_ctz((unsigned)B);
      uint64_t per = 1;
      for (int k = Lv; k >= 1; --k) { t.per_group[k] = (uint32_t)(fi.K * per); per *= B; }
      for (int k = 1; k <= Lv; ++k) t.trav[k] = trav + 3 * fi.level_off[k];
      t.sorted_rays = sc->sorted_rays.as<float4>(); t.tri_e = sc->tri_e.as<float4>();
      t.sorted_slot = sc->sorted_slot.as<uint32_t>(); t.rays = sc->rays.as<float4>();
      t.tri_sph = sc->tri_sph.as<float4>();
      t.masks = sc->masks.as<uint32_t>(); t.W = W; t.n_meshes = sc->n_meshes;
      t.mesh_first = sc->mesh_first.as<uint32_t>(); t.mesh_count = sc->mesh_count.as<uint32_t>();
      if (objt || pf) {
        t.tri_order = sc->cl_order.as<int32_t>(); t.tri_sph_ord = sc->tri_sph_ord.as<float4>();
        t.mesh_cluster_first = sc->cl_first.as<uint32_t>(); t.cluster_sph = sc->cl_sph.as<float4>();
        t.cluster_pf = sc->cl_pf.as<float4>();
      }
      t.items = sc->items.as<uint4>(); t.fd = fd; t.ticket = tickets + T_TRAV; t.M = (uint32_t)sc->M;
      t.obj_list_cap = fi.obj_list;
      t.best = sc->best.as<unsigned long long>(); t.counters = counters; t.n_seg = fi.n_seg;
      const bool small = fi.GR <= SMALL_GROUP_RAYS;
      const TravSmem L = TravSmem::make(fi.K, B, sc->n_meshes, Lv, small, t.per_group, fi.GR);
      auto launch = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
        if (e != cudaSuccess) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TRAV_THREADS, L.total);
        if (e != cudaSuccess) return e;
        per_sm = std::max(1, per_sm);
        kern<<<per_sm * sc->sm_count, TRAV_THREADS, L.total, st>>>(t, L);
        return cudaGetLastError();
      };
      auto pick = [&](auto obj) -> cudaError_t {
        constexpr bool O = decltype(obj)::value;
        if (!O && pf)
          return fi.top_prefilter ? launch(k_traverse<true, 8, 8, 2, false, 2>) : launch(k_traverse<true, 8, 8, 2, false, 1>);
        if (B == 8 && B0 == 8 && Lv == 2 && fi.K == 8)
          return small ? launch(k_traverse<true, 8, 8, 2, O>) : launch(k_traverse<false, 8, 8, 2, O>);
        if (B == 8 && B0 == 8) return small ? launch(k_traverse<true, 8, 8, 0, O>) : launch(k_traverse<false, 8, 8, 0, O>);
        return small ? launch(k_traverse<true, 0, 0, 0, O>) : launch(k_traverse<false, 0, 0, 0, O>);
      };
      if (fi.flags & CRSH_F_OBJTREE) CK(pick(std::true_type()));
      else CK(pick(std::false_type()));
      ++nl;
    }
    CK(mark(7));
    {
      UnpackArgs a{};
      a.fd = fd; a.group_rays = fi.GR; a.n_seg = fi.n_seg;
      a.sorted_slot = sc->sorted_slot.as<uint32_t>(); a.best = sc->best.as<unsigned long long>();
      a.out_hit = out_hit; a.out_t = out_t; a.out_packed = out_packed; a.peer = peer; a.counters = counters;
      a.n_slots = (uint32_t)S;
      k_unpack<<<cdiv(std::max<uint64_t>(fi.Np_max, 1), 256), 256, 0, st>>>(a);
      CK(cudaGetLastError());
      ++nl;
    }
  }
  if (dist) {   // a14: merge the per-rank results into hit_tri / t on every rank, sum the counters
    unsigned long long* wb = static_cast<unsigned long long*>(dist->wbuf);
    if (dist->mode == MERGE_PEER) {
      k_lsa_barrier<<<1, 128, 0, st>>>(dist->dev);   // every rank's stores have landed in every window
      CK(cudaGetLastError());
      ++nl;
    } else {
      NCK(ncclAllReduce(wb, wb, S, ncclUint64, ncclMin, dist->comm, st));
    }
    k_unpack_packed<<<std::min<uint32_t>(cdiv(S, 256), 8 * sc->sm_count), 256, 0, st>>>(wb, S, out_hit, out_t);
    CK(cudaGetLastError());
    ++nl;
    NCK(ncclAllReduce(counters, counters, (size_t)MAX_SEG * CTR_STRIDE, ncclUint64, ncclSum, dist->comm, st));
  }
  CK(mark(8));
  CK(cudaMemcpyAsync(sc->h_counters, counters, 8 * MAX_SEG * CTR_STRIDE, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(sc->h_fd, fd, sizeof(FrameDesc), cudaMemcpyDeviceToHost, st));
  *n_launch = nl;
  return CRSH_OK;
}

crsh_status dist_window(crsh_scene* sc, size_t bytes);

crsh_status trace_impl(crsh_scene* sc, const crsh_primary_hits* h, const float* lights, int32_t n_lights,
                       uint32_t types, const crsh_opts* o, int32_t* out_hit, float* out_t,
                       unsigned long long* out_packed, const PeerOut& peer_in, cudaStream_t st, bool graph_ok = true,
                       const float4* in_rays = nullptr, bool use_dist = false) {
  if (!sc || !h || !o) return fail(CRSH_EINVAL, "null scene / hits / opts");
  if (h->width <= 0 || h->height <= 0) return fail(CRSH_EINVAL, "width/height must be positive");
  const uint64_t P64 = (uint64_t)h->width * (uint64_t)h->height;
  if (P64 >= (1ull << 31)) return fail(CRSH_ELIMIT, "too many pixels");
  const int32_t P = (int32_t)P64;
  if (n_lights < 0 || n_lights > 16) return fail(CRSH_ELIMIT, "n_lights must be in [0, 16] (4-bit light field)");
  if (n_lights > 0 && !lights) return fail(CRSH_EINVAL, "lights is null");
  if (types == 0 || (types & ~7u)) return fail(CRSH_EINVAL, "bad ray_types");
  if (!h->pos || !h->nrm || !h->mat || (h->n_mat > 0 && !h->materials) || h->n_mat < 0)
    return fail(CRSH_EINVAL, "null G-buffer pointer");
  const int Lv = o->levels, B0 = o->leaf_size, B = o->branching;
  if (Lv < 1 || Lv > MAX_LEVELS) return fail(CRSH_EINVAL, "levels must be in [1, 8]");
  if (!is_pow2(B0) || B0 < 2 || B0 > 64) return fail(CRSH_EINVAL, "leaf_size must be a power of 2 in [2, 64]");
  if (!is_pow2(B) || B < 2 || B > 32) return fail(CRSH_EINVAL, "branching must be a power of 2 in [2, 32]");
  uint64_t span = B0;
  for (int k = 1; k < Lv; ++k) span *= B;
  if (span > (1ull << 22)) return fail(CRSH_ELIMIT, "leaf_size * branching^(levels-1) > 2^22");
  int world = std::max(1, o->shard_world), rank = o->shard_rank;
  if (rank < 0 || rank >= world) return fail(CRSH_EINVAL, "bad shard rank/world");
  const Dist* dist = (use_dist && sc && sc->dist) ? sc->dist : nullptr;
  if (dist) {   // the scene's NCCL world decides the shard (crsh_dist_init)
    if (world > 1 && (world != dist->world || rank != dist->rank))
      return fail(CRSH_EINVAL, "opts shard (%d of %d) differs from crsh_dist_init (%d of %d)", rank, world,
                  dist->rank, dist->world);
    rank = dist->rank;
    world = dist->world;
  }
  PeerOut peer = peer_in;
  if ((o->flags & ~127u) != 0) return fail(CRSH_EINVAL, "unknown flags");
  if (!peer.n && !out_packed && (!out_hit || !out_t)) return fail(CRSH_EINVAL, "null output");
  if (dist && (peer.n || out_packed || in_rays)) return fail(CRSH_EINVAL, "internal: dist merge with explicit outputs");

  // ---------------------------------------------------------------- static plan
  FrameInfo fi;
  fi.Lv = Lv; fi.B0 = B0; fi.B = B;
  fi.span = (uint32_t)span;
  fi.K = span >= 512 ? 1 : (int)std::min<uint64_t>(32, 512 / span);
  fi.GR = fi.K * fi.span;
  fi.flags = o->flags;
  fi.sorted = (o->flags & CRSH_F_SORT) != 0;
  fi.timed = (o->flags & CRSH_F_STAGE_TIMING) != 0;
  fi.ktimed = (o->flags & CRSH_F_KERNEL_TIMING) != 0;
  fi.brute = (o->flags & CRSH_F_BRUTE) != 0;
  fi.rank = rank; fi.world = world;
  fi.in_rays = in_rays;
  uint64_t S = 0;
  const int type_bits[3] = {1, 2, 4};
  for (int t = 0; t < 3; ++t) {
    if (!(types & type_bits[t])) continue;
    const uint64_t ns = (t == 0) ? (uint64_t)P * n_lights : (uint64_t)P;
    if (ns == 0) continue;
    fi.seg_type[fi.n_seg] = t;
    fi.seg_slot_start[fi.n_seg] = (uint32_t)S;
    ++fi.n_seg;
    S += ns;
  }
  if (S >= (1ull << 30)) return fail(CRSH_ELIMIT, "slots >= 2^30");
  fi.seg_slot_start[fi.n_seg] = (uint32_t)S;
  fi.S = S;
  fi.Np_max = roundup(S + (uint64_t)fi.n_seg * fi.GR, fi.GR);
  fi.G_max = fi.Np_max / fi.GR;
  {
    size_t off = 0;
    uint64_t per = B0;
    for (int k = 1; k <= Lv; ++k) {
      fi.level_off[k] = off;
      fi.level_max[k] = fi.Np_max / per;
      off += fi.level_max[k];
      per *= B;
    }
  }
  CK(cudaSetDevice(sc->device));
  if (dist && S > 0) {   // the packed frame lives in the symmetric window (collective growth)
    crsh_status rc = dist_window(sc, 8 * S);
    if (rc != CRSH_OK) return rc;
    if (dist->mode == MERGE_PEER) peer = dist->peers;
    else out_packed = static_cast<unsigned long long*>(dist->wbuf);
  }
  sc->last_stream = st;
  sc->fi = fi;
  sc->fi.valid = false;
  if (S == 0) {
    std::memset(sc->h_counters, 0, 8 * MAX_SEG * CTR_STRIDE);
    std::memset(sc->h_fd, 0, sizeof(FrameDesc));
    sc->launches = 0;
    sc->fi.valid = true;
    return CRSH_OK;
  }

  // ---------------------------------------------------------------- buffers (upper bounds)
  const ZeroLayout Z = ZeroLayout::make(S, fi.G_max);
  size_t total_nodes = 0;
  for (int k = 1; k <= Lv; ++k) total_nodes += fi.level_max[k];
  const int W = (sc->n_meshes + 31) / 32;
  fi.item_tris = item_tris_for(fi.G_max, world, sc->sm_count, (fi.flags & CRSH_F_OBJTREE) != 0);
  fi.obj_list = obj_list_for(fi.K);
  {
    const char* e = std::getenv("CRSH_NO_PREFILTER");
    fi.prefilter = (e && std::atoi(e) != 0) ? 0 : 1;
    // the top-level prefilter pays where most top-level tests fail: with the
    // Z-order hash (cfg4 Z-order 332 -> 408 Mrays/s), not with R6 (70 % of
    // the top-level tests pass: 23.7 -> 22.7)
    const char* t = std::getenv("CRSH_TOP_PREFILTER");
    fi.top_prefilter = t ? (std::atoi(t) != 0) : ((fi.flags & CRSH_F_ZORDER) ? 1 : 0);
  }
  {   // decompression-scan tile size; radix histograms built by k_rle (A/B at cfg4: scan 178 -> 162 us with
      // 8192-entry tiles; sort 340 -> 319 us without the histogram pass). Overrides CRSH_BIG_TILES, CRSH_RLE_HIST.
    const char* e = std::getenv("CRSH_BIG_TILES");
    fi.big_tiles = e ? std::atoi(e) != 0 : S >= (1ull << 21);
    const char* h2 = std::getenv("CRSH_RLE_HIST");
    fi.rle_hist = h2 ? std::atoi(h2) != 0 : true;
  }
  sc->fi.big_tiles = fi.big_tiles;
  sc->fi.rle_hist = fi.rle_hist;
  sc->fi.item_tris = fi.item_tris;
  sc->fi.obj_list = fi.obj_list;
  sc->fi.prefilter = fi.prefilter;
  sc->fi.top_prefilter = fi.top_prefilter;
  // a group's virtual range is at most M, or M + 31 per mesh when meshes are
  // padded to whole clusters (object tree, K8-PF)
  const int64_t M_virt = sc->M + (int64_t)(CLUSTER_TRIS - 1) * sc->n_meshes;
  const uint64_t items_cap = std::max<uint64_t>(fi.G_max, 1) * cdiv(std::max<int64_t>(M_virt, 1), fi.item_tris);
  CK(grow(sc, sc->zero, Z.total));
  CK(grow(sc, sc->rays, 32 * S));
  CK(grow(sc, sc->px_tiles, 12 * ((size_t)cdiv((uint64_t)h->width * h->height, px_tile(2)) + 1)));
  CK(grow(sc, sc->keys_c, 4 * S));
  CK(grow(sc, sc->vals_c, 4 * S));
  if (!fi.brute) {
    CK(grow(sc, sc->ckey, 4 * S));
    CK(grow(sc, sc->cbase, 4 * (S + 1)));
    CK(grow(sc, sc->k1, 4 * S)); CK(grow(sc, sc->v1, 4 * S));
    CK(grow(sc, sc->k2, 4 * S)); CK(grow(sc, sc->v2, 4 * S));
    CK(grow(sc, sc->pos, 4 * (S + 1)));
    CK(grow(sc, sc->first_chunk, 4 * ((size_t)cdiv(S, EXP_TILE) + 1)));
    CK(grow(sc, sc->sorted_key, 4 * fi.Np_max));
    CK(grow(sc, sc->sorted_slot, 4 * fi.Np_max));
    CK(grow(sc, sc->sorted_rays, 32 * fi.Np_max));
    CK(grow(sc, sc->nodes, 32 * total_nodes));
    CK(grow(sc, sc->trav, 48 * total_nodes));
    CK(grow(sc, sc->masks, 4 * (size_t)fi.G_max * fi.K * W + 4));
    CK(grow(sc, sc->gwork, 8 * (size_t)fi.G_max + 8));
    CK(grow(sc, sc->gstat, 16 * (size_t)fi.G_max + 16));
    CK(grow(sc, sc->best, 8 * fi.Np_max));
    CK(grow(sc, sc->items, 16 * items_cap));
  }

  // ---------------------------------------------------------------- graph replay or capture
  CallKey key{};
  key.pos = h->pos; key.nrm = h->nrm; key.mat = h->mat; key.materials = h->materials; key.dir = h->dir;
  key.out_hit = out_hit; key.out_t = out_t; key.out_packed = out_packed; key.peer = peer;
  key.W = h->width; key.H = h->height; key.n_mat = h->n_mat; key.n_lights = n_lights;
  for (int i = 0; i < 3; ++i) key.eye[i] = h->eye[i];
  for (int i = 0; i < 3 * n_lights; ++i) key.lights[i] = lights[i];
  key.types = types; key.o = *o; key.gen = sc->gen; key.item_tris = fi.item_tris; key.obj_list = fi.obj_list; key.prefilter = fi.prefilter;
  key.top_prefilter = fi.top_prefilter;
  key.tiles = (fi.big_tiles ? 1u : 0u) | (fi.rle_hist ? 2u : 0u);
  std::vector<unsigned char> kb(sizeof(CallKey));
  std::memcpy(kb.data(), &key, sizeof(CallKey));
  static const bool use_graph = !std::getenv("CRSH_NO_GRAPH");
  if (!use_graph || !graph_ok) {
    int64_t nl = 0;
    crsh_status rc = enqueue_frame(sc, fi, h, lights, n_lights, out_hit, out_t, out_packed, peer, st, &nl, dist);
    if (rc != CRSH_OK) return rc;
    sc->launches = nl;
  } else {
    if (!sc->gexec || kb != sc->gkey) {
      if (sc->gexec) { cudaGraphExecDestroy(sc->gexec); sc->gexec = nullptr; }
      CK(cudaStreamBeginCapture(sc->gstream, cudaStreamCaptureModeThreadLocal));
      int64_t nl = 0;
      crsh_status rc = enqueue_frame(sc, fi, h, lights, n_lights, out_hit, out_t, out_packed, peer, sc->gstream, &nl,
                                     dist);
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(sc->gstream, &g);
      if (rc != CRSH_OK) { if (g) cudaGraphDestroy(g); return rc; }
      CK(e);
      e = cudaGraphInstantiate(&sc->gexec, g, 0);
      cudaGraphDestroy(g);
      CK(e);
      sc->gkey = kb;
      sc->graph_launches = nl;
    }
    CK(cudaEventRecord(sc->ev_in, st));
    CK(cudaStreamWaitEvent(sc->gstream, sc->ev_in, 0));
    CK(cudaGraphLaunch(sc->gexec, sc->gstream));
    CK(cudaEventRecord(sc->ev_out, sc->gstream));
    CK(cudaStreamWaitEvent(st, sc->ev_out, 0));
    sc->launches = sc->graph_launches;
  }
  sc->fi.valid = true;
  sc->fi.fd_fresh = false;
  return CRSH_OK;
}

// wait for the last frame and refresh the host copy of its FrameDesc
crsh_status sync_frame(crsh_scene* sc) {
  CK(cudaSetDevice(sc->device));
  CK(cudaStreamSynchronize(sc->last_stream));
  if (sc->gstream) CK(cudaStreamSynchronize(sc->gstream));
  if (CRSH_CHECKED) {   // checked build: the first failed device bounds check (common.cuh)
    unsigned int chk = 0;
    CK(cudaMemcpyFromSymbol(&chk, g_crsh_check, sizeof chk));
    if (chk) return fail(CRSH_ECUDA, "device bounds check %u failed (checked build)", chk);
  }
  if (sc->dist) {
    ncclResult_t ae = ncclSuccess;
    NCK(ncclCommGetAsyncError(sc->dist->comm, &ae));
    if (ae != ncclSuccess) return fail(CRSH_ENCCL, "NCCL asynchronous error: %s", ncclGetErrorString(ae));
  }
  if (sc->fi.valid && !sc->fi.fd_fresh) {
    sc->fi.fd = *sc->h_fd;
    sc->fi.fd_fresh = true;
  }
  return CRSH_OK;
}

// Grow the symmetric window that holds the packed frame (collective: every
// rank calls it in the same trace, with the same slot count). No frame may
// still use the old window.
crsh_status dist_window(crsh_scene* sc, size_t bytes) {
  Dist* d = sc->dist;
  if (d->wbuf && d->wcap >= bytes) return CRSH_OK;
  CK(cudaStreamSynchronize(sc->last_stream));
  if (sc->gstream) CK(cudaStreamSynchronize(sc->gstream));
  if (d->win) { NCK(ncclCommWindowDeregister(d->comm, d->win)); d->win = nullptr; }
  if (d->wbuf) { NCK(ncclMemFree(d->wbuf)); d->wbuf = nullptr; d->wcap = 0; }
  const size_t want = roundup(std::max<size_t>(bytes + bytes / 8, 4096), NCCL_WIN_REQUIRED_ALIGNMENT);
  NCK(ncclMemAlloc(&d->wbuf, want));
  d->wcap = want;
  if (d->mode == MERGE_PEER) {
    NCK(ncclCommWindowRegister(d->comm, d->wbuf, want, &d->win, NCCL_WIN_COLL_SYMMETRIC));
    k_window_peers<<<1, 32>>>(d->win, d->world, d->d_ptrs);
    CK(cudaGetLastError());
    unsigned long long h[MAX_PEERS] = {0};
    CK(cudaMemcpy(h, d->d_ptrs, 8 * d->world, cudaMemcpyDeviceToHost));
    d->peers = PeerOut{};
    for (int r = 0; r < d->world; ++r) {
      if (!h[r]) return fail(CRSH_ENCCL, "no load/store pointer to the window of rank %d", r);
      d->peers.p[r] = reinterpret_cast<unsigned long long*>(h[r]);
    }
    d->peers.n = d->world;
  }
  ++sc->gen;   // the frame graph holds the window addresses: recapture
  return CRSH_OK;
}

}  // namespace

// ============================================================== C ABI
extern "C" {

crsh_status crsh_dist_unique_id(void* uid) {
  if (!uid) return fail(CRSH_EINVAL, "uid is null");
  ncclUniqueId id;
  NCK(ncclGetUniqueId(&id));
  std::memcpy(uid, &id, sizeof id);
  return CRSH_OK;
}

crsh_status crsh_dist_init(crsh_scene_t sc, const void* nccl_uid, int32_t rank, int32_t world) {
  if (!sc || !nccl_uid) return fail(CRSH_EINVAL, "null argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(CRSH_EINVAL, "bad rank %d / world %d", rank, world);
  if (sc->dist) return fail(CRSH_EINVAL, "crsh_dist_init already called on this scene");
  CK(cudaSetDevice(sc->device));
  auto* d = new Dist();
  d->rank = rank;
  d->world = world;
  ncclUniqueId id;
  std::memcpy(&id, nccl_uid, sizeof id);
  ncclResult_t r = ncclCommInitRank(&d->comm, world, id, rank);
  if (r != ncclSuccess) {
    delete d;
    return fail(CRSH_ENCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  sc->dist = d;   // from here on crsh_scene_destroy releases it
  // the fused merge needs every rank reachable by load/store (one NVLink
  // domain), at most MAX_PEERS ranks and the device API; the NCCL all-reduce
  // merge is the fallback (or CRSH_DIST_MERGE=nccl). All ranks agree.
  const char* want = std::getenv("CRSH_DIST_MERGE");
  int peer_ok = (!want || std::strcmp(want, "nccl") != 0) && world <= MAX_PEERS &&
                ncclTeamLsa(d->comm).nRanks == world;
  if (peer_ok) {
    ncclDevCommRequirements req{};
    req.lsaBarrierCount = 1;
    peer_ok = ncclDevCommCreate(d->comm, &req, &d->dev) == ncclSuccess;
    d->dev_ok = peer_ok != 0;
  }
  CK(cudaMalloc(&d->d_ptrs, 8 * MAX_PEERS + 8));
  int* flag = reinterpret_cast<int*>(d->d_ptrs + MAX_PEERS);
  CK(cudaMemcpy(flag, &peer_ok, sizeof(int), cudaMemcpyHostToDevice));
  NCK(ncclAllReduce(flag, flag, 1, ncclInt32, ncclMin, d->comm, sc->gstream));
  CK(cudaStreamSynchronize(sc->gstream));
  CK(cudaMemcpy(&peer_ok, flag, sizeof(int), cudaMemcpyDeviceToHost));
  d->mode = peer_ok ? MERGE_PEER : MERGE_NCCL;
  ++sc->gen;
  return CRSH_OK;
}

const char* crsh_last_error(void) { return g_err.c_str(); }

int64_t crsh_num_slots(int32_t P, int32_t n_lights, uint32_t t) {
  if (P < 0 || n_lights < 0) return 0;
  return (int64_t)P * (((t & 1u) ? n_lights : 0) + ((t & 2u) ? 1 : 0) + ((t & 4u) ? 1 : 0));
}

crsh_status crsh_scene_create(const float* tris, const int32_t* mesh_ids, int64_t M, int32_t device,
                              crsh_scene_t* out) {
  if (!out) return fail(CRSH_EINVAL, "out is null");
  *out = nullptr;
  if (!tris || !mesh_ids) return fail(CRSH_EINVAL, "null geometry");
  if (M < 1 || M >= (1ll << 31)) return fail(CRSH_ELIMIT, "M must be in [1, 2^31)");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return fail(CRSH_ECUDA, "no CUDA device: %s", cudaGetErrorString(e));
  if (device < 0 || device >= ndev) return fail(CRSH_EINVAL, "bad device ordinal");
  CK(cudaSetDevice(device));
  std::vector<float> ht(9 * (size_t)M);
  std::vector<int32_t> hm((size_t)M);
  CK(cudaMemcpy(ht.data(), tris, 36 * (size_t)M, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hm.data(), mesh_ids, 4 * (size_t)M, cudaMemcpyDeviceToHost));
  if (hm[0] != 0) return fail(CRSH_EINVAL, "mesh ids must start at 0");
  for (int64_t t = 1; t < M; ++t)
    if (hm[t] < hm[t - 1] || hm[t] > hm[t - 1] + 1) return fail(CRSH_EINVAL, "mesh ids must be non-decreasing and dense");
  const int32_t n_meshes = hm[M - 1] + 1;
  if (n_meshes > 2048) return fail(CRSH_ELIMIT, "more than 2048 meshes");
  auto* sc = new crsh_scene();
  sc->device = device;
  sc->M = M;
  sc->n_meshes = n_meshes;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) sc->sm_count = prop.multiProcessorCount;
  for (int k = 0; k < 3; ++k) { sc->box_min[k] = INFINITY; sc->box_max[k] = -INFINITY; }
  for (int64_t i = 0; i < 9 * M; ++i) {   // every vertex coordinate
    const int k = (int)(i % 3);
    sc->box_min[k] = std::min(sc->box_min[k], ht[i]);
    sc->box_max[k] = std::max(sc->box_max[k], ht[i]);
  }
  double diag = 0.0;
  for (int k = 0; k < 3; ++k) {
    const double ext = (double)sc->box_max[k] - (double)sc->box_min[k];
    diag += ext * ext;
    sc->box_ext[k] = sc->box_max[k] - sc->box_min[k];
  }
  diag = std::sqrt(diag);
  sc->pad = (float)(1e-5 * diag);
  sc->eps_t = (float)(1e-4 * diag);
  auto bail = [&](crsh_status s) { crsh_scene_destroy(sc); return s; };
  crsh_status rc = CRSH_OK;
  auto ck = [&](cudaError_t err, const char* what) {
    if (err != cudaSuccess && rc == CRSH_OK)
      rc = fail(err == cudaErrorMemoryAllocation ? CRSH_ENOMEM : CRSH_ECUDA, "%s: %s", what, cudaGetErrorString(err));
  };
  ck(ensure(sc->tri_e, 48 * (size_t)M), "alloc tri_e");
  ck(ensure(sc->tri_sph, 16 * (size_t)M), "alloc tri_sph");
  ck(ensure(sc->mesh_sph, 16 * (size_t)n_meshes), "alloc mesh_sph");
  ck(ensure(sc->mesh_first, 4 * (size_t)n_meshes), "alloc mesh_first");
  ck(ensure(sc->mesh_count, 4 * (size_t)n_meshes), "alloc mesh_count");
  ck(cudaMallocHost(&sc->h_counters, 8 * MAX_SEG * CTR_STRIDE), "alloc pinned");
  ck(cudaMallocHost(&sc->h_fd, sizeof(FrameDesc)), "alloc pinned");
  ck(cudaStreamCreateWithFlags(&sc->gstream, cudaStreamNonBlocking), "graph stream");
  ck(cudaEventCreateWithFlags(&sc->ev_in, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&sc->ev_out, cudaEventDisableTiming), "event");
  for (int i = 0; i < 10 && rc == CRSH_OK; ++i) ck(cudaEventCreate(&sc->ev[i]), "event");
  if (rc != CRSH_OK) return bail(rc);
  std::memset(sc->h_counters, 0, 8 * MAX_SEG * CTR_STRIDE);
  k_tri_prep<<<std::min<int64_t>((M + 255) / 256, 8 * sc->sm_count), 256>>>(tris, M, sc->pad, sc->tri_e.as<float4>(),
                                                                          sc->tri_sph.as<float4>());
  ck(cudaGetLastError(), "k_tri_prep");
  std::vector<uint32_t> first(n_meshes, 0), count(n_meshes, 0);
  for (int64_t t = 0; t < M; ++t) {
    if (count[hm[t]] == 0) first[hm[t]] = (uint32_t)t;
    ++count[hm[t]];
  }
  sc->h_mesh_sph.assign(4 * (size_t)n_meshes, 0.0f);
  for (int m = 0; m < n_meshes; ++m) {
    if (count[m] == 0) { sc->h_mesh_sph[4 * m + 3] = -1.0f; continue; }
    mesh_sphere(ht.data(), first[m], first[m] + count[m], sc->pad, &sc->h_mesh_sph[4 * m]);
  }
  ck(cudaMemcpy(sc->mesh_sph.p, sc->h_mesh_sph.data(), 16 * (size_t)n_meshes, cudaMemcpyHostToDevice), "copy mesh_sph");
  sc->h_mesh_sph0 = sc->h_mesh_sph;
  ck(ensure(sc->tris0, 36 * (size_t)M), "alloc tris0");
  ck(ensure(sc->mesh_ids, 4 * (size_t)M), "alloc mesh_ids");
  if (rc == CRSH_OK) {
    ck(cudaMemcpy(sc->tris0.p, tris, 36 * (size_t)M, cudaMemcpyDeviceToDevice), "copy tris0");
    ck(cudaMemcpy(sc->mesh_ids.p, mesh_ids, 4 * (size_t)M, cudaMemcpyDeviceToDevice), "copy mesh ids");
  }
  ck(cudaMemcpy(sc->mesh_first.p, first.data(), 4 * (size_t)n_meshes, cudaMemcpyHostToDevice), "copy first");
  ck(cudaMemcpy(sc->mesh_count.p, count.data(), 4 * (size_t)n_meshes, cudaMemcpyHostToDevice), "copy count");
  for (int32_t m = 0; m < n_meshes; ++m) sc->n_nonempty += count[m] ? 1 : 0;
  {   // object sphere-tree (CRSH_F_OBJTREE): cluster order on the host, spheres on the device
    std::vector<int32_t> order;
    std::vector<uint32_t> cfirst, crange;
    cluster_order(ht.data(), first, count, order, cfirst, crange);
    sc->n_clusters = (int64_t)(crange.size() / 2);
    ck(ensure(sc->cl_order, 4 * (size_t)M), "alloc cl_order");
    ck(ensure(sc->cl_first, 4 * ((size_t)n_meshes + 1)), "alloc cl_first");
    ck(ensure(sc->cl_range, 8 * (size_t)std::max<int64_t>(sc->n_clusters, 1)), "alloc cl_range");
    ck(ensure(sc->cl_sph, 16 * (size_t)std::max<int64_t>(sc->n_clusters, 1)), "alloc cl_sph");
    ck(ensure(sc->tri_sph_ord, 16 * (size_t)M), "alloc tri_sph_ord");
    ck(ensure(sc->cl_pf, 16 * (size_t)std::max<int64_t>(sc->n_clusters, 1)), "alloc cl_pf");
    if (rc == CRSH_OK) {
      ck(cudaMemcpy(sc->cl_order.p, order.data(), 4 * (size_t)M, cudaMemcpyHostToDevice), "copy cl_order");
      ck(cudaMemcpy(sc->cl_first.p, cfirst.data(), 4 * cfirst.size(), cudaMemcpyHostToDevice), "copy cl_first");
      if (!crange.empty())
        ck(cudaMemcpy(sc->cl_range.p, crange.data(), 4 * crange.size(), cudaMemcpyHostToDevice), "copy cl_range");
    }
    if (rc == CRSH_OK) {
      const int grid = (int)std::min<int64_t>((std::max<int64_t>(sc->n_clusters, M) + 255) / 256, 8 * sc->sm_count);
      k_cluster_prep<<<grid, 256>>>(tris, sc->cl_order.as<int32_t>(), sc->cl_range.as<uint2>(), sc->n_clusters, sc->pad,
                                    sc->cl_sph.as<float4>());
      k_permute_sph<<<grid, 256>>>(sc->tri_sph.as<float4>(), sc->cl_order.as<int32_t>(), M, sc->tri_sph_ord.as<float4>());
      k_cluster_pf<<<grid, 256>>>(sc->cl_sph.as<float4>(), sc->tri_sph_ord.as<float4>(), sc->cl_range.as<uint2>(),
                                  sc->n_clusters, sc->cl_pf.as<float4>());
      ck(cudaGetLastError(), "k_cluster_prep");
    }
  }
  ck(cudaDeviceSynchronize(), "scene prep");
  if (rc != CRSH_OK) return bail(rc);
  *out = sc;
  return CRSH_OK;
}

void crsh_scene_destroy(crsh_scene_t sc) {
  if (!sc) return;
  cudaSetDevice(sc->device);
  Buf* bufs[] = {&sc->tri_e, &sc->tri_sph, &sc->mesh_sph, &sc->mesh_first, &sc->mesh_count, &sc->rays, &sc->keys_c,
                 &sc->vals_c, &sc->ckey, &sc->cbase, &sc->k1, &sc->v1, &sc->k2, &sc->v2, &sc->pos, &sc->first_chunk,
                 &sc->sorted_key, &sc->sorted_slot, &sc->sorted_rays, &sc->px_tiles, &sc->nodes, &sc->trav, &sc->masks, &sc->gwork, &sc->gstat, &sc->items,
                 &sc->best, &sc->zero, &sc->stage_in, &sc->stage_out};
  for (Buf* b : bufs) b->release();
  for (auto& w : sc->wb) for (auto& b : w) b.release();
  sc->w_hit.release(); sc->w_t.release(); sc->w_zero.release(); sc->prim_rays.release();
  sc->tris0.release(); sc->mesh_ids.release(); sc->tris_cur.release(); sc->xf.release(); sc->boxk.release();
  sc->cl_order.release(); sc->cl_range.release(); sc->cl_first.release(); sc->cl_sph.release(); sc->tri_sph_ord.release(); sc->cl_pf.release();
  if (sc->dist) {
    Dist* d = sc->dist;
    if (d->win) ncclCommWindowDeregister(d->comm, d->win);
    if (d->wbuf) ncclMemFree(d->wbuf);
    if (d->dev_ok) ncclDevCommDestroy(d->comm, &d->dev);
    if (d->d_ptrs) cudaFree(d->d_ptrs);
    if (d->comm) ncclCommDestroy(d->comm);
    delete d;
    sc->dist = nullptr;
  }
  if (sc->h_counters) cudaFreeHost(sc->h_counters);
  if (sc->h_fd) cudaFreeHost(sc->h_fd);
  if (sc->gexec) cudaGraphExecDestroy(sc->gexec);
  if (sc->gstream) cudaStreamDestroy(sc->gstream);
  if (sc->ev_in) cudaEventDestroy(sc->ev_in);
  if (sc->ev_out) cudaEventDestroy(sc->ev_out);
  for (auto& e : sc->ev) if (e) cudaEventDestroy(e);
  delete sc;
}

crsh_status crsh_trace_secondary(crsh_scene_t sc, const crsh_primary_hits* h, const float* lights, int32_t n_lights,
                                 uint32_t types, const crsh_opts* o, int32_t* hit_tri, float* t, void* stream) {
  return trace_impl(sc, h, lights, n_lights, types, o, hit_tri, t, nullptr, PeerOut{}, (cudaStream_t)stream, true,
                    nullptr, true);
}

crsh_status crsh_trace_secondary_packed(crsh_scene_t sc, const crsh_primary_hits* h, const float* lights,
                                        int32_t n_lights, uint32_t types, const crsh_opts* o, uint64_t* packed,
                                        void* stream) {
  if (!packed) return fail(CRSH_EINVAL, "packed is null");
  return trace_impl(sc, h, lights, n_lights, types, o, nullptr, nullptr,
                    reinterpret_cast<unsigned long long*>(packed), PeerOut{}, (cudaStream_t)stream);
}

crsh_status crsh_trace_secondary_peer(crsh_scene_t sc, const crsh_primary_hits* h, const float* lights,
                                      int32_t n_lights, uint32_t types, const crsh_opts* o, uint64_t* const* dst,
                                      int32_t n_dst, void* stream) {
  if (!dst || n_dst < 1 || n_dst > MAX_PEERS) return fail(CRSH_EINVAL, "dst must hold 1..8 device pointers");
  PeerOut peer{};
  for (int d = 0; d < n_dst; ++d) {
    if (!dst[d]) return fail(CRSH_EINVAL, "null destination pointer");
    peer.p[d] = reinterpret_cast<unsigned long long*>(dst[d]);
  }
  peer.n = n_dst;
  return trace_impl(sc, h, lights, n_lights, types, o, nullptr, nullptr, nullptr, peer, (cudaStream_t)stream);
}

}  // extern "C"

namespace {
// largest singular value of the 3x3 part of a row-major [A | b]: sqrt of the
// largest eigenvalue of A^T A by the closed trigonometric form (double)
double sigma_max3(const float* x) {
  double A[3][3], S[3][3];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) A[r][c] = (double)x[4 * r + c];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) S[i][j] = A[0][i] * A[0][j] + A[1][i] * A[1][j] + A[2][i] * A[2][j];
  const double off = S[0][1] * S[0][1] + S[0][2] * S[0][2] + S[1][2] * S[1][2];
  double lam;
  if (off == 0.0) {
    lam = std::max(S[0][0], std::max(S[1][1], S[2][2]));
  } else {
    const double q = (S[0][0] + S[1][1] + S[2][2]) / 3.0;
    const double p2 = (S[0][0] - q) * (S[0][0] - q) + (S[1][1] - q) * (S[1][1] - q) + (S[2][2] - q) * (S[2][2] - q) + 2.0 * off;
    const double p = std::sqrt(p2 / 6.0);
    double Bm[3][3];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) Bm[i][j] = (S[i][j] - (i == j ? q : 0.0)) / p;
    const double det = Bm[0][0] * (Bm[1][1] * Bm[2][2] - Bm[1][2] * Bm[2][1]) -
                       Bm[0][1] * (Bm[1][0] * Bm[2][2] - Bm[1][2] * Bm[2][0]) +
                       Bm[0][2] * (Bm[1][0] * Bm[2][1] - Bm[1][1] * Bm[2][0]);
    const double r = det / 2.0;
    const double phi = r <= -1.0 ? M_PI / 3.0 : (r >= 1.0 ? 0.0 : std::acos(r) / 3.0);
    lam = q + 2.0 * p * std::cos(phi);
  }
  return std::sqrt(std::max(lam, 0.0));
}
inline int float_key(float f) { const int i = __builtin_bit_cast(int, f); return i >= 0 ? i : (i ^ 0x7FFFFFFF); }
inline float key_float(int k) { return __builtin_bit_cast(float, k >= 0 ? k : (k ^ 0x7FFFFFFF)); }
}  // namespace

extern "C" {

crsh_status crsh_scene_transform(crsh_scene_t sc, const float* xforms) {
  if (!sc || !xforms) return fail(CRSH_EINVAL, "null argument");
  CK(cudaSetDevice(sc->device));
  // an in-flight frame (on the caller's stream or the scene's graph stream,
  // both possibly non-blocking) still reads the geometry rewritten below
  CK(cudaStreamSynchronize(sc->last_stream));
  if (sc->gstream) CK(cudaStreamSynchronize(sc->gstream));
  const int n = sc->n_meshes;
  for (int i = 0; i < 12 * n; ++i)
    if (!std::isfinite(xforms[i])) return fail(CRSH_EINVAL, "non-finite transform");
  CK(ensure(sc->tris_cur, 36 * (size_t)sc->M));
  CK(ensure(sc->xf, 48 * (size_t)n));
  CK(ensure(sc->boxk, 32));
  CK(cudaMemcpy(sc->xf.p, xforms, 48 * (size_t)n, cudaMemcpyHostToDevice));
  const int init[6] = {float_key(INFINITY), float_key(INFINITY), float_key(INFINITY),
                       float_key(-INFINITY), float_key(-INFINITY), float_key(-INFINITY)};
  CK(cudaMemcpy(sc->boxk.p, init, sizeof init, cudaMemcpyHostToDevice));
  const int grid = (int)std::min<int64_t>((sc->M + 255) / 256, 8 * sc->sm_count);
  k_transform<<<grid, 256>>>(sc->tris0.as<float>(), sc->mesh_ids.as<int32_t>(), sc->M, sc->xf.as<float>(),
                             sc->tris_cur.as<float>(), sc->boxk.as<float>());
  CK(cudaGetLastError());
  k_tri_prep<<<grid, 256>>>(sc->tris_cur.as<float>(), sc->M, sc->pad, sc->tri_e.as<float4>(), sc->tri_sph.as<float4>());
  CK(cudaGetLastError());
  // object-tree clusters: creation-time order, spheres of the moved vertices
  k_cluster_prep<<<grid, 256>>>(sc->tris_cur.as<float>(), sc->cl_order.as<int32_t>(), sc->cl_range.as<uint2>(),
                                sc->n_clusters, sc->pad, sc->cl_sph.as<float4>());
  k_permute_sph<<<grid, 256>>>(sc->tri_sph.as<float4>(), sc->cl_order.as<int32_t>(), sc->M, sc->tri_sph_ord.as<float4>());
  k_cluster_pf<<<grid, 256>>>(sc->cl_sph.as<float4>(), sc->tri_sph_ord.as<float4>(), sc->cl_range.as<uint2>(),
                              sc->n_clusters, sc->cl_pf.as<float4>());
  CK(cudaGetLastError());
  int box[6];
  CK(cudaMemcpy(box, sc->boxk.p, sizeof box, cudaMemcpyDeviceToHost));
  for (int k = 0; k < 3; ++k) {
    sc->box_min[k] = key_float(box[k]);
    sc->box_max[k] = key_float(box[3 + k]);
    sc->box_ext[k] = sc->box_max[k] - sc->box_min[k];
  }
  // bounding-volume update: centre transformed, radius scaled by
  // sigma_max and rounded up -- the creation-time spheres are not recomputed
  for (int m = 0; m < n; ++m) {
    const float* s0 = &sc->h_mesh_sph0[4 * m];
    float* s1 = &sc->h_mesh_sph[4 * m];
    if (s0[3] < 0.0f) { for (int k = 0; k < 4; ++k) s1[k] = s0[k]; continue; }
    const float* a = xforms + 12 * m;
    for (int r = 0; r < 3; ++r)
      s1[r] = std::fmaf(a[4 * r], s0[0], std::fmaf(a[4 * r + 1], s0[1], std::fmaf(a[4 * r + 2], s0[2], a[4 * r + 3])));
    const double want = (double)s0[3] * sigma_max3(a);
    float rf = (float)want;
    if ((double)rf < want) rf = std::nextafter(rf, INFINITY);
    s1[3] = rf;
  }
  CK(cudaMemcpy(sc->mesh_sph.p, sc->h_mesh_sph.data(), 16 * (size_t)n, cudaMemcpyHostToDevice));
  ++sc->gen;   // scene constants changed: recapture the frame graph
  return CRSH_OK;
}

crsh_status crsh_trace_rays(crsh_scene_t sc, const float* rays, int64_t n, const crsh_opts* o, int32_t* hit_tri,
                            float* t, void* stream) {
  if (!sc || !o || !hit_tri || !t || (n > 0 && !rays)) return fail(CRSH_EINVAL, "null argument");
  if (n < 0 || n >= (1ll << 30)) return fail(CRSH_ELIMIT, "n must be in [0, 2^30)");
  if (n == 0) return CRSH_OK;
  // a one-segment frame (the bounce-type segment, slot i = ray i) whose K1
  // reads the given rays instead of generating them from a G-buffer
  crsh_primary_hits h{};
  h.width = (int32_t)n; h.height = 1;
  h.pos = rays; h.nrm = rays; h.mat = reinterpret_cast<const int32_t*>(rays);
  h.n_mat = 0;
  return trace_impl(sc, &h, nullptr, 0, CRSH_REFLECT, o, hit_tri, t, nullptr, PeerOut{}, (cudaStream_t)stream, true,
                    reinterpret_cast<const float4*>(rays));
}

crsh_status crsh_primary_gbuffer(crsh_scene_t sc, const crsh_camera* cam, int32_t width, int32_t height,
                                 const int32_t* tri_mat, const crsh_opts* o, float* pos, float* nrm, int32_t* mat,
                                 int32_t* hit_tri, float* t, void* stream) {
  if (!sc || !cam || !tri_mat || !o || !pos || !nrm || !mat || !hit_tri || !t) return fail(CRSH_EINVAL, "null argument");
  if (width <= 0 || height <= 0 || (int64_t)width * height >= (1ll << 30)) return fail(CRSH_ELIMIT, "bad image size");
  if (o->shard_world > 1) return fail(CRSH_EINVAL, "the primary pass runs on one rank");
  const int64_t P = (int64_t)width * height;
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(sc->device));
  CK(ensure(sc->prim_rays, 32 * (size_t)P));
  CameraArgs c{};
  for (int k = 0; k < 3; ++k) {
    c.eye[k] = cam->eye[k]; c.right[k] = cam->right[k]; c.up[k] = cam->up[k]; c.fwd[k] = cam->fwd[k];
  }
  c.tan_half = cam->tan_half_vfov; c.W = width; c.H = height; c.rays = sc->prim_rays.as<float4>();
  k_camera_rays<<<cdiv((uint64_t)P, 256), 256, 0, st>>>(c);
  CK(cudaGetLastError());
  crsh_status rc = crsh_trace_rays(sc, sc->prim_rays.as<float>(), P, o, hit_tri, t, stream);
  if (rc != CRSH_OK) return rc;
  GbufArgs g{};
  g.P = P; g.rays = c.rays; g.hit_tri = hit_tri; g.t = t; g.tri_e = sc->tri_e.as<float4>(); g.tri_mat = tri_mat;
  g.pos = pos; g.nrm = nrm; g.mat = mat;
  k_gbuffer<<<cdiv((uint64_t)P, 256), 256, 0, st>>>(g);
  CK(cudaGetLastError());
  sc->launches += 2;
  return CRSH_OK;
}

crsh_status crsh_render_whitted(crsh_scene_t sc, const crsh_primary_hits* gbuf, const float* lights, int32_t n_lights,
                                const int32_t* tri_mat, int32_t depth, const crsh_opts* o, float* image,
                                crsh_whitted_stats_t* wst, void* stream) {
  if (!sc || !gbuf || !o || !image || !tri_mat) return fail(CRSH_EINVAL, "null argument");
  if (depth < 0 || depth > CRSH_MAX_BOUNCES) return fail(CRSH_EINVAL, "depth must be in [0, 8]");
  if (o->shard_world > 1) return fail(CRSH_EINVAL, "crsh_render_whitted runs on one rank");
  if (o->flags & CRSH_F_BRUTE) return fail(CRSH_EINVAL, "crsh_render_whitted traces with the hierarchy");
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaSetDevice(sc->device));
  if (wst) { std::memset(wst, 0, sizeof(*wst)); wst->bounces = depth; }
  if ((int)sc->wb.size() < depth + 1) sc->wb.resize(depth + 1);
  crsh_primary_hits cur = *gbuf;
  std::vector<int64_t> Pd;
  int last = -1;
  int64_t launches = 0;
  for (int d = 0; d <= depth; ++d) {
    const int64_t P = (int64_t)cur.width * cur.height;
    Pd.push_back(P);
    last = d;
    auto& B = sc->wb[d];
    for (int i = 4; i < 8; ++i) CK(ensure(B[i], 4 * (size_t)std::max<int64_t>(P, 1)));
    if (wst) wst->vertices[d] = P;
    if (P == 0) break;
    const uint32_t types = (n_lights > 0 ? (uint32_t)CRSH_SHADOW : 0u) |
                           (d < depth ? (uint32_t)(CRSH_REFLECT | CRSH_REFRACT) : 0u);
    if (types == 0) {   // no lights at the last bounce: no direct term, no children
      CK(cudaMemsetAsync(B[4].p, 0, 4 * (size_t)P, st));
      break;
    }
    const int64_t S = crsh_num_slots((int32_t)P, n_lights, types);
    CK(ensure(sc->w_hit, 4 * (size_t)S));
    CK(ensure(sc->w_t, 4 * (size_t)S));
    int32_t* hit = sc->w_hit.as<int32_t>();
    float* tt = sc->w_t.as<float>();
    crsh_status rc = trace_impl(sc, &cur, lights, n_lights, types, o, hit, tt, nullptr, PeerOut{}, st, false);
    if (rc != CRSH_OK) return rc;
    launches += sc->launches;
    const FrameInfo fi = sc->fi;
    if (wst) {
      crsh_stats_t bs;
      rc = crsh_stats(sc, &bs);
      if (rc != CRSH_OK) return rc;
      for (int q = 0; q < 3; ++q) {
        wst->rays[d] += (int64_t)bs.rays[q];
        for (int k = 1; k <= MAX_LEVELS; ++k) wst->tests[d] += bs.tests[q][k];
        wst->final_tests[d] += bs.final_tests[q];
      }
    }
    // KW1: direct term + child placement
    const uint32_t tiles = cdiv((uint64_t)P, SCAN_TILE);
    CK(ensure(sc->w_zero, 8 * ((size_t)tiles + 2)));
    CK(cudaMemsetAsync(sc->w_zero.p, 0, 8 * ((size_t)tiles + 2), st));
    ShadeArgs a{};
    a.rg = raygen_def(sc, fi, &cur, lights, n_lights);
    a.hit_tri = hit;
    a.sh_slots = (types & CRSH_SHADOW) ? n_lights * (int32_t)P : 0;
    a.re0 = (types & CRSH_REFLECT) ? a.sh_slots : -1;
    a.rr0 = (types & CRSH_REFRACT) ? a.sh_slots + (int32_t)P : -1;
    a.spawn = d < depth ? 1 : 0;
    a.direct = B[4].as<float>(); a.c_re = B[5].as<int32_t>(); a.c_rr = B[6].as<int32_t>();
    a.count = sc->w_zero.as<uint32_t>();
    a.ticket = sc->w_zero.as<uint32_t>() + 1;
    a.status = sc->w_zero.as<unsigned long long>() + 1;
    k_shade<<<tiles, SCAN_THREADS, 0, st>>>(a);
    CK(cudaGetLastError());
    ++launches;
    if (d == depth) break;
    uint32_t k = 0;
    CK(cudaMemcpyAsync(&k, a.count, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (k == 0) break;   // no reflection / refraction hit: the last bounce
    // KW2: the children become the next bounce's vertex set
    auto& N = sc->wb[d + 1];
    for (int i = 0; i < 3; ++i) CK(ensure(N[i], 12 * (size_t)k));
    CK(ensure(N[3], 4 * (size_t)k));
    SpawnArgs sp{};
    sp.rg = a.rg; sp.hit_tri = hit; sp.t = tt; sp.re0 = a.re0; sp.rr0 = a.rr0;
    sp.c_re = a.c_re; sp.c_rr = a.c_rr; sp.tri_e = sc->tri_e.as<float4>(); sp.tri_mat = tri_mat; sp.k = k;
    sp.npos = N[0].as<float>(); sp.nnrm = N[1].as<float>(); sp.ndir = N[2].as<float>(); sp.nmat = N[3].as<int32_t>();
    k_spawn<<<cdiv((uint64_t)P, 256), 256, 0, st>>>(sp);
    CK(cudaGetLastError());
    ++launches;
    cur.width = (int32_t)k; cur.height = 1;
    cur.pos = sp.npos; cur.nrm = sp.nnrm; cur.mat = sp.nmat; cur.dir = sp.ndir;
  }
  // KW3: radiance from the deepest bounce up; bounce 0 writes the image
  for (int d = last; d >= 0; --d) {
    const int64_t P = Pd[d];
    if (P == 0) continue;
    auto& B = sc->wb[d];
    const bool has_next = d < last && Pd[d + 1] > 0;
    const int32_t* mat = d == 0 ? gbuf->mat : sc->wb[d][3].as<int32_t>();
    k_backprop<<<cdiv((uint64_t)P, 256), 256, 0, st>>>(
        (int32_t)P, mat, gbuf->materials, gbuf->n_mat, B[4].as<float>(), has_next ? B[5].as<int32_t>() : nullptr,
        has_next ? B[6].as<int32_t>() : nullptr, has_next ? sc->wb[d + 1][7].as<float>() : nullptr,
        d == 0 ? image : B[7].as<float>());
    CK(cudaGetLastError());
    ++launches;
  }
  sc->launches = launches;
  return CRSH_OK;
}

crsh_status crsh_unpack_hits(crsh_scene_t sc, const uint64_t* packed, int64_t slots, int32_t* hit_tri, float* t,
                             void* stream) {
  if (!sc || !packed || !hit_tri || !t || slots < 0) return fail(CRSH_EINVAL, "bad unpack arguments");
  if (slots == 0) return CRSH_OK;
  CK(cudaSetDevice(sc->device));
  k_unpack_packed<<<std::min<int64_t>((slots + 255) / 256, 8 * sc->sm_count), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const unsigned long long*>(packed), (uint64_t)slots, hit_tri, t);
  CK(cudaGetLastError());
  return CRSH_OK;
}

crsh_status crsh_trace_secondary_host(crsh_scene_t sc, const crsh_primary_hits* h, const float* lights,
                                      int32_t n_lights, uint32_t types, const crsh_opts* o, int32_t* hit_tri,
                                      float* t, void* stream) {
  if (!sc || !h || !hit_tri || !t) return fail(CRSH_EINVAL, "null argument");
  if (h->width <= 0 || h->height <= 0) return fail(CRSH_EINVAL, "width/height must be positive");
  CK(cudaSetDevice(sc->device));
  const size_t P = (size_t)h->width * h->height;
  const int64_t S = crsh_num_slots((int32_t)P, n_lights, types);
  cudaStream_t st = (cudaStream_t)stream;
  if (h->dir) return fail(CRSH_EINVAL, "dir must be NULL for crsh_trace_secondary_host");
  const size_t in_bytes = 28 * P + 12 * (size_t)std::max(h->n_mat, 0);
  CK(ensure(sc->stage_in, in_bytes + 64));
  CK(ensure(sc->stage_out, 8 * (size_t)std::max<int64_t>(S, 1)));
  char* din = sc->stage_in.as<char>();
  float* dpos = reinterpret_cast<float*>(din);
  float* dnrm = dpos + 3 * P;
  int32_t* dmat = reinterpret_cast<int32_t*>(dnrm + 3 * P);
  float* dmats = reinterpret_cast<float*>(dmat + P);
  CK(cudaMemcpyAsync(dpos, h->pos, 12 * P, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dnrm, h->nrm, 12 * P, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dmat, h->mat, 4 * P, cudaMemcpyHostToDevice, st));
  if (h->n_mat > 0) CK(cudaMemcpyAsync(dmats, h->materials, 12 * (size_t)h->n_mat, cudaMemcpyHostToDevice, st));
  crsh_primary_hits dh = *h;
  dh.pos = dpos; dh.nrm = dnrm; dh.mat = dmat; dh.materials = dmats;
  int32_t* dhit = sc->stage_out.as<int32_t>();
  float* dt = reinterpret_cast<float*>(dhit + S);
  crsh_status rc = trace_impl(sc, &dh, lights, n_lights, types, o, dhit, dt, nullptr, PeerOut{}, st, true, nullptr, true);
  if (rc != CRSH_OK) return rc;
  CK(cudaMemcpyAsync(hit_tri, dhit, 4 * (size_t)S, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(t, dt, 4 * (size_t)S, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return CRSH_OK;
}

crsh_status crsh_stats(crsh_scene_t sc, crsh_stats_t* out) {
  if (!sc || !out) return fail(CRSH_EINVAL, "null argument");
  crsh_status rc = sync_frame(sc);
  if (rc != CRSH_OK) return rc;
  std::memset(out, 0, sizeof(*out));
  const FrameInfo& fi = sc->fi;
  if (!fi.valid) return CRSH_OK;
  out->levels = fi.Lv;
  out->merge = sc->dist ? sc->dist->mode : MERGE_NONE;
  for (int s = 0; s < fi.n_seg; ++s) {
    const int ty = fi.seg_type[s];
    const unsigned long long* c = sc->h_counters + s * CTR_STRIDE;
    out->rays[ty] = fi.fd.seg_n[s];
    out->slots[ty] = fi.seg_slot_start[s + 1] - fi.seg_slot_start[s];
    out->chunks[ty] = (fi.sorted && !fi.brute) ? fi.fd.seg_C[s] : 0;
    for (int k = 1; k <= MAX_LEVELS; ++k) { out->tests[ty][k] = c[CTR_TESTS + k]; out->hits[ty][k] = c[CTR_HITS + k]; }
    out->mesh_tests[ty] = c[CTR_MESH_TESTS];
    out->mesh_hits[ty] = c[CTR_MESH_HITS];
    out->final_tests[ty] = c[CTR_FINAL_TESTS];
    out->final_hits[ty] = c[CTR_FINAL_HITS];
    out->rays_hit[ty] = c[CTR_RAYS_HIT];
    out->cluster_tests[ty] = c[CTR_CL_TESTS];
    out->cluster_hits[ty] = c[CTR_CL_HITS];
    out->skipped_tests[ty] = c[CTR_CH_SKIP];
    out->prefilter_tests[ty] = c[CTR_PF_TESTS];
    out->brute[ty] = (uint64_t)fi.fd.seg_n[s] * (uint64_t)sc->M;
  }
  if ((fi.timed || fi.ktimed) && fi.fd.N > 0) {
    for (int i = 0; i < 8; ++i) {
      if (!fi.timed && i != 6) continue;
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, sc->ev[i], sc->ev[i + 1]) == cudaSuccess) out->stage_ms[i] = ms;
      else out->stage_ms[i] = -1.0f;
    }
    (void)cudaGetLastError();   // a failed timing query must not poison the next launch check
  }
  return CRSH_OK;
}

int64_t crsh_launch_count(crsh_scene_t sc) { return sc ? sc->launches : 0; }

crsh_status crsh_debug_tap(crsh_scene_t sc, int32_t tap, int32_t seg_type, int32_t level, void* host_dst,
                           size_t cap_bytes, size_t* n_out) {
  if (!sc || !n_out) return fail(CRSH_EINVAL, "null argument");
  crsh_status rc0 = sync_frame(sc);
  if (rc0 != CRSH_OK) return rc0;
  *n_out = 0;
  const FrameInfo& fi = sc->fi;
  const FrameDesc& fd = fi.fd;
  const void* src = nullptr;
  size_t n = 0, esz = 4;
  std::vector<uint32_t> rel;
  if (tap == CRSH_TAP_TRI_SPHERES) { src = sc->tri_sph.p; n = (size_t)sc->M; esz = 16; }
  else if (tap == CRSH_TAP_MESH_SPHERES) { src = sc->mesh_sph.p; n = (size_t)sc->n_meshes; esz = 16; }
  else if (tap == CRSH_TAP_CLUSTER_SPHERES) { src = sc->cl_sph.p; n = (size_t)sc->n_clusters; esz = 16; }
  else if (tap == CRSH_TAP_CLUSTER_ORDER) { src = sc->cl_order.p; n = (size_t)sc->M; esz = 4; }
  else if (tap == CRSH_TAP_SCENE_CONSTS) {
    float c[8] = {sc->box_min[0], sc->box_min[1], sc->box_min[2], sc->box_max[0], sc->box_max[1], sc->box_max[2], sc->pad, sc->eps_t};
    *n_out = 8;
    if (cap_bytes < sizeof c) return fail(CRSH_EIO, "buffer too small");
    std::memcpy(host_dst, c, sizeof c);
    return CRSH_OK;
  } else if (tap == CRSH_TAP_GROUP_RANGE || tap == CRSH_TAP_GROUP_WORK) {
    if (!fi.valid) return fail(CRSH_EINVAL, "no trace yet");
    if (tap == CRSH_TAP_GROUP_RANGE) {
      const uint32_t r[3] = {fd.g_lo, fd.g_hi, fd.G};
      *n_out = 3;
      if (cap_bytes < sizeof r) return fail(CRSH_EIO, "buffer too small");
      std::memcpy(host_dst, r, sizeof r);
      return CRSH_OK;
    }
    if (fi.world <= 1 || fi.brute) return CRSH_OK;
    src = sc->gwork.p; n = fd.G; esz = 8;
  } else {
    if (!fi.valid) return fail(CRSH_EINVAL, "no trace yet");
    int s = -1;
    for (int q = 0; q < fi.n_seg; ++q) if (fi.seg_type[q] == seg_type) s = q;
    if (s < 0) return CRSH_OK;   // segment not present: empty
    const size_t ns = fd.seg_n[s];
    switch (tap) {
      case CRSH_TAP_KEYS: src = sc->keys_c.as<uint32_t>() + fd.seg_comp_start[s]; n = ns; break;
      case CRSH_TAP_VALS: src = sc->vals_c.as<uint32_t>() + fd.seg_comp_start[s]; n = ns; break;
      case CRSH_TAP_CHUNK_KEYS:
        if (!fi.sorted || fi.brute) return CRSH_OK;
        src = sc->ckey.as<uint32_t>() + fd.seg_chunk_start[s]; n = fd.seg_C[s]; break;
      case CRSH_TAP_CHUNK_BASE: {
        if (!fi.sorted || fi.brute) return CRSH_OK;
        n = fd.seg_C[s];
        rel.resize(n);
        if (n) CK(cudaMemcpy(rel.data(), sc->cbase.as<uint32_t>() + fd.seg_chunk_start[s], 4 * n, cudaMemcpyDeviceToHost));
        for (auto& v : rel) v -= fd.seg_comp_start[s];
        *n_out = n;
        if (cap_bytes < 4 * n) return fail(CRSH_EIO, "buffer too small");
        if (n) std::memcpy(host_dst, rel.data(), 4 * n);
        return CRSH_OK;
      }
      case CRSH_TAP_SORTED_KEYS: src = sc->sorted_key.as<uint32_t>() + fd.seg_pad_base[s]; n = ns; break;
      case CRSH_TAP_SORTED_SLOTS: src = sc->sorted_slot.as<uint32_t>() + fd.seg_pad_base[s]; n = ns; break;
      case CRSH_TAP_SORTED_RAYS:
        src = sc->sorted_rays.as<float4>() + 2 * (size_t)fd.seg_pad_base[s]; n = ns; esz = 32;
        if (fi.GR <= SMALL_GROUP_RAYS && ns) {   // not materialised (K8 gathers): gather them here
          CK(ensure(sc->stage_out, 32 * ns));
          k_gather_sorted<<<cdiv(ns, 256), 256>>>(sc->sorted_slot.as<uint32_t>() + fd.seg_pad_base[s],
                                                  sc->rays.as<float4>(), (uint32_t)ns, sc->stage_out.as<float4>());
          CK(cudaGetLastError());
          CK(cudaDeviceSynchronize());
          src = sc->stage_out.p;
        }
        break;
      case CRSH_TAP_NODES: {
        if (level < 1 || level > fi.Lv) return fail(CRSH_EINVAL, "bad level");
        uint64_t per = fi.B0;
        for (int k = 1; k < level; ++k) per *= fi.B;
        n = (size_t)((ns + per - 1) / per);
        src = sc->nodes.as<float4>() + 2 * (fi.level_off[level] + fd.seg_pad_base[s] / per);
        esz = 32;
        break;
      }
      default: return fail(CRSH_EINVAL, "unknown tap");
    }
  }
  *n_out = n;
  if (cap_bytes < n * esz) return fail(CRSH_EIO, "buffer too small");
  if (n) CK(cudaMemcpy(host_dst, src, n * esz, cudaMemcpyDeviceToHost));
  return CRSH_OK;
}

}  // extern "C"
