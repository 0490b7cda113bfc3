/* workloads/raster.c — z-buffer rasteriser that produces the G-buffer input.
 *
 * This is the paper's step 1, "Rasterization is performed as a first step"
 * (§3.2): the fragment shader writes position, normal and
 * material per pixel. It is an INPUT GENERATOR shared by the oracle and the
 * CUDA path; it holds none of the method's arithmetic (no secondary rays, no
 * hashing, no ray-triangle test). Coverage is decided in 2-D screen space with
 * edge functions; the fragment position is the intersection of the pixel's
 * primary ray with the covering triangle's plane (perspective-correct depth).
 * All arithmetic is double precision; outputs are rounded to float32
 * ("four 32 bit floats per pixel").
 *
 * Camera: eye, orthonormal (right, up, fwd), vertical field of view vfov_deg,
 * W x H pixels; pixel (i, j), j = 0 at the top, has index p = j*W + i and its
 * primary ray passes through the pixel centre.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double x, y, z; } d3;
static d3 mk(double x, double y, double z) { d3 r = {x, y, z}; return r; }
static d3 sub(d3 a, d3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
static double dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static d3 cross(d3 a, d3 b) {
  return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

#define NEAR_Z 1e-3

/* Clip polygon (camera space) against z >= NEAR_Z; returns new vertex count. */
static int clip_near(const d3* in, int n, d3* out) {
  int m = 0;
  for (int i = 0; i < n; ++i) {
    d3 a = in[i], b = in[(i + 1) % n];
    int ain = a.z >= NEAR_Z, bin = b.z >= NEAR_Z;
    if (ain) out[m++] = a;
    if (ain != bin) {
      double s = (NEAR_Z - a.z) / (b.z - a.z);
      out[m++] = mk(a.x + s * (b.x - a.x), a.y + s * (b.y - a.y), NEAR_Z);
    }
  }
  return m;
}

/* tris: [M][9] float (v0, v1, v2); tri_mat: [M] material id per triangle.
 * Outputs: pos [3][P], nrm [3][P] (SoA float32), mat [P] (-1 = no hit),
 * tri_id [P] (visible triangle or -1; for diagnostics only). */
int raster_gbuffer(const float* tris, const int32_t* tri_mat, int64_t M,
                   const double* eye_in, const double* fwd_in, const double* up_in,
                   double vfov_deg, int32_t W, int32_t H,
                   float* pos, float* nrm, int32_t* mat, int32_t* tri_id) {
  const int64_t P = (int64_t)W * H;
  d3 eye = mk(eye_in[0], eye_in[1], eye_in[2]);
  d3 fwd = mk(fwd_in[0], fwd_in[1], fwd_in[2]);
  d3 up0 = mk(up_in[0], up_in[1], up_in[2]);
  double fl = sqrt(dot(fwd, fwd));
  fwd = mk(fwd.x / fl, fwd.y / fl, fwd.z / fl);
  d3 right = cross(fwd, up0);
  double rl = sqrt(dot(right, right));
  if (!(rl > 0)) return 2;
  right = mk(right.x / rl, right.y / rl, right.z / rl);
  d3 up = cross(right, fwd);
  const double th = tan(vfov_deg * M_PI / 360.0);
  const double aspect = (double)W / (double)H;

  double* depth = (double*)malloc(sizeof(double) * (size_t)P);
  if (!depth) return 5;
  for (int64_t p = 0; p < P; ++p) { depth[p] = INFINITY; tri_id[p] = -1; }

  for (int64_t t = 0; t < M; ++t) {
    const float* v = tris + 9 * t;
    d3 w[3], c[3];
    for (int k = 0; k < 3; ++k) {
      w[k] = mk(v[3 * k], v[3 * k + 1], v[3 * k + 2]);
      d3 q = sub(w[k], eye);
      c[k] = mk(dot(q, right), dot(q, up), dot(q, fwd));
    }
    d3 n = cross(sub(w[1], w[0]), sub(w[2], w[0]));
    if (dot(n, n) == 0.0) continue; /* degenerate: covers nothing */
    d3 poly[8];
    int np = clip_near(c, 3, poly);
    if (np < 3) continue;
    /* screen coordinates: u in [0, W), v in [0, H) (v down) */
    double su[8], sv[8];
    double umin = 1e300, umax = -1e300, vmin = 1e300, vmax = -1e300;
    for (int k = 0; k < np; ++k) {
      double nx = poly[k].x / (poly[k].z * th * aspect);
      double ny = poly[k].y / (poly[k].z * th);
      su[k] = (nx + 1.0) * 0.5 * W;
      sv[k] = (1.0 - ny) * 0.5 * H;
      if (su[k] < umin) umin = su[k];
      if (su[k] > umax) umax = su[k];
      if (sv[k] < vmin) vmin = sv[k];
      if (sv[k] > vmax) vmax = sv[k];
    }
    int i0 = (int)fmax(0.0, ceil(umin - 0.5)), i1 = (int)fmin(W - 1.0, floor(umax - 0.5));
    int j0 = (int)fmax(0.0, ceil(vmin - 0.5)), j1 = (int)fmin(H - 1.0, floor(vmax - 0.5));
    if (i0 > i1 || j0 > j1) continue;
    for (int f = 1; f + 1 < np; ++f) { /* fan of the clipped polygon */
      const double ax = su[0], ay = sv[0], bx = su[f], by = sv[f], cx = su[f + 1], cy = sv[f + 1];
      double area = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
      if (area == 0.0) continue;
      for (int j = j0; j <= j1; ++j) {
        double py = j + 0.5;
        for (int i = i0; i <= i1; ++i) {
          double px = i + 0.5;
          double e0 = (bx - ax) * (py - ay) - (by - ay) * (px - ax);
          double e1 = (cx - bx) * (py - by) - (cy - by) * (px - bx);
          double e2 = (ax - cx) * (py - cy) - (ay - cy) * (px - cx);
          int inside = area > 0 ? (e0 >= 0 && e1 >= 0 && e2 >= 0) : (e0 <= 0 && e1 <= 0 && e2 <= 0);
          if (!inside) continue;
          double ndx = ((i + 0.5) / W) * 2.0 - 1.0;
          double ndy = 1.0 - ((j + 0.5) / H) * 2.0;
          d3 dir = mk(fwd.x + ndx * th * aspect * right.x + ndy * th * up.x,
                      fwd.y + ndx * th * aspect * right.y + ndy * th * up.y,
                      fwd.z + ndx * th * aspect * right.z + ndy * th * up.z);
          double dn = dot(n, dir);
          if (dn == 0.0) continue;
          double tt = dot(n, sub(w[0], eye)) / dn; /* along unnormalised dir */
          if (!(tt > 0)) continue;
          int64_t p = (int64_t)j * W + i;
          if (tt < depth[p]) { depth[p] = tt; tri_id[p] = (int32_t)t; }
        }
      }
    }
  }

  for (int64_t p = 0; p < P; ++p) {
    int64_t t = tri_id[p];
    if (t < 0) {
      mat[p] = -1;
      pos[p] = pos[P + p] = pos[2 * P + p] = 0.0f;
      nrm[p] = nrm[P + p] = 0.0f;
      nrm[2 * P + p] = 1.0f;
      continue;
    }
    int i = (int)(p % W), j = (int)(p / W);
    double ndx = ((i + 0.5) / W) * 2.0 - 1.0;
    double ndy = 1.0 - ((j + 0.5) / H) * 2.0;
    d3 dir = mk(fwd.x + ndx * th * aspect * right.x + ndy * th * up.x,
                fwd.y + ndx * th * aspect * right.y + ndy * th * up.y,
                fwd.z + ndx * th * aspect * right.z + ndy * th * up.z);
    double tt = depth[p];
    pos[p] = (float)(eye.x + tt * dir.x);
    pos[P + p] = (float)(eye.y + tt * dir.y);
    pos[2 * P + p] = (float)(eye.z + tt * dir.z);
    const float* v = tris + 9 * t;
    d3 a = mk(v[0], v[1], v[2]), b = mk(v[3], v[4], v[5]), c = mk(v[6], v[7], v[8]);
    d3 n = cross(sub(b, a), sub(c, a));
    double nl = sqrt(dot(n, n));
    n = mk(n.x / nl, n.y / nl, n.z / nl);
    if (dot(n, dir) > 0) n = mk(-n.x, -n.y, -n.z); /* faces the camera */
    nrm[p] = (float)n.x;
    nrm[P + p] = (float)n.y;
    nrm[2 * P + p] = (float)n.z;
    mat[p] = tri_mat[t];
  }
  free(depth);
  return 0;
}
