// k_primary.cuh — GPU primary pass ("a G-buffer
// producer in the library instead of rasterization"): pixel-centre
// camera rays are traced through the same CRSH pipeline (ray-batch mode of
// K1), and the closest hits become the G-buffer the secondary pass reads
// (position, camera-facing geometric normal, material).
#pragma once
#include "common.cuh"
#include "numspec.cuh"

namespace crsh {

struct CameraArgs {
  float eye[3], right[3], up[3], fwd[3];
  float tan_half;              // tan(vfov / 2)
  int32_t W, H;
  float4* rays;                // [P][2] out: {eye, 0}, {d, +inf}
};

// pixel (i, j), j = 0 at the top: u = ((2i+1)/W - 1) tan aspect,
// v = (1 - (2j+1)/H) tan, d = norm(u right + v up + fwd) (fma order below)
__global__ void __launch_bounds__(256) k_camera_rays(const CameraArgs a) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= (int64_t)a.W * a.H) return;
  const int32_t i = (int32_t)(p % a.W), j = (int32_t)(p / a.W);
  const float ax = a.tan_half * ((float)a.W / (float)a.H);
  const float u = ((float)(2 * i + 1) / (float)a.W - 1.0f) * ax;
  const float v = (1.0f - (float)(2 * j + 1) / (float)a.H) * a.tan_half;
  const f3 dd = mk3(__fmaf_rn(u, a.right[0], __fmaf_rn(v, a.up[0], a.fwd[0])),
                    __fmaf_rn(u, a.right[1], __fmaf_rn(v, a.up[1], a.fwd[1])),
                    __fmaf_rn(u, a.right[2], __fmaf_rn(v, a.up[2], a.fwd[2])));
  const f3 d = norm3(dd);
  a.rays[2 * p] = make_float4(a.eye[0], a.eye[1], a.eye[2], 0.0f);
  a.rays[2 * p + 1] = make_float4(d.x, d.y, d.z, __int_as_float(0x7f800000));
}

struct GbufArgs {
  int64_t P;
  const float4* rays;
  const int32_t* hit_tri;
  const float* t;
  const float4* tri_e;         // {v0},{e1},{e2}
  const int32_t* tri_mat;
  float* pos;                  // [3][P]
  float* nrm;                  // [3][P]
  int32_t* mat;                // [P]
};

// hit: pos = fma(t, d, o) per axis, n = norm(e1 x e2) turned to face the
// camera (dot(d, n) > 0 -> -n), material of the triangle; miss: 0, 0, -1
__global__ void __launch_bounds__(256) k_gbuffer(const GbufArgs a) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= a.P) return;
  const int32_t h = a.hit_tri[p];
  const size_t P = (size_t)a.P;
  if (h < 0) {
    a.pos[p] = a.pos[P + p] = a.pos[2 * P + p] = 0.0f;
    a.nrm[p] = a.nrm[P + p] = a.nrm[2 * P + p] = 0.0f;
    a.mat[p] = -1;
    return;
  }
  const float4 r0 = a.rays[2 * p], r1 = a.rays[2 * p + 1];
  const float th = a.t[p];
  const float4 e1 = __ldg(a.tri_e + 3 * (size_t)h + 1), e2 = __ldg(a.tri_e + 3 * (size_t)h + 2);
  f3 n = norm3(cross3(mk3(e1.x, e1.y, e1.z), mk3(e2.x, e2.y, e2.z)));
  const f3 d = mk3(r1.x, r1.y, r1.z);
  if (dot3(d, n) > 0.0f) n = neg3(n);
  a.pos[p] = __fmaf_rn(th, r1.x, r0.x);
  a.pos[P + p] = __fmaf_rn(th, r1.y, r0.y);
  a.pos[2 * P + p] = __fmaf_rn(th, r1.z, r0.z);
  a.nrm[p] = n.x; a.nrm[P + p] = n.y; a.nrm[2 * P + p] = n.z;
  a.mat[p] = __ldg(a.tri_mat + h);
}

}  // namespace crsh
