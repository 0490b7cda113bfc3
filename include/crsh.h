/* crsh.h — C ABI of the B200-native Coherent Ray-Space Hierarchy (CRSH)
 * secondary-ray path (Reis, Costa & Pereira, arXiv 2312.06538).
 *
 * Citations: "P:n" = line n of the paper text; "S:n" = line n of
 * SPEC.md; "R#" = a reading in DESIGN.md §3. The library is libcrsh.so in
 * paper_2312_06538_b200/ (hand-written sm_100a CUDA + C++ host runtime).
 *
 * Conventions for every call:
 *  - Pointers documented "device" must be CUDA device pointers on the scene's
 *    device; "host" pointers are ordinary host memory. No torch types.
 *  - All calls return a crsh_status; argument and limit errors are detected
 *    synchronously before any work is enqueued (CRSH_EINVAL / CRSH_ELIMIT).
 *    Asynchronous CUDA failures surface as CRSH_ECUDA from the failing call or
 *    from the next crsh_stats(). crsh_last_error() gives a thread-local text.
 *  - One scene is used by one host thread and one stream at a time.
 *  - There is no CPU fallback: without a usable CUDA device every compute call
 *    fails with CRSH_ECUDA.
 *  - Environment (read when a frame is planned; A/B and test hooks, none
 *    changes a result): CRSH_NO_GRAPH=1 launches the frame's kernels directly
 *    instead of replaying a CUDA graph; CRSH_ITEM_TRIS=<n> fixes the
 *    triangles per traversal work item; CRSH_BIG_TILES / CRSH_RLE_HIST = 0|1
 *    select the decompression-scan tile size / where the radix histograms are
 *    counted; CRSH_SLOT_MAJOR=1 selects the slot-major ray generator;
 *    CRSH_OBJ_LIST_CAP=<n> bounds the object tree's per-round cluster list;
 *    CRSH_NO_PREFILTER=1 disables K8's child prefilter and CRSH_TOP_PREFILTER=0|1
 *    overrides the per-hash choice of its top-level prefilter (crsh_stats_t);
 *    CRSH_DIST_MERGE=nccl (read by crsh_dist_init) the all-reduce merge.
 */
#ifndef CRSH_H_
#define CRSH_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct crsh_scene* crsh_scene_t;

/* Status codes; 2/3/4 mirror the CPU program's exit codes. */
typedef enum {
  CRSH_OK = 0,
  CRSH_EINVAL = 2, /* bad argument (null pointer, bad mesh ids, bad option) */
  CRSH_EIO = 3,    /* host buffer too small for a tap */
  CRSH_ELIMIT = 4, /* exceeds an encoding limit (lights > 16, slots >= 2^30, ...). The slot bound is 2^30,
                      not SURVEY §8(b)'s 2^32: the single-pass scans publish a flag and a 30-bit count in
                      one 32-bit look-back word (k_onesweep), and 2^30 slots already cover a 7680x4320
                      frame with 16 lights (and every frame of this path's configurations by far) */
  CRSH_ENOMEM = 5, /* device allocation failed */
  CRSH_ECUDA = 6,  /* CUDA runtime error (incl. no device) */
  CRSH_ENCCL = 7   /* NCCL failure (crsh_dist_*, the multi-GPU merge, asynchronous errors) */
} crsh_status;

/* Ray types (bitmask), "Batches can consist of any combination of
 * shadow rays, reflection rays or refraction rays". One hierarchy segment per
 * type (R5): segment 0 = SH (all lights), 1 = RE, 2 = RR. */
enum { CRSH_SHADOW = 1u, CRSH_REFLECT = 2u, CRSH_REFRACT = 4u };

/* Option flags. CRSH_F_SORT | CRSH_F_MESH_CULL is the paper's CRSH; neither is
 * the RAH baseline of P:47-49 (rays in generation order, no mesh spheres).
 * CRSH_F_ZORDER selects the Z-order (bit-interleaved) hash layout instead of
 * the concatenated layout of R6.
 * CRSH_F_STAGE_TIMING records per-stage CUDA-event times into stage_ms.
 * CRSH_F_BRUTE replaces the hierarchy by the N x M baseline (final_tests =
 * rays * M); the other flags are then ignored. */
enum {
  CRSH_F_SORT = 1u,
  CRSH_F_MESH_CULL = 2u,
  CRSH_F_ZORDER = 4u,
  CRSH_F_STAGE_TIMING = 8u,
  CRSH_F_BRUTE = 16u,  /* naive N x M ray tracing: every ray
                          against every triangle, no hierarchy; same outputs */
  CRSH_F_KERNEL_TIMING = 32u, /* time only the traversal kernel (stage_ms[6]) */
  CRSH_F_OBJTREE = 64u  /* object sphere-tree below the mesh spheres ("combine our
                           coherent ray hierarchy with a deeper object hierarchy"): each mesh's triangles in
                           Morton order of their centroids, in clusters of 32 with a bounding sphere each
                           (reading O1); a top node tests a kept mesh's cluster spheres (Eq 9) before
                           the triangles of the clusters that pass. Same hits; cluster_tests / cluster_hits
                           count the extra level and tests[Lv] only the triangles of passing clusters. */
};

/* Build a scene (untimed preparation): copies the geometry, computes
 * per-triangle v0/e1/e2 and padded minimal bounding spheres (R1, R2),
 * per-mesh minimal bounding spheres [Gar99], the scene AABB,
 * pad = 1e-5*diag and eps_t = 1e-4*diag (R2, R3).
 *   tris     device [M][9] float32: v0.xyz, v1.xyz, v2.xyz (row-major)
 *   mesh_ids device [M] int32, non-decreasing, dense from 0
 *   M        number of triangles, 1 <= M < 2^31
 *   device   CUDA device ordinal
 *   out      receives the scene handle (owned by the caller; destroy with
 *            crsh_scene_destroy). The caller may free tris/mesh_ids on return.
 * Errors: EINVAL (null / bad mesh ids), ELIMIT (M, meshes > 2048), ECUDA, ENOMEM. */
crsh_status crsh_scene_create(const float* tris, const int32_t* mesh_ids, int64_t M, int32_t device,
                              crsh_scene_t* out);
void crsh_scene_destroy(crsh_scene_t scene);

/* The primary-hit buffer (the paper's G-buffer: position, normal and
 * material per pixel). P = width*height; pixel p = y*width + x.
 *   pos, nrm  [3][P] float32 structure-of-arrays (x plane, y plane, z plane);
 *             nrm is the unit geometric normal
 *   mat       [P] int32 material index, -1 = no primary hit
 *   materials [n_mat][3] float32: reflectivity, transmissivity, ior
 *   eye       camera position (view vector for reflection/refraction)
 *   dir       optional [3][P] float32 SoA incident directions (unit), used
 *             instead of norm(pos - eye) as the view vector i of RE/RR rays:
 *             the vertices of a later Whitted bounce, whose incident rays
 *             are the previous bounce's secondary rays. NULL =
 *             the camera at `eye` (the primary G-buffer).
 * For crsh_trace_secondary these are device pointers; for
 * crsh_trace_secondary_host they are host pointers (dir must be NULL). */
typedef struct {
  int32_t width, height;
  const float* pos;
  const float* nrm;
  const int32_t* mat;
  const float* materials;
  int32_t n_mat;
  float eye[3];
  const float* dir;
} crsh_primary_hits;

/* Hierarchy and run options.
 *   levels      Lv, number of RSH levels built and traversed, 1..8;
 *               the paper's "hierarchy depth of 2" is Lv = 2
 *   leaf_size   B0, rays per bottom-level node, power of 2 in [2, 64]
 *   branching   B, children per upper node ("node subdivision"),
 *               power of 2 in [2, 32]; B0*B^(Lv-1) <= 2^22
 *   flags       CRSH_F_* bits
 *   shard_rank, shard_world  hash-range sharding: this call traverses only
 *               its contiguous range of top-node groups. The
 *               range is cut on the device at equal WORK (top-level tests
 *               after the whole-mesh cull, which every rank runs over all
 *               groups), the same cut on every rank, so the ranks' ranges
 *               partition the groups and summed counters / min-merged hits
 *               equal the world-1 result; world 1 = everything. */
typedef struct {
  int32_t levels, leaf_size, branching;
  uint32_t flags;
  int32_t shard_rank, shard_world;
} crsh_opts;

/* Ray-primitive test counters of the last trace (Tables 1-4), per
 * segment s (0 = SH, 1 = RE, 2 = RR) and level k (1 = leaves .. Lv = top;
 * index 0 unused). Node-vs-mesh-sphere tests are reported separately and are
 * not part of the paper's totals. brute = rays * M. */
typedef struct {
  uint64_t rays[3], slots[3], chunks[3];
  uint64_t mesh_tests[3], mesh_hits[3];
  uint64_t tests[3][9], hits[3][9];
  uint64_t final_tests[3], final_hits[3], rays_hit[3], brute[3];
  int32_t levels;
  int32_t merge;     /* multi-GPU merge of the last trace: 0 none (one rank), 1 NCCL all-reduce MIN,
                        2 fused peer stores into the symmetric window (crsh_dist_init) */
  float stage_ms[8]; /* generate+trim, compress, sort, decompress, build,
                        mesh-cull+plan, traverse+final, output */
  uint64_t cluster_tests[3], cluster_hits[3];   /* CRSH_F_OBJTREE: node-vs-cluster-sphere tests / passes */
  /* Work K8 actually evaluated, beside the paper's counts above (which do not
   * depend on it): of the counted Eq 9 tests, skipped_tests were never
   * evaluated because a conservative bound proved them failing -- the child
   * nodes (and, with CRSH_TOP_PREFILTER=1, the top nodes) tested against a
   * sphere containing the 32 triangle spheres of the slice, with a rounding
   * margin (cull_pf in k_traverse.cuh); prefilter_tests counts those bound
   * tests. Hits and every paper count are identical with and without the
   * prefilter (CRSH_NO_PREFILTER=1 disables it; then both are 0). */
  uint64_t skipped_tests[3], prefilter_tests[3];
} crsh_stats_t;

/* Number of ray slots: P * (n_lights*[SH] + [RE] + [RR]). Slot order (the ray
 * id): SH light 0 pixels 0..P-1, SH light 1 pixels, ..., then RE pixels, then
 * RR pixels; only requested types get slots. */
int64_t crsh_num_slots(int32_t P, int32_t n_lights, uint32_t ray_types);

/* Trace one frame of secondary rays: generate + hash + trim,
 * compress, radix sort, decompress, build the Lv-level sphere-cone hierarchy,
 * cull against mesh spheres, traverse, closest-hit Moller-Trumbore tests.
 *   hits        device G-buffer (see crsh_primary_hits)
 *   lights      host [n_lights][3] float32, 0 <= n_lights <= 16 (4-bit light
 *               field of the shadow hash)
 *   ray_types   CRSH_SHADOW | CRSH_REFLECT | CRSH_REFRACT
 *   hit_tri     device [slots] int32 out: closest triangle, -1 miss, -2 no ray
 *   t           device [slots] float32 out: hit distance, +inf on miss / no ray
 *   stream      cudaStream_t (NULL = legacy default stream). The call does not
 *               synchronise: the whole frame is one CUDA graph (captured on the
 *               first call with these arguments, replayed afterwards) that runs
 *               on the scene's internal stream, ordered after the work already
 *               on `stream` and before anything enqueued on `stream` later.
 *               Data-dependent counts stay on the device (every grid is sized
 *               from upper bounds). Set CRSH_NO_GRAPH=1 to launch directly.
 * Ties in t go to the smaller triangle index. */
crsh_status crsh_trace_secondary(crsh_scene_t scene, const crsh_primary_hits* hits, const float* lights,
                                 int32_t n_lights, uint32_t ray_types, const crsh_opts* opts, int32_t* hit_tri,
                                 float* t, void* stream);

/* Sharded variant for hash-range multi-GPU runs: writes, for
 * every slot, a packed uint64 that is min-reducible across ranks:
 *   owned hit  (float_bits(t) << 32) | tri
 *   owned miss 0x7F800000FFFFFFFF
 *   otherwise  0x7FFFFFFFFFFFFFFF (empty slot, or a ray owned by another rank)
 * packed: device [slots] uint64. After an element-wise MIN across ranks
 * (e.g. an NCCL all-reduce on int64), crsh_unpack_hits gives hit_tri / t. */
crsh_status crsh_trace_secondary_packed(crsh_scene_t scene, const crsh_primary_hits* hits, const float* lights,
                                        int32_t n_lights, uint32_t ray_types, const crsh_opts* opts,
                                        uint64_t* packed, void* stream);
/* Fused multi-GPU variant ("fused variant"): the epilogue of
 * each rank stores the packed result (encoding above) of every ray it owns
 * straight into EVERY destination buffer in dst -- its own and its peers',
 * e.g. the NVLink peer pointers of a symmetric allocation -- and the empty
 * sentinel into every slot that has no ray; slots whose ray another rank owns
 * are not touched. Each slot of each destination is thus written with its
 * final value by exactly one rank (empty slots: the same value by all), so
 * once all ranks' calls have completed every destination holds the merged
 * frame with no reduction step. Ordering is the caller's: a cross-rank
 * barrier after the calls before reading, and before the next frame writes
 * into buffers a peer may still be reading.
 * dst: host array of n_dst (1..8) device pointers, each [slots] uint64,
 * writable from this scene's device. Errors: EINVAL for a bad dst. */
crsh_status crsh_trace_secondary_peer(crsh_scene_t scene, const crsh_primary_hits* hits, const float* lights,
                                      int32_t n_lights, uint32_t ray_types, const crsh_opts* opts,
                                      uint64_t* const* dst, int32_t n_dst, void* stream);
/* Dynamic scenes (§3.3.1 Bounding Volume Update,
 * P:75-77): move every mesh by an affine transform of its
 * CREATION-time vertices. xforms: host [n_meshes][12] float32, row-major
 * [A | b] (3x4); vertex' = (fma(a00, x, fma(a01, y, fma(a02, z, b0))), ...).
 * Triangle data (e1, e2, minimal spheres) is rebuilt from the moved vertices
 * with the creation pad; the mesh spheres are UPDATED, not recomputed
 * ("since we only update the center and the radius there is no need to
 * recalculate the bounding spheres"): c' = A c + b (same fma order),
 * r' = r * sigma_max(A) rounded up (conservative; rigid motions keep r);
 * the hash box becomes the moved vertices' AABB; eps_t stays. Synchronous.
 * Errors: EINVAL for a null pointer or a non-finite entry. */
crsh_status crsh_scene_transform(crsh_scene_t scene, const float* xforms);

/* Trace an arbitrary batch of rays through the same pipeline (hash of the
 * bounce-ray layout, compress, sort, decompress, hierarchy, cull, traverse,
 * closest hit): the re-entry point the paper describes for the next set of
 * rays ("output these rays onto the ray array ... and continue from the
 * ray-sorting step") and the engine of the GPU primary pass.
 *   rays     device [n][8] float32: o.xyz, tmin, d.xyz (unit), tmax; a ray
 *            with !(tmax > tmin) is an empty slot (hit -2)
 *   hit_tri, t  device [n] outputs as crsh_trace_secondary
 * Counters go to segment 1 (the bounce-ray segment) of crsh_stats. */
crsh_status crsh_trace_rays(crsh_scene_t scene, const float* rays, int64_t n, const crsh_opts* opts, int32_t* hit_tri,
                            float* t, void* stream);

/* Pinhole camera of the GPU primary pass: orthonormal basis (right, up, fwd),
 * tan_half_vfov = tan(vertical field of view / 2). Pixel (i, j), j = 0 at the
 * top, p = j*width + i, ray through the pixel centre:
 *   u = ((2i+1)/W - 1) * tan_half_vfov * (W/H),  v = (1 - (2j+1)/H) * tan_half_vfov,
 *   d = norm(fma(u, right, fma(v, up, fwd))),  o = eye, tmin = 0, tmax = +inf. */
typedef struct {
  float eye[3], right[3], up[3], fwd[3];
  float tan_half_vfov;
} crsh_camera;

/* GPU primary pass (the G-buffer the paper rasterises,
 * P:67-71, produced in the library instead): camera rays traced with
 * crsh_trace_rays; per pixel pos = fma(t, d, o), nrm = norm(e1 x e2) of the
 * hit triangle turned toward the camera, mat = tri_mat[hit]; a miss gives
 * pos = nrm = 0, mat = -1. The outputs are a crsh_primary_hits-compatible
 * G-buffer (device SoA [3][P] pos / nrm, [P] mat) plus the primary hit_tri / t
 * (device [P]). tri_mat: device [M] int32. One rank. */
crsh_status crsh_primary_gbuffer(crsh_scene_t scene, const crsh_camera* cam, int32_t width, int32_t height,
                                 const int32_t* tri_mat, const crsh_opts* opts, float* pos, float* nrm, int32_t* mat,
                                 int32_t* hit_tri, float* t, void* stream);

/* Multi-bounce Whitted rendering on top of the secondary pass (SURVEY §8(f)
 * NEXT-2; "accumulate shading ... output another set of secondary
 * rays onto the ray array that we used initially and continue"; [Whi80]).
 * Bounce d traces a vertex set V_d (V_0 = gbuf) with crsh_trace_secondary's
 * pipeline: shadow rays to every light give the direct term, and while
 * d < depth the reflection / refraction rays' closest hits become V_{d+1}
 * (hit point o + t d, winding normal of the hit triangle, its material,
 * incident direction d -- the `dir` field of the next bounce's buffer). The
 * radiance is then assembled from the deepest bounce up:
 *   L(v) = kd sum_l vis_l max(0, n.l_hat) / n_lights
 *          + refl L(reflection child) + trans L(refraction child),
 *   kd = max(0, 1 - refl - trans), n turned toward the incoming ray,
 *   white lights, background 0 (readings W1-W4).
 *   gbuf      device G-buffer of the pixels (bounce 0), as crsh_trace_secondary
 *   tri_mat   device [M] int32 material index of every triangle
 *   depth     reflection/refraction bounces, 0..8 (0 = direct light only)
 *   opts      hierarchy options and flags (one rank; no CRSH_F_BRUTE)
 *   image     device [P] float32 out: radiance per pixel (0 where mat < 0)
 *   stats     optional host out: per-bounce vertices, rays, tests
 * Synchronises `stream` once per bounce (the next vertex count). */
#define CRSH_MAX_BOUNCES 8
typedef struct {
  int32_t bounces, reserved;
  int64_t vertices[CRSH_MAX_BOUNCES + 1];     /* vertices of bounce d */
  int64_t rays[CRSH_MAX_BOUNCES + 1];         /* non-empty rays traced at bounce d */
  uint64_t tests[CRSH_MAX_BOUNCES + 1];       /* ray-node tests (all levels) at bounce d */
  uint64_t final_tests[CRSH_MAX_BOUNCES + 1]; /* Moller-Trumbore tests at bounce d */
} crsh_whitted_stats_t;
crsh_status crsh_render_whitted(crsh_scene_t scene, const crsh_primary_hits* gbuf, const float* lights,
                                int32_t n_lights, const int32_t* tri_mat, int32_t depth, const crsh_opts* opts,
                                float* image, crsh_whitted_stats_t* stats, void* stream);

/* packed: device [slots]; hit_tri, t: device [slots] outputs. */
crsh_status crsh_unpack_hits(crsh_scene_t scene, const uint64_t* packed, int64_t slots, int32_t* hit_tri, float* t,
                             void* stream);

/* End-to-end variant with HOST buffers: hits->pos/nrm/mat/materials and the
 * outputs hit_tri/t are host pointers. The call copies the G-buffer to the
 * device, traces, copies the results back and synchronises `stream`. */
crsh_status crsh_trace_secondary_host(crsh_scene_t scene, const crsh_primary_hits* hits, const float* lights,
                                      int32_t n_lights, uint32_t ray_types, const crsh_opts* opts, int32_t* hit_tri,
                                      float* t, void* stream);

/* Counters of the last trace (synchronises its stream). out: host. */
crsh_status crsh_stats(crsh_scene_t scene, crsh_stats_t* out);

/* ---------------------------------------------------------------------------
 * Multi-GPU data plane (SURVEY §8(b) crsh_dist_init, §8(e); BASELINE.json
 * north_star: "Sorted rays are sharded by contiguous hash range across the GPUs
 * of one 8xB200 box. Each GPU builds and traverses its own sub-hierarchy, and
 * the per-pixel hits are gathered with NCCL over NVLink"; the paper itself is
 * single-GPU). One process per GPU; every rank holds the same scene
 * and G-buffer and makes the same calls.
 *
 * crsh_dist_unique_id: a fresh NCCL unique id (128 bytes, host) that rank 0
 * creates and every rank receives out of band (e.g. a torch.distributed
 * broadcast). Errors: EINVAL (null), ENCCL.
 *
 * crsh_dist_init: joins `scene` (on its device) to an NCCL communicator of
 * `world` ranks built from `nccl_uid` (host, 128 bytes); collective over the
 * ranks. From then on crsh_trace_secondary / crsh_trace_secondary_host on
 * this scene trace rank `rank`'s work-balanced share of the top-node groups
 * (opts.shard_rank / shard_world must be 0 / 1 or equal to rank / world) and
 * MERGE inside the call: every rank's hit_tri / t receive the whole frame and
 * crsh_stats reports the counters summed over the ranks (stats.merge says
 * which merge ran). The merge is the fused one of §8(e) -- each rank's
 * epilogue stores its owned packed results into every rank's symmetric NCCL
 * window over NVLink (LSA pointers), bracketed by device-side LSA barriers --
 * when all ranks share one load/store domain of <= 8 GPUs, else (or with the
 * environment variable CRSH_DIST_MERGE=nccl at init) ncclAllReduce(ncclMin,
 * ncclUint64) of the packed frames; counters use ncclAllReduce(ncclSum).
 * Both run inside the frame's CUDA graph on the scene's stream. The window
 * (8 bytes per slot, ncclMemAlloc) grows collectively on the first trace
 * that needs more. crsh_trace_secondary_packed / _peer / crsh_trace_rays /
 * crsh_render_whitted / crsh_primary_gbuffer are unaffected (no merge).
 * crsh_scene_destroy releases the communicator. Called once per scene.
 * Errors: EINVAL (bad rank/world, second call), ENCCL (communicator or window
 * setup), ECUDA. Asynchronous NCCL errors surface as ENCCL from crsh_stats
 * (ncclCommGetAsyncError). */
crsh_status crsh_dist_unique_id(void* uid);
crsh_status crsh_dist_init(crsh_scene_t scene, const void* nccl_uid, int32_t rank, int32_t world);

/* Number of CUDA kernels the library launched during the last trace. */
int64_t crsh_launch_count(crsh_scene_t scene);

/* Thread-local description of the last non-OK status. */
const char* crsh_last_error(void);

/* Debug taps: copy an intermediate array of the last trace to host memory
 * (synchronises). segment in {0,1,2}; level used by CRSH_TAP_NODES only.
 *   host_dst host buffer of cap_bytes; *n_out receives the element count.
 * Returns CRSH_EIO if cap_bytes is too small (n_out still set). */
enum {
  CRSH_TAP_KEYS = 1,         /* u32 compacted keys of the segment, slot order (Fig 4) */
  CRSH_TAP_VALS = 2,         /* u32 compacted slot ids */
  CRSH_TAP_CHUNK_KEYS = 3,   /* u32 chunk keys (Fig 5) */
  CRSH_TAP_CHUNK_BASE = 4,   /* u32 chunk bases, relative to the segment */
  CRSH_TAP_SORTED_KEYS = 5,  /* u32 sorted keys (Fig 6) */
  CRSH_TAP_SORTED_SLOTS = 6, /* u32 sorted slot ids (the permutation) */
  CRSH_TAP_NODES = 7,        /* float[8] nodes (c.xyz, r, a.xyz, alpha) at `level` */
  CRSH_TAP_SORTED_RAYS = 8,  /* float[8] rays (o.xyz, tmin, d.xyz, tmax) in sorted order */
  CRSH_TAP_TRI_SPHERES = 9,  /* float[4] padded triangle spheres (scene) */
  CRSH_TAP_MESH_SPHERES = 10,/* float[4] padded mesh spheres (scene) */
  CRSH_TAP_SCENE_CONSTS = 11,/* float[8]: aabb min.xyz, max.xyz, pad, eps_t */
  CRSH_TAP_GROUP_RANGE = 12, /* u32[3]: this rank's groups [g_lo, g_hi) and G (frame-wide) */
  CRSH_TAP_GROUP_WORK = 13,  /* u64[G]: per-group work the cut balanced (shard_world > 1 only) */
  CRSH_TAP_CLUSTER_SPHERES = 14, /* float[4] padded object-tree cluster spheres, mesh by mesh (scene) */
  CRSH_TAP_CLUSTER_ORDER = 15    /* i32[M] triangle ids in cluster order (Morton within each mesh; scene) */
};
crsh_status crsh_debug_tap(crsh_scene_t scene, int32_t tap, int32_t segment, int32_t level, void* host_dst,
                           size_t cap_bytes, size_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* CRSH_H_ */
