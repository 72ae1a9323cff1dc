/* pgg.h — C ABI of the B200 screen-space path-guiding pass (libpgg.so).
 *
 * Drop-in boundary for the reference package `pgtrace` (arXiv 2112.09728
 * desk-scale implementation; paths relative to /root/reference/pkg/src/pgtrace).
 * The reference exposes Python functions on NumPy arrays and has no FFI of
 * its own; each entry point below replaces one of them (see INTEGRATION.md
 * for the ctypes binding that the Python shim uses):
 *
 *   pgg_guiding_pass ..... guide_buffers.reproject      guide_buffers.py:78-137
 *                          guide_buffers.training_pass  guide_buffers.py:262-283
 *                          ptrace._sample_first_bounce  ptrace.py:161-220 (+ the
 *                          per-pixel lane setup of ptrace.py:449-475)
 *                          any subset of the three, fused into one kernel
 *   pgg_train_records .... guide_buffers.gather_training_batch  guide_buffers.py:234-259
 *   pgg_sample_lanes ..... ptrace._sample_first_bounce  ptrace.py:161-220 and
 *                          mixture.sample_mixture       mixture.py:193-259 on
 *                          caller-owned PCG32 states (in/out)
 *   pgg_lobe ............. mixture.lobe_from_stats      mixture.py:129-155
 *   pgg_mixture_lanes .... mixture.gaussian_pdf_square / mixture_pdf / box_muller /
 *                          e_step_responsibility / neighbor_count  mixture.py:158-190, 262-273, 324-328
 *   pgg_sample_gauss ..... the Gaussian branch of mixture.sample_mixture (mixture.py:208-235)
 *                          for callers with their own BRDF callbacks
 *   pgg_trunc_mass ....... mixture.truncation_mass      mixture.py:84-126 (its rule, float64)
 *   pgg_m_step ........... mixture.m_step_update        mixture.py:276-321
 *   pgg_make_streams ..... rng.make_streams             rng.py:25-39
 *   pgg_next_u32 ......... rng.next_u32                 rng.py:42-50
 *   pgg_frame_key ........ the lane-independent prefix of rng.make_streams
 *   pgg_pack_* / pgg_gamma_* layout conversion at the API edge (pgg_pack_gbuffer_mat: from
 *                          material ids + the scene's table)
 *
 * The render pass that feeds it:
 *   pgg_gbuffer_pass ..... ptrace.gbuffer_pass          ptrace.py:97-129
 *                          ptrace.motion_vectors        ptrace.py:132-150
 *   pgg_render_pass ...... ptrace.render_frame / _render_chunk / _trace_lanes
 *                          ptrace.py:223-355, 382-586 (scene.intersect,
 *                          occluded, sample_emitter, brdf_* scene.py:158-414)
 *   pgg_image_error ...... metrics.mse / rel_mse         metrics.py:24-38
 *
 * Conventions: every pointer is a DEVICE pointer owned by the caller unless
 * stated otherwise; calls are asynchronous on `stream` (a cudaStream_t, NULL =
 * legacy default stream), keep no global mutable state, never throw, and
 * return 0 or a pgg_status code.  Safe to call concurrently from several host
 * threads on different streams.
 *
 * Device layouts (P = pixels of a row band, row-major, width = frame width):
 *   Gamma      two float4 planes  g0 = (mu_x, mu_y, m2_xx, m2_yy)
 *                                 g1 = (m2_xy, w_sum, pi, k)
 *   G-buffer   flags u8 (bit0 valid, bit1 has_history, bit2 glossy, bit3 front)
 *              nd float4 (normal.xyz, depth)      pr float4 (pos.xyz, roughness)
 *              va float4 (view.xyz, albedo.r)     am float4 (albedo.g, albedo.b, motion.xy)
 *              mat int32 plane (material id, -1 on a miss; render pass only)
 *   VPLs (Pi)  y float4 (pos.xyz, usable = valid && strategy==BRDF ? 1 : 0)
 *              L float4 (radiance.rgb, valid | strategy << 1)
 *   samples    per lane (pixel*spp + s): dir float4 (wi.xyz world, pdf),
 *              tag u8 (bit0 strategy GAUSSIAN, bit1 valid, bits 2..7 the
 *              number of PCG32 draws the depth-0 sampler consumed after the
 *              NEE draws, so the render pass continues the lane's stream)
 */
#ifndef PGG_H_
#define PGG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PGG_ABI_VERSION 2

enum pgg_status {
  PGG_OK = 0,
  PGG_ERR_ARGUMENT = 1,    /* bad dimensions / null pointer where required */
  PGG_ERR_CUDA = 2,        /* kernel launch failed (see pgg_last_cuda_error) */
  PGG_ERR_UNSUPPORTED = 3  /* device is not sm_100 */
};

/* A row band [row0, row0 + rows) of a G-buffer in the packed layout. */
typedef struct pgg_gbuffer {
  const uint8_t* flags;
  const float* nd;
  const float* pr;
  const float* va;
  const float* am;
  int32_t row0;
  int32_t rows;
} pgg_gbuffer;

/* Read-only Gamma planes holding rows [row0, row0 + rows). */
typedef struct pgg_gamma_in {
  const float* g0;
  const float* g1;
  int32_t row0;
  int32_t rows;
} pgg_gamma_in;

/* Gamma planes written for the call's own band (cfg.row0, cfg.rows). */
typedef struct pgg_gamma_out {
  float* g0;
  float* g1;
} pgg_gamma_out;

/* VPL planes holding rows [row0, row0 + rows) (own band + EM halo). */
typedef struct pgg_vpl {
  const float* y;
  const float* L;
  int32_t row0;
  int32_t rows;
} pgg_vpl;

/* Depth-0 samples of the call's own band, lane = pixel * spp + s. */
typedef struct pgg_samples {
  float* dir;  /* float4 per lane */
  uint8_t* tag;
} pgg_samples;

typedef struct pgg_config {
  int32_t width, height;       /* full frame */
  int32_t row0, rows;          /* band produced by this call */
  int32_t spp;                 /* lanes per pixel (ptrace.py:460-475) */
  int32_t nee_draws;           /* draws consumed before the depth-0 scatter (3 with NEE + emitters) */
  int32_t k_max;               /* mixture.KMAX_DEFAULT = 64 */
  int32_t rotate_mean;         /* ReprojectionPolicy.rotate_mean */
  double radius;               /* training neighbour radius (guide_buffers.py:19) */
  double depth_rel_tol;        /* ReprojectionPolicy.depth_rel_tol */
  double normal_dot_min;       /* ReprojectionPolicy.normal_dot_min */
  double rough_min_guide;      /* PathConfig.roughness_min_guide */
  double prev_cam[3];          /* previous frame camera origin (GBuffer.cam_origin) */
  uint64_t key_sample;         /* pgg_frame_key(seed, frame, 0) */
  uint64_t key_train;          /* pgg_frame_key(seed, frame, 1) */
} pgg_config;

/* Fused guiding pass over the band cfg.row0..: for every pixel
 *   Gamma  = prev ? reproject(gamma_prev, prev, cur) : gamma_prev
 *   (gamma_reproj) <- Gamma                       if gamma_reproj != NULL
 *   samples <- depth-0 guided/BRDF sampling       if samples != NULL
 *   gamma_out <- one EM epoch over the VPL disk   if vpl != NULL (gamma_out required)
 * gamma_prev / prev must hold every row a motion vector of the band reaches
 * (reprojection halo); vpl must hold the band +- rint(radius) rows clipped to
 * the frame (EM halo).  References outside the supplied rows are counted in
 * *halo_misses (device int32, may be NULL) and treated as out of frame.
 * With prev, gamma_out / gamma_reproj must not share planes with gamma_prev
 * (reprojection reads other pixels' Gamma): PGG_ERR_ARGUMENT; without prev
 * the update may be in place. */
int pgg_guiding_pass(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gbuffer* prev,
                     const pgg_gamma_in* gamma_prev, const pgg_vpl* vpl, const pgg_gamma_out* gamma_reproj,
                     const pgg_gamma_out* gamma_out, const pgg_samples* samples, int32_t* halo_misses,
                     void* stream);

/* One stage of the pass each (= pgg_guiding_pass with that stage only):
 *   pgg_reproject ............ guide_buffers.reproject (guide_buffers.py:78-137)
 *   pgg_train ................ guide_buffers.training_pass (guide_buffers.py:262-283)
 *                              on an already reprojected Gamma
 *   pgg_sample_first_bounce .. the render's depth-0 sampling (ptrace.py:161-220,
 *                              449-475) for every pixel x spp lane */
int pgg_reproject(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gbuffer* prev,
                  const pgg_gamma_in* gamma_prev, const pgg_gamma_out* gamma_out, int32_t* halo_misses, void* stream);
int pgg_train(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gamma_in* gamma, const pgg_vpl* vpl,
              const pgg_gamma_out* gamma_out, int32_t* halo_misses, void* stream);
int pgg_sample_first_bounce(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gamma_in* gamma,
                            const pgg_samples* samples, void* stream);

/* Training records of n pixels (pix_xy: n x int32 (x, y)) for
 * guide_buffers.gather_training_batch (guide_buffers.py:234-259): the EM
 * candidate draws come from the caller's per-pixel PCG32 states (states is
 * W*H, indexed by pixel, not advanced here).  records: n x 20 x float4
 * (sq_x, sq_y, weight, valid) in slot order. */
int pgg_train_records(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gamma_in* gamma, const pgg_vpl* vpl,
                      int64_t n, const int32_t* pix_xy, const uint64_t* states, float* records, void* stream);

/* Per-lane depth-0 sampling on caller-owned PCG32 states (in/out).
 * Inputs per lane: normal/view float4 (w unused), roughness, glossy (u8),
 * guided (u8), pi, lobe float x6 (mu_x, mu_y, l11, l21, l22, trunc_z).
 * world != 0: lanes are world-space (ptrace._sample_first_bounce: plain lanes
 * sample the BRDF about `normal`, guided lanes the mixture in its tangent
 * frame); world == 0: mixture.sample_mixture in the local frame (normal
 * ignored, `view` holds wo in local coordinates, every lane guided).
 * Outputs: dir float4 (direction, pdf), tag u8 (bit0 GAUSSIAN, bit1 valid). */
int pgg_sample_lanes(int64_t n, int32_t world, const float* normal, const float* view, const float* rough,
                     const uint8_t* glossy, const uint8_t* guided, const float* pi, const float* lobe6,
                     uint64_t* states, float* dir, uint8_t* tag, void* stream);

/* lobe_from_stats on n rows of float64 stats (n x 8): mu (n x 2),
 * cov (n x 4 row-major 2x2), chol (n x 4), trunc_z (n), reset flag (n, may be NULL). */
int pgg_lobe(int64_t n, const double* stats, double* mu, double* cov, double* chol, double* trunc_z,
             uint8_t* reset, void* stream);

/* truncation_mass(mu (n x 2), cov (n x 4)) -> z (n). */
int pgg_trunc_mass(int64_t n, const double* mu, const double* cov, double* z, void* stream);

/* m_step_update(stats (n x 8), sq (n x c x 2), weight, resp (n x c),
 * valid (n x c u8 or NULL), k_max) -> out (n x 8), all float64. */
int pgg_m_step(int64_t n, int32_t c, const double* stats, const double* sq, const double* weight,
               const double* resp, const uint8_t* valid, int32_t k_max, double* out, void* stream);

/* Host function: the (seed, frame, stream_id) prefix of rng.make_streams. */
uint64_t pgg_frame_key(uint64_t seed, uint64_t frame, uint64_t stream_id);

/* make_streams: states[i] = PCG32 lane state of lanes[i] under `key`. */
int pgg_make_streams(uint64_t key, int64_t n, const uint64_t* lanes, uint64_t* states, void* stream);

/* next_u32: advance every state once (in place), outputs u32. */
int pgg_next_u32(int64_t n, uint64_t* states, uint32_t* out, void* stream);

/* Pack reference-layout G-buffer fields (float32/uint8/int32 device arrays,
 * P pixels) into the planes above.  motion/has_history may be NULL. */
int pgg_pack_gbuffer(int64_t p, const uint8_t* valid, const float* pos, const float* normal,
                     const float* depth, const int32_t* kind, const float* albedo, const float* rough,
                     const float* view, const float* motion, const uint8_t* has_history, uint8_t* flags,
                     float* nd, float* pr, float* va, float* am, void* stream);

/* The same planes from the G-buffer's material ids (int32, -1 = miss) and the
 * scene's material table (n_mat kinds, albedo rgb, roughness; the lookups of
 * ptrace.gbuffer_pass, ptrace.py:97-129) instead of per-pixel kind / albedo
 * / roughness: 16 B/px less to upload.  Bitwise the same planes. */
int pgg_pack_gbuffer_mat(int64_t p, const uint8_t* valid, const float* pos, const float* normal,
                         const float* depth, const int32_t* mat, int32_t n_mat, const int32_t* mat_kind,
                         const float* mat_albedo, const float* mat_rough, const float* view, const float* motion,
                         const uint8_t* has_history, uint8_t* flags, float* nd, float* pr, float* va, float* am,
                         void* stream);

/* Pack VplBuffer fields (valid u8, y f32 x3, radiance f32 x3, strategy u8). */
int pgg_pack_vpl(int64_t p, const uint8_t* valid, const float* y, const float* radiance,
                 const uint8_t* strategy, float* vy, float* vl, void* stream);

/* Gamma (P x 8 float32, the reference's (H,W,8) layout) <-> planes. */
int pgg_gamma_split(int64_t p, const float* aos, float* g0, float* g1, void* stream);
int pgg_gamma_join(int64_t p, const float* g0, const float* g1, float* aos, void* stream);
/* Fresh Gamma (mixture.init_stats) into the planes. */
int pgg_gamma_init(int64_t p, float* g0, float* g1, void* stream);

/* ---------------------------------------------------------------------
 * Render pass (the producer of the G-buffer and the VPLs). */

/* Scene table (device, float64; built by paper_2112_09728_b200/scene.py
 * Scene.pack): n_mat x 12 (kind, albedo rgb, roughness, emission rgb, albedo/pi rgb, pad),
 * n_sph x 8 (center xyz, radius, material, pad), n_quad x 16 (corner, edge_u,
 * edge_v, unit normal, area, material, |edge_u|^2, |edge_v|^2), n_emit
 * emitter quad indices.  At most 6144 doubles (staged in shared memory). */
typedef struct pgg_scene {
  const double* table;
  int32_t n_mat, n_sph, n_quad, n_emit;
  double background[3];
} pgg_scene;

/* Pinhole camera of one frame (scene.camera_at, scene.py:94-117). */
typedef struct pgg_camera {
  double origin[3], forward[3], right[3], up[3];
  double tan_half_fov;
} pgg_camera;

/* Primary hit per pixel centre of rows [row0, row0 + rows) into the packed
 * G-buffer planes (+ material ids); prev_cam != NULL also writes the motion
 * vectors and has_history of motion_vectors(prev_cam, cam, gbuf). */
int pgg_gbuffer_pass(const pgg_scene* scene, const pgg_camera* cam, const pgg_camera* prev_cam, int32_t width,
                     int32_t height, int32_t row0, int32_t rows, uint8_t* flags, float* nd, float* pr, float* va,
                     float* am, int32_t* mat, void* stream);

typedef struct pgg_render_config {
  int32_t width, height;       /* full frame */
  int32_t row0, rows;          /* band rendered by this call */
  int32_t spp, max_depth, nee; /* PathConfig (ptrace.py:27-40) */
  int32_t reserved;
  uint64_t key;                /* pgg_frame_key(seed, frame, 0) */
} pgg_render_config;

typedef struct pgg_render_out {
  float* image;                   /* rows x W x 3, mean over spp */
  float* vpl_y;                   /* VPL planes of the band (layout above) */
  float* vpl_L;
  double* lum_moments;            /* rows x W x 2 (sum, sum of squares of luminance) or NULL */
  unsigned long long* counters;   /* [scatter segments, non-finite samples] accumulated, or NULL */
  uint64_t* states;               /* NULL: lane streams from cfg.key (ptrace.py:474-475); else the
                                     caller's PCG32 state per lane (band-local lane index), advanced in
                                     place (ptrace.trace_pixel, ptrace.py:358-376) */
} pgg_render_out;

/* Trace spp lanes per pixel from the G-buffer (gb + mat planes holding the
 * band): NEE at every vertex, BRDF scatter, VPL of the last lane.  depth0 !=
 * NULL (pg mode): the depth-0 scatter of every lane comes from the guiding
 * pass's samples of the same band and frame (pgg_guiding_pass with
 * nee_draws = nee && n_emit ? 3 : 0). */
int pgg_render_pass(const pgg_render_config* cfg, const pgg_scene* scene, const pgg_gbuffer* gb, const int32_t* mat,
                    const pgg_samples* depth0, const pgg_render_out* out, void* stream);

/* Scene routines of pg/scene.py as batch lane operations (float64, n lanes,
 * xyz triples interleaved):
 *   pgg_intersect ....... scene.intersect / occluded (scene.py:158-241):
 *                         any_hit != 0 writes only `hit` (occluded)
 *   pgg_sample_emitter .. scene.sample_emitter (scene.py:386-414), three
 *                         draws per lane from `states` (in/out)
 *   pgg_brdf ............ op 0 brdf_eval -> f (rgb), 1 brdf_pdf -> pdf,
 *                         2 brdf_sample -> wi, pdf, valid (two draws)
 *                         (scene.py:258-380)
 *   pgg_primary_rays .... scene.primary_ray_dirs (scene.py:125-135)
 *   pgg_project ......... scene.project_to_pixels (scene.py:138-151)
 *   pgg_motion_vectors .. ptrace.motion_vectors (ptrace.py:132-150) */
int pgg_intersect(const pgg_scene* scene, int64_t n, const double* origins, const double* dirs, const double* t_min,
                  const double* t_max, int32_t any_hit, uint8_t* hit, double* t, double* pos, double* normal,
                  int32_t* mat, uint8_t* front, void* stream);
int pgg_sample_emitter(const pgg_scene* scene, int64_t n, const double* points, uint64_t* states, double* dir,
                       double* dist, double* emitted, double* pdf, void* stream);
int pgg_brdf(int32_t op, int64_t n, const int32_t* kind, const double* albedo, const double* rough, double* wi,
             const double* wo, const double* normal, uint64_t* states, double* f, double* pdf, uint8_t* valid,
             void* stream);
int pgg_primary_rays(const pgg_camera* cam, int32_t width, int32_t height, int64_t n, const double* px,
                     const double* py, double* dirs, void* stream);
int pgg_project(const pgg_camera* cam, int32_t width, int32_t height, int64_t n, const double* points, double* px,
                double* py, uint8_t* in_front, void* stream);
/* ptrace.motion_vectors (ptrace.py:132-150) for a caller G-buffer: pos is
 * height x width x 3 hit points, valid its hit mask; writes motion (height x
 * width x 2, zero where no history) and has_history. */
int pgg_motion_vectors(const pgg_camera* prev_cam, int32_t width, int32_t height, const double* pos,
                       const uint8_t* valid, double* motion, uint8_t* has_history, void* stream);

/* sgmap.py:21-115 as float64 lane operations: op 0 square_to_disk (n x 2 ->
 * n x 2), 1 disk_to_square (2 -> 2), 2 square_to_hemisphere (2 -> 3),
 * 3 hemisphere_to_square (3 -> 2; the caller rejects z < -1e-9 first),
 * 4 build_tangent_frame (n x 3 -> n x (t, b) 6), 5 to_world and 6 to_local
 * (n x (t, b, n, v) 12 -> n x 3). */
int pgg_sgmap(int32_t op, int64_t n, const double* in, double* out, void* stream);

/* Image error (metrics.mse / metrics.rel_mse, metrics.py:24-38) of n
 * float32 elements: mean of (a - ref)^2, or of (a - ref)^2 / (ref^2 + 0.01)
 * when relative != 0, accumulated in float64 with a fixed reduction order
 * (deterministic).  scratch: PGG_IMAGE_ERROR_SCRATCH doubles of device
 * memory; out: one double (device). */
#define PGG_IMAGE_ERROR_SCRATCH 1184
int pgg_image_error(int64_t n, const float* a, const float* ref, int32_t relative, double* scratch, double* out,
                    void* stream);

const char* pgg_status_string(int status);
const char* pgg_last_cuda_error(void);
int pgg_abi_version(void);

/* mixture.py's remaining lane functions in float64 (device arrays, n lanes):
 *   op 0 gaussian_pdf_square  a = mu (n,2), b = chol (n,2,2), c = trunc_z (n), d = p (n,2)  mixture.py:158-169
 *   op 1 box_muller           a = u1, b = u2 -> out0 = z0, out1 = z1                       mixture.py:185-190
 *   op 2 e_step_responsibility a = pi, b = gauss pdf, c = brdf pdf                          mixture.py:262-273
 *   op 3 neighbor_count       a = k, k_max -> out0 = N (as double)                          mixture.py:324-328
 *   op 4 mixture_pdf          a = pi, b = per lane (mu_x, mu_y, l11, 0, l21, l22, trunc_z) (n,7),
 *                             c = square point of the direction (n,2), d = brdf pdf         mixture.py:172-182
 * (e is unused; out1 only for op 1) */
int pgg_mixture_lanes(int32_t op, int64_t n, const double* a, const double* b, const double* c, const double* d,
                      const double* e, double* out0, double* out1, int32_t k_max, void* stream);

/* Gaussian branch of mixture.sample_mixture (mixture.py:208-235) in float64
 * for callers that keep the reference's Python BRDF callbacks: per lane a
 * zeta draw (< pi) and up to 16 Box-Muller tries on `states` (advanced in
 * place); writes the accepted square point (n,2) and accepted[i] in {0,1}.
 * The BRDF fallback and pdf are the caller's (pg/ptrace.py:201-208). */
int pgg_sample_gauss(int64_t n, const double* pi, const double* mu, const double* chol, uint64_t* states, double* sq,
                     uint8_t* accepted, void* stream);

/* Diagnostics (test-only; not on the product path).  Each runs the device
 * functions of pgg_guiding_pass over a whole frame / batch and records the
 * discrete decisions the reference makes, so tests can compare them with the
 * reference's float64 arithmetic at frame scale:
 *   pgg_debug_em_offsets  the 19 candidate offsets (dx, dy) of every pixel,
 *       int8 [width*height][19][2], as training_pass draws them
 *       (guide_buffers.py:140-161: rint of 10 sqrt(u1) cos/sin(2 pi u2));
 *       *rechecks += number of offsets re-decided in float64 (guard band)
 *   pgg_debug_bm_accept   Box-Muller proposal acceptance p in [0,1]^2
 *       (mixture.py:216-230) for n proposals, lobe i / per_lobe from float32
 *       Gamma stats[8]; draws (u1, u2) as u32 pairs; out bit0 accepted, bit1
 *       re-decided in float64; proposals (nullable) the float32 p = mu + L z
 *   pgg_debug_reproject   reprojection decision per pixel of cfg's band
 *       (guide_buffers.py:78-137): bit0 accepted, bit1 gates re-decided in
 *       float64, bit2 rejected by the mean rotation (z < 0), bit3 rejected by
 *       the depth / normal gates */
/* Checked builds only (libpgg_checked.so, -DPGG_CHECKS=1: in-kernel index
 * bounds asserts on every tile / plane access of pgg_guiding_pass): copies
 * {failures, first site, operand a, operand b, blockIdx.x, blockIdx.y} to
 * host memory (synchronous) and optionally resets them.  Other builds return
 * PGG_ERR_UNSUPPORTED. */
int pgg_debug_checks(int32_t* host_out6, int32_t reset);
int pgg_debug_em_offsets(const pgg_config* cfg, int8_t* offsets, int32_t* rechecks, void* stream);
int pgg_debug_bm_accept(int64_t n, int32_t per_lobe, const float* stats, const uint32_t* draws, uint8_t* out,
                        float* proposals, int32_t* rechecks, void* stream);
/*   pgg_debug_trunc_bvn   the pass's float32 truncation mass (Genz BVN; the
 *       reference rule for |r| >= 0.999) of n lobes (mu n x 2, cov n x 2 x 2,
 *       float64) -- pgg_trunc_mass returns the reference's float64 rule */
int pgg_debug_trunc_bvn(int64_t n, const double* mu, const double* cov, double* z, void* stream);
/*   pgg_debug_brdf_draw   the sampler's local-frame BRDF draw (Lambert cosine
 *       or GGX VNDF, scene.py:311-351, with the float64 re-evaluation of rim
 *       samples) for n lanes: glossy u8, roughness, wo float4 (local), draws
 *       (u1, u2) as u32 pairs; out float4 (wi.xyz, valid); *rechecks += the
 *       draws re-evaluated in float64 */
int pgg_debug_brdf_draw(int64_t n, const uint8_t* glossy, const float* rough, const float* wo, const uint32_t* draws,
                        float* out, int32_t* rechecks, void* stream);
int pgg_debug_reproject(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gbuffer* prev,
                        const pgg_gamma_in* gamma_prev, uint8_t* decisions, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PGG_H_ */
