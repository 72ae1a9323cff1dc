// pgg_render.cu — the render pass that produces the guiding pass's inputs
// (SURVEY.md 8f rank 1): primary-ray G-buffer + camera motion vectors
// (pg/ptrace.py:97-150) and the path-traced lanes with next-event estimation
// that write the image and the per-pixel VPLs (pg/ptrace.py:223-355,
// 382-586; scene routines pg/scene.py:158-241, 247-414).
//
// Precision: the reference traces in float64 and its hit / visibility
// decisions are discontinuous, so this translation unit computes geometry,
// BRDFs and throughput in float64 with the reference's operation order and
// is compiled with -fmad=false (no contraction): primary rays, NEE and
// scatter decisions match the reference's bit for bit except where NumPy's
// BLAS dot products or libm transcendentals round differently (1 ulp).
// B200 runs FP64 at half the FP32 rate; the scene is a few dozen
// primitives held in shared memory, so a lane is latency- not bandwidth-
// bound (render pass).
//
// Lanes: one thread per pixel walks its spp lanes in order (lane key
// pixel * spp + s, pg/ptrace.py:474), so the per-pixel sums accumulate in the
// reference's order.  In pg mode the depth-0 scatter comes from the guiding
// pass's samples (pgg_guiding_pass, samples != NULL) and the lane's PCG32
// stream continues after the draws that sampler consumed (tag bits 2..7).

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "pgg.h"

namespace pgg_rt {
extern thread_local char g_cuda_err[256];
int check_launch();
int device_check();
}  // namespace pgg_rt

namespace {

// PCG32 lane streams (pg/rng.py:10-55; same chain as pgg_math.cuh)
constexpr uint64_t PCG_MUL = 6364136223846793005ULL;
constexpr uint64_t PCG_INC = 1442695040888963407ULL;
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t pcg_lane(uint64_t key, uint64_t lane) {
  return mix64(key ^ mix64(lane)) * PCG_MUL + PCG_INC;
}
__device__ __forceinline__ uint32_t pcg_next(uint64_t& s) {
  const uint64_t old = s;
  s = old * PCG_MUL + PCG_INC;
  const uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
  const uint32_t rot = (uint32_t)(old >> 59);
  return (xs >> rot) | (xs << ((32u - rot) & 31u));
}
__device__ __forceinline__ double u01d(uint32_t u) { return (double)u * 2.3283064365386963e-10; }

constexpr double PI_D = 3.141592653589793;
constexpr double RAY_EPS = 1e-4;  // pg/scene.py:24
constexpr int MAT_STRIDE = 12, SPH_STRIDE = 8, QUAD_STRIDE = 16;  // scene.py pack()
constexpr int MAX_TABLE = 6144;   // doubles staged in shared memory (48 KB)

struct D3 {
  double x, y, z;
};
__device__ __forceinline__ D3 d3(double x, double y, double z) { return {x, y, z}; }
__device__ __forceinline__ D3 operator+(D3 a, D3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ D3 operator-(D3 a, D3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ D3 operator*(D3 a, D3 b) { return {a.x * b.x, a.y * b.y, a.z * b.z}; }
__device__ __forceinline__ D3 operator*(D3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ D3 operator*(double s, D3 a) { return {s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ D3 operator/(D3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
__device__ __forceinline__ D3 neg(D3 a) { return {-a.x, -a.y, -a.z}; }
// np.sum(a * b, axis=-1): sequential over the three products
__device__ __forceinline__ double dot(D3 a, D3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
__device__ __forceinline__ double norm(D3 a) { return sqrt(dot(a, a)); }
// pg/scene.py:31-34
__device__ __forceinline__ D3 normalize(D3 a) { return a / fmax(norm(a), 1e-30); }
__device__ __forceinline__ D3 cross(D3 a, D3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
__device__ __forceinline__ bool any_pos(D3 a) { return a.x > 0.0 || a.y > 0.0 || a.z > 0.0; }
__device__ __forceinline__ bool finite3(D3 a) { return isfinite(a.x) && isfinite(a.y) && isfinite(a.z); }
__device__ __forceinline__ D3 ld3(const double* p) { return {p[0], p[1], p[2]}; }

// Scene table staged in shared memory (layout: paper_2112_09728_b200/scene.py)
struct SceneS {
  const double* mats;
  const double* sph;
  const double* quad;
  const double* emit;
  int nm, ns, nq, ne;
  D3 bg;
  __device__ int kind(int m) const { return (int)mats[m * MAT_STRIDE]; }
  __device__ D3 albedo(int m) const { return ld3(mats + m * MAT_STRIDE + 1); }
  __device__ double rough(int m) const { return mats[m * MAT_STRIDE + 4]; }
  __device__ D3 emission(int m) const { return ld3(mats + m * MAT_STRIDE + 5); }
  __device__ D3 albedo_pi(int m) const { return ld3(mats + m * MAT_STRIDE + 8); }  // albedo / pi (host-divided)
};

__device__ SceneS stage_scene(const pgg_scene& sc, double* smem) {
  const int n = sc.n_mat * MAT_STRIDE + sc.n_sph * SPH_STRIDE + sc.n_quad * QUAD_STRIDE + sc.n_emit;
  const int tid = threadIdx.x + blockDim.x * threadIdx.y;
  for (int i = tid; i < n; i += blockDim.x * blockDim.y) smem[i] = sc.table[i];
  __syncthreads();
  SceneS s;
  s.mats = smem;
  s.sph = s.mats + sc.n_mat * MAT_STRIDE;
  s.quad = s.sph + sc.n_sph * SPH_STRIDE;
  s.emit = s.quad + sc.n_quad * QUAD_STRIDE;
  s.nm = sc.n_mat;
  s.ns = sc.n_sph;
  s.nq = sc.n_quad;
  s.ne = sc.n_emit;
  s.bg = d3(sc.background[0], sc.background[1], sc.background[2]);
  return s;
}

// RN(n / e) in [0, 1] for e > 0 without the division: RN(n/e) <= 1 iff
// n <= e (n > e means n >= nextafter(e), so n/e > 1 + 2^-53 rounds above 1);
// RN(n/e) >= 0 iff n >= 0, or n < 0 underflowing to -0 (tiny n only).
__device__ __noinline__ bool tiny_negative_quotient_nonneg(double n, double e) { return n / e >= 0.0; }
__device__ __forceinline__ bool in_unit(double n, double e) {
  if (n > e) return false;
  if (n >= 0.0) return true;
  return n > -1e-280 && tiny_negative_quotient_nonneg(n, e);
}

__device__ __forceinline__ int table_doubles_d(const pgg_scene& sc) {
  return sc.n_mat * MAT_STRIDE + sc.n_sph * SPH_STRIDE + sc.n_quad * QUAD_STRIDE + sc.n_emit;
}

#ifndef PGG_QUAD_PREREJECT
#define PGG_QUAD_PREREJECT 1
#endif

struct Hit {
  bool hit, front;
  double t;
  D3 pos, nrm;
  int mat;
};

// Nearest hit, spheres then quads, strict t < best (pg/scene.py:158-235).
// any_hit: stop at the first primitive inside (t_min, t_max) (occluded()).
template <bool kAny>
__device__ Hit cast(const SceneS& S, D3 o, D3 d, double t_min, double t_max) {
  double best = INFINITY;
  int which = -1, prim = -1;
  for (int i = 0; i < S.ns; ++i) {
    const double* sp = S.sph + i * SPH_STRIDE;
    const D3 oc = o - ld3(sp);
    const double r = sp[3];
    const double b = dot(oc, d);
    const double c = dot(oc, oc) - r * r;
    const double disc = b * b - c;
    bool ok = disc > 0.0;
    const double root = sqrt(ok ? disc : 0.0);
    const double t0 = -b - root, t1 = -b + root;
    const double t = (t0 > t_min && t0 < t_max) ? t0 : t1;
    ok = ok && t > t_min && t < t_max && t < best;
    if (ok) {
      best = t;
      which = 0;
      prim = i;
      if (kAny) break;
    }
  }
  if (!kAny || which < 0) {
    for (int i = 0; i < S.nq; ++i) {
      const double* q = S.quad + i * QUAD_STRIDE;
      const D3 qn = ld3(q + 9);
      const double den = dot(d, qn);
      if (!(fabs(den) > 1e-12)) continue;
      const D3 corner = ld3(q);
      const double num = dot(corner - o, qn);
      // t = num / den > t_min > 0 needs num and den of one sign: the other
      // half of the planes is rejected without the division
      if (!(num > 0.0 ? den > 0.0 : (num < 0.0 && den < 0.0))) continue;
#if PGG_QUAD_PREREJECT
      // planes certainly beyond min(best, t_max) skip the division: with
      // |num| > bound |den| (1 + 2^-50) the exact quotient exceeds bound by
      // more than the product's rounding, so RN(num / den) >= bound
      {
        const double bound = fmin(best, t_max);
        if (fabs(num) > __dmul_rn(__dmul_rn(bound, fabs(den)), 1.0 + 0x1p-50)) continue;
      }
#endif
      const double t = num / den;
      if (!(t > t_min && t < t_max && t < best)) continue;
      const D3 rel = (o + d * t) - corner;
      // u = un / |eu|^2 in [0, 1] decided without dividing (exact for the
      // correctly rounded quotient, see in_unit)
      if (!in_unit(dot(rel, ld3(q + 3)), q[14]) || !in_unit(dot(rel, ld3(q + 6)), q[15])) continue;
      best = t;
      which = 1;
      prim = i;
      if (kAny) break;
    }
  }
  Hit h;
  h.hit = which >= 0;
  h.t = best;
  if (kAny || !h.hit) {
    h.front = false;
    h.mat = -1;
    return h;
  }
  h.pos = o + d * best;
  if (which == 0) {
    const double* sp = S.sph + prim * SPH_STRIDE;
    h.nrm = (h.pos - ld3(sp)) / sp[3];
    h.mat = (int)sp[4];
  } else {
    const double* q = S.quad + prim * QUAD_STRIDE;
    h.nrm = ld3(q + 9);
    h.mat = (int)q[13];
  }
  const double facing = dot(h.nrm, d);
  h.front = facing < 0.0;
  if (facing > 0.0) h.nrm = neg(h.nrm);
  return h;
}

// ---------------------------------------------------------------------------
// BRDFs in float64 (pg/scene.py:247-380), NumPy operation order

__device__ __forceinline__ double ggx_ndf(double alpha, double c) {
  const double a2 = alpha * alpha;
  const double d = c * c * (a2 - 1.0) + 1.0;
  return a2 / fmax(PI_D * d * d, 1e-30);
}
__device__ __forceinline__ double smith_g1(double alpha, double c) {
  const double a2 = alpha * alpha;
  return 2.0 * c / fmax(c + sqrt(a2 + (1.0 - a2) * c * c), 1e-30);
}

__device__ D3 brdf_eval(int kind, D3 alb, D3 alb_pi, double rough, D3 wi, D3 wo, D3 n) {
  const double ci = dot(wi, n), co = dot(wo, n);
  if (!(ci > 0.0 && co > 0.0)) return d3(0, 0, 0);
  if (kind != 1) return alb_pi;
  const double alpha = fmax(rough * rough, 1e-6);
  const D3 h = normalize(wi + wo);
  const double ch = fabs(dot(h, n));
  const double hw = dot(h, wi);
  const double d = ggx_ndf(alpha, ch);
  const double g = smith_g1(alpha, fabs(ci)) * smith_g1(alpha, fabs(co));
  const double p5 = pow(fmin(fmax(1.0 - fabs(hw), 0.0), 1.0), 5.0);
  const double sc = d * g / fmax(4.0 * ci * co, 1e-30);
  const D3 fres = alb + (d3(1, 1, 1) - alb) * p5;
  return fres * sc;
}

__device__ double brdf_pdf(int kind, double rough, D3 wi, D3 wo, D3 n) {
  const double ci = dot(wi, n), co = dot(wo, n);
  if (!(ci > 0.0 && co > 0.0)) return 0.0;
  if (kind != 1) return ci / PI_D;
  const double alpha = fmax(rough * rough, 1e-6);
  const D3 h = normalize(wi + wo);
  const double ch = fabs(dot(h, n));
  return smith_g1(alpha, fabs(co)) * ggx_ndf(alpha, ch) / fmax(4.0 * co, 1e-30);
}

// revised ONB keyed on sign(n_z) (pg/sgmap.py:85-98)
struct Onb {
  D3 t, b, n;
  __device__ D3 world(D3 v) const { return (t * v.x + b * v.y) + n * v.z; }
  __device__ D3 local(D3 v) const { return d3(dot(v, t), dot(v, b), dot(v, n)); }
};
__device__ Onb onb(D3 n) {
  const double s = copysign(1.0, n.z);
  const double a = -1.0 / (s + n.z);
  const double b = n.x * n.y * a;
  return {d3(1.0 + s * n.x * n.x * a, s * b, -s * n.x), d3(b, s + n.y * n.y * a, -n.y), n};
}

__device__ D3 vndf_local(double alpha, D3 wo_l, double u1, double u2) {
  const D3 vh = normalize(wo_l * d3(alpha, alpha, 1.0));
  const double lensq = vh.x * vh.x + vh.y * vh.y;
  const bool safe = lensq > 1e-18;
  const double inv = 1.0 / sqrt(safe ? lensq : 1.0);
  const D3 t1 = safe ? d3(-vh.y * inv, vh.x * inv, 0.0) : d3(1.0, 0.0, 0.0);
  const D3 t2 = cross(vh, t1);
  const double r = sqrt(u1);
  const double phi = 2.0 * PI_D * u2;
  double sp, cp;
  sincos(phi, &sp, &cp);
  const double p1 = r * cp;
  double p2 = r * sp;
  const double s = 0.5 * (1.0 + vh.z);
  p2 = (1.0 - s) * sqrt(fmax(1.0 - p1 * p1, 0.0)) + s * p2;
  const D3 nh = (t1 * p1 + t2 * p2) + vh * sqrt(fmax(1.0 - p1 * p1 - p2 * p2, 0.0));
  const D3 h = normalize(d3(alpha * nh.x, alpha * nh.y, fmax(nh.z, 1e-9)));
  return (2.0 * dot(wo_l, h)) * h - wo_l;
}

// world-space BRDF sample, two draws (pg/scene.py:354-380)
__device__ D3 brdf_sample(int kind, double rough, D3 wo, D3 n, uint64_t& st, double& pdf, bool& valid) {
  const double u1 = u01d(pcg_next(st));
  const double u2 = u01d(pcg_next(st));
  const Onb f = onb(n);
  D3 wl;
  if (kind == 1) {
    const double alpha = fmax(rough * rough, 1e-6);
    wl = vndf_local(alpha, f.local(wo), u1, u2);
  } else {
    const double r = sqrt(u1);
    const double ang = 2.0 * PI_D * u2;
    double sa, ca;
    sincos(ang, &sa, &ca);
    wl = d3(r * ca, r * sa, sqrt(fmax(1.0 - u1, 0.0)));
  }
  const D3 wi = f.world(wl);
  valid = dot(wi, n) > 1e-9 && dot(wo, n) > 0.0;
  pdf = brdf_pdf(kind, rough, wi, wo, n);
  valid = valid && pdf > 0.0;
  return wi;
}

// NEE toward one uniformly picked one-sided quad emitter, three draws
// (pg/scene.py:386-414)
__device__ void sample_emitter(const SceneS& S, D3 p, uint64_t& st, D3& dir, double& dist, D3& le, double& pdf) {
  const double up = u01d(pcg_next(st));
  const double u1 = u01d(pcg_next(st));
  const double u2 = u01d(pcg_next(st));
  long long pick = (long long)(up * (double)S.ne);
  if (pick > S.ne - 1) pick = S.ne - 1;
  const int qi = (int)S.emit[pick];
  const double* q = S.quad + qi * QUAD_STRIDE;
  const D3 y = (ld3(q) + ld3(q + 3) * u1) + ld3(q + 6) * u2;
  const D3 d = y - p;
  dist = fmax(norm(d), 1e-12);
  dir = d / dist;
  const double cos_l = -dot(dir, ld3(q + 9));
  const bool lit = cos_l > 1e-9;
  pdf = lit ? dist * dist / (q[12] * fmax(cos_l, 1e-12) * (double)S.ne) : 0.0;
  le = lit ? S.emission((int)q[13]) : d3(0, 0, 0);
}

// ---------------------------------------------------------------------------
// G-buffer kernel (pg/ptrace.py:97-150, pg/scene.py:125-151)

struct GbArgs {
  pgg_scene scene;
  pgg_camera cam, prev;
  int has_prev;
  int W, H, row0, rows;
  uint8_t* flags;
  float4 *nd, *pr, *va, *am;
  int32_t* mat;
};

__device__ __forceinline__ D3 cam3(const double* v) { return d3(v[0], v[1], v[2]); }

// scene.project_to_pixels (pg/scene.py:138-151) of one point: continuous pixel
// coordinates in camera `c`'s frame; returns in_front (z > 1e-9)
__device__ __forceinline__ bool project_px(const pgg_camera& c, int w, int h, const D3 p, double& px, double& py) {
  const double aspect = (double)w / (double)h;
  const D3 dd = p - cam3(c.origin);
  const double zc = dot(dd, cam3(c.forward));
  const bool fr = zc > 1e-9;
  const double z = fr ? zc : 1.0;
  const double xc = dot(dd, cam3(c.right)) / z;
  const double yc = dot(dd, cam3(c.up)) / z;
  px = (xc / (c.tan_half_fov * aspect) + 1.0) * 0.5 * (double)w - 0.5;
  py = (1.0 - yc / c.tan_half_fov) * 0.5 * (double)h - 0.5;
  return fr;
}

__global__ void __launch_bounds__(128) k_gbuffer(const GbArgs A) {
  extern __shared__ double smem[];
  const SceneS S = stage_scene(A.scene, smem);
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int yl = blockIdx.y * blockDim.y + threadIdx.y;
  if (x >= A.W || yl >= A.rows) return;
  const int y = A.row0 + yl;
  const int64_t o = (int64_t)yl * A.W + x;
  const double aspect = (double)A.W / (double)A.H;
  const double th = A.cam.tan_half_fov;
  const double ndc_x = (2.0 * ((double)x + 0.5) / (double)A.W - 1.0) * th * aspect;
  const double ndc_y = (1.0 - 2.0 * ((double)y + 0.5) / (double)A.H) * th;
  const D3 d = normalize((cam3(A.cam.forward) + cam3(A.cam.right) * ndc_x) + cam3(A.cam.up) * ndc_y);
  const Hit h = cast<false>(S, cam3(A.cam.origin), d, RAY_EPS, INFINITY);
  const D3 view = neg(d);
  if (!h.hit) {
    A.flags[o] = 0;
    A.nd[o] = make_float4(0.f, 0.f, 0.f, 0.f);
    A.pr[o] = make_float4(0.f, 0.f, 0.f, 0.f);
    A.va[o] = make_float4((float)view.x, (float)view.y, (float)view.z, 0.f);
    A.am[o] = make_float4(0.f, 0.f, 0.f, 0.f);
    A.mat[o] = -1;
    return;
  }
  const int m = h.mat;
  const D3 alb = S.albedo(m);
  float mx = 0.f, my = 0.f;
  bool has = false;
  if (A.has_prev) {
    // previous camera's projection of the hit (pg/scene.py:138-151, pg/ptrace.py:132-150)
    double px, py;
    const bool in_front = project_px(A.prev, A.W, A.H, h.pos, px, py);
    const double tx = rint(px), ty = rint(py);
    has = in_front && tx >= 0.0 && tx < (double)A.W && ty >= 0.0 && ty < (double)A.H;
    if (has) {
      mx = (float)(px - (double)x);
      my = (float)(py - (double)y);
    }
  }
  const bool glossy = S.kind(m) == 1;
  A.flags[o] = (uint8_t)(1 | (has ? 2 : 0) | (glossy ? 4 : 0) | (h.front ? 8 : 0));
  A.nd[o] = make_float4((float)h.nrm.x, (float)h.nrm.y, (float)h.nrm.z, (float)h.t);
  A.pr[o] = make_float4((float)h.pos.x, (float)h.pos.y, (float)h.pos.z, (float)S.rough(m));
  A.va[o] = make_float4((float)view.x, (float)view.y, (float)view.z, (float)alb.x);
  A.am[o] = make_float4((float)alb.y, (float)alb.z, mx, my);
  A.mat[o] = m;
}

// ---------------------------------------------------------------------------
// Path lanes (pg/ptrace.py:223-355) and the per-pixel accumulation of
// pg/ptrace.py:382-494

struct RenderArgs {
  pgg_render_config cfg;
  pgg_scene scene;
  pgg_gbuffer gb;
  const int32_t* mat;
  const float4* s_dir;  // depth-0 samples (pg mode) or NULL
  const uint8_t* s_tag;
  pgg_render_out out;
};

struct LaneResult {
  D3 L, Li, vy;
  bool vv;
  int vs;
  int segs;
};

// Lane accumulators (L, Li, T, Tr, vy: 15 doubles) parked in shared memory:
// they change once per bounce, and keeping them out of the register file
// leaves the intersection loops their registers.
struct Park {
  volatile double* p;  // field k of this thread at p[k * stride]
  int stride;
  __device__ D3 get(int k) const { return d3(p[(3 * k) * stride], p[(3 * k + 1) * stride], p[(3 * k + 2) * stride]); }
  __device__ void set(int k, D3 v) const {
    p[(3 * k) * stride] = v.x;
    p[(3 * k + 1) * stride] = v.y;
    p[(3 * k + 2) * stride] = v.z;
  }
};
enum { P_L = 0, P_LI = 1, P_T = 2, P_TR = 3, P_VY = 4, P_FIELDS = 5 };

__device__ LaneResult trace_lane(const RenderArgs& A, const SceneS& S, bool valid0, bool front0, D3 pos, D3 nrm,
                                 int mat, D3 wo, uint64_t& st, int64_t lane_own, const Park& pk) {
  const pgg_render_config& C = A.cfg;
  LaneResult R;
  R.vv = false;
  R.vs = 0;
  R.segs = 0;
  const D3 zero = d3(0, 0, 0);
  pk.set(P_LI, zero);
  pk.set(P_VY, zero);
  if (!valid0) {
    R.L = S.bg;
    R.Li = zero;
    R.vy = zero;
    return R;
  }
  pk.set(P_L, front0 ? zero + S.emission(mat) : zero);
  pk.set(P_T, d3(1, 1, 1));
  pk.set(P_TR, zero);
  const bool do_nee = C.nee && S.ne > 0;
  for (int depth = 0; depth < C.max_depth; ++depth) {
    const int kd = S.kind(mat);
    const D3 alb = S.albedo(mat);
    const D3 alb_pi = S.albedo_pi(mat);
    const double rg = S.rough(mat);
    if (do_nee) {
      D3 ld, le;
      double dist, lpdf;
      sample_emitter(S, pos, st, ld, dist, le, lpdf);
      const D3 f = brdf_eval(kd, alb, alb_pi, rg, ld, wo, nrm);
      const double cx = dot(ld, nrm);
      D3 c = d3(0, 0, 0);
      if (lpdf > 0.0 && cx > 0.0 && any_pos(f)) {
        if (!cast<true>(S, pos, ld, RAY_EPS, dist - RAY_EPS).hit) c = le * f * (cx / lpdf);
      }
      pk.set(P_L, pk.get(P_L) + pk.get(P_T) * c);
      if (depth >= 1) pk.set(P_LI, pk.get(P_LI) + pk.get(P_TR) * c);
    }
    D3 wi;
    double pdf;
    bool ok;
    int strat = 0;
    if (depth == 0 && A.s_dir) {
      // guided (or plain) depth-0 sample of the guiding pass; continue the
      // stream after the draws it consumed
      const float4 sd = A.s_dir[lane_own];
      const uint8_t tg = A.s_tag[lane_own];
      wi = d3(sd.x, sd.y, sd.z);
      pdf = (double)sd.w;
      ok = (tg & 2) != 0;
      strat = tg & 1;
      for (int k = tg >> 2; k > 0; --k) st = st * PCG_MUL + PCG_INC;
    } else {
      wi = brdf_sample(kd, rg, wo, nrm, st, pdf, ok);
    }
    const D3 f = brdf_eval(kd, alb, alb_pi, rg, wi, wo, nrm);
    const double ci = dot(wi, nrm);
    ok = ok && pdf > 0.0 && ci > 0.0;
    if (!ok) break;
    const D3 w = f * (ci / pdf);
    pk.set(P_T, pk.get(P_T) * w);
    if (depth >= 1) pk.set(P_TR, pk.get(P_TR) * w);
    if (depth == 0) R.vs = strat;
    const Hit h = cast<false>(S, pos, wi, RAY_EPS, INFINITY);
    ++R.segs;
    if (!h.hit) {
      pk.set(P_L, pk.get(P_L) + pk.get(P_T) * S.bg);
      if (depth >= 1) pk.set(P_LI, pk.get(P_LI) + pk.get(P_TR) * S.bg);
      break;
    }
    pos = h.pos;
    nrm = h.nrm;
    mat = h.mat;
    wo = neg(wi);
    if (depth == 0) {
      R.vv = true;
      pk.set(P_VY, h.pos);
      pk.set(P_TR, d3(1, 1, 1));
      if (h.front) pk.set(P_LI, pk.get(P_LI) + S.emission(h.mat));
    }
  }
  R.L = pk.get(P_L);
  R.Li = pk.get(P_LI);
  R.vy = pk.get(P_VY);
  return R;
}

#ifndef PGG_RENDER_MIN_BLOCKS
#define PGG_RENDER_MIN_BLOCKS 8  // 64 registers: 0.99 ms vs 1.11 (5 blocks) / 1.36 (3 blocks) at 1080p
#endif
constexpr int RT_W = 32, RT_H = 4;  // pixel tile of one 128-thread block

__device__ void render_pixel(const RenderArgs& A, const SceneS& S, int x, int yl, int& segs, int& bad, const Park& pk) {
  const pgg_render_config& C = A.cfg;
  const int y = C.row0 + yl;
  const int64_t own = (int64_t)yl * C.width + x;
  const int64_t gi = (int64_t)(y - A.gb.row0) * C.width + x;
  const uint8_t fl = A.gb.flags[gi];
  const bool valid = fl & 1, front = (fl & 8) != 0;
  const float4 nd = reinterpret_cast<const float4*>(A.gb.nd)[gi];
  const float4 pr = reinterpret_cast<const float4*>(A.gb.pr)[gi];
  const float4 va = reinterpret_cast<const float4*>(A.gb.va)[gi];
  const int m = valid ? A.mat[gi] : 0;
  const uint64_t pix = (uint64_t)y * (uint64_t)C.width + (uint64_t)x;
  D3 acc = d3(0, 0, 0);
  double lsum = 0.0, lsq = 0.0;
  LaneResult R;
  for (int s = 0; s < C.spp; ++s) {
    const int64_t lane = own * C.spp + s;
    uint64_t st = A.out.states ? A.out.states[lane] : pcg_lane(C.key, pix * (uint64_t)C.spp + (uint64_t)s);
    R = trace_lane(A, S, valid, front, d3(pr.x, pr.y, pr.z), d3(nd.x, nd.y, nd.z), m, d3(va.x, va.y, va.z), st,
                   own * C.spp + s, pk);
    if (A.out.states) A.out.states[lane] = st;
    segs += R.segs;
    if (!finite3(R.L)) {
      ++bad;
      R.L = d3(0, 0, 0);
    }
    if (!finite3(R.Li)) {
      R.Li = d3(0, 0, 0);
      R.vv = false;
    }
    acc = acc + R.L;
    const double lum = (R.L.x * 0.2126 + R.L.y * 0.7152) + R.L.z * 0.0722;
    lsum += lum;
    lsq += lum * lum;
  }
  const D3 img = acc / (double)C.spp;
  float* im = A.out.image + own * 3;
  im[0] = (float)img.x;
  im[1] = (float)img.y;
  im[2] = (float)img.z;
  // VPL of the last lane, in the guiding pass's packed layout
  const bool usable = R.vv && R.vs == 0;
  reinterpret_cast<float4*>(A.out.vpl_y)[own] =
      make_float4((float)R.vy.x, (float)R.vy.y, (float)R.vy.z, usable ? 1.0f : 0.0f);
  reinterpret_cast<float4*>(A.out.vpl_L)[own] =
      make_float4((float)R.Li.x, (float)R.Li.y, (float)R.Li.z, (float)((R.vv ? 1 : 0) | (R.vs << 1)));
  if (A.out.lum_moments) {
    A.out.lum_moments[2 * own] = lsum;
    A.out.lum_moments[2 * own + 1] = lsq;
  }
}

// One 32 x 4 pixel tile per block; the scene table is staged in shared
// memory per block (a persistent-grid variant measured no faster: 1.01 vs
// 0.99 ms at 1080p).
__global__ void __launch_bounds__(RT_W * RT_H, PGG_RENDER_MIN_BLOCKS) k_render(const RenderArgs A) {
  extern __shared__ double smem[];
  const SceneS S = stage_scene(A.scene, smem);
  const pgg_render_config& C = A.cfg;
  int segs = 0, bad = 0;
  const int x = blockIdx.x * RT_W + threadIdx.x;
  const int yl = blockIdx.y * RT_H + threadIdx.y;
  const int tid = threadIdx.x + RT_W * threadIdx.y;
  const Park pk{smem + table_doubles_d(A.scene) + tid, RT_W * RT_H};
  if (x < C.width && yl < C.rows) render_pixel(A, S, x, yl, segs, bad, pk);
  if (A.out.counters) {
    const unsigned sg = __reduce_add_sync(0xffffffffu, (unsigned)segs);
    const unsigned bd = __reduce_add_sync(0xffffffffu, (unsigned)bad);
    if ((threadIdx.x & 31) == 0) {
      if (sg) atomicAdd(A.out.counters, (unsigned long long)sg);
      if (bd) atomicAdd(A.out.counters + 1, (unsigned long long)bd);
    }
  }
}

// ---------------------------------------------------------------------------
// Image error metrics (pg/metrics.py:24-47): float64 per-element terms,
// deterministic two-level reduction (fixed grid, fixed tree), no atomics.

#ifndef PGG_ERR_UNROLL
#define PGG_ERR_UNROLL 1
#endif
#ifndef PGG_ERR_GRID
#define PGG_ERR_GRID PGG_IMAGE_ERROR_SCRATCH
#endif
constexpr int ERR_BLOCKS = PGG_ERR_GRID;  // 8 x 148 SMs, one partial per block
constexpr int ERR_THREADS = 256;

__device__ __forceinline__ double err_term(float a, float r, int rel) {
  const double d = (double)a - (double)r;
  const double e = d * d;
  if (!rel) return e;
  const double rr = (double)r;
  return e / (rr * rr + 0.01);
}

__device__ __forceinline__ double err4(const float4& x, const float4& y, int rel) {
  return ((err_term(x.x, y.x, rel) + err_term(x.y, y.y, rel)) + err_term(x.z, y.z, rel)) + err_term(x.w, y.w, rel);
}

__device__ double block_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = 0.0;
  if (w == 0) {
    v = l < (int)(blockDim.x >> 5) ? sh[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;
}

// HBM-bound: 8 bytes read per element.  Four independent float4 pairs are
// loaded per step so each thread keeps several requests in flight.
__global__ void __launch_bounds__(ERR_THREADS) k_err_partial(int64_t n, const float* __restrict__ a,
                                                            const float* __restrict__ r, int rel, double* part) {
  __shared__ double sh[32];
  double acc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n4 = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(r)) & 15) ? 0 : n / 4;
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* r4 = reinterpret_cast<const float4*>(r);
  int64_t i = t0;
#if PGG_ERR_UNROLL
  for (; i + 3 * stride < n4; i += 4 * stride) {
    const float4 x0 = __ldcs(a4 + i), y0 = __ldcs(r4 + i);
    const float4 x1 = __ldcs(a4 + i + stride), y1 = __ldcs(r4 + i + stride);
    const float4 x2 = __ldcs(a4 + i + 2 * stride), y2 = __ldcs(r4 + i + 2 * stride);
    const float4 x3 = __ldcs(a4 + i + 3 * stride), y3 = __ldcs(r4 + i + 3 * stride);
    acc += err4(x0, y0, rel);
    acc += err4(x1, y1, rel);
    acc += err4(x2, y2, rel);
    acc += err4(x3, y3, rel);
  }
#endif
  for (; i < n4; i += stride) acc += err4(a4[i], r4[i], rel);
  for (int64_t j = n4 * 4 + t0; j < n; j += stride) acc += err_term(a[j], r[j], rel);
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void __launch_bounds__(ERR_THREADS) k_err_final(int nb, const double* part, int64_t n, double* out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) acc += part[i];
  const double s = block_sum(acc, sh);
  if (threadIdx.x == 0) *out = s / (double)n;
}


// ---------------------------------------------------------------------------
// Lane kernels: the scene routines of pg/scene.py as batch operations
// (intersect / occluded, sample_emitter, brdf_eval / brdf_pdf /
// brdf_sample, primary_ray_dirs, project_to_pixels), float64 in / out.

__device__ __forceinline__ D3 ldd3(const double* p, int64_t i) { return d3(p[3 * i], p[3 * i + 1], p[3 * i + 2]); }
__device__ __forceinline__ void std3(double* p, int64_t i, D3 v) {
  p[3 * i] = v.x;
  p[3 * i + 1] = v.y;
  p[3 * i + 2] = v.z;
}

__global__ void __launch_bounds__(128) k_lane_intersect(const pgg_scene sc, int64_t n, const double* o, const double* d,
                                                        const double* t_min, const double* t_max, int any_hit,
                                                        uint8_t* hit, double* t, double* pos, double* nrm,
                                                        int32_t* mat, uint8_t* front) {
  extern __shared__ double smem[];
  const SceneS S = stage_scene(sc, smem);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const D3 oi = ldd3(o, i), di = ldd3(d, i);
  if (any_hit) {
    hit[i] = cast<true>(S, oi, di, t_min[i], t_max[i]).hit ? 1 : 0;
    return;
  }
  const Hit h = cast<false>(S, oi, di, t_min[i], t_max[i]);
  hit[i] = h.hit ? 1 : 0;
  t[i] = h.hit ? h.t : INFINITY;
  // the reference's pos = o + best_t d is non-finite on a miss (best_t = inf)
  std3(pos, i, h.hit ? h.pos : oi + di * INFINITY);
  std3(nrm, i, h.hit ? h.nrm : d3(0, 0, 0));
  mat[i] = h.hit ? h.mat : -1;
  front[i] = h.front ? 1 : 0;
}

__global__ void __launch_bounds__(128) k_lane_emitter(const pgg_scene sc, int64_t n, const double* pts,
                                                      uint64_t* states, double* dir, double* dist, double* le,
                                                      double* pdf) {
  extern __shared__ double smem[];
  const SceneS S = stage_scene(sc, smem);
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || S.ne == 0) return;
  uint64_t st = states[i];
  D3 w, e;
  double ds, p;
  sample_emitter(S, ldd3(pts, i), st, w, ds, e, p);
  states[i] = st;
  std3(dir, i, w);
  dist[i] = ds;
  std3(le, i, e);
  pdf[i] = p;
}

// op 0: eval (f rgb), 1: pdf, 2: sample (wi, pdf, valid; two draws per lane)
__global__ void __launch_bounds__(128) k_lane_brdf(int op, int64_t n, const int32_t* kind, const double* alb,
                                                   const double* rough, double* wi, const double* wo, const double* nn,
                                                   uint64_t* states, double* f, double* pdf, uint8_t* valid) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int k = kind[i];
  const D3 woi = ldd3(wo, i), ni = ldd3(nn, i);
  if (op == 0) {
    const D3 a = ldd3(alb, i);
    std3(f, i, brdf_eval(k, a, a / PI_D, rough[i], ldd3(wi, i), woi, ni));
  } else if (op == 1) {
    pdf[i] = brdf_pdf(k, rough[i], ldd3(wi, i), woi, ni);
  } else {
    uint64_t st = states[i];
    double p;
    bool ok;
    const D3 w = brdf_sample(k, rough[i], woi, ni, st, p, ok);
    states[i] = st;
    std3(wi, i, w);
    pdf[i] = p;
    valid[i] = ok ? 1 : 0;
  }
}

// primary_ray_dirs (pg/scene.py:125-135) and project_to_pixels (138-151)
__global__ void k_lane_rays(pgg_camera cam, int w, int h, int64_t n, const double* px, const double* py, double* dirs) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double aspect = (double)w / (double)h;
  const double nx = (2.0 * (px[i] + 0.5) / (double)w - 1.0) * cam.tan_half_fov * aspect;
  const double ny = (1.0 - 2.0 * (py[i] + 0.5) / (double)h) * cam.tan_half_fov;
  std3(dirs, i, normalize((cam3(cam.forward) + cam3(cam.right) * nx) + cam3(cam.up) * ny));
}

__global__ void k_lane_project(pgg_camera cam, int w, int h, int64_t n, const double* pts, double* px, double* py,
                               uint8_t* in_front) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x, y;
  const bool fr = project_px(cam, w, h, ldd3(pts, i), x, y);
  px[i] = x;
  py[i] = y;
  in_front[i] = fr ? 1 : 0;
}

// ptrace.motion_vectors (pg/ptrace.py:132-150) over a caller G-buffer's hit
// points: offset to the previous camera's projection where the pixel is
// valid, in front of that camera and rounds (np.rint) inside the frame
__global__ void k_motion_vectors(pgg_camera prev, int w, int h, const double* pos, const uint8_t* valid,
                                 double* motion, uint8_t* has) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)w * h) return;
  double px, py;
  const bool fr = project_px(prev, w, h, ldd3(pos, i), px, py);
  const double tx = rint(px), ty = rint(py);
  const bool ok = valid[i] && fr && tx >= 0.0 && tx < (double)w && ty >= 0.0 && ty < (double)h;
  motion[2 * i] = ok ? px - (double)(i % w) : 0.0;
  motion[2 * i + 1] = ok ? py - (double)(i / w) : 0.0;
  has[i] = ok ? 1 : 0;
}


// ---------------------------------------------------------------------------
// Equal-area square <-> hemisphere map and tangent frames as lane kernels
// (sgmap.py:21-115), float64: op 0 square->disk (2 -> 2), 1 disk->square
// (2 -> 2), 2 square->hemisphere (2 -> 3), 3 hemisphere->square (3 -> 2),
// 4 tangent frame of a normal (3 -> t 3, b 3), 5 local->world and 6
// world->local (t, b, n, v: 12 -> 3).

__device__ void conc_disk(double px, double py, double& x, double& y) {
  const double a = 2.0 * px - 1.0, b = 2.0 * py - 1.0;
  double r = b, phi;
  if (fabs(a) > fabs(b)) {
    r = a;
    phi = (0.25 * PI_D) * (b / a);
  } else if (b != 0.0) {
    phi = 0.5 * PI_D - (0.25 * PI_D) * (a / b);
  } else {
    phi = 0.0;  // the centre
  }
  double sp, cp;
  sincos(phi, &sp, &cp);
  x = r * cp;
  y = r * sp;
}

__device__ void conc_square(double x, double y, double& u, double& v) {
  const double rho = hypot(x, y);
  double a = 0.0, b = 0.0;
  if (rho != 0.0) {
    if (fabs(x) >= fabs(y)) {
      a = copysign(rho, x);
      b = atan(y / x) * (4.0 / PI_D) * a;
    } else {
      b = copysign(rho, y);
      a = atan(x / y) * (4.0 / PI_D) * b;
    }
  }
  u = fmin(fmax((a + 1.0) * 0.5, 0.0), 1.0);
  v = fmin(fmax((b + 1.0) * 0.5, 0.0), 1.0);
}

__global__ void k_lane_sgmap(int op, int64_t n, const double* __restrict__ in, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  switch (op) {
    case 0: conc_disk(in[2 * i], in[2 * i + 1], out[2 * i], out[2 * i + 1]); break;
    case 1: conc_square(in[2 * i], in[2 * i + 1], out[2 * i], out[2 * i + 1]); break;
    case 2: {
      double x, y;
      conc_disk(in[2 * i], in[2 * i + 1], x, y);
      const double r2 = x * x + y * y;  // Lambert lift (sgmap.py:59-65)
      const double lift = sqrt(fmax(2.0 - r2, 0.0));
      std3(out, i, d3(x * lift, y * lift, 1.0 - r2));
      break;
    }
    case 3: {
      const D3 w = ldd3(in, i);
      const double s = sqrt(fmax(1.0 + w.z, 1e-30));
      conc_square(w.x / s, w.y / s, out[2 * i], out[2 * i + 1]);
      break;
    }
    case 4: {
      const Onb f = onb(ldd3(in, i));
      std3(out, 2 * i, f.t);
      std3(out, 2 * i + 1, f.b);
      break;
    }
    default: {
      const Onb f{ldd3(in, 4 * i), ldd3(in, 4 * i + 1), ldd3(in, 4 * i + 2)};
      const D3 v = ldd3(in, 4 * i + 3);
      std3(out, i, op == 5 ? f.world(v) : f.local(v));
    }
  }
}

int table_doubles(const pgg_scene* s) {
  return s->n_mat * MAT_STRIDE + s->n_sph * SPH_STRIDE + s->n_quad * QUAD_STRIDE + s->n_emit;
}

bool scene_ok(const pgg_scene* s) {
  return s && s->table && s->n_mat > 0 && s->n_sph >= 0 && s->n_quad >= 0 && s->n_emit >= 0 &&
         s->n_emit <= s->n_quad && table_doubles(s) <= MAX_TABLE;
}

}  // namespace

extern "C" {

int pgg_gbuffer_pass(const pgg_scene* scene, const pgg_camera* cam, const pgg_camera* prev_cam, int32_t width,
                     int32_t height, int32_t row0, int32_t rows, uint8_t* flags, float* nd, float* pr, float* va,
                     float* am, int32_t* mat, void* stream) {
  if (!scene_ok(scene) || !cam || width <= 0 || height <= 0 || row0 < 0 || rows < 0 || row0 + rows > height ||
      !flags || !nd || !pr || !va || !am || !mat)
    return PGG_ERR_ARGUMENT;
  if (rows == 0) return PGG_OK;
  GbArgs A;
  A.scene = *scene;
  A.cam = *cam;
  A.has_prev = prev_cam != nullptr;
  if (prev_cam) A.prev = *prev_cam;
  A.W = width;
  A.H = height;
  A.row0 = row0;
  A.rows = rows;
  A.flags = flags;
  A.nd = reinterpret_cast<float4*>(nd);
  A.pr = reinterpret_cast<float4*>(pr);
  A.va = reinterpret_cast<float4*>(va);
  A.am = reinterpret_cast<float4*>(am);
  A.mat = mat;
  const dim3 blk(32, 4), grd((width + 31) / 32, (rows + 3) / 4);
  if (const int rc = pgg_rt::device_check()) return rc;
  k_gbuffer<<<grd, blk, table_doubles(scene) * sizeof(double), reinterpret_cast<cudaStream_t>(stream)>>>(A);
  return pgg_rt::check_launch();
}

int pgg_render_pass(const pgg_render_config* cfg, const pgg_scene* scene, const pgg_gbuffer* gb, const int32_t* mat,
                    const pgg_samples* depth0, const pgg_render_out* out, void* stream) {
  if (!cfg || !scene_ok(scene) || !gb || !mat || !out || !out->image || !out->vpl_y || !out->vpl_L)
    return PGG_ERR_ARGUMENT;
  if (cfg->width <= 0 || cfg->height <= 0 || cfg->row0 < 0 || cfg->rows < 0 || cfg->row0 + cfg->rows > cfg->height ||
      cfg->spp < 1 || cfg->max_depth < 1 || cfg->spp * 35 > (1 << 30))
    return PGG_ERR_ARGUMENT;
  if (gb->row0 > cfg->row0 || gb->row0 + gb->rows < cfg->row0 + cfg->rows || !gb->flags || !gb->nd || !gb->pr ||
      !gb->va)
    return PGG_ERR_ARGUMENT;
  if (depth0 && (!depth0->dir || !depth0->tag)) return PGG_ERR_ARGUMENT;
  if (cfg->rows == 0) return PGG_OK;
  RenderArgs A;
  A.cfg = *cfg;
  A.scene = *scene;
  A.gb = *gb;
  A.mat = mat;
  A.s_dir = depth0 ? reinterpret_cast<const float4*>(depth0->dir) : nullptr;
  A.s_tag = depth0 ? depth0->tag : nullptr;
  A.out = *out;
  const dim3 grd((cfg->width + RT_W - 1) / RT_W, (cfg->rows + RT_H - 1) / RT_H);
  const size_t smem = (table_doubles(scene) + 3 * P_FIELDS * RT_W * RT_H) * sizeof(double);
  if (const int rc = pgg_rt::device_check()) return rc;
  k_render<<<grd, dim3(RT_W, RT_H), smem, reinterpret_cast<cudaStream_t>(stream)>>>(A);
  return pgg_rt::check_launch();
}

int pgg_image_error(int64_t n, const float* a, const float* ref, int32_t relative, double* scratch, double* out,
                    void* stream) {
  if (n <= 0 || !a || !ref || !scratch || !out) return PGG_ERR_ARGUMENT;
  const cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (const int rc = pgg_rt::device_check()) return rc;
  k_err_partial<<<ERR_BLOCKS, ERR_THREADS, 0, st>>>(n, a, ref, relative ? 1 : 0, scratch);
  k_err_final<<<1, ERR_THREADS, 0, st>>>(ERR_BLOCKS, scratch, n, out);
  return pgg_rt::check_launch();
}

static inline unsigned lane_blocks(int64_t n) { return (unsigned)((n + 127) / 128); }

int pgg_intersect(const pgg_scene* scene, int64_t n, const double* origins, const double* dirs, const double* t_min,
                  const double* t_max, int32_t any_hit, uint8_t* hit, double* t, double* pos, double* normal,
                  int32_t* mat, uint8_t* front, void* stream) {
  if (!scene_ok(scene) || n < 0 || !origins || !dirs || !t_min || !t_max || !hit) return PGG_ERR_ARGUMENT;
  if (!any_hit && (!t || !pos || !normal || !mat || !front)) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = pgg_rt::device_check()) return rc;
  k_lane_intersect<<<lane_blocks(n), 128, table_doubles(scene) * sizeof(double), reinterpret_cast<cudaStream_t>(stream)>>>(
      *scene, n, origins, dirs, t_min, t_max, any_hit, hit, t, pos, normal, mat, front);
  return pgg_rt::check_launch();
}

int pgg_sample_emitter(const pgg_scene* scene, int64_t n, const double* points, uint64_t* states, double* dir,
                       double* dist, double* emitted, double* pdf, void* stream) {
  if (!scene_ok(scene) || scene->n_emit < 1 || n < 0 || !points || !states || !dir || !dist || !emitted || !pdf)
    return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = pgg_rt::device_check()) return rc;
  k_lane_emitter<<<lane_blocks(n), 128, table_doubles(scene) * sizeof(double), reinterpret_cast<cudaStream_t>(stream)>>>(
      *scene, n, points, states, dir, dist, emitted, pdf);
  return pgg_rt::check_launch();
}

int pgg_brdf(int32_t op, int64_t n, const int32_t* kind, const double* albedo, const double* rough, double* wi,
             const double* wo, const double* normal, uint64_t* states, double* f, double* pdf, uint8_t* valid,
             void* stream) {
  if (op < 0 || op > 2 || n < 0 || !kind || !rough || !wi || !wo || !normal) return PGG_ERR_ARGUMENT;
  if ((op == 0 && (!albedo || !f)) || (op == 1 && !pdf) || (op == 2 && (!states || !pdf || !valid)))
    return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = pgg_rt::device_check()) return rc;
  k_lane_brdf<<<lane_blocks(n), 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(op, n, kind, albedo, rough, wi, wo,
                                                                                  normal, states, f, pdf, valid);
  return pgg_rt::check_launch();
}

int pgg_primary_rays(const pgg_camera* cam, int32_t width, int32_t height, int64_t n, const double* px,
                     const double* py, double* dirs, void* stream) {
  if (!cam || width <= 0 || height <= 0 || n < 0 || !px || !py || !dirs) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = pgg_rt::device_check()) return rc;
  k_lane_rays<<<lane_blocks(n), 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*cam, width, height, n, px, py,
                                                                                  dirs);
  return pgg_rt::check_launch();
}

int pgg_project(const pgg_camera* cam, int32_t width, int32_t height, int64_t n, const double* points, double* px,
                double* py, uint8_t* in_front, void* stream) {
  if (!cam || width <= 0 || height <= 0 || n < 0 || !points || !px || !py || !in_front) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = pgg_rt::device_check()) return rc;
  k_lane_project<<<lane_blocks(n), 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*cam, width, height, n, points,
                                                                                     px, py, in_front);
  return pgg_rt::check_launch();
}

int pgg_motion_vectors(const pgg_camera* prev_cam, int32_t width, int32_t height, const double* pos,
                       const uint8_t* valid, double* motion, uint8_t* has_history, void* stream) {
  if (!prev_cam || width < 0 || height < 0 || !pos || !valid || !motion || !has_history) return PGG_ERR_ARGUMENT;
  const int64_t n = (int64_t)width * height;
  if (n == 0) return PGG_OK;
  if (const int rc = pgg_rt::device_check()) return rc;
  k_motion_vectors<<<lane_blocks(n), 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*prev_cam, width, height, pos,
                                                                                       valid, motion, has_history);
  return pgg_rt::check_launch();
}

int pgg_sgmap(int32_t op, int64_t n, const double* in, double* out, void* stream) {
  if (op < 0 || op > 6 || n < 0 || !in || !out) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = pgg_rt::device_check()) return rc;
  k_lane_sgmap<<<lane_blocks(n), 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(op, n, in, out);
  return pgg_rt::check_launch();
}

}  // extern "C"
