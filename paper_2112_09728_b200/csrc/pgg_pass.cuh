// pgg_pass.cuh — per-pixel / per-lane bodies of the guiding pass.
//
// The CUDA kernels (pgg_kernels.cu) are thin grid loops over these
// functions; the test-only host build (pgg_hostcheck.cpp) runs the very same
// bodies on the CPU so the device formulas can be checked against the oracle
// without a GPU.  Reference semantics cited per stage.
#pragma once

#include <string.h>

#include "pgg.h"
#include "pgg_math.cuh"

namespace pgg {

#ifndef PGG_SMP_UNIFORM_PDF
#define PGG_SMP_UNIFORM_PDF 1
#endif
#ifndef PGG_SHARE_LANE_HASH
#define PGG_SHARE_LANE_HASH 1
#endif
#ifndef PGG_GATES_F32
#define PGG_GATES_F32 1  // reprojection gates: float32 first, float64 only near the thresholds (0.5176 -> 0.5153 ms)
#endif
constexpr int SLOTS = 20;                 // guide_buffers.py:20

// Checked builds (-DPGG_CHECKS=1, libpgg_checked.so): every shared-memory
// tile read, global plane read and output store of the pass asserts its
// index bounds; failures are counted (first one recorded) in device globals
// read back by pgg_debug_checks().  compute-sanitizer is not available on
// this pool; this is its in-kernel substitute (tests/test_gpu_checked.py).
#ifndef PGG_CHECKS
#define PGG_CHECKS 0
#endif
#if PGG_CHECKS && defined(__CUDACC__)
__device__ int g_pgg_check[6];  // failures, first site, its two operands, blockIdx.x, blockIdx.y
#endif
#if PGG_CHECKS && defined(__CUDA_ARCH__)
__device__ __noinline__ void pgg_check_fail(int site, int a, int b) {
  if (atomicAdd(&g_pgg_check[0], 1) == 0) {
    g_pgg_check[1] = site;
    g_pgg_check[2] = a;
    g_pgg_check[3] = b;
    g_pgg_check[4] = blockIdx.x;
    g_pgg_check[5] = blockIdx.y;
  }
}
#define PGG_CHK(site, cond, a, b) \
  do {                            \
    if (!(cond)) pgg_check_fail(site, (int)(a), (int)(b)); \
  } while (0)
#else
#define PGG_CHK(site, cond, a, b) \
  do {                            \
  } while (0)
#endif
enum : int { CHK_TILE = 1, CHK_CUR = 2, CHK_GIN = 3, CHK_PREV = 4, CHK_VPL = 5, CHK_OUT = 6, CHK_SMP = 7 };
#ifndef PGG_PROF_TRIES
#define PGG_PROF_TRIES 16  // measurement-only override
#endif
constexpr int GAUSS_TRIES = PGG_PROF_TRIES;  // mixture.py:28 (16)
constexpr uint64_t J3_MUL = pcg_jump_mul(3);
constexpr uint64_t J3_ADD = pcg_jump_add(3);
constexpr uint64_t J19_MUL = pcg_jump_mul(SLOTS - 1);
constexpr uint64_t J19_ADD = pcg_jump_add(SLOTS - 1);

struct PassArgs {
  pgg_config cfg;
  pgg_gbuffer cur;
  pgg_gbuffer prev;
  pgg_gamma_in gin;
  pgg_vpl vpl;
  pgg_gamma_out grep;
  pgg_gamma_out gout;
  pgg_samples smp;
  int has_prev, has_vpl, has_grep, has_smp;
  int32_t* halo_misses;
  // record-loop constants precomputed on the host (kernel parameters, so the
  // loop reads them as constant-bank operands instead of holding registers)
  float em_radius16;  // (float) cfg.radius * 2^-16 (exact): R sqrt(u 2^-32) = em_radius16 sqrt(u)
  float em_hband;     // 0.5 - the candidate-offset rounding guard band
};

// fills the derived PassArgs fields from cfg (every construction site)
inline void pass_args_finish(PassArgs& A) {
  const float rf = (float)A.cfg.radius;
  A.em_radius16 = rf * 1.52587890625e-05f;
  A.em_hband = 0.5f - 4e-6f * (rf + 1.0f);
}

PGG_HD float4 f4(float x, float y, float z, float w) {
  float4 v;
  v.x = x;
  v.y = y;
  v.z = z;
  v.w = w;
  return v;
}

PGG_HD float4 ld4(const float* base, int64_t i) {
#ifdef __CUDA_ARCH__
  return __ldg(reinterpret_cast<const float4*>(base) + i);
#else
  const float* p = base + 4 * i;
  return f4(p[0], p[1], p[2], p[3]);
#endif
}

PGG_HD void st4(float* base, int64_t i, const float4& v) {
#ifdef __CUDA_ARCH__
  reinterpret_cast<float4*>(base)[i] = v;
#else
  float* p = base + 4 * i;
  p[0] = v.x;
  p[1] = v.y;
  p[2] = v.z;
  p[3] = v.w;
#endif
}

PGG_HD uint8_t ldu8(const uint8_t* p, int64_t i) {
#ifdef __CUDA_ARCH__
  return __ldg(p + i);
#else
  return p[i];
#endif
}

PGG_HD void count_miss(int32_t* c, int n = 1) {
  if (!c) return;
#ifdef __CUDA_ARCH__
  atomicAdd(c, n);
#else
  *c += n;
#endif
}

PGG_HD void init_gamma(float4& g0, float4& g1) {  // mixture.py:44-59
  g0 = f4(0.5f, 0.5f, 0.5f, 0.5f);
  g1 = f4(0.25f, 0.0f, 0.05f, 0.0f);
}

// float64 Cholesky of the lobe (guard-band re-evaluation of Box-Muller
// acceptance only); same arithmetic as make_lobe
PGG_HD void lobe_chol_d(float mxf, float myf, float m2xx, float m2yy, float m2xy, double& l11, double& l21,
                        double& l22) {
  const double mx = mxf, my = myf;
  double sxx = radd(rsub((double)m2xx, rmul(mx, mx)), 1e-4);
  double syy = radd(rsub((double)m2yy, rmul(my, my)), 1e-4);
  double sxy = rsub((double)m2xy, rmul(mx, my));
  const double half = rmul(0.5, radd(sxx, syy));
  const double dd = rsub(sxx, syy);
  const double q = radd(rmul(0.25, rmul(dd, dd)), rmul(sxy, sxy));
  if (rsub(half, sqrt(fmax(q, 0.0))) < 1e-6) {
    sxx = 0.05;
    syy = 0.05;
    sxy = 0.0;
  }
  l11 = sqrt(sxx);
  l21 = sxy / l11;
  l22 = sqrt(fmax(rsub(syy, rmul(l21, l21)), 1e-30));
}

// ---------------------------------------------------------------------------
// reprojection of one pixel (guide_buffers.py:78-137)

// sin(pi t), cos(pi t) for |t| <= 1/4: Taylor series in x = pi t to x^17 /
// x^18 (truncation < 1e-19 on |x| <= pi/4)
PGG_HD void sincospi_quarter(double t, double& s, double& c) {
  const double x = 3.141592653589793 * t;
  const double u = x * x;
  double ps = 2.8114572543455206e-15;             // 1/17!
  ps = fma(ps, u, -7.647163731819816e-13);        // -1/15!
  ps = fma(ps, u, 1.6059043836821613e-10);        // 1/13!
  ps = fma(ps, u, -2.505210838544172e-08);        // -1/11!
  ps = fma(ps, u, 2.7557319223985893e-06);        // 1/9!
  ps = fma(ps, u, -0.0001984126984126984);        // -1/7!
  ps = fma(ps, u, 0.008333333333333333);          // 1/5!
  ps = fma(ps, u, -0.16666666666666666);          // -1/3!
  s = fma(ps * u, x, x);
  double pc = -1.5619206968586225e-16;            // -1/18!
  pc = fma(pc, u, 4.779477332387385e-14);         // 1/16!
  pc = fma(pc, u, -1.1470745597729725e-11);       // -1/14!
  pc = fma(pc, u, 2.08767569878681e-09);          // 1/12!
  pc = fma(pc, u, -2.755731922398589e-07);        // -1/10!
  pc = fma(pc, u, 2.48015873015873e-05);          // 1/8!
  pc = fma(pc, u, -0.001388888888888889);         // -1/6!
  pc = fma(pc, u, 0.041666666666666664);          // 1/4!
  pc = fma(pc, u, -0.5);                          // -1/2!
  c = fma(pc, u, 1.0);
}

// sq_to_dir<double> (sgmap.py:21-33, 59-65) with the concentric angle
// reduced to |t| <= 1/4 (the else-branch angle pi (1/2 - t) swaps sin/cos)
PGG_HD V3<double> sq_to_dir_f64(float px, float py) {
  const double a = 2.0 * (double)px - 1.0;
  const double b = 2.0 * (double)py - 1.0;
  double r, s, c;
  if (fabs(a) > fabs(b)) {
    r = a;
    sincospi_quarter(0.25 * (b * d_rcp(a)), s, c);
  } else if (b != 0.0) {
    r = b;
    sincospi_quarter(0.25 * (a * d_rcp(b)), c, s);  // sin(pi/2 - x) = cos x
  } else {
    r = 0.0;
    s = 0.0;
    c = 1.0;
  }
  const double r2 = r * r;
  const double l2 = fmax(2.0 - r2, 0.0);
  const double lift = l2 > 0.0 ? l2 * d_rsqrt(l2) : 0.0;
  return {r * c * lift, r * s * lift, 1.0 - r2};
}

// dir_to_sq<double> (sgmap.py:67-77, 41-56) on the fast reciprocals
PGG_HD void dir_to_sq_f64(const V3<double>& v, double& sx, double& sy) {
  const double is = d_rsqrt(fmax(1.0 + v.z, 1e-30));
  const double x = v.x * is;
  const double y = v.y * is;
  const double r2 = x * x + y * y;
  double a, b;
  if (r2 == 0.0) {
    a = 0.0;
    b = 0.0;
  } else {
    const double rho = r2 * d_rsqrt(r2);
    if (fabs(x) >= fabs(y)) {
      a = copysign(rho, x);
      b = atan(y * d_rcp(x)) * (4.0 * K<double>::inv_pi) * a;
    } else {
      b = copysign(rho, y);
      a = atan(x * d_rcp(y)) * (4.0 * K<double>::inv_pi) * b;
    }
  }
  sx = fmin(fmax((a + 1.0) * 0.5, 0.0), 1.0);
  sy = fmin(fmax((b + 1.0) * 0.5, 0.0), 1.0);
}

// Mean rotation between the previous and current tangent frames
// (guide_buffers.py:117-133), in float64: M2 is carried unrotated, so the
// covariance M2 - mu mu^T of the next lobe cancels and amplifies any error
// in the rotated mean ~1/Sigma-fold; float64 keeps the float32-rounded mean
// identical to the reference's in all but boundary-rounding cases.
PGG_COLD void rotate_or_reject(const V3<float>& np_, const V3<float>& nc, float mux, float muy, bool& keep,
                             float& ox, float& oy) {
  keep = true;
  ox = mux;
  oy = muy;
  // identical normals: the rotation is the identity and the float64 round
  // trip of an interior mean rounds back to the same float32
  if (np_.x == nc.x && np_.y == nc.y && np_.z == nc.z && mux >= 1e-6f && mux <= 1.0f - 1e-6f &&
      muy >= 1e-6f && muy <= 1.0f - 1e-6f)
    return;
#if defined(__CUDA_ARCH__) && PGG_FAST_F64
  // float64 throughout, with range-reduced polynomials and Newton-refined
  // MUFU seeds instead of the library's general sincospi / division / sqrt
  // (~1 ulp of float64; the result is rounded to float32)
  const V3<double> dl = sq_to_dir_f64(mux, muy);
  V3<double> dc = make_frame_fast(cvt<double>(nc)).to_local(make_frame_fast(cvt<double>(np_)).to_world(dl));
#else
  const V3<double> dl = sq_to_dir<double>((double)mux, (double)muy);
  V3<double> dc = make_frame(cvt<double>(nc)).to_local(make_frame(cvt<double>(np_)).to_world(dl));
#endif
  if (dc.z < 0.0) {
    keep = false;
    return;
  }
  double sx, sy;
#if defined(__CUDA_ARCH__) && PGG_FAST_F64
  dir_to_sq_f64(dc, sx, sy);
#else
  dir_to_sq<double>(dc, sx, sy);
#endif
  ox = (float)sx;
  oy = (float)sy;
}

// Decision record of one pixel's reprojection (diagnostic builds of the same
// body, kDbg): bit0 accepted, bit1 the depth/normal gates were re-decided in
// float64 (float32 within the guard band), bit2 the mean rotation rejected
// (z < 0), bit3 the gates rejected.
enum : uint8_t { RP_ACCEPT = 1, RP_GATE_F64 = 2, RP_ROT_REJECT = 4, RP_GATE_REJECT = 8 };

template <bool kDbg = false>
PGG_HD void reproject_px(const PassArgs& A, int x, int y, uint8_t fl, const float4& nd, const float4& pr,
                         const float4& am, float4& g0, float4& g1, uint8_t* dbg = nullptr) {
  const pgg_config& C = A.cfg;
  init_gamma(g0, g1);
  if (kDbg) *dbg = 0;
  if ((fl & 3) != 3) return;  // valid & has_history
  const double tx = rint((double)x + (double)am.z);
  const double ty = rint((double)y + (double)am.w);
  if (!(tx >= 0.0 && tx < (double)C.width && ty >= 0.0 && ty < (double)C.height)) return;
  const int sx = (int)tx, sy = (int)ty;
  if (sy < A.prev.row0 || sy >= A.prev.row0 + A.prev.rows || sy < A.gin.row0 || sy >= A.gin.row0 + A.gin.rows) {
    count_miss(A.halo_misses);
    return;
  }
  const int64_t sp = (int64_t)(sy - A.prev.row0) * C.width + sx;
  const int64_t gi = (int64_t)(sy - A.gin.row0) * C.width + sx;
  PGG_CHK(CHK_PREV, sy - A.prev.row0 >= 0 && sy - A.prev.row0 < A.prev.rows && sx >= 0 && sx < C.width, sy, sx);
  PGG_CHK(CHK_GIN, sy - A.gin.row0 >= 0 && sy - A.gin.row0 < A.gin.rows, sy, A.gin.row0);
  // the source's gate planes and Gamma in flight together
  const uint8_t pfl = ldu8(A.prev.flags, sp);
  const float4 ndp = ld4(A.prev.nd, sp);
  float4 p0 = ld4(A.gin.g0, gi);
  const float4 p1 = ld4(A.gin.g1, gi);
  if (!(pfl & 1)) return;
#if PGG_GATES_F32
  // depth and normal gates decided in float32 when clear of the threshold,
  // else in float64 with the reference's operation order.  Depth band: an
  // absolute bound on the float32 error of lhs - rhs -- the rounding of
  // (float)prev_cam (|cam| 2^-24 per component), of the differences, of the
  // norm (a few ulps of def) and of ndp.w, rhs -- taken as 2^-19 (def + |ndp.w|
  // + |cam|_1) (>= 8x the worst case), plus 1e-5 relative to rhs.
  int gate = 0;  // 1 pass, -1 reject, 0 undecided
  {
    const float cx = (float)C.prev_cam[0], cy = (float)C.prev_cam[1], cz = (float)C.prev_cam[2];
    const float fx = pr.x - cx, fy = pr.y - cy, fz = pr.z - cz;
    const float def = sqrtf(fx * fx + fy * fy + fz * fz);
    const float lhs = fabsf(ndp.w - def), rhs = (float)C.depth_rel_tol * fmaxf(def, 1e-12f);
    const float nf = ndp.x * nd.x + ndp.y * nd.y + ndp.z * nd.z, tn = (float)C.normal_dot_min;
    const float eps = 1.9073486328125e-06f * (def + fabsf(ndp.w) + fabsf(cx) + fabsf(cy) + fabsf(cz)) + 1e-5f * rhs;
    const bool dpass = lhs < rhs - eps, dfail = lhs > rhs + eps;
    const bool npass = nf > tn + 1e-5f, nfail = nf < tn - 1e-5f;
    if (dfail || nfail) gate = -1;
    else if (dpass && npass) gate = 1;
  }
  if (gate < 0) {
    if (kDbg) *dbg |= RP_GATE_REJECT;
    return;
  }
  if (gate == 0) {
    if (kDbg) *dbg |= RP_GATE_F64;
#endif
  // depth and normal gates in float64, reference operation order
  const double dx = rsub((double)pr.x, C.prev_cam[0]);
  const double dy = rsub((double)pr.y, C.prev_cam[1]);
  const double dz = rsub((double)pr.z, C.prev_cam[2]);
  const double de = sqrt(radd(radd(rmul(dx, dx), rmul(dy, dy)), rmul(dz, dz)));
  if (!(fabs(rsub((double)ndp.w, de)) < rmul(C.depth_rel_tol, fmax(de, 1e-12)))) {
    if (kDbg) *dbg |= RP_GATE_REJECT;
    return;
  }
  const double ndot = radd(radd(rmul((double)ndp.x, (double)nd.x), rmul((double)ndp.y, (double)nd.y)),
                           rmul((double)ndp.z, (double)nd.z));
  if (!(ndot > C.normal_dot_min)) {
    if (kDbg) *dbg |= RP_GATE_REJECT;
    return;
  }
#if PGG_GATES_F32
  }
#endif
  if (C.rotate_mean) {
    bool keep;
    float ox, oy;
#ifdef PGG_PROF_NO_ROT
    keep = true, ox = p0.x, oy = p0.y;  // measurement-only build
#else
    rotate_or_reject(v3(ndp.x, ndp.y, ndp.z), v3(nd.x, nd.y, nd.z), p0.x, p0.y, keep, ox, oy);
#endif
    if (!keep) {
      if (kDbg) *dbg |= RP_ROT_REJECT;
      return;
    }
    p0.x = ox;
    p0.y = oy;
  }
  g0 = p0;
  g1 = p1;
  if (kDbg) *dbg |= RP_ACCEPT;
}

// ---------------------------------------------------------------------------
// depth-0 sampling of one lane (ptrace.py:161-220, mixture.py:193-259,
// scene.py:354-380).  `wo` is in world space; `n` the shading normal.
// Returns dir (world), pdf, strategy, valid.  `state` is advanced exactly as
// the reference advances it.

struct LaneOut {
  V3<float> wi;
  float pdf;
  int gauss;
  int valid;
  int draws;  // PCG32 draws consumed (the render continues the stream after them)
};

// float64 Cholesky provider for the rare guard-band acceptance recheck
struct CholD {
  float mx, my, m2xx, m2yy, m2xy;  // raw moments (pass), or
  int from_floats;                 // 1: use the float lobe upcast (lane API)
  float l11f, l21f, l22f;
  PGG_MHD void get(double& l11, double& l21, double& l22) const {
    if (from_floats) {
      l11 = l11f;
      l21 = l21f;
      l22 = l22f;
    } else {
      lobe_chol_d(mx, my, m2xx, m2yy, m2xy, l11, l21, l22);
    }
  }
};

// Box-Muller acceptance p in [0,1]^2 re-decided in float64 (the reference's
// arithmetic, mixture.py:216-224) when float32 lands within 1e-5 of an edge
PGG_COLD bool accept_d(const CholD& cd, float mx, float my, uint32_t a, uint32_t b) {
  double l11, l21, l22, d0, d1;
  cd.get(l11, l21, l22);
  box_muller_d(a, b, d0, d1);
  const double qx = radd((double)mx, rmul(l11, d0));
  const double qy = radd(radd((double)my, rmul(l21, d0)), rmul(l22, d1));
  return qx >= 0.0 && qx <= 1.0 && qy >= 0.0 && qy <= 1.0;
}

// float32 p = mu + L z carries <= ~1e-6 absolute error (|L z| <= 2): re-decide
// within 3e-6 of an edge
PGG_HD bool near_edge(float v) { return fabsf(v) < 3e-6f || fabsf(1.0f - v) < 3e-6f; }

PGG_COLD V3<float> brdf_draw_local_d(const Mat<float>& mf, float alpha, const V3<float>& wol, bool co_pos,
                                     uint32_t a, uint32_t b, bool& ok) {
  const Mat<double> md{mf.glossy, (double)mf.a2, (double)mf.kappa};
  bool ill_d;
  const V3<double> wd = brdf_sample_local<double>(md, (double)alpha, cvt<double>(wol), a, b, ill_d);
  ok = wd.z > 1e-9 && co_pos;
  return cvt<float>(wd);
}

// local-frame BRDF draw with its validity (wl.z > 1e-9, wo.z > 0); float64
// re-evaluation for the VNDF rim case and near the z threshold
PGG_HD V3<float> brdf_draw_local(const Mat<float>& mf, float alpha, const V3<float>& wol, bool co_pos, uint32_t a,
                                 uint32_t b, bool& ok, int* rechecks = nullptr) {
  bool ill;
  V3<float> wl = brdf_sample_local<float>(mf, alpha, wol, a, b, ill);
#ifdef PGG_PROF_NO_VNDF_RECHECK
  ill = false;  // measurement-only build
#endif
  if (ill || fabsf(wl.z) < 1e-6f) {
    if (rechecks) ++*rechecks;
    return brdf_draw_local_d(mf, alpha, wol, co_pos, a, b, ok);
  }
  ok = wl.z > 1e-9f && co_pos;
  return wl;
}

// One Box-Muller proposal p = mu + L z of the guided branch and its [0,1]^2
// acceptance (mixture.py:216-230): float32, re-decided in float64 within the
// guard band of an edge (*rechecked set then).
PGG_HD bool bm_propose(const LobeF& L, const CholD& cd, uint32_t a, uint32_t b, float& px, float& py,
                       bool* rechecked = nullptr) {
  float z0, z1;
  box_muller_f(a, b, z0, z1);
  px = L.mx + L.l11 * z0;
  py = L.my + L.l21 * z0 + L.l22 * z1;
  if (near_edge(px) || near_edge(py)) {
    if (rechecked) *rechecked = true;
    return accept_d(cd, L.mx, L.my, a, b);
  }
  return px >= 0.0f && px <= 1.0f && py >= 0.0f && py <= 1.0f;
}

PGG_HD LaneOut sample_lane(const PixelFrame& pf, bool glossy, float rough, bool guided, const LobeF& L,
                           const CholD& cd, uint64_t& st) {
  const Frame<float>& fr = pf.fr;
  const V3<float>& wol = pf.wol;
  const bool co_pos = pf.co_pos;
  const double r2d = (double)rough * (double)rough;
  const float alpha = (float)fmax(r2d, 1e-6);
  const float a2 = alpha * alpha;
  const Mat<float> mf{glossy, a2, guided ? a2 : kappa_world(pf.om_nn, a2)};
  LaneOut o;
  if (!guided) {
    // plain BRDF lane in the world frame (scene.py:354-380)
    const uint32_t a = pcg_next(st), b = pcg_next(st);
    bool ok;
    const V3<float> wl = brdf_draw_local(mf, alpha, wol, co_pos, a, b, ok);
    o.wi = fr.to_world(wl);
    o.pdf = co_pos ? brdf_pdf_local(mf, wl, wol) : 0.0f;
    o.gauss = 0;
    o.valid = ok && o.pdf > 0.0f;
    o.draws = 2;
    return o;
  }
  const uint32_t uz = pcg_next(st);
  o.draws = 1;
  bool acc = false;
  float sx = 0.0f, sy = 0.0f;
  if (u01d(uz) < (double)L.pi) {
    for (int t = 0; t < GAUSS_TRIES; ++t) {
      const uint32_t a = pcg_next(st), b = pcg_next(st);
      o.draws += 2;
      float px, py;
      if (bm_propose(L, cd, a, b, px, py)) {
        acc = true;
        sx = m_clamp01(px);
        sy = m_clamp01(py);
        break;
      }
    }
  }
  V3<float> dl;
  bool ok = true;
  if (acc) {
    dl = sq_to_dir<float>(sx, sy);
  } else {
    const uint32_t a = pcg_next(st), b = pcg_next(st);
    o.draws += 2;
    dl = brdf_draw_local(mf, alpha, wol, co_pos, a, b, ok);
  }
  o.gauss = acc ? 1 : 0;
  o.pdf = 0.0f;
  if (ok) {
    const float bp = co_pos ? brdf_pdf_local(mf, dl, wol) : 0.0f;
#if PGG_SMP_UNIFORM_PDF
    // every valid lane maps its direction back to the square, as the
    // reference does (mixture.py:250-256: hemisphere_to_square of the
    // direction); one path for Gaussian and BRDF lanes (no divergence)
    (void)sx;
    (void)sy;
    float qx, qy;
    {
      V3<float> dz = dl;
      dz.z = fmaxf(dz.z, 0.0f);
      dir_to_sq_f(dz, qx, qy);
    }
#else
    float qx = sx, qy = sy;
    if (!acc) {
      V3<float> dz = dl;
      dz.z = fmaxf(dz.z, 0.0f);
      dir_to_sq_f(dz, qx, qy);
    }
#endif
    const float g = gauss_sr(L, qx, qy);
    o.pdf = L.pi * g + (1.0f - L.pi) * bp;
  }
  o.valid = ok && o.pdf > 0.0f;
  o.wi = fr.to_world(dl);
  return o;
}

// ---------------------------------------------------------------------------
// EM training of one pixel (guide_buffers.py:140-231,262-283;
// mixture.py:262-321)

// candidate offset (rint of r cos, r sin) with float64 re-evaluation near
// the half-integer rounding boundary (guide_buffers.py:146-149)
struct Off2 {
  int x, y;
};

PGG_COLD Off2 disk_offset_d(uint32_t ua, uint32_t ub, double radius) {
  const double rd = radius * sqrt(u01d(ua));
  const double ang = 2.0 * K<double>::pi * u01d(ub);
  return {(int)rint(rd * cos(ang)), (int)rint(rd * sin(ang))};
}

#ifndef PGG_PI_FOLD
#define PGG_PI_FOLD 0  // 1: one multiply fewer per Lambert record; measured neutral (0.4276 vs 0.4276 ms), not kept
#endif
#if PGG_PI_FOLD
// 1/pi folded into the per-pixel constants (albedo, 1 - pi) and pi into G1(wo):
// the records' bp carries pi x the BRDF pdf and the Lambert bp is cos itself
constexpr float kLumR = (float)(0.2126 / 3.14159265358979323846), kLumG = (float)(0.7152 / 3.14159265358979323846),
                kLumB = (float)(0.0722 / 3.14159265358979323846);
#define PGG_LAMBERT_BP(cr) (cr)
#else
constexpr float kLumR = 0.2126f, kLumG = 0.7152f, kLumB = 0.0722f;
#define PGG_LAMBERT_BP(cr) ((cr) * K<float>::inv_pi)
#endif
#ifndef PGG_GAUSS_FMA
#define PGG_GAUSS_FMA 0  // 1: z by three FFMAs on pre-multiplied constants: -0.17 %, golden Gamma p99.99 2.7e-5 -> 3.6e-5 (not kept)
#endif
#ifndef PGG_W_UMASK
#define PGG_W_UMASK 1  // record weight test 0 < w <= FLT_MAX as one unsigned compare of the bits
#endif
#ifndef PGG_GGX_LA
#define PGG_GGX_LA 1  // GGX record weight as la + (luminance(L) - la) f5 (3 per-pixel invariants fewer): -0.45 %
#endif
#ifndef PGG_SB_JUMP
#define PGG_SB_JUMP 1  // the u2 stream derived from the u1 stream per slot (one live LCG state): -0.45 %, bitwise the same
#endif
#ifndef PGG_EM_RAW_RSQRT
#define PGG_EM_RAW_RSQRT 0  // 1: 0.6 % faster but golden Gamma p99.99 4.1e-5, and 1.07e-4 together with PGG_SQ_RAW
#endif
#ifndef PGG_EM_FAST
#define PGG_EM_FAST 1
#endif

// float32 candidate offset; values within `band` of a rounding boundary are
// re-evaluated in float64.  The band (4e-6 (R + 1)) bounds the float32
// error of r cos / r sin: on the device sin/cos come from MUFU.SIN/COS on
// [-pi, pi) (abs error < 2^-20.5, x R) and rint from the 1.5 * 2^23 add.
#ifndef PGG_TILE_OOB
#define PGG_TILE_OOB 1
#endif
#ifndef PGG_LOOP_TRIM
#define PGG_LOOP_TRIM 1
#endif
PGG_HD void disk_offset_k(uint32_t ua, uint32_t ub, double radius, float rf16, float hb, int& dx, int& dy,
                          int* rechecks = nullptr);
PGG_HD void disk_offset(uint32_t ua, uint32_t ub, double radius, int& dx, int& dy) {
  const float rf = (float)radius;
  disk_offset_k(ua, ub, radius, rf * 1.52587890625e-05f, 0.5f - 4e-6f * (rf + 1.0f), dx, dy);
}
// rf16 = (float)radius * 2^-16, hb = 0.5 - 4e-6 ((float)radius + 1)
PGG_HD void disk_offset_k(uint32_t ua, uint32_t ub, double radius, float rf16, float hb, int& dx, int& dy,
                          int* rechecks) {
  const float band = 0.5f - hb;
  const float rf = rf16 * 65536.0f;
#if defined(__CUDA_ARCH__) && PGG_EM_FAST
#if PGG_LOOP_TRIM
  // sqrt(u 2^-32) = sqrt(u) 2^-16 exactly: the scale joins the radius
  (void)rf;
  const float r = rf16 * f_sqrt_mufu((float)ua);
#else
  const float r = rf * f_sqrt(u01f(ua));
#endif
  const float th = (float)(int32_t)ub * 1.4629180792671596e-09f;  // 2 pi u - (u >= 1/2 ? 2 pi : 0)
  const float fx = r * __cosf(th), fy = r * __sinf(th);
  const float kM = 12582912.0f;  // 1.5 * 2^23: x + kM rounds x to the nearest integer (even on ties)
  const float tx = fx + kM, ty = fy + kM;
  const float rx = fx - (tx - kM), ry = fy - (ty - kM);
#if PGG_LOOP_TRIM
  if (fabsf(rx) > hb || fabsf(ry) > hb) {  // one compare on |r| per coordinate
#else
  if (0.5f - fabsf(rx) < band || 0.5f - fabsf(ry) < band) {
#endif
    if (rechecks) ++*rechecks;
    const Off2 o = disk_offset_d(ua, ub, radius);
    dx = o.x;
    dy = o.y;
    return;
  }
  dx = __float_as_int(tx) - 0x4B400000;
  dy = __float_as_int(ty) - 0x4B400000;
#else
  (void)band;
  const float r = rf * f_sqrt(u01f(ua));
  float s, c;
  sincos_turn(ub, &s, &c);
  const float fx = r * c, fy = r * s;
  const float ex = fabsf(fx - floorf(fx) - 0.5f);
  const float ey = fabsf(fy - floorf(fy) - 0.5f);
  if (ex < band || ey < band) {
    if (rechecks) ++*rechecks;
    const Off2 o = disk_offset_d(ua, ub, radius);
    dx = o.x;
    dy = o.y;
    return;
  }
  dx = (int)rintf(fx);
  dy = (int)rintf(fy);
#endif
}

// Per-pixel EM context: everything a record needs about its receiver.
// Built once per pixel (stage 1) and shared by the 8 lanes that process the
// pixel's candidate slots (stage 2).
struct EmSetup {
  V3<float> x;       // receiver position
  Frame<float> fr;   // orthonormal frame about n/|n|
  V3<float> n_raw;   // stored normal (float64 validity re-check)
  V3<float> wol;     // view in the local frame
  float alb_r, alb_g, alb_b;  // luminance-weighted albedo (0.2126 r, 0.7152 g, 0.0722 b)
  float a2, kappa, g1o;  // g1o = G1(cos_o) / (4 cos_o)
  float mx, my, il11, l21, il22;  // il11, il22 x c and l21 / c, c = sqrt(log2(e) / 2)
  float pg, qpi;                    // pi x (Gaussian normaliser), 1 - pi
  int flags;         // bit0 train this pixel, bit1 glossy, bit2 cos_o > 0
  int nb;            // neighbour budget N (mixture.py:324-328)
  uint64_t s0;       // EM stream (seed, frame, pixel, stream_id=1)
};

// standardised square coordinates z = L^-1 (q - mu) (scaled by c) of a record
PGG_HD void em_z(const EmSetup& S, float qx, float qy, float& z1, float& z2) {
#if PGG_GAUSS_FMA
  // z1 = qx il11 - mx il11, z2 = qy il22 - my il22 - (l21 il22) z1: three
  // fused multiply-adds on pre-multiplied per-pixel constants
  z1 = fmaf(qx, S.il11, -S.mx);
  z2 = fmaf(qy, S.il22, fmaf(-S.l21, z1, -S.my));
#else
  z1 = (qx - S.mx) * S.il11;
  z2 = ((qy - S.my) - S.l21 * z1) * S.il22;
#endif
}

// jump table: state after n LCG steps is J_MUL[n] * s + J_ADD[n], n = 0..37
// (every draw position of the 38-draw EM candidate block)
constexpr int JUMPS = 38;
#define PGG_J2(F, b) F(b + 0), F(b + 1)
#define PGG_J6(F, b) PGG_J2(F, b), PGG_J2(F, b + 2), PGG_J2(F, b + 4)
#define PGG_JTAB(F) PGG_J6(F, 0), PGG_J6(F, 6), PGG_J6(F, 12), PGG_J6(F, 18), PGG_J6(F, 24), PGG_J6(F, 30), \
    PGG_J2(F, 36)
#ifdef __CUDACC__
__constant__ uint64_t c_jmul[JUMPS] = {PGG_JTAB(pcg_jump_mul)};
__constant__ uint64_t c_jadd[JUMPS] = {PGG_JTAB(pcg_jump_add)};
#endif
PGG_HD void jump_tables(uint64_t* mul, uint64_t* add) {
  uint64_t m = 1, a = 0;
  for (int n = 0; n < JUMPS; ++n) {
    mul[n] = m;
    add[n] = a;
    m *= PCG_MUL;
    a = a * PCG_MUL + PCG_INC;
  }
}


// XSH-RR output of a state (without advancing it)
PGG_HD uint32_t pcg_out(uint64_t old) {
  const uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
  const uint32_t rot = (uint32_t)(old >> 59);
  return (xs >> rot) | (xs << ((32u - rot) & 31u));
}

// validity thresholds dist > 1e-9 and cos > 1e-9 decided in float64:
// returns the float64 receiver cosine (the reference's cos_r,
// guide_buffers.py:186-196) rounded to float32 for a valid record, -1
// otherwise.  Near the horizon the float32 cosine of the loop is ~6e-8
// absolute off (the position difference is rounded): a 0.6 % weight error
// at cos = 1e-5, which moved one 4K pixel's Gamma by 8e-4 relative where that
// record held the responsibility mass.
#ifndef PGG_GRAZE
#define PGG_GRAZE 1e-3f  // |cos| below which a record's cosine is re-evaluated in float64
#endif
#ifndef PGG_GRAZE_FIX
#define PGG_GRAZE_FIX 1
#endif
PGG_HD float record_cos_d_inl(float yx, float yy, float yz, V3<float> x, V3<float> n) {
  const V3<double> dd = cvt<double>(v3(yx, yy, yz)) - cvt<double>(x);
  const double dd2 = dot(dd, dd);
#if PGG_FAST_F64 && defined(__CUDA_ARCH__)
  const double c = dot(dd, cvt<double>(n)) * d_rsqrt(fmax(dd2, 1e-300));
#else
  const double c = dot(dd, cvt<double>(n)) / sqrt(fmax(dd2, 1e-300));
#endif
  return (dd2 > 1e-18 && c > 1e-9) ? (float)c : -1.0f;
}
PGG_COLD float record_cos_d(float yx, float yy, float yz, V3<float> x, V3<float> n) {
  const V3<double> dd = cvt<double>(v3(yx, yy, yz)) - cvt<double>(x);
  const double distd = sqrt(dot(dd, dd));
  const V3<double> omd = dd * (1.0 / fmax(distd, 1e-12));
  const double c = dot(omd, cvt<double>(n));
  return (distd > 1e-9 && c > 1e-9) ? (float)c : -1.0f;
}


// VPL accessors for the record loop: straight from global memory (L2), or
// from a shared-memory tile (own 32 x 8 block + EM halo) staged by TMA.
struct VplGlobal {
  static constexpr bool kZeroOOB = false;  // no padding: out-of-frame candidates must be tested
  const float* y;
  const float* L;
  int width, row0;
  int rows;  // rows held (bounds checks of checked builds)
  PGG_MHD float4 get_y(int cx, int cy) const { return y_at(index(cx, cy)); }
  PGG_MHD float4 get_L(int cx, int cy) const { return L_at(index(cx, cy)); }
  PGG_MHD int64_t index(int cx, int cy) const { return (int64_t)(cy - row0) * width + cx; }
  PGG_MHD int stride() const { return width; }
  PGG_MHD float4 y_at(int64_t i) const {
    PGG_CHK(CHK_VPL, i >= 0 && i < (int64_t)rows * width, i, rows);
    return ld4(y, i);
  }
  PGG_MHD float4 L_at(int64_t i) const {
    PGG_CHK(CHK_VPL, i >= 0 && i < (int64_t)rows * width, i, rows);
    return ld4(L, i);
  }
};
struct VplTile {
  static constexpr bool kZeroOOB = true;  // TMA zero-fills tile elements outside the frame
  const float4* y;  // shared memory, [rows][cols]
  const float4* L;
  int x0, y0, cols;  // frame coordinates of tile element (0, 0)
  PGG_MHD float4 get_y(int cx, int cy) const { return y[(cy - y0) * cols + (cx - x0)]; }
  PGG_MHD float4 get_L(int cx, int cy) const { return L[(cy - y0) * cols + (cx - x0)]; }
  PGG_MHD int index(int cx, int cy) const { return (cy - y0) * cols + (cx - x0); }
  PGG_MHD int stride() const { return cols; }
  PGG_MHD float4 y_at(int i) const { return y[i]; }
  PGG_MHD float4 L_at(int i) const { return L[i]; }
};

// The same tile through 32-bit shared-memory addresses (ld.shared.v4): one
// base register instead of two generic pointers, L at a fixed offset.
// Device-only (the host build reads VplGlobal).
struct VplTileS {
  static constexpr bool kZeroOOB = true;  // TMA zero-fills tile elements outside the frame
  uint32_t y;      // shared address of tile element (0, 0) of the y plane
  uint32_t off_l;  // byte offset of the L plane
  int x0, y0, cols;
  int n;           // elements per plane (bounds checks of checked builds)
  PGG_MHD static float4 lds(uint32_t a) {
    float4 v;
#ifdef __CUDA_ARCH__
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
#else
    (void)a;
    v = float4{0.f, 0.f, 0.f, 0.f};
#endif
    return v;
  }
  PGG_MHD int index(int cx, int cy) const { return (cy - y0) * cols + (cx - x0); }
  PGG_MHD int stride() const { return cols; }
  PGG_MHD float4 y_at(int i) const {
    PGG_CHK(CHK_TILE, i >= 0 && i < n, i, n);
    return lds(y + 16u * (uint32_t)i);
  }
  PGG_MHD float4 L_at(int i) const {
    PGG_CHK(CHK_TILE, i >= 0 && i < n, i, n);
    return lds(y + off_l + 16u * (uint32_t)i);
  }
  PGG_MHD float4 get_y(int cx, int cy) const { return y_at(index(cx, cy)); }
  PGG_MHD float4 get_L(int cx, int cy) const { return L_at(index(cx, cy)); }
};

// One training record (guide_buffers.py:186-230): receiver S, VPL (y, L).
// Returns the reference's geometric validity (dist > 1e-9, cos > 1e-9) and
// fills w (luminance weight), r (E-step responsibility) and the square
// point; kAll also evaluates records whose weight is known to be zero
// (view below the surface), which the accumulating path skips.
struct Rec {
  float w, r, qx, qy;
};

template <bool kAll, class VS>
PGG_HD bool em_eval(const EmSetup& S, const float4& vy, const VS& V, int cx, int cy, Rec& o) {
  const V3<float> d = v3(vy.x, vy.y, vy.z) - S.x;
  const float dist2 = dot(d, d);
  const float rinv = r_rsqrt(fmaxf(dist2, 1e-24f));
  const V3<float> om = d * rinv;
  const V3<float> dl = S.fr.to_local(om);
  float cr = dl.z;
  if (dist2 < 1e-12f || fabsf(dl.z) < PGG_GRAZE) {
    cr = record_cos_d(vy.x, vy.y, vy.z, S.x, S.n_raw);
    if (!(cr > 0.0f)) return false;
  } else if (!(dl.z > 1e-9f)) {
    return false;
  }
  const bool co_pos = (S.flags & 4) != 0;
  o.w = 0.0f;
  o.r = 0.0f;
  if (!co_pos && !kAll) return true;  // f = 0 and brdf_pdf = 0: zero weight
  float bp = 0.0f;
  if (co_pos) {
    const float4 lv = V.get_L(cx, cy);
    if (!(S.flags & 2)) {
      // Lambert: luminance(L albedo / pi) cos, pdf cos / pi (scene.py:269, 296)
      bp = PGG_LAMBERT_BP(cr);
      o.w = (lv.x * S.alb_r + lv.y * S.alb_g + lv.z * S.alb_b) * bp;
    } else {
      // GGX (scene.py:271-283, 298-307); G1(wo)/(4 cos_o) is a pixel constant
      const V3<float> hr = dl + S.wol;
      const float D = ggx_d_fast(S.a2, S.kappa, hr);
      bp = S.g1o * D;
      const float spec = bp * ggx_g1_fast(S.a2, cr);
      const float hi = fabsf(dot(hr, dl)) * m_rsqrt(fmaxf(dot(hr, hr), 1e-30f));
      const float t = fminf(fmaxf(1.0f - hi, 0.0f), 1.0f);
      const float t2 = t * t;
      const float f5 = t2 * t2 * t;
      // luma_c F_c = la_c + (luma_c - la_c) f5 (Schlick, F0 = albedo)
      const float kr = fmaf(kLumR - S.alb_r, f5, S.alb_r);
      const float kg = fmaf(kLumG - S.alb_g, f5, S.alb_g);
      const float kb = fmaf(kLumB - S.alb_b, f5, S.alb_b);
      // f cos = F D G1(wi) G1(wo) / (4 cos_i cos_o) * cos_i
      o.w = (lv.x * kr + lv.y * kg + lv.z * kb) * spec;
    }
    if (!kAll && !(isfinite(o.w) && o.w >= 0.0f)) return true;  // dropped by the M-step
  }
  dir_to_sq_f(dl, o.qx, o.qy);
  float z1, z2;
  em_z(S, o.qx, o.qy, z1, z2);
  const float num = S.pg * f_exp2(-(z1 * z1 + z2 * z2));
  const float den = num + S.qpi * bp;
  o.r = num * f_rcp(fmaxf(den, 1e-30f));  // den = 0 only with num = 0 -> r = 0
  return true;
}

// Accumulates w, w r, w r x, w r y, w r x^2, w r y^2, w r x y of one record,
// branch-light: the candidate's validity `ok` masks the sums instead of
// branching (a warp with mixed validity pays the full record either way),
// so the record and the next slot's draws form one schedulable block.
template <class VS, class IDX, class NRM>
PGG_HD void em_accumulate(const EmSetup& S, const float4& vy, const VS& V, IDX idx, bool ok, float* acc,
                          const NRM& n_raw) {
  const V3<float> d = v3(vy.x, vy.y, vy.z) - S.x;
  const float dist2 = dot(d, d);
#if PGG_EM_RAW_RSQRT
  const float rinv = m_rsqrt(fmaxf(dist2, 1e-24f));  // MUFU only (rel. error < 2^-22.9)
#else
  const float rinv = r_rsqrt(fmaxf(dist2, 1e-24f));
#endif
  const V3<float> dl = S.fr.to_local(d * rinv);
#if PGG_GRAZE_FIX
  // near-horizon records: the receiver cosine in float64 (weight and
  // Lambert pdf are linear in it; float32 is ~6e-8 absolute off)
  float cz = dl.z;
  if (ok && (dist2 < 1e-12f || fabsf(dl.z) < PGG_GRAZE)) {
#if PGG_GRAZE_FIX == 2
    cz = record_cos_d_inl(vy.x, vy.y, vy.z, S.x, n_raw());
#else
    cz = record_cos_d(vy.x, vy.y, vy.z, S.x, n_raw());  // stored normal, reloaded: not live in the loop
#endif
    ok = cz > 0.0f;
  } else {
    ok = ok && dl.z > 1e-9f;
  }
  const float cr = fmaxf(cz, 0.0f);
#else
  if (ok && (dist2 < 1e-12f || fabsf(dl.z) < 1e-6f)) {
    ok = record_cos_d(vy.x, vy.y, vy.z, S.x, n_raw()) > 0.0f;  // stored normal, reloaded: not live in the loop
  } else {
    ok = ok && dl.z > 1e-9f;
  }
  const float cr = fmaxf(dl.z, 0.0f);
#endif
  const float4 lv = V.L_at(idx);
  // Lambert (scene.py:269, 296)
  float bp = PGG_LAMBERT_BP(cr);
  // S.alb_c = luminance weight x albedo: la = luminance(L albedo)
  const float la = lv.x * S.alb_r + lv.y * S.alb_g + lv.z * S.alb_b;
  float w = la * bp;
  if (S.flags & 2) {
    // GGX (scene.py:271-283, 298-307); G1(wo)/(4 cos_o) is a pixel constant
    const V3<float> hr = dl + S.wol;
    const float D = ggx_d_fast(S.a2, S.kappa, hr);
    bp = S.g1o * D;
    const float spec = bp * ggx_g1_fast(S.a2, cr);
    const float hi = fabsf(dot(hr, dl)) * m_rsqrt(fmaxf(dot(hr, hr), 1e-30f));
    const float t = fminf(fmaxf(1.0f - hi, 0.0f), 1.0f);
    const float t2 = t * t;
    const float f5 = t2 * t2 * t;
#if PGG_GGX_LA
    // luminance(L F), Schlick F_c = albedo_c + (1 - albedo_c) f5, as
    // la + (luminance(L) - la) f5: no per-pixel (lum_c - albedo_c) invariants
    const float ll = fmaf(kLumB, lv.z, fmaf(kLumG, lv.y, kLumR * lv.x));
    w = fmaf(ll - la, f5, la) * spec;
#else
    const float kr = fmaf(kLumR - S.alb_r, f5, S.alb_r);
    const float kg = fmaf(kLumG - S.alb_g, f5, S.alb_g);
    const float kb = fmaf(kLumB - S.alb_b, f5, S.alb_b);
    w = (lv.x * kr + lv.y * kg + lv.z * kb) * spec;
#endif
  }
  // non-finite or zero weights are dropped / add nothing (mixture.py:291)
#if PGG_W_UMASK && defined(__CUDA_ARCH__)
  // 0 < w <= FLT_MAX as one unsigned compare of the bits (negative, +-0,
  // inf and NaN fall outside)
  ok = ok && (__float_as_uint(w) - 1u) < 0x7F7FFFFFu;
#else
  ok = ok && w > 0.0f && w <= 3.402823466e38f;
#endif
  float qx, qy;
  dir_to_sq_f(dl, qx, qy);
  float z1, z2;
  em_z(S, qx, qy, z1, z2);
#if PGG_LOOP_TRIM
  // -(z1^2 + z2^2) with the negation folded into the products (same value);
  // r is finite, so the masked w r is 0 * r = 0 as before
  const float num = S.pg * f_exp2(fmaf(-z1, z1, -(z2 * z2)));
  const float den = num + S.qpi * bp;
  const float r = num * f_rcp(fmaxf(den, 1e-30f));
  const float wv = ok ? w : 0.0f;
  const float wr = wv * r;
#else
  const float num = S.pg * f_exp2(-(z1 * z1 + z2 * z2));
  const float den = num + S.qpi * bp;
  const float r = num * f_rcp(fmaxf(den, 1e-30f));
  const float wv = ok ? w : 0.0f;
  const float wr = ok ? w * r : 0.0f;
#endif
  // qx, qy are finite even for masked records (dir_to_sq_f clamps, NaN -> 0)
  acc[0] += wv;
  acc[1] += wr;
  acc[2] = fmaf(wr, qx, acc[2]);
  acc[3] = fmaf(wr, qy, acc[3]);
  acc[4] = fmaf(wr * qx, qx, acc[4]);
  acc[5] = fmaf(wr * qy, qy, acc[5]);
  acc[6] = fmaf(wr * qx, qy, acc[6]);
}

template <class VS>
PGG_HD void em_record(const EmSetup& S, const float4& vy, const VS& V, int cx, int cy, float* acc) {
  em_accumulate(S, vy, V, V.index(cx, cy), true, acc, [&]() { return S.n_raw; });
}

// EM sums of one pixel over its candidate slots 0..N-1.  Slot 0 is the
// pixel's own VPL; slot s >= 1 draws u1 = draw s-1 and u2 = draw 18+s of
// the pixel's stream (the reference draws all 19 u1 then all 19 u2,
// guide_buffers.py:144-145) and rounds the disk offset.
// kFull: the VPL planes cover the whole frame (every launch but a row band's),
// so no candidate can miss them and no halo misses are counted.
#ifndef PGG_EM_PAIR
// 2: all candidate slots in pairs (0, 1), (2, 3), ... with the record math in
// packed FP32 (FFMA2 / FMUL2 / FADD2, pgg_pair.cuh).  Measured on B200 (1080p
// bench): 5.7 % fewer warp-instructions but issue utilisation 70.5 -> 63.7 %
// (long-scoreboard, instruction-fetch and math-pipe-throttle stalls up),
// 0.4967 vs 0.4725 ms -- slower, also at 2 blocks/SM without spills
// (0.4966 ms); off.  DESIGN.md section 4.
#define PGG_EM_PAIR 0
#endif
#if PGG_GAUSS_FMA && PGG_EM_PAIR == 2
#error "PGG_GAUSS_FMA changes the EmSetup constants the pair path reads"
#endif
}  // namespace pgg
#include "pgg_pair.cuh"
namespace pgg {

#ifdef __CUDA_ARCH__
// disk_offset_k for two slots: the float32 arithmetic packed (FFMA2 / FADD2),
// sin / cos / sqrt per slot on MUFU, the same guard band and float64
// re-decision per slot
PGG_PI void disk_offset_k2(uint32_t ua0, uint32_t ub0, uint32_t ua1, uint32_t ub1, double radius, float rf16,
                           float hb, int& dx0, int& dy0, int& dx1, int& dy1, int* rechecks0 = nullptr,
                           int* rechecks1 = nullptr) {
  const F2 r = f2(f_sqrt_mufu((float)ua0), f_sqrt_mufu((float)ua1)) * rf16;
  const float th0 = (float)(int32_t)ub0 * 1.4629180792671596e-09f;
  const float th1 = (float)(int32_t)ub1 * 1.4629180792671596e-09f;
  const F2 fx = r * f2(__cosf(th0), __cosf(th1)), fy = r * f2(__sinf(th0), __sinf(th1));
  const float kM = 12582912.0f;  // 1.5 * 2^23: x + kM rounds x to the nearest integer (even on ties)
  const F2 tx = fx + kM, ty = fy + kM;
  const F2 rx = fx - (tx - kM), ry = fy - (ty - kM);
  if (fabsf(lo(rx)) > hb || fabsf(lo(ry)) > hb) {
    if (rechecks0) ++*rechecks0;
    const Off2 o = disk_offset_d(ua0, ub0, radius);
    dx0 = o.x;
    dy0 = o.y;
  } else {
    dx0 = __float_as_int(lo(tx)) - 0x4B400000;
    dy0 = __float_as_int(lo(ty)) - 0x4B400000;
  }
  if (fabsf(hi(rx)) > hb || fabsf(hi(ry)) > hb) {
    if (rechecks1) ++*rechecks1;
    const Off2 o = disk_offset_d(ua1, ub1, radius);
    dx1 = o.x;
    dy1 = o.y;
  } else {
    dx1 = __float_as_int(hi(tx)) - 0x4B400000;
    dy1 = __float_as_int(hi(ty)) - 0x4B400000;
  }
}
#endif

template <bool kFull = false, class VS>
PGG_HD void em_partial(const PassArgs& A, const VS& V, const EmSetup& S, int x, int y, const uint64_t* jmul,
                       const uint64_t* jadd, float* acc) {
  const pgg_config& C = A.cfg;
  const unsigned W = (unsigned)C.width, H = (unsigned)C.height;
  const int vr0 = A.vpl.row0;
  const unsigned vrows = (unsigned)A.vpl.rows;
  if (S.nb <= 0) return;
  if (!kFull && (unsigned)(y - vr0) >= vrows) {  // own row outside the VPL rows: every slot misses
    count_miss(A.halo_misses);
    return;
  }
  const auto base = V.index(x, y);
  const int stride = V.stride();
  const auto n_raw = [&]() {
    const float4 nd = ld4(A.cur.nd, (int64_t)(y - A.cur.row0) * C.width + x);
    return v3(nd.x, nd.y, nd.z);
  };
#if defined(__CUDA_ARCH__) && PGG_EM_PAIR == 2
  {
    // every slot in pairs (0, 1), (2, 3), ...; slot 0 is the pixel's own VPL
    // (offset 0, no draws): the streams start one step before draws 0 / 19
    constexpr bool kNoBounds2 = PGG_TILE_OOB && kFull && VS::kZeroOOB;
    uint64_t sa = (S.s0 - PCG_INC) * PCG_MUL_INV;
    uint64_t sb = jmul[18] * S.s0 + jadd[18];
    int misses = 0;
    F2 acc2[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) acc2[k] = f2s(0.0f);
    for (int s = 0; s < S.nb; s += 2) {
      const uint32_t ua0 = pcg_out(sa), ub0 = pcg_out(sb);
      sa = sa * PCG_MUL + PCG_INC;
      sb = sb * PCG_MUL + PCG_INC;
      const uint32_t ua1 = pcg_out(sa), ub1 = pcg_out(sb);
      sa = sa * PCG_MUL + PCG_INC;
      sb = sb * PCG_MUL + PCG_INC;
      const bool has1 = s + 1 < S.nb;
      int dx0, dy0, dx1, dy1;
      disk_offset_k2(ua0, ub0, ua1, ub1, C.radius, A.em_radius16, A.em_hband, dx0, dy0, dx1, dy1);
      if (s == 0) dx0 = dy0 = 0;  // self
      const int cx0 = x + dx0, cy0 = y + dy0, cx1 = x + dx1, cy1 = y + dy1;
      const bool inf0 = kNoBounds2 || ((unsigned)cx0 < W && (unsigned)cy0 < H);
      const bool inf1 = kNoBounds2 || ((unsigned)cx1 < W && (unsigned)cy1 < H);
      const bool inv0 = kFull || (unsigned)(cy0 - vr0) < vrows;
      const bool inv1 = kFull || (unsigned)(cy1 - vr0) < vrows;
      if (!kFull) misses += ((inf0 && !inv0) ? 1 : 0) + ((has1 && inf1 && !inv1) ? 1 : 0);
      bool ok0 = inf0 && inv0;
      bool ok1 = has1 && inf1 && inv1;
      const auto idx0 = (kNoBounds2 || ok0) ? base + (decltype(base))dy0 * stride + dx0 : base;
      const auto idx1 = (kNoBounds2 || ok1) ? base + (decltype(base))dy1 * stride + dx1 : base;
      const float4 vy0 = V.y_at(idx0), vy1 = V.y_at(idx1);
      ok0 = ok0 && vy0.w != 0.0f;  // VPL invalid or not BRDF-strategy
      ok1 = ok1 && vy1.w != 0.0f;
      em_accumulate2(S, vy0, vy1, V, idx0, idx1, ok0, ok1, acc2, n_raw);
    }
#pragma unroll
    for (int k = 0; k < 7; ++k) acc[k] += lo(acc2[k]) + hi(acc2[k]);
    if (!kFull && misses) count_miss(A.halo_misses, misses);
    return;
  }
#endif
  {
    const float4 vy = V.y_at(base);
    em_accumulate(S, vy, V, base, vy.w != 0.0f, acc, n_raw);
  }
  int s = 1;
  if (s >= S.nb) return;
  uint64_t sa = jmul[0] * S.s0 + jadd[0];     // draw 0: u1 of slot 1
#if !PGG_SB_JUMP
  uint64_t sb = jmul[19] * S.s0 + jadd[19];   // draw 19: u2 of slot 1
#endif
  int misses = 0;  // in-frame candidates outside the supplied VPL rows (halo misses)
  // whole-frame VPLs staged by TMA: every candidate (|d| <= R) lies in the
  // tile and those outside the frame read TMA's zero fill, i.e. an invalid
  // VPL (w = 0) -- the reference's "out of frame -> unused" without a test
  constexpr bool kNoBounds = PGG_TILE_OOB && kFull && VS::kZeroOOB;
  for (; s < S.nb; ++s) {
#if PGG_SB_JUMP
    // the u2 stream is the u1 stream 19 draws ahead: one live state, the
    // other derived per slot (the same instruction count as a second step)
    const uint64_t sb = lcg_jump<J19_MUL, J19_ADD>(sa);
    const uint32_t ua = pcg_out(sa), ub = pcg_out(sb);
    sa = lcg_step(sa);
#else
    const uint32_t ua = pcg_out(sa), ub = pcg_out(sb);
    sa = lcg_step(sa);
    sb = lcg_step(sb);
#endif
    int dx, dy;
    disk_offset_k(ua, ub, C.radius, A.em_radius16, A.em_hband, dx, dy);
    const int cx = x + dx, cy = y + dy;
    const bool in_frame = kNoBounds || ((unsigned)cx < W && (unsigned)cy < H);
    const bool in_vpl = kFull || (unsigned)(cy - vr0) < vrows;
    if (!kFull) misses += (in_frame && !in_vpl) ? 1 : 0;
    bool ok = in_frame && in_vpl;
    const auto idx = (kNoBounds || ok) ? base + (decltype(base))dy * stride + dx : base;
    const float4 vy = V.y_at(idx);
    ok = ok && vy.w != 0.0f;  // VPL invalid or not BRDF-strategy
    em_accumulate(S, vy, V, idx, ok, acc, n_raw);
  }
  if (!kFull && misses) count_miss(A.halo_misses, misses);
}

// Online M-step (mixture.py:276-321) in float64 from the float32 sums.
PGG_HD void m_step_apply(const float4& g0, const float4& g1, const float* acc, int kmax, float4& o0, float4& o1) {
  o0 = g0;
  o1 = g1;
  const float sw = acc[0], swr = acc[1];
  if (!(sw > 0.0f)) return;  // no information: unchanged, k unchanged
  const double k = g1.w;
#if PGG_FAST_F64 && defined(__CUDA_ARCH__)
  // reciprocals to ~1 ulp of float64; the results are rounded to float32
  const double eta = d_rcp(fmin(k + 1.0, (double)kmax));  // = max(1/(k+1), 1/kMax)
  const double om1 = 1.0 - eta;
  const double ed = eta * d_rcp(fmax((double)swr, 1e-8));
#else
  const double eta = 1.0 / fmin(k + 1.0, (double)kmax);  // = max(1/(k+1), 1/kMax): division is monotone
  const double om1 = 1.0 - eta;
  const double ed = eta / fmax((double)swr, 1e-8);
#endif
  o0.x = (float)(om1 * g0.x + ed * (double)acc[2]);
  o0.y = (float)(om1 * g0.y + ed * (double)acc[3]);
  o0.z = (float)(om1 * g0.z + ed * (double)acc[4]);
  o0.w = (float)(om1 * g0.w + ed * (double)acc[5]);
  o1.x = (float)(om1 * g1.x + ed * (double)acc[6]);
  o1.y = (float)(om1 * g1.y + eta * (double)swr);
#if PGG_FAST_F64 && defined(__CUDA_ARCH__)
  const double pit = (double)swr * d_rcp(fmax((double)sw, 1e-8));
#else
  const double pit = (double)swr / fmax((double)sw, 1e-8);
#endif
  o1.z = (float)fmin(fmax(om1 * g1.z + eta * pit, 0.05), 0.95);
  o1.w = (float)(k + 1.0);
}

constexpr double GAUSS_C = 0.84932180028801904272;  // sqrt(log2(e) / 2)

// EM context of a valid pixel from its G-buffer planes, frame and lobe
PGG_HD void em_setup(const float4& pr, const float4& va, const float4& am, bool glossy, const PixelFrame& pf,
                     const LobeF& L, float k, int kmax, uint64_t s0, EmSetup& S) {
  const double r2d = (double)pr.w * (double)pr.w;
  const float alpha = (float)fmax(r2d, 1e-6);
  S.x = v3(pr.x, pr.y, pr.z);
  S.fr = pf.fr;
  S.wol = pf.wol;
  S.alb_r = kLumR * va.w;
  S.alb_g = kLumG * am.x;
  S.alb_b = kLumB * am.y;
  S.a2 = alpha * alpha;
  S.kappa = kappa_world(pf.om_nn, S.a2);
  S.g1o = glossy ? ggx_g1(S.a2, fabsf(pf.wol.z)) / fmaxf(4.0f * pf.wol.z, 1e-30f) : 0.0f;
#if PGG_PI_FOLD
  S.g1o *= 3.14159265358979323846f;
#endif
  // exponent -(z1^2 + z2^2)/2 evaluated as exp2(-(z1'^2 + z2'^2)) with z' = c z
  const double il11c = (double)L.il11 * GAUSS_C, il22c = (double)L.il22 * GAUSS_C;
  const double l21c = (double)L.l21 * (1.0 / GAUSS_C);  // constant reciprocal: no float64 division
  S.il11 = (float)il11c;
  S.il22 = (float)il22c;
#if PGG_GAUSS_FMA
  // em_z's fused form: mu and the cross term pre-multiplied
  S.mx = (float)((double)L.mx * il11c);
  S.my = (float)((double)L.my * il22c);
  S.l21 = (float)(l21c * il22c);
#else
  S.mx = L.mx;
  S.my = L.my;
  S.l21 = (float)l21c;
#endif
  S.pg = L.pi * L.gnorm;
#if PGG_PI_FOLD
  S.qpi = (1.0f - L.pi) * K<float>::inv_pi;
#else
  S.qpi = 1.0f - L.pi;
#endif
  S.flags = 1 | (glossy ? 2 : 0) | (pf.co_pos ? 4 : 0);
  S.nb = neighbor_budget(k, kmax);
#ifdef PGG_PROF_NO_EM
  S.nb = 0;  // measurement-only build: stage 1 alone
#endif
  S.s0 = s0;
}

// ---------------------------------------------------------------------------
// Stage 1 of a pixel (own band, y_local yl): Gamma (reprojected or read),
// optional reprojection output, depth-0 samples, and the EM context.
// Returns false when the pixel has nothing to train (invalid G-buffer:
// Gamma passes through unchanged, guide_buffers.py:279-280).

// Depth-0 samples of one pixel's spp lanes (ptrace.py:161-220, 449-475).
PGG_HD void sample_pixel(const PassArgs& A, int64_t own, uint64_t pix, const PixelFrame& pf, bool glossy,
                         float rough, const LobeF& L, const float4& g0, const float4& g1) {
  const pgg_config& C = A.cfg;
#ifdef PGG_PROF_NO_GUIDE
  const bool guided = false;  // measurement-only build
#else
  const bool guided = (!glossy || (double)rough >= C.rough_min_guide) && g1.w >= 1.0f;
#endif
  CholD cd;
  cd.mx = g0.x;
  cd.my = g0.y;
  cd.m2xx = g0.z;
  cd.m2yy = g0.w;
  cd.m2xy = g1.x;
  cd.from_floats = 0;
#if PGG_SHARE_LANE_HASH
  const uint64_t hpix = splitmix64(pix);
#endif
  for (int s = 0; s < C.spp; ++s) {
#if PGG_SHARE_LANE_HASH
    // spp == 1: the sampling lane key equals the pixel key of the EM stream
    uint64_t st = (C.spp == 1 ? splitmix64(C.key_sample ^ hpix)
                              : splitmix64(C.key_sample ^ splitmix64(pix * (uint64_t)C.spp + (uint64_t)s))) *
                      PCG_MUL + PCG_INC;
#else
    uint64_t st = pcg_lane(C.key_sample, pix * (uint64_t)C.spp + (uint64_t)s);
#endif
    if (C.nee_draws == 3) {
      st = st * J3_MUL + J3_ADD;  // the three NEE draws as one jump
    } else {
      for (int k = 0; k < C.nee_draws; ++k) st = st * PCG_MUL + PCG_INC;
    }
    const LaneOut o = sample_lane(pf, glossy, rough, guided, L, cd, st);
    st4(A.smp.dir, own * C.spp + s, f4(o.wi.x, o.wi.y, o.wi.z, o.pdf));
    A.smp.tag[own * C.spp + s] = (uint8_t)(o.gauss | (o.valid << 1) | (o.draws << 2));
  }
}

// kStage: 0 every stage the arguments select (the fused pass), 1 reprojection
// + depth-0 sampling only (no EM code), 2 EM only (no reprojection or
// sampling code; Gamma from gin).
template <int kStage = 0>
PGG_HD bool pixel_stage(const PassArgs& A, int x, int yl, float4& g0, float4& g1, EmSetup& S) {
  const pgg_config& C = A.cfg;
  const int W = C.width;
  const int y = C.row0 + yl;
  const int64_t own = (int64_t)yl * W + x;
  const int64_t ci = (int64_t)(y - A.cur.row0) * W + x;
  PGG_CHK(CHK_CUR, y - A.cur.row0 >= 0 && y - A.cur.row0 < A.cur.rows && x >= 0 && x < W, y, x);
  PGG_CHK(CHK_OUT, yl >= 0 && yl < C.rows, yl, C.rows);
  const uint8_t fl = ldu8(A.cur.flags, ci);
  const bool valid = fl & 1;
  // all own-pixel loads in flight together (invalid pixels are ~10 %)
  const float4 nd = ld4(A.cur.nd, ci);
  const float4 pr = ld4(A.cur.pr, ci);
  const float4 am = ld4(A.cur.am, ci);
  const float4 va = ld4(A.cur.va, ci);
#ifdef PGG_PROF_NO_REPROJ
  if (false) {  // measurement-only build
#else
  if (kStage != 2 && A.has_prev) {
#endif
    reproject_px(A, x, y, fl, nd, pr, am, g0, g1);
  } else {
    const int64_t gi = (int64_t)(y - A.gin.row0) * W + x;
    PGG_CHK(CHK_GIN, y - A.gin.row0 >= 0 && y - A.gin.row0 < A.gin.rows, y, A.gin.row0);
    g0 = ld4(A.gin.g0, gi);
    g1 = ld4(A.gin.g1, gi);
  }
  if (A.has_grep) {
    st4(A.grep.g0, own, g0);
    st4(A.grep.g1, own, g1);
  }
  S.flags = 0;
  S.nb = 0;
  if (!A.has_smp && !A.has_vpl) return false;
  if (!valid) {
    if (kStage != 2 && A.has_smp) {
      for (int s = 0; s < C.spp; ++s) {
        st4(A.smp.dir, own * C.spp + s, f4(0, 0, 0, 0));
        A.smp.tag[own * C.spp + s] = 0;
      }
    }
    return false;
  }
  const LobeF L = make_lobe(g0.x, g0.y, g0.z, g0.w, g1.x, g1.z);
  const V3<float> n = v3(nd.x, nd.y, nd.z);
  const V3<float> wo = v3(va.x, va.y, va.z);
  const float rough = pr.w;
  const bool glossy = (fl & 4) != 0;
  const PixelFrame pf = make_pixel_frame(n, wo);
  const uint64_t pix = (uint64_t)y * (uint64_t)W + (uint64_t)x;
#if PGG_SHARE_LANE_HASH
  const uint64_t hpix = splitmix64(pix);  // rng.make_streams' lane hash, shared by both streams
#endif
#ifdef PGG_PROF_NO_SMP
  if (false) {  // measurement-only build
#else
  if (kStage != 2 && A.has_smp) {
#endif
    sample_pixel(A, own, pix, pf, glossy, rough, L, g0, g1);
  }
  if (kStage == 1 || !A.has_vpl) return false;
#if PGG_SHARE_LANE_HASH
  em_setup(pr, va, am, glossy, pf, L, g1.w, C.k_max, splitmix64(C.key_train ^ hpix) * PCG_MUL + PCG_INC, S);
#else
  em_setup(pr, va, am, glossy, pf, L, g1.w, C.k_max, pcg_lane(C.key_train, pix), S);
#endif
  S.n_raw = n;
  // view below the surface: every record has f = 0, so the batch carries no
  // weight and the reference leaves Gamma (and k) unchanged -- skip the EM
  return pf.co_pos;
}

// Record dump of one pixel for gather_training_batch (guide_buffers.py:234-259):
// Gamma from gamma_in, EM stream state `s0` supplied by the caller; writes
// per slot (qx, qy, w, valid) for slots < N, valid = 0 beyond.
PGG_HD void em_dump(const PassArgs& A, int x, int y, uint64_t s0, const uint64_t* jmul, const uint64_t* jadd,
                    float* out) {
  const pgg_config& C = A.cfg;
  const int W = C.width, H = C.height;
  for (int s = 0; s < SLOTS; ++s) {
    out[4 * s + 0] = 0.5f;
    out[4 * s + 1] = 0.5f;
    out[4 * s + 2] = 0.0f;
    out[4 * s + 3] = 0.0f;
  }
  const int64_t ci = (int64_t)(y - A.cur.row0) * W + x;
  const uint8_t fl = ldu8(A.cur.flags, ci);
  if (!(fl & 1)) return;
  const float4 nd = ld4(A.cur.nd, ci), pr = ld4(A.cur.pr, ci), va = ld4(A.cur.va, ci), am = ld4(A.cur.am, ci);
  const int64_t gi = (int64_t)(y - A.gin.row0) * W + x;
  const float4 g0 = ld4(A.gin.g0, gi), g1 = ld4(A.gin.g1, gi);
  const LobeF L = make_lobe(g0.x, g0.y, g0.z, g0.w, g1.x, g1.z);
  const PixelFrame pf = make_pixel_frame(v3(nd.x, nd.y, nd.z), v3(va.x, va.y, va.z));
  EmSetup S;
  em_setup(pr, va, am, (fl & 4) != 0, pf, L, g1.w, C.k_max, s0, S);
  S.n_raw = v3(nd.x, nd.y, nd.z);
  const VplGlobal V{A.vpl.y, A.vpl.L, W, A.vpl.row0, A.vpl.rows};
  for (int s = 0; s < S.nb; ++s) {
    int cx = x, cy = y;
    if (s > 0) {
      const uint32_t ua = pcg_out(jmul[s - 1] * s0 + jadd[s - 1]);
      const uint32_t ub = pcg_out(jmul[s + 18] * s0 + jadd[s + 18]);
      int dx, dy;
      disk_offset(ua, ub, C.radius, dx, dy);
      cx += dx;
      cy += dy;
      if (cx < 0 || cx >= W || cy < 0 || cy >= H) continue;
    }
    if (cy < A.vpl.row0 || cy >= A.vpl.row0 + A.vpl.rows) continue;
    const float4 vy = V.get_y(cx, cy);
    if (vy.w == 0.0f) continue;
    Rec o;
    if (!em_eval<true>(S, vy, V, cx, cy, o)) continue;
    out[4 * s + 0] = o.qx;
    out[4 * s + 1] = o.qy;
    out[4 * s + 2] = o.w;
    out[4 * s + 3] = 1.0f;
  }
}

// Whole pixel on one thread (host build of the device code path).
PGG_HD void pass_pixel(const PassArgs& A, int x, int yl, const uint64_t* jmul, const uint64_t* jadd) {
  float4 g0, g1;
  EmSetup S;
  const bool train = pixel_stage(A, x, yl, g0, g1, S);
  if (!A.has_vpl) return;
  const int64_t own = (int64_t)yl * A.cfg.width + x;
  float4 o0 = g0, o1 = g1;
  if (train) {
    float acc[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const VplGlobal V{A.vpl.y, A.vpl.L, A.cfg.width, A.vpl.row0, A.vpl.rows};
    em_partial(A, V, S, x, A.cfg.row0 + yl, jmul, jadd, acc);
    m_step_apply(g0, g1, acc, A.cfg.k_max, o0, o1);
  }
  st4(A.gout.g0, own, o0);
  st4(A.gout.g1, own, o1);
}

}  // namespace pgg
