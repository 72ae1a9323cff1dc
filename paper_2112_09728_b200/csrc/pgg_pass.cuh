// pgg_pass.cuh — per-pixel / per-lane bodies of the guiding pass.
//
// The CUDA kernels (pgg_kernels.cu) are thin grid loops over these
// functions; the test-only host build (pgg_hostcheck.cpp) runs the very same
// bodies on the CPU so the device formulas can be checked against the oracle
// without a GPU.  Reference semantics cited per stage.
#pragma once

#include "pgg.h"
#include "pgg_math.cuh"

namespace pgg {

constexpr int SLOTS = 20;                 // guide_buffers.py:20
constexpr int GAUSS_TRIES = 16;           // mixture.py:28
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
};

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

PGG_HD void count_miss(int32_t* c) {
  if (!c) return;
#ifdef __CUDA_ARCH__
  atomicAdd(c, 1);
#else
  *c += 1;
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

// Mean rotation between the previous and current tangent frames
// (guide_buffers.py:117-133), in float64: M2 is carried unrotated, so the
// covariance M2 - mu mu^T of the next lobe cancels and amplifies any error
// in the rotated mean ~1/Sigma-fold; float64 keeps the float32-rounded mean
// identical to the reference's in all but boundary-rounding cases.
PGG_HD void rotate_or_reject(const V3<float>& np_, const V3<float>& nc, float mux, float muy, bool& keep,
                             float& ox, float& oy) {
  keep = true;
  ox = mux;
  oy = muy;
  // identical normals: the rotation is the identity and the float64 round
  // trip of an interior mean rounds back to the same float32
  if (np_.x == nc.x && np_.y == nc.y && np_.z == nc.z && mux >= 1e-6f && mux <= 1.0f - 1e-6f &&
      muy >= 1e-6f && muy <= 1.0f - 1e-6f)
    return;
  const V3<double> dl = sq_to_dir<double>((double)mux, (double)muy);
  V3<double> dc = make_frame(cvt<double>(nc)).to_local(make_frame(cvt<double>(np_)).to_world(dl));
  if (dc.z < 0.0) {
    keep = false;
    return;
  }
  double sx, sy;
  dir_to_sq<double>(dc, sx, sy);
  ox = (float)sx;
  oy = (float)sy;
}

PGG_HD void reproject_px(const PassArgs& A, int x, int y, uint8_t fl, const float4& nd, const float4& pr,
                         const float4& am, float4& g0, float4& g1) {
  const pgg_config& C = A.cfg;
  init_gamma(g0, g1);
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
  if (!(ldu8(A.prev.flags, sp) & 1)) return;
  // depth and normal gates in float64, reference operation order
  const double dx = rsub((double)pr.x, C.prev_cam[0]);
  const double dy = rsub((double)pr.y, C.prev_cam[1]);
  const double dz = rsub((double)pr.z, C.prev_cam[2]);
  const double de = sqrt(radd(radd(rmul(dx, dx), rmul(dy, dy)), rmul(dz, dz)));
  const float4 ndp = ld4(A.prev.nd, sp);
  if (!(fabs(rsub((double)ndp.w, de)) < rmul(C.depth_rel_tol, fmax(de, 1e-12)))) return;
  const double ndot = radd(radd(rmul((double)ndp.x, (double)nd.x), rmul((double)ndp.y, (double)nd.y)),
                           rmul((double)ndp.z, (double)nd.z));
  if (!(ndot > C.normal_dot_min)) return;
  const int64_t gi = (int64_t)(sy - A.gin.row0) * C.width + sx;
  float4 p0 = ld4(A.gin.g0, gi);
  const float4 p1 = ld4(A.gin.g1, gi);
  if (C.rotate_mean) {
    bool keep;
    float ox, oy;
    rotate_or_reject(v3(ndp.x, ndp.y, ndp.z), v3(nd.x, nd.y, nd.z), p0.x, p0.y, keep, ox, oy);
    if (!keep) return;
    p0.x = ox;
    p0.y = oy;
  }
  g0 = p0;
  g1 = p1;
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

PGG_HD bool near_edge(float v) { return fabsf(v) < 1e-5f || fabsf(1.0f - v) < 1e-5f; }

// local-frame BRDF draw with its validity (wl.z > 1e-9, wo.z > 0); float64
// re-evaluation for the VNDF rim case and near the z threshold
PGG_HD V3<float> brdf_draw_local(const Mat<float>& mf, float alpha, const V3<float>& wol, bool co_pos, uint32_t a,
                                 uint32_t b, bool& ok) {
  bool ill;
  V3<float> wl = brdf_sample_local<float>(mf, alpha, wol, a, b, ill);
  if (ill || fabsf(wl.z) < 1e-6f) {
    const Mat<double> md{mf.glossy, (double)mf.a2, (double)mf.kappa};
    bool ill_d;
    const V3<double> wd = brdf_sample_local<double>(md, (double)alpha, cvt<double>(wol), a, b, ill_d);
    ok = wd.z > 1e-9 && co_pos;
    return cvt<float>(wd);
  }
  ok = wl.z > 1e-9f && co_pos;
  return wl;
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
    return o;
  }
  const uint32_t uz = pcg_next(st);
  bool acc = false;
  float sx = 0.0f, sy = 0.0f;
  if (u01d(uz) < (double)L.pi) {
    for (int t = 0; t < GAUSS_TRIES; ++t) {
      const uint32_t a = pcg_next(st), b = pcg_next(st);
      float z0, z1;
      box_muller_f(a, b, z0, z1);
      const float px = L.mx + L.l11 * z0;
      const float py = L.my + L.l21 * z0 + L.l22 * z1;
      bool inside;
      if (near_edge(px) || near_edge(py)) {
        double l11, l21, l22, d0, d1;
        cd.get(l11, l21, l22);
        box_muller_d(a, b, d0, d1);
        const double qx = radd((double)L.mx, rmul(l11, d0));
        const double qy = radd(radd((double)L.my, rmul(l21, d0)), rmul(l22, d1));
        inside = qx >= 0.0 && qx <= 1.0 && qy >= 0.0 && qy <= 1.0;
      } else {
        inside = px >= 0.0f && px <= 1.0f && py >= 0.0f && py <= 1.0f;
      }
      if (inside) {
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
    dl = brdf_draw_local(mf, alpha, wol, co_pos, a, b, ok);
  }
  o.gauss = acc ? 1 : 0;
  o.pdf = 0.0f;
  if (ok) {
    const float bp = co_pos ? brdf_pdf_local(mf, dl, wol) : 0.0f;
    float qx = sx, qy = sy;
    if (!acc) {
      V3<float> dz = dl;
      dz.z = fmaxf(dz.z, 0.0f);
      dir_to_sq<float>(dz, qx, qy);
    }
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
PGG_HD void disk_offset(uint32_t ua, uint32_t ub, double radius, int& dx, int& dy) {
  const float r = (float)radius * sqrtf(u01f(ua));
  float s, c;
  m_sincospi(2.0f * u01f(ub), &s, &c);
  const float fx = r * c, fy = r * s;
  const float band = 4e-6f * ((float)radius + 1.0f);
  const float ex = fabsf(fabsf(fx - floorf(fx)) - 0.5f);
  const float ey = fabsf(fabsf(fy - floorf(fy)) - 0.5f);
  if (ex < band || ey < band) {
    const double rd = radius * sqrt(u01d(ua));
    const double ang = 2.0 * K<double>::pi * u01d(ub);
    dx = (int)rint(rd * cos(ang));
    dy = (int)rint(rd * sin(ang));
    return;
  }
  dx = (int)rintf(fx);
  dy = (int)rintf(fy);
}

struct Px {
  V3<float> x, n, wo;
  float alb_r, alb_g, alb_b;
  float rough;
  bool glossy;
};

PGG_HD void train_px(const PassArgs& A, int x, int y, const Px& P, const PixelFrame& pf, const LobeF& L,
                     const float4& g0, const float4& g1, float4& o0, float4& o1) {
  const pgg_config& C = A.cfg;
  const int W = C.width, H = C.height;
  const int nb = neighbor_budget(g1.w, C.k_max);
  const double r2d = (double)P.rough * (double)P.rough;
  const float alpha = (float)fmax(r2d, 1e-6);
  const float a2 = alpha * alpha;
  const float kap = kappa_world(pf.om_nn, a2);
  const Frame<float>& fr = pf.fr;
  const V3<float>& wol = pf.wol;
  const float co = wol.z;
  const bool co_pos = pf.co_pos;
  // luminance-weighted albedo (diffuse f = albedo / pi)
  const float kr = 0.2126f * P.alb_r, kg = 0.7152f * P.alb_g, kb = 0.0722f * P.alb_b;
  const float g1o = P.glossy ? ggx_g1(a2, fabsf(co)) : 0.0f;
  const uint64_t pix = (uint64_t)y * (uint64_t)W + (uint64_t)x;
  uint64_t sa = pcg_lane(C.key_train, pix);
  uint64_t sb = sa * J19_MUL + J19_ADD;
  float sw = 0.f, swr = 0.f, sx = 0.f, sy = 0.f, sxx = 0.f, syy = 0.f, sxy = 0.f;
  const int vr0 = A.vpl.row0, vr1 = A.vpl.row0 + A.vpl.rows;
  for (int slot = 0; slot < nb; ++slot) {
    int cx = x, cy = y;
    if (slot > 0) {
      const uint32_t ua = pcg_next(sa);
      const uint32_t ub = pcg_next(sb);
      int dx, dy;
      disk_offset(ua, ub, C.radius, dx, dy);
      cx += dx;
      cy += dy;
      if (cx < 0 || cx >= W || cy < 0 || cy >= H) continue;
    }
    if (cy < vr0 || cy >= vr1) {
      count_miss(A.halo_misses);
      continue;
    }
    const int64_t vi = (int64_t)(cy - vr0) * W + cx;
    const float4 vy = ld4(A.vpl.y, vi);
    if (vy.w == 0.0f) continue;  // VPL invalid or not BRDF-strategy
    const V3<float> d = v3(vy.x, vy.y, vy.z) - P.x;
    const float dist = sqrtf(dot(d, d));
    const V3<float> om = d * (1.0f / fmaxf(dist, 1e-12f));
    const V3<float> dl = fr.to_local(om);
    if (dist < 1e-6f || fabsf(dl.z) < 1e-6f) {
      const V3<double> dd = cvt<double>(v3(vy.x, vy.y, vy.z)) - cvt<double>(P.x);
      const double distd = sqrt(dot(dd, dd));
      const V3<double> omd = dd * (1.0 / fmax(distd, 1e-12));
      if (!(distd > 1e-9 && dot(omd, cvt<double>(P.n)) > 1e-9)) continue;
    } else if (!(dl.z > 1e-9f)) {
      continue;
    }
    const float cr = dl.z;
    const float4 lv = ld4(A.vpl.L, vi);
    float w, bp;
    if (!P.glossy) {
      w = co_pos ? (lv.x * kr + lv.y * kg + lv.z * kb) * (cr * K<float>::inv_pi) : 0.0f;
      bp = co_pos ? cr * K<float>::inv_pi : 0.0f;
    } else if (co_pos) {
      const V3<float> hr = dl + wol;
      const float D = ggx_d(a2, kap, hr);
      const float spec = D * ggx_g1(a2, cr) * g1o / fmaxf(4.0f * cr * co, 1e-30f);
      const float hi = fabsf(dot(hr, dl)) * m_rsqrt(fmaxf(dot(hr, hr), 1e-30f));
      const float t = fminf(fmaxf(1.0f - hi, 0.0f), 1.0f);
      const float t2 = t * t;
      const float f5 = t2 * t2 * t;
      const float fr_ = P.alb_r + (1.0f - P.alb_r) * f5;
      const float fg_ = P.alb_g + (1.0f - P.alb_g) * f5;
      const float fb_ = P.alb_b + (1.0f - P.alb_b) * f5;
      w = ((lv.x * fr_) * 0.2126f + (lv.y * fg_) * 0.7152f + (lv.z * fb_) * 0.0722f) * (spec * cr);
      bp = g1o * D / fmaxf(4.0f * co, 1e-30f);
    } else {
      w = 0.0f;
      bp = 0.0f;
    }
    if (!(isfinite(w) && w >= 0.0f)) continue;
    float qx, qy;
    dir_to_sq<float>(dl, qx, qy);
    const float g = gauss_sr(L, qx, qy);
    const float num = L.pi * g;
    const float den = num + (1.0f - L.pi) * bp;
    const float r = den > 0.0f ? num / den : 0.0f;
    const float wr = w * r;
    sw += w;
    swr += wr;
    sx = fmaf(wr, qx, sx);
    sy = fmaf(wr, qy, sy);
    sxx = fmaf(wr * qx, qx, sxx);
    syy = fmaf(wr * qy, qy, syy);
    sxy = fmaf(wr * qx, qy, sxy);
  }
  o0 = g0;
  o1 = g1;
  if (!(sw > 0.0f)) return;  // no information: unchanged, k unchanged
  const double k = g1.w;
  const double eta = fmax(1.0 / (k + 1.0), 1.0 / (double)C.k_max);
  const double om1 = 1.0 - eta;
  const double den = fmax((double)swr, 1e-8);
  o0.x = (float)(om1 * g0.x + eta * ((double)sx / den));
  o0.y = (float)(om1 * g0.y + eta * ((double)sy / den));
  o0.z = (float)(om1 * g0.z + eta * ((double)sxx / den));
  o0.w = (float)(om1 * g0.w + eta * ((double)syy / den));
  o1.x = (float)(om1 * g1.x + eta * ((double)sxy / den));
  o1.y = (float)(om1 * g1.y + eta * (double)swr);
  const double pit = (double)swr / fmax((double)sw, 1e-8);
  o1.z = (float)fmin(fmax(om1 * g1.z + eta * pit, 0.05), 0.95);
  o1.w = (float)(k + 1.0);
}

// ---------------------------------------------------------------------------
// the fused per-pixel body; y_local indexes the call's own band

PGG_HD void pass_pixel(const PassArgs& A, int x, int yl) {
  const pgg_config& C = A.cfg;
  const int W = C.width;
  const int y = C.row0 + yl;
  const int64_t own = (int64_t)yl * W + x;
  const int64_t ci = (int64_t)(y - A.cur.row0) * W + x;
  const uint8_t fl = ldu8(A.cur.flags, ci);
  const bool valid = fl & 1;
  float4 nd = f4(0, 0, 1, 0), pr = f4(0, 0, 0, 0), am = f4(0, 0, 0, 0);
  if (valid) {
    nd = ld4(A.cur.nd, ci);
    pr = ld4(A.cur.pr, ci);
    am = ld4(A.cur.am, ci);
  }
  float4 g0, g1;
  if (A.has_prev) {
    reproject_px(A, x, y, fl, nd, pr, am, g0, g1);
  } else {
    const int64_t gi = (int64_t)(y - A.gin.row0) * W + x;
    g0 = ld4(A.gin.g0, gi);
    g1 = ld4(A.gin.g1, gi);
  }
  if (A.has_grep) {
    st4(A.grep.g0, own, g0);
    st4(A.grep.g1, own, g1);
  }
  if (!A.has_smp && !A.has_vpl) return;
  if (!valid) {
    if (A.has_smp) {
      for (int s = 0; s < C.spp; ++s) {
        st4(A.smp.dir, own * C.spp + s, f4(0, 0, 0, 0));
        A.smp.tag[own * C.spp + s] = 0;
      }
    }
    if (A.has_vpl) {
      st4(A.gout.g0, own, g0);
      st4(A.gout.g1, own, g1);
    }
    return;
  }
  const LobeF L = make_lobe(g0.x, g0.y, g0.z, g0.w, g1.x, g1.z);
  const float4 va = ld4(A.cur.va, ci);
  Px P;
  P.x = v3(pr.x, pr.y, pr.z);
  P.n = v3(nd.x, nd.y, nd.z);
  P.wo = v3(va.x, va.y, va.z);
  P.alb_r = va.w;
  P.alb_g = am.x;
  P.alb_b = am.y;
  P.rough = pr.w;
  P.glossy = (fl & 4) != 0;
  const PixelFrame pf = make_pixel_frame(P.n, P.wo);
  if (A.has_smp) {
    const bool guided = (!P.glossy || (double)P.rough >= C.rough_min_guide) && g1.w >= 1.0f;
    CholD cd;
    cd.mx = g0.x;
    cd.my = g0.y;
    cd.m2xx = g0.z;
    cd.m2yy = g0.w;
    cd.m2xy = g1.x;
    cd.from_floats = 0;
    const uint64_t pix = (uint64_t)y * (uint64_t)W + (uint64_t)x;
    for (int s = 0; s < C.spp; ++s) {
      uint64_t st = pcg_lane(C.key_sample, pix * (uint64_t)C.spp + (uint64_t)s);
      for (int k = 0; k < C.nee_draws; ++k) st = st * PCG_MUL + PCG_INC;
      const LaneOut o = sample_lane(pf, P.glossy, P.rough, guided, L, cd, st);
      st4(A.smp.dir, own * C.spp + s, f4(o.wi.x, o.wi.y, o.wi.z, o.pdf));
      A.smp.tag[own * C.spp + s] = (uint8_t)(o.gauss | (o.valid << 1));
    }
  }
  if (A.has_vpl) {
    float4 o0, o1;
    train_px(A, x, y, P, pf, L, g0, g1, o0, o1);
    st4(A.gout.g0, own, o0);
    st4(A.gout.g1, own, o1);
  }
}

}  // namespace pgg
