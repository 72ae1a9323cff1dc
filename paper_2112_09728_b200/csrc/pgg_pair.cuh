// pgg_pair.cuh — two EM candidate slots per thread in packed FP32 (sm_100a).
//
// Blackwell issues fma/mul/add.f32x2 (SASS FFMA2 / FMUL2 / FADD2) as ONE
// warp-instruction for two float32 operations per thread, with a scalar
// register broadcast as either operand.  The record loop of the pass is
// issue-bound, so slots s and s+1 of a pixel run side
// by side: every float32 add / mul / fma of the record math is one packed
// instruction for both; the MUFU transcendentals, compares, selects and the
// 64-bit PCG arithmetic stay per slot.  Per-pixel constants (EmSetup) are
// scalars broadcast into the packed operations.  The arithmetic per slot is
// em_accumulate's (pgg_pass.cuh; guide_buffers.py:186-231, mixture.py:262-
// 273), evaluated with the same formulas; the two slots' sums are kept as
// separate partial sums and added once per pixel.
//
// Device-only: the host build (pgg_hostcheck.cpp) runs the scalar loop.
#pragma once

#ifdef __CUDA_ARCH__

#include <stdint.h>

namespace pgg {

#define PGG_PI __device__ __forceinline__

struct F2 {
  uint64_t v;  // (lo, hi) = (slot s, slot s + 1)
};

PGG_PI F2 f2(float a, float b) {
  F2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(a), "f"(b));
  return r;
}
PGG_PI F2 f2s(float a) { return f2(a, a); }  // broadcast: ptxas folds it into the packed operand
PGG_PI float lo(F2 a) {
  float x, y;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a.v));
  return x;
}
PGG_PI float hi(F2 a) {
  float x, y;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a.v));
  return y;
}
PGG_PI F2 operator+(F2 a, F2 b) {
  F2 r;
  asm("add.ftz.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
PGG_PI F2 operator-(F2 a, F2 b) {
  F2 r;
  asm("sub.ftz.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
PGG_PI F2 operator*(F2 a, F2 b) {
  F2 r;
  asm("mul.ftz.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
  return r;
}
PGG_PI F2 fma2(F2 a, F2 b, F2 c) {
  F2 r;
  asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return r;
}
PGG_PI F2 operator+(F2 a, float b) { return a + f2s(b); }
PGG_PI F2 operator-(F2 a, float b) { return a - f2s(b); }
PGG_PI F2 operator-(float a, F2 b) { return f2s(a) - b; }
PGG_PI F2 operator*(F2 a, float b) { return a * f2s(b); }
PGG_PI F2 fma2(F2 a, float b, F2 c) { return fma2(a, f2s(b), c); }
PGG_PI F2 fma2(F2 a, F2 b, float c) { return fma2(a, b, f2s(c)); }
PGG_PI F2 fma2(F2 a, float b, float c) { return fma2(a, f2s(b), f2s(c)); }
// per-slot (scalar) helpers
template <class Fn>
PGG_PI F2 each(F2 a, Fn f) {
  return f2(f(lo(a)), f(hi(a)));
}
PGG_PI F2 max2(F2 a, float b) { return f2(fmaxf(lo(a), b), fmaxf(hi(a), b)); }
PGG_PI F2 rsqrt2(F2 a) { return f2(rsqrtf(lo(a)), rsqrtf(hi(a))); }
PGG_PI F2 rcp2(F2 a) { return f2(f_rcp(lo(a)), f_rcp(hi(a))); }
PGG_PI F2 ex22(F2 a) { return f2(f_exp2(lo(a)), f_exp2(hi(a))); }
PGG_PI F2 sel2(bool p0, bool p1, F2 a, float b) { return f2(p0 ? lo(a) : b, p1 ? hi(a) : b); }

struct V3F2 {
  F2 x, y, z;
};

// rsqrt refined by one Newton step (r_rsqrt, pgg_math.cuh)
PGG_PI F2 r_rsqrt2(F2 x) {
  const F2 y = rsqrt2(x);
  const F2 e = f2s(1.0f) - (x * y) * y;
  return fma2(y * 0.5f, e, y);
}

// dir_to_sq_f on two directions (pgg_math.cuh; sgmap.py:67-77 then 41-56)
PGG_PI void dir_to_sq2(const V3F2& v, F2& sx, F2& sy) {
  const F2 rs = rsqrt2(max2(v.z + 1.0f, 1e-30f));
  const F2 x = v.x * rs, y = v.y * rs;
  const float ax0 = fabsf(lo(x)), ay0 = fabsf(lo(y)), ax1 = fabsf(hi(x)), ay1 = fabsf(hi(y));
  const F2 rho2 = fma2(x, x, y * y);
  const F2 rho = rho2 * rsqrt2(max2(rho2, 1e-36f));
  const F2 t = f2(fminf(ax0, ay0), fminf(ax1, ay1)) * rcp2(f2(fmaxf(fmaxf(ax0, ay0), 1e-36f), fmaxf(fmaxf(ax1, ay1), 1e-36f)));
  const F2 u2 = t * t;
  F2 p = fma2(u2, -0.005162642803043127f, 0.02783750370144844f);
  p = fma2(p, u2, f2s(-0.07119078189134598f));
  p = fma2(p, u2, f2s(0.12276896089315414f));
  p = fma2(p, u2, f2s(-0.17709042131900787f));
  p = fma2(p, u2, f2s(0.25396761298179626f));
  p = fma2(p, u2, f2s(-0.4243689775466919f));
  p = fma2(p, u2, f2s(1.2732386589050293f));
  const F2 u = (t * p) * rho;
  const bool xd0 = ax0 >= ay0, xd1 = ax1 >= ay1;
  const F2 a = f2(copysignf(xd0 ? lo(rho) : lo(u), lo(x)), copysignf(xd1 ? hi(rho) : hi(u), hi(x)));
  const F2 b = f2(copysignf(xd0 ? lo(u) : lo(rho), lo(y)), copysignf(xd1 ? hi(u) : hi(rho), hi(y)));
  const F2 qa = fma2(a, 0.5f, 0.5f), qb = fma2(b, 0.5f, 0.5f);
  sx = f2(__saturatef(lo(qa)), __saturatef(hi(qa)));
  sy = f2(__saturatef(lo(qb)), __saturatef(hi(qb)));
}

// Records of two candidate slots of one receiver (em_accumulate, pgg_pass.cuh),
// summed into the packed partial sums acc2[0..6] (lo: slot s, hi: slot s+1).
template <class VS, class NRM>
PGG_PI void em_accumulate2(const EmSetup& S, const float4& vy0, const float4& vy1, const VS& V, int idx0, int idx1,
                           bool ok0, bool ok1, F2* acc2, const NRM& n_raw) {
  const V3F2 d{f2(vy0.x, vy1.x) - S.x.x, f2(vy0.y, vy1.y) - S.x.y, f2(vy0.z, vy1.z) - S.x.z};
  const F2 dist2 = fma2(d.x, d.x, fma2(d.y, d.y, d.z * d.z));
  const F2 rinv = r_rsqrt2(max2(dist2, 1e-24f));
  const V3F2 om{d.x * rinv, d.y * rinv, d.z * rinv};
  const Frame<float>& fr = S.fr;
  const V3F2 dl{fma2(om.x, fr.t.x, fma2(om.y, fr.t.y, om.z * fr.t.z)),
                fma2(om.x, fr.b.x, fma2(om.y, fr.b.y, om.z * fr.b.z)),
                fma2(om.x, fr.n.x, fma2(om.y, fr.n.y, om.z * fr.n.z))};
  const float dz0 = lo(dl.z), dz1 = hi(dl.z);
  if (ok0 && (lo(dist2) < 1e-12f || fabsf(dz0) < 1e-6f)) {
    ok0 = record_cos_d(vy0.x, vy0.y, vy0.z, S.x, n_raw()) > 0.0f;
  } else {
    ok0 = ok0 && dz0 > 1e-9f;
  }
  if (ok1 && (hi(dist2) < 1e-12f || fabsf(dz1) < 1e-6f)) {
    ok1 = record_cos_d(vy1.x, vy1.y, vy1.z, S.x, n_raw()) > 0.0f;
  } else {
    ok1 = ok1 && dz1 > 1e-9f;
  }
  const F2 cr = f2(fmaxf(dz0, 0.0f), fmaxf(dz1, 0.0f));
  const float4 lv0 = V.L_at(idx0), lv1 = V.L_at(idx1);
  // Lambert (scene.py:269, 296)
  F2 bp = cr * K<float>::inv_pi;
  F2 w = f2(lv0.x * S.alb_r + lv0.y * S.alb_g + lv0.z * S.alb_b, lv1.x * S.alb_r + lv1.y * S.alb_g + lv1.z * S.alb_b) * bp;
  if (S.flags & 2) {
    // GGX (scene.py:271-283, 298-307); G1(wo)/(4 cos_o) is a pixel constant
    const V3F2 hr{dl.x + S.wol.x, dl.y + S.wol.y, dl.z + S.wol.z};
    // ggx_d_fast
    const F2 c2 = hr.z * hr.z;
    const F2 s2 = fma2(hr.x, hr.x, hr.y * hr.y);
    const F2 n2 = s2 + c2;
    const F2 dq = fma2(c2, S.kappa, s2) * rcp2(n2);
    const F2 dd = f2(lo(n2) > 0.0f ? lo(dq) : 1.0f, hi(n2) > 0.0f ? hi(dq) : 1.0f);
    const F2 D = rcp2(max2((dd * K<float>::pi) * dd, 1e-30f)) * S.a2;
    bp = D * S.g1o;
    // ggx_g1_fast(a2, cr)
    const F2 ga = fma2(cr * (1.0f - S.a2), cr, f2s(S.a2));
    const F2 gs = f2(lo(ga) > 0.0f ? lo(ga) * rsqrtf(lo(ga)) : 0.0f, hi(ga) > 0.0f ? hi(ga) * rsqrtf(hi(ga)) : 0.0f);
    const F2 g1 = (cr * 2.0f) * rcp2(max2(cr + gs, 1e-30f));
    const F2 spec = bp * g1;
    const F2 hd = fma2(hr.x, dl.x, fma2(hr.y, dl.y, hr.z * dl.z));
    const F2 hh = fma2(hr.x, hr.x, fma2(hr.y, hr.y, hr.z * hr.z));
    const F2 hrs = rsqrt2(max2(hh, 1e-30f));
    const F2 hi_ = f2(fabsf(lo(hd)) * lo(hrs), fabsf(hi(hd)) * hi(hrs));
    const F2 tq = f2s(1.0f) - hi_;
    const F2 t = f2(fminf(fmaxf(lo(tq), 0.0f), 1.0f), fminf(fmaxf(hi(tq), 0.0f), 1.0f));
    const F2 t2 = t * t;
    const F2 f5 = (t2 * t2) * t;
    const F2 kr = fma2(f5, 0.2126f - S.alb_r, f2s(S.alb_r));
    const F2 kg = fma2(f5, 0.7152f - S.alb_g, f2s(S.alb_g));
    const F2 kb = fma2(f5, 0.0722f - S.alb_b, f2s(S.alb_b));
    w = f2(lv0.x * lo(kr) + lv0.y * lo(kg) + lv0.z * lo(kb), lv1.x * hi(kr) + lv1.y * hi(kg) + lv1.z * hi(kb)) * spec;
  }
  // non-finite or zero weights are dropped / add nothing (mixture.py:291)
  ok0 = ok0 && lo(w) > 0.0f && lo(w) <= 3.402823466e38f;
  ok1 = ok1 && hi(w) > 0.0f && hi(w) <= 3.402823466e38f;
  F2 qx, qy;
  dir_to_sq2(dl, qx, qy);
  const F2 z1 = (qx - S.mx) * S.il11;
  const F2 z2 = ((qy - S.my) - z1 * S.l21) * S.il22;
  const F2 num = ex22(f2s(0.0f) - fma2(z1, z1, z2 * z2)) * S.pg;
  const F2 den = fma2(bp, S.qpi, num);
  const F2 r = num * rcp2(max2(den, 1e-30f));
  const F2 wv = sel2(ok0, ok1, w, 0.0f);
  const F2 wr = wv * r;
  // qx, qy are finite even for masked records (clamped to [0,1])
  const F2 wrx = wr * qx, wry = wr * qy;
  acc2[0] = acc2[0] + wv;
  acc2[1] = acc2[1] + wr;
  acc2[2] = acc2[2] + wrx;
  acc2[3] = acc2[3] + wry;
  acc2[4] = fma2(wrx, qx, acc2[4]);
  acc2[5] = fma2(wry, qy, acc2[5]);
  acc2[6] = fma2(wrx, qy, acc2[6]);
}

}  // namespace pgg

#endif  // __CUDA_ARCH__
