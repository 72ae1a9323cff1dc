// pgg_math.cuh — scalar math of the screen-space guiding pass.
//
// One source for the device (sm_100a) and for the test-only host build
// (csrc/pgg_hostcheck.cpp, compiled with g++ -ffp-contract=off).  Every
// function is templated on the scalar type T: the hot path instantiates it
// in float, and the few decisions that must agree with the float64 reference
// exactly (candidate-offset rint, Box-Muller acceptance, rotated-mean
// hemisphere test, record validity) are re-evaluated in double inside a
// guard band around the threshold.
//
// Reference semantics (file:line under /root/reference/pkg/src/pgtrace):
//   PCG32 + SplitMix key chain ........ rng.py:10-55
//   concentric/Lambert map, ONB ....... sgmap.py:21-115
//   GGX / Lambert eval, pdf, sample ... scene.py:247-380
//   lobe, truncation mass, pdfs ....... mixture.py:62-190
#pragma once

#include <stdint.h>
#include <vector_types.h>

#ifdef __CUDACC__
#define PGG_HD __host__ __device__ __forceinline__
#define PGG_MHD __host__ __device__ __forceinline__
#define PGG_COLD __host__ __device__ __noinline__
#else
#include <math.h>
#define PGG_HD static inline
#define PGG_MHD inline
#define PGG_COLD static
#endif

namespace pgg {

// ---------------------------------------------------------------------------
// scalar wrappers (float / double overloads, device intrinsics vs libm)

PGG_HD float m_sqrt(float x) { return sqrtf(x); }
PGG_HD double m_sqrt(double x) { return sqrt(x); }
PGG_HD float m_rsqrt(float x) {
#ifdef __CUDA_ARCH__
  return rsqrtf(x);
#else
  return 1.0f / sqrtf(x);
#endif
}
PGG_HD float m_exp(float x) { return expf(x); }
// fast float32 variants for the hot loops (device intrinsics, ~2 ulp)
PGG_HD float f_exp(float x) {
#ifdef __CUDA_ARCH__
  return __expf(x);
#else
  return expf(x);
#endif
}
PGG_HD float f_exp2(float x) {
#ifdef __CUDA_ARCH__
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#else
  return exp2f(x);
#endif
}
PGG_HD float f_rcp(float x) {
#ifdef __CUDA_ARCH__
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#else
  return 1.0f / x;
#endif
}
PGG_HD float f_div(float a, float b) {
#ifdef __CUDA_ARCH__
  return __fdividef(a, b);
#else
  return a / b;
#endif
}
PGG_HD float f_sin(float x) {
#ifdef __CUDA_ARCH__
  return __sinf(x);
#else
  return sinf(x);
#endif
}
// rsqrt and division refined by one Newton step (~1 ulp) for the
// accuracy-sensitive record mapping (square point -> Gaussian exponent)
PGG_HD float r_rsqrt(float x) {
#ifdef __CUDA_ARCH__
  const float y = rsqrtf(x);
  const float e = fmaf(-(x * y), y, 1.0f);
  return fmaf(0.5f * y, e, y);
#else
  return 1.0f / sqrtf(x);
#endif
}
PGG_HD float r_div(float a, float b) {
#ifdef __CUDA_ARCH__
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(b));
  const float q = a * r;
  return fmaf(r, fmaf(-b, q, a), q);
#else
  return a / b;
#endif
}

// sqrt via rsqrt (~2 ulp), 0 -> 0
// sqrt.approx (one MUFU.SQRT; relative error ~2^-22) for non-negative x
PGG_HD float f_sqrt_mufu(float x) {
#ifdef __CUDA_ARCH__
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
#else
  return sqrtf(x);
#endif
}
PGG_HD float f_sqrt(float x) {
#ifdef __CUDA_ARCH__
  return x > 0.0f ? x * rsqrtf(x) : 0.0f;
#else
  return sqrtf(x);
#endif
}

// sin and cos of 2 pi u / 2^32 for a raw 32-bit draw: quadrant from the top
// bits (exact), the remainder in [-pi/4, pi/4) by degree-9/8 polynomials
// (max error 1.3e-10 before float32 rounding).  Reference: 2 pi u2 angles
// of pg/guide_buffers.py:147, pg/mixture.py:189, pg/scene.py:313,334.
PGG_HD void sincos_turn(uint32_t u, float* s, float* c) {
  const uint32_t v = u + 0x20000000u;
  const uint32_t q = v >> 30;
  const int32_t f = (int32_t)(v & 0x3FFFFFFFu) - 0x20000000;
  const float th = (float)f * 1.4629180792671596e-09f;  // (pi/2) / 2^30
  const float uu = th * th;
  float ps = 2.7155285907043094e-06f;
  ps = fmaf(ps, uu, -0.0001983892565139517f);
  ps = fmaf(ps, uu, 0.008333327385762281f);
  ps = fmaf(ps, uu, -0.1666666660556111f);
  ps = fmaf(ps, uu, 0.9999999999826111f);
  const float s0 = th * ps;
  float pc = 2.4401924905735495e-05f;
  pc = fmaf(pc, uu, -0.0013886863579152262f);
  pc = fmaf(pc, uu, 0.04166662507354549f);
  pc = fmaf(pc, uu, -0.49999999704175707f);
  const float c0 = fmaf(pc, uu, 0.9999999999668368f);
  const float ss = (q & 1u) ? c0 : s0;
  const float cc = (q & 1u) ? s0 : c0;
  *s = (q & 2u) ? -ss : ss;
  *c = ((q + 1u) & 2u) ? -cc : cc;
}
PGG_HD void sincos_turn(uint32_t u, double* s, double* c) {
  const double ang = 2.0 * 3.14159265358979323846 * ((double)u * 2.3283064365386963e-10);
  *s = sin(ang);
  *c = cos(ang);
}

// atan on |t| <= 1: odd minimax polynomial t P(t^2), max error 5.8e-9
PGG_HD float atan_unit(float t) {
  const float u = t * t;
  float p = 0.0024566648549691015f;
  p = fmaf(p, u, -0.014401109845298344f);
  p = fmaf(p, u, 0.03978079996771651f);
  p = fmaf(p, u, -0.0723481905704511f);
  p = fmaf(p, u, 0.10498926387366457f);
  p = fmaf(p, u, -0.14161223468972228f);
  p = fmaf(p, u, 0.19985905886585464f);
  p = fmaf(p, u, -0.3333259696770105f);
  p = fmaf(p, u, 0.9999998863709554f);
  return t * p;
}
PGG_HD double atan_unit(double t) { return atan(t); }
PGG_HD float q_div(float a, float b) { return f_div(a, b); }
PGG_HD double q_div(double a, double b) { return a / b; }
PGG_HD double m_exp(double x) { return exp(x); }
PGG_HD float m_log(float x) { return logf(x); }
PGG_HD double m_log(double x) { return log(x); }
PGG_HD float m_log1p(float x) { return log1pf(x); }
PGG_HD double m_log1p(double x) { return log1p(x); }
PGG_HD float m_atan(float x) { return atanf(x); }
PGG_HD double m_atan(double x) { return atan(x); }
PGG_HD float m_abs(float x) { return fabsf(x); }
PGG_HD double m_abs(double x) { return fabs(x); }
PGG_HD float m_max(float a, float b) { return fmaxf(a, b); }
PGG_HD double m_max(double a, double b) { return fmax(a, b); }
PGG_HD float m_min(float a, float b) { return fminf(a, b); }
PGG_HD double m_min(double a, double b) { return fmin(a, b); }
PGG_HD float m_copysign(float a, float b) { return copysignf(a, b); }
PGG_HD double m_copysign(double a, double b) { return copysign(a, b); }
PGG_HD float m_rint(float x) { return rintf(x); }
PGG_HD double m_rint(double x) { return rint(x); }
PGG_HD float m_clamp01(float x) { return fminf(fmaxf(x, 0.0f), 1.0f); }
PGG_HD double m_clamp01(double x) { return fmin(fmax(x, 0.0), 1.0); }
PGG_HD bool m_isfinite(float x) { return isfinite(x); }
PGG_HD bool m_isfinite(double x) { return isfinite(x); }

// square roots on the sampler's float paths (Lambert lift, Box-Muller
// radius): MUFU-based on the device when PGG_SMP_SQRT_FAST (~1e-7 relative,
// inside the acceptance guard band and the direction tolerance)
#ifndef PGG_SMP_SQRT_FAST
#define PGG_SMP_SQRT_FAST 1
#endif
PGG_HD float smp_sqrt(float x) {
#if defined(__CUDA_ARCH__) && PGG_SMP_SQRT_FAST
  return f_sqrt(x);
#else
  return m_sqrt(x);
#endif
}
PGG_HD double smp_sqrt(double x) { return m_sqrt(x); }

// sin/cos of pi*x (exact argument scaling on the device)
#ifndef PGG_SMP_MUFU_TRIG
#define PGG_SMP_MUFU_TRIG 1  // concentric-map sin/cos on MUFU (abs error < 2^-20.5): 0.5387 -> 0.5364 ms
#endif
#ifndef PGG_SMP_MUFU_LOG
#define PGG_SMP_MUFU_LOG 1  // Box-Muller ln u (u < 1/2) on lg2.approx: 0.5387 -> 0.5360 ms
#endif
#ifndef PGG_SMP_LN_UNIFIED
#define PGG_SMP_LN_UNIFIED 1
#endif
PGG_HD void m_sincospi(float x, float* s, float* c) {
#if defined(__CUDA_ARCH__) && PGG_SMP_MUFU_TRIG
  const float a = 3.14159265358979323846f * x;  // |x| <= 3/4 (concentric map)
  *s = __sinf(a);
  *c = __cosf(a);
#elif defined(__CUDA_ARCH__)
  sincospif(x, s, c);
#else
  const double a = 3.14159265358979323846 * (double)x;
  *s = (float)sin(a);
  *c = (float)cos(a);
#endif
}
PGG_HD void m_sincospi(double x, double* s, double* c) {
#ifdef __CUDA_ARCH__
  sincospi(x, s, c);
#else
  const double a = 3.14159265358979323846 * x;
  *s = sin(a);
  *c = cos(a);
#endif
}

// standard normal CDF
PGG_HD float m_ndtr(float x) {
#ifdef __CUDA_ARCH__
  return normcdff(x);
#else
  return (float)(0.5 * erfc(-(double)x * 0.70710678118654752440));
#endif
}
PGG_HD double m_ndtr(double x) {
#ifdef __CUDA_ARCH__
  return normcdf(x);
#else
  return 0.5 * erfc(-x * 0.70710678118654752440);
#endif
}

// float64 ops that must not be contracted into FMAs (bitwise agreement with
// NumPy's separately rounded * and +)
PGG_HD double rmul(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
PGG_HD double radd(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
PGG_HD double rsub(double a, double b) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}

PGG_HD double rdiv(double a, double b) { return a / b; }  // IEEE round-to-nearest in float64

template <class T> struct K {
  static constexpr T pi = T(3.14159265358979323846);
  static constexpr T inv_pi = T(0.31830988618379067154);
  static constexpr T inv_2pi = T(0.15915494309189533577);
};

// ---------------------------------------------------------------------------
// PCG32 streams (rng.py:10-55)

constexpr uint64_t PCG_MUL = 6364136223846793005ULL;
constexpr uint64_t PCG_INC = 1442695040888963407ULL;
// PCG_MUL^-1 mod 2^64 (Newton: each step doubles the correct low bits)
constexpr uint64_t inv_mod64(uint64_t a) {
  uint64_t x = a;  // a odd: a * a = 1 mod 8
  for (int i = 0; i < 5; ++i) x *= 2 - a * x;
  return x;
}
constexpr uint64_t PCG_MUL_INV = inv_mod64(PCG_MUL);
static_assert(PCG_MUL * PCG_MUL_INV == 1, "PCG multiplier inverse");

PGG_HD uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// lane state = mix(key ^ mix(lane)) after one warm-up LCG step; key is the
// per-(seed, frame, stream) prefix of the hash chain (rng.py:34-39)
PGG_HD uint64_t pcg_lane(uint64_t key, uint64_t lane) {
  return splitmix64(key ^ splitmix64(lane)) * PCG_MUL + PCG_INC;
}

// One LCG step s * PCG_MUL + PCG_INC (mod 2^64).  On the device the
// increment is added with carry-chained immediates (IADD3 / IADD3.X) instead
// of the 64-bit addend of IMAD.WIDE, which ptxas rematerialises into a
// register pair (two MOVs) on every step of the record loop.
#ifndef PGG_LCG_IMM
#define PGG_LCG_IMM 1
#endif
PGG_HD uint64_t lcg_step(uint64_t s) {
#if defined(__CUDA_ARCH__) && PGG_LCG_IMM
  uint64_t r;
  asm("{\n\t.reg .u64 m;\n\t.reg .u32 lo, hi;\n\t"
      "mul.lo.u64 m, %1, 6364136223846793005;\n\t"
      "mov.b64 {lo, hi}, m;\n\t"
      "add.cc.u32 lo, lo, 4150755663;\n\t"
      "addc.u32 hi, hi, 335903614;\n\t"
      "mov.b64 %0, {lo, hi};\n\t}"
      : "=l"(r)
      : "l"(s));
  return r;
#else
  return s * PCG_MUL + PCG_INC;
#endif
}
static_assert((PCG_INC & 0xFFFFFFFFull) == 4150755663ull && (PCG_INC >> 32) == 335903614ull, "PCG increment halves");

// s * M + C for compile-time (M, C) (a jump-ahead), carry-chained like lcg_step
template <uint64_t M, uint64_t C> PGG_HD uint64_t lcg_jump(uint64_t s) {
#if defined(__CUDA_ARCH__) && PGG_LCG_IMM
  uint64_t r;
  asm("{\n\t.reg .u64 m;\n\t.reg .u32 lo, hi;\n\t"
      "mul.lo.u64 m, %1, %2;\n\t"
      "mov.b64 {lo, hi}, m;\n\t"
      "add.cc.u32 lo, lo, %3;\n\t"
      "addc.u32 hi, hi, %4;\n\t"
      "mov.b64 %0, {lo, hi};\n\t}"
      : "=l"(r)
      : "l"(s), "n"(M), "n"((uint32_t)(C & 0xFFFFFFFFull)), "n"((uint32_t)(C >> 32)));
  return r;
#else
  return s * M + C;
#endif
}

PGG_HD uint32_t pcg_next(uint64_t& s) {
  const uint64_t old = s;
  s = lcg_step(old);
  const uint32_t xs = (uint32_t)(((old >> 18) ^ old) >> 27);
  const uint32_t rot = (uint32_t)(old >> 59);
  return (xs >> rot) | (xs << ((32u - rot) & 31u));
}

// n LCG steps collapsed into one affine map s -> mul*s + add
constexpr uint64_t pcg_jump_mul(unsigned n) {
  uint64_t m = 1;
  for (unsigned i = 0; i < n; ++i) m *= PCG_MUL;
  return m;
}
constexpr uint64_t pcg_jump_add(unsigned n) {
  uint64_t a = 0;
  for (unsigned i = 0; i < n; ++i) a = a * PCG_MUL + PCG_INC;
  return a;
}

PGG_HD float u01f(uint32_t u) { return (float)u * 2.3283064365386963e-10f; }
PGG_HD double u01d(uint32_t u) { return (double)u * 2.3283064365386963e-10; }

// ---------------------------------------------------------------------------
// 3-vectors

template <class T> struct V3 {
  T x, y, z;
};
template <class T> PGG_HD V3<T> v3(T x, T y, T z) { return V3<T>{x, y, z}; }
template <class T> PGG_HD T dot(const V3<T>& a, const V3<T>& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class T> PGG_HD V3<T> operator+(const V3<T>& a, const V3<T>& b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class T> PGG_HD V3<T> operator-(const V3<T>& a, const V3<T>& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class T> PGG_HD V3<T> operator*(const V3<T>& a, T s) { return {a.x * s, a.y * s, a.z * s}; }
template <class T> PGG_HD V3<T> cross(const V3<T>& a, const V3<T>& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
// Fast float64 reciprocal / reciprocal square root for values that are
// rounded to float32 afterwards: MUFU seed (rcp / rsqrt .approx.f64, ~2^-23)
// and two Newton steps (~1 ulp of float64) instead of the correctly rounded
// division / sqrt sequences with their slow-path branches.
#ifndef PGG_FAST_F64
#define PGG_FAST_F64 1
#endif
PGG_HD double d_rcp(double x) {
#if defined(__CUDA_ARCH__) && PGG_FAST_F64
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
#else
  return 1.0 / x;
#endif
}
PGG_HD double d_rsqrt(double x) {
#if defined(__CUDA_ARCH__) && PGG_FAST_F64
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return fma(y, fma(-h * y, y, 0.5), y);
#else
  return 1.0 / sqrt(x);
#endif
}

// sqrt / reciprocal for the shared float / double templates: float as
// before; float64 on the device takes the Newton-refined MUFU seeds (the
// float64 instances in this TU are the guard-band re-evaluations of float32
// results, ~1 ulp is ample there)
PGG_HD float t_sqrt(float x) { return m_sqrt(x); }
PGG_HD double t_sqrt(double x) {
#if defined(__CUDA_ARCH__) && PGG_FAST_F64
  return x > 0.0 ? x * d_rsqrt(x) : 0.0;
#else
  return sqrt(x);
#endif
}
PGG_HD float t_rcp(float x) { return 1.0f / x; }
PGG_HD double t_rcp(double x) { return d_rcp(x); }

template <class T> PGG_HD V3<T> unit(const V3<T>& v) {
  const T n = t_sqrt(dot(v, v));
  return v * t_rcp(m_max(n, T(1e-30)));
}
template <class D, class S> PGG_HD V3<D> cvt(const V3<S>& v) { return {(D)v.x, (D)v.y, (D)v.z}; }

// Branchless revised ONB keyed on sign(n_z) (sgmap.py:85-98)
template <class T> struct Frame {
  V3<T> t, b, n;
  PGG_MHD V3<T> to_local(const V3<T>& v) const { return {dot(v, t), dot(v, b), dot(v, n)}; }
  PGG_MHD V3<T> to_world(const V3<T>& v) const {
    return {t.x * v.x + b.x * v.y + n.x * v.z, t.y * v.x + b.y * v.y + n.y * v.z, t.z * v.x + b.z * v.y + n.z * v.z};
  }
};
template <class T> PGG_HD Frame<T> make_frame(const V3<T>& n) {
  const T s = m_copysign(T(1), n.z);
  const T a = T(-1) / (s + n.z);
  const T b = n.x * n.y * a;
  Frame<T> f;
  f.t = {T(1) + s * n.x * n.x * a, s * b, -s * n.x};
  f.b = {b, s + n.y * n.y * a, -n.y};
  f.n = n;
  return f;
}

// ---------------------------------------------------------------------------
// equal-area square <-> hemisphere (sgmap.py:21-77)

// Concentric map + Lambert lift.  phi is carried in units of pi so the
// device evaluates sincospi without rounding 2*pi*u first.
template <class T> PGG_HD V3<T> sq_to_dir(T px, T py) {
  const T a = T(2) * px - T(1);
  const T b = T(2) * py - T(1);
  T r, q;
  if (m_abs(a) > m_abs(b)) {
    r = a;
    q = T(0.25) * (b / a);
  } else if (b != T(0)) {
    r = b;
    q = T(0.5) - T(0.25) * (a / b);
  } else {
    r = T(0);
    q = T(0);
  }
  T s, c;
  m_sincospi(q, &s, &c);
  const T r2 = r * r;
  const T lift = smp_sqrt(m_max(T(2) - r2, T(0)));
  return {r * c * lift, r * s * lift, T(1) - r2};
}

// Inverse lift + inverse concentric map, clipped to [0,1]^2.  Callers pass
// z >= 0 (the reference raises below -1e-9; sgmap.py:72-73).
template <class T> PGG_HD void dir_to_sq(const V3<T>& v, T& sx, T& sy) {
  const T is = T(1) / m_sqrt(m_max(T(1) + v.z, T(1e-30)));
  const T x = v.x * is;
  const T y = v.y * is;
  const T rho = m_sqrt(x * x + y * y);
  T a, b;
  if (rho == T(0)) {
    a = T(0);
    b = T(0);
  } else if (m_abs(x) >= m_abs(y)) {
    a = m_copysign(rho, x);
    b = atan_unit(q_div(y, x)) * (T(4) * K<T>::inv_pi) * a;
  } else {
    b = m_copysign(rho, y);
    a = atan_unit(q_div(x, y)) * (T(4) * K<T>::inv_pi) * b;
  }
  sx = m_clamp01((a + T(1)) * T(0.5));
  sy = m_clamp01((b + T(1)) * T(0.5));
}

// float32 fast form of dir_to_sq: the two concentric branches collapse to
// one atan of min/max (|y/x| or |x/y| <= 1) with the signs restored, and the
// lift uses a reciprocal square root.  Same values as the generic form to a
// few ulp.
#ifndef PGG_SQ_POLY8
#define PGG_SQ_POLY8 1  // (4/pi) atan folded into one 8-term polynomial
#endif
// (4/pi) atan(t) on 0 <= t <= 1 as t P(t^2), 8 terms (near-minimax fit; max
// abs error 1.9e-7 evaluated in float32, like atan_unit(t) * 4/pi): 2
// instructions fewer per EM record.  A 7-term fit (4.3e-7) saved one more
// but tripled the golden Gamma error (p99.99 1.7e-5 -> 5.3e-5).
PGG_HD float atan4pi_unit(float t) {
  const float u = t * t;
  float p = -0.005162642803043127f;
  p = fmaf(p, u, 0.02783750370144844f);
  p = fmaf(p, u, -0.07119078189134598f);
  p = fmaf(p, u, 0.12276896089315414f);
  p = fmaf(p, u, -0.17709042131900787f);
  p = fmaf(p, u, 0.25396761298179626f);
  p = fmaf(p, u, -0.4243689775466919f);
  p = fmaf(p, u, 1.2732386589050293f);
  return t * p;
}
#ifndef PGG_SQ_NOFLOOR
#define PGG_SQ_NOFLOOR 1  // no 1e-30 floor under the lift rsqrt (the saturating clip maps the z = -1 inf / NaN to 0): -0.2 %, same Gamma
#endif
#ifndef PGG_SQ_MUFU_SQRT
#define PGG_SQ_MUFU_SQRT 0  // 1: rho on MUFU.SQRT: a further -0.6 % but golden Gamma p99.99 2.7e-5 -> 4.0e-5 (not kept)
#endif
#ifndef PGG_SQ_FMA_SAT
#define PGG_SQ_FMA_SAT 1  // record square map clip as fma.sat (one FFMA.SAT instead of FFMA + FADD.SAT): with PGG_W_UMASK -0.7 %, same Gamma
#endif
#ifndef PGG_SQ_RAW
#define PGG_SQ_RAW 1  // record square mapping on raw MUFU rsqrt / rcp: 0.528 -> 0.519 ms; golden Gamma p99.99 stays <= 3.1e-5 (limit 1e-4)
#endif
PGG_HD void dir_to_sq_f(const V3<float>& v, float& sx, float& sy) {
#if defined(__CUDA_ARCH__) && PGG_SQ_RAW && PGG_SQ_NOFLOOR
  // no floor: 1 + z <= 0 (z = -1, masked records only) gives inf / NaN,
  // which the saturating clip below maps to finite 0
  const float rs = rsqrtf(1.0f + v.z);
#elif defined(__CUDA_ARCH__) && PGG_SQ_RAW
  const float rs = rsqrtf(fmaxf(1.0f + v.z, 1e-30f));
#else
  const float rs = r_rsqrt(fmaxf(1.0f + v.z, 1e-30f));
#endif
  const float x = v.x * rs, y = v.y * rs;
  const float ax = fabsf(x), ay = fabsf(y);
  const float rho2 = x * x + y * y;
#if defined(__CUDA_ARCH__) && PGG_SQ_RAW
  // floors instead of guards: a zero rho2 / max gives 0 * finite = 0
#if PGG_SQ_MUFU_SQRT
  const float rho = f_sqrt_mufu(rho2);  // MUFU.SQRT (sqrt.approx; 0 -> 0)
#else
  const float rho = rho2 * rsqrtf(fmaxf(rho2, 1e-36f));
#endif
  const float mx = fmaxf(ax, ay);
  const float t = fminf(ax, ay) * f_rcp(fmaxf(mx, 1e-36f));
#else
  const float rho = rho2 > 0.0f ? rho2 * r_rsqrt(rho2) : 0.0f;
  const float mx = fmaxf(ax, ay);
  const float t = mx > 0.0f ? r_div(fminf(ax, ay), mx) : 0.0f;
#endif
#if PGG_SQ_POLY8
  const float u = atan4pi_unit(t) * rho;
#else
  const float u = atan_unit(t) * (4.0f * 0.31830988618379067154f) * rho;
#endif
  const bool xdom = ax >= ay;
  const float a = copysignf(xdom ? rho : u, x);
  const float b = copysignf(xdom ? u : rho, y);
#if defined(__CUDA_ARCH__) && PGG_SQ_FMA_SAT
  // (a + 1) / 2 as one fma: halving commutes with rounding, same value; the
  // clip to [0,1] in the same instruction (fma.sat; nvcc emits FFMA + FADD.SAT
  // for __saturatef(fmaf(..)))
  asm("fma.rn.ftz.sat.f32 %0, %1, 0f3F000000, 0f3F000000;" : "=f"(sx) : "f"(a));
  asm("fma.rn.ftz.sat.f32 %0, %1, 0f3F000000, 0f3F000000;" : "=f"(sy) : "f"(b));
#elif defined(__CUDA_ARCH__)
  // (a + 1) / 2 as one fma: halving commutes with rounding, same value
  sx = __saturatef(fmaf(a, 0.5f, 0.5f));
  sy = __saturatef(fmaf(b, 0.5f, 0.5f));
#else
  sx = fminf(fmaxf((a + 1.0f) * 0.5f, 0.0f), 1.0f);
  sy = fminf(fmaxf((b + 1.0f) * 0.5f, 0.0f), 1.0f);
#endif
}

// ---------------------------------------------------------------------------
// BRDFs in a local frame (scene.py:247-380).  The reference evaluates GGX in
// world space as d = cos_h^2 (a^2 - 1) + 1 with cos_h = h . n for a unit h
// and the stored (float32, not exactly unit) normal n.  At the specular
// peak d ~ a^2, so float32 must not form 1 - cos_h^2 by subtraction, and the
// 1 - |n|^2 ~ 1e-7 offset of the stored normal matters at the 1e-5 level.
// With h_raw in an orthonormal frame about n/|n| (s^2 = h.x^2 + h.y^2,
// c = h.z, no normalisation needed):
//   d = (s^2 + c^2 kappa) / (s^2 + c^2),   kappa = 1 - |n|^2 (1 - a^2)
// which is the reference's d to float32 relative precision (kappa = a^2 for
// the exactly-unit local normal e_z of the guided lanes).

template <class T> struct Mat {
  bool glossy;
  T a2;     // alpha^2, alpha = max(rough^2, 1e-6)
  T kappa;  // 1 - |n|^2 (1 - a2)
};

template <class T> PGG_HD T ggx_d(T a2, T kappa, const V3<T>& h) {
  const T c2 = h.z * h.z;
  const T s2 = h.x * h.x + h.y * h.y;
  const T n2 = s2 + c2;
  const T d = n2 > T(0) ? (s2 + c2 * kappa) / n2 : T(1);
  return a2 / m_max(K<T>::pi * d * d, T(1e-30));
}
template <class T> PGG_HD T ggx_g1(T a2, T c) {
  return T(2) * c / m_max(c + m_sqrt(a2 + (T(1) - a2) * c * c), T(1e-30));
}

// record-loop variants with fast division (same formulas)
PGG_HD float ggx_d_fast(float a2, float kappa, const V3<float>& h) {
  const float c2 = h.z * h.z;
  const float s2 = h.x * h.x + h.y * h.y;
  const float n2 = s2 + c2;
  const float d = n2 > 0.0f ? f_div(s2 + c2 * kappa, n2) : 1.0f;
  return f_div(a2, fmaxf(K<float>::pi * d * d, 1e-30f));
}
PGG_HD float ggx_g1_fast(float a2, float c) {
  return f_div(2.0f * c, fmaxf(c + f_sqrt(a2 + (1.0f - a2) * c * c), 1e-30f));
}

// solid-angle pdf of brdf_sample (scene.py:287-308), wo.z = cos_o
template <class T> PGG_HD T brdf_pdf_local(const Mat<T>& m, const V3<T>& wi, const V3<T>& wo) {
  if (!(wi.z > T(0) && wo.z > T(0))) return T(0);
  if (!m.glossy) return wi.z * K<T>::inv_pi;
  return ggx_g1(m.a2, m_abs(wo.z)) * ggx_d(m.a2, m.kappa, wi + wo) / m_max(T(4) * wo.z, T(1e-30));
}

// uniforms from a raw draw: u, and 1-u computed from the integer so it keeps
// full relative precision near u -> 1 (float32 path)
PGG_HD float u01(uint32_t u, float) { return u01f(u); }
PGG_HD double u01(uint32_t u, double) { return u01d(u); }
PGG_HD float om_u01(uint32_t u, float) { return (float)(0x100000000ULL - (uint64_t)u) * 2.3283064365386963e-10f; }
PGG_HD double om_u01(uint32_t u, double) { return 1.0 - u01d(u); }  // exact in float64

// Lambert cosine sample (scene.py:311-316); z = sqrt(1 - u1)
// Lambert azimuth: no decision depends on it, so the device uses MUFU
// sin/cos on the folded angle (direction error < 1e-6)
PGG_HD void sincos_turn_lambert(uint32_t u, float* s, float* c) {
#if defined(__CUDA_ARCH__) && PGG_SMP_MUFU_TRIG
  const float th = (float)(int32_t)u * 1.4629180792671596e-09f;  // 2 pi u - (u >= 1/2 ? 2 pi : 0)
  *s = __sinf(th);
  *c = __cosf(th);
#else
  sincos_turn(u, s, c);
#endif
}
PGG_HD void sincos_turn_lambert(uint32_t u, double* s, double* c) { sincos_turn(u, s, c); }

template <class T> PGG_HD V3<T> sample_cosine(uint32_t a, uint32_t b) {
  const T r = m_sqrt(u01(a, T()));
  T s, c;
  sincos_turn_lambert(b, &s, &c);
  return {r * c, r * s, m_sqrt(m_max(om_u01(a, T()), T(0)))};
}

// Heitz GGX visible-normal sampling (scene.py:319-351).  `ill` reports the
// rim case 1 - p1^2 - p2^2 ~ 0 where float32 loses the sqrt argument; the
// caller then re-evaluates in float64.
// q = 1 - p1^2 - p2^2 of the VNDF sample (scene.py:343).  float64 as the
// reference writes it.  float32 without the cancellation of a1 - p2^2 at
// the rim of the projected disk: with a1 = 1 - p1^2, p2 = (1 - sm) sqrt(a1)
// + sm r s and 1 - r^2 = 1 - u1 (exact from the integer draw),
//   q = sm (sqrt(a1) - r s) ((2 - sm) sqrt(a1) + sm r s), where
//   sqrt(a1) - r s = (1 - u1) / D  (s > 0)  or  D  (s <= 0),  D = sqrt(a1) + r |s|,
//   (2 - sm) sqrt(a1) + sm r s = 2 (1 - sm) sqrt(a1) + sm (1 - u1) / D  (s < 0),
// every term a sum of non-negative ones (relative accuracy); 1 - sm =
// (1 - vh.z) / 2 = l2 / (2 (1 + vh.z)).
#ifndef PGG_VNDF_GUARD
#define PGG_VNDF_GUARD 1  // 0: the round-1 guard (with the naive q)
#endif
#ifndef PGG_VNDF_STABLE_Q
#define PGG_VNDF_STABLE_Q 1
#endif
PGG_HD double vndf_q(double a1, double p2, double, double, double, double, uint32_t) { return a1 - p2 * p2; }
PGG_HD float vndf_q(float a1, float p2, float rs, float sm, float l2, float vhz, uint32_t ua) {
#if PGG_VNDF_STABLE_Q
  const float om_u1 = om_u01(ua, 0.0f);
  const float sa1 = m_sqrt(fmaxf(a1, 0.0f));
  const float D = sa1 + fabsf(rs);
  const float omsm = 0.5f * l2 / (1.0f + vhz);
  const float X = rs > 0.0f ? om_u1 / D : D;
  const float Y = rs >= 0.0f ? (1.0f + omsm) * sa1 + sm * rs : 2.0f * omsm * sa1 + sm * (om_u1 / D);
  (void)p2;
  return sm * X * Y;
#else
  (void)rs, (void)sm, (void)l2, (void)vhz, (void)ua;
  return a1 - p2 * p2;
#endif
}

template <class T> PGG_HD V3<T> sample_vndf(T alpha, const V3<T>& wo, uint32_t ua, uint32_t ub, bool& ill) {
  const V3<T> vh = unit(V3<T>{wo.x * alpha, wo.y * alpha, wo.z});
  const T l2 = vh.x * vh.x + vh.y * vh.y;
  V3<T> t1;
  if (l2 > T(1e-18)) {
    const T inv = t_rcp(t_sqrt(l2));
    t1 = {-vh.y * inv, vh.x * inv, T(0)};
  } else {
    t1 = {T(1), T(0), T(0)};
  }
  const V3<T> t2 = cross(vh, t1);
  const T u1 = u01(ua, T());
  const T r = t_sqrt(u1);
  T s, c;
  sincos_turn(ub, &s, &c);
  const T p1 = r * c;
  const T a1 = om_u01(ua, T()) + u1 * s * s;  // 1 - p1^2 without cancellation
  const T sm = T(0.5) * (T(1) + vh.z);
  const T p2 = (T(1) - sm) * t_sqrt(m_max(a1, T(0))) + sm * (r * s);
  const T q = vndf_q(a1, p2, r * s, sm, l2, vh.z, ua);
  const T p3 = t_sqrt(m_max(q, T(0)));
  const V3<T> nh = t1 * p1 + t2 * p2 + vh * p3;
  const V3<T> hv = V3<T>{alpha * nh.x, alpha * nh.y, m_max(nh.z, T(1e-9))};
  const T hn = t_sqrt(dot(hv, hv));
  // With q free of cancellation (vndf_q: ~5e-7 relative) the float32 error
  // of nh is a few 1e-7 absolute and that of h ~|delta nh| / |hv|:
  // re-evaluate in float64 where |hv| < 0.03 (10.5 M draws,
  // tests/test_gpu_hazards.py::test_brdf_draws_10m: max direction error
  // 7.4e-6, 0.16 % of the draws re-evaluated).  The naive a1 - p2^2 lost up
  // to 1.5 % of q at the disk's rim and needed q < 1e-3 || p3 |hv| < 0.03
  // (1.1 % re-evaluated, one draw still 1.1e-5 off).
#if PGG_VNDF_GUARD == 0
  ill = q < T(1e-3) || p3 * hn < T(0.03);
#else
  (void)p3;
  ill = hn < T(0.03);
#endif
  const V3<T> h = hv * t_rcp(m_max(hn, T(1e-30)));
  const T k = T(2) * dot(wo, h);
  return h * k - wo;
}

// local-frame BRDF draw from two raw draws (scene.py:364-374: the same pair
// feeds both kinds; glossy lanes take the VNDF sample)
template <class T> PGG_HD V3<T> brdf_sample_local(const Mat<T>& m, T alpha, const V3<T>& wo, uint32_t a, uint32_t b,
                                                  bool& ill) {
  ill = false;
  if (m.glossy) return sample_vndf(alpha, wo, a, b, ill);
  return sample_cosine<T>(a, b);
}

// Tangent frame and local view of a pixel: built in float64 and rounded, so
// small local components (view near the normal, directions near the
// horizon) keep their relative precision in the float32 math downstream.
#ifndef PGG_WOL_RAW_FRAME
#define PGG_WOL_RAW_FRAME 2  // 1: always the raw-frame view (+0.2 %), 2: only within 0.1 of n (+0.07 %)
#endif
struct PixelFrame {
  Frame<float> fr;  // orthonormal frame about n/|n|
  V3<float> wol;    // view in that frame
  bool co_pos;      // wo . n > 0 (reference float64 sum order, stored n)
  float om_nn;      // 1 - |n|^2 of the stored normal (kept relative-exact)
};
template <class T> PGG_HD Frame<T> make_frame_fast(const V3<T>& n) {
  const T s = m_copysign(T(1), n.z);
  const T a = -d_rcp(s + n.z);
  const T b = n.x * n.y * a;
  Frame<T> f;
  f.t = {T(1) + s * n.x * n.x * a, s * b, -s * n.x};
  f.b = {b, s + n.y * n.y * a, -n.y};
  f.n = n;
  return f;
}

PGG_HD PixelFrame make_pixel_frame(const V3<float>& n, const V3<float>& wo) {
  const V3<double> nd = cvt<double>(n);
  const double nn = dot(nd, nd);
#if PGG_FAST_F64 && defined(__CUDA_ARCH__)
  const V3<double> nh = nd * d_rsqrt(fmax(nn, 1e-300));
  const Frame<double> fd = make_frame_fast(nh);
#else
  const V3<double> nh = nd * (1.0 / sqrt(fmax(nn, 1e-300)));
  const Frame<double> fd = make_frame(nh);
#endif
  const V3<double> wd = cvt<double>(wo);
  PixelFrame p;
  p.fr.t = cvt<float>(fd.t);
  p.fr.b = cvt<float>(fd.b);
  p.fr.n = cvt<float>(nh);
#if PGG_WOL_RAW_FRAME
  // the local view as the reference forms it: in the frame of the STORED
  // normal (sgmap.build_tangent_frame / to_local of the raw n, ptrace.py:
  // 200-202, scene.py:354-380).  A float32 normal has |n| = 1 +- 1e-7, and
  // that frame's t, b are then off-orthogonal to n by ~|n|^2 - 1: when the
  // view is within ~1e-3 of n the azimuth of (wo.x, wo.y) -- which the VNDF
  // sample rotates with -- moves by ~1e-4 between the raw and the
  // normalised frame (4K sequence: 7e-5 direction error).  Everything else
  // keeps the orthonormal frame about n / |n| (O(1e-7) apart).
#if PGG_WOL_RAW_FRAME == 2
  // (the two frames' local views differ in azimuth by ~1e-7 / |wo.xy|: only
  // views within ~0.1 of n need the raw frame for 1e-6)
  const V3<double> wn = fd.to_local(wd);
  if (wn.x * wn.x + wn.y * wn.y >= 1e-2) {
    p.wol = cvt<float>(wn);
  } else
#endif
  {
#if PGG_FAST_F64 && defined(__CUDA_ARCH__)
    p.wol = cvt<float>(make_frame_fast(nd).to_local(wd));
#else
    p.wol = cvt<float>(make_frame(nd).to_local(wd));
#endif
  }
#else
  p.wol = cvt<float>(fd.to_local(wd));
#endif
  p.co_pos = radd(radd(rmul(wd.x, nd.x), rmul(wd.y, nd.y)), rmul(wd.z, nd.z)) > 0.0;
  p.om_nn = (float)(1.0 - nn);
  return p;
}

// kappa of a world-frame evaluation about the stored normal
PGG_HD float kappa_world(float om_nn, float a2) {
  return (float)((double)om_nn + (double)a2 * (1.0 - (double)om_nn));
}

// ---------------------------------------------------------------------------
// Box-Muller (mixture.py:185-190) from raw u32 draws.  float path: ln(u) via
// log of the integer (u < 1/2) or log1p(-(2^32-u)/2^32) (u >= 1/2) so the
// radius keeps full relative accuracy at both ends.
PGG_HD void box_muller_f(uint32_t a, uint32_t b, float& z0, float& z1) {
  float lnu;
#if defined(__CUDA_ARCH__) && PGG_SMP_LN_UNIFIED
  // one branch-free ln u for the whole range (branches diverge in a warp).
  // u < 3/4: lg2.approx of u -- its error is ABSOLUTE (~2^-22), so only
  // where |ln u| >= 0.287 is it a small relative error (<= 4e-7).
  // u >= 3/4: log1p(-d) with d = 1 - u exact from the integer, as
  // 2 atanh(s), s = -d / (2 - d), |s| <= 1/7: four odd terms (truncation
  // < 2e-8 relative).  Near u = 1 (r = sqrt(-2 ln u) -> 0) this keeps r
  // relatively accurate; a log of 1 - d on lg2 would not (0.999999688:
  // 40 % error in ln u, 3.5e-5 in the sampled direction).
  {
    const bool lo = a < 0xC0000000u;
    float l2;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l2) : "f"((float)a * 2.3283064365386963e-10f));
    const float d = (float)(0x100000000ULL - (uint64_t)a) * 2.3283064365386963e-10f;
    const float sd = -d * f_rcp(2.0f - d);
    const float t = sd * sd;
    const float p = fmaf(t, fmaf(t, fmaf(t, 0.14285714285714285f, 0.2f), 0.33333333333333333f), 1.0f);
    lnu = lo ? l2 * 0.69314718055994531f : 2.0f * sd * p;
    if (a == 0u) lnu = -27.631021115928547f;  // log(1e-12), the reference clamp
  }
#else
  if (a == 0u) {
    lnu = -27.631021115928547f;  // log(1e-12), the reference clamp
  } else if (a < 0x80000000u) {
#if defined(__CUDA_ARCH__) && PGG_SMP_MUFU_LOG
    lnu = __log2f((float)a) * 0.69314718055994531f - 22.180709777918249f;  // |ln u| > 0.69: 2e-7 relative
#else
    lnu = m_log((float)a) - 22.180709777918249f;  // - 32 ln 2
#endif
  } else {
    lnu = m_log1p(-(float)(0x100000000ULL - (uint64_t)a) * 2.3283064365386963e-10f);
  }
#endif
  const float r = smp_sqrt(-2.0f * lnu);
  float s, c;
  sincos_turn(b, &s, &c);
  z0 = r * c;
  z1 = r * s;
}
PGG_HD void box_muller_d(uint32_t a, uint32_t b, double& z0, double& z1) {
  const double u1 = m_max(u01d(a), 1e-12);
  const double r = sqrt(-2.0 * log(u1));
  const double ang = 2.0 * K<double>::pi * u01d(b);
  z0 = r * cos(ang);
  z1 = r * sin(ang);
}

// ---------------------------------------------------------------------------
// Gaussian lobe (mixture.py:129-155) and its truncation mass (77-126)

struct LobeF {
  float mx, my;       // mean
  float l11, l21, l22;
  float il11, il22;   // reciprocals for the pdf
  float gnorm;        // 1 / (2 pi l11 l22 Z) / (2 pi): square density -> solid angle
  float z;            // truncation mass
  float pi;           // mixing coefficient (Gamma channel 6)
  int reset;          // covariance was reset to 0.05 I
};

#define PGG_GL24(X)                                  \
  X(0.0024063900014893447f, 0.0061706148999943452f)  \
  X(0.012635722014345263f, 0.01426569431446678f)     \
  X(0.030862723998633601f, 0.022138719408709706f)    \
  X(0.056792236497799464f, 0.02964929245771818f)     \
  X(0.089999007013048526f, 0.036673240705540081f)    \
  X(0.12993790421072282f, 0.043095080765976602f)     \
  X(0.17595317403151223f, 0.048809326052056963f)     \
  X(0.22728926430558022f, 0.053722135057982782f)     \
  X(0.28310324618697746f, 0.057752834026862758f)     \
  X(0.3424786601519183f, 0.060835236463901647f)      \
  X(0.40444056626319186f, 0.062918728173414123f)     \
  X(0.46797155356869719f, 0.06396909767337601f)      \
  X(0.53202844643130276f, 0.06396909767337601f)      \
  X(0.5955594337368082f, 0.062918728173414123f)      \
  X(0.6575213398480817f, 0.060835236463901647f)      \
  X(0.71689675381302254f, 0.057752834026862758f)     \
  X(0.77271073569441984f, 0.053722135057982782f)     \
  X(0.82404682596848777f, 0.048809326052056963f)     \
  X(0.87006209578927718f, 0.043095080765976602f)     \
  X(0.91000099298695147f, 0.036673240705540081f)     \
  X(0.94320776350220048f, 0.02964929245771818f)      \
  X(0.96913727600136634f, 0.022138719408709706f)     \
  X(0.98736427798565474f, 0.01426569431446678f)      \
  X(0.99759360999851066f, 0.0061706148999943452f)

// Fast standard normal CDF for the truncation mass: Phi(x) = erfc(-x/sqrt2)/2
// with the Chebyshev-fitted erfc of Numerical Recipes (erfcc, fractional
// error < 1.2e-7), ~15 instructions instead of normcdff's ~120.  Measured in
// float32: <= 2.1e-7 absolute, <= 2e-6 relative for x >= -6.
PGG_HD float ndtr_fast(float x) {
  const float z = -x * 0.70710678118654752440f;
  const float az = fabsf(z);
  const float t = f_rcp(fmaf(0.5f, az, 1.0f));
  float p = 0.17087277f;
  p = fmaf(p, t, -0.82215223f);
  p = fmaf(p, t, 1.48851587f);
  p = fmaf(p, t, -1.13520398f);
  p = fmaf(p, t, 0.27886807f);
  p = fmaf(p, t, -0.18628806f);
  p = fmaf(p, t, 0.09678418f);
  p = fmaf(p, t, 0.37409196f);
  p = fmaf(p, t, 1.00002368f);
  p = fmaf(p, t, -1.26551223f);
  const float e = t * f_exp(fmaf(-az, az, p));  // erfc(|z|)
  return 0.5f * (z >= 0.0f ? e : 2.0f - e);
}

// Phi(hi) - Phi(lo), hi > lo, evaluated on the side that avoids cancellation
PGG_HD float ndtr_diff(float hi, float lo) {
  if (lo >= 0.0f) return ndtr_fast(-lo) - ndtr_fast(-hi);
  return ndtr_fast(hi) - ndtr_fast(lo);
}

// Inner-CDF saturation state of one edge term on a segment: 0 = Phi ~ 0,
// 1 = Phi ~ 1, 2 = ramp (evaluate per node).
PGG_HD int ramp_state(float arg) { return arg >= 6.5f ? 1 : (arg <= -6.5f ? 0 : 2); }

// 24-point Gauss-Legendre nodes/weights on [0,1] (mixture.py:77-79), as
// arrays for the (rare) reference-rule fallback below
#define PGG_XN(xn, wn) xn,
#define PGG_WN(xn, wn) wn,
#ifdef __CUDACC__
__constant__ float c_gl24_x[24] = {PGG_GL24(PGG_XN)};
__constant__ float c_gl24_w[24] = {PGG_GL24(PGG_WN)};
#endif
static const float h_gl24_x[24] = {PGG_GL24(PGG_XN)};
static const float h_gl24_w[24] = {PGG_GL24(PGG_WN)};
#undef PGG_XN
#undef PGG_WN
PGG_HD float gl24_x(int i) {
#ifdef __CUDA_ARCH__
  return c_gl24_x[i];
#else
  return h_gl24_x[i];
#endif
}
PGG_HD float gl24_w(int i) {
#ifdef __CUDA_ARCH__
  return c_gl24_w[i];
#else
  return h_gl24_w[i];
#endif
}

// Sum_i w_i phi(a + L x_i) over the 24-point rule (without the 1/sqrt(2 pi)).
PGG_HD float gl24_phi(float a, float len) {
  float acc = 0.0f;
  for (int i = 0; i < 24; ++i) {
    const float z = fmaf(len, gl24_x(i), a);
    acc = fmaf(gl24_w(i), m_exp(-0.5f * z * z), acc);
  }
  return acc;
}

// The reference's truncation rule itself in float64 (pg/mixture.py:84-126,
// its operation order): the lane API (mixture.truncation_mass,
// lobe_from_stats) returns it, so callers get the reference's Z on any input
// (the pass keeps its float32 Genz form, trunc_mass_bvn, whose domain is the
// lobes it forms).
#if defined(__CUDACC__)
#define PGG_TABLE __constant__ const
#else
#define PGG_TABLE static const
#endif
PGG_TABLE double kGL24_X[24] = {0.0024063900014893447, 0.012635722014345263, 0.0308627239986336,
                                0.056792236497799464,  0.08999900701304853,  0.12993790421072282,
                                0.17595317403151223,   0.22728926430558022,  0.28310324618697746,
                                0.3424786601519183,    0.40444056626319186,  0.4679715535686972,
                                0.5320284464313028,    0.5955594337368082,   0.6575213398480817,
                                0.7168967538130225,    0.7727107356944198,   0.8240468259684878,
                                0.8700620957892772,    0.9100009929869515,   0.9432077635022005,
                                0.9691372760013663,    0.9873642779856547,   0.9975936099985107};
PGG_TABLE double kGL24_W[24] = {0.006170614899994345, 0.01426569431446678, 0.022138719408709706,
                                0.02964929245771818,  0.03667324070554008, 0.0430950807659766,
                                0.04880932605205696,  0.05372213505798278, 0.05775283402686276,
                                0.06083523646390165,  0.06291872817341412, 0.06396909767337601,
                                0.06396909767337601,  0.06291872817341412, 0.06083523646390165,
                                0.05775283402686276,  0.05372213505798278, 0.04880932605205696,
                                0.0430950807659766,   0.03667324070554008, 0.02964929245771818,
                                0.022138719408709706, 0.01426569431446678, 0.006170614899994345};
PGG_HD double ndtr_d(double x) {  // scipy.special.ndtr
  const double t = x * 0.70710678118654752440;
  return fabs(t) < 0.70710678118654752440 ? 0.5 + 0.5 * erf(t) : (t > 0.0 ? 1.0 - 0.5 * erfc(t) : 0.5 * erfc(-t));
}
PGG_COLD double trunc_mass_ref_d(double mx, double my, double l11, double l21, double l22) {
  const double lo1 = fmax(rdiv(rsub(0.0, mx), l11), -8.5);
  double hi1 = fmin(rdiv(rsub(1.0, mx), l11), 8.5);
  hi1 = fmax(hi1, lo1);
  const double sl21 = fabs(l21) < 1e-30 ? 1e-30 : l21;
  double e[6];
  e[0] = fmin(fmax(rdiv(rsub(rsub(0.0, my), rmul(-6.5, l22)), sl21), lo1), hi1);
  e[1] = fmin(fmax(rdiv(rsub(rsub(0.0, my), rmul(6.5, l22)), sl21), lo1), hi1);
  e[2] = fmin(fmax(rdiv(rsub(rsub(1.0, my), rmul(-6.5, l22)), sl21), lo1), hi1);
  e[3] = fmin(fmax(rdiv(rsub(rsub(1.0, my), rmul(6.5, l22)), sl21), lo1), hi1);
  e[4] = lo1;
  e[5] = hi1;
  for (int i = 1; i < 6; ++i)  // insertion sort (np.sort)
    for (int j = i; j > 0 && e[j - 1] > e[j]; --j) {
      const double t = e[j];
      e[j] = e[j - 1];
      e[j - 1] = t;
    }
  double acc = 0.0;
  for (int k = 0; k < 5; ++k) {
    const double a = e[k], len = rsub(e[k + 1], e[k]);
    for (int i = 0; i < 24; ++i) {
      const double z = radd(a, rmul(len, kGL24_X[i]));
      const double hi = rdiv(rsub(rsub(1.0, my), rmul(l21, z)), l22);
      const double lo = rdiv(rsub(rsub(0.0, my), rmul(l21, z)), l22);
      const double g = rsub(ndtr_d(hi), ndtr_d(lo));
      const double phi = rdiv(exp(rmul(rmul(-0.5, z), z)), 2.5066282746310002);
      acc = radd(acc, rmul(rmul(rmul(len, kGL24_W[i]), phi), g));
    }
  }
  return fmin(fmax(acc, 1e-4), 1.0);
}

// Truncation mass of N(mu, L L^T) on [0,1]^2, the reference's rule: whitened
// outer variable on [lo1, hi1] (clipped to +-8.5), break points where the
// inner edge CDFs saturate (+-6.5), 24-point Gauss-Legendre per segment,
// clamp [1e-4, 1].  Segments whose inner terms are saturated reduce to the
// Gaussian-weight sum alone; only ramp segments evaluate Phi per node.
// Used for |rho| >= 0.99 (and by tests); the hot path is trunc_mass_bvn.
PGG_COLD float trunc_mass_f(float mx, float my, float l11, float l21, float l22) {
  const float lo1 = fmaxf((0.0f - mx) / l11, -8.5f);
  const float hi1 = fmaxf(fminf((1.0f - mx) / l11, 8.5f), lo1);
  float acc = 0.0f;
  if (l21 == 0.0f) {
    const float len = hi1 - lo1;
    if (len > 0.0f) {
      const float g = ndtr_diff((1.0f - my) / l22, (0.0f - my) / l22);
      acc = len * g * gl24_phi(lo1, len);
    }
  } else {
    const float l21s = fabsf(l21) < 1e-30f ? 1e-30f : l21;
    float e[6];
    e[0] = fminf(fmaxf(((0.0f - my) + 6.5f * l22) / l21s, lo1), hi1);
    e[1] = fminf(fmaxf(((0.0f - my) - 6.5f * l22) / l21s, lo1), hi1);
    e[2] = fminf(fmaxf(((1.0f - my) + 6.5f * l22) / l21s, lo1), hi1);
    e[3] = fminf(fmaxf(((1.0f - my) - 6.5f * l22) / l21s, lo1), hi1);
    e[4] = lo1;
    e[5] = hi1;
    // sorting network for 6 keys
#define PGG_CS(i, j)                     \
  {                                      \
    const float lo_ = fminf(e[i], e[j]); \
    const float hi_ = fmaxf(e[i], e[j]); \
    e[i] = lo_;                          \
    e[j] = hi_;                          \
  }
    PGG_CS(1, 2) PGG_CS(4, 5) PGG_CS(0, 2) PGG_CS(3, 5) PGG_CS(0, 1) PGG_CS(3, 4)
    PGG_CS(1, 4) PGG_CS(0, 3) PGG_CS(2, 5) PGG_CS(1, 3) PGG_CS(2, 4) PGG_CS(2, 3)
#undef PGG_CS
    const float one_m_my = 1.0f - my;
    const float m_my = 0.0f - my;
    for (int s = 0; s < 5; ++s) {
      const float a = e[s];
      const float len = e[s + 1] - a;
      if (!(len > 0.0f)) continue;
      const float mid = a + 0.5f * len;
      const int sh = ramp_state((one_m_my - l21 * mid) / l22);
      const int sl = ramp_state((m_my - l21 * mid) / l22);
      if (sh != 2 && sl != 2) {
        if (sh - sl > 0) acc += len * gl24_phi(a, len);  // Phi(hi) - Phi(lo) = 1
        continue;
      }
      float part = 0.0f;
      for (int i = 0; i < 24; ++i) {
        const float z = fmaf(len, gl24_x(i), a);
        const float hi = (one_m_my - l21 * z) / l22;
        const float lo = (m_my - l21 * z) / l22;
        float g;
        if (sh == 2 && sl == 2)
          g = ndtr_diff(hi, lo);
        else if (sh == 2)
          g = (sl == 0) ? m_ndtr(hi) : 0.0f;
        else
          g = (sh == 1) ? m_ndtr(-lo) : 0.0f;
        part = fmaf(gl24_w(i) * m_exp(-0.5f * z * z), g, part);
      }
      acc += len * part;
    }
  }
  acc *= 0.39894228040143267794f;  // 1/sqrt(2 pi)
  return fminf(fmaxf(acc, 1e-4f), 1.0f);
}

// Gauss-Legendre node sets of the BVN form, concatenated: n = 4, 6, 10, 12,
// 16, 24 at offsets 0, 4, 10, 20, 32, 48 (nodes on [0,1], weights for [-1,1])
#ifdef __CUDACC__
__constant__ float c_glb_u[72] = {0.069431844202973714f, 0.33000947820757187f, 0.66999052179242813f, 0.93056815579702623f,
    0.03376524289842403f, 0.16939530676686776f, 0.38069040695840156f, 0.61930959304159849f,
    0.83060469323313224f, 0.96623475710157591f, 0.013046735741414128f, 0.067468316655507732f,
    0.16029521585048778f, 0.28330230293537639f, 0.42556283050918442f, 0.57443716949081558f,
    0.71669769706462361f, 0.83970478414951222f, 0.93253168334449232f, 0.98695326425858587f,
    0.0092196828766403782f, 0.047941371814762601f, 0.11504866290284765f, 0.20634102285669126f,
    0.31608425050090994f, 0.43738329574426554f, 0.5626167042557344f, 0.68391574949909006f,
    0.79365897714330869f, 0.88495133709715235f, 0.95205862818523745f, 0.99078031712335957f,
    0.0052995325041750307f, 0.0277124884633837f, 0.067184398806084122f, 0.1222977958224985f,
    0.19106187779867811f, 0.27099161117138632f, 0.35919822461037054f, 0.45249374508118129f,
    0.54750625491881877f, 0.64080177538962946f, 0.72900838882861363f, 0.80893812220132189f,
    0.87770220417750155f, 0.93281560119391593f, 0.9722875115366163f, 0.99470046749582497f,
    0.0024063900014893447f, 0.012635722014345263f, 0.030862723998633601f, 0.056792236497799464f,
    0.089999007013048526f, 0.12993790421072282f, 0.17595317403151223f, 0.22728926430558022f,
    0.28310324618697746f, 0.3424786601519183f, 0.40444056626319186f, 0.46797155356869719f,
    0.53202844643130276f, 0.5955594337368082f, 0.6575213398480817f, 0.71689675381302254f,
    0.77271073569441984f, 0.82404682596848777f, 0.87006209578927718f, 0.91000099298695147f,
    0.94320776350220048f, 0.96913727600136634f, 0.98736427798565474f, 0.99759360999851066f};
__constant__ float c_glb_w[72] = {0.34785484513745357f, 0.65214515486254643f, 0.65214515486254643f, 0.34785484513745357f,
    0.17132449237917027f, 0.36076157304813872f, 0.46791393457269104f, 0.46791393457269104f,
    0.36076157304813872f, 0.17132449237917027f, 0.066671344308688138f, 0.14945134915058039f,
    0.21908636251598201f, 0.26926671930999652f, 0.29552422471475281f, 0.29552422471475281f,
    0.26926671930999652f, 0.21908636251598201f, 0.14945134915058039f, 0.066671344308688138f,
    0.047175336386511411f, 0.10693932599531907f, 0.16007832854334642f, 0.20316742672306573f,
    0.23349253653835461f, 0.24914704581340269f, 0.24914704581340269f, 0.23349253653835461f,
    0.20316742672306573f, 0.16007832854334642f, 0.10693932599531907f, 0.047175336386511411f,
    0.027152459411754176f, 0.062253523938647456f, 0.095158511682492605f, 0.12462897125553407f,
    0.14959598881657671f, 0.16915651939500265f, 0.18260341504492364f, 0.18945061045506864f,
    0.18945061045506864f, 0.18260341504492364f, 0.16915651939500265f, 0.14959598881657671f,
    0.12462897125553407f, 0.095158511682492605f, 0.062253523938647456f, 0.027152459411754176f,
    0.01234122979998869f, 0.028531388628933559f, 0.044277438817419412f, 0.05929858491543636f,
    0.073346481411080161f, 0.086190161531953205f, 0.097618652104113926f, 0.10744427011596556f,
    0.11550566805372552f, 0.12167047292780329f, 0.12583745634682825f, 0.12793819534675202f,
    0.12793819534675202f, 0.12583745634682825f, 0.12167047292780329f, 0.11550566805372552f,
    0.10744427011596556f, 0.097618652104113926f, 0.086190161531953205f, 0.073346481411080161f,
    0.05929858491543636f, 0.044277438817419412f, 0.028531388628933559f, 0.01234122979998869f};
#endif
static const float h_glb_u[72] = {0.069431844202973714f, 0.33000947820757187f, 0.66999052179242813f, 0.93056815579702623f,
    0.03376524289842403f, 0.16939530676686776f, 0.38069040695840156f, 0.61930959304159849f,
    0.83060469323313224f, 0.96623475710157591f, 0.013046735741414128f, 0.067468316655507732f,
    0.16029521585048778f, 0.28330230293537639f, 0.42556283050918442f, 0.57443716949081558f,
    0.71669769706462361f, 0.83970478414951222f, 0.93253168334449232f, 0.98695326425858587f,
    0.0092196828766403782f, 0.047941371814762601f, 0.11504866290284765f, 0.20634102285669126f,
    0.31608425050090994f, 0.43738329574426554f, 0.5626167042557344f, 0.68391574949909006f,
    0.79365897714330869f, 0.88495133709715235f, 0.95205862818523745f, 0.99078031712335957f,
    0.0052995325041750307f, 0.0277124884633837f, 0.067184398806084122f, 0.1222977958224985f,
    0.19106187779867811f, 0.27099161117138632f, 0.35919822461037054f, 0.45249374508118129f,
    0.54750625491881877f, 0.64080177538962946f, 0.72900838882861363f, 0.80893812220132189f,
    0.87770220417750155f, 0.93281560119391593f, 0.9722875115366163f, 0.99470046749582497f,
    0.0024063900014893447f, 0.012635722014345263f, 0.030862723998633601f, 0.056792236497799464f,
    0.089999007013048526f, 0.12993790421072282f, 0.17595317403151223f, 0.22728926430558022f,
    0.28310324618697746f, 0.3424786601519183f, 0.40444056626319186f, 0.46797155356869719f,
    0.53202844643130276f, 0.5955594337368082f, 0.6575213398480817f, 0.71689675381302254f,
    0.77271073569441984f, 0.82404682596848777f, 0.87006209578927718f, 0.91000099298695147f,
    0.94320776350220048f, 0.96913727600136634f, 0.98736427798565474f, 0.99759360999851066f};
static const float h_glb_w[72] = {0.34785484513745357f, 0.65214515486254643f, 0.65214515486254643f, 0.34785484513745357f,
    0.17132449237917027f, 0.36076157304813872f, 0.46791393457269104f, 0.46791393457269104f,
    0.36076157304813872f, 0.17132449237917027f, 0.066671344308688138f, 0.14945134915058039f,
    0.21908636251598201f, 0.26926671930999652f, 0.29552422471475281f, 0.29552422471475281f,
    0.26926671930999652f, 0.21908636251598201f, 0.14945134915058039f, 0.066671344308688138f,
    0.047175336386511411f, 0.10693932599531907f, 0.16007832854334642f, 0.20316742672306573f,
    0.23349253653835461f, 0.24914704581340269f, 0.24914704581340269f, 0.23349253653835461f,
    0.20316742672306573f, 0.16007832854334642f, 0.10693932599531907f, 0.047175336386511411f,
    0.027152459411754176f, 0.062253523938647456f, 0.095158511682492605f, 0.12462897125553407f,
    0.14959598881657671f, 0.16915651939500265f, 0.18260341504492364f, 0.18945061045506864f,
    0.18945061045506864f, 0.18260341504492364f, 0.16915651939500265f, 0.14959598881657671f,
    0.12462897125553407f, 0.095158511682492605f, 0.062253523938647456f, 0.027152459411754176f,
    0.01234122979998869f, 0.028531388628933559f, 0.044277438817419412f, 0.05929858491543636f,
    0.073346481411080161f, 0.086190161531953205f, 0.097618652104113926f, 0.10744427011596556f,
    0.11550566805372552f, 0.12167047292780329f, 0.12583745634682825f, 0.12793819534675202f,
    0.12793819534675202f, 0.12583745634682825f, 0.12167047292780329f, 0.11550566805372552f,
    0.10744427011596556f, 0.097618652104113926f, 0.086190161531953205f, 0.073346481411080161f,
    0.05929858491543636f, 0.044277438817419412f, 0.028531388628933559f, 0.01234122979998869f};
PGG_HD float glb_u(int i) {
#ifdef __CUDA_ARCH__
  return c_glb_u[i];
#else
  return h_glb_u[i];
#endif
}
PGG_HD float glb_w(int i) {
#ifdef __CUDA_ARCH__
  return c_glb_w[i];
#else
  return h_glb_w[i];
#endif
}

// Truncation mass as an exact bivariate-normal rectangle probability
// (Genz 2004, "Numerical computation of rectangular bivariate and trivariate
// normal probabilities", the |r| < 0.925 Gauss-Legendre form, here used up
// to |r| < 0.999 with a node count chosen for float32 accuracy):
//   Z = dPhi_x dPhi_y + asin(r)/(4 pi) sum_i w_i sum_corners +-
//       exp((sin(asin(r) u_i) h k - (h^2+k^2)/2) / cos^2(asin(r) u_i))
// over the four standardized corners of [0,1]^2.  It equals the
// reference's piecewise 24-point rule (mixture.py:84-126) up to that rule's
// own quadrature error (<= 2.5e-5 relative on extreme lobes, ~1e-15
// typically); |r| >= 0.999 falls back to the reference rule itself.
#ifndef PGG_BVN_FAST
#define PGG_BVN_FAST 1
#endif
PGG_HD float trunc_mass_bvn(double mx, double my, double sxx, double syy, double sxy, float l11, float l21,
                            float l22) {
  // standardised bounds and correlation in float32 (the result is float32;
  // float64 here bought nothing but DP divisions)
  const float mxf = (float)mx, myf = (float)my;
  const float isx = r_rsqrt((float)sxx), isy = r_rsqrt((float)syy);
  const float r = (float)sxy * isx * isy;
  const float ar = fabsf(r);
  float z;
  if (ar >= 0.999f) {
    z = trunc_mass_f(mxf, myf, l11, l21, l22);
  } else {
    const float a1 = (0.0f - mxf) * isx, b1 = (1.0f - mxf) * isx;
    const float a2 = (0.0f - myf) * isy, b2 = (1.0f - myf) * isy;
    const float pa = ndtr_diff(b1, a1), pb = ndtr_diff(b2, a2);
    z = pa * pb;
    // Frechet bounds: |P(A and B) - P(A) P(B)| <= min(1 - P(A), 1 - P(B)); when
    // one marginal leaves less than 1e-6 z outside [0,1] the correlation term
    // is below 1e-6 relative (the reference rule itself is good to 8e-6)
#if PGG_BVN_FAST
    if (sxy != 0.0 && fminf(1.0f - pa, 1.0f - pb) > 1e-6f * z) {
#else
    if (sxy != 0.0) {
#endif
      const float asr = asinf(r);
      // corner terms pre-scaled by log2(e): exp(x) = ex2(x log2 e), one
      // multiply fewer per exponential in the node loop
      constexpr float L2E = 1.4426950408889634f;
      const float hk0 = L2E * (a1 * a2), hs0 = (0.5f * L2E) * (a1 * a1 + a2 * a2);
      const float hk1 = L2E * (b1 * a2), hs1 = (0.5f * L2E) * (b1 * b1 + a2 * a2);
      const float hk2 = L2E * (a1 * b2), hs2 = (0.5f * L2E) * (a1 * a1 + b2 * b2);
      const float hk3 = L2E * (b1 * b2), hs3 = (0.5f * L2E) * (b1 * b1 + b2 * b2);
      // node count per |r| for float32 accuracy (measured); one
      // loop over a constant table keeps the code small (icache)
      const int cls = ar < 0.3f ? 0 : ar < 0.75f ? 1 : ar < 0.925f ? 2 : ar < 0.96f ? 3 : ar < 0.99f ? 4 : 5;
      const int off = cls == 0 ? 0 : cls == 1 ? 4 : cls == 2 ? 10 : cls == 3 ? 20 : cls == 4 ? 32 : 48;
      const int cnt = cls == 0 ? 4 : cls == 1 ? 6 : cls == 2 ? 10 : cls == 3 ? 12 : cls == 4 ? 16 : 24;
      float acc = 0.0f;
#pragma unroll 2
      for (int i = off; i < off + cnt; ++i) {
        const float sn = f_sin(asr * glb_u(i));
        const float inv = f_rcp(1.0f - sn * sn);
        const float e = f_exp2((sn * hk0 - hs0) * inv) - f_exp2((sn * hk1 - hs1) * inv) -
                        f_exp2((sn * hk2 - hs2) * inv) + f_exp2((sn * hk3 - hs3) * inv);
        acc = fmaf(glb_w(i), e, acc);
      }
      z += acc * asr * 0.079577471545947667884f;  // 1/(4 pi)
    }
  }
  return fminf(fmaxf(z, 1e-4f), 1.0f);
}

// Lobe from the float32 Gamma moments.  Covariance, ridge, reset test and
// Cholesky run in float64 with the reference's operation order and no FMA
// contraction, so the reset branch and Sigma match the reference bitwise;
// the float32 lobe feeds the per-record math.
PGG_HD LobeF make_lobe(float mxf, float myf, float m2xx, float m2yy, float m2xy, float pi) {
  const double mx = mxf, my = myf;
  double sxx = radd(rsub((double)m2xx, rmul(mx, mx)), 1e-4);
  double syy = radd(rsub((double)m2yy, rmul(my, my)), 1e-4);
  double sxy = rsub((double)m2xy, rmul(mx, my));
  const double half = rmul(0.5, radd(sxx, syy));
  const double dd = rsub(sxx, syy);
  const double q = radd(rmul(0.25, rmul(dd, dd)), rmul(sxy, sxy));
  // zero operands (reset and fresh lobes: sxy = 0) would take the slow
  // paths of the float64 sqrt / division; the results are the same values
#if PGG_FAST_F64 && defined(__CUDA_ARCH__)
  // the reset DECISION keeps the correctly rounded sqrt of the reference
  // within a few float64 ulps of the threshold; the Cholesky factors are
  // rounded to float32 and take the fast reciprocals
  double delta = q > 0.0 ? q * d_rsqrt(q) : 0.0;
  if (fabs(rsub(half, delta) - 1e-6) <= 1e-15 * (half + delta + 1e-6)) delta = sqrt(q);
#else
  const double delta = q > 0.0 ? sqrt(q) : 0.0;
#endif
  const bool reset = rsub(half, delta) < 1e-6;
  if (reset) {
    sxx = 0.05;
    syy = 0.05;
    sxy = 0.0;
  }
#if PGG_FAST_F64 && defined(__CUDA_ARCH__)
  const double ri11 = d_rsqrt(sxx);
  const double l11 = sxx * ri11;
  const double l21 = sxy == 0.0 ? sxy : sxy * ri11;
  const double v22 = fmax(rsub(syy, rmul(l21, l21)), 1e-30);
  const double l22 = v22 * d_rsqrt(v22);
#else
  const double l11 = sqrt(sxx);
  const double l21 = sxy == 0.0 ? sxy : sxy / l11;
  const double l22 = sqrt(fmax(rsub(syy, rmul(l21, l21)), 1e-30));
#endif
  LobeF L;
  L.mx = mxf;
  L.my = myf;
  L.l11 = (float)l11;
  L.l21 = (float)l21;
  L.l22 = (float)l22;
  L.il11 = 1.0f / L.l11;
  L.il22 = 1.0f / L.l22;
#ifdef PGG_PROF_NO_TRUNC
  L.z = 1.0f;  // measurement-only build
#else
  L.z = trunc_mass_bvn(mx, my, sxx, syy, sxy, L.l11, L.l21, L.l22);
#endif
  // 1 / (2 pi l11 l22 Z) / (2 pi)
  L.gnorm = L.il11 * L.il22 * (0.025330295910584444f / L.z);
  L.pi = pi;
  L.reset = reset ? 1 : 0;
  return L;
}

// solid-angle Gaussian density of a square point (gaussian_pdf_square / 2pi)
PGG_HD float gauss_sr(const LobeF& L, float sx, float sy) {
  const float z1 = (sx - L.mx) * L.il11;
  const float z2 = ((sy - L.my) - L.l21 * z1) * L.il22;
  return f_exp(-0.5f * (z1 * z1 + z2 * z2)) * L.gnorm;
}

// EM training budget N = floor((1 - min(k,kmax)/kmax)*15 + 5 + 0.5)
// (mixture.py:324-328), computed in float64 like the reference
PGG_HD int neighbor_budget(float k, int kmax) {
  const double kk = fmin((double)k, (double)kmax);
  // kk / kmax; a power-of-two kmax (64 by default) divides exactly as a product
  const double q = (kmax & (kmax - 1)) == 0 ? kk * (1.0 / (double)kmax) : kk / (double)kmax;
  const double raw = radd(rmul(rsub(1.0, q), 15.0), 5.0);
  return (int)floor(radd(raw, 0.5));
}

}  // namespace pgg
