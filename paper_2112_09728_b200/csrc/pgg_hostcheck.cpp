// pgg_hostcheck.cpp — TEST-ONLY host build of the device bodies.
//
// Compiles pgg_pass.cuh / pgg_math.cuh with g++ (-ffp-contract=off) so the
// CPU test suite can compare the exact per-pixel formulas of the CUDA kernels
// with the oracle in a container without a GPU.  Loaded only by tests/; the
// product shim (paper_2112_09728_b200/_lib.py) never loads it and has no CPU
// path.  Same argument conventions as include/pgg.h, host pointers.
#include <string.h>

#include "pgg.h"
#include "pgg_pass.cuh"

using namespace pgg;

extern "C" {

int pgghc_guiding_pass(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gbuffer* prev,
                       const pgg_gamma_in* gamma_prev, const pgg_vpl* vpl, const pgg_gamma_out* gamma_reproj,
                       const pgg_gamma_out* gamma_out, const pgg_samples* samples, int32_t* halo_misses) {
  if (!cfg || !cur || !gamma_prev) return PGG_ERR_ARGUMENT;
  PassArgs A;
  memset(&A, 0, sizeof(A));
  A.cfg = *cfg;
  pass_args_finish(A);
  A.cur = *cur;
  if (prev) A.prev = *prev;
  A.gin = *gamma_prev;
  if (vpl) A.vpl = *vpl;
  if (gamma_reproj) A.grep = *gamma_reproj;
  if (gamma_out) A.gout = *gamma_out;
  if (samples) A.smp = *samples;
  A.has_prev = prev != nullptr;
  A.has_vpl = vpl != nullptr;
  A.has_grep = gamma_reproj != nullptr;
  A.has_smp = samples != nullptr;
  A.halo_misses = halo_misses;
  uint64_t jm[JUMPS], ja[JUMPS];
  jump_tables(jm, ja);
  for (int yl = 0; yl < cfg->rows; ++yl)
    for (int x = 0; x < cfg->width; ++x) pass_pixel(A, x, yl, jm, ja);
  return PGG_OK;
}

int pgghc_trunc_mass(int64_t n, const float* mx, const float* my, const float* l11, const float* l21,
                     const float* l22, float* z) {
  for (int64_t i = 0; i < n; ++i) z[i] = trunc_mass_f(mx[i], my[i], l11[i], l21[i], l22[i]);
  return PGG_OK;
}

// lobe of float32 Gamma rows: out 10 floats per row
// (mx, my, l11, l21, l22, z, gnorm, reset, il11, il22)
int pgghc_lobe_f(int64_t n, const float* st, float* out) {
  for (int64_t i = 0; i < n; ++i) {
    const float* s = st + 8 * i;
    const LobeF L = make_lobe(s[0], s[1], s[2], s[3], s[4], s[6]);
    float* o = out + 10 * i;
    o[0] = L.mx;
    o[1] = L.my;
    o[2] = L.l11;
    o[3] = L.l21;
    o[4] = L.l22;
    o[5] = L.z;
    o[6] = L.gnorm;
    o[7] = (float)L.reset;
    o[8] = L.il11;
    o[9] = L.il22;
  }
  return PGG_OK;
}

int pgghc_sq_to_dir(int64_t n, const float* sq, float* d) {
  for (int64_t i = 0; i < n; ++i) {
    const V3<float> v = sq_to_dir<float>(sq[2 * i], sq[2 * i + 1]);
    d[3 * i] = v.x;
    d[3 * i + 1] = v.y;
    d[3 * i + 2] = v.z;
  }
  return PGG_OK;
}

int pgghc_dir_to_sq(int64_t n, const float* d, float* sq) {
  for (int64_t i = 0; i < n; ++i) dir_to_sq<float>(v3(d[3 * i], d[3 * i + 1], d[3 * i + 2]), sq[2 * i], sq[2 * i + 1]);
  return PGG_OK;
}

int pgghc_box_muller(int64_t n, const uint32_t* a, const uint32_t* b, float* z) {
  for (int64_t i = 0; i < n; ++i) box_muller_f(a[i], b[i], z[2 * i], z[2 * i + 1]);
  return PGG_OK;
}

int pgghc_disk_offset(int64_t n, const uint32_t* a, const uint32_t* b, double radius, int32_t* d) {
  for (int64_t i = 0; i < n; ++i) {
    int dx, dy;
    disk_offset(a[i], b[i], radius, dx, dy);
    d[2 * i] = dx;
    d[2 * i + 1] = dy;
  }
  return PGG_OK;
}

int pgghc_neighbor_budget(int64_t n, const float* k, int32_t kmax, int32_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = neighbor_budget(k[i], kmax);
  return PGG_OK;
}

}  // extern "C"

extern "C" int pgghc_train_records(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gamma_in* gamma,
                                   const pgg_vpl* vpl, int64_t n, const int32_t* pix_xy, const uint64_t* states,
                                   float* records) {
  PassArgs A;
  memset(&A, 0, sizeof(A));
  A.cfg = *cfg;
  pass_args_finish(A);
  A.cur = *cur;
  A.gin = *gamma;
  A.vpl = *vpl;
  A.has_vpl = 1;
  uint64_t jm[JUMPS], ja[JUMPS];
  jump_tables(jm, ja);
  for (int64_t i = 0; i < n; ++i) {
    const int x = pix_xy[2 * i], y = pix_xy[2 * i + 1];
    em_dump(A, x, y, states[(int64_t)y * cfg->width + x], jm, ja, records + i * SLOTS * 4);
  }
  return PGG_OK;
}
