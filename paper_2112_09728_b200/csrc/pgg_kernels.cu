// pgg_kernels.cu — sm_100a kernels and the C ABI of libpgg.so (include/pgg.h).
//
// Build (see __graft_entry__.build):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17
//        -shared -Xcompiler -fPIC -I include csrc/pgg_kernels.cu -o libpgg.so
#include <cuda.h>
#include <algorithm>
#include <atomic>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pgg.h"
#include "pgg_math.cuh"
#include "pgg_pass.cuh"

using namespace pgg;

// shared with the render translation unit (pgg_render.cu)
namespace pgg_rt {
thread_local char g_cuda_err[256] = "";

int check_launch() {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s", cudaGetErrorString(e));
    return PGG_ERR_CUDA;
  }
  return PGG_OK;
}
}  // namespace pgg_rt

namespace {

using pgg_rt::check_launch;
using pgg_rt::g_cuda_err;

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#ifndef PGG_TILE_H
// 32 x 12 tiles at 2 blocks/SM (24 warps, 80 registers): 0.4365 vs 0.4405 ms
// for 32 x 8 at 3 blocks (less VPL halo per pixel: 56 x 36 tile elements
// for 384 pixels at R = 10-12); 32 x 6 at 4 and 32 x 24 at 1 are slower
// (0.482 / 0.460 ms)
#define PGG_TILE_H 12
#endif
constexpr int TILE_W = 32, TILE_H = PGG_TILE_H, THREADS = TILE_W * TILE_H;
constexpr int MAX_TILE_R = 12;  // EM halo staged in shared memory up to this radius

#ifndef PGG_PHASE_SYNC
#define PGG_PHASE_SYNC 0  // block-wide barrier between stage 1 and the EM loop: helped in round 1 (0.5585 vs 0.5623 ms), costs 0.4 % now (0.4642 vs 0.4624 ms)
#endif
#ifndef PGG_TILE_S
#define PGG_TILE_S 1
#endif
#ifndef PGG_OPAQUE_Y
#define PGG_OPAQUE_Y 1
#endif
#ifndef PGG_STASH
#define PGG_STASH 1
#endif
#ifndef PGG_STAGE_KERNELS
#define PGG_STAGE_KERNELS 1  // single-stage calls on stage-specialised instantiations
#endif
#ifndef PGG_MIN_BLOCKS
#define PGG_MIN_BLOCKS 2  // 80 registers, 24 warps/SM with 32 x 12 tiles (round 1: 3 blocks of 32 x 8)
#endif

// shared-memory carve-up of one block
struct SmemLayout {
  int R, cols, rows;
  size_t tile_bytes, off_l, off_em, off_sum, off_bar, total;
  __host__ __device__ SmemLayout(int r, bool tile) : R(r), cols(TILE_W + 2 * r), rows(TILE_H + 2 * r) {
    tile_bytes = tile ? (size_t)cols * rows * 16 : 0;
    off_l = (tile_bytes + 127) & ~(size_t)127;
    off_em = off_l + ((tile_bytes + 127) & ~(size_t)127);
    // the lane's Gamma (2 float4) parked during the EM loop
    const size_t em_bytes = (size_t)THREADS * 32;
    const size_t sum_bytes = 0;
    off_sum = off_em + em_bytes;
    off_bar = off_sum + sum_bytes;
    total = off_bar + 16;
  }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// TMA: 2-D tiled bulk copy global -> shared, completion on an mbarrier
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// ---------------------------------------------------------------------------
// The guiding pass.  A block is a 32 x TILE_H pixel tile, one warp per row, one
// lane per pixel end to end.
//   stage 0  (kTile) one thread issues two TMA loads of the block's VPL tile
//            plus the EM halo (Pi y and L planes) into shared memory; they
//            land while stage 1 runs
//   stage 1  reproject Gamma, lobe + truncation mass, depth-0 sampling, EM
//            context (registers)
//   stage 2  EM over the pixel's candidate slots, VPLs from the tile
//   stage 3  float64 M-step, Gamma' store
// Measured alternatives (2/4/8 lanes per pixel with a butterfly reduction,
// a split stage-1 / EM kernel pair) were slower; see DESIGN.md section 4.

template <bool kTile, bool kFull, int kStage = 0>
__global__ void __launch_bounds__(THREADS, PGG_MIN_BLOCKS)
    k_guiding_pass(const PassArgs A, const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmL,
                   int R) {
  extern __shared__ __align__(128) unsigned char smem[];
  const SmemLayout SL(R, kTile);
  float4* tile_y = reinterpret_cast<float4*>(smem);
  float4* tile_l = reinterpret_cast<float4*>(smem + SL.off_l);
  float* s_em = reinterpret_cast<float*>(smem + SL.off_em);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SL.off_bar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int band_y0 = A.cfg.row0 + blockIdx.y * TILE_H;  // frame row of the tile's first row
  if (kStage != 1 && kTile && A.has_vpl) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      const uint32_t bytes = (uint32_t)(2 * SL.tile_bytes);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                   : "memory");
      const int c0 = (int)(blockIdx.x * TILE_W - R) * 4;
      const int c1 = band_y0 - R - A.vpl.row0;
      tma_load_2d(tile_y, &tmY, c0, c1, bar);
      tma_load_2d(tile_l, &tmL, c0, c1, bar);
    }
    __syncthreads();  // barrier initialised before anyone waits on it
  }
  const int x = blockIdx.x * TILE_W + lane;
  const int yl = blockIdx.y * TILE_H + warp;
  const bool active = x < A.cfg.width && yl < A.cfg.rows;
  float4 g0 = f4(0, 0, 0, 0), g1 = f4(0, 0, 0, 0);
  EmSetup S;
  S.flags = 0;
  S.nb = 0;
  bool train = false;
  if (active) train = pixel_stage<kStage>(A, x, yl, g0, g1, S);
  if constexpr (kStage == 1) {
    return;  // reprojection + sampling launch: no EM code at all
  } else {
  if (!A.has_vpl) return;  // uniform across the grid
  if (!train) {
    S.flags = 0;
    S.nb = 0;
  }
  // one lane per pixel end to end: the EM context stays in registers
#if PGG_PHASE_SYNC
  __syncthreads();  // keep a block's warps in one code phase (instruction-cache locality)
#endif
  if (kTile) mbar_wait(bar, 0);
  if (!active) return;
  float acc[7] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#if PGG_OPAQUE_Y
  // through a shuffle, opaque to the register allocator: under pressure the
  // row is then kept or spilled (one reload) instead of being rebuilt from
  // tid / ctaid / kernel parameters in every slot of the record loop
  const int y = __shfl_sync(__activemask(), A.cfg.row0 + yl, lane);
#else
  const int y = A.cfg.row0 + yl;
#endif
#if PGG_STASH
  // park Gamma in shared memory: 8 registers fewer live across the EM loop
  float4* stash = reinterpret_cast<float4*>(s_em);
  stash[threadIdx.x] = g0;
  stash[THREADS + threadIdx.x] = g1;
#endif
  if (train) {
    if (kTile) {
#if PGG_TILE_S
      const VplTileS V{smem_u32(tile_y), (uint32_t)SL.off_l, (int)(blockIdx.x * TILE_W) - R, band_y0 - R, SL.cols,
                       SL.cols * SL.rows};
#else
      const VplTile V{tile_y, tile_l, (int)(blockIdx.x * TILE_W) - R, band_y0 - R, SL.cols};
#endif
      em_partial<kFull>(A, V, S, x, y, c_jmul, c_jadd, acc);
    } else {
      const VplGlobal V{A.vpl.y, A.vpl.L, A.cfg.width, A.vpl.row0, A.vpl.rows};
      em_partial<kFull>(A, V, S, x, y, c_jmul, c_jadd, acc);
    }
  }
  const int64_t own = (int64_t)yl * A.cfg.width + x;
#if PGG_STASH
  g0 = stash[threadIdx.x];
  g1 = stash[THREADS + threadIdx.x];
#endif
  float4 o0 = g0, o1 = g1;
  if (train) m_step_apply(g0, g1, acc, A.cfg.k_max, o0, o1);
  PGG_CHK(CHK_OUT, yl >= 0 && yl < A.cfg.rows && x < A.cfg.width, yl, x);
  st4(A.gout.g0, own, o0);
  st4(A.gout.g1, own, o1);
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// link-time dependency on libcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// VPL plane (rows x W float4) as a 2-D float32 tensor of 4W x rows, box of
// the tile + halo
bool encode_vpl_map(CUtensorMap* m, const float* plane, int width, int rows, int R) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)4 * width, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)4 * width * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)(4 * (TILE_W + 2 * R)), (cuuint32_t)(TILE_H + 2 * R)};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(plane), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Per-device state of the calling process: the dynamic-shared-memory opt-in
// is an attribute of a kernel in one device context, so it is set once per
// (instantiation, device).  Lock-free: concurrent first calls may both set
// the (idempotent) attribute; the bit is published only after it succeeded.
constexpr int MAX_DEVICES = 64;

template <bool kTile, bool kFull, int kStage>
int ensure_smem_opt_in(int dev) {
  static std::atomic<uint64_t> done{0};
  if (dev < 0 || dev >= MAX_DEVICES) return PGG_ERR_UNSUPPORTED;
  const uint64_t bit = 1ull << dev;
  if (done.load(std::memory_order_acquire) & bit) return PGG_OK;
  const SmemLayout big(kTile ? MAX_TILE_R : 0, kTile);  // the largest layout this instantiation can use
  const cudaError_t e =
      cudaFuncSetAttribute(k_guiding_pass<kTile, kFull, kStage>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)big.total);
  if (e != cudaSuccess) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return PGG_ERR_CUDA;
  }
  done.fetch_or(bit, std::memory_order_release);
  return PGG_OK;
}

template <bool kTile, bool kFull, int kStage = 0>
int launch_pass_t(const PassArgs& A, const CUtensorMap& my, const CUtensorMap& ml, int R, cudaStream_t st) {
  const SmemLayout SL(R, kTile);
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return check_launch();
  const int rc = ensure_smem_opt_in<kTile, kFull, kStage>(dev);
  if (rc != PGG_OK) return rc;
  const dim3 grid((A.cfg.width + TILE_W - 1) / TILE_W, (A.cfg.rows + TILE_H - 1) / TILE_H);
  k_guiding_pass<kTile, kFull, kStage><<<grid, THREADS, SL.total, st>>>(A, my, ml, R);
  return check_launch();
}

// VPL planes that cover every candidate row of the launch (the whole frame,
// or a row band with its full ceil(radius) halo) take the instantiation
// without the per-candidate halo checks: no candidate can miss them
template <bool kTile, int kStage = 0>
int launch_pass(const PassArgs& A, const CUtensorMap& my, const CUtensorMap& ml, int R, cudaStream_t st) {
  const int halo = (int)ceil(A.cfg.radius > 0.0 ? A.cfg.radius : 0.0);
  const int lo = std::max(0, A.cfg.row0 - halo);
  const int hi = std::min(A.cfg.height, A.cfg.row0 + A.cfg.rows + halo);
  if (A.vpl.row0 <= lo && A.vpl.row0 + A.vpl.rows >= hi) return launch_pass_t<kTile, true, kStage>(A, my, ml, R, st);
  return launch_pass_t<kTile, false, kStage>(A, my, ml, R, st);
}

// ---------------------------------------------------------------------------
// per-lane sampling on caller-owned states

__global__ void k_sample_lanes(int64_t n, int world, const float4* __restrict__ normal,
                               const float4* __restrict__ view, const float* __restrict__ rough,
                               const uint8_t* __restrict__ glossy, const uint8_t* __restrict__ guided,
                               const float* __restrict__ pi, const float* __restrict__ lobe6,
                               uint64_t* __restrict__ states, float4* __restrict__ dir, uint8_t* __restrict__ tag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float4 vv = view[i];
  PixelFrame pf;
  if (world) {
    const float4 nn = normal[i];
    pf = make_pixel_frame(v3(nn.x, nn.y, nn.z), v3(vv.x, vv.y, vv.z));
  } else {
    pf.fr.t = v3(1.f, 0.f, 0.f);
    pf.fr.b = v3(0.f, 1.f, 0.f);
    pf.fr.n = v3(0.f, 0.f, 1.f);
    pf.wol = v3(vv.x, vv.y, vv.z);
    pf.co_pos = vv.z > 0.0f;
  }
  const float* l = lobe6 + 6 * i;
  LobeF L;
  L.mx = l[0];
  L.my = l[1];
  L.l11 = l[2];
  L.l21 = l[3];
  L.l22 = l[4];
  L.z = l[5];
  L.il11 = 1.0f / L.l11;
  L.il22 = 1.0f / L.l22;
  L.gnorm = (float)(1.0 / (2.0 * K<double>::pi * (double)L.l11 * (double)L.l22) / (double)L.z * K<double>::inv_2pi);
  L.pi = pi[i];
  L.reset = 0;
  CholD cd;
  cd.from_floats = 1;
  cd.l11f = L.l11;
  cd.l21f = L.l21;
  cd.l22f = L.l22;
  uint64_t st = states[i];
  const bool gd = world ? (guided[i] != 0) : true;
  const LaneOut o = sample_lane(pf, glossy[i] != 0, rough[i], gd, L, cd, st);
  states[i] = st;
  dir[i] = f4(o.wi.x, o.wi.y, o.wi.z, o.pdf);
  tag[i] = (uint8_t)(o.gauss | (o.valid << 1) | (o.draws << 2));
}

// ---------------------------------------------------------------------------
// training-record dump (gather_training_batch)

__global__ void k_train_records(const PassArgs A, int64_t n, const int32_t* __restrict__ pix_xy,
                                const uint64_t* __restrict__ states, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int x = pix_xy[2 * i], y = pix_xy[2 * i + 1];
  const uint64_t s0 = states[(int64_t)y * A.cfg.width + x];
  em_dump(A, x, y, s0, c_jmul, c_jadd, out + i * SLOTS * 4);
}

// ---------------------------------------------------------------------------
// small batch kernels of the API edge

__global__ void k_lobe(int64_t n, const double* __restrict__ st, double* mu, double* cov, double* chol, double* z,
                       uint8_t* reset) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* s = st + 8 * i;
  // mixture.py:129-155 on the caller's float64 stats
  const double mx = s[0], my = s[1];
  double sxx = radd(rsub(s[2], rmul(mx, mx)), 1e-4);
  double syy = radd(rsub(s[3], rmul(my, my)), 1e-4);
  double sxy = rsub(s[4], rmul(mx, my));
  const double half = rmul(0.5, radd(sxx, syy));
  const double dd = rsub(sxx, syy);
  const double q = radd(rmul(0.25, rmul(dd, dd)), rmul(sxy, sxy));
  const bool bad = rsub(half, sqrt(fmax(q, 0.0))) < 1e-6;
  if (bad) {
    sxx = 0.05;
    syy = 0.05;
    sxy = 0.0;
  }
  const double l11 = sqrt(sxx);
  const double l21 = sxy / l11;
  const double l22 = sqrt(fmax(rsub(syy, rmul(l21, l21)), 1e-30));
  mu[2 * i] = mx;
  mu[2 * i + 1] = my;
  cov[4 * i] = sxx;
  cov[4 * i + 1] = sxy;
  cov[4 * i + 2] = sxy;
  cov[4 * i + 3] = syy;
  chol[4 * i] = l11;
  chol[4 * i + 1] = 0.0;
  chol[4 * i + 2] = l21;
  chol[4 * i + 3] = l22;
  z[i] = trunc_mass_ref_d(mx, my, l11, l21, l22);  // the reference's rule in float64
  if (reset) reset[i] = bad ? 1 : 0;
}

__global__ void k_trunc(int64_t n, const double* __restrict__ mu, const double* __restrict__ cov, double* z) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = cov[4 * i], c = cov[4 * i + 1], b = cov[4 * i + 3];
  const double l11 = sqrt(a);
  const double l21 = c / l11;
  const double l22 = sqrt(fmax(rsub(b, rmul(l21, l21)), 1e-30));
  z[i] = trunc_mass_ref_d(mu[2 * i], mu[2 * i + 1], l11, l21, l22);  // the reference's rule in float64
}

__global__ void k_m_step(int64_t n, int c, const double* __restrict__ st, const double* __restrict__ sq,
                         const double* __restrict__ wt, const double* __restrict__ rs,
                         const uint8_t* __restrict__ valid, int kmax, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // mixture.py:276-321
  double bw = 0, bwr = 0, m[5] = {0, 0, 0, 0, 0};
  for (int j = 0; j < c; ++j) {
    const int64_t r = i * c + j;
    const double w = wt[r];
    if (!(isfinite(w) && w >= 0.0) || (valid && !valid[r])) continue;
    const double wr = w * rs[r];
    const double x = sq[2 * r], y = sq[2 * r + 1];
    bw += w;
    bwr += wr;
    m[0] += wr * x;
    m[1] += wr * y;
    m[2] += wr * (x * x);
    m[3] += wr * (y * y);
    m[4] += wr * (x * y);
  }
  const double* s = st + 8 * i;
  double* o = out + 8 * i;
  for (int k = 0; k < 8; ++k) o[k] = s[k];
  if (!(bw > 0.0)) return;
  const double k = s[7];
  const double eta = fmax(1.0 / (k + 1.0), 1.0 / (double)kmax);
  const double den = fmax(bwr, 1e-8);
  for (int q = 0; q < 5; ++q) o[q] = (1.0 - eta) * s[q] + eta * (m[q] / den);
  o[6] = fmin(fmax((1.0 - eta) * s[6] + eta * (bwr / fmax(bw, 1e-8)), 0.05), 0.95);
  o[5] = (1.0 - eta) * s[5] + eta * bwr;
  o[7] = k + 1.0;
}

__global__ void k_make_streams(uint64_t key, int64_t n, const uint64_t* __restrict__ lanes, uint64_t* states) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) states[i] = pcg_lane(key, lanes[i]);
}

__global__ void k_next_u32(int64_t n, uint64_t* states, uint32_t* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t s = states[i];
  out[i] = pcg_next(s);
  states[i] = s;
}

__global__ void k_pack_gbuffer(int64_t p, const uint8_t* __restrict__ valid, const float* __restrict__ pos,
                               const float* __restrict__ nrm, const float* __restrict__ depth,
                               const int32_t* __restrict__ kind, const float* __restrict__ alb,
                               const float* __restrict__ rough, const float* __restrict__ view,
                               const float* __restrict__ motion, const uint8_t* __restrict__ hist,
                               uint8_t* flags, float4* nd, float4* pr, float4* va, float4* am) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p) return;
  const uint8_t v = valid[i] ? 1 : 0;
  const uint8_t h = (hist && hist[i]) ? 2 : 0;
  const uint8_t g = (kind[i] == 1) ? 4 : 0;
  flags[i] = v | h | g;
  nd[i] = f4(nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2], depth[i]);
  pr[i] = f4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], rough[i]);
  va[i] = f4(view[3 * i], view[3 * i + 1], view[3 * i + 2], alb[3 * i]);
  am[i] = f4(alb[3 * i + 1], alb[3 * i + 2], motion ? motion[2 * i] : 0.f, motion ? motion[2 * i + 1] : 0.f);
}

// the same planes from the material ids the reference's G-buffer carries
// (pg/ptrace.py:97-129 looks kind / albedo / roughness up per material;
// mat -1 = miss -> zeros), with the scene's material table: 16 B/px fewer
// to move than per-pixel albedo / roughness / kind
__global__ void k_pack_gbuffer_mat(int64_t p, const uint8_t* __restrict__ valid, const float* __restrict__ pos,
                                   const float* __restrict__ nrm, const float* __restrict__ depth,
                                   const int32_t* __restrict__ mat, int n_mat, const int32_t* __restrict__ mkind,
                                   const float* __restrict__ malb, const float* __restrict__ mrough,
                                   const float* __restrict__ view, const float* __restrict__ motion,
                                   const uint8_t* __restrict__ hist, uint8_t* flags, float4* nd, float4* pr,
                                   float4* va, float4* am) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p) return;
  const int m = mat[i];
  const bool has = m >= 0 && m < n_mat;
  const int k = has ? mkind[m] : 0;
  const float ar = has ? malb[3 * m] : 0.f, ag = has ? malb[3 * m + 1] : 0.f, ab = has ? malb[3 * m + 2] : 0.f;
  const float ro = has ? mrough[m] : 0.f;
  const uint8_t v = valid[i] ? 1 : 0;
  const uint8_t h = (hist && hist[i]) ? 2 : 0;
  const uint8_t g = (k == 1) ? 4 : 0;
  flags[i] = v | h | g;
  nd[i] = f4(nrm[3 * i], nrm[3 * i + 1], nrm[3 * i + 2], depth[i]);
  pr[i] = f4(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], ro);
  va[i] = f4(view[3 * i], view[3 * i + 1], view[3 * i + 2], ar);
  am[i] = f4(ag, ab, motion ? motion[2 * i] : 0.f, motion ? motion[2 * i + 1] : 0.f);
}

__global__ void k_pack_vpl(int64_t p, const uint8_t* __restrict__ valid, const float* __restrict__ y,
                           const float* __restrict__ rad, const uint8_t* __restrict__ strat, float4* vy,
                           float4* vl) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p) return;
  const float use = (valid[i] && strat[i] == 0) ? 1.0f : 0.0f;  // mixture.STRATEGY_BRDF
  vy[i] = f4(y[3 * i], y[3 * i + 1], y[3 * i + 2], use);
  vl[i] = f4(rad[3 * i], rad[3 * i + 1], rad[3 * i + 2], 0.0f);
}

__global__ void k_gamma_split(int64_t p, const float4* __restrict__ aos, float4* g0, float4* g1) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p) return;
  g0[i] = aos[2 * i];
  g1[i] = aos[2 * i + 1];
}

__global__ void k_gamma_join(int64_t p, const float4* __restrict__ g0, const float4* __restrict__ g1, float4* aos) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p) return;
  aos[2 * i] = g0[i];
  aos[2 * i + 1] = g1[i];
}

__global__ void k_gamma_init(int64_t p, float4* g0, float4* g1) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= p) return;
  float4 a, b;
  init_gamma(a, b);
  g0[i] = a;
  g1[i] = b;
}

// ---------------------------------------------------------------------------
// The remaining mixture.py entry points as float64 lane kernels, with the
// reference's operation order (no FMA contraction: rmul / radd / rsub).

enum MixOp { MIX_GAUSS_PDF = 0, MIX_BOX_MULLER = 1, MIX_E_STEP = 2, MIX_NEIGHBORS = 3, MIX_PDF = 4 };

// gaussian_pdf_square (mixture.py:158-169): mu (2), chol (4: l11, 0, l21, l22), z
__device__ __forceinline__ double gauss_pdf_d(const double* mu, const double* ch, double z, double px, double py) {
  const double l11 = ch[0], l21 = ch[2], l22 = ch[3];
  const double z1 = rsub(px, mu[0]) / l11;
  const double z2 = rsub(rsub(py, mu[1]), rmul(l21, z1)) / l22;
  const double e = exp(rmul(-0.5, radd(rmul(z1, z1), rmul(z2, z2))));
  return rmul(e, 1.0 / rmul(rmul(2.0 * K<double>::pi, l11), l22)) / z;
}

__global__ void k_mixture_lanes(int op, int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                                const double* __restrict__ c, const double* __restrict__ d,
                                const double* __restrict__ e, double* __restrict__ o0, double* __restrict__ o1,
                                int kmax) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  switch (op) {
    case MIX_GAUSS_PDF:  // a = mu (n,2), b = chol (n,4), c = z (n), d = p (n,2)
      o0[i] = gauss_pdf_d(a + 2 * i, b + 4 * i, c[i], d[2 * i], d[2 * i + 1]);
      break;
    case MIX_BOX_MULLER: {  // a = u1, b = u2 (mixture.py:185-190)
      const double u1 = fmax(a[i], 1e-12);
      const double r = sqrt(rmul(-2.0, log(u1)));
      const double ang = rmul(2.0 * K<double>::pi, b[i]);
      o0[i] = rmul(r, cos(ang));
      o1[i] = rmul(r, sin(ang));
      break;
    }
    case MIX_E_STEP: {  // a = pi, b = gauss pdf, c = brdf pdf (mixture.py:262-273)
      const double num = rmul(a[i], b[i]);
      const double den = radd(num, rmul(rsub(1.0, a[i]), c[i]));
      o0[i] = den > 0.0 ? num / den : 0.0;
      break;
    }
    case MIX_NEIGHBORS: {  // a = k (mixture.py:324-328); integer result stored as double
      const double kk = fmin(a[i], (double)kmax);
      o0[i] = floor(radd(radd(rmul(rsub(1.0, kk / (double)kmax), 15.0), 5.0), 0.5));
      break;
    }
    case MIX_PDF: {  // a = pi, b = mu|chol|z packed (n,7), c = square point (n,2), d = brdf pdf (mixture.py:172-182)
      const double* L = b + 7 * i;
      const double g = gauss_pdf_d(L, L + 2, L[6], c[2 * i], c[2 * i + 1]) / (2.0 * K<double>::pi);
      o0[i] = radd(rmul(a[i], g), rmul(rsub(1.0, a[i]), d[i]));
      break;
    }
  }
}

// Gaussian branch of sample_mixture (mixture.py:208-235) in float64 for
// callers with their own BRDF callbacks: zeta draw, up to 16 Box-Muller
// tries on the lane's stream; out: accepted flag, square point
__global__ void k_sample_gauss(int64_t n, const double* __restrict__ pi, const double* __restrict__ mu,
                               const double* __restrict__ chol, uint64_t* __restrict__ states, double* __restrict__ sq,
                               uint8_t* __restrict__ acc) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t st = states[i];
  const uint32_t uz = pcg_next(st);
  uint8_t hit = 0;
  double px = 0.0, py = 0.0;
  if (u01d(uz) < pi[i]) {
    const double mx = mu[2 * i], my = mu[2 * i + 1];
    const double l11 = chol[4 * i], l21 = chol[4 * i + 2], l22 = chol[4 * i + 3];
    for (int t = 0; t < GAUSS_TRIES; ++t) {
      const uint32_t ua = pcg_next(st), ub = pcg_next(st);
      double z0, z1;
      box_muller_d(ua, ub, z0, z1);
      const double qx = radd(mx, rmul(l11, z0));
      const double qy = radd(radd(my, rmul(l21, z0)), rmul(l22, z1));
      if (qx >= 0.0 && qx <= 1.0 && qy >= 0.0 && qy <= 1.0) {
        hit = 1;
        px = qx;
        py = qy;
        break;
      }
    }
  }
  states[i] = st;
  sq[2 * i] = px;
  sq[2 * i + 1] = py;
  acc[i] = hit;
}

// ---------------------------------------------------------------------------
// Diagnostics (tests only): the pass's discrete decisions over whole frames,
// through the same device functions the fused kernel runs.

// warp-aggregated counter add
__device__ __forceinline__ void count_add(int32_t* c, int n) {
  const unsigned m = __activemask();
  int tot = n;
  for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(m, tot, o);
  if ((threadIdx.x & 31) == (__ffs(m) - 1) && tot) atomicAdd(c, tot);
}

// the 19 candidate offsets of every pixel of the frame, as em_partial draws
// them (jump tables, two interleaved streams, disk_offset_k with the pass's
// radius / guard-band parameters)
__global__ void k_debug_em_offsets(const PassArgs A, int8_t* __restrict__ out, int32_t* rechecks) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t P = (int64_t)A.cfg.width * A.cfg.height;
  int n = 0;
  if (p < P) {
    const uint64_t s0 = pcg_lane(A.cfg.key_train, (uint64_t)p);
    uint64_t sa = c_jmul[0] * s0 + c_jadd[0];
    uint64_t sb = c_jmul[19] * s0 + c_jadd[19];
#if defined(__CUDA_ARCH__) && PGG_EM_PAIR
    // the pass's paired path (em_partial) computes each slot's offset with
    // disk_offset_k2; the partner slot does not change a slot's arithmetic
    for (int s = 1; s < SLOTS; s += 2) {
      const uint32_t ua0 = pcg_out(sa), ub0 = pcg_out(sb);
      sa = sa * PCG_MUL + PCG_INC;
      sb = sb * PCG_MUL + PCG_INC;
      const uint32_t ua1 = pcg_out(sa), ub1 = pcg_out(sb);
      sa = sa * PCG_MUL + PCG_INC;
      sb = sb * PCG_MUL + PCG_INC;
      int dx0, dy0, dx1, dy1, m0 = 0, m1 = 0;
      disk_offset_k2(ua0, ub0, ua1, ub1, A.cfg.radius, A.em_radius16, A.em_hband, dx0, dy0, dx1, dy1, &m0, &m1);
      n += m0 + (s + 1 < SLOTS ? m1 : 0);  // slot 20 does not exist: the last pair's partner is masked
      out[(p * (SLOTS - 1) + (s - 1)) * 2] = (int8_t)dx0;
      out[(p * (SLOTS - 1) + (s - 1)) * 2 + 1] = (int8_t)dy0;
      if (s + 1 < SLOTS) {
        out[(p * (SLOTS - 1) + s) * 2] = (int8_t)dx1;
        out[(p * (SLOTS - 1) + s) * 2 + 1] = (int8_t)dy1;
      }
    }
#else
    for (int s = 1; s < SLOTS; ++s) {
      const uint32_t ua = pcg_out(sa), ub = pcg_out(sb);
      sa = sa * PCG_MUL + PCG_INC;
      sb = sb * PCG_MUL + PCG_INC;
      int dx, dy;
      disk_offset_k(ua, ub, A.cfg.radius, A.em_radius16, A.em_hband, dx, dy, &n);
      out[(p * (SLOTS - 1) + (s - 1)) * 2] = (int8_t)dx;
      out[(p * (SLOTS - 1) + (s - 1)) * 2 + 1] = (int8_t)dy;
    }
#endif
  }
  count_add(rechecks, n);
}

// Box-Muller proposals of the guided branch: lobe from float32 Gamma
// (make_lobe, as pixel_stage), acceptance via bm_propose
// the pass's float32 truncation mass (Genz BVN, reference rule at |r| >=
// 0.999) on caller lobes, for accuracy sweeps against the reference rule
__global__ void k_debug_trunc_bvn(int64_t n, const double* __restrict__ mu, const double* __restrict__ cov,
                                  double* z) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double a = cov[4 * i], c = cov[4 * i + 1], b = cov[4 * i + 3];
  const double l11 = sqrt(a);
  const double l21 = c / l11;
  const double l22 = sqrt(fmax(rsub(b, rmul(l21, l21)), 1e-30));
  z[i] = trunc_mass_bvn(mu[2 * i], mu[2 * i + 1], a, b, c, (float)l11, (float)l21, (float)l22);
}

__global__ void k_debug_bm_accept(int64_t n, int per, const float* __restrict__ stats, const uint32_t* __restrict__ ab,
                                  uint8_t* __restrict__ out, float* __restrict__ p_out, int32_t* rechecks) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int c = 0;
  if (i < n) {
    const float* g = stats + 8 * (i / per);
    const LobeF L = make_lobe(g[0], g[1], g[2], g[3], g[4], g[6]);
    CholD cd;
    cd.mx = g[0];
    cd.my = g[1];
    cd.m2xx = g[2];
    cd.m2yy = g[3];
    cd.m2xy = g[4];
    cd.from_floats = 0;
    bool rc = false;
    float px, py;
    const bool in = bm_propose(L, cd, ab[2 * i], ab[2 * i + 1], px, py, &rc);
    out[i] = (uint8_t)((in ? 1 : 0) | (rc ? 2 : 0));
    if (p_out) {
      p_out[2 * i] = px;
      p_out[2 * i + 1] = py;
    }
    c = rc ? 1 : 0;
  }
  count_add(rechecks, c);
}

// local-frame BRDF draws of the sampler (brdf_draw_local: Lambert cosine or
// GGX VNDF with the float64 rim re-evaluation), one per lane: glossy[i],
// roughness[i], wo (float4 local, w unused), raw draws (a, b)
__global__ void k_debug_brdf_draw(int64_t n, const uint8_t* __restrict__ glossy, const float* __restrict__ rough,
                                  const float4* __restrict__ wo, const uint32_t* __restrict__ ab,
                                  float4* __restrict__ out, int32_t* rechecks) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int c = 0;
  if (i < n) {
    const double r2d = (double)rough[i] * (double)rough[i];
    const float alpha = (float)fmax(r2d, 1e-6);
    const float a2 = alpha * alpha;
    const Mat<float> mf{glossy[i] != 0, a2, a2};
    const float4 w = wo[i];
    const V3<float> wol = v3(w.x, w.y, w.z);
    bool ok;
    const V3<float> d = brdf_draw_local(mf, alpha, wol, w.z > 0.0f, ab[2 * i], ab[2 * i + 1], ok, &c);
    out[i] = f4(d.x, d.y, d.z, ok ? 1.0f : 0.0f);
  }
  count_add(rechecks, c);
}

// reprojection decision record of every pixel of the call's band
__global__ void k_debug_reproject(const PassArgs A, uint8_t* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int yl = blockIdx.y;
  if (x >= A.cfg.width) return;
  const int y = A.cfg.row0 + yl;
  const int64_t ci = (int64_t)(y - A.cur.row0) * A.cfg.width + x;
  float4 g0, g1;
  uint8_t d;
  reproject_px<true>(A, x, y, ldu8(A.cur.flags, ci), ld4(A.cur.nd, ci), ld4(A.cur.pr, ci), ld4(A.cur.am, ci), g0,
                     g1, &d);
  out[(int64_t)yl * A.cfg.width + x] = d;
}

inline unsigned blocks(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

namespace pgg_rt {
// PGG_ERR_UNSUPPORTED unless the calling thread's current device is sm_100
// (the library holds sm_100a code only); cached per device, lock-free
int device_check() {
  static std::atomic<uint8_t> state[64];  // 0 unknown, 1 sm_100, 2 other
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s", cudaGetErrorString(e));
    return PGG_ERR_CUDA;
  }
  if (dev < 0 || dev >= 64) return PGG_ERR_UNSUPPORTED;
  uint8_t st = state[dev].load(std::memory_order_relaxed);
  if (st == 0) {
    int major = 0, minor = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
      return check_launch();
    st = (major == 10 && minor == 0) ? 1 : 2;
    state[dev].store(st, std::memory_order_relaxed);
  }
  return st == 1 ? PGG_OK : PGG_ERR_UNSUPPORTED;
}
}  // namespace pgg_rt

namespace {
using pgg_rt::device_check;

}  // namespace

extern "C" {

int pgg_abi_version(void) { return PGG_ABI_VERSION; }

const char* pgg_status_string(int s) {
  switch (s) {
    case PGG_OK: return "ok";
    case PGG_ERR_ARGUMENT: return "invalid argument";
    case PGG_ERR_CUDA: return "CUDA launch error";
    case PGG_ERR_UNSUPPORTED: return "unsupported device";
    default: return "unknown status";
  }
}

const char* pgg_last_cuda_error(void) { return g_cuda_err; }

uint64_t pgg_frame_key(uint64_t seed, uint64_t frame, uint64_t stream_id) {
  uint64_t h = splitmix64(seed);
  h = splitmix64(h ^ splitmix64(frame));
  return splitmix64(h ^ splitmix64(stream_id + 0xA02BDBF7BB3C0A7ULL));
}

int pgg_guiding_pass(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gbuffer* prev,
                     const pgg_gamma_in* gamma_prev, const pgg_vpl* vpl, const pgg_gamma_out* gamma_reproj,
                     const pgg_gamma_out* gamma_out, const pgg_samples* samples, int32_t* halo_misses,
                     void* stream) {
  if (!cfg || !cur || !gamma_prev) return PGG_ERR_ARGUMENT;
  if (cfg->width <= 0 || cfg->height <= 0 || cfg->rows < 0 || cfg->row0 < 0 || cfg->row0 + cfg->rows > cfg->height)
    return PGG_ERR_ARGUMENT;
  if (cfg->rows == 0) return PGG_OK;
  if (cur->row0 > cfg->row0 || cur->row0 + cur->rows < cfg->row0 + cfg->rows) return PGG_ERR_ARGUMENT;
  if (!cur->flags || !cur->nd || !cur->pr || !cur->va || !cur->am) return PGG_ERR_ARGUMENT;
  if (!gamma_prev->g0 || !gamma_prev->g1) return PGG_ERR_ARGUMENT;
  if (!prev && (gamma_prev->row0 > cfg->row0 || gamma_prev->row0 + gamma_prev->rows < cfg->row0 + cfg->rows))
    return PGG_ERR_ARGUMENT;
  if (vpl && (!gamma_out || !vpl->y || !vpl->L || cfg->k_max < 1)) return PGG_ERR_ARGUMENT;
  if (samples && (!samples->dir || !samples->tag || cfg->spp < 1 || cfg->nee_draws < 0)) return PGG_ERR_ARGUMENT;
  // every supplied row range lies inside the frame: the whole-frame
  // instantiation relies on TMA's zero fill beyond the VPL plane's rows for
  // out-of-frame candidates, so a plane extending past the frame is refused
  const auto in_frame = [&](int32_t r0, int32_t n) { return r0 >= 0 && n >= 0 && (int64_t)r0 + n <= cfg->height; };
  if (!in_frame(cur->row0, cur->rows) || !in_frame(gamma_prev->row0, gamma_prev->rows)) return PGG_ERR_ARGUMENT;
  if (prev && !in_frame(prev->row0, prev->rows)) return PGG_ERR_ARGUMENT;
  if (vpl && !in_frame(vpl->row0, vpl->rows)) return PGG_ERR_ARGUMENT;
  // reprojection reads Gamma at OTHER pixels (the motion source): an output
  // plane that is also the input would race with it (without reprojection
  // every pixel reads and writes only its own Gamma: in place is fine)
  if (prev) {
    const auto aliases = [&](const pgg_gamma_out* o) {
      return o && (o->g0 == gamma_prev->g0 || o->g0 == gamma_prev->g1 || o->g1 == gamma_prev->g0 ||
                   o->g1 == gamma_prev->g1);
    };
    if (aliases(gamma_out) || aliases(gamma_reproj)) return PGG_ERR_ARGUMENT;
  }
  if (const int rc = device_check()) return rc;
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
  A.has_grep = gamma_reproj != nullptr && gamma_reproj->g0 && gamma_reproj->g1;
  A.has_smp = samples != nullptr;
  A.halo_misses = halo_misses;
  // stage the VPL neighbourhood through shared memory (TMA) when the halo fits
  const int R = (int)ceil(cfg->radius > 0.0 ? cfg->radius : 0.0);
  CUtensorMap my, ml;
  memset(&my, 0, sizeof(my));
  memset(&ml, 0, sizeof(ml));
  const bool tile = vpl && R <= MAX_TILE_R && encode_vpl_map(&my, vpl->y, cfg->width, vpl->rows, R) &&
                    encode_vpl_map(&ml, vpl->L, cfg->width, vpl->rows, R);
#if PGG_STAGE_KERNELS
  // single-stage calls take instantiations holding only their stages' code:
  // training alone (training_pass, the frame loop's EM launch) without the
  // sampler's state (no EM-loop spills), reprojection / sampling alone
  // without the EM loop.  Calls with both halves stay fused: as two launches
  // the latency-bound first half runs alone (0.514 vs 0.436 ms at 1080p,
  // bitwise the same results).
  if (A.has_vpl && !A.has_prev && !A.has_smp) {
    if (tile) return launch_pass<true, 2>(A, my, ml, R, S(stream));
    return launch_pass<false, 2>(A, my, ml, 0, S(stream));
  }
  if (!A.has_vpl) return launch_pass_t<false, false, 1>(A, my, ml, 0, S(stream));
#endif
  if (tile) return launch_pass<true>(A, my, ml, R, S(stream));
  return launch_pass<false>(A, my, ml, 0, S(stream));
}

// Single-stage conveniences over the fused pass (the entry points SURVEY 8b
// names): each is pgg_guiding_pass with one stage selected.
int pgg_reproject(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gbuffer* prev,
                  const pgg_gamma_in* gamma_prev, const pgg_gamma_out* gamma_out, int32_t* halo_misses, void* stream) {
  if (!prev || !gamma_out) return PGG_ERR_ARGUMENT;
  return pgg_guiding_pass(cfg, cur, prev, gamma_prev, nullptr, gamma_out, nullptr, nullptr, halo_misses, stream);
}

int pgg_train(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gamma_in* gamma, const pgg_vpl* vpl,
              const pgg_gamma_out* gamma_out, int32_t* halo_misses, void* stream) {
  if (!vpl || !gamma_out) return PGG_ERR_ARGUMENT;
  return pgg_guiding_pass(cfg, cur, nullptr, gamma, vpl, nullptr, gamma_out, nullptr, halo_misses, stream);
}

int pgg_sample_first_bounce(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gamma_in* gamma,
                            const pgg_samples* samples, void* stream) {
  if (!samples) return PGG_ERR_ARGUMENT;
  return pgg_guiding_pass(cfg, cur, nullptr, gamma, nullptr, nullptr, nullptr, samples, nullptr, stream);
}

int pgg_train_records(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gamma_in* gamma, const pgg_vpl* vpl,
                      int64_t n, const int32_t* pix_xy, const uint64_t* states, float* records, void* stream) {
  if (!cfg || !cur || !gamma || !vpl || n < 0 || !pix_xy || !states || !records || cfg->k_max < 1)
    return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  PassArgs A;
  memset(&A, 0, sizeof(A));
  A.cfg = *cfg;
  pass_args_finish(A);
  A.cur = *cur;
  A.gin = *gamma;
  A.vpl = *vpl;
  A.has_vpl = 1;
  if (const int rc = device_check()) return rc;
  k_train_records<<<blocks(n, 64), 64, 0, S(stream)>>>(A, n, pix_xy, states, records);
  return check_launch();
}

int pgg_sample_lanes(int64_t n, int32_t world, const float* normal, const float* view, const float* rough,
                     const uint8_t* glossy, const uint8_t* guided, const float* pi, const float* lobe6,
                     uint64_t* states, float* dir, uint8_t* tag, void* stream) {
  if (n < 0 || !view || !rough || !glossy || !pi || !lobe6 || !states || !dir || !tag) return PGG_ERR_ARGUMENT;
  if (world && (!normal || !guided)) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_sample_lanes<<<blocks(n, 128), 128, 0, S(stream)>>>(
      n, world, reinterpret_cast<const float4*>(normal), reinterpret_cast<const float4*>(view), rough, glossy,
      guided, pi, lobe6, states, reinterpret_cast<float4*>(dir), tag);
  return check_launch();
}

int pgg_lobe(int64_t n, const double* stats, double* mu, double* cov, double* chol, double* trunc_z, uint8_t* reset,
             void* stream) {
  if (n < 0 || !stats || !mu || !cov || !chol || !trunc_z) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_lobe<<<blocks(n, 128), 128, 0, S(stream)>>>(n, stats, mu, cov, chol, trunc_z, reset);
  return check_launch();
}

int pgg_trunc_mass(int64_t n, const double* mu, const double* cov, double* z, void* stream) {
  if (n < 0 || !mu || !cov || !z) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_trunc<<<blocks(n, 128), 128, 0, S(stream)>>>(n, mu, cov, z);
  return check_launch();
}

int pgg_m_step(int64_t n, int32_t c, const double* stats, const double* sq, const double* weight, const double* resp,
               const uint8_t* valid, int32_t k_max, double* out, void* stream) {
  if (n < 0 || c < 0 || !stats || !out || k_max < 1) return PGG_ERR_ARGUMENT;
  if (c > 0 && (!sq || !weight || !resp)) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_m_step<<<blocks(n, 128), 128, 0, S(stream)>>>(n, c, stats, sq, weight, resp, valid, k_max, out);
  return check_launch();
}

int pgg_make_streams(uint64_t key, int64_t n, const uint64_t* lanes, uint64_t* states, void* stream) {
  if (n < 0 || !lanes || !states) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_make_streams<<<blocks(n, 256), 256, 0, S(stream)>>>(key, n, lanes, states);
  return check_launch();
}

int pgg_next_u32(int64_t n, uint64_t* states, uint32_t* out, void* stream) {
  if (n < 0 || !states || !out) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_next_u32<<<blocks(n, 256), 256, 0, S(stream)>>>(n, states, out);
  return check_launch();
}

int pgg_pack_gbuffer(int64_t p, const uint8_t* valid, const float* pos, const float* normal, const float* depth,
                     const int32_t* kind, const float* albedo, const float* rough, const float* view,
                     const float* motion, const uint8_t* has_history, uint8_t* flags, float* nd, float* pr,
                     float* va, float* am, void* stream) {
  if (p < 0 || !valid || !pos || !normal || !depth || !kind || !albedo || !rough || !view || !flags || !nd || !pr ||
      !va || !am)
    return PGG_ERR_ARGUMENT;
  if (p == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_pack_gbuffer<<<blocks(p, 256), 256, 0, S(stream)>>>(
      p, valid, pos, normal, depth, kind, albedo, rough, view, motion, has_history, flags,
      reinterpret_cast<float4*>(nd), reinterpret_cast<float4*>(pr), reinterpret_cast<float4*>(va),
      reinterpret_cast<float4*>(am));
  return check_launch();
}

int pgg_pack_gbuffer_mat(int64_t p, const uint8_t* valid, const float* pos, const float* normal, const float* depth,
                         const int32_t* mat, int32_t n_mat, const int32_t* mat_kind, const float* mat_albedo,
                         const float* mat_rough, const float* view, const float* motion, const uint8_t* has_history,
                         uint8_t* flags, float* nd, float* pr, float* va, float* am, void* stream) {
  if (p < 0 || n_mat < 0 || !valid || !pos || !normal || !depth || !mat || !view || !flags || !nd || !pr || !va ||
      !am)
    return PGG_ERR_ARGUMENT;
  if (n_mat > 0 && (!mat_kind || !mat_albedo || !mat_rough)) return PGG_ERR_ARGUMENT;
  if (p == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_pack_gbuffer_mat<<<blocks(p, 256), 256, 0, S(stream)>>>(
      p, valid, pos, normal, depth, mat, n_mat, mat_kind, mat_albedo, mat_rough, view, motion, has_history, flags,
      reinterpret_cast<float4*>(nd), reinterpret_cast<float4*>(pr), reinterpret_cast<float4*>(va),
      reinterpret_cast<float4*>(am));
  return check_launch();
}

int pgg_pack_vpl(int64_t p, const uint8_t* valid, const float* y, const float* radiance, const uint8_t* strategy,
                 float* vy, float* vl, void* stream) {
  if (p < 0 || !valid || !y || !radiance || !strategy || !vy || !vl) return PGG_ERR_ARGUMENT;
  if (p == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_pack_vpl<<<blocks(p, 256), 256, 0, S(stream)>>>(p, valid, y, radiance, strategy, reinterpret_cast<float4*>(vy),
                                                    reinterpret_cast<float4*>(vl));
  return check_launch();
}

int pgg_gamma_split(int64_t p, const float* aos, float* g0, float* g1, void* stream) {
  if (p < 0 || !aos || !g0 || !g1) return PGG_ERR_ARGUMENT;
  if (p == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_gamma_split<<<blocks(p, 256), 256, 0, S(stream)>>>(p, reinterpret_cast<const float4*>(aos),
                                                       reinterpret_cast<float4*>(g0), reinterpret_cast<float4*>(g1));
  return check_launch();
}

int pgg_gamma_join(int64_t p, const float* g0, const float* g1, float* aos, void* stream) {
  if (p < 0 || !aos || !g0 || !g1) return PGG_ERR_ARGUMENT;
  if (p == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_gamma_join<<<blocks(p, 256), 256, 0, S(stream)>>>(p, reinterpret_cast<const float4*>(g0),
                                                      reinterpret_cast<const float4*>(g1),
                                                      reinterpret_cast<float4*>(aos));
  return check_launch();
}

int pgg_debug_em_offsets(const pgg_config* cfg, int8_t* offsets, int32_t* rechecks, void* stream) {
  if (!cfg || !offsets || !rechecks || cfg->width <= 0 || cfg->height <= 0) return PGG_ERR_ARGUMENT;
  PassArgs A;
  memset(&A, 0, sizeof(A));
  A.cfg = *cfg;
  pass_args_finish(A);
  const int64_t P = (int64_t)cfg->width * cfg->height;
  if (const int rc = device_check()) return rc;
  k_debug_em_offsets<<<blocks(P, 256), 256, 0, S(stream)>>>(A, offsets, rechecks);
  return check_launch();
}

int pgg_debug_trunc_bvn(int64_t n, const double* mu, const double* cov, double* z, void* stream) {
  if (n < 0 || !mu || !cov || !z) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_debug_trunc_bvn<<<blocks(n, 128), 128, 0, S(stream)>>>(n, mu, cov, z);
  return check_launch();
}

int pgg_debug_bm_accept(int64_t n, int32_t per_lobe, const float* stats, const uint32_t* draws, uint8_t* out,
                        float* proposals, int32_t* rechecks, void* stream) {
  if (n < 0 || per_lobe < 1 || !stats || !draws || !out || !rechecks) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_debug_bm_accept<<<blocks(n, 256), 256, 0, S(stream)>>>(n, per_lobe, stats, draws, out, proposals, rechecks);
  return check_launch();
}

int pgg_debug_brdf_draw(int64_t n, const uint8_t* glossy, const float* rough, const float* wo, const uint32_t* draws,
                        float* out, int32_t* rechecks, void* stream) {
  if (n < 0 || !glossy || !rough || !wo || !draws || !out || !rechecks) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_debug_brdf_draw<<<blocks(n, 256), 256, 0, S(stream)>>>(n, glossy, rough, reinterpret_cast<const float4*>(wo),
                                                           draws, reinterpret_cast<float4*>(out), rechecks);
  return check_launch();
}

int pgg_debug_reproject(const pgg_config* cfg, const pgg_gbuffer* cur, const pgg_gbuffer* prev,
                        const pgg_gamma_in* gamma_prev, uint8_t* decisions, void* stream) {
  if (!cfg || !cur || !prev || !gamma_prev || !decisions) return PGG_ERR_ARGUMENT;
  if (cfg->width <= 0 || cfg->rows < 0 || cfg->row0 < 0 || cfg->row0 + cfg->rows > cfg->height) return PGG_ERR_ARGUMENT;
  if (cfg->rows == 0) return PGG_OK;
  PassArgs A;
  memset(&A, 0, sizeof(A));
  A.cfg = *cfg;
  pass_args_finish(A);
  A.cur = *cur;
  A.prev = *prev;
  A.gin = *gamma_prev;
  A.has_prev = 1;
  if (const int rc = device_check()) return rc;
  k_debug_reproject<<<dim3(blocks(cfg->width, 128), cfg->rows), 128, 0, S(stream)>>>(A, decisions);
  return check_launch();
}

int pgg_mixture_lanes(int32_t op, int64_t n, const double* a, const double* b, const double* c, const double* d,
                      const double* e, double* out0, double* out1, int32_t k_max, void* stream) {
  if (n < 0 || op < 0 || op > 4 || !a || !out0) return PGG_ERR_ARGUMENT;
  if ((op == MIX_GAUSS_PDF || op == MIX_PDF) && (!b || !c || !d)) return PGG_ERR_ARGUMENT;
  if (op == MIX_BOX_MULLER && (!b || !out1)) return PGG_ERR_ARGUMENT;
  if (op == MIX_E_STEP && (!b || !c)) return PGG_ERR_ARGUMENT;
  if (op == MIX_NEIGHBORS && k_max < 1) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_mixture_lanes<<<blocks(n, 128), 128, 0, S(stream)>>>(op, n, a, b, c, d, e, out0, out1, k_max);
  return check_launch();
}

int pgg_sample_gauss(int64_t n, const double* pi, const double* mu, const double* chol, uint64_t* states, double* sq,
                     uint8_t* accepted, void* stream) {
  if (n < 0 || !pi || !mu || !chol || !states || !sq || !accepted) return PGG_ERR_ARGUMENT;
  if (n == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_sample_gauss<<<blocks(n, 128), 128, 0, S(stream)>>>(n, pi, mu, chol, states, sq, accepted);
  return check_launch();
}

int pgg_debug_checks(int32_t* host_out6, int32_t reset) {
#if PGG_CHECKS
  if (!host_out6) return PGG_ERR_ARGUMENT;
  cudaError_t e = cudaMemcpyFromSymbol(host_out6, g_pgg_check, 6 * sizeof(int32_t));
  if (e == cudaSuccess && reset) {
    const int32_t z[6] = {0, 0, 0, 0, 0, 0};
    e = cudaMemcpyToSymbol(g_pgg_check, z, sizeof(z));
  }
  if (e != cudaSuccess) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s", cudaGetErrorString(e));
    return PGG_ERR_CUDA;
  }
  return PGG_OK;
#else
  (void)host_out6;
  (void)reset;
  return PGG_ERR_UNSUPPORTED;  // not a checked build
#endif
}

int pgg_gamma_init(int64_t p, float* g0, float* g1, void* stream) {
  if (p < 0 || !g0 || !g1) return PGG_ERR_ARGUMENT;
  if (p == 0) return PGG_OK;
  if (const int rc = device_check()) return rc;
  k_gamma_init<<<blocks(p, 256), 256, 0, S(stream)>>>(p, reinterpret_cast<float4*>(g0), reinterpret_cast<float4*>(g1));
  return check_launch();
}

}  // extern "C"
