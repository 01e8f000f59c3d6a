// Shared device helpers of the dock-and-score kernels (vs_dock.cu,
// vs_kernels.cu): RNG, TMA bulk staging, field/wall/pair terms, per-warp
// shared-memory layout, torsion chain, sweep key, start draws.
#pragma once
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "vs_detmath.cuh"
#include "vs_types.h"

namespace vs {

// The pocket reaches every kernel as a `const __grid_constant__ PocketDev`
// launch parameter (constant bank, uniform loads); the helpers below read it
// through a reference to that parameter.  No process-wide device state, so
// concurrent handles and streams never see each other's pocket.

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned long long kGolden = 0x9e3779b97f4a7c15ull;
constexpr double kPiD = 3.14159265358979323846;
constexpr double kHalfPiD = 1.57079632679489661923;
constexpr float kPiF = 3.14159274f;     // (float)pi, rounds up
constexpr float kHalfPiF = 1.57079637f;  // (float)(pi / 2)
constexpr float kTwoPiF = 6.28318548f;  // (float)(2 pi)

// ------------------------------------------------------------------ RNG --
// Counter-based splitmix64 of rng.hpp:14-41, evaluated at an explicit
// counter so that any draw of any start attempt is random-access.
__device__ __forceinline__ unsigned long long rng_mix(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned long long rng_draw(unsigned long long key,
                                                       unsigned long long ctr) {
  return rng_mix(key + kGolden * ctr);
}
__device__ __forceinline__ double rng_unit(unsigned long long u) {
  return static_cast<double>(u >> 11) * 0x1.0p-53;
}

// ------------------------------------------------------ TMA bulk staging --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---------------------------------------------------------------- field --
__device__ __forceinline__ float site_sum(const SiteF* __restrict__ s, int n, float x, float y,
                                          float z) {
  float acc = 0.0f;
  for (int k = 0; k < n; ++k) {
    const float4 c = *reinterpret_cast<const float4*>(&s[k].cx);
    const float inv = s[k].inv2s2;
    const float dx = x - c.x, dy = y - c.y, dz = z - c.z;
    const float e = det_exp_neg(-(det_norm2(dx, dy, dz) * inv));
    acc = fmaf(c.w, e, acc);
  }
  return acc;
}

// One corner-packed cell (32 B, one sector) in a single 256-bit load
// (LDG.E.ENL2.256 on sm_100a): one L1 request per lookup instead of two.
__device__ __forceinline__ void ldg_cell(const float4* c, float4& lo, float4& hi) {
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(lo.x), "=f"(lo.y), "=f"(lo.z), "=f"(lo.w), "=f"(hi.x), "=f"(hi.y),
                 "=f"(hi.z), "=f"(hi.w)
               : "l"(c));
}

// One FP16 corner cell (16 B, LDG.128), widened to FP32 exactly.
__device__ __forceinline__ void ldg_hcell(const uint4* c, float4& lo, float4& hi) {
  uint4 u;
  asm("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
      : "l"(c));
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  const float2 d = __half22float2(*reinterpret_cast<const __half2*>(&u.z));
  const float2 e = __half22float2(*reinterpret_cast<const __half2*>(&u.w));
  lo = make_float4(a.x, a.y, b.x, b.y);
  hi = make_float4(d.x, d.y, e.x, e.y);
}

// the same cell through the texture path (TEX: its own L1 data pipe)
__device__ __forceinline__ void tex_hcell(unsigned long long tex, unsigned idx, float4& lo,
                                          float4& hi) {
  const uint4 u = tex1Dfetch<uint4>(static_cast<cudaTextureObject_t>(tex), static_cast<int>(idx));
  const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
  const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
  const float2 d = __half22float2(*reinterpret_cast<const __half2*>(&u.z));
  const float2 e = __half22float2(*reinterpret_cast<const __half2*>(&u.w));
  lo = make_float4(a.x, a.y, b.x, b.y);
  hi = make_float4(d.x, d.y, e.x, e.y);
}

// floor(g) and its integer value for a cell lookup without the XU pipe:
// y = 2^23 + g rounded toward zero (FADD.RZ, FMA pipe) holds floor(g) in its
// low mantissa bits for 0 <= g < 2^23, so floor(g) = y - 2^23 exactly and
// i = bits(y) - bits(2^23).  Every g < 0 gives i < 0 (or, below -2^23, a
// value above any grid extent when read unsigned), i.e. "off the grid" as
// floorf would: the in-grid decision and, in the grid, the fraction g -
// floor(g) are bit-identical to floorf / F2I (which run on the quarter-rate
// XU pipe, 6 per lookup).
__device__ __forceinline__ int floor_cell(float g, float* fl) {
  const float y = __fadd_rz(g, 8388608.0f);
  *fl = y - 8388608.0f;
  return __float_as_int(y) - 0x4B000000;
}

// Packed FP32 pairs (sm_100a FFMA2 / FADD2): two IEEE FP32 operations per
// instruction, each element rounded exactly as its scalar form, so code
// written with them gives the scalar code's bits with fewer issue slots.
// A pair built from one scalar (f2s) becomes ptxas's broadcast operand.
__device__ __forceinline__ unsigned long long f2pack(float2 v) {
  unsigned long long u;
  asm("mov.b64 %0, {%1, %2};" : "=l"(u) : "f"(v.x), "f"(v.y));
  return u;
}
__device__ __forceinline__ float2 f2unpack(unsigned long long u) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(u));
  return v;
}
__device__ __forceinline__ float2 f2s(float x) { return make_float2(x, x); }
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {  // a * b + c, .rn
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2pack(a)), "l"(f2pack(b)), "l"(f2pack(c)));
  return f2unpack(d);
}
__device__ __forceinline__ float2 f2add_rz(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rz.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2pack(a)), "l"(f2pack(b)));
  return f2unpack(d);
}
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {  // a - b, .rn
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2pack(a)), "l"(f2pack(b)));
  return f2unpack(d);
}

// One trilinear lookup split in two halves so that callers can issue the
// next lookup's loads before consuming this one.
struct TriCell {
  float4 lo, hi;  // corners (000,100,010,110), (001,101,011,111)
  float tx, ty, tz;
  bool in;
};

// address + fractional part + the two cell loads (issued, not consumed)
__device__ __forceinline__ TriCell tri_issue(const GridDev& g, const float4* __restrict__ cells,
                                             float x, float y, float z) {
  const float gx = (x - g.ox) * g.inv_h;
  const float gy = (y - g.oy) * g.inv_h;
  const float gz = (z - g.oz) * g.inv_h;
  float fx, fy, fz;
  const int ix = floor_cell(gx, &fx), iy = floor_cell(gy, &fy), iz = floor_cell(gz, &fz);
  // gx < 0 <=> ix < 0 (floor), so one unsigned compare per axis covers both
  // ends; out-of-grid lanes read cell 0 and are zeroed (no divergent branch)
  TriCell c;
  c.in = static_cast<unsigned>(ix) <= static_cast<unsigned>(g.nx - 2) &&
         static_cast<unsigned>(iy) <= static_cast<unsigned>(g.ny - 2) &&
         static_cast<unsigned>(iz) <= static_cast<unsigned>(g.nz - 2);
  c.tx = gx - fx;
  c.ty = gy - fy;
  c.tz = gz - fz;
  const unsigned cell = static_cast<unsigned>(iz * g.cxy + iy * g.cx + ix);
  ldg_cell(cells + 2 * (c.in ? cell : 0u), c.lo, c.hi);
  return c;
}

__device__ __forceinline__ float tri_finish(const TriCell& c) {
  const float c00 = det_lerp(c.lo.x, c.lo.y, c.tx), c10 = det_lerp(c.lo.z, c.lo.w, c.tx);
  const float c01 = det_lerp(c.hi.x, c.hi.y, c.tx), c11 = det_lerp(c.hi.z, c.hi.w, c.tx);
  const float c0 = det_lerp(c00, c10, c.ty), c1 = det_lerp(c01, c11, c.ty);
  return c.in ? det_lerp(c0, c1, c.tz) : 0.0f;
}

// Trilinear interpolation on one corner-packed cell (two 16 B loads of the
// same 32 B sector).  Same corner values and lerp order as the node layout,
// so the result is bit-identical to interpolating the node map.
__device__ __forceinline__ float trilinear(const GridDev& g, const float4* __restrict__ cells,
                                           float x, float y, float z) {
  return tri_finish(tri_issue(g, cells, x, y, z));
}

template <int kGrid>
__device__ __forceinline__ float field_steric(const PocketDev& pk, float x, float y, float z) {
  if (kGrid) return trilinear(pk.grid, pk.grid.steric_c, x, y, z);
  return site_sum(pk.sites, pk.n_steric, x, y, z);
}

// kind bonus of rescore (dock.cpp:304-314): C -> lipophilic, N/O -> hbond
template <int kGrid>
__device__ __forceinline__ float atom_bonus(const PocketDev& pk, int cls, float x, float y,
                                            float z) {
  if (cls == 1) {
    if (kGrid) return trilinear(pk.grid, pk.grid.lipo_c, x, y, z);
    return site_sum(pk.sites + pk.n_steric + pk.n_hbond, pk.n_lipo, x, y, z);
  }
  if (cls == 2) {
    if (kGrid) return trilinear(pk.grid, pk.grid.hbond_c, x, y, z);
    return site_sum(pk.sites + pk.n_steric, pk.n_hbond, x, y, z);
  }
  return 0.0f;
}

// wall softplus of one atom (dock.cpp:31-44, 98-101)
__device__ __forceinline__ float wall_of(const PocketDev& P, float x, float y, float z) {
  const float d0 = x - P.lo[0], d1 = P.hi[0] - x;
  const float d2 = y - P.lo[1], d3 = P.hi[1] - y;
  const float d4 = z - P.lo[2], d5 = P.hi[2] - z;
  const float w = fminf(fminf(fminf(d0, d1), fminf(d2, d3)), fminf(d4, d5));
  return det_softplus((P.r - w) * 10.0f);
}
__device__ __forceinline__ float wall_term(const PocketDev& pk, float x, float y, float z) {
  return wall_of(pk, x, y, z);
}

// pair clash softplus (dock.cpp:86-97) from an FP64 difference
__device__ __forceinline__ float pair_term_d(const PocketDev& pk, double dx, double dy,
                                             double dz) {
  const double d2 = det_norm2_d(dx, dy, dz);
  if (d2 > pk.cut2_d) return 0.0f;
  return det_softplus((pk.r - sqrtf(static_cast<float>(d2))) * 10.0f);
}
// clash softplus of a pair inside the cutoff, from its FP64 squared distance
__device__ __forceinline__ float pair_soft(const PocketDev& pk, double d2) {
  return det_softplus((pk.r - sqrtf(static_cast<float>(d2))) * 10.0f);
}
// search-only pair term (SWEEP_V1.md §3.4): the clash softplus of a pair
// inside the cutoff read from the d^2 table by linear interpolation
__device__ __forceinline__ float pair_soft_tab(const PocketDev& pk, const float2* tab, double d2) {
  const float x = static_cast<float>(d2) * pk.soft_inv_h;
  const int i = min(static_cast<int>(x), kSoftN - 1);
  const float2 e = tab[i];
  return fmaf(x - static_cast<float>(i), e.y, e.x);
}
// cross pair of the flex search from FP32 coordinates (SWEEP_V1.md §3.4):
// FP32 squared distance, FP32 cutoff, tabulated softplus
__device__ __forceinline__ float pair_term_f(const PocketDev& pk, const float2* tab, float dx, float dy, float dz,
                                             int& n_active) {
  const float d2 = det_norm2(dx, dy, dz);
  if (d2 > pk.cut2) return 0.0f;
  ++n_active;
  const float x = d2 * pk.soft_inv_h;
  const int i = min(static_cast<int>(x), kSoftN - 1);
  const float2 e = tab[i];
  return fmaf(x - static_cast<float>(i), e.y, e.x);
}
// pair term of the flex search: tabulated (kTab) or exact, counting pairs
// inside the cutoff (work counter)
template <bool kTab>
__device__ __forceinline__ float pair_term_s(const PocketDev& pk, const float2* tab, double dx, double dy, double dz,
                                             int& n_active) {
  const double d2 = det_norm2_d(dx, dy, dz);
  if (d2 > pk.cut2_d) return 0.0f;
  ++n_active;
  return kTab ? pair_soft_tab(pk, tab, d2) : pair_soft(pk, d2);
}
// same as pair_term_d, counting the pairs inside the cutoff (work counter)
__device__ __forceinline__ float pair_term_d(const PocketDev& pk, double dx, double dy, double dz,
                                             int& n_active) {
  const double d2 = det_norm2_d(dx, dy, dz);
  if (d2 > pk.cut2_d) return 0.0f;
  ++n_active;
  return pair_soft(pk, d2);
}

// per-atom field + wall of local coordinate y under (R, t), FP64 transform
template <int kGrid>
__device__ __forceinline__ void atom_terms(const PocketDev& pk, const Mat3d& R, double tx,
                                           double ty, double tz, double yx, double yy, double yz,
                                           float* f, float* w, float* xo = nullptr) {
  double x, y, z;
  det_apply_d(R, yx, yy, yz, tx, ty, tz, &x, &y, &z);
  const float xf = static_cast<float>(x), yf = static_cast<float>(y), zf = static_cast<float>(z);
  *f = field_steric<kGrid>(pk, xf, yf, zf);
  *w = wall_term(pk, xf, yf, zf);
  if (xo) {
    xo[0] = xf;
    xo[1] = yf;
    xo[2] = zf;
  }
}

// same, with the warp-uniform transform read from shared memory at each use
// (keeps 24 FP64 registers free in the flex loops)
template <int kGrid>
__device__ __forceinline__ void atom_terms_s(const PocketDev& pk, const double* pm, double yx, double yy, double yz,
                                             float* f, float* w) {
  const volatile double* v = pm;
  const double x = fma(v[0], yx, fma(v[1], yy, fma(v[2], yz, v[9])));
  const double y = fma(v[3], yx, fma(v[4], yy, fma(v[5], yz, v[10])));
  const double z = fma(v[6], yx, fma(v[7], yy, fma(v[8], yz, v[11])));
  const float xf = static_cast<float>(x), yf = static_cast<float>(y), zf = static_cast<float>(z);
  *f = field_steric<kGrid>(pk, xf, yf, zf);
  *w = wall_term(pk, xf, yf, zf);
}

__device__ __forceinline__ float warp_sum(float v) {
  for (int off = 16; off > 0; off >>= 1) v = v + __shfl_xor_sync(kFull, v, off);
  return v;
}

// ------------------------------------------------- per-warp shared layout --
// rescore kernel: kCand pose columns per warp, kLanesPerPose lanes each
constexpr int kCand = 4;
constexpr int kLanesPerPose = 8;

struct WarpSmem {
  double4* y0;    // conformer (x, y, z, class), FP64
  double4* ys;    // state local coordinates (torsions applied), FP64
  double* pose;   // flex: posed transform R (row-major 9) and t (3), FP64, warp-uniform
  float4* ysf;    // FP32 copy of the state (sweep); with kLayPairs followed by
                  // its atom pairs (pairs_of)
  float4* xf;     // posed coordinates under test (FP32, decisions)
  float* fa;      // per-atom field term of the posed state
  float* wa;      // per-atom wall term of the posed state
  int4* ax;       // torsion axes
  float* theta;   // state torsions
  uint8_t* mov;   // moving lists
  unsigned* mask; // all-zero moving set (4 words; rigid ligands)
  unsigned* tmask;  // moving set of each torsion (4 words per torsion)
  double* axl;      // 1 / |y0[b_j] - y0[a_j]| per torsion (0 for a degenerate axis)
  double* col;    // rescore kernel only: pose columns [i][c][16], FP64
  float* kscore;  // kept-pose scores
  int* kinv;      // rank -> kept index
  float* kresc;   // survivor rescores by rank
  uint64_t* bar;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Layout parts: a kernel carves only the arrays its phases touch.
enum : int {
  kLayLig = 1,     // y0, ax, mov, mask, tmask, axl (ligand topology)
  kLayState = 2,   // ys (FP64 state), theta
  kLaySweep = 4,   // ysf
  kLayPosed = 8,   // xf
  kLayFlex = 16,   // pose, fa, wa
  kLayKept = 32,   // kscore, kinv, kresc
  kLayCols = 64,   // rescore pose columns
  // ysf and xf alias the conformer y0 (a kernel that no longer needs y0
  // after staging: the flex kernel) -> 32 B/atom less shared memory, more L1
  kLayAliasY0 = 128,
  kLayPairs = 256,  // ysf's atom pairs (the grid-mode sweep key, eval_key)
  kLayAll = kLayLig | kLayState | kLaySweep | kLayPosed | kLayFlex | kLayKept,
};

// byte offsets of every part (0 size when absent), in carve order
__host__ __device__ inline size_t warp_layout(int nmax, int tmax, int mvmax, int lay,
                                              size_t* off) {
  const size_t n = size_t(nmax), t = size_t(tmax);
  const size_t sz[18] = {
      (lay & kLayLig) ? 32 * n : 0,                 // 0 y0
      (lay & kLayState) ? 32 * n : 0,               // 1 ys
      (lay & kLayFlex) ? size_t(96) : 0,                    // 2 pose
      (lay & kLaySweep) && !(lay & kLayAliasY0)
          ? 16 * n + ((lay & kLayPairs) ? 16 * ((n + 1) / 2) + align16(8 * ((n + 1) / 2)) : 0)
          : 0,                                      // 3 ysf (+ pairs)
      (lay & kLayPosed) && !(lay & kLayAliasY0) ? 16 * n : 0,  // 4 xf
      (lay & kLayFlex) ? align16(4 * n) : 0,        // 5 fa
      (lay & kLayFlex) ? align16(4 * n) : 0,        // 6 wa
      (lay & kLayLig) ? 16 * t : 0,                 // 7 ax
      (lay & kLayState) ? align16(4 * t) : 0,       // 8 theta
      (lay & kLayLig) ? align16(size_t(mvmax)) : 0, // 9 mov
      (lay & kLayLig) ? size_t(16) : 0,                     // 10 mask
      (lay & kLayLig) ? 16 * t : 0,                 // 11 tmask
      (lay & kLayLig) ? align16(8 * t) : 0,         // 12 axl
      (lay & kLayCols) ? 8 * n * 3 * kCand : 0,     // 13 col
      (lay & kLayKept) ? size_t(4 * kMaxRestarts) : 0,      // 14 kscore
      (lay & kLayKept) ? size_t(4 * kMaxRestarts) : 0,      // 15 kinv
      (lay & kLayKept) ? size_t(4 * kMaxRestarts) : 0,      // 16 kresc
      16};                                          // 17 mbarrier
  size_t o = 0;
  for (int k = 0; k < 18; ++k) {
    if (off) off[k] = o;
    o += sz[k];
  }
  return o;
}

__host__ __device__ inline size_t warp_smem_bytes(int nmax, int tmax, int mvmax, int lay) {
  return (warp_layout(nmax, tmax, mvmax, lay, nullptr) + 127) & ~size_t(127);  // 128 B bases
}

__device__ inline WarpSmem carve(unsigned char* base, int nmax, int tmax, int mvmax, int lay) {
  size_t o[18];
  warp_layout(nmax, tmax, mvmax, lay, o);
  WarpSmem s;
  s.y0 = (lay & kLayLig) ? reinterpret_cast<double4*>(base + o[0]) : nullptr;
  s.ys = (lay & kLayState) ? reinterpret_cast<double4*>(base + o[1]) : nullptr;
  s.pose = (lay & kLayFlex) ? reinterpret_cast<double*>(base + o[2]) : nullptr;
  s.ysf = (lay & kLaySweep) ? reinterpret_cast<float4*>(base + o[3]) : nullptr;
  s.xf = (lay & kLayPosed) ? reinterpret_cast<float4*>(base + o[4]) : nullptr;
  if ((lay & kLayAliasY0) && (lay & kLayLig)) {
    if (lay & kLaySweep) s.ysf = reinterpret_cast<float4*>(base + o[0]);
    if (lay & kLayPosed) s.xf = reinterpret_cast<float4*>(base + o[0] + 16 * size_t(nmax));
  }
  s.fa = (lay & kLayFlex) ? reinterpret_cast<float*>(base + o[5]) : nullptr;
  s.wa = (lay & kLayFlex) ? reinterpret_cast<float*>(base + o[6]) : nullptr;
  s.ax = (lay & kLayLig) ? reinterpret_cast<int4*>(base + o[7]) : nullptr;
  s.theta = (lay & kLayState) ? reinterpret_cast<float*>(base + o[8]) : nullptr;
  s.mov = (lay & kLayLig) ? base + o[9] : nullptr;
  s.mask = (lay & kLayLig) ? reinterpret_cast<unsigned*>(base + o[10]) : nullptr;
  s.tmask = (lay & kLayLig) ? reinterpret_cast<unsigned*>(base + o[11]) : nullptr;
  s.axl = (lay & kLayLig) ? reinterpret_cast<double*>(base + o[12]) : nullptr;
  s.col = (lay & kLayCols) ? reinterpret_cast<double*>(base + o[13]) : nullptr;
  s.kscore = (lay & kLayKept) ? reinterpret_cast<float*>(base + o[14]) : nullptr;
  s.kinv = (lay & kLayKept) ? reinterpret_cast<int*>(base + o[15]) : nullptr;
  s.kresc = (lay & kLayKept) ? reinterpret_cast<float*>(base + o[16]) : nullptr;
  s.bar = reinterpret_cast<uint64_t*>(base + o[17]);
  return s;
}

// Stage one ligand's atoms, axes and moving lists with TMA bulk copies.
__device__ inline void stage_ligand(const LibDev& lib, int lig, const WarpSmem& s, int lane,
                                    uint32_t& phase, int4& meta) {
  meta = lib.meta[lig];
  const int2 mv = lib.mov[lig];
  __syncwarp();
  if (lane == 0) {
    fence_proxy_async();
    const uint32_t bytes = 32u * meta.y + 16u * meta.w + static_cast<uint32_t>(mv.y);
    mbar_expect_tx(s.bar, bytes);
    bulk_g2s(s.y0, lib.atoms + meta.x, 32u * meta.y, s.bar);
    if (meta.w > 0) bulk_g2s(s.ax, lib.axes + meta.z, 16u * meta.w, s.bar);
    if (mv.y > 0) bulk_g2s(s.mov, lib.moving + mv.x, static_cast<uint32_t>(mv.y), s.bar);
  }
  mbar_wait(s.bar, phase);
  phase ^= 1u;
  // per-ligand torsion tables: moving-set bitmasks and inverse axis lengths
  // of the conformer (the axis length is invariant under the torsion chain)
  const int T = meta.w;
  if (lane < 4) s.mask[lane] = 0u;
  for (int e = lane; e < 4 * T; e += 32) {
    const int j = e >> 2, w = e & 3;
    const int4 a = s.ax[j];
    unsigned bits = 0u;
    for (int q = 0; q < a.w; ++q) {
      const int idx = s.mov[a.z + q];
      if ((idx >> 5) == w) bits |= 1u << (idx & 31);
    }
    s.tmask[e] = bits;
  }
  for (int j = lane; j < T; j += 32) {
    const int4 a = s.ax[j];
    const double4 o = s.y0[a.x], b = s.y0[a.y];
    const double n = sqrt(det_norm2_d(b.x - o.x, b.y - o.y, b.z - o.z));
    s.axl[j] = n > 0.0 ? 1.0 / n : 0.0;
  }
  __syncwarp();
}

// s.ys = y0 with torsions [0, T) at s.theta (dock.cpp:54-63); lanes over
// the moving atoms of each torsion in turn.
static __device__ __noinline__ void chain_coop(const WarpSmem& s, int N, int T, int lane) {
  for (int i = lane; i < N; i += 32) s.ys[i] = s.y0[i];
  __syncwarp();
  for (int j = 0; j < T; ++j) {
    const int4 a = s.ax[j];
    const double4 o = s.ys[a.x], b = s.ys[a.y];
    const Mat3d M = det_torsion_mat_d(o.x, o.y, o.z, b.x, b.y, b.z, s.theta[j], s.axl[j]);
    for (int m = lane; m < a.w; m += 32) {
      const int idx = s.mov[a.z + m];
      double4 v = s.ys[idx];
      det_apply_d(M, v.x - o.x, v.y - o.y, v.z - o.z, o.x, o.y, o.z, &v.x, &v.y, &v.z);
      s.ys[idx] = v;
    }
    __syncwarp();
  }
}

// s.xf = (float)(R s.ys + t) over all atoms (lanes over atoms)
static __device__ __noinline__ void pose_coop(const WarpSmem& s, int N, const Mat3d& R, double tx, double ty,
                                 double tz, int lane) {
  for (int i = lane; i < N; i += 32) {
    const double4 v = s.ys[i];
    double x, y, z;
    det_apply_d(R, v.x, v.y, v.z, tx, ty, tz, &x, &y, &z);
    s.xf[i] = make_float4(static_cast<float>(x), static_cast<float>(y), static_cast<float>(z), 0.0f);
  }
  __syncwarp();
}

// Sweep key of one rigid pose over the FP32 state copy (SWEEP_V1.md §2.3),
// one atom (analytic) or one atom pair (grid) per iteration and never
// unrolled, so the loop body stays resident in the ~6 KB L0 instruction
// cache next to the other warps' flex loops.
//  analytic: F - lam W (parity sums of field and wall)
//  grid:     sum of the key map K = S - lam W interpolated at the atom, the
//            pose composed with the grid frame (g = (R/h) y + (t - o)/h) so
//            one FMA chain yields cell coordinates; atoms off the grid score
//            the linear wall -lam * 10 (r - w) at x = g h + o.
__device__ __forceinline__ float off_grid_term(const PocketDev& pk, float gx, float gy, float gz) {
  // -lam * 10 (r - w), w the (negative) signed distance to the box: the wall
  // softplus at z = 10 (r - w) >= 10 (r + pad) is z to ~1e-11 there
  const GridDev& g = pk.grid;
  const float x = fmaf(gx, g.h, g.ox), y = fmaf(gy, g.h, g.oy), z = fmaf(gz, g.h, g.oz);
  const float w = fminf(fminf(fminf(x - pk.lo[0], pk.hi[0] - x),
                              fminf(y - pk.lo[1], pk.hi[1] - y)),
                        fminf(z - pk.lo[2], pk.hi[2] - z));
  return -(pk.lam * ((pk.r - w) * 10.0f));
}

// The atoms a sweep key reads: the FP32 state (analytic mode) and its atom
// pairs (grid mode, built by build_pairs).
struct KeyAtoms {
  const float4* ysf;
  const float4* p4;
  const float2* p2;
};

// ysf[nmax] is followed (kLayPairs) by the atom pairs: (x0, x1, y0, y1)
// float4s, then (z0, z1) float2s; an odd last pair repeats the last atom
__device__ __forceinline__ KeyAtoms pairs_of(const float4* ysf, int nmax) {
  const float4* p4 = ysf + nmax;
  return KeyAtoms{ysf, p4, reinterpret_cast<const float2*>(p4 + (nmax + 1) / 2)};
}

// the pairs from ysf: lanes over atom pairs
__device__ __forceinline__ void build_pairs(const KeyAtoms& ka, int N, int lane) {
  float4* p4 = const_cast<float4*>(ka.p4);
  float2* p2 = const_cast<float2*>(ka.p2);
  for (int j = lane; j < (N + 1) / 2; j += 32) {
    const float4 a = ka.ysf[2 * j], b = ka.ysf[2 * j + 1 < N ? 2 * j + 1 : N - 1];
    p4[j] = make_float4(a.x, b.x, a.y, b.y);
    p2[j] = make_float2(a.z, b.z);
  }
  __syncwarp();
}

// Grid mode takes two atoms per iteration in FP32 pairs (FFMA2 / FADD2:
// the transform, the cell floor and fraction, the cell polynomial), every
// element the scalar operation of SWEEP_V1.md §2.3, and sums the atom terms
// in atom order into one FP32 accumulator: the key bits of the one-atom
// form with ~30 % fewer issued instructions.  An odd last pair repeats the
// last atom and drops its term.
template <int kGrid, bool kTex = false>
static __device__ __forceinline__ float eval_key(const PocketDev& pk, const KeyAtoms& A, int N,
                                                 const Mat3 R, float tx, float ty, float tz) {
  if (kGrid) {
    const GridDev& g = pk.grid;
    const float ih = g.inv_h;
    const float a00 = R.m00 * ih, a01 = R.m01 * ih, a02 = R.m02 * ih;
    const float a10 = R.m10 * ih, a11 = R.m11 * ih, a12 = R.m12 * ih;
    const float a20 = R.m20 * ih, a21 = R.m21 * ih, a22 = R.m22 * ih;
    const float ux = (tx - g.ox) * ih, uy = (ty - g.oy) * ih, uz = (tz - g.oz) * ih;
    const unsigned mx = static_cast<unsigned>(g.nx - 2), my = static_cast<unsigned>(g.ny - 2),
                   mz = static_cast<unsigned>(g.nz - 2);
    const float2 M23 = f2s(8388608.0f);
    float k = 0.0f;
#pragma unroll 1
    for (int i0 = 0; i0 < N; i0 += 2) {
      const float4 xy = A.p4[i0 >> 1];
      const float2 Z = A.p2[i0 >> 1];
      const float2 X = make_float2(xy.x, xy.y), Y = make_float2(xy.z, xy.w);
      const float2 GX = f2fma(f2s(a00), X, f2fma(f2s(a01), Y, f2fma(f2s(a02), Z, f2s(ux))));
      const float2 GY = f2fma(f2s(a10), X, f2fma(f2s(a11), Y, f2fma(f2s(a12), Z, f2s(uy))));
      const float2 GZ = f2fma(f2s(a20), X, f2fma(f2s(a21), Y, f2fma(f2s(a22), Z, f2s(uz))));
      // floor_cell of both atoms: y = g + 2^23 (RZ), floor = y - 2^23
      const float2 FX = f2add_rz(GX, M23), FY = f2add_rz(GY, M23), FZ = f2add_rz(GZ, M23);
      const int ix0 = __float_as_int(FX.x) - 0x4B000000, ix1 = __float_as_int(FX.y) - 0x4B000000;
      const int iy0 = __float_as_int(FY.x) - 0x4B000000, iy1 = __float_as_int(FY.y) - 0x4B000000;
      const int iz0 = __float_as_int(FZ.x) - 0x4B000000, iz1 = __float_as_int(FZ.y) - 0x4B000000;
      const bool in0 = static_cast<unsigned>(ix0) <= mx && static_cast<unsigned>(iy0) <= my &&
                       static_cast<unsigned>(iz0) <= mz;
      const bool in1 = static_cast<unsigned>(ix1) <= mx && static_cast<unsigned>(iy1) <= my &&
                       static_cast<unsigned>(iz1) <= mz;
      const unsigned c0 = static_cast<unsigned>(iz0 * g.cxy + iy0 * g.cx + ix0);
      const unsigned c1 = static_cast<unsigned>(iz1 * g.cxy + iy1 * g.cx + ix1);
      float4 lo0, hi0, lo1, hi1;
      if (kTex) {
        tex_hcell(g.key_tex, in0 ? c0 : 0u, lo0, hi0);
        tex_hcell(g.key_tex, in1 ? c1 : 0u, lo1, hi1);
      } else {
        ldg_hcell(g.key_h + (in0 ? c0 : 0u), lo0, hi0);
        ldg_hcell(g.key_h + (in1 ? c1 : 0u), lo1, hi1);
      }
      const float2 TX = f2sub(GX, f2sub(FX, M23)), TY = f2sub(GY, f2sub(FY, M23)),
                   TZ = f2sub(GZ, f2sub(FZ, M23));
      // the cells' trilinear polynomials (vs_pack_half_kernel), 7 FFMA2
      const float2 Pw = f2fma(make_float2(hi0.w, hi1.w), TZ, make_float2(lo0.w, lo1.w));
      const float2 Py = f2fma(make_float2(hi0.y, hi1.y), TZ, make_float2(lo0.y, lo1.y));
      const float2 Pz = f2fma(make_float2(hi0.z, hi1.z), TZ, make_float2(lo0.z, lo1.z));
      const float2 Px = f2fma(make_float2(hi0.x, hi1.x), TZ, make_float2(lo0.x, lo1.x));
      const float2 Tm = f2fma(f2fma(Pw, TY, Py), TX, f2fma(Pz, TY, Px));
      k = k + (in0 ? Tm.x : off_grid_term(pk, GX.x, GY.x, GZ.x));
      if (i0 + 1 < N) k = k + (in1 ? Tm.y : off_grid_term(pk, GX.y, GY.y, GZ.y));
    }
    return k;
  }
  const float4* ys = A.ysf;
  float fe = 0.0f, fo = 0.0f, we = 0.0f, wo = 0.0f;
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    const float4 a = ys[i];
    float x, y, z;
    det_apply(R, a.x, a.y, a.z, tx, ty, tz, &x, &y, &z);
    const float f = field_steric<kGrid>(pk, x, y, z);
    const float w = wall_term(pk, x, y, z);
    if (i & 1) {
      fo = fo + f;
      wo = wo + w;
    } else {
      fe = fe + f;
      we = we + w;
    }
  }
  return (fe + fo) - pk.lam * (we + wo);
}

// the sweep key at grid coordinates g (the FP32 flex search, SWEEP_V1.md
// §3.4): the key map's cell polynomial, or the linear wall off the grid,
// as in eval_key
__device__ __forceinline__ float key_at_grid(const PocketDev& pk, float gx, float gy, float gz) {
  const GridDev& g = pk.grid;
  float fx, fy, fz;
  const int ix = floor_cell(gx, &fx), iy = floor_cell(gy, &fy), iz = floor_cell(gz, &fz);
  const bool in = static_cast<unsigned>(ix) <= static_cast<unsigned>(g.nx - 2) &&
                  static_cast<unsigned>(iy) <= static_cast<unsigned>(g.ny - 2) &&
                  static_cast<unsigned>(iz) <= static_cast<unsigned>(g.nz - 2);
  if (!in) return off_grid_term(pk, gx, gy, gz);
  float4 a, b;
  ldg_hcell(g.key_h + static_cast<unsigned>(iz * g.cxy + iy * g.cx + ix), a, b);
  const float tx1 = gx - fx, ty1 = gy - fy, tz1 = gz - fz;
  return fmaf(fmaf(fmaf(b.w, tz1, a.w), ty1, fmaf(b.y, tz1, a.y)), tx1,
              fmaf(fmaf(b.z, tz1, a.z), ty1, fmaf(b.x, tz1, a.x)));
}

// all kept poses at RMSD >= delta from s.xf (dock.cpp:335-340, 392-401)
static __device__ __noinline__ bool diverse_from_kept(const WarpSmem& s, const float4* kx, int nk, int nmax,
                                         int N, float delta, int lane) {
  bool ok = true;
  for (int k = lane; k < nk; k += 32) {
    const float4* X = kx + static_cast<size_t>(k) * nmax;
    float acc = 0.0f;
    for (int i = 0; i < N; ++i) {
      const float4 a = s.xf[i], b = X[i];
      acc = acc + det_norm2(a.x - b.x, a.y - b.y, a.z - b.z);
    }
    if (sqrtf(acc / static_cast<float>(N)) < delta) ok = false;
  }
  return __all_sync(kFull, ok);
}

// Translation-sweep lattice: l = 0 is the current point, l = 1..26 the
// non-zero offsets of {-1,0,1}^3 in x-fastest order, scaled by sc.
constexpr int kTransIters = 16;
constexpr float kTransMin = 1.0f / 64.0f;
__device__ __forceinline__ void trans_offset(int l, float sc, float* ox, float* oy, float* oz) {
  if (l == 0) {
    *ox = *oy = *oz = 0.0f;
    return;
  }
  const int m = l - 1 < 13 ? l - 1 : l;
  *ox = static_cast<float>(m % 3 - 1) * sc;
  *oy = static_cast<float>((m / 3) % 3 - 1) * sc;
  *oz = static_cast<float>(m / 9 - 1) * sc;
}

// Start attempt `att` of restart key rkey (dock.cpp:346-354): writes
// s.theta and returns t (FP32) and q (FP64-normalized, cast to FP32).
static __device__ __noinline__ void draw_start(const PocketDev& pk, unsigned long long rkey, int att, int T,
                                  const WarpSmem& s, int lane, float* t, float* q) {
  const unsigned long long base = static_cast<unsigned long long>(att) * (11ull + T);
  double tv = 0.0, nv = 0.0;
  for (int l = lane; l < 7 + T; l += 32) {
    if (l < 3) {
      const double u = rng_unit(rng_draw(rkey, base + 1 + l));
      tv = pk.lo_d[l] + (pk.hi_d[l] - pk.lo_d[l]) * u;
    } else if (l < 7) {
      const int m = l - 3;
      const unsigned long long ua = rng_draw(rkey, base + 4 + 2 * m);
      const unsigned long long ub = rng_draw(rkey, base + 5 + 2 * m);
      const double u1 = static_cast<double>((ua >> 11) + 1) * 0x1.0p-53;
      const double u2 = rng_unit(ub);
      nv = sqrt(-2.0 * log(u1)) * cos(2.0 * kPiD * u2);
    } else {
      const double u = rng_unit(rng_draw(rkey, base + 12 + (l - 7)));
      s.theta[l - 7] = static_cast<float>(-kPiD + (kPiD - -kPiD) * u);
    }
  }
  t[0] = static_cast<float>(__shfl_sync(kFull, tv, 0));
  t[1] = static_cast<float>(__shfl_sync(kFull, tv, 1));
  t[2] = static_cast<float>(__shfl_sync(kFull, tv, 2));
  const double w = __shfl_sync(kFull, nv, 3), x = __shfl_sync(kFull, nv, 4),
               y = __shfl_sync(kFull, nv, 5), z = __shfl_sync(kFull, nv, 6);
  const double n = sqrt(w * w + x * x + y * y + z * z);
  if (n > 1e-12) {
    q[0] = static_cast<float>(w / n);
    q[1] = static_cast<float>(x / n);
    q[2] = static_cast<float>(y / n);
    q[3] = static_cast<float>(z / n);
  } else {
    q[0] = 1.0f;
    q[1] = q[2] = q[3] = 0.0f;
  }
  __syncwarp();
}

// Rotation of the flex move: moving_j rotated about the state's axis j by
// delta = th_new - th_old (FP64 of two FP32 angles), unit axis d * inv_len.
// The half angle is folded into [-pi/2, pi/2] by q -> -q (same matrix).
__device__ __forceinline__ Mat3d flex_mat(double ox, double oy, double oz, double bx, double by,
                                          double bz, float th_new, float th_old, double inv_len) {
  const double dx = bx - ox, dy = by - oy, dz = bz - oz;
  double hh = 0.5 * (static_cast<double>(th_new) - static_cast<double>(th_old));
  if (hh > kHalfPiD) hh = hh - kPiD;
  else if (hh < -kHalfPiD) hh = hh + kPiD;
  double s, c;
  det_sincos_d(hh, &s, &c);
  const double ks = s * inv_len;
  return det_quat_mat_d(c, dx * ks, dy * ks, dz * ks);
}

__device__ __forceinline__ bool in_mask(const unsigned* mask, int i) {
  return (mask[i >> 5] >> (i & 31)) & 1u;
}

}  // namespace vs
