// sm_100a kernels of the dock-and-score path.
//
//   vs_dock_kernel     K2+K3+K4a  sweep-v1 pose generation (rigid
//                      roto-translation sweep + incremental torsion flex),
//                      canonical scoring, diversity, keep-top filter,
//                      rescore, per-ligand best and top-k key.  One warp per
//                      ligand, persistent warps pulling ligands from an
//                      atomic counter (LPT order from the packer).
//   vs_rescore_kernel  K3a  geometric_score / rescore of given poses.
//   vs_grid_kernel     N1   pocket grid maps (steric / hbond / lipophilic),
//   vs_pack_kernel          + corner-packed cells for one-sector lookups.
//   vs_topk_kernel     K4b  block-bitonic tournament top-k over u64 keys.
//
// Ligand records are staged into shared memory with one-dimensional TMA
// bulk copies (cp.async.bulk + mbarrier complete_tx).  All arithmetic that
// feeds a score or a decision is the deterministic arithmetic of
// vs_detmath.cuh with fixed-order sums (docs/SWEEP_V1.md §3), so the CPU
// oracle reproduces every score and decision bit for bit.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "vs_detmath.cuh"
#include "vs_types.h"

namespace vs {

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned long long kGolden = 0x9e3779b97f4a7c15ull;
constexpr double kPiD = 3.14159265358979323846;
constexpr double kHalfPiD = 1.57079632679489661923;
constexpr float kPiF = 3.14159274f;     // (float)pi, rounds up
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

// Trilinear interpolation on one corner-packed cell (two 16 B loads of the
// same 32 B sector).  Same corner values and lerp order as the node layout,
// so the result is bit-identical to interpolating the node map.
__device__ __forceinline__ float trilinear(const GridDev& g, const float4* __restrict__ cells,
                                           float x, float y, float z) {
  const float gx = (x - g.ox) * g.inv_h;
  const float gy = (y - g.oy) * g.inv_h;
  const float gz = (z - g.oz) * g.inv_h;
  const float fx = floorf(gx), fy = floorf(gy), fz = floorf(gz);
  const int ix = static_cast<int>(fx), iy = static_cast<int>(fy), iz = static_cast<int>(fz);
  if (gx < 0.0f || gy < 0.0f || gz < 0.0f || ix > g.nx - 2 || iy > g.ny - 2 || iz > g.nz - 2)
    return 0.0f;
  const float tx = gx - fx, ty = gy - fy, tz = gz - fz;
  const float4* c = cells + 2 * ((static_cast<long>(iz) * (g.ny - 1) + iy) * (g.nx - 1) + ix);
  const float4 lo = __ldg(c), hi = __ldg(c + 1);  // (000,100,010,110), (001,101,011,111)
  const float c00 = det_lerp(lo.x, lo.y, tx), c10 = det_lerp(lo.z, lo.w, tx);
  const float c01 = det_lerp(hi.x, hi.y, tx), c11 = det_lerp(hi.z, hi.w, tx);
  const float c0 = det_lerp(c00, c10, ty), c1 = det_lerp(c01, c11, ty);
  return det_lerp(c0, c1, tz);
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
__device__ __forceinline__ float wall_term(const PocketDev& pk, float x, float y, float z) {
  const float d0 = x - pk.lo[0], d1 = pk.hi[0] - x;
  const float d2 = y - pk.lo[1], d3 = pk.hi[1] - y;
  const float d4 = z - pk.lo[2], d5 = pk.hi[2] - z;
  const float w = fminf(fminf(fminf(d0, d1), fminf(d2, d3)), fminf(d4, d5));
  return det_softplus((pk.r - w) * 10.0f);
}

// pair clash softplus (dock.cpp:86-97) from an FP64 difference
__device__ __forceinline__ float pair_term_d(const PocketDev& pk, double dx, double dy,
                                             double dz) {
  const double d2 = det_norm2_d(dx, dy, dz);
  if (d2 > static_cast<double>(pk.cut2)) return 0.0f;
  return det_softplus((pk.r - sqrtf(static_cast<float>(d2))) * 10.0f);
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

__device__ __forceinline__ float warp_sum(float v) {
  for (int off = 16; off > 0; off >>= 1) v = v + __shfl_xor_sync(kFull, v, off);
  return v;
}

// ------------------------------------------------- per-warp shared layout --
constexpr int kCand = 16;  // rescore kernel: pose columns (one lane pair each)

struct WarpSmem {
  double4* y0;    // conformer (x, y, z, class), FP64
  double4* ys;    // state local coordinates (torsions applied), FP64
  float4* ysf;    // FP32 copy of the state (sweep)
  float4* xf;     // posed coordinates under test (FP32, decisions)
  float* fa;      // per-atom field term of the posed state
  float* wa;      // per-atom wall term of the posed state
  int4* ax;       // torsion axes
  float* theta;   // state torsions
  uint8_t* mov;   // moving lists
  unsigned* mask; // moving set of the current flex axis (4 words)
  double* col;    // rescore kernel only: pose columns [i][c][16], FP64
  float* kscore;  // kept-pose scores
  int* kinv;      // rank -> kept index
  float* kresc;   // survivor rescores by rank
  uint64_t* bar;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline size_t warp_smem_bytes(int nmax, int tmax, int mvmax, bool cols) {
  size_t b = 0;
  b += 2 * 32 * size_t(nmax);                 // y0, ys
  b += 2 * 16 * size_t(nmax);                 // ysf, xf
  b += 2 * align16(4 * size_t(nmax));         // fa, wa
  b += 16 * size_t(tmax);                     // ax
  b += align16(4 * size_t(tmax));             // theta
  b += align16(size_t(mvmax));                // mov
  b += 16;                                    // mask
  if (cols) b += 8 * size_t(nmax) * 3 * kCand;
  b += 3 * 4 * kMaxRestarts;                  // kscore, kinv, kresc
  b += 16;                                    // mbarrier
  return b;
}

__device__ inline WarpSmem carve(unsigned char* base, int nmax, int tmax, int mvmax, bool cols) {
  WarpSmem s;
  size_t o = 0;
  s.y0 = reinterpret_cast<double4*>(base + o); o += 32 * size_t(nmax);
  s.ys = reinterpret_cast<double4*>(base + o); o += 32 * size_t(nmax);
  s.ysf = reinterpret_cast<float4*>(base + o); o += 16 * size_t(nmax);
  s.xf = reinterpret_cast<float4*>(base + o); o += 16 * size_t(nmax);
  s.fa = reinterpret_cast<float*>(base + o); o += align16(4 * size_t(nmax));
  s.wa = reinterpret_cast<float*>(base + o); o += align16(4 * size_t(nmax));
  s.ax = reinterpret_cast<int4*>(base + o); o += 16 * size_t(tmax);
  s.theta = reinterpret_cast<float*>(base + o); o += align16(4 * size_t(tmax));
  s.mov = base + o; o += align16(size_t(mvmax));
  s.mask = reinterpret_cast<unsigned*>(base + o); o += 16;
  s.col = nullptr;
  if (cols) {
    s.col = reinterpret_cast<double*>(base + o);
    o += 8 * size_t(nmax) * 3 * kCand;
  }
  s.kscore = reinterpret_cast<float*>(base + o); o += 4 * kMaxRestarts;
  s.kinv = reinterpret_cast<int*>(base + o); o += 4 * kMaxRestarts;
  s.kresc = reinterpret_cast<float*>(base + o); o += 4 * kMaxRestarts;
  s.bar = reinterpret_cast<uint64_t*>(base + o);
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
}

// s.ys = y0 with torsions [0, T) at s.theta (dock.cpp:54-63); lanes over
// the moving atoms of each torsion in turn.
__device__ inline void chain_coop(const WarpSmem& s, int N, int T, int lane) {
  for (int i = lane; i < N; i += 32) s.ys[i] = s.y0[i];
  __syncwarp();
  for (int j = 0; j < T; ++j) {
    const int4 a = s.ax[j];
    const double4 o = s.ys[a.x], b = s.ys[a.y];
    const Mat3d M = det_torsion_mat_d(o.x, o.y, o.z, b.x, b.y, b.z, s.theta[j]);
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
__device__ inline void pose_coop(const WarpSmem& s, int N, const Mat3d& R, double tx, double ty,
                                 double tz, int lane) {
  for (int i = lane; i < N; i += 32) {
    const double4 v = s.ys[i];
    double x, y, z;
    det_apply_d(R, v.x, v.y, v.z, tx, ty, tz, &x, &y, &z);
    s.xf[i] = make_float4(static_cast<float>(x), static_cast<float>(y), static_cast<float>(z), 0.0f);
  }
  __syncwarp();
}

// Rigid-variant key of one sweep pose: F - lam W over the FP32 state coords.
template <int kGrid>
__device__ inline float eval_rigid(const PocketDev& pk, const float4* ys, int N, const Mat3& R,
                                   float tx, float ty, float tz) {
  float fe = 0.0f, fo = 0.0f, we = 0.0f, wo = 0.0f;
  int i = 0;
  for (; i + 1 < N; i += 2) {
    const float4 a = ys[i], b = ys[i + 1];
    float x0, y0, z0, x1, y1, z1;
    det_apply(R, a.x, a.y, a.z, tx, ty, tz, &x0, &y0, &z0);
    det_apply(R, b.x, b.y, b.z, tx, ty, tz, &x1, &y1, &z1);
    const float f0 = field_steric<kGrid>(pk, x0, y0, z0);
    const float f1 = field_steric<kGrid>(pk, x1, y1, z1);
    fe = fe + f0;
    we = we + wall_term(pk, x0, y0, z0);
    fo = fo + f1;
    wo = wo + wall_term(pk, x1, y1, z1);
  }
  if (i < N) {
    const float4 a = ys[i];
    float x, y, z;
    det_apply(R, a.x, a.y, a.z, tx, ty, tz, &x, &y, &z);
    fe = fe + field_steric<kGrid>(pk, x, y, z);
    we = we + wall_term(pk, x, y, z);
  }
  return (fe + fo) - pk.lam * (we + wo);
}

// all kept poses at RMSD >= delta from s.xf (dock.cpp:335-340, 392-401)
__device__ inline bool diverse_from_kept(const WarpSmem& s, const float4* kx, int nk, int nmax,
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
__device__ inline void draw_start(const PocketDev& pk, unsigned long long rkey, int att, int T,
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
// delta = th_new - th_old (FP64 of two FP32 angles).  The half angle is
// folded into [-pi/2, pi/2] by q -> -q (same matrix).
__device__ __forceinline__ Mat3d flex_mat(double ox, double oy, double oz, double bx, double by,
                                          double bz, float th_new, float th_old) {
  const double dx = bx - ox, dy = by - oy, dz = bz - oz;
  const double n = sqrt(det_norm2_d(dx, dy, dz));
  double hh = 0.5 * (static_cast<double>(th_new) - static_cast<double>(th_old));
  if (hh > kHalfPiD) hh = hh - kPiD;
  else if (hh < -kHalfPiD) hh = hh + kPiD;
  double s, c;
  det_sincos_d(hh, &s, &c);
  const double ks = n > 0.0 ? s / n : 0.0;
  return det_quat_mat_d(c, dx * ks, dy * ks, dz * ks);
}

__device__ __forceinline__ bool in_mask(const unsigned* mask, int i) {
  return (mask[i >> 5] >> (i & 31)) & 1u;
}

// ============================================================= dock kernel
template <int kGrid>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 4)
    vs_dock_kernel(const LibDev lib, const PocketDev pk, const float4* __restrict__ rots,
                   const DockParams prm, const int* __restrict__ order, int n_order,
                   int* __restrict__ work_counter, int nmax, int tmax, int mvmax,
                   float4* __restrict__ scratch_xyz, float* __restrict__ scratch_par,
                   int* __restrict__ scratch_meta, DockOut out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const WarpSmem s =
      carve(smem_raw + wib * warp_smem_bytes(nmax, tmax, mvmax, false), nmax, tmax, mvmax, false);
  const long gwarp = static_cast<long>(blockIdx.x) * kWarpsPerBlock + wib;
  const int R = prm.R;
  const int parw = 8 + tmax;
  float4* kx = scratch_xyz + gwarp * R * nmax;
  float* kp = scratch_par + gwarp * R * parw;
  int* km = scratch_meta + gwarp * R * 4;

  if (lane == 0) mbar_init(s.bar);
  __syncwarp();
  uint32_t phase = 0;

  const int a_lane = lane & 15;
  const int h = lane >> 4;
  const float step = kTwoPiF / static_cast<float>(prm.A);

  while (true) {
    int w = 0;
    if (lane == 0) w = atomicAdd(work_counter, 1);
    w = __shfl_sync(kFull, w, 0);
    if (w >= n_order) break;
    const int lig = order[w];
    int4 meta;
    stage_ligand(lib, lig, s, lane, phase, meta);
    const int N = meta.y, T = meta.w;
    const unsigned long long root = rng_mix(lib.seeds[lig] ^ kGolden);
    int nk = 0;
    unsigned long long st_trans = 0, st_att = 0, st_flex = 0;

    for (int r = 0; r < R; ++r) {
      const unsigned long long rkey =
          rng_mix(root ^ rng_mix(static_cast<unsigned long long>(r) + kGolden));
      float t[3], q[4];
      int att = 0;
      bool have_chain = false;
      for (; att < 50; ++att) {
        draw_start(pk, rkey, att, T, s, lane, t, q);
        if (nk == 0) break;
        chain_coop(s, N, T, lane);
        have_chain = true;
        pose_coop(s, N, det_pose_mat_d(q[0], q[1], q[2], q[3]), t[0], t[1], t[2], lane);
        if (diverse_from_kept(s, kx, nk, nmax, N, prm.delta, lane)) break;
      }
      if (att == 50) att = 49;
      if (!have_chain) chain_coop(s, N, T, lane);
      st_att += static_cast<unsigned long long>(att) + 1;
      for (int i = lane; i < N; i += 32) {
        const double4 v = s.ys[i];
        s.ysf[i] = make_float4(static_cast<float>(v.x), static_cast<float>(v.y),
                               static_cast<float>(v.z), 0.0f);
      }
      __syncwarp();

      // ---- rigid sweep: K orientations about the posed centroid (FP32 key)
      float qs0 = q[0], qs1 = q[1], qs2 = q[2], qs3 = q[3];
      det_quat_normalize(&qs0, &qs1, &qs2, &qs3);
      float cx = 0.0f, cy = 0.0f, cz = 0.0f;
      for (int i = 0; i < N; ++i) {
        const float4 v = s.ysf[i];
        cx = cx + v.x;
        cy = cy + v.y;
        cz = cz + v.z;
      }
      const float fN = static_cast<float>(N);
      cx = cx / fN;
      cy = cy / fN;
      cz = cz / fN;
      float Cx, Cy, Cz;
      det_apply(det_quat_mat(qs0, qs1, qs2, qs3), cx, cy, cz, t[0], t[1], t[2], &Cx, &Cy, &Cz);

      float best_key = -INFINITY;
      int best_k = 0x7fffffff;
      for (int k = lane; k < prm.K; k += 32) {
        const float4 rq = rots[k];
        float w4, x4, y4, z4;
        det_quat_mul(rq.x, rq.y, rq.z, rq.w, qs0, qs1, qs2, qs3, &w4, &x4, &y4, &z4);
        det_quat_normalize(&w4, &x4, &y4, &z4);
        const Mat3 Rk = det_quat_mat(w4, x4, y4, z4);
        float vx, vy, vz;
        det_apply(Rk, cx, cy, cz, 0.0f, 0.0f, 0.0f, &vx, &vy, &vz);
        const float key = eval_rigid<kGrid>(pk, s.ysf, N, Rk, Cx - vx, Cy - vy, Cz - vz);
        if (key > best_key) {
          best_key = key;
          best_k = k;
        }
      }
      for (int off = 16; off > 0; off >>= 1) {
        const float ok = __shfl_xor_sync(kFull, best_key, off);
        const int oi = __shfl_xor_sync(kFull, best_k, off);
        if (ok > best_key || (ok == best_key && oi < best_k)) {
          best_key = ok;
          best_k = oi;
        }
      }
      float pw, px, py, pz;
      {
        const float4 rq = rots[best_k];
        det_quat_mul(rq.x, rq.y, rq.z, rq.w, qs0, qs1, qs2, qs3, &pw, &px, &py, &pz);
        det_quat_normalize(&pw, &px, &py, &pz);
      }
      float ptx, pty, ptz;
      {
        const Mat3 RS = det_quat_mat(pw, px, py, pz);
        float vx, vy, vz;
        det_apply(RS, cx, cy, cz, 0.0f, 0.0f, 0.0f, &vx, &vy, &vz);
        ptx = Cx - vx;
        pty = Cy - vy;
        ptz = Cz - vz;
      }
      // ---- translation sweep: compass search over the 26 lattice
      // neighbours at step sc, halving sc when no neighbour improves
      {
        const Mat3 RS = det_quat_mat(pw, px, py, pz);
        float sc = 1.0f;
        for (int it = 0; it < kTransIters && sc >= kTransMin; ++it) {
          float key = -INFINITY, ox = 0.0f, oy = 0.0f, oz = 0.0f;
          if (lane < 27) {
            trans_offset(lane, sc, &ox, &oy, &oz);
            key = eval_rigid<kGrid>(pk, s.ysf, N, RS, ptx + ox, pty + oy, ptz + oz);
          }
          int li = lane < 27 ? lane : 0x7fffffff;
          for (int off = 16; off > 0; off >>= 1) {
            const float ok = __shfl_xor_sync(kFull, key, off);
            const int oi = __shfl_xor_sync(kFull, li, off);
            if (ok > key || (ok == key && oi < li)) {
              key = ok;
              li = oi;
            }
          }
          if (li != 0) {
            float wx, wy, wz;
            trans_offset(li, sc, &wx, &wy, &wz);
            ptx = ptx + wx;
            pty = pty + wy;
            ptz = ptz + wz;
          } else {
            sc = sc * 0.5f;
          }
          ++st_trans;
        }
      }
      const Mat3d RD = det_pose_mat_d(pw, px, py, pz);
      const double tdx = ptx, tdy = pty, tdz = ptz;

      // ---- incremental torsion flex (docs/SWEEP_V1.md §2.5): per-atom
      // terms of the posed state, then for each (pass, axis j) 16 candidate
      // angles scored as  base(state, atoms/pairs not touched by moving_j)
      // + moved part(candidate, moving_j atoms and their cross pairs).
      for (int i = lane; i < N; i += 32) {
        const double4 v = s.ys[i];
        atom_terms<kGrid>(pk, RD, tdx, tdy, tdz, v.x, v.y, v.z, &s.fa[i], &s.wa[i]);
      }
      __syncwarp();
      const bool do_flex = T > 0 && prm.F > 0;
      const int steps = do_flex ? prm.F * T : 1;
      st_flex += do_flex ? static_cast<unsigned long long>(steps) * prm.A : 1ull;
      float S_cur = 0.0f;
      for (int st = 0; st < steps; ++st) {
        const int j = do_flex ? st % T : -1;
        const int4 ax = do_flex ? s.ax[j] : make_int4(0, 0, 0, 0);
        const int m = ax.w;
        if (lane < 4) {
          unsigned wd = 0;
          for (int q2 = 0; q2 < m; ++q2) {
            const int idx = s.mov[ax.z + q2];
            if ((idx >> 5) == lane) wd |= 1u << (idx & 31);
          }
          s.mask[lane] = wd;
        }
        __syncwarp();
        // base sums: lane l accumulates atoms i = l (mod 32) outside the
        // moving set and pairs p = l (mod 32) (row-major index over all
        // pairs) that do not cross it; then an xor butterfly
        float fb = 0.0f, wb = 0.0f, pb = 0.0f;
        for (int i = lane; i < N; i += 32) {
          if (!in_mask(s.mask, i)) {
            fb = fb + s.fa[i];
            wb = wb + s.wa[i];
          }
        }
        {
          int ps = 0;
          for (int i = 0; i + 1 < N; ++i) {
            const double4 yi = s.ys[i];
            const bool mi = in_mask(s.mask, i);
            for (int k = i + 1 + ((lane - ps) & 31); k < N; k += 32) {
              if (mi != in_mask(s.mask, k)) continue;
              const double4 yk = s.ys[k];
              pb = pb + pair_term_d(pk, yi.x - yk.x, yi.y - yk.y, yi.z - yk.z);
            }
            ps += N - 1 - i;
          }
        }
        fb = warp_sum(fb);
        wb = warp_sum(wb);
        pb = warp_sum(pb);
        // candidates: lane pair (a, h); lane h takes moving positions = h mod 2
        const bool active = do_flex && a_lane < prm.A;
        float th_new = 0.0f;
        float fm = 0.0f, wm = 0.0f, pc = 0.0f;
        if (active) {
          const float th_old = s.theta[j];
          th_new = th_old;
          if (a_lane > 0) {
            float v = th_old + static_cast<float>(a_lane) * step;
            if (v >= kPiF) v = v - kTwoPiF;
            th_new = v;
          }
          const double4 o = s.ys[ax.x], b = s.ys[ax.y];
          const Mat3d M = flex_mat(o.x, o.y, o.z, b.x, b.y, b.z, th_new, th_old);
          for (int q2 = h; q2 < m; q2 += 2) {
            const int idx = s.mov[ax.z + q2];
            const double4 v = s.ys[idx];
            double yx, yy, yz;
            det_apply_d(M, v.x - o.x, v.y - o.y, v.z - o.z, o.x, o.y, o.z, &yx, &yy, &yz);
            float fi, wi;
            atom_terms<kGrid>(pk, RD, tdx, tdy, tdz, yx, yy, yz, &fi, &wi);
            fm = fm + fi;
            wm = wm + wi;
            for (int k = 0; k < N; ++k) {
              if (in_mask(s.mask, k)) continue;
              const double4 yk = s.ys[k];
              pc = pc + pair_term_d(pk, yx - yk.x, yy - yk.y, yz - yk.z);
            }
          }
        }
        const float fm2 = __shfl_xor_sync(kFull, fm, 16);
        const float wm2 = __shfl_xor_sync(kFull, wm, 16);
        const float pc2 = __shfl_xor_sync(kFull, pc, 16);
        float S = (fb + (fm + fm2)) - pk.lam * ((pb + (pc + pc2)) + (wb + (wm + wm2)));
        if (do_flex && !active) S = -INFINITY;
        int ai = (do_flex && !active) ? 0x7fffffff : a_lane;
        for (int off = 8; off > 0; off >>= 1) {
          const float oS = __shfl_xor_sync(kFull, S, off);
          const int oa = __shfl_xor_sync(kFull, ai, off);
          if (oS > S || (oS == S && oa < ai)) {
            S = oS;
            ai = oa;
          }
        }
        S_cur = S;
        if (do_flex && ai != 0) {  // move the state to the winning angle
          const float th_old = s.theta[j];
          const float th_win = __shfl_sync(kFull, th_new, ai);
          const double4 o = s.ys[ax.x], b = s.ys[ax.y];
          const Mat3d M = flex_mat(o.x, o.y, o.z, b.x, b.y, b.z, th_win, th_old);
          __syncwarp();
          for (int q2 = lane; q2 < m; q2 += 32) {
            const int idx = s.mov[ax.z + q2];
            double4 v = s.ys[idx];
            det_apply_d(M, v.x - o.x, v.y - o.y, v.z - o.z, o.x, o.y, o.z, &v.x, &v.y, &v.z);
            s.ys[idx] = v;
            atom_terms<kGrid>(pk, RD, tdx, tdy, tdz, v.x, v.y, v.z, &s.fa[idx], &s.wa[idx]);
          }
          if (lane == 0) s.theta[j] = th_win;
        }
        __syncwarp();
      }

      // ---- final coordinates and diversity against kept (dock.cpp:359-361)
      pose_coop(s, N, RD, tdx, tdy, tdz, lane);
      const bool keep = nk == 0 || diverse_from_kept(s, kx, nk, nmax, N, prm.delta, lane);
      if (keep) {
        for (int i = lane; i < N; i += 32) kx[static_cast<size_t>(nk) * nmax + i] = s.xf[i];
        float* P = kp + static_cast<size_t>(nk) * parw;
        if (lane == 0) {
          P[0] = ptx; P[1] = pty; P[2] = ptz;
          P[3] = pw; P[4] = px; P[5] = py; P[6] = pz;
          P[7] = S_cur;
          km[nk * 4 + 0] = r;
          km[nk * 4 + 1] = att;
          km[nk * 4 + 2] = best_k;
          s.kscore[nk] = S_cur;
        }
        for (int jj = lane; jj < T; jj += 32) P[8 + jj] = s.theta[jj];
        ++nk;
      }
      __syncwarp();
    }

    // ---- stable sort by score desc (dock.cpp:364-366), keep-top filter
    // (dock.cpp:373-390), rescore (dock.cpp:297-316), best (pipeline.cpp:508)
    int m_pass = 0;
    for (int k = lane; k < nk; k += 32) {
      const float sk = s.kscore[k];
      int rank = 0;
      for (int m2 = 0; m2 < nk; ++m2) {
        const float sm = s.kscore[m2];
        rank += (sm > sk || (sm == sk && m2 < k)) ? 1 : 0;
      }
      s.kinv[rank] = k;
      m_pass += (static_cast<double>(sk) >= prm.min_score) ? 1 : 0;
    }
    for (int off = 16; off > 0; off >>= 1) m_pass += __shfl_xor_sync(kFull, m_pass, off);
    __syncwarp();
    const int n_surv = min(m_pass, prm.keep_top);

    if (prm.write_all) {
      for (int rank = lane; rank < nk; rank += 32) {
        const int k = s.kinv[rank];
        const float* P = kp + static_cast<size_t>(k) * parw;
        PoseOut o;
        o.t[0] = P[0]; o.t[1] = P[1]; o.t[2] = P[2];
        o.q[0] = P[3]; o.q[1] = P[4]; o.q[2] = P[5]; o.q[3] = P[6];
        o.score = P[7];
        o.rescore = 0.0f;
        o.restart = static_cast<int16_t>(km[k * 4]);
        o.attempt = static_cast<int16_t>(km[k * 4 + 1]);
        o.rot = static_cast<int16_t>(km[k * 4 + 2]);
        o.pad = 0;
        out.all[static_cast<size_t>(lig) * R + rank] = o;
        float* tt = out.all_tors + static_cast<size_t>(meta.z) * R + static_cast<size_t>(rank) * T;
        for (int jj = 0; jj < T; ++jj) tt[jj] = P[8 + jj];
      }
      __syncwarp();
    }

    for (int base = 0; base < n_surv; base += 16) {
      const int p = base + a_lane;
      float B = 0.0f;
      if (p < n_surv) {
        const float4* X = kx + static_cast<size_t>(s.kinv[p]) * nmax;
        for (int i = h; i < N; i += 2) {
          const float4 v = X[i];
          B = B + atom_bonus<kGrid>(pk, static_cast<int>(s.y0[i].w), v.x, v.y, v.z);
        }
      }
      const float B2 = __shfl_xor_sync(kFull, B, 16);
      if (p < n_surv && h == 0) {
        const int k = s.kinv[p];
        const float* P = kp + static_cast<size_t>(k) * parw;
        const float resc = P[7] + (B + B2);
        s.kresc[p] = resc;
        PoseOut o;
        o.t[0] = P[0]; o.t[1] = P[1]; o.t[2] = P[2];
        o.q[0] = P[3]; o.q[1] = P[4]; o.q[2] = P[5]; o.q[3] = P[6];
        o.score = P[7];
        o.rescore = resc;
        o.restart = static_cast<int16_t>(km[k * 4]);
        o.attempt = static_cast<int16_t>(km[k * 4 + 1]);
        o.rot = static_cast<int16_t>(km[k * 4 + 2]);
        o.pad = 0;
        out.surv[static_cast<size_t>(lig) * prm.keep_top + p] = o;
        float* tt = out.surv_tors + static_cast<size_t>(meta.z) * prm.keep_top +
                    static_cast<size_t>(p) * T;
        for (int jj = 0; jj < T; ++jj) tt[jj] = P[8 + jj];
        if (prm.write_all) out.all[static_cast<size_t>(lig) * R + p].rescore = resc;
      }
    }
    __syncwarp();
    if (lane == 0) {
      // best = max rescore over survivors (pipeline.cpp:508-510)
      float bmax = -INFINITY;
      for (int p = 0; p < n_surv; ++p) bmax = p == 0 ? s.kresc[p] : fmaxf(bmax, s.kresc[p]);
      out.best[lig] = bmax;
      out.n_kept[lig] = nk;
      out.n_surv[lig] = n_surv;
      out.keys[lig] =
          n_surv > 0 ? ((static_cast<unsigned long long>(~det_orderable(bmax)) << 32) |
                        lib.id_rank[lig])
                     : ~0ull;
      if (out.stats) {
        atomicAdd(out.stats + 0, st_trans);
        atomicAdd(out.stats + 1, st_trans * static_cast<unsigned long long>(N));
        atomicAdd(out.stats + 2, st_att);
        atomicAdd(out.stats + 3, st_flex);
      }
    }
    __syncwarp();
  }
}

// ========================================================= rescore kernel
__device__ __forceinline__ double& cold(double* col, int i, int c, int a) {
  return col[(i * 3 + c) * kCand + a];
}

// Pose column a (lane pair (a, h)): conformer with all torsions of the pose
// applied in order (dock.cpp:54-63); lanes h = 0/1 split atoms and moving
// lists, __syncwarp between torsions.
__device__ inline void chain_pose(const WarpSmem& s, int N, int T, int a, int h, bool active,
                                  const float* th) {
  double* col = s.col;
  if (active) {
    for (int i = h; i < N; i += 2) {
      const double4 v = s.y0[i];
      cold(col, i, 0, a) = v.x;
      cold(col, i, 1, a) = v.y;
      cold(col, i, 2, a) = v.z;
    }
  }
  __syncwarp();
  for (int k = 0; k < T; ++k) {
    if (active) {
      const int4 ax = s.ax[k];
      const double ox = cold(col, ax.x, 0, a), oy = cold(col, ax.x, 1, a),
                   oz = cold(col, ax.x, 2, a);
      const Mat3d M = det_torsion_mat_d(ox, oy, oz, cold(col, ax.y, 0, a), cold(col, ax.y, 1, a),
                                        cold(col, ax.y, 2, a), th[k]);
      for (int m = h; m < ax.w; m += 2) {
        const int idx = s.mov[ax.z + m];
        double vx, vy, vz;
        det_apply_d(M, cold(col, idx, 0, a) - ox, cold(col, idx, 1, a) - oy,
                    cold(col, idx, 2, a) - oz, ox, oy, oz, &vx, &vy, &vz);
        cold(col, idx, 0, a) = vx;
        cold(col, idx, 1, a) = vy;
        cold(col, idx, 2, a) = vz;
      }
    }
    __syncwarp();
  }
}

// Work item w: ligand ligs[w], poses [pose_off[w], pose_off[w+1]) (float4 t,
// float4 q = (w,x,y,z)), torsions at tors_base[w] + (p - pose_off[w]) * T.
// Canonical score of a given pose: parity-h lane sums over atoms i = h mod 2
// and pairs p = h mod 2 (row-major), combined across the lane pair.
template <int kGrid>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    vs_rescore_kernel(const LibDev lib, const PocketDev pk, const int* __restrict__ ligs,
                      int n_ligs, int* __restrict__ work_counter, const int* __restrict__ pose_off,
                      const long* __restrict__ tors_base, const float4* __restrict__ pose_t,
                      const float4* __restrict__ pose_q, const float* __restrict__ pose_tors,
                      int nmax, int tmax, int mvmax, float* __restrict__ geo,
                      float* __restrict__ resc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const WarpSmem s =
      carve(smem_raw + wib * warp_smem_bytes(nmax, tmax, mvmax, true), nmax, tmax, mvmax, true);
  if (lane == 0) mbar_init(s.bar);
  __syncwarp();
  uint32_t phase = 0;
  const int a = lane & 15;
  const int h = lane >> 4;
  while (true) {
    int w = 0;
    if (lane == 0) w = atomicAdd(work_counter, 1);
    w = __shfl_sync(kFull, w, 0);
    if (w >= n_ligs) break;
    const int lig = ligs[w];
    int4 meta;
    stage_ligand(lib, lig, s, lane, phase, meta);
    const int N = meta.y, T = meta.w;
    const int p0 = pose_off[w], p1 = pose_off[w + 1];
    for (int base = p0; base < p1; base += 16) {
      const int p = base + a;
      const bool active = p < p1;
      const float* th = pose_tors + tors_base[w] + static_cast<long>(active ? p - p0 : 0) * T;
      chain_pose(s, N, T, a, h, active, th);
      float F = 0.0f, W = 0.0f, P = 0.0f, B = 0.0f;
      if (active) {
        const float4 tt = pose_t[p];
        const float4 qq = pose_q[p];
        const Mat3d Rm = det_pose_mat_d(qq.x, qq.y, qq.z, qq.w);
        const double tx = tt.x, ty = tt.y, tz = tt.z;
        const double* col = s.col;
        for (int i = h; i < N; i += 2) {
          float fi, wi, xo[3];
          atom_terms<kGrid>(pk, Rm, tx, ty, tz, col[(i * 3) * kCand + a],
                            col[(i * 3 + 1) * kCand + a], col[(i * 3 + 2) * kCand + a], &fi, &wi,
                            xo);
          F = F + fi;
          W = W + wi;
          B = B + atom_bonus<kGrid>(pk, static_cast<int>(s.y0[i].w), xo[0], xo[1], xo[2]);
        }
        int ps = 0;
        for (int i = 0; i + 1 < N; ++i) {
          const double xi = col[(i * 3) * kCand + a], yi = col[(i * 3 + 1) * kCand + a],
                       zi = col[(i * 3 + 2) * kCand + a];
          for (int jj = i + 1 + ((h ^ ps) & 1); jj < N; jj += 2) {
            P = P + pair_term_d(pk, xi - col[(jj * 3) * kCand + a],
                                yi - col[(jj * 3 + 1) * kCand + a],
                                zi - col[(jj * 3 + 2) * kCand + a]);
          }
          ps += N - 1 - i;
        }
      }
      const float F2 = __shfl_xor_sync(kFull, F, 16);
      const float W2 = __shfl_xor_sync(kFull, W, 16);
      const float P2 = __shfl_xor_sync(kFull, P, 16);
      const float B2 = __shfl_xor_sync(kFull, B, 16);
      if (active && h == 0) {
        const float S = (F + F2) - pk.lam * ((P + P2) + (W + W2));
        geo[p] = S;
        resc[p] = S + (B + B2);
      }
      __syncwarp();
    }
    __syncwarp();
  }
}

// ============================================================ grid kernels
__global__ void vs_grid_kernel(const PocketDev pk, float* __restrict__ steric,
                               float* __restrict__ hbond, float* __restrict__ lipo) {
  const GridDev& g = pk.grid;
  const long n = static_cast<long>(g.nx) * g.ny * g.nz;
  for (long id = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; id < n;
       id += static_cast<long>(gridDim.x) * blockDim.x) {
    const int ix = static_cast<int>(id % g.nx);
    const int iy = static_cast<int>((id / g.nx) % g.ny);
    const int iz = static_cast<int>(id / (static_cast<long>(g.nx) * g.ny));
    const float x = fmaf(static_cast<float>(ix), g.h, g.ox);
    const float y = fmaf(static_cast<float>(iy), g.h, g.oy);
    const float z = fmaf(static_cast<float>(iz), g.h, g.oz);
    steric[id] = site_sum(pk.sites, pk.n_steric, x, y, z);
    hbond[id] = site_sum(pk.sites + pk.n_steric, pk.n_hbond, x, y, z);
    lipo[id] = site_sum(pk.sites + pk.n_steric + pk.n_hbond, pk.n_lipo, x, y, z);
  }
}

// node map -> corner-packed cells (000,100,010,110 | 001,101,011,111)
__global__ void vs_pack_kernel(const GridDev g, const float* __restrict__ node,
                               float4* __restrict__ cells) {
  const long cx = g.nx - 1, cy = g.ny - 1, cz = g.nz - 1;
  const long n = cx * cy * cz;
  const long sx = 1, sy = g.nx, sz = static_cast<long>(g.nx) * g.ny;
  for (long id = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; id < n;
       id += static_cast<long>(gridDim.x) * blockDim.x) {
    const long ix = id % cx, iy = (id / cx) % cy, iz = id / (cx * cy);
    const float* p = node + iz * sz + iy * sy + ix;
    cells[2 * id] = make_float4(p[0], p[sx], p[sy], p[sy + sx]);
    cells[2 * id + 1] = make_float4(p[sz], p[sz + sx], p[sz + sy], p[sz + sy + sx]);
  }
}

// ============================================================ top-k kernel
// Block b sorts keys [b*C, (b+1)*C) ascending (bitonic, shared memory) and
// writes its k smallest to out[b*k ...].  Keys are unique (id_rank in the low
// word) except the ~0 padding, so the result is deterministic.
constexpr int kTopkC = 4096;
__global__ void __launch_bounds__(1024)
    vs_topk_kernel(const unsigned long long* __restrict__ in, long n,
                   unsigned long long* __restrict__ out, int k) {
  __shared__ unsigned long long sk[kTopkC];
  const long base = static_cast<long>(blockIdx.x) * kTopkC;
  for (int i = threadIdx.x; i < kTopkC; i += blockDim.x) {
    const long g = base + i;
    sk[i] = g < n ? in[g] : ~0ull;
  }
  __syncthreads();
  for (int size = 2; size <= kTopkC; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < kTopkC / 2; i += blockDim.x) {
        const int lo = 2 * i - (i & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const unsigned long long a = sk[lo], b = sk[hi];
        if ((a > b) == up) {
          sk[lo] = b;
          sk[hi] = a;
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < k; i += blockDim.x)
    out[static_cast<long>(blockIdx.x) * k + i] = sk[i];
}

// ====================================================== peak microbenchmarks
// Independent FMA / MUFU chains per thread; the result is stored only under a
// never-true predicate so the chains are not dead code.
__global__ void vs_peak_fp32(float* out, int iters, float seed) {
  float a[8];
  for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-7f + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(a[k], 0.999999f, 1e-7f);
  }
  float s = 0.0f;
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == -1.2345f) out[threadIdx.x] = s;
}
__global__ void vs_peak_fp64(double* out, int iters, double seed) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], 0.999999999, 1e-9);
  }
  double s = 0.0;
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == -1.2345) out[threadIdx.x] = s;
}
__global__ void vs_peak_xu(float* out, int iters, float seed) {
  float a[8];
  for (int k = 0; k < 8; ++k) a[k] = seed * 1e-3f + threadIdx.x * 1e-9f + k * 1e-3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[k]));
  }
  float s = 0.0f;
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == -1.2345f) out[threadIdx.x] = s;
}

}  // namespace vs

// ------------------------------------------------------ launch wrappers --
namespace vs {

size_t dock_smem_per_block(int nmax, int tmax, int mvmax) {
  return kWarpsPerBlock * warp_smem_bytes(nmax, tmax, mvmax, false);
}

size_t rescore_smem_per_block(int nmax, int tmax, int mvmax) {
  return kWarpsPerBlock * warp_smem_bytes(nmax, tmax, mvmax, true);
}

template <class K>
static void prep(K kernel, size_t smem) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
}

cudaError_t launch_dock(bool grid, int blocks, size_t smem, cudaStream_t st, const LibDev& lib,
                        const PocketDev& pk, const float4* rots, const DockParams& prm,
                        const int* order, int n_order, int* counter, int nmax, int tmax,
                        int mvmax, float4* sx, float* sp, int* sm, const DockOut& out) {
  if (grid) {
    prep(vs_dock_kernel<1>, smem);
    vs_dock_kernel<1><<<blocks, kWarpsPerBlock * 32, smem, st>>>(
        lib, pk, rots, prm, order, n_order, counter, nmax, tmax, mvmax, sx, sp, sm, out);
  } else {
    prep(vs_dock_kernel<0>, smem);
    vs_dock_kernel<0><<<blocks, kWarpsPerBlock * 32, smem, st>>>(
        lib, pk, rots, prm, order, n_order, counter, nmax, tmax, mvmax, sx, sp, sm, out);
  }
  return cudaGetLastError();
}

int dock_blocks_per_sm(bool grid, size_t smem) {
  int nb = 0;
  if (grid) {
    prep(vs_dock_kernel<1>, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, vs_dock_kernel<1>, kWarpsPerBlock * 32,
                                                  smem);
  } else {
    prep(vs_dock_kernel<0>, smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, vs_dock_kernel<0>, kWarpsPerBlock * 32,
                                                  smem);
  }
  return nb;
}

cudaError_t launch_rescore(bool grid, int blocks, size_t smem, cudaStream_t st, const LibDev& lib,
                           const PocketDev& pk, const int* ligs, int n_ligs, int* counter,
                           const int* pose_off, const long* tors_base, const float4* pt,
                           const float4* pq, const float* ptors, int nmax, int tmax, int mvmax,
                           float* geo, float* resc) {
  if (grid) {
    prep(vs_rescore_kernel<1>, smem);
    vs_rescore_kernel<1><<<blocks, kWarpsPerBlock * 32, smem, st>>>(
        lib, pk, ligs, n_ligs, counter, pose_off, tors_base, pt, pq, ptors, nmax, tmax, mvmax,
        geo, resc);
  } else {
    prep(vs_rescore_kernel<0>, smem);
    vs_rescore_kernel<0><<<blocks, kWarpsPerBlock * 32, smem, st>>>(
        lib, pk, ligs, n_ligs, counter, pose_off, tors_base, pt, pq, ptors, nmax, tmax, mvmax,
        geo, resc);
  }
  return cudaGetLastError();
}

cudaError_t launch_grid(cudaStream_t st, const PocketDev& pk, float* steric, float* hb,
                        float* lipo, float4* cells) {
  const GridDev& g = pk.grid;
  const long n = static_cast<long>(g.nx) * g.ny * g.nz;
  int blocks = static_cast<int>((n + 255) / 256);
  if (blocks > 148 * 64) blocks = 148 * 64;
  vs_grid_kernel<<<blocks, 256, 0, st>>>(pk, steric, hb, lipo);
  const long nc = static_cast<long>(g.nx - 1) * (g.ny - 1) * (g.nz - 1);
  int cb = static_cast<int>((nc + 255) / 256);
  if (cb > 148 * 64) cb = 148 * 64;
  vs_pack_kernel<<<cb, 256, 0, st>>>(g, steric, cells);
  vs_pack_kernel<<<cb, 256, 0, st>>>(g, hb, cells + 2 * nc);
  vs_pack_kernel<<<cb, 256, 0, st>>>(g, lipo, cells + 4 * nc);
  return cudaGetLastError();
}

int topk_chunk() { return kTopkC; }

cudaError_t launch_topk(cudaStream_t st, const unsigned long long* in, long n,
                        unsigned long long* out, int k, int blocks) {
  vs_topk_kernel<<<blocks, 1024, 0, st>>>(in, n, out, k);
  return cudaGetLastError();
}

// kind 0 fp32 fma, 1 fp64 fma, 2 ex2; returns ops/s (best of 3)
double measure_peak(int kind, int sms) {
  void* buf = nullptr;
  cudaMalloc(&buf, 1024 * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    if (kind == 0) vs_peak_fp32<<<blocks, threads>>>(static_cast<float*>(buf), iters, 1.0f);
    else if (kind == 1) vs_peak_fp64<<<blocks, threads>>>(static_cast<double*>(buf), iters, 1.0);
    else vs_peak_xu<<<blocks, threads>>>(static_cast<float*>(buf), iters, 1.0f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = static_cast<double>(blocks) * threads * iters * 8 * (kind == 2 ? 1.0 : 2.0);
    if (rep > 0) best = std::max(best, ops / (ms * 1e-3));
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  return best;
}

}  // namespace vs
