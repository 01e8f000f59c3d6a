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
//   vs_pack_kernel          + the sweep-key map and corner-packed cells for
//                           one-sector lookups.
//   vs_topk_kernel     K4b  block-bitonic tournament top-k over u64 keys.
//
// Ligand records are staged into shared memory with one-dimensional TMA
// bulk copies (cp.async.bulk + mbarrier complete_tx).  All arithmetic that
// feeds a score or a decision is the deterministic arithmetic of
// vs_detmath.cuh with fixed-order sums (docs/SWEEP_V1.md §3), so the CPU
// oracle reproduces every score and decision bit for bit.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "vs_detmath.cuh"
#include "vs_types.h"

#include "vs_common.cuh"

namespace vs {

// ========================================================= rescore kernel
// the parts the rescore kernel touches: the ligand (conformer, axes, moving
// lists, axis lengths) and the pose columns
constexpr int kLayRescore = kLayLig | kLayCols;
__device__ __forceinline__ double& cold(double* col, int i, int c, int a) {
  return col[(i * 3 + c) * kCand + a];
}

// Pose column a (lanes 8a .. 8a + 7, slice h): conformer with all torsions
// of the pose applied in order (dock.cpp:54-63); the 8 lanes split atoms and
// moving lists, __syncwarp between torsions.
__device__ inline void chain_pose(const WarpSmem& s, int N, int T, int a, int h, bool active,
                                  const float* th) {
  double* col = s.col;
  if (active) {
    for (int i = h; i < N; i += kLanesPerPose) {
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
                                        cold(col, ax.y, 2, a), th[k], s.axl[k]);
      for (int m = h; m < ax.w; m += kLanesPerPose) {
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

// sum over the 8 lanes of a pose column: xor butterfly 1, 2, 4, i.e.
// ((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7)) on every lane
__device__ __forceinline__ float column_sum(float v) {
  v = v + __shfl_xor_sync(kFull, v, 1);
  v = v + __shfl_xor_sync(kFull, v, 2);
  v = v + __shfl_xor_sync(kFull, v, 4);
  return v;
}

// Work item w: ligand ligs[w] and its poses (PoseSrc), kCand = 4 at a time.
// Canonical score of a given pose, lanes 8a + h: slice h sums atoms
// i = h (mod 8) and pairs p = h (mod 8) (row-major), then the column's
// butterfly.  A ligand with up to 4 poses (keep_top 4) uses every lane.
#ifndef VS_MINB_RESCORE
#define VS_MINB_RESCORE 8  // C5: 0.531 ms vs 0.600 (no bound), 0.551 (6), 0.567 (10)
#endif
template <int kGrid>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, VS_MINB_RESCORE)
    vs_rescore_kernel(const __grid_constant__ LibDev lib, const __grid_constant__ PocketDev pk,
                      const int* __restrict__ ligs, int n_ligs, int* __restrict__ work_counter,
                      const __grid_constant__ PoseSrc src, int nmax, int tmax, int mvmax) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const WarpSmem s =
      carve(smem_raw + wib * warp_smem_bytes(nmax, tmax, mvmax, kLayRescore), nmax, tmax, mvmax,
            kLayRescore);
  if (lane == 0) mbar_init(s.bar);
  __syncwarp();
  uint32_t phase = 0;
  const int a = lane / kLanesPerPose;
  const int h = lane % kLanesPerPose;
  const bool flat = src.t3 != nullptr;
  while (true) {
    int w = 0;
    if (lane == 0) w = atomicAdd(work_counter, 1);
    w = __shfl_sync(kFull, w, 0);
    if (w >= n_ligs) break;
    const int lig = ligs[w];
    const int np = flat ? src.count[lig] : src.n_surv[lig];
    if (np <= 0) continue;
    int4 meta;
    stage_ligand(lib, lig, s, lane, phase, meta);
    const int N = meta.y, T = meta.w;
    const long p0 = flat ? src.first[lig] : static_cast<long>(lig) * src.keep_top;
    for (int base = 0; base < np; base += kCand) {
      const int j = base + a;
      const bool active = j < np;
      const int jj0 = active ? j : 0;
      const long p = p0 + jj0;
      const float* th = flat ? src.tors + src.tb[lig] + static_cast<long>(jj0) * T
                             : src.surv_tors + static_cast<long>(meta.z) * src.keep_top +
                                   static_cast<long>(jj0) * T;
      chain_pose(s, N, T, a, h, active, th);
      float F = 0.0f, W = 0.0f, P = 0.0f, B = 0.0f;
      if (active) {
        float tq[7];
        if (flat) {
          for (int c = 0; c < 3; ++c) tq[c] = src.t3[3 * p + c];
          for (int c = 0; c < 4; ++c) tq[3 + c] = src.q4[4 * p + c];
        } else {
          const PoseOut& o = src.surv[p];
          for (int c = 0; c < 3; ++c) tq[c] = o.t[c];
          for (int c = 0; c < 4; ++c) tq[3 + c] = o.q[c];
        }
        const Mat3d Rm = det_pose_mat_d(tq[3], tq[4], tq[5], tq[6]);
        const double tx = tq[0], ty = tq[1], tz = tq[2];
        const double* col = s.col;
        for (int i = h; i < N; i += kLanesPerPose) {
          float fi, wi, xo[3];
          atom_terms<kGrid>(pk, Rm, tx, ty, tz, col[(i * 3) * kCand + a],
                            col[(i * 3 + 1) * kCand + a], col[(i * 3 + 2) * kCand + a], &fi, &wi,
                            xo);
          F = F + fi;
          W = W + wi;
          B = B + atom_bonus<kGrid>(pk, static_cast<int>(s.y0[i].w), xo[0], xo[1], xo[2]);
        }
        // pairs in row-major order, pair index q = h (mod 8) on this slice
        int ps = 0;  // pairs before row i
        for (int i = 0; i + 1 < N; ++i) {
          const double xi = col[(i * 3) * kCand + a], yi = col[(i * 3 + 1) * kCand + a],
                       zi = col[(i * 3 + 2) * kCand + a];
          const int first = i + 1 + ((h - ps) % kLanesPerPose + kLanesPerPose) % kLanesPerPose;
          for (int jx = first; jx < N; jx += kLanesPerPose) {
            P = P + pair_term_d(pk, xi - col[(jx * 3) * kCand + a],
                                yi - col[(jx * 3 + 1) * kCand + a],
                                zi - col[(jx * 3 + 2) * kCand + a]);
          }
          ps += N - 1 - i;
        }
      }
      F = column_sum(F);
      W = column_sum(W);
      P = column_sum(P);
      B = column_sum(B);
      if (active && h == 0) {
        const float S = F - pk.lam * (P + W);
        src.geo[p] = S;
        src.resc[p] = S + B;
      }
      __syncwarp();
    }
    __syncwarp();
  }
}

// ============================================================ grid kernels
__global__ void vs_grid_kernel(const __grid_constant__ PocketDev pk, float* __restrict__ steric,
                               float* __restrict__ hbond, float* __restrict__ lipo,
                               float* __restrict__ key) {
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
    // the sweep-key map is stored in FP16 (node map holds the rounded value)
    key[id] = __half2float(__float2half_rn(fmaf(-pk.lam, wall_of(pk, x, y, z), steric[id])));
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

// FP16 node map -> 16 B cells holding the trilinear polynomial of the cell
// (SWEEP_V1.md §3.2): c000, c100, c010, c110 | c001, c101, c011, c111, from
// the corner values in the fixed FP32 order below, each rounded to FP16.
// The sweep key evaluates it with 7 FMAs (the 7 lerps took 14 instructions).
__global__ void vs_pack_half_kernel(const GridDev g, const float* __restrict__ node,
                                    uint4* __restrict__ cells) {
  const long cx = g.nx - 1, cy = g.ny - 1, cz = g.nz - 1;
  const long n = cx * cy * cz;
  const long sx = 1, sy = g.nx, sz = static_cast<long>(g.nx) * g.ny;
  for (long id = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; id < n;
       id += static_cast<long>(gridDim.x) * blockDim.x) {
    const long ix = id % cx, iy = (id / cx) % cy, iz = id / (cx * cy);
    const float* p = node + iz * sz + iy * sy + ix;
    auto h2 = [](float a, float b) {
      const __half2 v = __floats2half2_rn(a, b);
      return *reinterpret_cast<const unsigned*>(&v);
    };
    const float v000 = p[0], v100 = p[sx], v010 = p[sy], v110 = p[sy + sx];
    const float v001 = p[sz], v101 = p[sz + sx], v011 = p[sz + sy], v111 = p[sz + sy + sx];
    const float c100 = v100 - v000, c010 = v010 - v000, c001 = v001 - v000;
    const float c110 = (v110 - v100) - c010, c101 = (v101 - v100) - c001;
    const float c011 = (v011 - v010) - c001;
    const float c111 = ((v111 - v110) - (v101 - v100)) - c011;
    cells[id] = make_uint4(h2(v000, c100), h2(c010, c110), h2(c001, c101), h2(c011, c111));
  }
}

// =========================================== search pair-softplus table
// node k: x_k = k * (cut2 / kSoftN) (FP32), g_k = softplus((r - sqrt(x_k)) * 10)
__global__ void vs_softtab_kernel(float r, float cut2, float2* __restrict__ tab) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= kSoftN) return;
  const float h = cut2 * (1.0f / static_cast<float>(kSoftN));
  const float g0 = det_softplus((r - sqrtf(static_cast<float>(k) * h)) * 10.0f);
  const float g1 = det_softplus((r - sqrtf(static_cast<float>(k + 1) * h)) * 10.0f);
  tab[k] = make_float2(g0, g1 - g0);
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

// random 16 B gathers: 8 independent LCG streams per thread over n cells
// (n a power of two); the loaded words feed an xor kept under a never-true
// predicate
__global__ void vs_peak_gather(const uint4* __restrict__ cells, unsigned mask, int iters,
                               unsigned* out) {
  unsigned h[8];
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < 8; ++k) h[k] = t * 2654435761u + 0x9E3779B9u * (k + 1);
  unsigned acc = 0u;
  for (int i = 0; i < iters; ++i) {
    uint4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      h[k] = h[k] * 1664525u + 1013904223u;
      const uint4* c = cells + ((h[k] >> 7) & mask);
      asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[k].x), "=r"(v[k].y), "=r"(v[k].z), "=r"(v[k].w) : "l"(c));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc ^= v[k].x ^ v[k].w;
  }
  if (acc == 0x9E3779B9u) out[0] = acc;
}

// the same with 32 B loads (ld.global.nc.v8.f32, one whole sector per lane:
// the FP32 corner cell of SURVEY §8(d)'s L2_B = 8 corners x 4 B per lookup)
__global__ void vs_peak_gather32(const float4* __restrict__ cells, unsigned mask, int iters,
                                 unsigned* out) {
  unsigned h[8];
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  for (int k = 0; k < 8; ++k) h[k] = t * 2654435761u + 0x9E3779B9u * (k + 1);
  float acc = 0.0f;
  for (int i = 0; i < iters; ++i) {
    float4 lo[8], hi[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      h[k] = h[k] * 1664525u + 1013904223u;
      ldg_cell(cells + 2 * ((h[k] >> 7) & mask), lo[k], hi[k]);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += lo[k].x + hi[k].w;
  }
  if (acc == 1.2345f) out[0] = 1u;
}

}  // namespace vs

// ------------------------------------------------------ launch wrappers --
namespace vs {

size_t rescore_smem_per_block(int nmax, int tmax, int mvmax) {
  return kWarpsPerBlock * warp_smem_bytes(nmax, tmax, mvmax, kLayRescore);
}

template <class K>
static void prep(K kernel, size_t smem) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
}

cudaError_t launch_rescore(bool grid, int blocks, size_t smem, cudaStream_t st, const LibDev& lib,
                           const PocketDev& pk, const int* ligs, int n_ligs, int* counter,
                           const PoseSrc& src, int nmax, int tmax, int mvmax) {
  if (grid) {
    prep(vs_rescore_kernel<1>, smem);
    vs_rescore_kernel<1><<<blocks, kWarpsPerBlock * 32, smem, st>>>(lib, pk, ligs, n_ligs, counter,
                                                                   src, nmax, tmax, mvmax);
  } else {
    prep(vs_rescore_kernel<0>, smem);
    vs_rescore_kernel<0><<<blocks, kWarpsPerBlock * 32, smem, st>>>(lib, pk, ligs, n_ligs, counter,
                                                                   src, nmax, tmax, mvmax);
  }
  return cudaGetLastError();
}

cudaError_t launch_grid(cudaStream_t st, const PocketDev& pk, float* steric, float* hb,
                        float* lipo, float* key, float4* cells) {
  const GridDev& g = pk.grid;
  const long n = static_cast<long>(g.nx) * g.ny * g.nz;
  int blocks = static_cast<int>((n + 255) / 256);
  if (blocks > 148 * 64) blocks = 148 * 64;
  vs_grid_kernel<<<blocks, 256, 0, st>>>(pk, steric, hb, lipo, key);
  const long nc = static_cast<long>(g.nx - 1) * (g.ny - 1) * (g.nz - 1);
  int cb = static_cast<int>((nc + 255) / 256);
  if (cb > 148 * 64) cb = 148 * 64;
  vs_pack_kernel<<<cb, 256, 0, st>>>(g, steric, cells);
  vs_pack_kernel<<<cb, 256, 0, st>>>(g, hb, cells + 2 * nc);
  vs_pack_kernel<<<cb, 256, 0, st>>>(g, lipo, cells + 4 * nc);
  vs_pack_half_kernel<<<cb, 256, 0, st>>>(g, key, const_cast<uint4*>(g.key_h));
  return cudaGetLastError();
}

int topk_chunk() { return kTopkC; }

cudaError_t launch_softtab(cudaStream_t st, float r, float cut2, float2* tab) {
  vs_softtab_kernel<<<(kSoftN + 255) / 256, 256, 0, st>>>(r, cut2, tab);
  return cudaGetLastError();
}

cudaError_t launch_topk(cudaStream_t st, const unsigned long long* in, long n,
                        unsigned long long* out, int k, int blocks) {
  vs_topk_kernel<<<blocks, 1024, 0, st>>>(in, n, out, k);
  return cudaGetLastError();
}

// kind 0 fp32 fma, 1 fp64 fma, 2 ex2; returns ops/s (best of 3)
double measure_gather_peak(int sms, int bytes) {
  const unsigned n = 1u << 19;  // 512 Ki cells x 16 B = 8 MB (x 32 B = 16 MB; L2-resident)
  const size_t cb = bytes == 32 ? 32 : 16;
  void* buf = nullptr;
  if (cudaMalloc(&buf, size_t(n) * cb + 256) != cudaSuccess) return 0.0;
  cudaMemset(buf, 0, size_t(n) * cb + 256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 8, threads = 256, iters = 256;
  double best = 0.0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(a);
    unsigned* sink = reinterpret_cast<unsigned*>(static_cast<char*>(buf) + size_t(n) * cb);
    if (cb == 32)
      vs_peak_gather32<<<blocks, threads>>>(static_cast<const float4*>(buf), n - 1, iters, sink);
    else
      vs_peak_gather<<<blocks, threads>>>(static_cast<const uint4*>(buf), n - 1, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, a, b);
    const double loads = static_cast<double>(blocks) * threads * iters * 8;
    if (rep > 0) best = std::max(best, loads / (ms * 1e-3));
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  return best;
}

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
