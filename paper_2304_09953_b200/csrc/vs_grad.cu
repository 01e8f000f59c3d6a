// score_gradient (dock.cpp:117-160, 278-295) on the GPU, FP64: one warp per
// pose.  The reference's semantics are restated, not its code:
//   - torsion chain in axis order, each axis normalized from the current
//     coordinates, half-angle quaternion, v + 2w(u x v) + 2u x (u x v)
//     (dock.cpp:52-67, geom.hpp:38-53);
//   - score_positions with its per-atom gradient (dock.cpp:70-105):
//     steric Gaussians, pair and wall softplus, sigmoid derivatives;
//   - translation gradient = sum of atom gradients; rotation gradient =
//     d(R(q) y)/dq at unit q projected on the tangent of S^3; torsion
//     gradients by central differences with h = 1e-5.
// Lanes split atoms (gradients: each lane owns its atoms and visits every
// partner, so no cross-lane accumulation) and reductions are fixed xor
// butterflies: results are deterministic; against the reference's serial
// FP64 sums they agree to rounding (tests/test_gpu_parity.py).
#include <cuda_runtime.h>
#include <stdint.h>

#include "vs_types.h"

namespace vs {

struct GradPocket {
  const SiteD* sites;
  int n_sites;
  double lo[3], hi[3];
  double r, lam;
};

constexpr double kSharp = 0.1;  // kClashSharpness (dock.cpp:17)

__device__ __forceinline__ double ref_softplus(double z) { return z > 30.0 ? z : log1p(exp(z)); }
__device__ __forceinline__ double ref_sigmoid(double z) {
  if (z >= 0.0) return 1.0 / (1.0 + exp(-z));
  const double e = exp(z);
  return e / (1.0 + e);
}

__device__ __forceinline__ double wsum(double v) {
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  return v;
}

// v + 2w(u x v) + 2u x (u x v)
__device__ __forceinline__ double3 qrot(double w, double ux, double uy, double uz, double3 v) {
  const double cx = uy * v.z - uz * v.y, cy = uz * v.x - ux * v.z, cz = ux * v.y - uy * v.x;
  const double ex = uy * cz - uz * cy, ey = uz * cx - ux * cz, ez = ux * cy - uy * cx;
  return make_double3(v.x + 2.0 * w * cx + 2.0 * ex, v.y + 2.0 * w * cy + 2.0 * ey,
                      v.z + 2.0 * w * cz + 2.0 * ez);
}

// y = conformer with the torsions applied in axis order (dock.cpp:52-63);
// the moving lists are addressed through the ligand's byte offset
__device__ void grad_chain_mv(const LibDev& lib, int4 meta, int mov_off, const double* th,
                              double3* y, int lane) {
  const int N = meta.y, T = meta.w;
  for (int i = lane; i < N; i += 32) {
    const double4 a = lib.atoms[meta.x + i];
    y[i] = make_double3(a.x, a.y, a.z);
  }
  __syncwarp();
  for (int j = 0; j < T; ++j) {
    const int4 ax = lib.axes[meta.z + j];
    const double3 o = y[ax.x], b = y[ax.y];
    const double dx = b.x - o.x, dy = b.y - o.y, dz = b.z - o.z;
    const double n = sqrt(dx * dx + dy * dy + dz * dz);
    double ux = 0.0, uy = 0.0, uz = 0.0;
    if (n > 0.0) {
      ux = dx / n;
      uy = dy / n;
      uz = dz / n;
    }
    const double h = 0.5 * th[j];
    const double s = sin(h), c = cos(h);
    __syncwarp();
    for (int m = lane; m < ax.w; m += 32) {
      const int idx = lib.moving[mov_off + ax.z + m];
      const double3 v = make_double3(y[idx].x - o.x, y[idx].y - o.y, y[idx].z - o.z);
      const double3 r = qrot(c, ux * s, uy * s, uz * s, v);
      y[idx] = make_double3(o.x + r.x, o.y + r.y, o.z + r.z);
    }
    __syncwarp();
  }
}

// score_positions (dock.cpp:70-105); with g != nullptr also d(score)/dx
__device__ double grad_score(const GradPocket& pk, const double3* x, int N, double3* g,
                             int lane) {
  double s = 0.0;
  for (int a = lane; a < N; a += 32) {
    double gx = 0.0, gy = 0.0, gz = 0.0;
    for (int k = 0; k < pk.n_sites; ++k) {
      const SiteD st = pk.sites[k];
      if (st.kind != 0) continue;
      const double dx = x[a].x - st.cx, dy = x[a].y - st.cy, dz = x[a].z - st.cz;
      const double val = st.w * exp(-(dx * dx + dy * dy + dz * dz) * st.inv2s2);
      s += val;
      const double f = val * 2.0 * st.inv2s2;
      gx -= dx * f;
      gy -= dy * f;
      gz -= dz * f;
    }
    for (int b = 0; b < N; ++b) {
      if (b == a) continue;
      const double dx = x[a].x - x[b].x, dy = x[a].y - x[b].y, dz = x[a].z - x[b].z;
      const double dist = sqrt(dx * dx + dy * dy + dz * dz);
      const double z = (pk.r - dist) / kSharp;
      if (b > a) s -= pk.lam * ref_softplus(z);
      if (g && dist > 1e-12) {
        const double f = pk.lam * ref_sigmoid(z) / (kSharp * dist);
        gx += dx * f;
        gy += dy * f;
        gz += dz * f;
      }
    }
    // wall_distance (dock.cpp:31-44): first minimum of the six faces
    const double d6[6] = {x[a].x - pk.lo[0], pk.hi[0] - x[a].x, x[a].y - pk.lo[1],
                          pk.hi[1] - x[a].y, x[a].z - pk.lo[2], pk.hi[2] - x[a].z};
    int best = 0;
    for (int i = 1; i < 6; ++i)
      if (d6[i] < d6[best]) best = i;
    const double z = (pk.r - d6[best]) / kSharp;
    s -= pk.lam * ref_softplus(z);
    if (g) {
      const double f = pk.lam * ref_sigmoid(z) / kSharp;
      const double sgn = (best & 1) ? -1.0 : 1.0;
      if (best < 2) gx += sgn * f;
      else if (best < 4) gy += sgn * f;
      else gz += sgn * f;
      g[a] = make_double3(gx, gy, gz);
    }
  }
  return wsum(s);
}

// x = R(q) y + t with q normalized (dock.cpp:64-65)
__device__ void grad_pose(const double3* y, int N, double qw, double qx, double qy, double qz,
                          const double* t, double3* x, int lane) {
  for (int i = lane; i < N; i += 32) {
    const double3 r = qrot(qw, qx, qy, qz, y[i]);
    x[i] = make_double3(r.x + t[0], r.y + t[1], r.z + t[2]);
  }
  __syncwarp();
}

__global__ void __launch_bounds__(128)
    vs_grad_kernel(const __grid_constant__ LibDev lib, const __grid_constant__ GradPocket pk,
                   long n_poses, const int* __restrict__ pose_lig, const long* __restrict__ tb,
                   const double* __restrict__ t, const double* __restrict__ q,
                   const double* __restrict__ tors, int nmax, int tmax, double* __restrict__ score,
                   double* __restrict__ gt, double* __restrict__ gq, double* __restrict__ gtor,
                   double* __restrict__ resc) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double3* y = reinterpret_cast<double3*>(smem) + static_cast<size_t>(wib) * 3 * nmax;
  double3* x = y + nmax;
  double3* g = x + nmax;
  double* th = reinterpret_cast<double*>(reinterpret_cast<double3*>(smem) +
                                         static_cast<size_t>(blockDim.x >> 5) * 3 * nmax) +
               static_cast<size_t>(wib) * tmax;
  const long p = static_cast<long>(blockIdx.x) * (blockDim.x >> 5) + wib;
  if (p >= n_poses) return;
  const int lig = pose_lig[p];
  const int4 meta = lib.meta[lig];
  const int N = meta.y, T = meta.w;
  const int mov_off = lib.mov[lig].x;
  // unit q (Quat::normalized)
  const double n = sqrt(q[4 * p] * q[4 * p] + q[4 * p + 1] * q[4 * p + 1] +
                        q[4 * p + 2] * q[4 * p + 2] + q[4 * p + 3] * q[4 * p + 3]);
  const double qw = q[4 * p] / n, qx = q[4 * p + 1] / n, qy = q[4 * p + 2] / n,
               qz = q[4 * p + 3] / n;
  for (int j = lane; j < T; j += 32) th[j] = tors[tb[p] + j];
  __syncwarp();
  grad_chain_mv(lib, meta, mov_off, th, y, lane);
  grad_pose(y, N, qw, qx, qy, qz, t + 3 * p, x, lane);
  const bool with_grad = gt != nullptr;
  const double s0 = grad_score(pk, x, N, with_grad ? g : nullptr, lane);
  __syncwarp();
  if (!with_grad) {
    // score-only (geometric_score, dock.cpp:278-282), plus the kind bonuses
    // of rescore (dock.cpp:297-316): hbond sites over N/O atoms (class 2),
    // lipophilic sites over C atoms (class 1), FP64
    double b = 0.0;
    if (resc) {
      for (int a = lane; a < N; a += 32) {
        const int cls = static_cast<int>(lib.atoms[meta.x + a].w);
        if (cls == 0) continue;
        const int kind = cls == 2 ? 1 : 2;
        for (int k = 0; k < pk.n_sites; ++k) {
          const SiteD st = pk.sites[k];
          if (st.kind != kind) continue;
          const double dx = x[a].x - st.cx, dy = x[a].y - st.cy, dz = x[a].z - st.cz;
          b += st.w * exp(-(dx * dx + dy * dy + dz * dz) * st.inv2s2);
        }
      }
      b = wsum(b);
    }
    if (lane == 0) {
      score[p] = s0;
      if (resc) resc[p] = s0 + b;
    }
    return;
  }
  // translation and raw rotation derivatives, then the tangent projection
  double gtx = 0.0, gty = 0.0, gtz = 0.0, r0 = 0.0, r1 = 0.0, r2 = 0.0, r3 = 0.0;
  for (int i = lane; i < N; i += 32) {
    const double3 v = y[i], gi = g[i];
    gtx += gi.x;
    gty += gi.y;
    gtz += gi.z;
    // u x v
    const double cx = qy * v.z - qz * v.y, cy = qz * v.x - qx * v.z, cz = qx * v.y - qy * v.x;
    r0 += gi.x * 2.0 * cx + gi.y * 2.0 * cy + gi.z * 2.0 * cz;
    const double e[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    double rj[3];
    for (int j = 0; j < 3; ++j) {
      const double ex = e[j][0], ey = e[j][1], ez = e[j][2];
      // e x v
      const double a1 = ey * v.z - ez * v.y, a2 = ez * v.x - ex * v.z, a3 = ex * v.y - ey * v.x;
      // e x (u x v)
      const double b1 = ey * cz - ez * cy, b2 = ez * cx - ex * cz, b3 = ex * cy - ey * cx;
      // u x (e x v)
      const double c1 = qy * a3 - qz * a2, c2 = qz * a1 - qx * a3, c3 = qx * a2 - qy * a1;
      const double dvx = 2.0 * qw * a1 + 2.0 * b1 + 2.0 * c1;
      const double dvy = 2.0 * qw * a2 + 2.0 * b2 + 2.0 * c2;
      const double dvz = 2.0 * qw * a3 + 2.0 * b3 + 2.0 * c3;
      rj[j] = gi.x * dvx + gi.y * dvy + gi.z * dvz;
    }
    r1 += rj[0];
    r2 += rj[1];
    r3 += rj[2];
  }
  gtx = wsum(gtx);
  gty = wsum(gty);
  gtz = wsum(gtz);
  r0 = wsum(r0);
  r1 = wsum(r1);
  r2 = wsum(r2);
  r3 = wsum(r3);
  const double radial = r0 * qw + r1 * qx + r2 * qy + r3 * qz;
  if (lane == 0) {
    score[p] = s0;
    gt[3 * p] = gtx;
    gt[3 * p + 1] = gty;
    gt[3 * p + 2] = gtz;
    gq[4 * p] = r0 - radial * qw;
    gq[4 * p + 1] = r1 - radial * qx;
    gq[4 * p + 2] = r2 - radial * qy;
    gq[4 * p + 3] = r3 - radial * qz;
  }
  // torsions: central differences, h = 1e-5 (dock.cpp:150-157)
  const double h = 1e-5;
  for (int j = 0; j < T; ++j) {
    double sv[2];
    for (int sgn = 0; sgn < 2; ++sgn) {
      __syncwarp();
      if (lane == 0) th[j] = tors[tb[p] + j] + (sgn == 0 ? h : -h);
      __syncwarp();
      grad_chain_mv(lib, meta, mov_off, th, y, lane);
      grad_pose(y, N, qw, qx, qy, qz, t + 3 * p, x, lane);
      sv[sgn] = grad_score(pk, x, N, nullptr, lane);
    }
    __syncwarp();
    if (lane == 0) {
      th[j] = tors[tb[p] + j];
      gtor[tb[p] + j] = (sv[0] - sv[1]) / (2.0 * h);
    }
  }
}

// ---- the reference ascent (dock.cpp:168-203) per pose, device-resident
// (refine.ascend_poses_device).  State t (registers), q (registers, as given:
// the evaluations normalize it like transformed() does), torsions in shared
// memory; every score and gradient is the arithmetic of vs_grad_kernel.

// score and gradient at (t, q, th); the torsion gradient goes to G
__device__ double ascent_grad(const LibDev& lib, const GradPocket& pk, int4 meta, int mov_off,
                              double* th, const double* t, const double* q, double3* y,
                              double3* x, double3* g, double* gt, double* gq, double* G,
                              int lane) {
  const int N = meta.y, T = meta.w;
  const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  const double qw = q[0] / n, qx = q[1] / n, qy = q[2] / n, qz = q[3] / n;
  grad_chain_mv(lib, meta, mov_off, th, y, lane);
  grad_pose(y, N, qw, qx, qy, qz, t, x, lane);
  const double s0 = grad_score(pk, x, N, g, lane);
  __syncwarp();
  double gtx = 0.0, gty = 0.0, gtz = 0.0, r0 = 0.0, r1 = 0.0, r2 = 0.0, r3 = 0.0;
  for (int i = lane; i < N; i += 32) {
    const double3 v = y[i], gi = g[i];
    gtx += gi.x;
    gty += gi.y;
    gtz += gi.z;
    const double cx = qy * v.z - qz * v.y, cy = qz * v.x - qx * v.z, cz = qx * v.y - qy * v.x;
    r0 += gi.x * 2.0 * cx + gi.y * 2.0 * cy + gi.z * 2.0 * cz;
    const double e[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    double rj[3];
    for (int j = 0; j < 3; ++j) {
      const double ex = e[j][0], ey = e[j][1], ez = e[j][2];
      const double a1 = ey * v.z - ez * v.y, a2 = ez * v.x - ex * v.z, a3 = ex * v.y - ey * v.x;
      const double b1 = ey * cz - ez * cy, b2 = ez * cx - ex * cz, b3 = ex * cy - ey * cx;
      const double c1 = qy * a3 - qz * a2, c2 = qz * a1 - qx * a3, c3 = qx * a2 - qy * a1;
      const double dvx = 2.0 * qw * a1 + 2.0 * b1 + 2.0 * c1;
      const double dvy = 2.0 * qw * a2 + 2.0 * b2 + 2.0 * c2;
      const double dvz = 2.0 * qw * a3 + 2.0 * b3 + 2.0 * c3;
      rj[j] = gi.x * dvx + gi.y * dvy + gi.z * dvz;
    }
    r1 += rj[0];
    r2 += rj[1];
    r3 += rj[2];
  }
  gt[0] = wsum(gtx);
  gt[1] = wsum(gty);
  gt[2] = wsum(gtz);
  r0 = wsum(r0);
  r1 = wsum(r1);
  r2 = wsum(r2);
  r3 = wsum(r3);
  const double radial = r0 * qw + r1 * qx + r2 * qy + r3 * qz;
  gq[0] = r0 - radial * qw;
  gq[1] = r1 - radial * qx;
  gq[2] = r2 - radial * qy;
  gq[3] = r3 - radial * qz;
  const double h = 1e-5;
  for (int j = 0; j < T; ++j) {
    const double v = th[j];
    double sv[2];
    for (int sgn = 0; sgn < 2; ++sgn) {
      __syncwarp();
      if (lane == 0) th[j] = v + (sgn == 0 ? h : -h);
      __syncwarp();
      grad_chain_mv(lib, meta, mov_off, th, y, lane);
      grad_pose(y, N, qw, qx, qy, qz, t, x, lane);
      sv[sgn] = grad_score(pk, x, N, nullptr, lane);
    }
    __syncwarp();
    if (lane == 0) {
      th[j] = v;
      G[j] = (sv[0] - sv[1]) / (2.0 * h);
    }
  }
  __syncwarp();
  return s0;
}

__global__ void __launch_bounds__(128)
    vs_ascend_kernel(const __grid_constant__ LibDev lib, const __grid_constant__ GradPocket pk,
                     long n_poses, const int* __restrict__ pose_lig, const long* __restrict__ tb,
                     double* __restrict__ t, double* __restrict__ q, double* __restrict__ tors,
                     int nmax, int tmax, int max_steps, double* __restrict__ score,
                     int* __restrict__ steps_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  double3* y = reinterpret_cast<double3*>(smem) + static_cast<size_t>(wib) * 3 * nmax;
  double3* x = y + nmax;
  double3* g = x + nmax;
  double* th = reinterpret_cast<double*>(reinterpret_cast<double3*>(smem) +
                                         static_cast<size_t>(nw) * 3 * nmax) +
               static_cast<size_t>(wib) * 3 * tmax;
  double* G = th + tmax;
  double* th2 = G + tmax;
  const long p = static_cast<long>(blockIdx.x) * nw + wib;
  if (p >= n_poses) return;
  const int lig = pose_lig[p];
  const int4 meta = lib.meta[lig];
  const int T = meta.w;
  const int mov_off = lib.mov[lig].x;
  double pt[3] = {t[3 * p], t[3 * p + 1], t[3 * p + 2]};
  double pq[4];
  {  // p.q = p.q.normalized() (dock.cpp:169)
    const double* q0 = q + 4 * p;
    const double n = sqrt(q0[0] * q0[0] + q0[1] * q0[1] + q0[2] * q0[2] + q0[3] * q0[3]);
    for (int c = 0; c < 4; ++c) pq[c] = q0[c] / n;
  }
  for (int j = lane; j < T; j += 32) th[j] = tors[tb[p] + j];
  __syncwarp();
  double gt[3], gq[4];
  double s = ascent_grad(lib, pk, meta, mov_off, th, pt, pq, y, x, g, gt, gq, G, lane);
  int step = 0;
  for (; step < max_steps; ++step) {
    // |g|^2 in the reference's order (dock.cpp:176-177)
    double gn2 = gt[0] * gt[0] + gt[1] * gt[1] + gt[2] * gt[2] + gq[0] * gq[0] + gq[1] * gq[1] +
                 gq[2] * gq[2] + gq[3] * gq[3];
    for (int j = 0; j < T; ++j) gn2 += G[j] * G[j];
    if (sqrt(gn2) < 1e-6) break;
    double alpha = 0.5;
    bool accepted = false;
    while (alpha > 1e-14) {
      double tt[3], tq[4];
      for (int c = 0; c < 3; ++c) tt[c] = pt[c] + gt[c] * alpha;
      for (int c = 0; c < 4; ++c) tq[c] = pq[c] + gq[c] * alpha;
      const double n = sqrt(tq[0] * tq[0] + tq[1] * tq[1] + tq[2] * tq[2] + tq[3] * tq[3]);
      for (int c = 0; c < 4; ++c) tq[c] = tq[c] / n;
      for (int j = lane; j < T; j += 32) th2[j] = th[j] + G[j] * alpha;
      __syncwarp();
      // obj.eval(trial): score only
      const double nn = sqrt(tq[0] * tq[0] + tq[1] * tq[1] + tq[2] * tq[2] + tq[3] * tq[3]);
      grad_chain_mv(lib, meta, mov_off, th2, y, lane);
      grad_pose(y, meta.y, tq[0] / nn, tq[1] / nn, tq[2] / nn, tq[3] / nn, tt, x, lane);
      const double st = grad_score(pk, x, meta.y, nullptr, lane);
      if (st >= s + 1e-4 * alpha * gn2) {
        for (int c = 0; c < 3; ++c) pt[c] = tt[c];
        for (int c = 0; c < 4; ++c) pq[c] = tq[c];
        __syncwarp();
        for (int j = lane; j < T; j += 32) th[j] = th2[j];
        __syncwarp();
        s = st;
        accepted = true;
        break;
      }
      alpha *= 0.5;
    }
    if (!accepted) break;
    s = ascent_grad(lib, pk, meta, mov_off, th, pt, pq, y, x, g, gt, gq, G, lane);
  }
  if (lane == 0) {
    for (int c = 0; c < 3; ++c) t[3 * p + c] = pt[c];
    for (int c = 0; c < 4; ++c) q[4 * p + c] = pq[c];
    score[p] = s;
    steps_out[p] = step;
  }
  for (int j = lane; j < T; j += 32) tors[tb[p] + j] = th[j];
}

size_t ascend_smem_per_block(int nmax, int tmax) {
  return 4 * (3 * static_cast<size_t>(nmax) * sizeof(double3) + 3 * static_cast<size_t>(tmax) * 8);
}

cudaError_t launch_ascend(cudaStream_t st, const LibDev& lib, const SiteD* sites, int n_sites,
                          const double lo[3], const double hi[3], double r, double lam,
                          long n_poses, const int* pose_lig, const long* tb, double* t, double* q,
                          double* tors, int nmax, int tmax, int max_steps, double* score,
                          int* steps) {
  GradPocket pk;
  pk.sites = sites;
  pk.n_sites = n_sites;
  for (int c = 0; c < 3; ++c) {
    pk.lo[c] = lo[c];
    pk.hi[c] = hi[c];
  }
  pk.r = r;
  pk.lam = lam;
  const size_t smem = ascend_smem_per_block(nmax, tmax);
  cudaFuncSetAttribute(vs_ascend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  const long blocks = (n_poses + 3) / 4;
  vs_ascend_kernel<<<static_cast<unsigned>(blocks), 128, smem, st>>>(
      lib, pk, n_poses, pose_lig, tb, t, q, tors, nmax, tmax, max_steps, score, steps);
  return cudaGetLastError();
}

size_t grad_smem_per_block(int nmax, int tmax) {
  return 4 * (3 * static_cast<size_t>(nmax) * sizeof(double3) + static_cast<size_t>(tmax) * 8);
}

cudaError_t launch_grad(cudaStream_t st, const LibDev& lib, const SiteD* sites, int n_sites,
                        const double lo[3], const double hi[3], double r, double lam,
                        long n_poses, const int* pose_lig, const long* tb, const double* t,
                        const double* q, const double* tors, int nmax, int tmax, double* score,
                        double* gt, double* gq, double* gtor, double* resc) {
  GradPocket pk;
  pk.sites = sites;
  pk.n_sites = n_sites;
  for (int c = 0; c < 3; ++c) {
    pk.lo[c] = lo[c];
    pk.hi[c] = hi[c];
  }
  pk.r = r;
  pk.lam = lam;
  const size_t smem = grad_smem_per_block(nmax, tmax);
  cudaFuncSetAttribute(vs_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  const long blocks = (n_poses + 3) / 4;
  vs_grad_kernel<<<static_cast<unsigned>(blocks), 128, smem, st>>>(
      lib, pk, n_poses, pose_lig, tb, t, q, tors, nmax, tmax, score, gt, gq, gtor, resc);
  return cudaGetLastError();
}

}  // namespace vs
