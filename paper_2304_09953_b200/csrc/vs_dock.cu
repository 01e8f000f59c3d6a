// The dock kernels (K2 + K3 + K4a of DESIGN.md §3): sweep-v1 pose
// generation, canonical scoring, diversity, keep-top filter, rescore,
// per-ligand best and top-k key — one warp per ligand, persistent warps
// pulling ligands from an atomic counter over one global LPT order (largest
// ligands first), one kernel per phase and restart (start, sweep, flex,
// polish + keep; then finish), the per-ligand state handed over in HBM.
//
// The phases are inlined into their kernels (out-of-line phases paid ABI
// register saves on every call); the hot inner loops are kept small instead
// (sweep key: ~54 SASS instructions, never unrolled) so they stay resident in
// the SM's ~6 KB L0 instruction cache.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "vs_common.cuh"

#define VS_PHASE __forceinline__  // see header comment

// key-map gathers through the texture path (TEX) or LDG: the sweep
// kernel's (rotation sweep + compass) run faster on TEX (same bits), the
// polish kernel's on LDG (profiles/e2e_pipeline_r2.txt)
#ifndef VS_TEX_SWEEP
#define VS_TEX_SWEEP true
#endif
#ifndef VS_TEX_POLISH
#define VS_TEX_POLISH false
#endif

namespace vs {

struct Dims {
  int nmax, tmax, mvmax, lay;
};

struct PoseF {
  float t[3];
  float q[4];
};

__device__ __forceinline__ WarpSmem dock_smem(const Dims d) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  return carve(smem_raw + (threadIdx.x >> 5) * warp_smem_bytes(d.nmax, d.tmax, d.mvmax, d.lay),
               d.nmax, d.tmax, d.mvmax, d.lay);
}

// ---- start of restart r (dock.cpp:343-356): first attempt whose start
// coordinates are at RMSD >= delta from every kept pose (or the 50th);
// leaves the torsion-applied state in s.ys / s.ysf and s.theta.
static __device__ VS_PHASE int start_phase(const PocketDev& pk, const Dims d,
                                               unsigned long long rkey, int N, int T,
                                               const float4* kx, int kstride, int nk, float delta,
                                               int lane, PoseF* P) {
  const WarpSmem s = dock_smem(d);
  float t[3], q[4];
  int att = 0;
  bool have_chain = false;
  for (; att < 50; ++att) {
    draw_start(pk, rkey, att, T, s, lane, t, q);
    if (nk == 0) break;
    chain_coop(s, N, T, lane);
    have_chain = true;
    pose_coop(s, N, det_pose_mat_d(q[0], q[1], q[2], q[3]), t[0], t[1], t[2], lane);
    if (diverse_from_kept(s, kx, nk, kstride, N, delta, lane)) break;
  }
  if (att == 50) att = 49;
  if (!have_chain) chain_coop(s, N, T, lane);
  if (s.ysf) {
    for (int i = lane; i < N; i += 32) {
      const double4 v = s.ys[i];
      s.ysf[i] = make_float4(static_cast<float>(v.x), static_cast<float>(v.y),
                             static_cast<float>(v.z), 0.0f);
    }
  }
  __syncwarp();
  for (int c = 0; c < 3; ++c) P->t[c] = t[c];
  for (int c = 0; c < 4; ++c) P->q[c] = q[c];
  return att;
}

// ---- rigid roto-translation sweep (SWEEP_V1.md §2.3-2.4): K orientations
// about the posed centroid (lanes over rotations), then a compass search
// over the 26 lattice neighbours with halving steps.  FP32 key F - lam W.

// ---- rigid compass of the polish (SWEEP_V1.md §3.5), on the FP32 state
// copy with the sweep key.  Lane l < 31 is candidate l: 0 keeps the pose;
// 1..6 rotate by +-ang about world x y z through the posed centroid (cx, cy,
// cz); 7..12 translate by +-sc along x y z; 13..18 rotate by +-3 ang,
// 19..24 translate by +-2 sc; 25..30 translate by +-12 sc.  Argmax, ties to
// the lowest lane; l = 0 halves the steps, a winner l >= 13 doubles them
// while ang < kPolishAngMax.  At most kPolishIters iterations; the long
// jumps only in the first kLongJumpIters.
constexpr float kPolishAng0 = 0.28125f;
constexpr float kPolishSc0 = 0.5f;
constexpr float kPolishAngMin = 0.015625f;
constexpr float kPolishAngMax = 0.5625f;
constexpr int kPolishIters = 8;
constexpr int kCompassLanes = 31;
constexpr int kLongJumpIters = 4;

template <int kGrid, bool kTex>
static __device__ __forceinline__ int rigid_compass(const PocketDev& pk, const KeyAtoms& ka, int N,
                                                    float cx, float cy, float cz, PoseF* P,
                                                    int lane) {
  float qw = P->q[0], qx = P->q[1], qy = P->q[2], qz = P->q[3];
  float tx = P->t[0], ty = P->t[1], tz = P->t[2];
  float ang = kPolishAng0, sc = kPolishSc0;
  int it = 0;
  for (; it < kPolishIters && ang >= kPolishAngMin; ++it) {
    const Mat3 R0 = det_quat_mat(qw, qx, qy, qz);
    float Cx, Cy, Cz;
    det_apply(R0, cx, cy, cz, tx, ty, tz, &Cx, &Cy, &Cz);
    float w2 = qw, x2 = qx, y2 = qy, z2 = qz, u2 = tx, v2 = ty, s2 = tz;
    float key = -INFINITY;
    // the long jumps (lanes 25..30) take part in the first kLongJumpIters
    // iterations only
    const int n_lanes = it < kLongJumpIters ? kCompassLanes : 25;
    if (lane < n_lanes) {
      const bool big = lane >= 13;
      const bool huge = lane >= 25;
      const int lm = huge ? lane - 18 : (big ? lane - 12 : lane);
      const float a2 = big ? 3.0f * ang : ang;
      const float sc2 = huge ? 12.0f * sc : (big ? 2.0f * sc : sc);
      Mat3 R2 = R0;
      if (lm >= 1 && lm <= 6) {
        const int ax = (lm - 1) >> 1;
        float sh, ch;
        det_sincos(0.5f * a2, &sh, &ch);
        const float sg = ((lm - 1) & 1) ? -sh : sh;
        det_quat_mul(ch, ax == 0 ? sg : 0.0f, ax == 1 ? sg : 0.0f, ax == 2 ? sg : 0.0f, qw, qx,
                     qy, qz, &w2, &x2, &y2, &z2);
        det_quat_normalize(&w2, &x2, &y2, &z2);
        R2 = det_quat_mat(w2, x2, y2, z2);
        float vx, vy, vz;
        det_apply(R2, cx, cy, cz, 0.0f, 0.0f, 0.0f, &vx, &vy, &vz);
        u2 = Cx - vx;
        v2 = Cy - vy;
        s2 = Cz - vz;
      } else if (lm >= 7) {
        const int ax = (lm - 7) >> 1;
        const bool neg = (lm - 7) & 1;
        if (ax == 0) u2 = neg ? tx - sc2 : tx + sc2;
        if (ax == 1) v2 = neg ? ty - sc2 : ty + sc2;
        if (ax == 2) s2 = neg ? tz - sc2 : tz + sc2;
      }
      key = eval_key<kGrid, kTex>(pk, ka, N, R2, u2, v2, s2);
    }
    int li = lane < n_lanes ? lane : 0x7fffffff;
    for (int off = 16; off > 0; off >>= 1) {
      const float ok = __shfl_xor_sync(kFull, key, off);
      const int oi = __shfl_xor_sync(kFull, li, off);
      if (ok > key || (ok == key && oi < li)) {
        key = ok;
        li = oi;
      }
    }
    if (li == 0) {
      ang = ang * 0.5f;
      sc = sc * 0.5f;
    } else {
      qw = __shfl_sync(kFull, w2, li);
      qx = __shfl_sync(kFull, x2, li);
      qy = __shfl_sync(kFull, y2, li);
      qz = __shfl_sync(kFull, z2, li);
      tx = __shfl_sync(kFull, u2, li);
      ty = __shfl_sync(kFull, v2, li);
      tz = __shfl_sync(kFull, s2, li);
      if (li >= 13 && ang < kPolishAngMax) {
        ang = ang * 2.0f;
        sc = sc * 2.0f;
      }
    }
  }
  P->q[0] = qw;
  P->q[1] = qx;
  P->q[2] = qy;
  P->q[3] = qz;
  P->t[0] = tx;
  P->t[1] = ty;
  P->t[2] = tz;
  return it;
}

// Lanes take the rotations in the locality order `perm` (host: rotation
// clusters of 32, so the 32 lanes of one key-cell gather hold nearby
// orientations and touch fewer 128 B lines); the argmax breaks ties on the
// rotation index k itself, so the winner is the one of the index-ordered
// sweep (SWEEP_V1.md §2.3), bit for bit.
template <int kGrid>
static __device__ VS_PHASE int sweep_phase(const PocketDev& pk, const Dims d,
                                               const float4* __restrict__ rots,
                                               const float4* __restrict__ rots_p,
                                               const int* __restrict__ perm, int K, int N,
                                               int lane, PoseF* P, int* n_trans, int polish) {
  const WarpSmem s = dock_smem(d);
  const KeyAtoms ka = pairs_of(s.ysf, d.nmax);
  float qs0 = P->q[0], qs1 = P->q[1], qs2 = P->q[2], qs3 = P->q[3];
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
  det_apply(det_quat_mat(qs0, qs1, qs2, qs3), cx, cy, cz, P->t[0], P->t[1], P->t[2], &Cx, &Cy,
            &Cz);

  float best_key = -INFINITY;
  int best_k = 0x7fffffff;
  for (int p = lane; p < K; p += 32) {
    const int k = perm[p];
    const float4 rq = rots_p[p];  // = rots[k], loaded independently of k
    float w4, x4, y4, z4;
    det_quat_mul(rq.x, rq.y, rq.z, rq.w, qs0, qs1, qs2, qs3, &w4, &x4, &y4, &z4);
    det_quat_normalize(&w4, &x4, &y4, &z4);
    const Mat3 Rk = det_quat_mat(w4, x4, y4, z4);
    float vx, vy, vz;
    det_apply(Rk, cx, cy, cz, 0.0f, 0.0f, 0.0f, &vx, &vy, &vz);
    const float key = eval_key<kGrid, VS_TEX_SWEEP>(pk, ka, N, Rk, Cx - vx, Cy - vy, Cz - vz);
    if (key > best_key || (key == best_key && k < best_k)) {
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
  const Mat3 RS = det_quat_mat(pw, px, py, pz);
  float ptx, pty, ptz;
  {
    float vx, vy, vz;
    det_apply(RS, cx, cy, cz, 0.0f, 0.0f, 0.0f, &vx, &vy, &vz);
    ptx = Cx - vx;
    pty = Cy - vy;
    ptz = Cz - vz;
  }
  if (polish >= 1) {  // §3.5: the rigid compass replaces the translation lattice
    P->t[0] = ptx;
    P->t[1] = pty;
    P->t[2] = ptz;
    P->q[0] = pw;
    P->q[1] = px;
    P->q[2] = py;
    P->q[3] = pz;
    *n_trans += rigid_compass<kGrid, VS_TEX_SWEEP>(pk, ka, N, cx, cy, cz, P, lane);
    return best_k;
  }
  float sc = 1.0f;
  int it = 0;
  for (; it < kTransIters && sc >= kTransMin; ++it) {
    float key = -INFINITY, ox = 0.0f, oy = 0.0f, oz = 0.0f;
    if (lane < 27) {
      trans_offset(lane, sc, &ox, &oy, &oz);
      key = eval_key<kGrid, VS_TEX_SWEEP>(pk, ka, N, RS, ptx + ox, pty + oy, ptz + oz);
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
  }
  *n_trans += it;
  P->t[0] = ptx;
  P->t[1] = pty;
  P->t[2] = ptz;
  P->q[0] = pw;
  P->q[1] = px;
  P->q[2] = py;
  P->q[3] = pz;
  return best_k;
}

// ---- incremental greedy torsion flex (SWEEP_V1.md §2.5).  Per (pass,
// axis j) the 16 candidate angles are scored as base(state: atoms outside
// moving_j, pairs not crossing it; 32-lane strided sums + xor butterfly)
// + moved part(candidate: moving_j atoms rotated about the state's axis j
// and their cross pairs; lane pair (a, h), lane h takes moving positions
// = h mod 2).  Returns the score of the final state.
template <int kGrid, bool kPacked = false, bool kTab = false>
static __device__ VS_PHASE float flex_phase(const PocketDev& pk, const Dims d, int N, int T,
                                                int F, int A, float step, const PoseF* P,
                                                int lane, unsigned long long* n_active,
                                                int polish, const float2* tab = nullptr) {
  const WarpSmem s = dock_smem(d);
  const int a_lane = lane & 15;
  const int h = lane >> 4;
  // the FP32 search (polish >= 1, grid mode; SWEEP_V1.md §3.4) scores each
  // candidate's moved atoms on the sweep key in the pose's grid frame and
  // needs no per-atom caches (the base sums are not part of its score)
  constexpr bool kSearch32 = kTab && kGrid;
  if (lane == 0) {
    if (kSearch32) {
      const GridDev& g = pk.grid;
      const float ih = g.inv_h;
      const Mat3 R = det_quat_mat(P->q[0], P->q[1], P->q[2], P->q[3]);
      float4* gf = reinterpret_cast<float4*>(s.pose);
      gf[0] = make_float4(R.m00 * ih, R.m01 * ih, R.m02 * ih, (P->t[0] - g.ox) * ih);
      gf[1] = make_float4(R.m10 * ih, R.m11 * ih, R.m12 * ih, (P->t[1] - g.oy) * ih);
      gf[2] = make_float4(R.m20 * ih, R.m21 * ih, R.m22 * ih, (P->t[2] - g.oz) * ih);
    } else {
      const Mat3d RD = det_pose_mat_d(P->q[0], P->q[1], P->q[2], P->q[3]);
      double* pm = s.pose;
      pm[0] = RD.m00; pm[1] = RD.m01; pm[2] = RD.m02;
      pm[3] = RD.m10; pm[4] = RD.m11; pm[5] = RD.m12;
      pm[6] = RD.m20; pm[7] = RD.m21; pm[8] = RD.m22;
      pm[9] = P->t[0]; pm[10] = P->t[1]; pm[11] = P->t[2];
    }
  }
  __syncwarp();
  for (int i = lane; !kSearch32 && i < N; i += 32) {
    const double4 v = s.ys[i];
    atom_terms_s<kGrid>(pk, s.pose, v.x, v.y, v.z, &s.fa[i], &s.wa[i]);
  }
  __syncwarp();
  const bool do_flex = T > 0 && F > 0;
  const int steps0 = do_flex ? F * T : 1;
  // polish 2: one more pass over the torsions with fine candidate angles
  const int steps = steps0 + ((do_flex && polish >= 2) ? T : 0);
  const int W = (N + 31) >> 5;
  int quiet = 0;  // consecutive coarse steps without a move
  float S_cur = 0.0f;
  int nact = 0;  // pair softplus evaluations of this lane (work counter)
  for (int st = 0; st < steps; ++st) {
    const int j = do_flex ? st % T : -1;
    const int4 ax = do_flex ? s.ax[j] : make_int4(0, 0, 0, 0);
    const int m = ax.w;
    const unsigned* mk = do_flex ? s.tmask + 4 * j : s.mask;
    // base sums (atoms outside moving_j, pairs not crossing it): common to
    // every candidate of the step, so the search with the polish (§3.4)
    // ranks the candidates without them
    float fb = 0.0f, wb = 0.0f, pb = 0.0f;
    for (int i = lane; !kTab && i < N; i += 32) {
      if (!in_mask(mk, i)) {
        fb = fb + s.fa[i];
        wb = wb + s.wa[i];
      }
    }
    if (!kTab) {
      // lane l takes the pairs p = l, l + 32, ... of the row-major (i < k)
      // order, (i, k) advanced incrementally: every lane busy, same pairs and
      // per-lane order as a 32-strided walk of each row
      int i = 0, k = lane + 1;
      while (i < N - 1 && k >= N) {
        k = k - N + i + 2;
        ++i;
      }
      while (i < N - 1) {
        if (in_mask(mk, i) == in_mask(mk, k)) {
          const double4 yi = s.ys[i], yk = s.ys[k];
          pb = pb + pair_term_s<kTab>(pk, tab, yi.x - yk.x, yi.y - yk.y, yi.z - yk.z, nact);
        }
        k += 32;
        while (i < N - 1 && k >= N) {
          k = k - N + i + 2;
          ++i;
        }
      }
    }
    // kPacked: the partners of this step (atoms outside moving_j, ascending)
    // packed into the conformer's region, which the staged flex kernel no
    // longer reads; the candidate loop then walks a plain list
    int np = 0;
    if (kPacked && do_flex) {  // (np stays 0 otherwise)
      for (int i0 = 0; i0 < N; i0 += 32) {
        const int i = i0 + lane;
        const bool pt = i < N && !in_mask(mk, i);
        const unsigned bal = __ballot_sync(kFull, pt);
        if (pt) {
          const int p = np + __popc(bal & ((1u << lane) - 1u));
          const double4 v = s.ys[i];
          if (kTab)  // the search tests cross pairs in FP32
            reinterpret_cast<float4*>(s.y0)[p] = make_float4(
                static_cast<float>(v.x), static_cast<float>(v.y), static_cast<float>(v.z), 0.0f);
          else
            s.y0[p] = v;
        }
        np += __popc(bal);
      }
      __syncwarp();
    }
    if (!kTab) {
      fb = warp_sum(fb);
      wb = warp_sum(wb);
      pb = warp_sum(pb);
    }
    const bool active = do_flex && a_lane < A;
    float th_new = 0.0f;
    float fm = 0.0f, wm = 0.0f, pc = 0.0f;
    if (active) {
      const float th_old = s.theta[j];
      th_new = th_old;
      if (a_lane > 0) {
        float v;
        if (st >= steps0) {  // fine pass: offsets (-A/2, A/2] of step / 8
          const int off = a_lane <= A / 2 ? a_lane : a_lane - A;
          v = th_old + static_cast<float>(off) * (step * 0.125f);
          if (v < -kPiF) v = v + kTwoPiF;
        } else {
          v = th_old + static_cast<float>(a_lane) * step;
        }
        if (v >= kPiF) v = v - kTwoPiF;
        th_new = v;
      }
      const double4 o = s.ys[ax.x], b = s.ys[ax.y];
      if constexpr (kSearch32) {
        // FP32 candidate rotation about the state's axis by th_new - th_old
        const float ofx = static_cast<float>(o.x), ofy = static_cast<float>(o.y),
                    ofz = static_cast<float>(o.z);
        float hh = 0.5f * (th_new - th_old);
        if (hh > kHalfPiF) hh = hh - kPiF;
        else if (hh < -kHalfPiF) hh = hh + kPiF;
        float sn, cs;
        det_sincos(hh, &sn, &cs);
        const float ks = sn * static_cast<float>(s.axl[j]);
        const Mat3 Mf = det_quat_mat(cs, static_cast<float>(b.x - o.x) * ks,
                                     static_cast<float>(b.y - o.y) * ks,
                                     static_cast<float>(b.z - o.z) * ks);
        const float4* gf = reinterpret_cast<const float4*>(s.pose);
        const float4 r0 = gf[0], r1 = gf[1], r2 = gf[2];  // the pose's grid frame
        for (int q2 = h; q2 < m; q2 += 2) {
          const double4 v = s.ys[s.mov[ax.z + q2]];
          const float vx = static_cast<float>(v.x - o.x), vy = static_cast<float>(v.y - o.y),
                      vz = static_cast<float>(v.z - o.z);
          const float fx = fmaf(Mf.m00, vx, fmaf(Mf.m01, vy, fmaf(Mf.m02, vz, ofx)));
          const float fy = fmaf(Mf.m10, vx, fmaf(Mf.m11, vy, fmaf(Mf.m12, vz, ofy)));
          const float fz = fmaf(Mf.m20, vx, fmaf(Mf.m21, vy, fmaf(Mf.m22, vz, ofz)));
          fm = fm + key_at_grid(pk, fmaf(r0.x, fx, fmaf(r0.y, fy, fmaf(r0.z, fz, r0.w))),
                                fmaf(r1.x, fx, fmaf(r1.y, fy, fmaf(r1.z, fz, r1.w))),
                                fmaf(r2.x, fx, fmaf(r2.y, fy, fmaf(r2.z, fz, r2.w))));
          if constexpr (kPacked) {
            const float4* part = reinterpret_cast<const float4*>(s.y0);
            float4 yk = part[0];
            for (int p = 0; p < np; ++p) {
              const float4 yn = part[p + 1];
              pc = pc + pair_term_f(pk, tab, fx - yk.x, fy - yk.y, fz - yk.z, nact);
              yk = yn;
            }
          } else {
            for (int k = 0; k < N; ++k)
              if (!in_mask(mk, k)) {
                const double4 yk = s.ys[k];
                pc = pc + pair_term_f(pk, tab, fx - static_cast<float>(yk.x),
                                      fy - static_cast<float>(yk.y),
                                      fz - static_cast<float>(yk.z), nact);
              }
          }
        }
      } else {
      const Mat3d M = flex_mat(o.x, o.y, o.z, b.x, b.y, b.z, th_new, th_old, s.axl[j]);
      // partners: the atoms outside moving_j, walked as set bits of the
      // complemented mask (ascending k, same trip count in both halves)
      for (int q2 = h; q2 < m; q2 += 2) {
        const double4 v = s.ys[s.mov[ax.z + q2]];
        double yx, yy, yz;
        det_apply_d(M, v.x - o.x, v.y - o.y, v.z - o.z, o.x, o.y, o.z, &yx, &yy, &yz);
        float fi, wi;
        atom_terms_s<kGrid>(pk, s.pose, yx, yy, yz, &fi, &wi);
        fm = fm + fi;
        wm = wm + wi;
        if constexpr (kPacked && kTab) {
          // the search (§3.4): FP32 moved atom against the FP32 partner list
          const float4* part = reinterpret_cast<const float4*>(s.y0);
          const float fx = static_cast<float>(yx), fy = static_cast<float>(yy),
                      fz = static_cast<float>(yz);
          float4 yk = part[0];
          for (int p = 0; p < np; ++p) {
            const float4 yn = part[p + 1];
            pc = pc + pair_term_f(pk, tab, fx - yk.x, fy - yk.y, fz - yk.z, nact);
            yk = yn;
          }
        } else if constexpr (kPacked) {
          // next partner loaded before this pair's test; part[np] (np < N:
          // moving_j holds b_j) is in the buffer and unused
          const double4* part = s.y0;
          double4 yk = part[0];
          for (int p = 0; p < np; ++p) {
            const double4 yn = part[p + 1];
            pc = pc + pair_term_s<kTab>(pk, tab, yx - yk.x, yy - yk.y, yz - yk.z, nact);
            yk = yn;
          }
        } else {
          for (int wd = 0; wd < W; ++wd) {
            unsigned b2 = ~mk[wd];
            if (wd == W - 1 && (N & 31)) b2 &= (1u << (N & 31)) - 1u;
            if (!b2) continue;
            // the next partner's coordinates are loaded before this pair's
            // test (shared-memory latency off the dependent chain)
            const double4* yw = s.ys + wd * 32;
            double4 yk = yw[__ffs(b2) - 1];
            while (true) {
              b2 &= b2 - 1u;
              const double4 yn = yw[b2 ? __ffs(b2) - 1 : 0];
              if (kTab)  // the search (§3.4): FP32 cross pairs
                pc = pc + pair_term_f(pk, tab, static_cast<float>(yx) - static_cast<float>(yk.x),
                                      static_cast<float>(yy) - static_cast<float>(yk.y),
                                      static_cast<float>(yz) - static_cast<float>(yk.z), nact);
              else
                pc = pc + pair_term_s<kTab>(pk, tab, yx - yk.x, yy - yk.y, yz - yk.z, nact);
              if (!b2) break;
              yk = yn;
            }
          }
        }
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
      const Mat3d M = flex_mat(o.x, o.y, o.z, b.x, b.y, b.z, th_win, th_old, s.axl[j]);
      __syncwarp();
      for (int q2 = lane; q2 < m; q2 += 32) {
        const int idx = s.mov[ax.z + q2];
        double4 v = s.ys[idx];
        det_apply_d(M, v.x - o.x, v.y - o.y, v.z - o.z, o.x, o.y, o.z, &v.x, &v.y, &v.z);
        s.ys[idx] = v;
        if (!kSearch32) atom_terms_s<kGrid>(pk, s.pose, v.x, v.y, v.z, &s.fa[idx], &s.wa[idx]);
      }
      if (lane == 0) s.theta[j] = th_win;
    }
    // T coarse steps in a row without a move: every torsion is at its argmax
    // for the current state, so the remaining coarse steps would evaluate the
    // same states and keep them.  Skip to the last coarse step (its S is the
    // flex score when polish is 0) or, with the polish, past it.
    if (do_flex && st < steps0) {
      quiet = ai != 0 ? 0 : quiet + 1;
      if (quiet >= T && st < steps0 - 2) st = polish >= 1 ? steps0 - 1 : steps0 - 2;
    }
    __syncwarp();
  }
  for (int off = 16; off > 0; off >>= 1) nact += __shfl_xor_sync(kFull, nact, off);
  *n_active += static_cast<unsigned long long>(nact);
  return S_cur;
}

// ---- polish (SWEEP_V1.md §3.5) after the flex: the rigid compass on the
// flexed state, then the canonical score of the final pose as a flex step
// with an empty moving set (lane-strided atom and pair sums, butterflies).
template <int kGrid>
static __device__ VS_PHASE float polish_phase(const PocketDev& pk, const Dims d, int N, int lane,
                                              PoseF* P, int* n_iter) {
  const WarpSmem s = dock_smem(d);
  for (int i = lane; i < N; i += 32) {
    const double4 v = s.ys[i];
    s.ysf[i] = make_float4(static_cast<float>(v.x), static_cast<float>(v.y),
                           static_cast<float>(v.z), 0.0f);
  }
  __syncwarp();
  const KeyAtoms ka = pairs_of(s.ysf, d.nmax);
  if (kGrid) build_pairs(ka, N, lane);
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
  *n_iter += rigid_compass<kGrid, VS_TEX_POLISH>(pk, ka, N, cx, cy, cz, P, lane);
  const float qw = P->q[0], qx = P->q[1], qy = P->q[2], qz = P->q[3];
  const float tx = P->t[0], ty = P->t[1], tz = P->t[2];
  __syncwarp();
  if (lane == 0) {
    const Mat3d RD = det_pose_mat_d(qw, qx, qy, qz);
    double* pm = s.pose;
    pm[0] = RD.m00; pm[1] = RD.m01; pm[2] = RD.m02;
    pm[3] = RD.m10; pm[4] = RD.m11; pm[5] = RD.m12;
    pm[6] = RD.m20; pm[7] = RD.m21; pm[8] = RD.m22;
    pm[9] = tx; pm[10] = ty; pm[11] = tz;
  }
  __syncwarp();
  float fb = 0.0f, wb = 0.0f, pb = 0.0f;
  for (int i = lane; i < N; i += 32) {
    const double4 v = s.ys[i];
    float fi, wi;
    atom_terms_s<kGrid>(pk, s.pose, v.x, v.y, v.z, &fi, &wi);
    fb = fb + fi;
    wb = wb + wi;
  }
  {
    int i = 0, k = lane + 1;
    while (i < N - 1 && k >= N) {
      k = k - N + i + 2;
      ++i;
    }
    int nact = 0;
    while (i < N - 1) {
      const double4 yi = s.ys[i], yk = s.ys[k];
      pb = pb + pair_term_d(pk, yi.x - yk.x, yi.y - yk.y, yi.z - yk.z, nact);
      k += 32;
      while (i < N - 1 && k >= N) {
        k = k - N + i + 2;
        ++i;
      }
    }
  }
  fb = warp_sum(fb);
  wb = warp_sum(wb);
  pb = warp_sum(pb);
  return fb - pk.lam * (pb + wb);
}

// ---- final coordinates, diversity against kept (dock.cpp:359-361), store
static __device__ VS_PHASE bool keep_phase(const Dims d, int N, int T, const PoseF* P,
                                               float S, int r, int att, int best_k, float4* kx,
                                               int kstride, float* kp, int parw, int* km, int nk,
                                               float delta, int lane) {
  const WarpSmem s = dock_smem(d);
  pose_coop(s, N, det_pose_mat_d(P->q[0], P->q[1], P->q[2], P->q[3]), P->t[0], P->t[1], P->t[2],
            lane);
  const bool keep = nk == 0 || diverse_from_kept(s, kx, nk, kstride, N, delta, lane);
  if (keep) {
    for (int i = lane; i < N; i += 32) kx[static_cast<size_t>(nk) * kstride + i] = s.xf[i];
    float* Q = kp + static_cast<size_t>(nk) * parw;
    if (lane == 0) {
      for (int c = 0; c < 3; ++c) Q[c] = P->t[c];
      for (int c = 0; c < 4; ++c) Q[3 + c] = P->q[c];
      Q[7] = S;
      km[nk * 4 + 0] = r;
      km[nk * 4 + 1] = att;
      km[nk * 4 + 2] = best_k;
      if (s.kscore) s.kscore[nk] = S;
    }
    for (int jj = lane; jj < T; jj += 32) Q[8 + jj] = s.theta[jj];
  }
  __syncwarp();
  return keep;
}

__device__ __forceinline__ PoseOut pose_out(const float* Q, const int* kmk, float resc) {
  PoseOut o;
  o.t[0] = Q[0]; o.t[1] = Q[1]; o.t[2] = Q[2];
  o.q[0] = Q[3]; o.q[1] = Q[4]; o.q[2] = Q[5]; o.q[3] = Q[6];
  o.score = Q[7];
  o.rescore = resc;
  o.restart = static_cast<int16_t>(kmk[0]);
  o.attempt = static_cast<int16_t>(kmk[1]);
  o.rot = static_cast<int16_t>(kmk[2]);
  o.pad = 0;
  return o;
}

// ---- stable sort by score desc (dock.cpp:364-366), keep-top filter
// (dock.cpp:373-390), rescore (dock.cpp:297-316), best (pipeline.cpp:508)
template <int kGrid>
static __device__ VS_PHASE void finish_phase(const PocketDev& pk, const Dims d,
                                                 const DockParams& prm, const DockOut& out,
                                                 int lig, int4 meta, int nk, const float4* kx,
                                                 int kstride, const float* kp, int parw,
                                                 const int* km, unsigned id_rank, int lane,
                                                 const unsigned long long* st) {
  const WarpSmem s = dock_smem(d);
  const int N = meta.y, T = meta.w, R = prm.R;
  const int a_lane = lane & 15, h = lane >> 4;
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
      const float* Q = kp + static_cast<size_t>(k) * parw;
      out.all[static_cast<size_t>(lig) * R + rank] = pose_out(Q, km + k * 4, 0.0f);
      float* tt = out.all_tors + static_cast<size_t>(meta.z) * R + static_cast<size_t>(rank) * T;
      for (int jj = 0; jj < T; ++jj) tt[jj] = Q[8 + jj];
    }
    __syncwarp();
  }
  for (int base = 0; base < n_surv; base += 16) {
    const int p = base + a_lane;
    float B = 0.0f;
    if (p < n_surv) {
      const float4* X = kx + static_cast<size_t>(s.kinv[p]) * kstride;
      for (int i = h; i < N; i += 2) {
        const float4 v = X[i];
        B = B + atom_bonus<kGrid>(pk, static_cast<int>(s.y0[i].w), v.x, v.y, v.z);
      }
    }
    const float B2 = __shfl_xor_sync(kFull, B, 16);
    if (p < n_surv && h == 0) {
      const int k = s.kinv[p];
      const float* Q = kp + static_cast<size_t>(k) * parw;
      const float resc = Q[7] + (B + B2);
      s.kresc[p] = resc;
      out.surv[static_cast<size_t>(lig) * prm.keep_top + p] = pose_out(Q, km + k * 4, resc);
      float* tt = out.surv_tors + static_cast<size_t>(meta.z) * prm.keep_top +
                  static_cast<size_t>(p) * T;
      for (int jj = 0; jj < T; ++jj) tt[jj] = Q[8 + jj];
      if (prm.write_all) out.all[static_cast<size_t>(lig) * R + p].rescore = resc;
    }
  }
  __syncwarp();
  if (lane == 0) {
    float bmax = -INFINITY;
    for (int p = 0; p < n_surv; ++p) bmax = p == 0 ? s.kresc[p] : fmaxf(bmax, s.kresc[p]);
    out.best[lig] = bmax;
    out.n_kept[lig] = nk;
    out.n_surv[lig] = n_surv;
    out.keys[lig] = n_surv > 0 ? ((static_cast<unsigned long long>(~det_orderable(bmax)) << 32) |
                                  id_rank)
                               : ~0ull;
    if (out.stats) {
      atomicAdd(out.stats + 0, st[0]);
      atomicAdd(out.stats + 1, st[0] * static_cast<unsigned long long>(N));
      atomicAdd(out.stats + 2, st[1]);
      atomicAdd(out.stats + 3, st[2]);
      atomicAdd(out.stats + 8, st[3]);
      atomicAdd(out.stats + 9, st[3] * static_cast<unsigned long long>(N));
    }
  }
  __syncwarp();
}

// ===================================================== staged dock kernels
// One kernel per phase and restart, the per-ligand state handed over in HBM
// (StageBufs): each phase runs at its own occupancy and instruction footprint
// (the sweep needs ~40 registers and 1 KB of shared memory per warp; the flex
// needs 64 and ~5 KB), and an SM only ever holds one phase's code.  Launch
// order per restart r: start(r) -> sweep -> flex -> polish + keep(r); then
// finish.

__device__ __forceinline__ int next_item(int* counter, int lane) {
  int w = 0;
  if (lane == 0) w = atomicAdd(counter, 1);
  return __shfl_sync(kFull, w, 0);
}

// one TMA bulk copy of `bytes` (multiple of 16, 16 B aligned) into smem
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint32_t& phase, int lane) {
  __syncwarp();
  if (lane == 0) {
    fence_proxy_async();
    mbar_expect_tx(bar, bytes);
    bulk_g2s(dst, src, bytes, bar);
  }
  mbar_wait(bar, phase);
  phase ^= 1u;
}

#ifndef VS_MINB_START
#define VS_MINB_START 8
#endif
#ifndef VS_MINB_SWEEP
#define VS_MINB_SWEEP 8
#endif
#ifndef VS_MINB_POLISH
#define VS_MINB_POLISH 7  // 72 registers (4/5/6/8/10: slower, profiles/e2e_pipeline_r2.txt)
#endif
// the polish for ligands above kPolishSmallAtoms atoms (C4-size): fewer
// blocks, more registers
#ifndef VS_MINB_POLISH_BIG
#define VS_MINB_POLISH_BIG 6
#endif
constexpr int kPolishSmallAtoms = 48;
#ifndef VS_MINB_FLEX_BIG
#define VS_MINB_FLEX_BIG 6  // C4: 117.5 ms vs 119.3 at 8, 118.9 at 5, 125.4 at 4
#endif
#ifndef VS_MINB_FLEX
#define VS_MINB_FLEX 8
#endif

template <int kGrid>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, VS_MINB_START)
    vs_start_kernel(const __grid_constant__ LibDev lib, const __grid_constant__ PocketDev pk,
                    const __grid_constant__ DockParams prm,
                    const int* __restrict__ order, int n_order, int* __restrict__ counter,
                    int nmax, int tmax, int mvmax, int r, const __grid_constant__ StageBufs sb) {
  const Dims d{nmax, tmax, mvmax, kLayLig | kLayState | kLayPosed};
  const WarpSmem s = dock_smem(d);
  const int lane = threadIdx.x & 31;
  if (lane == 0) mbar_init(s.bar);
  __syncwarp();
  uint32_t phase = 0;
  for (int w = next_item(counter, lane); w < n_order; w = next_item(counter, lane)) {
    const int lig = order[w];
    int4 meta;
    stage_ligand(lib, lig, s, lane, phase, meta);
    const int N = meta.y, T = meta.w, R = prm.R;
    const long long c0 = clock64();
    const unsigned long long root = rng_mix(lib.seeds[lig] ^ kGolden);
    const unsigned long long rkey =
        rng_mix(root ^ rng_mix(static_cast<unsigned long long>(r) + kGolden));
    const int nk = r == 0 ? 0 : sb.nk[lig];
    const float4* kx = sb.kx + static_cast<size_t>(meta.x) * R;
    PoseF P;
    const int att = start_phase(pk, d, rkey, N, T, kx, N, nk, prm.delta, lane, &P);
    // start_phase leaves the FP32 copy in ysf; this layout has none, so the
    // FP32 state is written from ys here (same conversion)
    for (int i = lane; i < N; i += 32) {
      const double4 v = s.ys[i];
      sb.ys[meta.x + i] = v;
      sb.ysf[meta.x + i] = make_float4(static_cast<float>(v.x), static_cast<float>(v.y),
                                       static_cast<float>(v.z), 0.0f);
    }
    for (int j = lane; j < T; j += 32) sb.th[meta.z + j] = s.theta[j];
    if (lane == 0) {
      sb.pose[2 * lig] = make_float4(P.t[0], P.t[1], P.t[2], __int_as_float(att));
      sb.pose[2 * lig + 1] = make_float4(P.q[0], P.q[1], P.q[2], P.q[3]);
      if (r == 0) {
        sb.nk[lig] = 0;
        for (int c = 0; c < 8; ++c) sb.st[8 * lig + c] = 0ull;
      }
      atomicAdd(sb.st + 8 * lig + 1, static_cast<unsigned long long>(att) + 1);
      atomicAdd(sb.st + 8 * lig + 4, static_cast<unsigned long long>(clock64() - c0));
    }
    __syncwarp();
  }
}

template <int kGrid>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, VS_MINB_SWEEP)
    vs_sweep_kernel(const __grid_constant__ LibDev lib, const __grid_constant__ PocketDev pk,
                    const float4* __restrict__ rots, const float4* __restrict__ rots_p,
                    const int* __restrict__ perm, const __grid_constant__ DockParams prm, const int* __restrict__ order,
                    int n_order, int* __restrict__ counter, int nmax,
                    const __grid_constant__ StageBufs sb) {
  const Dims d{nmax, 0, 0, kLaySweep | kLayPairs};
  const WarpSmem s = dock_smem(d);
  const int lane = threadIdx.x & 31;
  if (lane == 0) mbar_init(s.bar);
  __syncwarp();
  uint32_t phase = 0;
  for (int w = next_item(counter, lane); w < n_order; w = next_item(counter, lane)) {
    const int lig = order[w];
    const int4 meta = lib.meta[lig];
    const int N = meta.y;
    // the pose loads issue before the bulk copy's wait (they do not depend on it)
    const float4 pt = sb.pose[2 * lig], pq = sb.pose[2 * lig + 1];
    tma_load(s.ysf, sb.ysf + meta.x, 16u * N, s.bar, phase, lane);
    if (kGrid) build_pairs(pairs_of(s.ysf, d.nmax), N, lane);
    const long long c0 = clock64();
    PoseF P;
    P.t[0] = pt.x;
    P.t[1] = pt.y;
    P.t[2] = pt.z;
    P.q[0] = pq.x;
    P.q[1] = pq.y;
    P.q[2] = pq.z;
    P.q[3] = pq.w;
    int n_trans = 0;
    const int best_k = sweep_phase<kGrid>(pk, d, rots, rots_p, perm, prm.K, N, lane, &P, &n_trans,
                                                prm.polish);
    if (lane == 0) {
      sb.pose[2 * lig] = make_float4(P.t[0], P.t[1], P.t[2], pt.w);
      sb.pose[2 * lig + 1] = make_float4(P.q[0], P.q[1], P.q[2], P.q[3]);
      sb.bk[lig] = best_k;
      atomicAdd(sb.st + 8 * lig + 0, static_cast<unsigned long long>(n_trans));
      atomicAdd(sb.st + 8 * lig + 5, static_cast<unsigned long long>(clock64() - c0));
    }
    __syncwarp();
  }
}

template <int kGrid, int kMinB>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, kMinB)
    vs_flex_kernel(const __grid_constant__ LibDev lib, const __grid_constant__ PocketDev pk,
                   const __grid_constant__ DockParams prm,
                   const int* __restrict__ order, int n_order, int* __restrict__ counter,
                   int nmax, int tmax, int mvmax, int r, const __grid_constant__ StageBufs sb) {
  const Dims d{nmax, tmax, mvmax,
               kLayLig | kLayState | kLayPosed | kLayFlex | kLaySweep | kLayAliasY0};
  const WarpSmem s = dock_smem(d);
  const int lane = threadIdx.x & 31;
  // the search pair-softplus table (polish >= 1) behind the warps' regions
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* tab = reinterpret_cast<float2*>(
      smem_raw + kWarpsPerBlock * warp_smem_bytes(d.nmax, d.tmax, d.mvmax, d.lay));
  if (prm.polish >= 1) {
    for (int k = threadIdx.x; k < kSoftN; k += blockDim.x) tab[k] = pk.soft_tab[k];
    __syncthreads();
  }
  if (lane == 0) mbar_init(s.bar);
  __syncwarp();
  uint32_t phase = 0;
  const float step = kTwoPiF / static_cast<float>(prm.A);
  for (int w = next_item(counter, lane); w < n_order; w = next_item(counter, lane)) {
    const int lig = order[w];
    int4 meta;
    const float4 pt = sb.pose[2 * lig], pq = sb.pose[2 * lig + 1];  // before the copies' waits
    stage_ligand(lib, lig, s, lane, phase, meta);
    const int N = meta.y, T = meta.w, R = prm.R;
    for (int j = lane; j < T; j += 32) s.theta[j] = sb.th[meta.z + j];
    tma_load(s.ys, sb.ys + meta.x, 32u * N, s.bar, phase, lane);
    const long long c0 = clock64();
    PoseF P;
    P.t[0] = pt.x;
    P.t[1] = pt.y;
    P.t[2] = pt.z;
    P.q[0] = pq.x;
    P.q[1] = pq.y;
    P.q[2] = pq.z;
    P.q[3] = pq.w;
    __syncwarp();
    unsigned long long nact = 0;
    float S = prm.polish >= 1
                  ? flex_phase<kGrid, true, true>(pk, d, N, T, prm.F, prm.A, step, &P, lane,
                                                  &nact, prm.polish, tab)
                  : flex_phase<kGrid, true, false>(pk, d, N, T, prm.F, prm.A, step, &P, lane,
                                                   &nact, prm.polish);
    if (prm.polish >= 1) {
      // the polish + keep run in vs_polish_kernel: hand over the flexed state
      for (int i = lane; i < N; i += 32) sb.ys[meta.x + i] = s.ys[i];
      for (int j = lane; j < T; j += 32) sb.th[meta.z + j] = s.theta[j];
      if (lane == 0) {
        atomicAdd(sb.st + 8 * lig + 2, nact);
        atomicAdd(sb.st + 8 * lig + 6, static_cast<unsigned long long>(clock64() - c0));
      }
      __syncwarp();
      continue;
    }
    const long long c1 = clock64();
    const int nk = sb.nk[lig];
    float4* kx = sb.kx + static_cast<size_t>(meta.x) * R;
    float* kp = sb.kp + (static_cast<size_t>(lig) * 8 + meta.z) * R;
    int* km = sb.km + static_cast<size_t>(lig) * R * 4;
    const bool kept = keep_phase(d, N, T, &P, S, r, __float_as_int(pt.w), sb.bk[lig], kx, N, kp,
                                 8 + T, km, nk, prm.delta, lane);
    if (lane == 0) {
      if (kept) sb.nk[lig] = nk + 1;
      atomicAdd(sb.st + 8 * lig + 2, nact);
      atomicAdd(sb.st + 8 * lig + 6, static_cast<unsigned long long>(c1 - c0));
      atomicAdd(sb.st + 8 * lig + 7, static_cast<unsigned long long>(clock64() - c1));
    }
    __syncwarp();
  }
}

// polish (SWEEP_V1.md §3.5) + keep of restart r on the flexed state: the
// compass runs here rather than in the flex kernel so it gets this kernel's
// small shared-memory footprint (no conformer / topology) and a large L1 for
// its key-map lookups.
template <int kGrid, int kMinB>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, kMinB)
    vs_polish_kernel(const __grid_constant__ LibDev lib, const __grid_constant__ PocketDev pk,
                     const __grid_constant__ DockParams prm,
                     const int* __restrict__ order, int n_order, int* __restrict__ counter,
                     int nmax, int tmax, int r, const __grid_constant__ StageBufs sb) {
  const Dims d{nmax, tmax, 0, kLayState | kLayPosed | kLayFlex | kLaySweep | kLayPairs};
  const WarpSmem s = dock_smem(d);
  const int lane = threadIdx.x & 31;
  if (lane == 0) mbar_init(s.bar);
  __syncwarp();
  uint32_t phase = 0;
  for (int w = next_item(counter, lane); w < n_order; w = next_item(counter, lane)) {
    const int lig = order[w];
    const int4 meta = lib.meta[lig];
    const int N = meta.y, T = meta.w, R = prm.R;
    // loads that do not depend on the bulk copy issue before its wait
    const float4 pt = sb.pose[2 * lig], pq = sb.pose[2 * lig + 1];
    const int nk = sb.nk[lig], bk = sb.bk[lig];
    for (int j = lane; j < T; j += 32) s.theta[j] = sb.th[meta.z + j];
    tma_load(s.ys, sb.ys + meta.x, 32u * N, s.bar, phase, lane);
    const long long c0 = clock64();
    PoseF P;
    P.t[0] = pt.x;
    P.t[1] = pt.y;
    P.t[2] = pt.z;
    P.q[0] = pq.x;
    P.q[1] = pq.y;
    P.q[2] = pq.z;
    P.q[3] = pq.w;
    __syncwarp();
    int n_post = 0;
    const float S = polish_phase<kGrid>(pk, d, N, lane, &P, &n_post);
    const long long c1 = clock64();
    float4* kx = sb.kx + static_cast<size_t>(meta.x) * R;
    float* kp = sb.kp + (static_cast<size_t>(lig) * 8 + meta.z) * R;
    int* km = sb.km + static_cast<size_t>(lig) * R * 4;
    const bool kept = keep_phase(d, N, T, &P, S, r, __float_as_int(pt.w), bk, kx, N, kp,
                                 8 + T, km, nk, prm.delta, lane);
    if (lane == 0) {
      if (kept) sb.nk[lig] = nk + 1;
      atomicAdd(sb.st + 8 * lig + 3, static_cast<unsigned long long>(n_post));
      atomicAdd(sb.st + 8 * lig + 6, static_cast<unsigned long long>(c1 - c0));
      atomicAdd(sb.st + 8 * lig + 7, static_cast<unsigned long long>(clock64() - c1));
    }
    __syncwarp();
  }
}

template <int kGrid>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 8)
    vs_finish_kernel(const __grid_constant__ LibDev lib, const __grid_constant__ PocketDev pk,
                     const __grid_constant__ DockParams prm,
                     const int* __restrict__ order, int n_order, int* __restrict__ counter,
                     int nmax, int tmax, int mvmax, const __grid_constant__ StageBufs sb,
                     const __grid_constant__ DockOut out) {
  const Dims d{nmax, tmax, mvmax, kLayLig | kLayKept};
  const WarpSmem s = dock_smem(d);
  const int lane = threadIdx.x & 31;
  if (lane == 0) mbar_init(s.bar);
  __syncwarp();
  uint32_t phase = 0;
  for (int w = next_item(counter, lane); w < n_order; w = next_item(counter, lane)) {
    const int lig = order[w];
    int4 meta;
    stage_ligand(lib, lig, s, lane, phase, meta);
    const int T = meta.w, R = prm.R;
    const int nk = sb.nk[lig];
    const float* kp = sb.kp + (static_cast<size_t>(lig) * 8 + meta.z) * R;
    for (int k = lane; k < nk; k += 32) s.kscore[k] = kp[static_cast<size_t>(k) * (8 + T) + 7];
    __syncwarp();
    const unsigned long long* st = sb.st + 8 * lig;
    finish_phase<kGrid>(pk, d, prm, out, lig, meta, nk, sb.kx + static_cast<size_t>(meta.x) * R,
                        meta.y, kp, 8 + T, sb.km + static_cast<size_t>(lig) * R * 4,
                        lib.id_rank[lig], lane, st);
    if (lane == 0 && out.stats)
      for (int c = 4; c < 8; ++c) atomicAdd(out.stats + c, st[c]);
  }
}

template <class K>
static void prep_dock(K kernel, size_t smem) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
}

// ---------------------------------------------------------- staged launch
template <class K>
static int stage_blocks(K kernel, size_t smem, int sms, int n_items, int target_per_sm) {
  prep_dock(kernel, smem);
  // shared-memory carveout just large enough for target_per_sm blocks: the
  // rest of the 256 KB stays L1 for the grid-cell gathers (the sweep kernel
  // needs ~32 KB of shared memory per SM and reuses cells across the
  // translation lattice); VSCREEN_CARVEOUT_MAXSHARED=1 restores max shared
  const char* ms = std::getenv("VSCREEN_CARVEOUT_MAXSHARED");
  if (!(ms && ms[0] == '1')) {
    const size_t need = static_cast<size_t>(target_per_sm) * (smem + 1024);
    int pct = static_cast<int>((need * 100 + 228 * 1024 - 1) / (228 * 1024)) + 1;
    pct = pct > 100 ? 100 : pct;
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kWarpsPerBlock * 32, smem);
  if (per_sm < 1) per_sm = 1;
  const int want = (n_items + kWarpsPerBlock - 1) / kWarpsPerBlock;
  return want < per_sm * sms ? (want > 0 ? want : 1) : per_sm * sms;
}

size_t stage_smem_per_block(int nmax, int tmax, int mvmax) {
  const int lays[5] = {kLayLig | kLayState | kLayPosed, kLaySweep | kLayPairs,
                       kLayLig | kLayState | kLayPosed | kLayFlex | kLaySweep | kLayAliasY0,
                       kLayState | kLayPosed | kLayFlex | kLaySweep | kLayPairs,  // polish
                       kLayLig | kLayKept};
  size_t m = 0;
  for (int l : lays) {
    const size_t b = kWarpsPerBlock * warp_smem_bytes(nmax, tmax, mvmax, l) +
                     ((l & kLayAliasY0) ? sizeof(float2) * kSoftN : 0);  // flex: softplus table
    m = b > m ? b : m;
  }
  return m;
}

template <int kGrid>
static cudaError_t staged_impl(int sms, cudaStream_t st, const LibDev& lib, const PocketDev& pk,
                               const float4* rots, const float4* rots_p, const int* perm,
                               const DockParams& prm,
                               const int* order, int n, int* counters, int nmax, int tmax,
                               int mvmax, const StageBufs& sb, const DockOut& out,
                               uint64_t* launches, cudaEvent_t* evs, int* kinds) {
  const size_t sm_start = kWarpsPerBlock * warp_smem_bytes(nmax, tmax, mvmax,
                                                           kLayLig | kLayState | kLayPosed);
  const size_t sm_sweep = kWarpsPerBlock * warp_smem_bytes(nmax, 0, 0, kLaySweep | kLayPairs);
  const size_t sm_flex = kWarpsPerBlock * warp_smem_bytes(
                                              nmax, tmax, mvmax,
                                              kLayLig | kLayState | kLayPosed | kLayFlex |
                                                  kLaySweep | kLayAliasY0) +
                         sizeof(float2) * kSoftN;  // search pair-softplus table
  const size_t sm_fin = kWarpsPerBlock * warp_smem_bytes(nmax, tmax, mvmax, kLayLig | kLayKept);
  const int b_start = stage_blocks(vs_start_kernel<kGrid>, sm_start, sms, n, VS_MINB_START);
  const int b_sweep = stage_blocks(vs_sweep_kernel<kGrid>, sm_sweep, sms, n, VS_MINB_SWEEP);
  const bool small = nmax <= kPolishSmallAtoms;
  const int b_flex = small ? stage_blocks(vs_flex_kernel<kGrid, VS_MINB_FLEX>, sm_flex, sms, n,
                                          VS_MINB_FLEX)
                           : stage_blocks(vs_flex_kernel<kGrid, VS_MINB_FLEX_BIG>, sm_flex, sms,
                                          n, VS_MINB_FLEX_BIG);
  const int b_fin = stage_blocks(vs_finish_kernel<kGrid>, sm_fin, sms, n, 8);
  const size_t sm_pol = kWarpsPerBlock * warp_smem_bytes(nmax, tmax, 0,
                                                         kLayState | kLayPosed | kLayFlex |
                                                             kLaySweep | kLayPairs);
  const bool pol_small = small;
  const int b_pol = pol_small
                        ? stage_blocks(vs_polish_kernel<kGrid, VS_MINB_POLISH>, sm_pol, sms, n,
                                       VS_MINB_POLISH)
                        : stage_blocks(vs_polish_kernel<kGrid, VS_MINB_POLISH_BIG>, sm_pol, sms, n,
                                       VS_MINB_POLISH_BIG);
  const int T = kWarpsPerBlock * 32;
  int c = 0;
  auto mark = [&](int kind, bool after) {  // event pair c: launch c (counter c)
    if (!evs) return;
    cudaEventRecord(evs[2 * c + (after ? 1 : 0)], st);
    kinds[c] = kind;
  };
  for (int r = 0; r < prm.R; ++r) {
    mark(0, false);
    vs_start_kernel<kGrid><<<b_start, T, sm_start, st>>>(lib, pk, prm, order, n, counters + c,
                                                        nmax, tmax, mvmax, r, sb);
    mark(0, true);
    ++c;
    mark(1, false);
    vs_sweep_kernel<kGrid><<<b_sweep, T, sm_sweep, st>>>(lib, pk, rots, rots_p, perm, prm, order, n,
                                                        counters + c, nmax, sb);
    mark(1, true);
    ++c;
    mark(2, false);
    if (small)
      vs_flex_kernel<kGrid, VS_MINB_FLEX><<<b_flex, T, sm_flex, st>>>(lib, pk, prm, order, n, counters + c, nmax,
                                                     tmax, mvmax, r, sb);
    else
      vs_flex_kernel<kGrid, VS_MINB_FLEX_BIG><<<b_flex, T, sm_flex, st>>>(lib, pk, prm, order, n, counters + c, nmax,
                                                     tmax, mvmax, r, sb);
    mark(2, true);
    ++c;
    *launches += 3;
    if (prm.polish >= 1) {
      mark(4, false);
      if (pol_small)
        vs_polish_kernel<kGrid, VS_MINB_POLISH><<<b_pol, T, sm_pol, st>>>(
            lib, pk, prm, order, n, counters + c, nmax, tmax, r, sb);
      else
        vs_polish_kernel<kGrid, VS_MINB_POLISH_BIG><<<b_pol, T, sm_pol, st>>>(
            lib, pk, prm, order, n, counters + c, nmax, tmax, r, sb);
      mark(4, true);
      ++c;
      *launches += 1;
    }
  }
  mark(3, false);
  vs_finish_kernel<kGrid><<<b_fin, T, sm_fin, st>>>(lib, pk, prm, order, n, counters + c, nmax,
                                                   tmax, mvmax, sb, out);
  mark(3, true);
  *launches += 1;
  return cudaGetLastError();
}

// ---- restart start draws (dock.cpp:343-354) of given (ligand, restart,
// attempt) triples, for the parity test against the reference Rng: one warp
// per triple, the same draw_start the start kernel runs.  Row i of `out`
// (stride floats): t[3], q[4] (w, x, y, z), theta[T].
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
    vs_draws_kernel(const __grid_constant__ PocketDev pk, const unsigned long long* __restrict__ seeds,
                    const int* __restrict__ n_tors, int n, int restarts, int attempts,
                    float* __restrict__ out, int stride) {
  __shared__ float theta[kWarpsPerBlock][kMaxTors];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const long total = static_cast<long>(n) * restarts * attempts;
  for (long w = static_cast<long>(blockIdx.x) * kWarpsPerBlock + wib; w < total;
       w += static_cast<long>(gridDim.x) * kWarpsPerBlock) {
    const int att = static_cast<int>(w % attempts);
    const int r = static_cast<int>((w / attempts) % restarts);
    const int lig = static_cast<int>(w / (static_cast<long>(attempts) * restarts));
    const int T = n_tors[lig];
    const unsigned long long root = rng_mix(seeds[lig] ^ kGolden);
    const unsigned long long rkey =
        rng_mix(root ^ rng_mix(static_cast<unsigned long long>(r) + kGolden));
    WarpSmem s{};
    s.theta = theta[wib];
    float t[3], q[4];
    draw_start(pk, rkey, att, T, s, lane, t, q);
    float* o = out + w * stride;
    if (lane == 0) {
      for (int c = 0; c < 3; ++c) o[c] = t[c];
      for (int c = 0; c < 4; ++c) o[3 + c] = q[c];
    }
    for (int j = lane; j < T; j += 32) o[7 + j] = s.theta[j];
    __syncwarp();
  }
}

cudaError_t launch_draws(cudaStream_t st, const PocketDev& pk, const unsigned long long* seeds,
                         const int* n_tors, int n, int restarts, int attempts, float* out,
                         int stride, int sms) {
  vs_draws_kernel<<<sms * 8, kWarpsPerBlock * 32, 0, st>>>(pk, seeds, n_tors, n, restarts,
                                                           attempts, out, stride);
  return cudaGetLastError();
}

// rots: the K rotations in index order; perm: the sweep's lane order (a
// permutation of 0..K-1, see sweep_phase); rots_p[p] = rots[perm[p]]
cudaError_t launch_staged(bool grid, int sms, cudaStream_t st, const LibDev& lib,
                          const PocketDev& pk, const float4* rots, const float4* rots_p,
                          const int* perm,
                          const DockParams& prm, const int* order, int n, int* counters,
                          int nmax, int tmax, int mvmax, const StageBufs& sb, const DockOut& out,
                          uint64_t* launches, cudaEvent_t* evs, int* kinds) {
  return grid ? staged_impl<1>(sms, st, lib, pk, rots, rots_p, perm, prm, order, n, counters, nmax, tmax,
                               mvmax, sb, out, launches, evs, kinds)
              : staged_impl<0>(sms, st, lib, pk, rots, rots_p, perm, prm, order, n, counters, nmax, tmax,
                               mvmax, sb, out, launches, evs, kinds);
}

}  // namespace vs
