// Device-side data layout of the dock-and-score path.
// Plain structs shared by the kernels (vs_kernels.cu) and the host runtime
// (vs_runtime.cpp).  Nothing here crosses the public C-ABI.
#pragma once
#include <stdint.h>

namespace vs {

constexpr int kMaxRestarts = 64;   // kept-pose bookkeeping in shared memory
constexpr int kMaxFlexAngles = 16; // one lane pair per candidate angle
constexpr int kMaxAtoms = 128;     // moving lists are u8 atom indices
constexpr int kMaxTors = 64;
constexpr int kWarpsPerBlock = 4;

// One analytic Gaussian site (dock.hpp:18-23) in FP32.
struct SiteF {
  float cx, cy, cz, w;
  float inv2s2;  // 1 / (2 sigma^2), computed in FP64 then rounded
  float pad[3];
};

// FP64 site for score_gradient (vs_grad.cu): pocket order, kind kept
struct SiteD {
  double cx, cy, cz, w, inv2s2;
  int kind, pad;
};

struct GridDev {
  float ox, oy, oz;  // node (0,0,0) position
  float h, inv_h;
  int nx, ny, nz;
  int cx, cxy;          // cell strides: nx - 1, (nx - 1)(ny - 1)
  const float* steric;  // node values, x fastest
  const float* hbond;
  const float* lipo;
  // corner-packed cells: 8 node values per cell (2 x float4, one 32 B
  // sector), cells x fastest over (nx-1)(ny-1)(nz-1); one sector per lookup
  const float4* steric_c;
  const float4* hbond_c;
  const float4* lipo_c;
  // sweep-key map K = steric - lam * wall at the nodes (SWEEP_V1.md §2.3)
  const float* key;
  const float4* key_c;
  const uint4* key_h;  // FP16 corner cells of the key map (8 halves, 16 B), the sweep's map
  unsigned long long key_tex;  // the same cells as a linear uint4 texture (TEX path)
};

struct PocketDev {
  float lo[3], hi[3];       // bounds (FP32) for the wall term
  double lo_d[3], hi_d[3];  // bounds (FP64) for the RNG start draws
  float r;                  // clash_radius
  float lam;                // clash_penalty
  float cut2;               // (r + 3)^2: pair skip threshold (z < -30)
  double cut2_d;            // the same threshold widened to FP64 (pair tests compare in FP64)
  int n_steric, n_hbond, n_lipo;
  const SiteF* sites;       // [steric | hbond | lipo], pocket order within kind
  int grid_mode;            // 0 analytic field, 1 grid maps
  GridDev grid;
  // search-only pair term (flex with polish >= 1, SWEEP_V1.md §3.4): the
  // clash softplus tabulated on d^2 in [0, cut2] at kSoftN + 1 nodes,
  // entry k = (g_k, g_{k+1} - g_k); soft_inv_h = kSoftN / cut2
  const float2* soft_tab;
  float soft_inv_h;
};
constexpr int kSoftN = 512;

// Output pose record (40 B); torsions live in a parallel float array.
struct PoseOut {
  float t[3];
  float q[4];
  float score;    // geometric score (canonical FP32)
  float rescore;  // geometric + kind bonuses
  int16_t restart;
  int16_t attempt;  // start attempt that was accepted (dock.cpp:345)
  int16_t rot;      // winning rotation index of the sweep
  int16_t pad;
};

struct LibDev {
  const int4* meta;        // {atom_off, n_atoms, tors_off, n_tors}
  const int2* mov;         // {byte offset (16B aligned), padded byte count}
  const double4* atoms;    // x, y, z, class (0 other, 1 C, 2 N/O), FP64
  const int4* axes;        // {a, b, mov_start (rel. to ligand), mov_cnt}
  const uint8_t* moving;
  const unsigned long long* seeds;
  const unsigned int* id_rank;
};

struct DockParams {
  int R, K, A, F;
  int keep_top;
  int write_all;
  float delta;
  double min_score;
  int polish;  // 0 off, 1 rigid compass, 2 + fine torsion pass (SWEEP_V1.md §3.5)
};

struct DockOut {
  PoseOut* surv;        // [n][keep_top]
  float* surv_tors;     // [tors_off * keep_top + slot * T + j]
  PoseOut* all;         // [n][R] (optional)
  float* all_tors;      // [tors_off * R + slot * T + j]
  float* best;          // [n]
  int* n_kept;          // [n]
  int* n_surv;          // [n]
  unsigned long long* keys;  // [n] top-k keys (score desc, id_rank asc)
  unsigned long long* stats; // [4] work counters (capi.h vs_last_stats)
};

// Poses for the rescoring kernel (K3a).  Flat mode (t3 != nullptr): the
// poses of ligand l are p in [first[l], first[l] + count[l]) of flat arrays
// t3[3p], q4[4p] (w, x, y, z), torsions at tb[l] + (p - first[l]) * T,
// results at geo[p] / resc[p].  Survivor mode (t3 == nullptr): the last
// dock's survivors of ligand l, surv[l * keep_top + k] for k < n_surv[l],
// torsions at surv_tors + tors_off(l) * keep_top + k * T, results at
// geo[l * keep_top + k].
struct PoseSrc {
  const int* first;
  const int* count;
  const long* tb;
  const float* t3;
  const float* q4;
  const float* tors;
  const PoseOut* surv;
  const float* surv_tors;
  const int* n_surv;
  int keep_top;
  float* geo;
  float* resc;
};

// Per-ligand state of the staged dock (one kernel per phase and restart):
// what one phase hands to the next through HBM.
struct StageBufs {
  double4* ys;               // [total_atoms] FP64 state after start (torsions applied)
  float4* ysf;               // [total_atoms] FP32 copy for the sweep
  float* th;                 // [total_tors] state torsions
  float4* pose;              // [n][2]: (t.xyz, attempt), q
  int* bk;                   // [n] winning rotation of the sweep
  int* nk;                   // [n] kept poses so far
  float4* kx;                // kept coordinates: ligand base atom_off * R, pose k at k * N
  float* kp;                 // kept (t, q, S, theta): base (lig * 8 + tors_off) * R, 8 + T each
  int* km;                   // [n][R][4] kept (restart, attempt, rotation)
  unsigned long long* st;    // [n][8] counters (trans iters, attempts, pairs, -, cycles x4)
};

}  // namespace vs
