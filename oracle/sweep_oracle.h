/* TEST INFRASTRUCTURE — the CPU oracle of the dock-and-score path.
 *
 * A plain-C restatement of sweep-v1 (docs/SWEEP_V1.md) built on the
 * reference's own semantics (proj/src/dock.cpp, proj/include/vscreen/rng.hpp,
 * proj/src/pipeline.cpp).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it; the product never does.
 *
 * Pinning: tests/test_oracle.py checks this oracle against the compiled
 * reference (oracle/_ref/libvsref.so): RNG streams bit-exact, per-pose
 * scores within 1e-5*max(|ref|,1) of dock::geometric_score / dock::rescore,
 * grid-node values against single-atom geometric scores, filter_poses /
 * rank_ligands / BatchQueue outputs exactly, and the reference's known-answer
 * tests (test_dock.cpp:40-61, 288-323, 361-376).
 */
#ifndef VS_SWEEP_ORACLE_H
#define VS_SWEEP_ORACLE_H
#include <stdint.h>

typedef struct {
  double center[3];
  double weight;
  double sigma;
  int32_t kind; /* 0 steric, 1 hbond, 2 lipophilic */
  int32_t reserved;
} vso_site;

typedef struct {
  const vso_site* sites;
  int32_t n_sites;
  int32_t reserved;
  double lo[3], hi[3];
  double clash_radius, clash_penalty;
  double grid_spacing; /* 0: analytic field */
  double grid_pad;
} vso_pocket_desc;

typedef struct {
  int32_t restarts, rotations, flex_angles, flex_passes;
  double diversity_delta;
  int32_t keep_top, write_all;
  double min_score;
  int32_t polish, reserved; /* 0 off, 1 rigid compass, 2 + fine torsion pass (SWEEP_V1.md §3.5) */
} vso_params;

typedef struct {
  float t[3];
  float q[4];
  float score;
  float rescore;
  int16_t restart, attempt, rot, reserved;
} vso_pose;

typedef struct {
  int32_t n_ligands;
  int32_t reserved;
  const int32_t* n_atoms;
  const int32_t* n_tors;
  const double* coords;
  const int32_t* atom_class;
  const int32_t* axis_a;
  const int32_t* axis_b;
  const int32_t* moving_count;
  const int32_t* moving;
  const uint64_t* seeds;
  const uint32_t* id_rank;
} vso_library;

typedef struct {
  float* best;
  int32_t* n_kept;
  int32_t* n_surv;
  vso_pose* surv;
  float* surv_tors;
  vso_pose* all;
  float* all_tors;
  uint64_t* keys;
} vso_results;

typedef struct vso_pocket vso_pocket;

int vso_pocket_new(const vso_pocket_desc* d, vso_pocket** out);
void vso_pocket_free(vso_pocket* p);
int vso_grid_info(const vso_pocket* p, int32_t dims[3], float origin[3], float* spacing);
int vso_grid_fetch(const vso_pocket* p, float* steric, float* hbond, float* lipo);

void vso_rotation_set(int32_t K, uint64_t seed, float* out /* K x 4 (w,x,y,z) */);

/* sweep-v1 over a library; `sel` (may be NULL) restricts to the listed
 * ligand indices (outputs still indexed by ligand).  threads >= 1. */
int vso_dock_library(const vso_pocket* p, const vso_library* lib, const int32_t* sel,
                     int32_t n_sel, const vso_params* prm, const float* rots, int32_t threads,
                     vso_results* out);

/* canonical FP32 geometric score + rescore of given poses (K3a) */
int vso_score_poses(const vso_pocket* p, const vso_library* lib, int64_t n_poses,
                    const int32_t* pose_lig, const float* t, const float* q, const float* tors,
                    float* geo, float* resc);

/* deterministic primitives, exposed for unit tests */
float vso_exp_neg(float x);
float vso_log1p01(float u);
float vso_softplus(float z);
void vso_sincos(float x, float* s, float* c);

/* top-k of keys (ascending), k <= n; returns count */
int vso_topk(const uint64_t* keys, int64_t n, int32_t k, uint64_t* out);

#endif
