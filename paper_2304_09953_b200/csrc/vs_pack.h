// Device ligand packer (vs_pack.cu) <-> runtime (vs_runtime.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "vs_types.h"

namespace vs {

// validation outcome codes (the host packer's status for each)
enum : int { kPkNoAtoms = 1, kPkCapacity = 2, kPkNegTors = 3, kPkTopology = 4, kPkNotTree = 5 };

// the stats buffer (ints): [0..3] in-class nmax, tmax, mvmax, count;
// [4 + 3c ..] per-class nmax, tmax, mvmax (c < kPkMaxClasses); the error key
// (u64) at kPkErr; the size classes (int4) from kPkClasses on
constexpr int kPkMaxClasses = 64;
constexpr int kPkErr = 4 + 3 * kPkMaxClasses;  // 196: 8-byte aligned
constexpr int kPkClasses = kPkErr + 4;         // 200: 16-byte aligned

// the caller's library arrays on the device (capi.h vs_library, as given)
struct PackIn {
  int n = 0;
  long total_atoms = 0, total_tors = 0, total_moving = 0;
  const int* n_atoms = nullptr;
  const int* n_tors = nullptr;
  const int* rot_bonds = nullptr;  // may be null: = n_tors
  const double* coords = nullptr;
  const int* atom_class = nullptr;
  const int* axis_a = nullptr;
  const int* axis_b = nullptr;
  const int* moving_count = nullptr;
  const int* moving = nullptr;
  const unsigned long long* seeds = nullptr;
  const unsigned* id_rank = nullptr;
  const int4* classes = nullptr;  // n_classes size classes (atom_lo, atom_hi, rot_lo, rot_hi)
};

// scratch: counts, their exclusive scans (n + 1 / T + 1 entries), sort keys
struct PackWork {
  long *cnt_a, *cnt_t, *cnt_m, *cnt_p;
  long *aoff, *toff, *msrc, *moff;
  int* cls;
  unsigned *key, *key_sorted;
  int* idx;
  int* stats;  // see kPkErr / kPkClasses
  unsigned long long* err;
};

// the packed layout (LibDev's arrays) + launch order
struct PackDev {
  int4* meta;
  int2* mov;
  double4* atoms;
  int4* axes;
  uint8_t* moving;
  unsigned long long* seeds;
  unsigned* id_rank;
  int* order;  // n entries: in-class ligands first, by descending cost
};

size_t pack_temp_bytes(int n, long total_tors);
// pass 1 (counts, classes, the count checks); the caller reads w.err before stage 2
cudaError_t pack_stage1(cudaStream_t st, const PackIn& in, const PackWork& w, int n_classes);
// scans, layout, topology checks, LPT order
cudaError_t pack_stage2(cudaStream_t st, const PackIn& in, const PackWork& w, const PackDev& out,
                        void* temp, size_t temp_bytes);

}  // namespace vs
