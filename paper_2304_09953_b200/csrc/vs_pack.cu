// North-star subsystem 1 on the device: the ligand batch packer.
//
// The caller's library arrays (capi.h vs_library: the reference's own
// Conformer / TorsionTopology data flattened) are DMA'd as
// they are — from pinned memory at full link rate — and these kernels build
// the dock's SoA layout in HBM: per-ligand meta, 32 B atom
// records (x, y, z, element class), per-torsion axes, the moving lists as
// 16 B-padded u8 segments (one TMA bulk copy each), the size class of every
// ligand (batcher.cpp:19-26, first containing class in list order), and the
// launch order: in-class ligands by descending cost (LPT, stable), so the
// persistent dock warps take the largest ligands first.  Validation follows
// the host packer's rules and precedence (vs_runtime.cu pack_library /
// check_nested): the lowest pass, then the lowest ligand, wins.
//
// Scans and the one radix sort are CUB device primitives; the gathers and
// scatters that make up the layout are the kernels below.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>

#include "vs_pack.h"

namespace vs {

namespace {

// error key: (pass << 56) | (ligand << 8) | code; atomicMin keeps the first
__device__ __forceinline__ void report(unsigned long long* err, int pass, long lig, int code) {
  const unsigned long long k = (static_cast<unsigned long long>(pass) << 56) |
                               (static_cast<unsigned long long>(lig) << 8) |
                               static_cast<unsigned long long>(code & 0xff);
  atomicMin(err, k);
}

__device__ __forceinline__ int ligand_of(const long* off, int n, long x) {
  // last i with off[i] <= x (off is non-decreasing, off[0] = 0)
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= x) lo = mid;
    else hi = mid;
  }
  return lo;
}

// pass 1: counts (clamped so every later kernel stays in bounds), classes
__global__ void pk_counts(PackIn in, PackWork w, int n_classes) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > in.n) return;
  if (i == in.n) {  // the scans' last element: offsets of the end
    w.cnt_a[i] = 0;
    w.cnt_t[i] = 0;
    return;
  }
  const int N = in.n_atoms[i], T = in.n_tors[i];
  if (N < 1) report(w.err, 1, i, kPkNoAtoms);
  else if (N > kMaxAtoms || T > kMaxTors) report(w.err, 1, i, kPkCapacity);
  else if (T < 0) report(w.err, 1, i, kPkNegTors);
  w.cnt_a[i] = N < 0 ? 0 : (N > kMaxAtoms ? kMaxAtoms : N);
  w.cnt_t[i] = T < 0 ? 0 : (T > kMaxTors ? kMaxTors : T);
  const int rot = in.rot_bonds ? in.rot_bonds[i] : T;
  int c = -1;
  if (n_classes > 0) {
    for (int k = 0; k < n_classes; ++k) {
      const int4 cl = in.classes[k];  // atom_lo, atom_hi, rot_lo, rot_hi (half-open)
      if (N >= cl.x && N < cl.y && rot >= cl.z && rot < cl.w) {
        c = k;
        break;
      }
    }
  } else {
    c = N <= 16 ? 0 : N <= 32 ? 1 : N <= 48 ? 2 : N <= 64 ? 3 : N <= 96 ? 4 : 5;
  }
  w.cls[i] = c;
}

// pass 2a: per torsion, the moving count (for the scan of raw offsets) and
// the axis atoms' range check
__global__ void pk_torsions(PackIn in, PackWork w) {
  const long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t > in.total_tors) return;
  if (t == in.total_tors) {
    w.cnt_m[t] = 0;
    return;
  }
  const int i = ligand_of(w.toff, in.n, t);
  const int N = in.n_atoms[i];
  const int a = in.axis_a[t], b = in.axis_b[t], c = in.moving_count[t];
  if (a < 0 || b < 0 || a >= N || b >= N || c < 0 || c > kMaxAtoms) report(w.err, 2, i, kPkTopology);
  w.cnt_m[t] = c < 0 ? 0 : (c > kMaxAtoms ? kMaxAtoms : c);
}

// per ligand: moving-list size (padded to 16 B), meta, cost key, maxima
__global__ void pk_ligands(PackIn in, PackWork w, PackDev out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > in.n) return;
  if (i == in.n) {
    w.cnt_p[i] = 0;
    return;
  }
  const long t0 = w.toff[i], t1 = w.toff[i + 1];
  const long mv = w.msrc[t1] - w.msrc[t0];
  w.cnt_p[i] = static_cast<int>((mv + 15) & ~15L);
  const int N = w.cnt_a[i], T = w.cnt_t[i];
  out.meta[i] = make_int4(static_cast<int>(w.aoff[i]), N, static_cast<int>(t0), T);
  out.seeds[i] = in.seeds ? in.seeds[i] : 0ull;
  out.id_rank[i] = in.id_rank ? in.id_rank[i] : static_cast<unsigned>(i);
  const long pairs = static_cast<long>(N) * (N - 1) / 2;
  const long cost = 256L * N + 32L * T * (N + pairs + mv);
  // ascending sort key: in-class ligands by descending cost, dropped last
  w.key[i] = w.cls[i] >= 0 ? ~static_cast<unsigned>(cost) : 0xffffffffu;
  w.idx[i] = i;
  const int c = w.cls[i];
  if (c >= 0) {
    const int mvp = static_cast<int>((mv + 15) & ~15L);
    atomicMax(&w.stats[0], N);
    atomicMax(&w.stats[1], T);
    atomicMax(&w.stats[2], mvp);
    atomicAdd(&w.stats[3], 1);
    if (c < kPkMaxClasses) {
      atomicMax(&w.stats[4 + 3 * c], N);
      atomicMax(&w.stats[5 + 3 * c], T);
      atomicMax(&w.stats[6 + 3 * c], mvp);
    }
  }
}

// pass 2b: axes and the u8 moving lists (each torsion writes its own span)
__global__ void pk_moving(PackIn in, PackWork w, PackDev out) {
  const long t = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= in.total_tors) return;
  const int i = ligand_of(w.toff, in.n, t);
  const int N = in.n_atoms[i];
  const long rel = w.msrc[t] - w.msrc[w.toff[i]];
  const int c = w.cnt_m[t];
  out.axes[t] = make_int4(in.axis_a[t], in.axis_b[t], static_cast<int>(rel), c);
  uint8_t* dst = out.moving + w.moff[i] + rel;
  const int* src = in.moving + w.msrc[t];
  for (int m = 0; m < c; ++m) {
    const int idx = src[m];
    if (idx < 0 || idx >= N) report(w.err, 2, i, kPkTopology);
    dst[m] = static_cast<uint8_t>(idx);
  }
}

// per ligand: moving segment descriptor and its zero padding
__global__ void pk_segments(PackIn in, PackWork w, PackDev out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= in.n) return;
  const long mv = w.msrc[w.toff[i + 1]] - w.msrc[w.toff[i]];
  out.mov[i] = make_int2(static_cast<int>(w.moff[i]), w.cnt_p[i]);
  for (long z = mv; z < w.cnt_p[i]; ++z) out.moving[w.moff[i] + z] = 0;
}

// 32 B atom records: x, y, z (FP64, as given), element class
__global__ void pk_atoms(PackIn in, PackDev out) {
  const long a = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= in.total_atoms) return;
  const double* c = in.coords + 3 * a;
  out.atoms[a] = make_double4(c[0], c[1], c[2], static_cast<double>(in.atom_class[a]));
}

// the torsion-tree property the incremental flex relies on (vs_runtime.cu
// check_nested): for j < k, moving_k and axis k lie inside moving_j (+ axis
// j) or are disjoint from it, and no later torsion moves axis j
__global__ void pk_nested(PackIn in, PackWork w, PackDev out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= in.n) return;
  const int T = w.cnt_t[i];
  if (T < 2) return;
  const int4* ax = out.axes + w.toff[i];
  const uint8_t* mv = out.moving + w.moff[i];
  unsigned long long set[kMaxTors][2];
  for (int j = 0; j < T; ++j) {
    set[j][0] = set[j][1] = 0ull;
    for (int m = 0; m < ax[j].w; ++m) set[j][mv[ax[j].z + m] >> 6] |= 1ull << (mv[ax[j].z + m] & 63);
  }
  auto has = [&](int j, int a) { return (set[j][a >> 6] >> (a & 63)) & 1ull; };
  for (int j = 0; j < T; ++j)
    for (int k = j + 1; k < T; ++k) {
      const bool sub = ((set[k][0] & ~set[j][0]) | (set[k][1] & ~set[j][1])) == 0 &&
                       (has(j, ax[k].x) || ax[k].x == ax[j].x || ax[k].x == ax[j].y) &&
                       (has(j, ax[k].y) || ax[k].y == ax[j].x || ax[k].y == ax[j].y);
      const bool dis = ((set[k][0] & set[j][0]) | (set[k][1] & set[j][1])) == 0 && !has(j, ax[k].x) &&
                       !has(j, ax[k].y);
      if ((!sub && !dis) || has(k, ax[j].x) || has(k, ax[j].y)) {
        report(w.err, 3, i, kPkNotTree);
        return;
      }
    }
}

}  // namespace

size_t pack_temp_bytes(int n, long total_tors) {
  size_t a = 0, b = 0, c = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, a, static_cast<const long*>(nullptr),
                                static_cast<long*>(nullptr), static_cast<long>(n) + 1);
  cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<const long*>(nullptr),
                                static_cast<long*>(nullptr), total_tors + 1);
  cub::DeviceRadixSort::SortPairs(nullptr, c, static_cast<const unsigned*>(nullptr),
                                  static_cast<unsigned*>(nullptr), static_cast<const int*>(nullptr),
                                  static_cast<int*>(nullptr), n);
  return std::max(a, std::max(b, c)) + 256;
}

static unsigned blocks_for(long n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

cudaError_t pack_stage1(cudaStream_t st, const PackIn& in, const PackWork& w, int n_classes) {
  pk_counts<<<blocks_for(in.n + 1, 256), 256, 0, st>>>(in, w, n_classes);
  return cudaGetLastError();
}

cudaError_t pack_stage2(cudaStream_t st, const PackIn& in, const PackWork& w, const PackDev& out,
                        void* temp, size_t temp_bytes) {
  const long n1 = static_cast<long>(in.n) + 1, t1 = in.total_tors + 1;
  size_t tb = temp_bytes;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, tb, w.cnt_a, w.aoff, n1, st);
  tb = temp_bytes;
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(temp, tb, w.cnt_t, w.toff, n1, st);
  if (e != cudaSuccess) return e;
  pk_torsions<<<blocks_for(t1, 256), 256, 0, st>>>(in, w);
  tb = temp_bytes;
  e = cub::DeviceScan::ExclusiveSum(temp, tb, w.cnt_m, w.msrc, t1, st);
  if (e != cudaSuccess) return e;
  pk_ligands<<<blocks_for(n1, 256), 256, 0, st>>>(in, w, out);
  tb = temp_bytes;
  e = cub::DeviceScan::ExclusiveSum(temp, tb, w.cnt_p, w.moff, n1, st);
  if (e != cudaSuccess) return e;
  if (in.total_tors > 0) pk_moving<<<blocks_for(in.total_tors, 256), 256, 0, st>>>(in, w, out);
  pk_segments<<<blocks_for(in.n, 256), 256, 0, st>>>(in, w, out);
  if (in.total_atoms > 0) pk_atoms<<<blocks_for(in.total_atoms, 256), 256, 0, st>>>(in, out);
  pk_nested<<<blocks_for(in.n, 128), 128, 0, st>>>(in, w, out);
  tb = temp_bytes;
  e = cub::DeviceRadixSort::SortPairs(temp, tb, w.key, w.key_sorted, w.idx, out.order, in.n, 0, 32,
                                      st);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// ---- per-ligand pose ranges of a device pose list (vs_rescore_device):
// pose_lig non-decreasing; first[l] / count[l] of its poses and tb[l], the
// offset of its first pose's torsions in the concatenated torsion array
namespace {
__global__ void pr_init(int* first, int* count, int n) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < n) {
    first[l] = 0x7fffffff;
    count[l] = 0;
  }
}
__global__ void pr_count(const int* pose_lig, long n_poses, LibDev lib, int* first, int* count,
                         long* tcnt) {
  const long p = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p > n_poses) return;
  if (p == n_poses) {
    tcnt[p] = 0;
    return;
  }
  const int l = pose_lig[p];
  atomicAdd(&count[l], 1);
  atomicMin(&first[l], static_cast<int>(p));
  tcnt[p] = lib.meta[l].w;
}
__global__ void pr_base(const int* first, const int* count, const long* tb_pose, long* tb, int n) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l < n) tb[l] = count[l] > 0 ? tb_pose[first[l]] : 0;
}
}  // namespace

size_t pose_ranges_temp_bytes(long n_poses) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<const long*>(nullptr),
                                static_cast<long*>(nullptr), n_poses + 1);
  return b + 256;
}

// tb_pose: 2 (n_poses + 1) longs of scratch (counts, then their scan)
cudaError_t launch_pose_ranges(cudaStream_t st, const int* pose_lig, long n_poses,
                               const LibDev& lib, int* first, int* count, long* tb_pose, long* tb,
                               int n_ligs, void* temp, size_t temp_bytes) {
  pr_init<<<blocks_for(n_ligs, 256), 256, 0, st>>>(first, count, n_ligs);
  long* tcnt = tb_pose + n_poses + 1;
  pr_count<<<blocks_for(n_poses + 1, 256), 256, 0, st>>>(pose_lig, n_poses, lib, first, count, tcnt);
  size_t tb2 = temp_bytes;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(temp, tb2, tcnt, tb_pose, n_poses + 1, st);
  if (e != cudaSuccess) return e;
  pr_base<<<blocks_for(n_ligs, 256), 256, 0, st>>>(first, count, tb_pose, tb, n_ligs);
  return cudaGetLastError();
}

}  // namespace vs
