// embed_3d's spring relaxation (chem.cpp:355-392, 434-445) on the GPU, one
// warp per ligand, FP64 in the reference's operation order so the result is
// bit-identical to the host embed (vs_ingest.cpp springs / closest_pair):
//   per iteration, grad[k] = bond terms of k in bond order, then the
//   non-bonded repulsion terms of k with partners in ascending index (the
//   order in which the reference's serial pair loop reaches atom k); then
//   step = grad * -0.05, clipped to length 0.2, pos += step for every atom.
// Lanes own atoms (no cross-lane sums); the new positions go to a second
// buffer so every gradient sees the previous iteration's positions.  The
// BFS placement runs on the host (bit-identical: glibc log/cos for the
// jitter) or, with seeds, here (place_dev: CUDA log/cos, within a tolerance).
#include <cuda_runtime.h>
#include <stdint.h>

namespace vs {

struct RelaxLib {
  const long long* atom_off;  // [n+1]
  const int* n_atoms;
  const long long* bond_off;  // [n+1]
  const int* n_bonds;
  const int2* bonds;
  double* coords;  // [3 * atoms], in / out
  const unsigned long long* seeds;  // embed seeds: place first (nullptr: relax only)
};

// Rng (rng.hpp:14-41) at explicit counters: split(0x3d) of Rng(seed), normal
// draw j from counters 2j + 1, 2j + 2 (single-value Box-Muller, no cache)
__device__ __forceinline__ unsigned long long emix(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
constexpr unsigned long long kGold = 0x9e3779b97f4a7c15ull;
__device__ __forceinline__ double enormal(unsigned long long key, long j) {
  const unsigned long long a = emix(key + kGold * static_cast<unsigned long long>(2 * j + 1));
  const unsigned long long b = emix(key + kGold * static_cast<unsigned long long>(2 * j + 2));
  const double u1 = static_cast<double>((a >> 11) + 1) * 0x1.0p-53;
  const double u2 = static_cast<double>(b >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

// BFS tetrahedral placement (chem.cpp:410-432): lane 0 walks the BFS (the
// neighbours of an atom in bond order = its incidence list), the lanes draw
// 32 placements' jitter at a time, lane 0 places them in BFS order:
// pos[w] = (pos[v] + dir * 1.5) + jit * 0.05.  Scratch: the q arrays.
__device__ void place_dev(double* px, double* py, double* pz, double* q, const int2* bd,
                          const short* io, const short* inc, int n, unsigned long long seed,
                          int lane) {
  int* ord = reinterpret_cast<int*>(q);  // BFS order (ord[0] = atom 0)
  int* par = ord + n;                    // parent of ord[m]
  int* slot = par + n;                   // tetrahedral direction of ord[m]
  int* kids = slot + n;                  // children placed so far
  int* seen = kids + n;
  if (lane == 0) {
    for (int k = 0; k < n; ++k) {
      kids[k] = 0;
      seen[k] = 0;
      px[k] = py[k] = pz[k] = 0.0;
    }
    ord[0] = 0;
    seen[0] = 1;
    int tail = 1;
    for (int qi = 0; qi < tail; ++qi) {
      const int v = ord[qi];
      for (int u = io[v]; u < io[v + 1]; ++u) {
        const int e = inc[u] >> 1;
        const int w = (inc[u] & 1) ? bd[e].x : bd[e].y;
        if (seen[w]) continue;
        seen[w] = 1;
        par[tail] = v;
        slot[tail] = kids[v] % 4;
        ++kids[v];
        ord[tail++] = w;
      }
    }
  }
  __syncwarp();
  const unsigned long long root = emix(seed ^ kGold);
  const unsigned long long key = emix(root ^ emix(0x3dull + kGold));
  const double t = 1.0 / sqrt(3.0);
  for (int c = 1; c < n; c += 32) {
    const int m = c + lane;  // placement m - 1 draws normals 3(m-1) .. 3(m-1) + 2
    double jx = 0.0, jy = 0.0, jz = 0.0;
    if (m < n) {
      jx = enormal(key, 3L * (m - 1));
      jy = enormal(key, 3L * (m - 1) + 1);
      jz = enormal(key, 3L * (m - 1) + 2);
    }
    for (int k = 0; k < 32 && c + k < n; ++k) {
      const double ax = __shfl_sync(0xffffffffu, jx, k), ay = __shfl_sync(0xffffffffu, jy, k),
                   az = __shfl_sync(0xffffffffu, jz, k);
      if (lane == 0) {
        const int w = ord[c + k], v = par[c + k], sl = slot[c + k];
        const double dx = (sl == 0 || sl == 1) ? t : -t;
        const double dy = (sl == 0 || sl == 2) ? t : -t;
        const double dz = (sl == 0 || sl == 3) ? t : -t;
        px[w] = (px[v] + dx * 1.5) + ax * 0.05;
        py[w] = (py[v] + dy * 1.5) + ay * 0.05;
        pz[w] = (pz[v] + dz * 1.5) + az * 0.05;
      }
    }
  }
  __syncwarp();
}

__device__ __forceinline__ double nrm(double x, double y, double z) {
  return sqrt(x * x + y * y + z * z);
}

// inc[ioff[k] .. ioff[k+1]): the bonds of atom k in bond order, as
// (bond index << 1) | (k is the bond's second atom)
__device__ void springs_dev(double* px, double* py, double* pz, double* qx, double* qy,
                            double* qz, const int2* bd, const short* ioff, const short* inc,
                            const unsigned* bonded, int n, int iters, int lane) {
  for (int it = 0; it < iters; ++it) {
    for (int k = lane; k < n; k += 32) {
      double gx = 0.0, gy = 0.0, gz = 0.0;
      for (int u = ioff[k]; u < ioff[k + 1]; ++u) {  // bonded rest length 1.5
        const int e = inc[u] >> 1;
        const int a = bd[e].x, b = bd[e].y;
        const double dx = px[a] - px[b], dy = py[a] - py[b], dz = pz[a] - pz[b];
        const double len = nrm(dx, dy, dz);
        if (len < 1e-12) continue;
        const double s = 2.0 * (len - 1.5) / len;
        if (!(inc[u] & 1)) {
          gx = gx + dx * s;
          gy = gy + dy * s;
          gz = gz + dz * s;
        } else {
          gx = gx - dx * s;
          gy = gy - dy * s;
          gz = gz - dz * s;
        }
      }
      const unsigned* bk = bonded + 4 * k;
      for (int p = 0; p < n; ++p) {  // non-bonded repulsion below 1.0
        if (p == k || ((bk[p >> 5] >> (p & 31)) & 1u)) continue;
        const int a = p < k ? p : k, b = p < k ? k : p;
        const double dx = px[a] - px[b], dy = py[a] - py[b], dz = pz[a] - pz[b];
        // sqrt is monotone and sqrt(1) = 1: |d|^2 >= 1 implies len >= 1, so
        // the far pairs skip the square root and keep the reference's outcome
        const double n2 = dx * dx + dy * dy + dz * dz;
        if (n2 >= 1.0) continue;
        const double len = sqrt(n2);
        if (len >= 1.0 || len < 1e-12) continue;
        const double s = -2.0 * (1.0 - len) / len;
        if (a == k) {
          gx = gx + dx * s;
          gy = gy + dy * s;
          gz = gz + dz * s;
        } else {
          gx = gx - dx * s;
          gy = gy - dy * s;
          gz = gz - dz * s;
        }
      }
      double sx = gx * -0.05, sy = gy * -0.05, sz = gz * -0.05;
      const double sn = nrm(sx, sy, sz);
      if (sn > 0.2) {
        const double f = 0.2 / sn;
        sx = sx * f;
        sy = sy * f;
        sz = sz * f;
      }
      qx[k] = px[k] + sx;
      qy[k] = py[k] + sy;
      qz[k] = pz[k] + sz;
    }
    __syncwarp();
    for (int k = lane; k < n; k += 32) {
      px[k] = qx[k];
      py[k] = qy[k];
      pz[k] = qz[k];
    }
    __syncwarp();
  }
}

// min over pairs of |a - b| (chem.cpp:394-400) as sqrt(min |a - b|^2): sqrt
// is monotone and correctly rounded, so the two agree bit for bit
__device__ double closest_dev(const double* px, const double* py, const double* pz, int n,
                              int lane) {
  double best = 1.0 / 0.0;
  for (int a = lane; a < n; a += 32)
    for (int b = a + 1; b < n; ++b) {
      const double dx = px[a] - px[b], dy = py[a] - py[b], dz = pz[a] - pz[b];
      best = fmin(best, dx * dx + dy * dy + dz * dz);
    }
  for (int off = 16; off > 0; off >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, off));
  return sqrt(best);
}

constexpr int kRelaxMaxAtoms = 128;
constexpr int kRelaxMaxBonds = 256;
constexpr int kRelaxWarps = 4;

// per-warp shared-memory region for ligands of <= amax atoms, <= bmax bonds
__host__ __device__ inline size_t relax_warp_bytes(int amax, int bmax) {
  const size_t a8 = 48u * amax;                      // p, q: 6 x amax doubles
  const size_t b8 = 8u * bmax;                       // bonds
  const size_t m4 = 16u * amax;                      // bonded bitmasks, 4 words per atom
  const size_t s2 = 2u * ((amax + 2) + 2 * bmax);    // incidence offsets + lists (short)
  return (a8 + b8 + m4 + s2 + 15u) & ~size_t(15);
}

__global__ void __launch_bounds__(kRelaxWarps * 32)
    vs_relax_kernel(const __grid_constant__ RelaxLib L, int n, int iterations, int amax,
                    int bmax) {
  extern __shared__ __align__(16) unsigned char relax_smem[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kRelaxWarps + w;
  if (i >= n) return;
  const int na = L.n_atoms[i], nb = L.n_bonds[i];
  if (na < 2 || na > amax || nb > bmax) return;
  unsigned char* base = relax_smem + w * relax_warp_bytes(amax, bmax);
  double* px = reinterpret_cast<double*>(base);
  double *py = px + amax, *pz = py + amax, *qx = pz + amax, *qy = qx + amax, *qz = qy + amax;
  int2* sb = reinterpret_cast<int2*>(qz + amax);
  unsigned* sbond = reinterpret_cast<unsigned*>(sb + bmax);
  short* io = reinterpret_cast<short*>(sbond + 4 * amax);
  short* inc = io + amax + 2;
  double* c = L.coords + 3 * L.atom_off[i];
  if (!L.seeds) {
    for (int k = lane; k < na; k += 32) {
      px[k] = c[3 * k];
      py[k] = c[3 * k + 1];
      pz[k] = c[3 * k + 2];
    }
  }
  for (int k = lane; k < 4 * na; k += 32) sbond[k] = 0u;
  for (int e = lane; e < nb; e += 32) sb[e] = L.bonds[L.bond_off[i] + e];
  __syncwarp();
  if (lane == 0) {
    for (int k = 0; k <= na; ++k) io[k] = 0;
    for (int e = 0; e < nb; ++e) {
      const int a = sb[e].x, b = sb[e].y;
      sbond[4 * a + (b >> 5)] |= 1u << (b & 31);
      sbond[4 * b + (a >> 5)] |= 1u << (a & 31);
      ++io[a + 1];
      if (b != a) ++io[b + 1];
    }
    for (int k = 0; k < na; ++k) io[k + 1] += io[k];
    int* fill = reinterpret_cast<int*>(qx);  // scratch until the springs run
    for (int k = 0; k < na; ++k) fill[k] = io[k];
    for (int e = 0; e < nb; ++e) {  // bond order within each atom's list
      const int a = sb[e].x, b = sb[e].y;
      inc[fill[a]++] = static_cast<short>(e << 1);
      if (b != a) inc[fill[b]++] = static_cast<short>((e << 1) | 1);
    }
  }
  __syncwarp();
  if (L.seeds) place_dev(px, py, pz, qx, sb, io, inc, na, L.seeds[i], lane);
  springs_dev(px, py, pz, qx, qy, qz, sb, io, inc, sbond, na, iterations, lane);
  for (int round = 0; round < 20 && closest_dev(px, py, pz, na, lane) < 0.5; ++round)
    springs_dev(px, py, pz, qx, qy, qz, sb, io, inc, sbond, na, 50, lane);
  for (int k = lane; k < na; k += 32) {
    c[3 * k] = px[k];
    c[3 * k + 1] = py[k];
    c[3 * k + 2] = pz[k];
  }
}

int relax_max_atoms() { return kRelaxMaxAtoms; }
int relax_max_bonds() { return kRelaxMaxBonds; }

cudaError_t launch_relax(cudaStream_t st, const long long* atom_off, const int* n_atoms,
                         const long long* bond_off, const int* n_bonds, const int2* bonds,
                         double* coords, int n, int iterations, int amax, int bmax,
                         const unsigned long long* seeds) {
  RelaxLib L{atom_off, n_atoms, bond_off, n_bonds, bonds, coords, seeds};
  const int blocks = (n + kRelaxWarps - 1) / kRelaxWarps;
  const size_t smem = kRelaxWarps * relax_warp_bytes(amax, bmax);
  cudaError_t e = cudaFuncSetAttribute(vs_relax_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  if (blocks > 0)
    vs_relax_kernel<<<blocks, kRelaxWarps * 32, smem, st>>>(L, n, iterations, amax, bmax);
  return cudaGetLastError();
}

}  // namespace vs
