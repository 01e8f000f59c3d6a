// embed_3d's spring relaxation (chem.cpp:355-392, 434-445) on the GPU, one
// warp per ligand, FP64 in the reference's operation order so the result is
// bit-identical to the host embed (vs_ingest.cpp springs / closest_pair):
//   per iteration, grad[k] = bond terms of k in bond order, then the
//   non-bonded repulsion terms of k with partners in ascending index (the
//   order in which the reference's serial pair loop reaches atom k); then
//   step = grad * -0.05, clipped to length 0.2, pos += step for every atom.
// Lanes own atoms (no cross-lane sums); the new positions go to a second
// buffer so every gradient sees the previous iteration's positions.  The
// BFS placement (RNG jitter through glibc log/cos) stays on the host.
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
};

__device__ __forceinline__ double nrm(double x, double y, double z) {
  return sqrt(x * x + y * y + z * z);
}

__device__ void springs_dev(double* px, double* py, double* pz, double* qx, double* qy,
                            double* qz, const int2* bd, int nb, const unsigned* bonded, int n,
                            int iters, int lane) {
  for (int it = 0; it < iters; ++it) {
    for (int k = lane; k < n; k += 32) {
      double gx = 0.0, gy = 0.0, gz = 0.0;
      for (int e = 0; e < nb; ++e) {  // bonded rest length 1.5
        const int a = bd[e].x, b = bd[e].y;
        if (a != k && b != k) continue;
        const double dx = px[a] - px[b], dy = py[a] - py[b], dz = pz[a] - pz[b];
        const double len = nrm(dx, dy, dz);
        if (len < 1e-12) continue;
        const double s = 2.0 * (len - 1.5) / len;
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
      for (int p = 0; p < n; ++p) {  // non-bonded repulsion below 1.0
        if (p == k || ((bonded[4 * k + (p >> 5)] >> (p & 31)) & 1u)) continue;
        const int a = p < k ? p : k, b = p < k ? k : p;
        const double dx = px[a] - px[b], dy = py[a] - py[b], dz = pz[a] - pz[b];
        const double len = nrm(dx, dy, dz);
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

__device__ double closest_dev(const double* px, const double* py, const double* pz, int n,
                              int lane) {
  double best = 1.0 / 0.0;
  for (int a = lane; a < n; a += 32)
    for (int b = a + 1; b < n; ++b)
      best = fmin(best, nrm(px[a] - px[b], py[a] - py[b], pz[a] - pz[b]));
  for (int off = 16; off > 0; off >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, off));
  return best;
}

constexpr int kRelaxMaxAtoms = 128;
constexpr int kRelaxMaxBonds = 256;
constexpr int kRelaxWarps = 4;

__global__ void __launch_bounds__(kRelaxWarps * 32)
    vs_relax_kernel(const __grid_constant__ RelaxLib L, int n, int iterations) {
  __shared__ double sp[kRelaxWarps][6][kRelaxMaxAtoms];
  __shared__ int2 sb[kRelaxWarps][kRelaxMaxBonds];
  __shared__ unsigned sbond[kRelaxWarps][4 * kRelaxMaxAtoms];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * kRelaxWarps + w;
  if (i >= n) return;
  const int na = L.n_atoms[i], nb = L.n_bonds[i];
  if (na < 2 || na > kRelaxMaxAtoms || nb > kRelaxMaxBonds) return;
  double *px = sp[w][0], *py = sp[w][1], *pz = sp[w][2];
  double *qx = sp[w][3], *qy = sp[w][4], *qz = sp[w][5];
  double* c = L.coords + 3 * L.atom_off[i];
  for (int k = lane; k < na; k += 32) {
    px[k] = c[3 * k];
    py[k] = c[3 * k + 1];
    pz[k] = c[3 * k + 2];
  }
  for (int k = lane; k < 4 * na; k += 32) sbond[w][k] = 0u;
  for (int e = lane; e < nb; e += 32) sb[w][e] = L.bonds[L.bond_off[i] + e];
  __syncwarp();
  if (lane == 0)
    for (int e = 0; e < nb; ++e) {
      const int a = sb[w][e].x, b = sb[w][e].y;
      sbond[w][4 * a + (b >> 5)] |= 1u << (b & 31);
      sbond[w][4 * b + (a >> 5)] |= 1u << (a & 31);
    }
  __syncwarp();
  springs_dev(px, py, pz, qx, qy, qz, sb[w], nb, sbond[w], na, iterations, lane);
  for (int round = 0; round < 20 && closest_dev(px, py, pz, na, lane) < 0.5; ++round)
    springs_dev(px, py, pz, qx, qy, qz, sb[w], nb, sbond[w], na, 50, lane);
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
                         double* coords, int n, int iterations) {
  RelaxLib L{atom_off, n_atoms, bond_off, n_bonds, bonds, coords};
  const int blocks = (n + kRelaxWarps - 1) / kRelaxWarps;
  if (blocks > 0) vs_relax_kernel<<<blocks, kRelaxWarps * 32, 0, st>>>(L, n, iterations);
  return cudaGetLastError();
}

}  // namespace vs
