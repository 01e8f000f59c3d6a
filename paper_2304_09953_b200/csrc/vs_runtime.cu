// GPU runtime behind the C-ABI (capi.h "GPU runtime" section): device
// handle, pocket upload + grid build, the library packer (size-class
// buckets, SoA, LPT order), dock launches per bucket, results, top-k and
// the rescoring path.  Host C++; the kernels live in vs_kernels.cu.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <functional>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vscreen_gpu/capi.h"
#include "vs_pack.h"
#include "vs_rng.h"
#include "vs_types.h"

namespace vs {
size_t rescore_smem_per_block(int nmax, int tmax, int mvmax);
size_t stage_smem_per_block(int nmax, int tmax, int mvmax);
constexpr int kStats = 10;  // work counters (capi.h vs_last_stats_ex)
// vs_dock_host pipelines libraries of at least kPipeMinLigands ligands in
// contiguous chunks cut at these fractions of the library
constexpr int kPipeMinLigands = 32768;
// (four equal chunks, two in flight: measured best of the shapes tried,
// tools/pipe_ab.sh; profiles/e2e_pipeline_r2.txt)
constexpr double kPipeSplit[] = {0.25, 0.5, 0.75};

cudaError_t launch_draws(cudaStream_t st, const PocketDev& pk, const unsigned long long* seeds,
                         const int* n_tors, int n, int restarts, int attempts, float* out,
                         int stride, int sms);
cudaError_t launch_staged(bool grid, int sms, cudaStream_t st, const LibDev& lib,
                          const PocketDev& pk, const float4* rots, const float4* rots_p,
                          const int* perm, const DockParams& prm, const int* order, int n, int* counters,
                          int nmax, int tmax, int mvmax, const StageBufs& sb, const DockOut& out,
                          uint64_t* launches, cudaEvent_t* evs, int* kinds);
cudaError_t launch_rescore(bool grid, int blocks, size_t smem, cudaStream_t st, const LibDev& lib,
                           const PocketDev& pk, const int* ligs, int n_ligs, int* counter,
                           const PoseSrc& src, int nmax, int tmax, int mvmax);
cudaError_t launch_pose_ranges(cudaStream_t st, const int* pose_lig, long n_poses,
                               const LibDev& lib, int* first, int* count, long* tb_pose, long* tb,
                               int n_ligs, void* temp, size_t temp_bytes);
size_t pose_ranges_temp_bytes(long n_poses);
size_t grad_smem_per_block(int nmax, int tmax);
size_t ascend_smem_per_block(int nmax, int tmax);
cudaError_t launch_ascend(cudaStream_t st, const LibDev& lib, const SiteD* sites, int n_sites,
                          const double lo[3], const double hi[3], double r, double lam,
                          long n_poses, const int* pose_lig, const long* tb, double* t, double* q,
                          double* tors, int nmax, int tmax, int max_steps, double* score,
                          int* steps);
int relax_max_atoms();
int relax_max_bonds();
cudaError_t launch_relax(cudaStream_t st, const long long* atom_off, const int* n_atoms,
                         const long long* bond_off, const int* n_bonds, const int2* bonds,
                         double* coords, int n, int iterations, int amax, int bmax,
                         const unsigned long long* seeds);
cudaError_t launch_grad(cudaStream_t st, const LibDev& lib, const SiteD* sites, int n_sites,
                        const double lo[3], const double hi[3], double r, double lam,
                        long n_poses, const int* pose_lig, const long* tb, const double* t,
                        const double* q, const double* tors, int nmax, int tmax, double* score,
                        double* gt, double* gq, double* gtor, double* resc = nullptr);
cudaError_t launch_grid(cudaStream_t st, const PocketDev& pk, float* steric, float* hb,
                        float* lipo, float* key, float4* cells);
int topk_chunk();
double measure_peak(int kind, int sms);
cudaError_t launch_softtab(cudaStream_t st, float r, float cut2, float2* tab);
double measure_gather_peak(int sms, int bytes);
cudaError_t launch_topk(cudaStream_t st, const unsigned long long* in, long n,
                        unsigned long long* out, int k, int blocks);
}  // namespace vs

using namespace vs;

namespace {

// grow-only device buffer
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t want = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct Bucket {
  int start = 0, count = 0;  // range in the order array
  int nmax = 1, tmax = 1, mvmax = 16;
};

// Packed library (host staging + device copies) for one set of ligands.
// Growable page-locked host array: the packed library is written straight
// into pinned memory, so the upload is one async DMA per array.
template <class T>
struct PinnedVec {
  T* p = nullptr;
  size_t n = 0, cap = 0;
  PinnedVec() = default;
  PinnedVec(const PinnedVec&) = delete;
  PinnedVec& operator=(const PinnedVec&) = delete;
  ~PinnedVec() {
    if (p) cudaFreeHost(p);
  }
  bool resize(size_t m) {
    if (m > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      cap = 0;
      const size_t want = std::max<size_t>(m + m / 4, 64);
      if (cudaHostAlloc(reinterpret_cast<void**>(&p), want * sizeof(T), cudaHostAllocDefault) !=
          cudaSuccess) {
        p = nullptr;
        n = 0;
        return false;
      }
      cap = want;
    }
    n = m;
    return true;
  }
  size_t size() const { return n; }
  bool empty() const { return n == 0; }
  T* data() { return p; }
  const T* data() const { return p; }
  T& operator[](size_t i) { return p[i]; }
  const T& operator[](size_t i) const { return p[i]; }
};

// the device packer's scratch (raw arrays as given, work arrays, CUB temp,
// pinned readback)
struct PackScratch {
  DBuf raw[9], pwork[13], ptemp;
  PinnedVec<int> pk_host;  // stats + error key + classes read back
  void release() {
    for (DBuf& b : raw) b.release();
    for (DBuf& b : pwork) b.release();
    ptemp.release();
  }
};

// a pack issued (pack_issue) and not yet read back (pack_finish)
struct PackPending {
  int n = 0, nc = 0;
  long A = 0, T = 0;
  size_t cls_at = 0;
  bool classes = false;
  int slot = 0;  // the PackScratch it uses
};

struct Packed {
  int n = 0;
  PinnedVec<int4> meta;
  PinnedVec<int2> mov;
  PinnedVec<double4> atoms;
  PinnedVec<int4> axes;
  PinnedVec<uint8_t> moving;
  PinnedVec<unsigned long long> seeds;
  PinnedVec<unsigned int> id_rank;
  std::vector<int> order;
  PinnedVec<int> order_pin;  // pinned copy of `order` (async H2D from a pipelined pack)
  std::vector<int> cls;          // class per ligand (-1 dropped)
  std::vector<long> tors_off;    // prefix sum of n_tors
  std::vector<Bucket> buckets;
  Bucket all;  // global LPT order (dock launch)
  long total_tors = 0;
  long total_atoms = 0;
  bool on_device = false;  // packed by gpu_pack: buckets[c] = size class c
  DBuf d_meta, d_mov, d_atoms, d_axes, d_moving, d_seeds, d_idr, d_order;
  void release() {
    d_meta.release(); d_mov.release(); d_atoms.release(); d_axes.release();
    d_moving.release(); d_seeds.release(); d_idr.release(); d_order.release();
  }
  LibDev dev() const {
    LibDev l;
    l.meta = d_meta.as<const int4>();
    l.mov = d_mov.as<const int2>();
    l.atoms = d_atoms.as<const double4>();
    l.axes = d_axes.as<const int4>();
    l.moving = d_moving.as<const uint8_t>();
    l.seeds = d_seeds.as<const unsigned long long>();
    l.id_rank = d_idr.as<const unsigned int>();
    return l;
  }
};

}  // namespace

// per-ligand state of one staged dock (StageBufs) + its launch counters
struct StageSet {
  DBuf ys, ysf, th, pose, bk, nk, kx, kp, km, st, counters;
  cudaError_t ensure(size_t na, size_t nt, size_t nn, size_t R) {
    cudaError_t e = cudaSuccess;
    auto en = [&](DBuf& d, size_t bytes) {
      if (e == cudaSuccess) e = d.ensure(bytes);
    };
    en(ys, na * sizeof(double4));
    en(ysf, na * sizeof(float4));
    en(th, nt * sizeof(float));
    en(pose, nn * 2 * sizeof(float4));
    en(bk, nn * sizeof(int));
    en(nk, nn * sizeof(int));
    en(kx, na * R * sizeof(float4));
    en(kp, (nn * 8 + nt) * R * sizeof(float));
    en(km, nn * R * 4 * sizeof(int));
    en(st, nn * 8 * sizeof(unsigned long long));
    en(counters, 320 * sizeof(int));
    return e;
  }
  StageBufs bufs() const {
    StageBufs sb;
    sb.ys = ys.as<double4>();
    sb.ysf = ysf.as<float4>();
    sb.th = th.as<float>();
    sb.pose = pose.as<float4>();
    sb.bk = bk.as<int>();
    sb.nk = nk.as<int>();
    sb.kx = kx.as<float4>();
    sb.kp = kp.as<float>();
    sb.km = km.as<int>();
    sb.st = st.as<unsigned long long>();
    return sb;
  }
  void release() {
    for (DBuf* b : {&ys, &ysf, &th, &pose, &bk, &nk, &kx, &kp, &km, &st, &counters}) b->release();
  }
};

struct vs_handle {
  int device = 0;
  cudaTextureObject_t key_tex = 0;  // the key-map cells as a linear texture
  cudaStream_t own = nullptr;
  cudaStream_t last = nullptr;
  std::string err;
  int sms = 148;
  char name[256] = {0};
  int clock_khz = 0;
  uint64_t launches = 0;
  // pocket
  bool has_pocket = false;
  bool empty_bounds = false;
  PocketDev pk{};
  DBuf d_sites, d_maps, d_softtab;
  DBuf d_sites64;               // FP64 sites, pocket order (score_gradient)
  int n_sites64 = 0;
  double box_lo[3] = {0, 0, 0}, box_hi[3] = {0, 0, 0}, r64 = 0.0, lam64 = 0.0;
  int gdims[3] = {0, 0, 0};
  // library + results
  bool has_lib = false;
  Packed libs[2];            // the resident library and the spare (prefetch) slot
  int cur = 0;               // libs[cur] is the resident one
  vs_dock_params last_prm{};
  bool has_results = false;
  DBuf d_surv, d_surv_tors, d_all, d_all_tors, d_best, d_nkept, d_nsurv, d_keys;
  DBuf d_rots, d_topk_a, d_topk_b, d_stats;
  StageSet sg;  // staged-dock state of vs_dock
  // what the last results cover: ligand count, class per ligand (-1 =
  // dropped), total torsions (vs_fetch_results, vs_topk)
  int res_n = 0;
  std::vector<int> res_cls;
  long res_tors = 0;
  // the pipelined vs_dock_host (dock_host_pipelined): two library slots and
  // stage sets, a compute stream per slot, H2D and D2H streams, pinned
  // result staging per slot
  Packed pipe_lib[2];
  StageSet pipe_sg[2];
  cudaStream_t pipe_s[2] = {nullptr, nullptr};
  cudaStream_t pipe_in = nullptr, pipe_out = nullptr;
  PinnedVec<uint8_t> pipe_stage[2];
  std::vector<cudaEvent_t> pipe_ev;
  int rots_k = -1;
  uint64_t rots_seed = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // end of the handle's last device operation (dock, top-k, gather) on
  // whichever stream it ran: later operations on other streams, and host
  // rewrites of the handle's buffers, are ordered after it
  cudaEvent_t done = nullptr;
  // NCCL communicator of the multi-GPU top-k gather (vs_comm_init /
  // vs_comm_attach); owned = created by vs_comm_init
  ncclComm_t comm = nullptr;
  bool comm_owned = false;
  DBuf d_gather;  // local top-k followed by the gathered keys of every rank
  std::vector<cudaEvent_t> pev;  // per-launch event pairs of the staged dock
  std::vector<int> pkind;        // kernel kind of each pair (0 start .. 3 finish)
  bool timed = false;
  bool staged_run = false;
  PinnedVec<uint8_t> fetch_stage;  // vs_fetch_results' pinned staging, reused across calls
  Packed rpack;              // vs_rescore's library staging, reused across calls
  // the per-pose FP64 paths (vs_score64, vs_score_gradient, vs_ascend):
  // library staging and pose arrays reused across calls, so a per-pose
  // caller (the C++ drop-in's geometric_score) allocates nothing per call
  Packed xpack;
  DBuf xbuf[10];
  // the device packer (vs_pack.cu): the caller's raw arrays, scratch, CUB temp
  PackScratch ps[2];       // the device packer's scratch, one per library slot
  // vs_dock_host_prefetch: the next library packing into libs[1 - cur] on
  // the copy stream while the current one docks
  cudaStream_t copy = nullptr;
  bool spare_pending = false;
  PackPending spare_pp;
  vs_library spare_L{};
  std::vector<vs_size_class> spare_cls;
  bool spare_has_cls = false;
  // per-class ligand lists of the resident library (the device rescoring
  // entries), rebuilt after each upload
  DBuf d_lib_lists;
  std::vector<std::pair<int, int>> lib_segs;
  int lib_lists_n = -1;
  DBuf rbuf[12];             // vs_rescore's pose / work arrays, reused across calls
  DBuf ebuf[7];              // the device embed's arrays, reused across calls
  PinnedVec<unsigned char> epin;  // their pinned host staging
  double rescore_ms = -1.0;  // device time of the rescore kernels of the last vs_rescore
  std::vector<cudaStream_t> fork;  // the rescoring's per-class streams (joined back)
  std::vector<cudaEvent_t> fork_ev;
  cudaEvent_t rev0 = nullptr, rev1 = nullptr;
};

namespace {

int fail(vs_handle* h, int code, const std::string& msg) {
  if (h) h->err = msg;
  return code;
}

int cuda_fail(vs_handle* h, cudaError_t e, const char* what) {
  return fail(h, VS_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define VS_CUDA(h, call)                                  \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return cuda_fail(h, e_, #call); \
  } while (0)

cudaStream_t pick(vs_handle* h, void* s) {
  h->last = s ? static_cast<cudaStream_t>(s) : h->own;
  return h->last;
}

// stream-side: `st` waits for the handle's previous device operation
cudaError_t after_prev(vs_handle* h, cudaStream_t st) { return cudaStreamWaitEvent(st, h->done, 0); }
// host-side: the previous device operation has finished (before buffers it
// reads are rewritten or freed: pocket, library, rescore staging)
cudaError_t quiesce(vs_handle* h) { return cudaEventSynchronize(h->done); }
cudaError_t mark_done(vs_handle* h, cudaStream_t st) { return cudaEventRecord(h->done, st); }

size_t align16z(size_t x) { return (x + 15) & ~size_t(15); }

// Validation + packing of a host library (SURVEY §8 row A7/A11 checks:
// AtomCountMismatch for empty conformers and axes outside the conformer).
// Stable sort of ligand indices by descending cost (ties keep index order):
// two-pass LSD radix sort on the 32-bit key ~cost (costs fit 32 bits for the
// GPU limits; a wider cost falls back to std::stable_sort).
void lpt_sort(std::vector<int>& idx, const std::vector<long>& cost) {
  long cmax = 0;
  for (int i : idx) cmax = std::max(cmax, cost[i]);
  if (cmax >= (1L << 32) || idx.size() < 4096) {
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    return;
  }
  std::vector<int> tmp(idx.size());
  std::vector<uint32_t> key(cost.size());
  for (int i : idx) key[i] = ~static_cast<uint32_t>(cost[i]);
  for (int pass = 0; pass < 2; ++pass) {
    const int sh = 16 * pass;
    std::vector<size_t> cnt(65537, 0);
    for (int i : idx) ++cnt[((key[i] >> sh) & 0xffffu) + 1];
    for (size_t d = 1; d < cnt.size(); ++d) cnt[d] += cnt[d - 1];
    for (int i : idx) tmp[cnt[(key[i] >> sh) & 0xffffu]++] = i;
    idx.swap(tmp);
  }
}

int upload_packed(vs_handle* h, Packed& P, cudaStream_t st, int parts);

// early: when non-null, the pinned arrays' DMA is issued on it as soon as they
// are filled, so it runs under the LPT sort and bucketing.
int pack_library(vs_handle* h, const vs_library* L, const vs_size_class* classes, int nc,
                 Packed& P, cudaStream_t early = nullptr) {
  const int n = L->n_ligands;
  if (n < 0) return fail(h, VS_ERR_INVALID_ARGUMENT, "negative ligand count");
  P.n = n;
  if (!P.seeds.resize(std::max(n, 1)) || !P.id_rank.resize(std::max(n, 1)))
    return fail(h, VS_ERR_CUDA, "pinned host allocation failed");
  P.cls.assign(n, -1);
  P.tors_off.assign(n + 1, 0);
  const auto pt0 = std::chrono::steady_clock::now();
  // pass 1: a sequential scan validates the counts (the lowest failing
  // ligand's error, as a sequential pass reports it) and lays out the atom
  // and torsion offsets; threads then take the moving-set sizes, classes,
  // seeds and LPT costs; a second scan lays out the moving-list offsets
  std::vector<long> cost(n, 0), aoff(n + 1, 0), moff(n + 1, 0), msrc(n + 1, 0), toff(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    const int N = L->n_atoms[i], T = L->n_tors[i];
    if (N < 1) return fail(h, VS_ERR_ATOM_COUNT, "conformer has no atoms (ligand " + std::to_string(i) + ")");
    if (N > kMaxAtoms || T > kMaxTors)
      return fail(h, VS_ERR_CAPACITY, "ligand " + std::to_string(i) + " exceeds GPU limits");
    if (T < 0) return fail(h, VS_ERR_INVALID_ARGUMENT, "negative torsion count");
    aoff[i + 1] = aoff[i] + N;
    toff[i + 1] = toff[i] + T;
  }
  std::vector<long> mvn(n, 0);
  const int nth1 = std::max(1, std::min<int>(32, static_cast<int>(std::thread::hardware_concurrency())));
  auto scan = [&](int t) {
    const int lo = static_cast<int>(static_cast<long>(n) * t / nth1);
    const int hi = static_cast<int>(static_cast<long>(n) * (t + 1) / nth1);
    for (int i = lo; i < hi; ++i) {
      const int N = L->n_atoms[i], T = L->n_tors[i];
      long mv = 0;
      for (int j = 0; j < T; ++j) mv += L->moving_count[toff[i] + j];
      mvn[i] = mv;
      P.tors_off[i] = toff[i];
      P.seeds[i] = L->seeds ? L->seeds[i] : 0ull;
      P.id_rank[i] = L->id_rank ? L->id_rank[i] : static_cast<unsigned>(i);
      const int rot = L->rot_bonds ? L->rot_bonds[i] : T;
      if (classes && nc > 0) {
        P.cls[i] = vs_size_class_of(N, rot, classes, nc);
        if (P.cls[i] < 0) P.cls[i] = -1;
      } else {
        P.cls[i] = N <= 16 ? 0 : N <= 32 ? 1 : N <= 48 ? 2 : N <= 64 ? 3 : N <= 96 ? 4 : 5;
      }
      const long pairs = static_cast<long>(N) * (N - 1) / 2;
      cost[i] = 256L * N + 32L * T * (N + pairs + mv);
    }
  };
  if (nth1 == 1 || n < 4096) {
    for (int t = 0; t < nth1; ++t) scan(t);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nth1; ++t) pool.emplace_back(scan, t);
    for (auto& th : pool) th.join();
  }
  for (int i = 0; i < n; ++i) {
    msrc[i + 1] = msrc[i] + mvn[i];
    moff[i + 1] = moff[i] + static_cast<long>(align16z(static_cast<size_t>(mvn[i])));
  }
  if (!P.meta.resize(std::max(n, 1)) || !P.mov.resize(std::max(n, 1)) ||
      !P.atoms.resize(std::max<long>(aoff[n], 1)) || !P.axes.resize(std::max<long>(toff[n], 1)) ||
      !P.moving.resize(std::max<long>(moff[n], 16)))
    return fail(h, VS_ERR_CUDA, "pinned host allocation failed");
  if (aoff[n] == 0) P.atoms[0] = double4{0, 0, 0, 0};
  if (toff[n] == 0) P.axes[0] = int4{0, 0, 0, 0};
  if (moff[n] == 0) std::memset(P.moving.data(), 0, 16);
  const auto pt1 = std::chrono::steady_clock::now();
  // pass 2 (threads over ligand ranges): fill + validate; the error of the
  // lowest failing ligand is the one reported (same as a sequential pass)
  const int nth = std::max(1, std::min<int>(32, static_cast<int>(std::thread::hardware_concurrency())));
  std::vector<int> bad(nth, -1), bad_code(nth, 0);
  std::vector<std::string> bad_msg(nth);
  auto fill = [&](int t) {
    const int lo = static_cast<int>(static_cast<long>(n) * t / nth);
    const int hi = static_cast<int>(static_cast<long>(n) * (t + 1) / nth);
    for (int i = lo; i < hi; ++i) {
      const int N = L->n_atoms[i], T = L->n_tors[i];
      P.meta[i] = int4{static_cast<int>(aoff[i]), N, static_cast<int>(toff[i]), T};
      for (int a = 0; a < N; ++a) {
        const double* c = L->coords + 3 * (aoff[i] + a);
        P.atoms[aoff[i] + a] = double4{c[0], c[1], c[2], static_cast<double>(L->atom_class[aoff[i] + a])};
      }
      long mo = msrc[i];
      int mv = 0;
      uint8_t* dst = P.moving.data() + moff[i];
      for (int j = 0; j < T; ++j) {
        const long tj = toff[i] + j;
        const int a = L->axis_a[tj], b = L->axis_b[tj], cnt = L->moving_count[tj];
        if (a < 0 || b < 0 || a >= N || b >= N) {
          bad[t] = i;
          bad_code[t] = VS_ERR_ATOM_COUNT;
          bad_msg[t] = "torsion topology does not fit conformer";
          return;
        }
        P.axes[tj] = int4{a, b, mv, cnt};
        for (int m = 0; m < cnt; ++m) {
          const int idx = L->moving[mo + m];
          if (idx < 0 || idx >= N) {
            bad[t] = i;
            bad_code[t] = VS_ERR_ATOM_COUNT;
            bad_msg[t] = "moving atom outside conformer";
            return;
          }
          dst[mv + m] = static_cast<uint8_t>(idx);
        }
        mo += cnt;
        mv += cnt;
      }
      for (long z = mv; z < moff[i + 1] - moff[i]; ++z) dst[z] = 0;
      P.mov[i] = int2{static_cast<int>(moff[i]), static_cast<int>(moff[i + 1] - moff[i])};
    }
  };
  if (nth == 1 || n < 4096) {
    for (int t = 0; t < nth; ++t) fill(t);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nth; ++t) pool.emplace_back(fill, t);
    for (auto& th : pool) th.join();
  }
  for (int t = 0; t < nth; ++t)
    if (bad[t] >= 0) return fail(h, bad_code[t], bad_msg[t]);
  const long to = toff[n];
  P.tors_off[n] = to;
  P.total_tors = to;
  P.total_atoms = aoff[n];
  P.on_device = false;
  // one stable LPT sort (descending cost, then index); the per-class buckets
  // are class-filtered views of it (same order inside each class), and the
  // global queue over every class is the dock launch's
  if (early) {
    const int urc = upload_packed(h, P, early, 1);
    if (urc) return urc;
  }
  std::vector<int> lpt;
  lpt.reserve(n);
  for (int i = 0; i < n; ++i)
    if (P.cls[i] >= 0) lpt.push_back(i);
  const auto pt2 = std::chrono::steady_clock::now();
  lpt_sort(lpt, cost);
  const auto pt3 = std::chrono::steady_clock::now();
  const int ncls = (classes && nc > 0) ? nc : 6;
  P.order.clear();
  P.order.reserve(2 * lpt.size() + 1);
  P.buckets.clear();
  {
    // one pass over the LPT order into per-class lists (LPT order kept)
    std::vector<std::vector<int>> per(static_cast<std::size_t>(ncls));
    for (int i : lpt) per[static_cast<std::size_t>(P.cls[i])].push_back(i);
    for (int c = 0; c < ncls; ++c) {
      Bucket b;
      b.start = static_cast<int>(P.order.size());
      for (int i : per[static_cast<std::size_t>(c)]) {
        b.nmax = std::max(b.nmax, P.meta[i].y);
        b.tmax = std::max(b.tmax, P.meta[i].w);
        b.mvmax = std::max(b.mvmax, P.mov[i].y);
        P.order.push_back(i);
      }
      b.count = static_cast<int>(P.order.size()) - b.start;
      if (b.count > 0) P.buckets.push_back(b);
    }
  }
  P.all = Bucket{};
  P.all.start = static_cast<int>(P.order.size());
  for (int i : lpt) {
    P.all.nmax = std::max(P.all.nmax, P.meta[i].y);
    P.all.tmax = std::max(P.all.tmax, P.meta[i].w);
    P.all.mvmax = std::max(P.all.mvmax, P.mov[i].y);
    P.order.push_back(i);
  }
  P.all.count = static_cast<int>(lpt.size());
  if (P.order.empty()) P.order.push_back(0);
  if (!P.order_pin.resize(P.order.size()))
    return fail(h, VS_ERR_CUDA, "pinned host allocation failed");
  std::memcpy(P.order_pin.data(), P.order.data(), P.order.size() * sizeof(int));
  if (const char* e = std::getenv("VSCREEN_UPLOAD_TIMING"); e && e[0] == '1') {
    const auto pt4 = std::chrono::steady_clock::now();
    auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    std::fprintf(stderr, "pack_library: pass1 %.2f ms, fill %.2f ms, lpt sort %.2f ms, buckets %.2f ms\n",
                 ms(pt0, pt1), ms(pt1, pt2), ms(pt2, pt3), ms(pt3, pt4));
  }
  return VS_OK;
}

// The incremental torsion flex (docs/SWEEP_V1.md §2.5) moves moving_j
// rigidly about the state's axis j.  That equals re-chaining the torsions
// from the conformer when the topology is a torsion tree: for j < k, either
// moving_k and axis k lie inside moving_j (+ axis j) or both are disjoint
// from moving_j, and no later torsion moves axis j.  Every topology that
// torsion_topology (dock.cpp:234-270) builds from a parsed SMILES graph has
// this property (b is the DFS child of a, moving = b's DFS subtree).
int check_nested(vs_handle* h, const Packed& P) {
  const int n = P.n;
  const int nth = std::max(1, std::min<int>(32, static_cast<int>(std::thread::hardware_concurrency())));
  std::vector<int> bad(nth, -1);
  auto run = [&](int t) {
    const int lo = static_cast<int>(static_cast<long>(n) * t / nth);
    const int hi = static_cast<int>(static_cast<long>(n) * (t + 1) / nth);
    std::array<uint64_t, 2> set[kMaxTors];
    for (int i = lo; i < hi; ++i) {
      const int T = P.meta[i].w;
      if (T < 2) continue;
      const int4* ax = P.axes.data() + P.meta[i].z;
      const uint8_t* mv = P.moving.data() + P.mov[i].x;
      for (int j = 0; j < T; ++j) {
        set[j] = {0ull, 0ull};
        for (int m = 0; m < ax[j].w; ++m)
          set[j][mv[ax[j].z + m] >> 6] |= 1ull << (mv[ax[j].z + m] & 63);
      }
      auto has = [&](int j, int a) { return (set[j][a >> 6] >> (a & 63)) & 1ull; };
      for (int j = 0; j < T; ++j) {
        for (int k = j + 1; k < T; ++k) {
          const bool sub = ((set[k][0] & ~set[j][0]) | (set[k][1] & ~set[j][1])) == 0 &&
                           (has(j, ax[k].x) || ax[k].x == ax[j].x || ax[k].x == ax[j].y) &&
                           (has(j, ax[k].y) || ax[k].y == ax[j].x || ax[k].y == ax[j].y);
          const bool dis = ((set[k][0] & set[j][0]) | (set[k][1] & set[j][1])) == 0 &&
                           !has(j, ax[k].x) && !has(j, ax[k].y);
          if ((!sub && !dis) || has(k, ax[j].x) || has(k, ax[j].y)) {
            bad[t] = i;
            return;
          }
        }
      }
    }
  };
  if (nth == 1 || n < 4096) {
    for (int t = 0; t < nth; ++t) run(t);
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nth; ++t) pool.emplace_back(run, t);
    for (auto& th : pool) th.join();
  }
  for (int t = 0; t < nth; ++t)
    if (bad[t] >= 0)
      return fail(h, VS_ERR_INVALID_ARGUMENT,
                  "ligand " + std::to_string(bad[t]) + ": torsion topology is not a torsion tree");
  return VS_OK;
}

// parts: 1 = the pinned arrays (async DMA, returns at once), 2 = the small
// pageable ones (a pageable H2D waits for the stream), 3 = both.
int upload_packed(vs_handle* h, Packed& P, cudaStream_t st, int parts) {
  auto up = [&](DBuf& d, const void* src, size_t bytes) -> cudaError_t {
    cudaError_t e = d.ensure(bytes);
    if (e != cudaSuccess) return e;
    return cudaMemcpyAsync(d.p, src, bytes, cudaMemcpyHostToDevice, st);
  };
  if (parts & 1) {
    VS_CUDA(h, up(P.d_meta, P.meta.data(), std::max<size_t>(16, P.meta.size() * sizeof(int4))));
    VS_CUDA(h, up(P.d_mov, P.mov.data(), std::max<size_t>(8, P.mov.size() * sizeof(int2))));
    VS_CUDA(h, up(P.d_atoms, P.atoms.data(), P.atoms.size() * sizeof(double4)));
    VS_CUDA(h, up(P.d_axes, P.axes.data(), P.axes.size() * sizeof(int4)));
    VS_CUDA(h, up(P.d_moving, P.moving.data(), P.moving.size()));
  }
  if (!(parts & 2)) return VS_OK;
  VS_CUDA(h, up(P.d_seeds, P.seeds.data(), std::max<size_t>(8, P.seeds.size() * 8)));
  VS_CUDA(h, up(P.d_idr, P.id_rank.data(), std::max<size_t>(4, P.id_rank.size() * 4)));
  VS_CUDA(h, up(P.d_order, P.order_pin.data(), P.order_pin.size() * sizeof(int)));
  return VS_OK;
}

int check_params(vs_handle* h, const vs_dock_params* p) {
  if (p->restarts < 1) return fail(h, VS_ERR_INVALID_ARGUMENT, "restarts must be >= 1");
  if (p->diversity_delta < 0.0)
    return fail(h, VS_ERR_INVALID_ARGUMENT, "diversity_delta must be >= 0");
  if (p->restarts > kMaxRestarts) return fail(h, VS_ERR_CAPACITY, "restarts > 64");
  if (p->flex_angles < 1 || p->flex_angles > kMaxFlexAngles)
    return fail(h, VS_ERR_CAPACITY, "flex_angles must be in [1, 16]");
  if (p->rotations < 1) return fail(h, VS_ERR_INVALID_ARGUMENT, "rotations must be >= 1");
  if (p->flex_passes < 0 || p->keep_top < 0)
    return fail(h, VS_ERR_INVALID_ARGUMENT, "negative flex_passes/keep_top");
  if (p->polish < 0 || p->polish > 2) return fail(h, VS_ERR_INVALID_ARGUMENT, "polish must be 0, 1 or 2");
  return VS_OK;
}

// Fixed rotation set of the sweep: k = 0 identity, k >= 1 the normalized
// 4-normal draw of Rng(seed).split(k) (FP64, then rounded to FP32).
std::vector<float4> rotation_set(int K, uint64_t seed) {
  std::vector<float4> r(static_cast<size_t>(K));
  const HostRng root(seed);
  for (int k = 0; k < K; ++k) {
    if (k == 0) {
      r[0] = float4{1.0f, 0.0f, 0.0f, 0.0f};
      continue;
    }
    HostRng g = root.split(static_cast<uint64_t>(k));
    const double w = g.normal(), x = g.normal(), y = g.normal(), z = g.normal();
    const double n = std::sqrt(w * w + x * x + y * y + z * z);
    r[k] = float4{static_cast<float>(w / n), static_cast<float>(x / n), static_cast<float>(y / n),
                  static_cast<float>(z / n)};
  }
  return r;
}

// Lane order of the rotation sweep (vs_dock.cu sweep_phase): the K rotations
// in groups of 32 (one warp-wide key-cell gather each) that are clusters on
// SO(3), so the 32 poses of one gather put each atom at nearby positions and
// touch fewer distinct 128 B lines of the key map.  Balanced k-means on the
// quaternion similarity |<qa, qb>| (capacity 32 per cluster, greedy
// assignment in order of decreasing similarity, ties by index), seeded by
// farthest-point sampling from rotation 0; fully deterministic.  The sweep's
// result does not depend on this order (argmax ties break on k).
std::vector<int> rotation_order(const std::vector<float4>& r) {
  const int K = static_cast<int>(r.size());
  std::vector<int> perm(static_cast<size_t>(K));
  std::iota(perm.begin(), perm.end(), 0);
  const int G = K / 32;
#ifdef VS_ROT_INDEX_ORDER  // A/B variant: lanes in index order
  return perm;
#endif
  if (G < 2) return perm;
  auto sim = [](const float4& a, const double* c) {
    return std::fabs(a.x * c[0] + a.y * c[1] + a.z * c[2] + a.w * c[3]);
  };
  std::vector<std::array<double, 4>> cent(static_cast<size_t>(G));
  std::vector<int> seeds{0};
  std::vector<double> near(static_cast<size_t>(K), 2.0);
  while (static_cast<int>(seeds.size()) < G) {
    const float4& s0 = r[static_cast<size_t>(seeds.back())];
    const double c0[4] = {s0.x, s0.y, s0.z, s0.w};
    int far = 0;
    for (int k = 0; k < K; ++k) {
      near[k] = std::min(near[k], 1.0 - sim(r[k], c0) + 0.0);
      if (near[k] > near[far]) far = k;
    }
    seeds.push_back(far);
  }
  for (int g = 0; g < G; ++g) {
    const float4& q = r[static_cast<size_t>(seeds[g])];
    cent[g] = {q.x, q.y, q.z, q.w};
  }
  std::vector<int> asg(static_cast<size_t>(K), -1);
  const int cap = 32;
  std::vector<std::pair<double, int>> pairs(static_cast<size_t>(K) * G);
  for (int it = 0; it < 16; ++it) {
    for (int k = 0; k < K; ++k)
      for (int g = 0; g < G; ++g) pairs[static_cast<size_t>(k) * G + g] = {-sim(r[k], cent[g].data()), k * G + g};
    std::sort(pairs.begin(), pairs.end());
    std::fill(asg.begin(), asg.end(), -1);
    std::vector<int> cnt(static_cast<size_t>(G), 0);
    for (const auto& pr : pairs) {
      const int k = pr.second / G, g = pr.second % G;
      if (asg[k] < 0 && cnt[g] < cap) {
        asg[k] = g;
        ++cnt[g];
      }
    }
    for (int g = 0; g < G; ++g) {
      double c[4] = {0, 0, 0, 0};
      for (int k = 0; k < K; ++k) {
        if (asg[k] != g) continue;
        const double d = r[k].x * cent[g][0] + r[k].y * cent[g][1] + r[k].z * cent[g][2] +
                         r[k].w * cent[g][3];
        const double sg = d < 0.0 ? -1.0 : 1.0;
        c[0] += sg * r[k].x;
        c[1] += sg * r[k].y;
        c[2] += sg * r[k].z;
        c[3] += sg * r[k].w;
      }
      const double n = std::sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2] + c[3] * c[3]);
      if (n > 0.0)
        for (int m = 0; m < 4; ++m) cent[g][m] = c[m] / n;
    }
  }
  int o = 0;
  for (int g = 0; g < G; ++g)
    for (int k = 0; k < K; ++k)
      if (asg[k] == g) perm[o++] = k;
  for (int k = 0; k < K; ++k)  // the K mod 32 rotations outside every cluster
    if (asg[k] < 0) perm[o++] = k;
  return perm;
}

}  // namespace

extern "C" {

int vs_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return VS_ERR_INVALID_ARGUMENT;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return VS_ERR_NO_DEVICE;
  }
  if (cudaHostAlloc(out, static_cast<size_t>(std::max<int64_t>(bytes, 1)), cudaHostAllocPortable) !=
      cudaSuccess) {
    cudaGetLastError();
    *out = nullptr;
    return VS_ERR_CUDA;
  }
  return VS_OK;
}

int vs_host_free(void* p) {
  if (p && cudaFreeHost(p) != cudaSuccess) {
    cudaGetLastError();
    return VS_ERR_CUDA;
  }
  return VS_OK;
}

int vs_create(int device, vs_handle** out) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return VS_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= count) return VS_ERR_NO_DEVICE;
  auto* h = new vs_handle;
  h->device = device;
  cudaSetDevice(device);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  h->sms = prop.multiProcessorCount;
  std::snprintf(h->name, sizeof(h->name), "%s", prop.name);
  cudaDeviceGetAttribute(&h->clock_khz, cudaDevAttrClockRate, device);
  if (cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking) != cudaSuccess) {
    delete h;
    return VS_ERR_CUDA;
  }
  cudaEventCreate(&h->ev0);
  cudaEventCreate(&h->ev1);
  cudaEventCreateWithFlags(&h->done, cudaEventDisableTiming);
  h->last = h->own;
  *out = h;
  return VS_OK;
}

void vs_destroy(vs_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->own);
  if (h->copy) {
    cudaStreamSynchronize(h->copy);
    cudaStreamDestroy(h->copy);
  }
  for (Packed& P : h->libs) P.release();
  h->rpack.release();
  h->xpack.release();
  for (DBuf& b : h->xbuf) b.release();
  for (PackScratch& x : h->ps) x.release();
  if (h->key_tex) cudaDestroyTextureObject(h->key_tex);
  for (DBuf& b : h->rbuf) b.release();
  for (DBuf& b : h->ebuf) b.release();
  for (DBuf* b : {&h->d_sites, &h->d_softtab, &h->d_sites64, &h->d_maps, &h->d_surv, &h->d_surv_tors, &h->d_all, &h->d_all_tors,
                  &h->d_best, &h->d_nkept, &h->d_nsurv, &h->d_keys, &h->d_rots, &h->d_topk_a, &h->d_topk_b, &h->d_stats})
    b->release();
  h->sg.release();
  for (int k = 0; k < 2; ++k) {
    h->pipe_sg[k].release();
    h->pipe_lib[k].release();
    if (h->pipe_s[k]) cudaStreamDestroy(h->pipe_s[k]);
  }
  if (h->pipe_in) cudaStreamDestroy(h->pipe_in);
  if (h->pipe_out) cudaStreamDestroy(h->pipe_out);
  for (cudaEvent_t e : h->pipe_ev) cudaEventDestroy(e);
  cudaEventDestroy(h->ev0);
  cudaEventDestroy(h->ev1);
  cudaEventDestroy(h->done);
  vs_comm_destroy(h);
  h->d_gather.release();
  for (cudaEvent_t e : h->pev) cudaEventDestroy(e);
  for (cudaStream_t x : h->fork) cudaStreamDestroy(x);
  for (cudaEvent_t e : h->fork_ev) cudaEventDestroy(e);
  if (h->rev0) cudaEventDestroy(h->rev0);
  if (h->rev1) cudaEventDestroy(h->rev1);
  cudaStreamDestroy(h->own);
  delete h;
}

const char* vs_last_error(const vs_handle* h) { return h ? h->err.c_str() : "null handle"; }

int vs_device_info(const vs_handle* h, char* name, int32_t* sm_count, int32_t* clock_khz) {
  if (name) std::snprintf(name, 256, "%s", h->name);
  if (sm_count) *sm_count = h->sms;
  if (clock_khz) *clock_khz = h->clock_khz;
  return VS_OK;
}

int vs_set_pocket(vs_handle* h, const vs_pocket* p, double spacing, double pad) {
  cudaSetDevice(h->device);
  VS_CUDA(h, quiesce(h));
  cudaStream_t st = h->own;
  std::vector<SiteF> sites;
  int counts[3] = {0, 0, 0};
  for (int kind = 0; kind < 3; ++kind) {
    for (int s = 0; s < p->n_sites; ++s) {
      const vs_site& v = p->sites[s];
      if (v.kind < 0 || v.kind > 2) return fail(h, VS_ERR_POCKET, "unknown site kind");
      if (!(v.sigma > 0.0)) return fail(h, VS_ERR_POCKET, "site sigma must be > 0");
      if (v.kind != kind) continue;
      SiteF f{};
      f.cx = static_cast<float>(v.center[0]);
      f.cy = static_cast<float>(v.center[1]);
      f.cz = static_cast<float>(v.center[2]);
      f.w = static_cast<float>(v.weight);
      f.inv2s2 = static_cast<float>(1.0 / (2.0 * v.sigma * v.sigma));
      sites.push_back(f);
      ++counts[kind];
    }
  }
  if (p->clash_penalty < 0.0) return fail(h, VS_ERR_POCKET, "clash_penalty must be >= 0");
  if (sites.empty()) sites.push_back(SiteF{});
  {
    std::vector<SiteD> sd(std::max(p->n_sites, 1));
    for (int s = 0; s < p->n_sites; ++s) {
      const vs_site& v = p->sites[s];
      sd[s] = SiteD{v.center[0], v.center[1], v.center[2], v.weight,
                    1.0 / (2.0 * v.sigma * v.sigma), v.kind, 0};
    }
    VS_CUDA(h, h->d_sites64.ensure(sd.size() * sizeof(SiteD)));
    VS_CUDA(h, cudaMemcpyAsync(h->d_sites64.p, sd.data(), sd.size() * sizeof(SiteD),
                               cudaMemcpyHostToDevice, st));
    VS_CUDA(h, cudaStreamSynchronize(st));
    h->n_sites64 = p->n_sites;
    for (int c = 0; c < 3; ++c) {
      h->box_lo[c] = p->lo[c];
      h->box_hi[c] = p->hi[c];
    }
    h->r64 = p->clash_radius;
    h->lam64 = p->clash_penalty;
  }
  VS_CUDA(h, h->d_sites.ensure(sites.size() * sizeof(SiteF)));
  VS_CUDA(h, cudaMemcpyAsync(h->d_sites.p, sites.data(), sites.size() * sizeof(SiteF),
                             cudaMemcpyHostToDevice, st));
  PocketDev& pk = h->pk;
  pk = PocketDev{};
  for (int c = 0; c < 3; ++c) {
    pk.lo[c] = static_cast<float>(p->lo[c]);
    pk.hi[c] = static_cast<float>(p->hi[c]);
    pk.lo_d[c] = p->lo[c];
    pk.hi_d[c] = p->hi[c];
  }
  h->empty_bounds = p->hi[0] <= p->lo[0] || p->hi[1] <= p->lo[1] || p->hi[2] <= p->lo[2];
  pk.r = static_cast<float>(p->clash_radius);
  pk.lam = static_cast<float>(p->clash_penalty);
  const float rr = pk.r + 3.0f;
  pk.cut2 = rr * rr;
  pk.cut2_d = static_cast<double>(pk.cut2);
  VS_CUDA(h, h->d_softtab.ensure(sizeof(float2) * kSoftN));
  VS_CUDA(h, launch_softtab(st, pk.r, pk.cut2, h->d_softtab.as<float2>()));
  ++h->launches;
  pk.soft_tab = h->d_softtab.as<const float2>();
  pk.soft_inv_h = static_cast<float>(kSoftN) / pk.cut2;
  pk.n_steric = counts[0];
  pk.n_hbond = counts[1];
  pk.n_lipo = counts[2];
  pk.sites = h->d_sites.as<const SiteF>();
  pk.grid_mode = 0;
  h->gdims[0] = h->gdims[1] = h->gdims[2] = 0;
  if (spacing > 0.0 && !h->empty_bounds) {
    GridDev& g = pk.grid;
    g.h = static_cast<float>(spacing);
    g.inv_h = 1.0f / g.h;
    g.ox = static_cast<float>(p->lo[0] - pad);
    g.oy = static_cast<float>(p->lo[1] - pad);
    g.oz = static_cast<float>(p->lo[2] - pad);
    int* dims[3] = {&g.nx, &g.ny, &g.nz};
    for (int c = 0; c < 3; ++c)
      *dims[c] = static_cast<int>(std::ceil((p->hi[c] - p->lo[c] + 2.0 * pad) / spacing)) + 1;
    g.cx = g.nx - 1;
    g.cxy = (g.nx - 1) * (g.ny - 1);
    const size_t nodes = static_cast<size_t>(g.nx) * g.ny * g.nz;
    const size_t cells = static_cast<size_t>(g.nx - 1) * (g.ny - 1) * (g.nz - 1);
    // cell arrays 256 B aligned: each 32 B cell is one 256-bit load (ldg_cell)
    const size_t node_bytes = (4 * nodes * sizeof(float) + 255) & ~size_t(255);
    VS_CUDA(h, h->d_maps.ensure(node_bytes + 4 * cells * 2 * sizeof(float4) + 512));
    float* m = h->d_maps.as<float>();
    float4* c = reinterpret_cast<float4*>(static_cast<char*>(h->d_maps.p) + node_bytes);
    g.steric = m;
    g.hbond = m + nodes;
    g.lipo = m + 2 * nodes;
    g.steric_c = c;
    g.hbond_c = c + 2 * cells;
    g.lipo_c = c + 4 * cells;
    g.key = m + 3 * nodes;
    g.key_c = c + 6 * cells;
    // the FP16 key cells at a 512 B boundary (texture alignment) inside the
    // key_c region, which they replace
    g.key_h = reinterpret_cast<const uint4*>(
        (reinterpret_cast<uintptr_t>(c + 6 * cells) + 511) & ~uintptr_t(511));
    if (h->key_tex) cudaDestroyTextureObject(h->key_tex);
    h->key_tex = 0;
    {
      cudaResourceDesc rd{};
      rd.resType = cudaResourceTypeLinear;
      rd.res.linear.devPtr = const_cast<uint4*>(g.key_h);
      rd.res.linear.desc = cudaCreateChannelDesc<uint4>();
      rd.res.linear.sizeInBytes = cells * sizeof(uint4);
      cudaTextureDesc td{};
      td.readMode = cudaReadModeElementType;
      VS_CUDA(h, cudaCreateTextureObject(&h->key_tex, &rd, &td, nullptr));
    }
    g.key_tex = h->key_tex;
    VS_CUDA(h, launch_grid(st, pk, m, m + nodes, m + 2 * nodes, m + 3 * nodes, c));
    h->launches += 5;
    pk.grid_mode = 1;
    h->gdims[0] = g.nx;
    h->gdims[1] = g.ny;
    h->gdims[2] = g.nz;
  }
  VS_CUDA(h, cudaStreamSynchronize(st));
  h->has_pocket = true;
  return VS_OK;
}

int vs_grid_info(const vs_handle* h, int32_t dims[3], float origin[3], float* spacing) {
  for (int c = 0; c < 3; ++c) dims[c] = h->gdims[c];
  origin[0] = h->pk.grid.ox;
  origin[1] = h->pk.grid.oy;
  origin[2] = h->pk.grid.oz;
  *spacing = h->pk.grid.h;
  return h->pk.grid_mode ? VS_OK : VS_ERR_STATE;
}

int vs_grid_fetch(vs_handle* h, float* steric, float* hbond, float* lipo) {
  if (!h->pk.grid_mode) return fail(h, VS_ERR_STATE, "no grid maps");
  const size_t nodes = static_cast<size_t>(h->gdims[0]) * h->gdims[1] * h->gdims[2];
  const float* m = h->d_maps.as<float>();
  VS_CUDA(h, cudaMemcpy(steric, m, nodes * 4, cudaMemcpyDeviceToHost));
  VS_CUDA(h, cudaMemcpy(hbond, m + nodes, nodes * 4, cudaMemcpyDeviceToHost));
  VS_CUDA(h, cudaMemcpy(lipo, m + 2 * nodes, nodes * 4, cudaMemcpyDeviceToHost));
  return VS_OK;
}

}  // extern "C"

namespace {

// The library packer on the device (north-star subsystem 1, vs_pack.cu):
// the caller's arrays DMA'd as given (pinned memory: full link rate), the
// SoA layout, size classes, checks and LPT order built by kernels on `st`,
// one synchronize to read back the outcome.  Leaves P ready for
// launch_packed (P.all over P.d_order, P.cls on the host).  The count
// checks run on the host first (they size the transfers).
// gpu_pack in two halves: pack_issue enqueues the transfers and kernels
// (async), pack_finish synchronizes `st` and reads back the outcome; a
// caller can do host work in between
int pack_issue(vs_handle* h, const vs_library* L, const vs_size_class* classes, int nc, Packed& P,
               cudaStream_t st, PackPending& pp, int slot = 0);
int pack_finish(vs_handle* h, Packed& P, cudaStream_t st, const PackPending& pp);

int gpu_pack(vs_handle* h, const vs_library* L, const vs_size_class* classes, int nc, Packed& P,
             cudaStream_t st, int slot = 0) {
  PackPending pp;
  const int rc = pack_issue(h, L, classes, nc, P, st, pp, slot);
  if (rc) return rc;
  return pack_finish(h, P, st, pp);
}

int pack_issue(vs_handle* h, const vs_library* L, const vs_size_class* classes, int nc, Packed& P,
               cudaStream_t st, PackPending& pp, int slot) {
  PackScratch& X = h->ps[slot];
  const int n = L->n_ligands;
  if (n < 0) return fail(h, VS_ERR_INVALID_ARGUMENT, "negative ligand count");
  long A = 0, T = 0, M = 0;
  for (int i = 0; i < n; ++i) {  // pass 1 of pack_library, same precedence
    const int N = L->n_atoms[i], t = L->n_tors[i];
    if (N < 1) return fail(h, VS_ERR_ATOM_COUNT, "conformer has no atoms (ligand " + std::to_string(i) + ")");
    if (N > kMaxAtoms || t > kMaxTors)
      return fail(h, VS_ERR_CAPACITY, "ligand " + std::to_string(i) + " exceeds GPU limits");
    if (t < 0) return fail(h, VS_ERR_INVALID_ARGUMENT, "negative torsion count");
    A += N;
    T += t;
  }
  for (long j = 0; j < T; ++j) M += std::max(0, L->moving_count[j]);
  const size_t n1 = static_cast<size_t>(n) + 1, t1 = static_cast<size_t>(T) + 1;
  // raw arrays (as given) -> device
  DBuf* r = X.raw;
  auto up = [&](DBuf& d, const void* src, size_t bytes) -> cudaError_t {
    cudaError_t e = d.ensure(std::max<size_t>(bytes, 16));
    if (e == cudaSuccess && bytes > 0 && src)
      e = cudaMemcpyAsync(d.p, src, bytes, cudaMemcpyHostToDevice, st);
    return e;
  };
  VS_CUDA(h, up(r[0], L->n_atoms, n * 4ul));
  VS_CUDA(h, up(r[1], L->n_tors, n * 4ul));
  VS_CUDA(h, up(r[2], L->rot_bonds, L->rot_bonds ? n * 4ul : 0));
  VS_CUDA(h, up(r[3], L->coords, A * 24ul));
  VS_CUDA(h, up(r[4], L->atom_class, A * 4ul));
  VS_CUDA(h, up(r[5], L->axis_a, T * 4ul));
  VS_CUDA(h, up(r[6], L->axis_b, T * 4ul));
  VS_CUDA(h, up(r[7], L->moving_count, T * 4ul));
  VS_CUDA(h, up(r[8], L->moving, M * 4ul));
  VS_CUDA(h, up(P.d_seeds, L->seeds, L->seeds ? n * 8ul : 0));
  VS_CUDA(h, up(P.d_idr, L->id_rank, L->id_rank ? n * 4ul : 0));
  // classes (int4 each) ride in the stats buffer's tail
  DBuf* w = X.pwork;
  VS_CUDA(h, w[0].ensure(n1 * 8));   // cnt_a
  VS_CUDA(h, w[1].ensure(n1 * 8));   // cnt_t
  VS_CUDA(h, w[2].ensure(t1 * 8));   // cnt_m
  VS_CUDA(h, w[3].ensure(n1 * 8));   // cnt_p
  VS_CUDA(h, w[4].ensure(n1 * 8));   // aoff
  VS_CUDA(h, w[5].ensure(n1 * 8));   // toff
  VS_CUDA(h, w[6].ensure(t1 * 8));   // msrc
  VS_CUDA(h, w[7].ensure(n1 * 8));   // moff
  VS_CUDA(h, w[8].ensure(n1 * 4));   // cls
  VS_CUDA(h, w[9].ensure(n1 * 4));   // key
  VS_CUDA(h, w[10].ensure(n1 * 4));  // key_sorted
  VS_CUDA(h, w[11].ensure(n1 * 4));  // idx
  if (nc > kPkMaxClasses) return fail(h, VS_ERR_CAPACITY, "more than 64 size classes");
  VS_CUDA(h, w[12].ensure(4 * kPkClasses + 16 * static_cast<size_t>(std::max(nc, 1))));
  const size_t tmp = pack_temp_bytes(n, T);
  VS_CUDA(h, X.ptemp.ensure(tmp));
  // packed outputs: M raw entries -> at most M + 15 n padded bytes
  VS_CUDA(h, P.d_meta.ensure(std::max<size_t>(16, n * 16ul)));
  VS_CUDA(h, P.d_mov.ensure(std::max<size_t>(8, n * 8ul)));
  VS_CUDA(h, P.d_atoms.ensure(std::max<size_t>(32, A * 32ul)));
  VS_CUDA(h, P.d_axes.ensure(std::max<size_t>(16, T * 16ul)));
  VS_CUDA(h, P.d_moving.ensure(std::max<size_t>(16, M + 15ul * n + 16)));
  VS_CUDA(h, P.d_seeds.ensure(std::max<size_t>(8, n * 8ul)));
  VS_CUDA(h, P.d_idr.ensure(std::max<size_t>(4, n * 4ul)));
  VS_CUDA(h, P.d_order.ensure(std::max<size_t>(4, n * 4ul)));
  int* stats = w[12].as<int>();
  unsigned long long* err = reinterpret_cast<unsigned long long*>(stats + kPkErr);
  int4* dcls = reinterpret_cast<int4*>(stats + kPkClasses);
  const size_t cls_at = kPkClasses + 4 * static_cast<size_t>(std::max(nc, 1));  // host: cls after
  if (!X.pk_host.resize(cls_at + n1)) return fail(h, VS_ERR_CUDA, "pinned host allocation failed");
  int* hs = X.pk_host.data();
  std::memset(hs, 0, kPkClasses * sizeof(int));
  *reinterpret_cast<unsigned long long*>(hs + kPkErr) = ~0ull;
  for (int k = 0; k < nc; ++k)
    reinterpret_cast<int4*>(hs + kPkClasses)[k] =
        int4{classes[k].atom_lo, classes[k].atom_hi, classes[k].rot_lo, classes[k].rot_hi};
  VS_CUDA(h, cudaMemcpyAsync(stats, hs, (kPkClasses + 4 * std::max(nc, 0)) * sizeof(int),
                             cudaMemcpyHostToDevice, st));
  PackIn in;
  in.n = n;
  in.total_atoms = A;
  in.total_tors = T;
  in.total_moving = M;
  in.n_atoms = r[0].as<const int>();
  in.n_tors = r[1].as<const int>();
  in.rot_bonds = L->rot_bonds ? r[2].as<const int>() : nullptr;
  in.coords = r[3].as<const double>();
  in.atom_class = r[4].as<const int>();
  in.axis_a = r[5].as<const int>();
  in.axis_b = r[6].as<const int>();
  in.moving_count = r[7].as<const int>();
  in.moving = r[8].as<const int>();
  in.seeds = L->seeds ? P.d_seeds.as<const unsigned long long>() : nullptr;
  in.id_rank = L->id_rank ? P.d_idr.as<const unsigned>() : nullptr;
  in.classes = dcls;
  PackWork pw{w[0].as<long>(), w[1].as<long>(), w[2].as<long>(), w[3].as<long>(),
              w[4].as<long>(), w[5].as<long>(), w[6].as<long>(), w[7].as<long>(),
              w[8].as<int>(),  w[9].as<unsigned>(), w[10].as<unsigned>(), w[11].as<int>(),
              stats, err};
  PackDev out{P.d_meta.as<int4>(), P.d_mov.as<int2>(), P.d_atoms.as<double4>(),
              P.d_axes.as<int4>(), P.d_moving.as<uint8_t>(), P.d_seeds.as<unsigned long long>(),
              P.d_idr.as<unsigned>(), P.d_order.as<int>()};
  VS_CUDA(h, pack_stage1(st, in, pw, classes ? nc : 0));
  VS_CUDA(h, pack_stage2(st, in, pw, out, X.ptemp.p, tmp));
  h->launches += 9;
  VS_CUDA(h, cudaMemcpyAsync(hs, stats, kPkClasses * sizeof(int), cudaMemcpyDeviceToHost, st));
  VS_CUDA(h, cudaMemcpyAsync(hs + cls_at, pw.cls, n * 4ul, cudaMemcpyDeviceToHost, st));
  pp.n = n;
  pp.nc = nc;
  pp.A = A;
  pp.T = T;
  pp.cls_at = cls_at;
  pp.classes = classes != nullptr;
  pp.slot = slot;
  return VS_OK;
}

int pack_finish(vs_handle* h, Packed& P, cudaStream_t st, const PackPending& pp) {
  VS_CUDA(h, cudaStreamSynchronize(st));
  const int n = pp.n, nc = pp.nc;
  const long A = pp.A, T = pp.T;
  const size_t cls_at = pp.cls_at;
  const int* hs = h->ps[pp.slot].pk_host.data();
  const unsigned long long ek = *reinterpret_cast<const unsigned long long*>(hs + kPkErr);
  if (ek != ~0ull) {
    const int code = static_cast<int>(ek & 0xff);
    const long lig = static_cast<long>((ek >> 8) & 0xffffffffffull);
    const std::string at = " (ligand " + std::to_string(lig) + ")";
    if (code == kPkTopology) return fail(h, VS_ERR_ATOM_COUNT, "torsion topology does not fit conformer" + at);
    if (code == kPkNotTree)
      return fail(h, VS_ERR_INVALID_ARGUMENT, "ligand " + std::to_string(lig) + ": torsion topology is not a torsion tree");
    if (code == kPkCapacity) return fail(h, VS_ERR_CAPACITY, "ligand exceeds GPU limits" + at);
    return fail(h, VS_ERR_ATOM_COUNT, "invalid ligand counts" + at);
  }
  P.n = n;
  P.total_atoms = A;
  P.total_tors = T;
  P.cls.assign(hs + cls_at, hs + cls_at + n);
  P.all = Bucket{};
  P.all.start = 0;
  P.all.count = hs[3];
  P.all.nmax = std::max(P.all.nmax, hs[0]);
  P.all.tmax = std::max(P.all.tmax, hs[1]);
  P.all.mvmax = std::max(P.all.mvmax, hs[2]);
  // per-class bounds (the rescoring launches, one per class); members are
  // listed by the caller from P.cls
  const int ncls = (pp.classes && nc > 0) ? nc : 6;
  P.on_device = true;
  P.buckets.assign(static_cast<size_t>(ncls), Bucket{});
  for (int c = 0; c < ncls; ++c) {
    Bucket& b = P.buckets[static_cast<size_t>(c)];
    b.nmax = std::max(b.nmax, hs[4 + 3 * c]);
    b.tmax = std::max(b.tmax, hs[5 + 3 * c]);
    b.mvmax = std::max(b.mvmax, hs[6 + 3 * c]);
  }
  return VS_OK;
}

bool device_pack_enabled() {
  const char* e = std::getenv("VSCREEN_HOST_PACK");
  return !(e && e[0] == '1');
}

}  // namespace

extern "C" {

int vs_upload_library(vs_handle* h, const vs_library* L, const vs_size_class* classes,
                      int32_t nc) {
  cudaSetDevice(h->device);
  VS_CUDA(h, quiesce(h));  // a dock on a caller stream may still read the library
  if (h->spare_pending) {  // a prefetch not taken: drain and drop it
    VS_CUDA(h, cudaStreamSynchronize(h->copy));
    h->spare_pending = false;
  }
  h->has_lib = false;
  h->lib_lists_n = -1;
  h->has_results = false;
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  if (device_pack_enabled()) {  // the device packer (VSCREEN_HOST_PACK=1: the host one)
    const int rc = gpu_pack(h, L, classes, nc, h->libs[h->cur], h->own, h->cur);
    if (rc) return rc;
    if (const char* e = std::getenv("VSCREEN_UPLOAD_TIMING"); e && e[0] == '1')
      std::fprintf(stderr, "vs_upload_library: device pack (raw H2D + kernels) %.2f ms\n",
                   std::chrono::duration<double, std::milli>(clk::now() - t0).count());
    h->has_lib = true;
    return VS_OK;
  }
  // the pinned arrays' DMA runs under the bucketing and the torsion-tree
  // check; a failure drains it before returning (the next pack rewrites them)
  int rc = pack_library(h, L, classes, nc, h->libs[h->cur], h->own);
  if (rc) {
    cudaStreamSynchronize(h->own);
    return rc;
  }
  const auto t1 = clk::now();
  rc = check_nested(h, h->libs[h->cur]);
  if (rc) {
    cudaStreamSynchronize(h->own);
    return rc;
  }
  const auto t2 = clk::now();
  rc = upload_packed(h, h->libs[h->cur], h->own, 2);
  if (rc) return rc;
  VS_CUDA(h, cudaStreamSynchronize(h->own));
  const auto t3 = clk::now();
  if (const char* e = std::getenv("VSCREEN_UPLOAD_TIMING"); e && e[0] == '1') {
    auto ms = [](clk::time_point a, clk::time_point b) {
      return std::chrono::duration<double, std::milli>(b - a).count();
    };
    std::fprintf(stderr, "vs_upload_library: pack %.2f ms, torsion-tree check (under the DMA) %.2f ms, rest of H2D %.2f ms\n",
                 ms(t0, t1), ms(t1, t2), ms(t2, t3));
  }
  h->has_lib = true;
  return VS_OK;
}

}  // extern "C"

namespace {

// the rotation set and the sweep's lane order, uploaded when they change
int ensure_rots(vs_handle* h, const vs_dock_params* prm, cudaStream_t st) {
  if (h->rots_k == prm->rotations && h->rots_seed == prm->rotation_seed) return VS_OK;
  // the K rotations in index order, the same in the sweep's lane order,
  // then the lane order itself
  const auto rs = rotation_set(prm->rotations, prm->rotation_seed);
  const auto perm = rotation_order(rs);
  std::vector<float4> rp(rs.size());
  for (size_t p = 0; p < rs.size(); ++p) rp[p] = rs[static_cast<size_t>(perm[p])];
  const size_t rb = rs.size() * sizeof(float4);
  std::vector<unsigned char> blob(2 * rb + perm.size() * sizeof(int));
  std::memcpy(blob.data(), rs.data(), rb);
  std::memcpy(blob.data() + rb, rp.data(), rb);
  std::memcpy(blob.data() + 2 * rb, perm.data(), perm.size() * sizeof(int));
  VS_CUDA(h, h->d_rots.ensure(blob.size()));
  VS_CUDA(h, cudaMemcpyAsync(h->d_rots.p, blob.data(), blob.size(), cudaMemcpyHostToDevice, st));
  VS_CUDA(h, cudaStreamSynchronize(st));
  h->rots_k = prm->rotations;
  h->rots_seed = prm->rotation_seed;
  return VS_OK;
}

// result arrays for n ligands / tt torsions, cleared on `st`: unused
// survivor / kept slots read as zeros (not a previous run's poses), keys ~0
int prepare_results(vs_handle* h, int n, long tt, const vs_dock_params* prm, cudaStream_t st) {
  const size_t nn = static_cast<size_t>(std::max(n, 1));
  const size_t R = static_cast<size_t>(prm->restarts), KT = static_cast<size_t>(std::max(prm->keep_top, 1));
  const size_t nt = static_cast<size_t>(std::max<long>(1, tt));
  VS_CUDA(h, h->d_surv.ensure(nn * KT * sizeof(PoseOut)));
  VS_CUDA(h, h->d_surv_tors.ensure(nt * KT * 4));
  if (prm->write_all_poses) {
    VS_CUDA(h, h->d_all.ensure(nn * R * sizeof(PoseOut)));
    VS_CUDA(h, h->d_all_tors.ensure(nt * R * 4));
  }
  VS_CUDA(h, h->d_best.ensure(nn * 4));
  VS_CUDA(h, h->d_nkept.ensure(nn * 4));
  VS_CUDA(h, h->d_nsurv.ensure(nn * 4));
  VS_CUDA(h, h->d_keys.ensure(nn * 8));
  VS_CUDA(h, h->d_stats.ensure(kStats * sizeof(unsigned long long)));
  VS_CUDA(h, cudaMemsetAsync(h->d_stats.p, 0, kStats * sizeof(unsigned long long), st));
  VS_CUDA(h, cudaMemsetAsync(h->d_keys.p, 0xff, nn * 8, st));
  VS_CUDA(h, cudaMemsetAsync(h->d_surv.p, 0, nn * KT * sizeof(PoseOut), st));
  VS_CUDA(h, cudaMemsetAsync(h->d_surv_tors.p, 0, nt * KT * 4, st));
  if (prm->write_all_poses) {
    VS_CUDA(h, cudaMemsetAsync(h->d_all.p, 0, nn * R * sizeof(PoseOut), st));
    VS_CUDA(h, cudaMemsetAsync(h->d_all_tors.p, 0, nt * R * 4, st));
  }
  VS_CUDA(h, cudaMemsetAsync(h->d_nkept.p, 0, nn * 4, st));
  VS_CUDA(h, cudaMemsetAsync(h->d_nsurv.p, 0, nn * 4, st));
  return VS_OK;
}

// the result arrays seen from ligand b (torsion offset tb) on: a chunk of a
// pipelined dock writes its own disjoint slice
DockOut results_view(vs_handle* h, const vs_dock_params* prm, long b, long tb) {
  const long R = prm->restarts, KT = prm->keep_top;
  DockOut out;
  out.surv = h->d_surv.as<PoseOut>() + b * KT;
  out.surv_tors = h->d_surv_tors.as<float>() + tb * KT;
  out.all = prm->write_all_poses ? h->d_all.as<PoseOut>() + b * R : nullptr;
  out.all_tors = prm->write_all_poses ? h->d_all_tors.as<float>() + tb * R : nullptr;
  out.best = h->d_best.as<float>() + b;
  out.n_kept = h->d_nkept.as<int>() + b;
  out.n_surv = h->d_nsurv.as<int>() + b;
  out.keys = h->d_keys.as<unsigned long long>() + b;
  out.stats = h->d_stats.as<unsigned long long>();
  return out;
}

// one launch per phase and restart over P's global LPT queue (every size
// bucket), shared memory sized for its largest ligand, the per-ligand state
// in `sg`; per-launch event pairs when `phases`
int launch_packed(vs_handle* h, const Packed& P, const vs_dock_params* prm, cudaStream_t st,
                  StageSet& sg, const DockOut& out, bool phases) {
  const Bucket& b = P.all;
  if (b.count == 0) return VS_OK;
  const size_t smem = stage_smem_per_block(b.nmax, b.tmax, b.mvmax);
  if (smem > 227 * 1024) return fail(h, VS_ERR_CAPACITY, "ligands need too much shared memory");
  const int R = prm->restarts;
  VS_CUDA(h, sg.ensure(std::max<size_t>(1, static_cast<size_t>(P.total_atoms)),
                       static_cast<size_t>(std::max<long>(1, P.total_tors)),
                       static_cast<size_t>(std::max(P.n, 1)), static_cast<size_t>(R)));
  VS_CUDA(h, cudaMemsetAsync(sg.counters.p, 0, 320 * sizeof(int), st));
  DockParams dp;
  dp.R = R;
  dp.K = prm->rotations;
  dp.A = prm->flex_angles;
  dp.F = prm->flex_passes;
  dp.keep_top = prm->keep_top;
  dp.write_all = prm->write_all_poses ? 1 : 0;
  dp.delta = static_cast<float>(prm->diversity_delta);
  dp.min_score = prm->min_score;
  dp.polish = prm->polish;
  cudaEvent_t* evs = nullptr;
  int* kinds = nullptr;
  if (phases) {
    const size_t npairs = 4 * static_cast<size_t>(R) + 1;  // start, sweep, flex, polish; finish
    while (h->pev.size() < 2 * npairs) {
      cudaEvent_t e;
      VS_CUDA(h, cudaEventCreate(&e));
      h->pev.push_back(e);
    }
    h->pkind.assign(npairs, -1);  // -1: no launch recorded in this slot
    evs = h->pev.data();
    kinds = h->pkind.data();
  }
  const float4* rots = h->d_rots.as<const float4>();
  const float4* rots_p = rots + prm->rotations;
  const int* perm = reinterpret_cast<const int*>(rots_p + prm->rotations);
  VS_CUDA(h, launch_staged(h->pk.grid_mode != 0, h->sms, st, P.dev(), h->pk, rots, rots_p, perm,
                           dp, P.d_order.as<int>() + b.start, b.count, sg.counters.as<int>(),
                           b.nmax, b.tmax, b.mvmax, sg.bufs(), out, &h->launches, evs, kinds));
  return VS_OK;
}

}  // namespace

extern "C" {

int vs_dock(vs_handle* h, const vs_dock_params* prm, void* stream) {
  cudaSetDevice(h->device);
  if (!h->has_pocket) return fail(h, VS_ERR_STATE, "no pocket");
  if (!h->has_lib) return fail(h, VS_ERR_STATE, "no library");
  if (h->empty_bounds) return fail(h, VS_ERR_EMPTY_BOUNDS, "pocket bounds box is empty");
  int rc = check_params(h, prm);
  if (rc) return rc;
  cudaStream_t st = pick(h, stream);
  VS_CUDA(h, after_prev(h, st));
  const Packed& P = h->libs[h->cur];
  rc = ensure_rots(h, prm, st);
  if (rc) return rc;
  rc = prepare_results(h, P.n, P.total_tors, prm, st);
  if (rc) return rc;
  VS_CUDA(h, cudaEventRecord(h->ev0, st));
  rc = launch_packed(h, P, prm, st, h->sg, results_view(h, prm, 0, 0), true);
  if (rc) return rc;
  h->staged_run = true;
  VS_CUDA(h, cudaEventRecord(h->ev1, st));
  VS_CUDA(h, mark_done(h, st));
  h->timed = true;
  h->last_prm = *prm;
  h->has_results = true;
  h->res_n = P.n;
  h->res_cls = P.cls;
  h->res_tors = P.total_tors;
  return VS_OK;
}

double vs_last_dock_ms(const vs_handle* h) {
  if (!h->timed) return -1.0;
  cudaEventSynchronize(h->ev1);
  float ms = 0.0f;
  cudaEventElapsedTime(&ms, h->ev0, h->ev1);
  return ms;
}

uint64_t vs_launch_count(const vs_handle* h) { return h->launches; }

double vs_last_rescore_ms(const vs_handle* h) { return h->rescore_ms; }

int vs_last_phase_ms(vs_handle* h, double out[4]) {
  if (!h->timed) return fail(h, VS_ERR_STATE, "no dock has run");
  for (int k = 0; k < 4; ++k) out[k] = 0.0;
  VS_CUDA(h, cudaEventSynchronize(h->ev1));
  if (!h->staged_run) {
    out[2] = vs_last_dock_ms(h);
    return VS_OK;
  }
  for (size_t i = 0; i < h->pkind.size(); ++i) {
    if (h->pkind[i] < 0) continue;
    float ms = 0.0f;
    VS_CUDA(h, cudaEventElapsedTime(&ms, h->pev[2 * i], h->pev[2 * i + 1]));
    out[h->pkind[i] == 4 ? 2 : h->pkind[i]] += ms;  // polish counted with flex+keep
  }
  return VS_OK;
}

int vs_last_phase_ms_ex(vs_handle* h, double* out, int32_t n) {
  if (!h->timed) return fail(h, VS_ERR_STATE, "no dock has run");
  double v[5] = {0, 0, 0, 0, 0};
  VS_CUDA(h, cudaEventSynchronize(h->ev1));
  if (!h->staged_run) {
    v[2] = vs_last_dock_ms(h);
  } else {
    for (size_t i = 0; i < h->pkind.size(); ++i) {
      if (h->pkind[i] < 0) continue;
      float ms = 0.0f;
      VS_CUDA(h, cudaEventElapsedTime(&ms, h->pev[2 * i], h->pev[2 * i + 1]));
      v[h->pkind[i]] += ms;
    }
  }
  const int k = std::max(0, std::min<int>(n, 5));
  for (int i = 0; i < k; ++i) out[i] = v[i];
  return k;
}

int vs_last_stats(vs_handle* h, uint64_t out[8]) {
  if (!h->has_results) return fail(h, VS_ERR_STATE, "no results");
  VS_CUDA(h, cudaStreamSynchronize(h->last));
  VS_CUDA(h, cudaMemcpy(out, h->d_stats.p, 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return VS_OK;
}

int vs_last_stats_ex(vs_handle* h, uint64_t* out, int32_t n) {
  if (!h->has_results) return fail(h, VS_ERR_STATE, "no results");
  if (n < 0) return fail(h, VS_ERR_INVALID_ARGUMENT, "negative count");
  const int m = n < kStats ? n : kStats;
  VS_CUDA(h, cudaStreamSynchronize(h->last));
  VS_CUDA(h, cudaMemcpy(out, h->d_stats.p, m * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return m;
}

int vs_measure_peaks(vs_handle* h, double* fp32, double* fp64, double* xu) {
  cudaSetDevice(h->device);
  VS_CUDA(h, cudaDeviceSynchronize());
  if (fp32) *fp32 = measure_peak(0, h->sms);
  if (fp64) *fp64 = measure_peak(1, h->sms);
  if (xu) *xu = measure_peak(2, h->sms);
  VS_CUDA(h, cudaGetLastError());
  return VS_OK;
}

int vs_measure_gather_peak(vs_handle* h, double* loads_per_s) {
  cudaSetDevice(h->device);
  VS_CUDA(h, cudaDeviceSynchronize());
  if (loads_per_s) *loads_per_s = measure_gather_peak(h->sms, 16);
  VS_CUDA(h, cudaGetLastError());
  return VS_OK;
}

int vs_measure_gather_peak_ex(vs_handle* h, int32_t bytes_per_load, double* loads_per_s) {
  cudaSetDevice(h->device);
  if (bytes_per_load != 16 && bytes_per_load != 32)
    return fail(h, VS_ERR_INVALID_ARGUMENT, "bytes_per_load must be 16 or 32");
  VS_CUDA(h, cudaDeviceSynchronize());
  if (loads_per_s) *loads_per_s = measure_gather_peak(h->sms, bytes_per_load);
  VS_CUDA(h, cudaGetLastError());
  return VS_OK;
}

}  // extern "C"

namespace {

// one result array slice: device source, caller destination, offset in the
// pinned staging buffer
struct FetchPart {
  void* dst;
  const void* src;
  size_t bytes;
  size_t off;
};

// the requested result arrays of ligands [b, b + n) (torsions [tb, tb + tt))
std::vector<FetchPart> fetch_parts(vs_handle* h, const vs_results* o, size_t b, size_t n,
                                   size_t tb, size_t tt, size_t* total) {
  const size_t KT = static_cast<size_t>(h->last_prm.keep_top);
  const size_t R = static_cast<size_t>(h->last_prm.restarts);
  const bool all = h->last_prm.write_all_poses != 0;
  std::vector<FetchPart> parts;
  *total = 0;
  auto add = [&](void* dst, const DBuf& src, size_t src_off, size_t bytes) {
    if (!dst || bytes == 0) return;
    parts.push_back(FetchPart{static_cast<uint8_t*>(dst) + src_off,
                              static_cast<const uint8_t*>(src.p) + src_off, bytes, *total});
    *total += (bytes + 255) & ~size_t(255);
  };
  add(o->best, h->d_best, b * 4, n * 4);
  add(o->n_kept, h->d_nkept, b * 4, n * 4);
  add(o->n_surv, h->d_nsurv, b * 4, n * 4);
  if (KT > 0) add(o->surv, h->d_surv, b * KT * sizeof(vs_pose), n * KT * sizeof(vs_pose));
  if (KT > 0) add(o->surv_tors, h->d_surv_tors, tb * KT * 4, tt * KT * 4);
  if (all) add(o->all, h->d_all, b * R * sizeof(vs_pose), n * R * sizeof(vs_pose));
  if (all) add(o->all_tors, h->d_all_tors, tb * R * 4, tt * R * 4);
  add(o->keys, h->d_keys, b * 8, n * 8);
  return parts;
}

// D2H of the parts into one pinned staging buffer (one DMA each at full
// link rate) on `st`, asynchronously
int fetch_issue(vs_handle* h, const std::vector<FetchPart>& parts, size_t total,
                PinnedVec<uint8_t>& stage, cudaStream_t st) {
  if (!stage.resize(std::max<size_t>(total, 256)))
    return fail(h, VS_ERR_CUDA, "pinned host allocation failed");
  for (const FetchPart& p : parts)
    VS_CUDA(h, cudaMemcpyAsync(stage.data() + p.off, p.src, p.bytes, cudaMemcpyDeviceToHost, st));
  return VS_OK;
}

// threaded copy from the staging buffer into the caller's (pageable)
// buffers, which also spreads their first-touch page faults; then the
// ligands outside every size class read as dropped
void fetch_copy_out(const std::vector<FetchPart>& parts, const uint8_t* stage, vs_results* o,
                    size_t b, const std::vector<int>& cls) {
  constexpr size_t kSlice = size_t(1) << 20;
  std::vector<std::array<size_t, 3>> slices;  // part, offset, bytes
  for (size_t k = 0; k < parts.size(); ++k)
    for (size_t x = 0; x < parts[k].bytes; x += kSlice)
      slices.push_back({k, x, std::min(kSlice, parts[k].bytes - x)});
  auto copy = [&](size_t t, size_t nt) {
    for (size_t i = t; i < slices.size(); i += nt) {
      const FetchPart& p = parts[slices[i][0]];
      std::memcpy(static_cast<uint8_t*>(p.dst) + slices[i][1], stage + p.off + slices[i][1],
                  slices[i][2]);
    }
  };
  const size_t nt = std::max<size_t>(
      1, std::min<size_t>({slices.size(), 16, std::max(1u, std::thread::hardware_concurrency())}));
  if (nt == 1) {
    copy(0, 1);
  } else {
    std::vector<std::thread> pool;
    for (size_t t = 0; t < nt; ++t) pool.emplace_back(copy, t, nt);
    for (auto& th : pool) th.join();
  }
  for (size_t i = 0; i < cls.size(); ++i) {
    const size_t g = b + i;
    if (cls[i] < 0) {
      if (o->n_kept) o->n_kept[g] = -1;
      if (o->n_surv) o->n_surv[g] = 0;
      if (o->best) o->best[g] = -INFINITY;
    } else if (o->best && o->n_surv && o->n_surv[g] == 0) {
      o->best[g] = -INFINITY;
    }
  }
}

}  // namespace

extern "C" {

int vs_fetch_results(vs_handle* h, vs_results* o) {
  cudaSetDevice(h->device);
  if (!h->has_results) return fail(h, VS_ERR_STATE, "no results");
  size_t total = 0;
  const auto parts = fetch_parts(h, o, 0, static_cast<size_t>(h->res_n), 0,
                                 static_cast<size_t>(h->res_tors), &total);
  // caller buffers in page-locked memory (cudaHostAlloc / registered): one
  // DMA per array straight into them, no staging copy
  bool pinned = true;
  for (const FetchPart& p : parts) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p.dst) != cudaSuccess || a.type != cudaMemoryTypeHost) {
      cudaGetLastError();  // clear the query's error state for unregistered memory
      pinned = false;
      break;
    }
  }
  if (pinned) {
    for (const FetchPart& p : parts)
      VS_CUDA(h, cudaMemcpyAsync(p.dst, p.src, p.bytes, cudaMemcpyDeviceToHost, h->last));
    VS_CUDA(h, cudaStreamSynchronize(h->last));
    fetch_copy_out({}, nullptr, o, 0, h->res_cls);  // the dropped-ligand fix-ups only
    return VS_OK;
  }
  int rc = fetch_issue(h, parts, total, h->fetch_stage, h->last);
  if (rc) return rc;
  VS_CUDA(h, cudaStreamSynchronize(h->last));
  fetch_copy_out(parts, h->fetch_stage.data(), o, 0, h->res_cls);
  return VS_OK;
}

}  // extern "C"

namespace {

// vs_dock_host for a large library as a pipeline of contiguous chunks: the
// host packs chunk k+1 and copies chunk k-1's results out while chunk k
// docks.  Chunk k uses library slot / stage set / compute stream k % 2, so
// two chunks' kernel sequences run concurrently and fill each other's
// launch tails; every chunk writes its own slice of the result arrays (one
// global LPT order per chunk, the global id ranks and seeds travel with the
// ligands, so results are those of the one-shot path, bit for bit).
//   host:  pack(k) [after H2D(k-2)]            copy-out(k-1) [after D2H(k-1)]
//   in:    H2D(k)  [after dock(k-2)]
//   s[k%2]: dock(k) [after H2D(k)]
//   out:   D2H(k)  [after dock(k)]
int dock_host_pipelined(vs_handle* h, const vs_library* L, const vs_size_class* classes,
                        int32_t nc, const vs_dock_params* prm, vs_results* out,
                        const std::vector<double>& split, bool concurrent) {
  const int chunks = static_cast<int>(split.size()) + 1;
  if (!h->has_pocket) return fail(h, VS_ERR_STATE, "no pocket");
  if (h->empty_bounds) return fail(h, VS_ERR_EMPTY_BOUNDS, "pocket bounds box is empty");
  int rc = check_params(h, prm);
  if (rc) return rc;
  VS_CUDA(h, quiesce(h));
  const int n = L->n_ligands;
  for (int i = 0; i < n; ++i)  // the counts the chunk views are cut from
    if (L->n_atoms[i] < 0 || L->n_tors[i] < 0)
      return fail(h, VS_ERR_INVALID_ARGUMENT, "negative atom or torsion count");
  std::vector<long> aoff(n + 1, 0), toff(n + 1, 0), moff(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    aoff[i + 1] = aoff[i] + L->n_atoms[i];
    toff[i + 1] = toff[i] + L->n_tors[i];
  }
  for (int i = 0; i < n; ++i) {
    long m = 0;
    for (long j = toff[i]; j < toff[i + 1]; ++j) m += L->moving_count[j];
    moff[i + 1] = moff[i] + m;
  }
  for (int k = 0; k < 2; ++k) {
    if (!h->pipe_s[k]) VS_CUDA(h, cudaStreamCreateWithFlags(&h->pipe_s[k], cudaStreamNonBlocking));
  }
  if (!h->pipe_in) VS_CUDA(h, cudaStreamCreateWithFlags(&h->pipe_in, cudaStreamNonBlocking));
  if (!h->pipe_out) VS_CUDA(h, cudaStreamCreateWithFlags(&h->pipe_out, cudaStreamNonBlocking));
  while (h->pipe_ev.size() < 3 * static_cast<size_t>(chunks)) {
    cudaEvent_t e;
    VS_CUDA(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h->pipe_ev.push_back(e);
  }
  cudaEvent_t* evH = h->pipe_ev.data();
  cudaEvent_t* evD = evH + chunks;
  cudaEvent_t* evR = evD + chunks;
  cudaStream_t st0 = h->own;
  rc = ensure_rots(h, prm, st0);
  if (rc) return rc;
  rc = prepare_results(h, n, toff[n], prm, st0);
  if (rc) return rc;
  VS_CUDA(h, cudaStreamSynchronize(st0));
  h->last_prm = *prm;
  h->has_lib = false;  // the library is not left resident (vs_upload_library does that)
  h->has_results = false;
  h->res_cls.assign(n, -1);
  std::vector<long> cb(chunks + 1, 0);
  for (int k = 1; k < chunks; ++k)
    cb[k] = std::max(cb[k - 1], std::min<long>(n, static_cast<long>(split[k - 1] * n)));
  cb[chunks] = n;
  std::vector<std::vector<FetchPart>> parts(chunks);
  std::vector<size_t> totals(chunks, 0);
  auto view = [&](int k) {
    vs_library c = *L;
    const long b = cb[k];
    c.n_ligands = static_cast<int32_t>(cb[k + 1] - b);
    c.n_atoms = L->n_atoms + b;
    c.n_tors = L->n_tors + b;
    c.rot_bonds = L->rot_bonds ? L->rot_bonds + b : nullptr;
    c.coords = L->coords + 3 * aoff[b];
    c.atom_class = L->atom_class + aoff[b];
    c.axis_a = L->axis_a + toff[b];
    c.axis_b = L->axis_b + toff[b];
    c.moving_count = L->moving_count + toff[b];
    c.moving = L->moving + moff[b];
    c.seeds = L->seeds ? L->seeds + b : nullptr;
    c.id_rank = L->id_rank ? L->id_rank + b : nullptr;
    return c;
  };
  using clk = std::chrono::steady_clock;
  const char* te = std::getenv("VSCREEN_UPLOAD_TIMING");
  const bool timing = te && te[0] == '1';
  std::vector<double> t_pack(chunks, 0.0), t_wait(chunks, 0.0), t_copy(chunks, 0.0);
  const auto t_start = clk::now();
  auto ms_since = [](clk::time_point a) {
    return std::chrono::duration<double, std::milli>(clk::now() - a).count();
  };
  auto copy_out = [&](int k) -> int {
    auto t0 = clk::now();
    VS_CUDA(h, cudaEventSynchronize(evR[k]));
    t_wait[k] = ms_since(t0);
    t0 = clk::now();
    const Packed& P = h->pipe_lib[k % 2];
    fetch_copy_out(parts[k], h->pipe_stage[k % 2].data(), out, static_cast<size_t>(cb[k]), P.cls);
    std::copy(P.cls.begin(), P.cls.end(), h->res_cls.begin() + cb[k]);
    t_copy[k] = ms_since(t0);
    return VS_OK;
  };
  // a failed chunk drains what is in flight before returning
  auto drain = [&](int r) {
    for (cudaStream_t x : {h->pipe_s[0], h->pipe_s[1], h->pipe_in, h->pipe_out})
      cudaStreamSynchronize(x);
    return r;
  };
  VS_CUDA(h, cudaEventRecord(h->ev0, h->pipe_s[0]));
  VS_CUDA(h, cudaStreamWaitEvent(h->pipe_s[1], h->ev0, 0));
  for (int k = 0; k < chunks; ++k) {
    const int s = k % 2;
    Packed& P = h->pipe_lib[s];
    if (k >= 2) VS_CUDA(h, cudaEventSynchronize(evH[k - 2]));  // pinned slot free
    const vs_library c = view(k);
    const auto tp = clk::now();
    rc = pack_library(h, &c, classes, nc, P, nullptr);
    if (rc == VS_OK) rc = check_nested(h, P);
    if (rc) return drain(rc);
    t_pack[k] = ms_since(tp);
    if (k >= 2) VS_CUDA(h, cudaStreamWaitEvent(h->pipe_in, evD[k - 2], 0));  // device slot free
    rc = upload_packed(h, P, h->pipe_in, 3);
    if (rc) return drain(rc);
    VS_CUDA(h, cudaEventRecord(evH[k], h->pipe_in));
    // concurrent: the chunks alternate between two compute streams (their
    // launch tails overlap); otherwise one stream runs them in order
    cudaStream_t cs = h->pipe_s[concurrent ? s : 0];
    VS_CUDA(h, cudaStreamWaitEvent(cs, evH[k], 0));
    rc = launch_packed(h, P, prm, cs, h->pipe_sg[concurrent ? s : 0],
                       results_view(h, prm, cb[k], toff[cb[k]]), false);
    if (rc) return drain(rc);
    VS_CUDA(h, cudaEventRecord(evD[k], cs));
    VS_CUDA(h, cudaStreamWaitEvent(h->pipe_out, evD[k], 0));
    parts[k] = fetch_parts(h, out, static_cast<size_t>(cb[k]), static_cast<size_t>(cb[k + 1] - cb[k]),
                           static_cast<size_t>(toff[cb[k]]),
                           static_cast<size_t>(toff[cb[k + 1]] - toff[cb[k]]), &totals[k]);
    rc = fetch_issue(h, parts[k], totals[k], h->pipe_stage[s], h->pipe_out);
    if (rc) return drain(rc);
    VS_CUDA(h, cudaEventRecord(evR[k], h->pipe_out));
    if (k >= 1) {
      rc = copy_out(k - 1);
      if (rc) return drain(rc);
    }
  }
  rc = copy_out(chunks - 1);
  if (rc) return drain(rc);
  if (timing) {
    std::fprintf(stderr, "vs_dock_host pipeline (%d chunks): total %.2f ms;", chunks, ms_since(t_start));
    for (int k = 0; k < chunks; ++k)
      std::fprintf(stderr, " [%d] pack %.2f wait %.2f copy-out %.2f", k, t_pack[k], t_wait[k], t_copy[k]);
    std::fprintf(stderr, "\n");
  }
  // the whole pipeline on the handle's timeline: ev0 .. ev1 spans every
  // chunk's dock; later operations wait for both compute streams
  VS_CUDA(h, cudaStreamWaitEvent(h->pipe_s[0], evD[chunks - 1], 0));
  if (chunks >= 2) VS_CUDA(h, cudaStreamWaitEvent(h->pipe_s[0], evD[chunks - 2], 0));
  VS_CUDA(h, cudaEventRecord(h->ev1, h->pipe_s[0]));
  VS_CUDA(h, mark_done(h, h->pipe_s[0]));
  h->last = h->pipe_s[0];
  h->timed = true;
  h->staged_run = false;  // no per-launch phase events in the pipeline
  h->has_results = true;
  h->res_n = n;
  h->res_tors = toff[n];
  return VS_OK;
}

}  // namespace

extern "C" {

int vs_dock_host(vs_handle* h, const vs_library* L, const vs_size_class* classes, int32_t nc,
                 const vs_dock_params* prm, vs_results* out) {
  // VSCREEN_PIPELINE=1: large libraries as a pipeline of chunks (host pack
  // / copy-out under the dock).  Off by default: with the device packer the
  // one-shot path is faster (chunked docks lose more device efficiency than
  // the overlap saves; profiles/e2e_pipeline_r2.txt)
  const char* pe = std::getenv("VSCREEN_PIPELINE");
  if (L->n_ligands >= kPipeMinLigands && pe && pe[0] == '1') {
    cudaSetDevice(h->device);
    // chunk boundaries as fractions of the library (VSCREEN_PIPE_SPLIT,
    // comma-separated; VSCREEN_PIPE_CONCURRENT=0 runs them on one stream)
    std::vector<double> split(kPipeSplit, kPipeSplit + sizeof(kPipeSplit) / sizeof(double));
    if (const char* e = std::getenv("VSCREEN_PIPE_SPLIT"); e && *e) {
      split.clear();
      for (const char* c = e; *c;) {
        char* end = nullptr;
        split.push_back(std::strtod(c, &end));
        c = (*end == ',') ? end + 1 : end;
        if (end == c && *c) break;
      }
    }
    const char* ce = std::getenv("VSCREEN_PIPE_CONCURRENT");
    return dock_host_pipelined(h, L, classes, nc, prm, out, split, !(ce && ce[0] == '0'));
  }
  int rc = vs_upload_library(h, L, classes, nc);
  if (rc) return rc;
  rc = vs_dock(h, prm, nullptr);
  if (rc) return rc;
  return vs_fetch_results(h, out);
}

namespace {
bool same_library(const vs_library& a, const vs_library* b) {
  return a.n_ligands == b->n_ligands && a.n_atoms == b->n_atoms && a.n_tors == b->n_tors &&
         a.rot_bonds == b->rot_bonds && a.coords == b->coords && a.atom_class == b->atom_class &&
         a.axis_a == b->axis_a && a.axis_b == b->axis_b && a.moving_count == b->moving_count &&
         a.moving == b->moving && a.seeds == b->seeds && a.id_rank == b->id_rank;
}
}  // namespace

int vs_dock_host_prefetch(vs_handle* h, const vs_library* L, const vs_library* next,
                          const vs_size_class* classes, int32_t nc, const vs_dock_params* prm,
                          vs_results* out) {
  cudaSetDevice(h->device);
  const bool cls_match =
      h->spare_has_cls == (classes != nullptr) &&
      (!classes || (static_cast<size_t>(std::max(nc, 0)) == h->spare_cls.size() &&
                    std::equal(h->spare_cls.begin(), h->spare_cls.end(), classes,
                               [](const vs_size_class& x, const vs_size_class& y) {
                                 return x.atom_lo == y.atom_lo && x.atom_hi == y.atom_hi &&
                                        x.rot_lo == y.rot_lo && x.rot_hi == y.rot_hi;
                               })));
  int rc;
  if (h->spare_pending && cls_match && same_library(h->spare_L, L)) {
    // adopt the prefetched pack: its outcome is read back (the same checks
    // and errors as a synchronous upload), then the slots swap
    VS_CUDA(h, quiesce(h));
    h->spare_pending = false;
    const int spare = 1 - h->cur;
    h->has_lib = false;
    h->lib_lists_n = -1;
    h->has_results = false;
    rc = pack_finish(h, h->libs[spare], h->copy, h->spare_pp);
    if (rc) return rc;
    h->cur = spare;
    h->has_lib = true;
  } else {
    rc = vs_upload_library(h, L, classes, nc);
    if (rc) return rc;
  }
  if (next) {
    // the spare slot is free (no dock reads it); the next library's DMA and
    // packer kernels run on the copy stream under this dock
    if (!h->copy) VS_CUDA(h, cudaStreamCreateWithFlags(&h->copy, cudaStreamNonBlocking));
    const int spare = 1 - h->cur;
    if (pack_issue(h, next, classes, nc, h->libs[spare], h->copy, h->spare_pp, spare) == VS_OK) {
      h->spare_pending = true;
      h->spare_L = *next;
      h->spare_has_cls = classes != nullptr;
      h->spare_cls.assign(classes ? classes : nullptr,
                          classes ? classes + std::max(nc, 0) : nullptr);
    } else {
      // a library the packer rejects is not prefetched: the call that docks
      // it uploads it and reports the error
      cudaStreamSynchronize(h->copy);
      h->err.clear();
    }
  }
  rc = vs_dock(h, prm, nullptr);
  if (rc) return rc;
  return vs_fetch_results(h, out);
}

// tournament: chunks of C keys -> k smallest each, until one chunk remains
static int topk_run(vs_handle* h, const unsigned long long* in, long n, int k,
                    unsigned long long* out_dev, cudaStream_t st) {
  const int C = topk_chunk();
  if (k < 1 || 2 * k > C) return fail(h, VS_ERR_CAPACITY, "top-k needs 1 <= k <= 2048");
  long cur = std::max<long>(n, 1);
  const unsigned long long* src = in;
  bool first = true;
  while (true) {
    const long blocks = (cur + C - 1) / C;
    unsigned long long* dst;
    if (blocks == 1) {
      dst = out_dev;
    } else {
      DBuf& tgt = (first || src == h->d_topk_b.as<unsigned long long>()) ? h->d_topk_a : h->d_topk_b;
      VS_CUDA(h, tgt.ensure(static_cast<size_t>(blocks) * k * 8));
      dst = tgt.as<unsigned long long>();
    }
    VS_CUDA(h, launch_topk(st, src, first ? n : cur, dst, k, static_cast<int>(blocks)));
    ++h->launches;
    if (blocks == 1) break;
    cur = blocks * k;
    src = dst;
    first = false;
  }
  return VS_OK;
}

int vs_topk_device(vs_handle* h, int32_t k, uint64_t* out_dev, void* stream) {
  cudaSetDevice(h->device);
  if (!h->has_results) return fail(h, VS_ERR_STATE, "no results");
  cudaStream_t st = pick(h, stream);
  VS_CUDA(h, after_prev(h, st));  // the keys of a dock on another stream
  const int rc = topk_run(h, h->d_keys.as<unsigned long long>(), h->res_n, k,
                          reinterpret_cast<unsigned long long*>(out_dev), st);
  if (rc == VS_OK) VS_CUDA(h, mark_done(h, st));
  return rc;
}

int vs_topk_merge_device(vs_handle* h, const uint64_t* keys_dev, int64_t n, int32_t k,
                         uint64_t* out_dev, void* stream) {
  cudaSetDevice(h->device);
  cudaStream_t st = pick(h, stream);
  VS_CUDA(h, after_prev(h, st));  // the handle's top-k scratch buffers
  const int rc = topk_run(h, reinterpret_cast<const unsigned long long*>(keys_dev),
                          static_cast<long>(n), k, reinterpret_cast<unsigned long long*>(out_dev),
                          st);
  if (rc == VS_OK) VS_CUDA(h, mark_done(h, st));
  return rc;
}

int vs_topk(vs_handle* h, int32_t k, uint64_t* out_keys) {
  DBuf tmp;
  VS_CUDA(h, tmp.ensure(static_cast<size_t>(k) * 8));
  int rc = vs_topk_device(h, k, tmp.as<uint64_t>(), nullptr);
  if (rc == VS_OK) {
    cudaError_t e = cudaMemcpyAsync(out_keys, tmp.p, static_cast<size_t>(k) * 8,
                                    cudaMemcpyDeviceToHost, h->last);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->last);
    if (e != cudaSuccess) rc = cuda_fail(h, e, "topk fetch");
  }
  tmp.release();
  return rc;
}

// ------------------------------------------------------------ NCCL gather
// libnccl is resolved at first use: the copy the process already has (the
// one torch.distributed loaded) or else the system libnccl.so.2, so the
// library carries no link-time NCCL dependency and never loads a second one.
namespace {
struct NcclApi {
  bool ok = false;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclCommCount) comm_count = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
};
const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!so) so = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!so) return a;
    a.get_unique_id = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(so, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(so, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(so, "ncclCommDestroy"));
    a.comm_count = reinterpret_cast<decltype(&ncclCommCount)>(dlsym(so, "ncclCommCount"));
    a.all_gather = reinterpret_cast<decltype(&ncclAllGather)>(dlsym(so, "ncclAllGather"));
    a.error_string = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(so, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.comm_count && a.all_gather &&
           a.error_string;
    return a;
  }();
  return api;
}
int nccl_fail(vs_handle* h, ncclResult_t r, const char* what) {
  return fail(h, VS_ERR_CUDA, std::string(what) + ": " + nccl().error_string(r));
}
}  // namespace

int vs_nccl_unique_id(uint8_t out[VS_NCCL_ID_BYTES]) {
  if (!nccl().ok) return VS_ERR_NO_DEVICE;
  ncclUniqueId id;
  if (nccl().get_unique_id(&id) != ncclSuccess) return VS_ERR_CUDA;
  std::memcpy(out, id.internal, VS_NCCL_ID_BYTES);
  return VS_OK;
}

int vs_comm_init(vs_handle* h, int32_t nranks, int32_t rank, const uint8_t id[VS_NCCL_ID_BYTES]) {
  cudaSetDevice(h->device);
  if (!nccl().ok) return fail(h, VS_ERR_NO_DEVICE, "libnccl.so.2 not available");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return fail(h, VS_ERR_INVALID_ARGUMENT, "rank must be in [0, nranks)");
  vs_comm_destroy(h);
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, VS_NCCL_ID_BYTES);
  ncclComm_t c = nullptr;
  const ncclResult_t r = nccl().comm_init_rank(&c, nranks, uid, rank);
  if (r != ncclSuccess) return nccl_fail(h, r, "ncclCommInitRank");
  h->comm = c;
  h->comm_owned = true;
  return VS_OK;
}

int vs_comm_attach(vs_handle* h, void* comm) {
  vs_comm_destroy(h);
  h->comm = static_cast<ncclComm_t>(comm);
  h->comm_owned = false;
  return VS_OK;
}

void vs_comm_destroy(vs_handle* h) {
  if (h->comm && h->comm_owned && nccl().ok) {
    cudaSetDevice(h->device);
    nccl().comm_destroy(h->comm);
  }
  h->comm = nullptr;
  h->comm_owned = false;
}

int vs_topk_allgather(vs_handle* h, void* comm, int32_t k, uint64_t* out_dev, void* stream) {
  cudaSetDevice(h->device);
  if (!h->has_results) return fail(h, VS_ERR_STATE, "no results");
  ncclComm_t c = comm ? static_cast<ncclComm_t>(comm) : h->comm;
  if (!c) return fail(h, VS_ERR_STATE, "no NCCL communicator (vs_comm_init / vs_comm_attach)");
  if (!nccl().ok) return fail(h, VS_ERR_NO_DEVICE, "libnccl.so.2 not available");
  int nranks = 0;
  ncclResult_t r = nccl().comm_count(c, &nranks);
  if (r != ncclSuccess) return nccl_fail(h, r, "ncclCommCount");
  cudaStream_t st = pick(h, stream);
  VS_CUDA(h, after_prev(h, st));
  VS_CUDA(h, h->d_gather.ensure(static_cast<size_t>(nranks + 1) * k * 8));
  auto* local = h->d_gather.as<unsigned long long>();
  auto* all = local + k;
  int rc = topk_run(h, h->d_keys.as<unsigned long long>(), h->res_n, k, local, st);
  if (rc) return rc;
  // one all-gather of k u64 keys per rank (8 KB at k = 1000), then the same
  // deterministic merge on every rank
  r = nccl().all_gather(local, all, static_cast<size_t>(k), ncclUint64, c, st);
  if (r != ncclSuccess) return nccl_fail(h, r, "ncclAllGather");
  rc = topk_run(h, all, static_cast<long>(nranks) * k, k,
                reinterpret_cast<unsigned long long*>(out_dev), st);
  if (rc) return rc;
  VS_CUDA(h, mark_done(h, st));
  return VS_OK;
}

// ---------------------------------------------------- restart start draws
int vs_start_draws(vs_handle* h, const uint64_t* seeds, const int32_t* n_tors, int32_t n,
                   int32_t restarts, int32_t attempts, int32_t stride, float* out) {
  cudaSetDevice(h->device);
  if (!h->has_pocket) return fail(h, VS_ERR_STATE, "no pocket");
  if (n < 0 || restarts < 1 || attempts < 1 || attempts > 50)
    return fail(h, VS_ERR_INVALID_ARGUMENT, "n >= 0, restarts >= 1, attempts in [1, 50]");
  int tmax = 0;
  for (int i = 0; i < n; ++i) tmax = std::max(tmax, n_tors[i]);
  if (tmax > kMaxTors) return fail(h, VS_ERR_CAPACITY, "torsions > 64");
  if (stride < 7 + tmax) return fail(h, VS_ERR_CAPACITY, "stride < 7 + max torsions");
  if (n == 0) return VS_OK;
  VS_CUDA(h, quiesce(h));
  cudaStream_t st = h->own;
  const size_t rows = static_cast<size_t>(n) * restarts * attempts;
  DBuf d_seeds, d_tors, d_out;
  VS_CUDA(h, d_seeds.ensure(static_cast<size_t>(n) * 8));
  VS_CUDA(h, d_tors.ensure(static_cast<size_t>(n) * 4));
  VS_CUDA(h, d_out.ensure(rows * stride * 4));
  int rc = VS_OK;
  cudaError_t e = cudaMemcpyAsync(d_seeds.p, seeds, static_cast<size_t>(n) * 8,
                                  cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_tors.p, n_tors, static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_out.p, 0, rows * stride * 4, st);
  if (e == cudaSuccess)
    e = launch_draws(st, h->pk, d_seeds.as<const unsigned long long>(), d_tors.as<const int>(), n,
                     restarts, attempts, d_out.as<float>(), stride, h->sms);
  if (e == cudaSuccess) {
    ++h->launches;
    e = cudaMemcpyAsync(out, d_out.p, rows * stride * 4, cudaMemcpyDeviceToHost, st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) rc = cuda_fail(h, e, "start draws");
  d_seeds.release();
  d_tors.release();
  d_out.release();
  return rc;
}

float vs_key_score(uint64_t key) {
  const uint32_t ord = ~static_cast<uint32_t>(key >> 32);
  const uint32_t bits = (ord & 0x80000000u) ? (ord & 0x7fffffffu) : ~ord;
  float f;
  std::memcpy(&f, &bits, 4);
  return f;
}

uint32_t vs_key_id_rank(uint64_t key) { return static_cast<uint32_t>(key & 0xffffffffu); }

}  // extern "C"

namespace vs {
// pinned staging for vs_libbuild_relax's flattened arrays (grow-only, owned
// by the handle): the copies in relax_on_device are then plain async DMA
void* relax_host_buffer(vs_handle* h, size_t bytes) {
  return h->epin.resize(bytes) ? h->epin.data() : nullptr;
}

// device half of vs_libbuild_relax (vs_host.cpp): the spring relaxation of
// embed_3d for a flattened batch of placed conformers, in place
int relax_on_device(vs_handle* h, int n, const int64_t* atom_off, const int32_t* n_atoms,
                    double* coords, const int64_t* bond_off, const int32_t* n_bonds,
                    const int32_t* bonds, int iterations, const uint64_t* place_seeds) {
  cudaSetDevice(h->device);
  if (iterations < 0) return fail(h, VS_ERR_INVALID_ARGUMENT, "iterations must be >= 0");
  int amax = 2, bmax = 1;
  for (int i = 0; i < n; ++i) {
    if (n_atoms[i] > relax_max_atoms() || n_bonds[i] > relax_max_bonds())
      return fail(h, VS_ERR_CAPACITY, "ligand " + std::to_string(i) + " too large for the device embed");
    amax = std::max(amax, static_cast<int>(n_atoms[i]));
    bmax = std::max(bmax, static_cast<int>(n_bonds[i]));
  }
  if (n == 0) return VS_OK;
  const size_t na = static_cast<size_t>(std::max<int64_t>(atom_off[n], 1));
  const size_t nbd = static_cast<size_t>(std::max<int64_t>(bond_off[n], 1));
  DBuf &d_ao = h->ebuf[0], &d_na = h->ebuf[1], &d_bo = h->ebuf[2], &d_nb = h->ebuf[3],
       &d_bd = h->ebuf[4], &d_xyz = h->ebuf[5], &d_seed = h->ebuf[6];
  cudaStream_t st = h->own;
  VS_CUDA(h, d_ao.ensure((n + 1) * 8));
  VS_CUDA(h, d_na.ensure(n * 4));
  VS_CUDA(h, d_bo.ensure((n + 1) * 8));
  VS_CUDA(h, d_nb.ensure(n * 4));
  VS_CUDA(h, d_bd.ensure(nbd * 8));
  VS_CUDA(h, d_xyz.ensure(na * 24));
  VS_CUDA(h, cudaMemcpyAsync(d_ao.p, atom_off, (n + 1) * 8, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, cudaMemcpyAsync(d_na.p, n_atoms, n * 4, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, cudaMemcpyAsync(d_bo.p, bond_off, (n + 1) * 8, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, cudaMemcpyAsync(d_nb.p, n_bonds, n * 4, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, cudaMemcpyAsync(d_bd.p, bonds, nbd * 8, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, cudaMemcpyAsync(d_xyz.p, coords, na * 24, cudaMemcpyHostToDevice, st));
  if (place_seeds) {
    VS_CUDA(h, d_seed.ensure(n * 8));
    VS_CUDA(h, cudaMemcpyAsync(d_seed.p, place_seeds, n * 8, cudaMemcpyHostToDevice, st));
  }
  VS_CUDA(h, launch_relax(st, d_ao.as<const long long>(), d_na.as<const int>(),
                          d_bo.as<const long long>(), d_nb.as<const int>(), d_bd.as<const int2>(),
                          d_xyz.as<double>(), n, iterations, amax, bmax,
                          place_seeds ? d_seed.as<const unsigned long long>() : nullptr));
  ++h->launches;
  VS_CUDA(h, cudaMemcpyAsync(coords, d_xyz.p, na * 24, cudaMemcpyDeviceToHost, st));
  VS_CUDA(h, cudaStreamSynchronize(st));
  return VS_OK;
}
}  // namespace vs

extern "C" {

namespace {
// FP64 score (+ gradient, or + rescore bonuses) of given poses on the device
int score64_run(vs_handle* h, const vs_library* L, int64_t n_poses, const int32_t* pose_lig,
                const double* t, const double* q, const double* tors, double* score,
                double* grad_t, double* grad_q, double* grad_tors, double* resc);
}  // namespace

int vs_score_gradient(vs_handle* h, const vs_library* L, int64_t n_poses,
                      const int32_t* pose_lig, const double* t, const double* q,
                      const double* tors, double* score, double* grad_t, double* grad_q,
                      double* grad_tors) {
  return score64_run(h, L, n_poses, pose_lig, t, q, tors, score, grad_t, grad_q, grad_tors,
                     nullptr);
}

int vs_score64(vs_handle* h, const vs_library* L, int64_t n_poses, const int32_t* pose_lig,
               const double* t, const double* q, const double* tors, double* geo, double* resc) {
  return score64_run(h, L, n_poses, pose_lig, t, q, tors, geo, nullptr, nullptr, nullptr, resc);
}

namespace {
int score64_run(vs_handle* h, const vs_library* L, int64_t n_poses, const int32_t* pose_lig,
                const double* t, const double* q, const double* tors, double* score,
                double* grad_t, double* grad_q, double* grad_tors, double* resc) {
  cudaSetDevice(h->device);
  const bool grad = grad_t != nullptr;
  // scoring takes any box (the reference checks bounds only in dock(),
  // dock.cpp:321): an empty box just puts every atom outside a wall
  if (!h->has_pocket) return fail(h, VS_ERR_STATE, "no pocket");
  if (n_poses < 0) return fail(h, VS_ERR_INVALID_ARGUMENT, "negative pose count");
  if (n_poses == 0) return VS_OK;
  VS_CUDA(h, quiesce(h));
  Packed& P = h->xpack;
  DBuf &d_pl = h->xbuf[0], &d_tb = h->xbuf[1], &d_t = h->xbuf[2], &d_q = h->xbuf[3],
       &d_th = h->xbuf[4], &d_s = h->xbuf[5], &d_gt = h->xbuf[6], &d_gq = h->xbuf[7],
       &d_gth = h->xbuf[8], &d_rs = h->xbuf[9];
  int rc = pack_library(h, L, nullptr, 0, P);
  if (rc) return rc;
  std::vector<long> tb(static_cast<size_t>(n_poses));
  long toff = 0;
  int nmax = 1, tmax = 1;
  for (int64_t p = 0; p < n_poses; ++p) {
    const int l = pose_lig[p];
    if (l < 0 || l >= P.n) return fail(h, VS_ERR_INVALID_ARGUMENT, "pose ligand index out of range");
    tb[p] = toff;
    toff += P.meta[l].w;
    nmax = std::max(nmax, P.meta[l].y);
    tmax = std::max(tmax, P.meta[l].w);
  }
  if (grad_smem_per_block(nmax, tmax) > 227 * 1024)
    return fail(h, VS_ERR_CAPACITY, "ligand too large for score_gradient");
  cudaStream_t st = h->own;
  rc = upload_packed(h, P, st, 3);
  if (rc) return rc;
  const size_t np = static_cast<size_t>(n_poses), nt = static_cast<size_t>(std::max<long>(toff, 1));
  VS_CUDA(h, d_pl.ensure(np * 4));
  VS_CUDA(h, d_tb.ensure(np * 8));
  VS_CUDA(h, d_t.ensure(np * 24));
  VS_CUDA(h, d_q.ensure(np * 32));
  VS_CUDA(h, d_th.ensure(nt * 8));
  VS_CUDA(h, d_s.ensure(np * 8));
  if (grad) {
    VS_CUDA(h, d_gt.ensure(np * 24));
    VS_CUDA(h, d_gq.ensure(np * 32));
    VS_CUDA(h, d_gth.ensure(nt * 8));
  }
  if (resc) VS_CUDA(h, d_rs.ensure(np * 8));
  VS_CUDA(h, cudaMemcpyAsync(d_pl.p, pose_lig, np * 4, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, cudaMemcpyAsync(d_tb.p, tb.data(), np * 8, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, cudaMemcpyAsync(d_t.p, t, np * 24, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, cudaMemcpyAsync(d_q.p, q, np * 32, cudaMemcpyHostToDevice, st));
  if (toff > 0) VS_CUDA(h, cudaMemcpyAsync(d_th.p, tors, toff * 8, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, launch_grad(st, P.dev(), h->d_sites64.as<const SiteD>(), h->n_sites64, h->box_lo,
                         h->box_hi, h->r64, h->lam64, n_poses, d_pl.as<const int>(),
                         d_tb.as<const long>(), d_t.as<const double>(), d_q.as<const double>(),
                         d_th.as<const double>(), nmax, tmax, d_s.as<double>(),
                         grad ? d_gt.as<double>() : nullptr, grad ? d_gq.as<double>() : nullptr,
                         grad ? d_gth.as<double>() : nullptr, resc ? d_rs.as<double>() : nullptr));
  ++h->launches;
  VS_CUDA(h, cudaMemcpyAsync(score, d_s.p, np * 8, cudaMemcpyDeviceToHost, st));
  if (grad) {
    VS_CUDA(h, cudaMemcpyAsync(grad_t, d_gt.p, np * 24, cudaMemcpyDeviceToHost, st));
    VS_CUDA(h, cudaMemcpyAsync(grad_q, d_gq.p, np * 32, cudaMemcpyDeviceToHost, st));
    if (toff > 0)
      VS_CUDA(h, cudaMemcpyAsync(grad_tors, d_gth.p, toff * 8, cudaMemcpyDeviceToHost, st));
  }
  if (resc) VS_CUDA(h, cudaMemcpyAsync(resc, d_rs.p, np * 8, cudaMemcpyDeviceToHost, st));
  VS_CUDA(h, cudaStreamSynchronize(st));
  return VS_OK;
}
}  // namespace

int vs_ascend(vs_handle* h, const vs_library* L, int64_t n_poses, const int32_t* pose_lig,
              double* t, double* q, double* tors, int32_t max_steps, double* score,
              int32_t* steps) {
  cudaSetDevice(h->device);
  if (!h->has_pocket) return fail(h, VS_ERR_STATE, "no pocket");
  if (h->empty_bounds) return fail(h, VS_ERR_EMPTY_BOUNDS, "pocket bounds are empty");
  if (n_poses < 0 || max_steps < 0) return fail(h, VS_ERR_INVALID_ARGUMENT, "negative count");
  if (n_poses == 0) return VS_OK;
  VS_CUDA(h, quiesce(h));
  Packed& P = h->xpack;
  DBuf &d_pl = h->xbuf[0], &d_tb = h->xbuf[1], &d_t = h->xbuf[2], &d_q = h->xbuf[3],
       &d_th = h->xbuf[4], &d_s = h->xbuf[5], &d_st = h->xbuf[6];
  int rc = pack_library(h, L, nullptr, 0, P);
  if (rc) return rc;
  std::vector<long> tb(static_cast<size_t>(n_poses));
  long toff = 0;
  int nmax = 1, tmax = 1;
  for (int64_t p = 0; p < n_poses; ++p) {
    const int l = pose_lig[p];
    if (l < 0 || l >= P.n) return fail(h, VS_ERR_INVALID_ARGUMENT, "pose ligand index out of range");
    tb[p] = toff;
    toff += P.meta[l].w;
    nmax = std::max(nmax, P.meta[l].y);
    tmax = std::max(tmax, P.meta[l].w);
  }
  if (ascend_smem_per_block(nmax, tmax) > 227 * 1024)
    return fail(h, VS_ERR_CAPACITY, "ligand too large for the ascent");
  cudaStream_t st = h->own;
  rc = upload_packed(h, P, st, 3);
  if (rc) return rc;
  const size_t np = static_cast<size_t>(n_poses), nt = static_cast<size_t>(std::max<long>(toff, 1));
  VS_CUDA(h, d_pl.ensure(np * 4));
  VS_CUDA(h, d_tb.ensure(np * 8));
  VS_CUDA(h, d_t.ensure(np * 24));
  VS_CUDA(h, d_q.ensure(np * 32));
  VS_CUDA(h, d_th.ensure(nt * 8));
  VS_CUDA(h, d_s.ensure(np * 8));
  VS_CUDA(h, d_st.ensure(np * 4));
  VS_CUDA(h, cudaMemcpyAsync(d_pl.p, pose_lig, np * 4, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, cudaMemcpyAsync(d_tb.p, tb.data(), np * 8, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, cudaMemcpyAsync(d_t.p, t, np * 24, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, cudaMemcpyAsync(d_q.p, q, np * 32, cudaMemcpyHostToDevice, st));
  if (toff > 0) VS_CUDA(h, cudaMemcpyAsync(d_th.p, tors, toff * 8, cudaMemcpyHostToDevice, st));
  VS_CUDA(h, launch_ascend(st, P.dev(), h->d_sites64.as<const SiteD>(), h->n_sites64, h->box_lo,
                           h->box_hi, h->r64, h->lam64, n_poses, d_pl.as<const int>(),
                           d_tb.as<const long>(), d_t.as<double>(), d_q.as<double>(),
                           d_th.as<double>(), nmax, tmax, max_steps, d_s.as<double>(),
                           d_st.as<int>()));
  ++h->launches;
  VS_CUDA(h, cudaMemcpyAsync(t, d_t.p, np * 24, cudaMemcpyDeviceToHost, st));
  VS_CUDA(h, cudaMemcpyAsync(q, d_q.p, np * 32, cudaMemcpyDeviceToHost, st));
  if (toff > 0) VS_CUDA(h, cudaMemcpyAsync(tors, d_th.p, toff * 8, cudaMemcpyDeviceToHost, st));
  if (score) VS_CUDA(h, cudaMemcpyAsync(score, d_s.p, np * 8, cudaMemcpyDeviceToHost, st));
  if (steps) VS_CUDA(h, cudaMemcpyAsync(steps, d_st.p, np * 4, cudaMemcpyDeviceToHost, st));
  VS_CUDA(h, cudaStreamSynchronize(st));
  return VS_OK;
}

// ---- dock() with the reference's contract (dock.cpp:318-371): sweep-v1
// restarts (vs_dock, every kept pose), each refined by the reference ascent
// on the device (vs_ascend, FP64, max_steps), then the reference's keep rule
// on the refined coordinates in restart order (RMSD >= delta from every
// kept pose, dock.cpp:359-361) and a stable sort by score descending
// (dock.cpp:364-366).  The RMSD bookkeeping (<= restarts poses per ligand)
// runs on the host in FP64 over apply_pose (dock.cpp:52-67, 392-401).
namespace {
// transformed() of one pose (dock.cpp:52-67): torsions in axis order about
// the current coordinates, then x = R(q / |q|) y + t
void pose_coords(const vs_library* L, int64_t aoff, int n, int64_t toff, int T, int64_t moff,
                 const double* t, const double* q, const double* th, std::vector<double>& x) {
  x.assign(L->coords + 3 * aoff, L->coords + 3 * (aoff + n));
  auto rot = [](double w, double ux, double uy, double uz, double v[3]) {
    const double cx = uy * v[2] - uz * v[1], cy = uz * v[0] - ux * v[2], cz = ux * v[1] - uy * v[0];
    const double ex = uy * cz - uz * cy, ey = uz * cx - ux * cz, ez = ux * cy - uy * cx;
    v[0] = v[0] + 2.0 * w * cx + 2.0 * ex;
    v[1] = v[1] + 2.0 * w * cy + 2.0 * ey;
    v[2] = v[2] + 2.0 * w * cz + 2.0 * ez;
  };
  int64_t m = moff;
  for (int j = 0; j < T; ++j) {
    const int a = L->axis_a[toff + j], b = L->axis_b[toff + j];
    const double o[3] = {x[3 * a], x[3 * a + 1], x[3 * a + 2]};
    double d[3] = {x[3 * b] - o[0], x[3 * b + 1] - o[1], x[3 * b + 2] - o[2]};
    const double nn = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    if (nn > 0.0)
      for (double& c : d) c /= nn;
    else
      d[0] = d[1] = d[2] = 0.0;
    const double hh = 0.5 * th[j], sn = std::sin(hh), cs = std::cos(hh);
    for (int k = 0; k < L->moving_count[toff + j]; ++k) {
      const int idx = L->moving[m + k];
      double v[3] = {x[3 * idx] - o[0], x[3 * idx + 1] - o[1], x[3 * idx + 2] - o[2]};
      rot(cs, d[0] * sn, d[1] * sn, d[2] * sn, v);
      for (int c = 0; c < 3; ++c) x[3 * idx + c] = o[c] + v[c];
    }
    m += L->moving_count[toff + j];
  }
  const double qn = std::sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  for (int i = 0; i < n; ++i) {
    double v[3] = {x[3 * i], x[3 * i + 1], x[3 * i + 2]};
    rot(q[0] / qn, q[1] / qn, q[2] / qn, q[3] / qn, v);
    for (int c = 0; c < 3; ++c) x[3 * i + c] = v[c] + t[c];
  }
}

double rmsd_host(const std::vector<double>& a, const std::vector<double>& b) {
  const size_t n = a.size() / 3;
  if (n == 0) return 0.0;
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double dx = a[3 * i] - b[3 * i], dy = a[3 * i + 1] - b[3 * i + 1],
                 dz = a[3 * i + 2] - b[3 * i + 2];
    s += dx * dx + dy * dy + dz * dz;
  }
  return std::sqrt(s / static_cast<double>(n));
}
}  // namespace

int vs_dock_refined_host(vs_handle* h, const vs_library* L, const vs_size_class* classes,
                         int32_t nc, const vs_dock_params* params, int32_t max_steps,
                         vs_refined* out) {
  if (max_steps < 0) return fail(h, VS_ERR_INVALID_ARGUMENT, "max_steps must be >= 0");
  const int n = L->n_ligands, R = params->restarts;
  if (n < 0) return fail(h, VS_ERR_INVALID_ARGUMENT, "negative ligand count");
  vs_dock_params prm = *params;
  prm.write_all_poses = 1;
  std::vector<int64_t> aoff(n + 1, 0), toff(n + 1, 0), moff(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    aoff[i + 1] = aoff[i] + L->n_atoms[i];
    toff[i + 1] = toff[i] + L->n_tors[i];
  }
  for (int i = 0; i < n; ++i) {
    int64_t m = 0;
    for (int64_t j = toff[i]; j < toff[i + 1]; ++j) m += L->moving_count[j];
    moff[i + 1] = moff[i] + m;
  }
  const size_t nr = static_cast<size_t>(std::max(n, 1)) * std::max(R, 1);
  std::vector<int32_t> n_kept(std::max(n, 1));
  std::vector<vs_pose> all(nr);
  std::vector<float> all_tors(std::max<int64_t>(toff[n], 1) * std::max(R, 1));
  vs_results res{};
  res.n_kept = n_kept.data();
  res.all = all.data();
  res.all_tors = all_tors.data();
  int rc = vs_dock_host(h, L, classes, nc, &prm, &res);
  if (rc) return rc;
  // every kept pose of every ligand, in restart order, FP64
  std::vector<int32_t> pl;
  std::vector<int> slot;  // rank in the ligand's `all` block
  std::vector<double> t, q, th;
  std::vector<int64_t> first(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    first[i] = static_cast<int64_t>(pl.size());
    const int k = std::max(n_kept[i], 0);
    std::vector<int> ord(k);
    std::iota(ord.begin(), ord.end(), 0);
    std::sort(ord.begin(), ord.end(), [&](int a, int b) {
      return all[static_cast<size_t>(i) * R + a].restart < all[static_cast<size_t>(i) * R + b].restart;
    });
    const int T = L->n_tors[i];
    for (int r : ord) {
      const vs_pose& p = all[static_cast<size_t>(i) * R + r];
      pl.push_back(i);
      slot.push_back(p.restart);
      for (int c = 0; c < 3; ++c) t.push_back(p.t[c]);
      for (int c = 0; c < 4; ++c) q.push_back(p.q[c]);
      const float* tt = all_tors.data() + toff[i] * R + static_cast<int64_t>(r) * T;
      for (int j = 0; j < T; ++j) th.push_back(tt[j]);
    }
  }
  first[n] = static_cast<int64_t>(pl.size());
  const int64_t np = static_cast<int64_t>(pl.size());
  std::vector<double> score(std::max<int64_t>(np, 1));
  if (th.empty()) th.push_back(0.0);
  rc = vs_ascend(h, L, np, pl.data(), t.data(), q.data(), th.data(), max_steps, score.data(),
                 nullptr);
  if (rc) return rc;
  // per ligand: the keep rule on the refined coordinates, then the sort
  std::vector<int64_t> tb(np + 1, 0);
  for (int64_t p = 0; p < np; ++p) tb[p + 1] = tb[p] + L->n_tors[pl[p]];
  std::vector<std::vector<double>> kept_x;
  std::vector<double> x;
  for (int i = 0; i < n; ++i) {
    out->n_poses[i] = n_kept[i] < 0 ? -1 : 0;
    if (n_kept[i] <= 0) continue;
    const int N = L->n_atoms[i], T = L->n_tors[i];
    std::vector<int64_t> keep;
    kept_x.clear();
    for (int64_t p = first[i]; p < first[i + 1]; ++p) {
      pose_coords(L, aoff[i], N, toff[i], T, moff[i], &t[3 * p], &q[4 * p], &th[tb[p]], x);
      bool diverse = true;
      for (const auto& kx : kept_x)
        if (rmsd_host(x, kx) < params->diversity_delta) {
          diverse = false;
          break;
        }
      if (!diverse) continue;
      keep.push_back(p);
      kept_x.push_back(x);
    }
    std::stable_sort(keep.begin(), keep.end(),
                     [&](int64_t a, int64_t b) { return score[a] > score[b]; });
    out->n_poses[i] = static_cast<int32_t>(keep.size());
    for (size_t r = 0; r < keep.size(); ++r) {
      const int64_t p = keep[r];
      const size_t o = static_cast<size_t>(i) * R + r;
      const double qn = std::sqrt(q[4 * p] * q[4 * p] + q[4 * p + 1] * q[4 * p + 1] +
                                  q[4 * p + 2] * q[4 * p + 2] + q[4 * p + 3] * q[4 * p + 3]);
      for (int c = 0; c < 3; ++c) out->t[3 * o + c] = t[3 * p + c];
      for (int c = 0; c < 4; ++c) out->q[4 * o + c] = q[4 * p + c] / qn;  // pose_of, dock.cpp:210
      out->score[o] = score[p];
      if (out->restart) out->restart[o] = slot[p];
      for (int j = 0; j < T; ++j) out->tors[toff[i] * R + static_cast<int64_t>(r) * T + j] = th[tb[p] + j];
    }
  }
  return VS_OK;
}

}  // extern "C"

namespace {

// work lists for the rescoring launches: the ligands of each size class of
// P (P.cls) that `keep` admits, concatenated; one (start, count) per class
void class_lists(const Packed& P, const std::function<bool(int)>& keep, std::vector<int>& ligs,
                 std::vector<std::pair<int, int>>& segs) {
  ligs.clear();
  segs.assign(P.buckets.size(), {0, 0});
  std::vector<int> cnt(P.buckets.size(), 0);
  for (int l = 0; l < P.n; ++l)
    if (P.cls[l] >= 0 && keep(l)) ++cnt[static_cast<size_t>(P.cls[l])];
  int o = 0;
  for (size_t c = 0; c < cnt.size(); ++c) {
    segs[c] = {o, 0};
    o += cnt[c];
  }
  ligs.resize(static_cast<size_t>(o));
  for (int l = 0; l < P.n; ++l) {
    if (P.cls[l] < 0 || !keep(l)) continue;
    auto& sg = segs[static_cast<size_t>(P.cls[l])];
    ligs[static_cast<size_t>(sg.first + sg.second++)] = l;
  }
}

// one rescoring launch per size class over `ligs` (device), events around
int rescore_launch(vs_handle* h, const Packed& P, const int* d_ligs,
                   const std::vector<std::pair<int, int>>& segs, const PoseSrc& src,
                   DBuf& counters, cudaStream_t st) {
  VS_CUDA(h, counters.ensure(std::max<size_t>(segs.size(), 1) * 4));
  VS_CUDA(h, cudaMemsetAsync(counters.p, 0, std::max<size_t>(segs.size(), 1) * 4, st));
  if (!h->rev0) {
    VS_CUDA(h, cudaEventCreate(&h->rev0));
    VS_CUDA(h, cudaEventCreate(&h->rev1));
  }
  const bool grid = h->pk.grid_mode != 0;
  VS_CUDA(h, cudaEventRecord(h->rev0, st));
  // the classes' launches run concurrently (a fork of `st` per class, joined
  // back): a class of few large ligands overlaps the bulk of small ones
  // instead of running after it at low occupancy.  The class with the largest
  // shared-memory footprint launches first, capped at `big` blocks per SM, so
  // that the others still find 8 - big block slots on every SM: both run from
  // the start instead of one after the other
  std::vector<size_t> ord;
  for (size_t c = 0; c < segs.size(); ++c)
    if (segs[c].second > 0) ord.push_back(c);
  auto smem_of = [&](size_t c) {
    const Bucket& b = P.buckets[c];
    return rescore_smem_per_block(b.nmax, b.tmax, b.mvmax);
  };
  std::stable_sort(ord.begin(), ord.end(),
                   [&](size_t a, size_t b) { return smem_of(a) > smem_of(b); });
  int big = 2;
  if (const char* e = std::getenv("VSCREEN_RESCORE_BIG"); e && *e) big = std::atoi(e);
  big = std::min(std::max(big, 1), 7);
  int k = 0;
  for (size_t c : ord) {
    const Bucket& b = P.buckets[c];
    const size_t smem = smem_of(c);
    if (smem > 227 * 1024) return fail(h, VS_ERR_CAPACITY, "ligands too large for rescoring");
    const int per_sm = ord.size() < 2 ? 8 : (k == 0 ? big : 8 - big);
    const int blocks = std::max(1, std::min((segs[c].second + kWarpsPerBlock - 1) / kWarpsPerBlock,
                                            per_sm * h->sms));
    cudaStream_t cs = st;
    if (k > 0) {
      if (h->fork.size() < static_cast<size_t>(k)) {
        cudaStream_t x;
        cudaEvent_t e;
        VS_CUDA(h, cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
        VS_CUDA(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->fork.push_back(x);
        h->fork_ev.push_back(e);
      }
      cs = h->fork[static_cast<size_t>(k - 1)];
      VS_CUDA(h, cudaStreamWaitEvent(cs, h->rev0, 0));
    }
    VS_CUDA(h, launch_rescore(grid, blocks, smem, cs, P.dev(), h->pk, d_ligs + segs[c].first,
                              segs[c].second, counters.as<int>() + c, src, b.nmax, b.tmax,
                              b.mvmax));
    if (k > 0) {
      VS_CUDA(h, cudaEventRecord(h->fork_ev[static_cast<size_t>(k - 1)], cs));
      VS_CUDA(h, cudaStreamWaitEvent(st, h->fork_ev[static_cast<size_t>(k - 1)], 0));
    }
    ++k;
    ++h->launches;
  }
  VS_CUDA(h, cudaEventRecord(h->rev1, st));
  return VS_OK;
}

}  // namespace

extern "C" {

// geometric_score + rescore of given poses (dock.cpp:278, 297).  The library
// goes through the device packer (raw arrays DMA'd as given), the pose
// arrays are DMA'd as given too, the per-ligand ranges are host bookkeeping
// over pose_lig, and the results are copied straight into geo / resc.
int vs_rescore(vs_handle* h, const vs_library* L, int64_t n_poses, const int32_t* pose_lig,
               const float* t, const float* q, const float* tors, float* geo, float* resc) {
  return vs_rescore_checked(h, L, n_poses, pose_lig, t, q, tors, -1, geo, resc);
}

int vs_rescore_checked(vs_handle* h, const vs_library* L, int64_t n_poses,
                       const int32_t* pose_lig, const float* t, const float* q, const float* tors,
                       int64_t n_tors_values, float* geo, float* resc) {
  cudaSetDevice(h->device);
  using clk = std::chrono::steady_clock;
  const auto r0 = clk::now();
  if (!h->has_pocket) return fail(h, VS_ERR_STATE, "no pocket");
  // pose indices are 32-bit on the device (first[], count[])
  if (n_poses < 0 || n_poses > INT32_MAX)
    return fail(h, VS_ERR_CAPACITY, "n_poses must be in [0, 2^31)");
  VS_CUDA(h, quiesce(h));
  const int n = L->n_ligands;
  cudaStream_t st = h->own;
  Packed& P = h->rpack;
  PackPending pp;
  int rc = pack_issue(h, L, nullptr, 0, P, st, pp, h->cur);  // the device packer runs under the
  if (rc) return rc;                                 // host bookkeeping below
  // the pose arrays queue right behind the library (DMA under the host work)
  DBuf* rb = h->rbuf;
  auto up = [&](DBuf& dst, const void* src, size_t bytes) -> cudaError_t {
    cudaError_t err = dst.ensure(std::max<size_t>(bytes, 16));
    if (err != cudaSuccess || bytes == 0) return err;
    return cudaMemcpyAsync(dst.p, src, bytes, cudaMemcpyHostToDevice, st);
  };
  const size_t np = static_cast<size_t>(n_poses);
  VS_CUDA(h, up(rb[0], t, np * 12));
  VS_CUDA(h, up(rb[1], q, np * 16));
  const auto r1 = clk::now();
  // checks, per-ligand pose ranges and torsion bases in one pass over the
  // poses while the library and poses are in flight; the work lists per class
  std::vector<int> first(std::max(n, 1), 0), count(std::max(n, 1), 0);
  std::vector<long> tb(std::max(n, 1), 0);
  long toff = 0;
  const char* bad = nullptr;
  for (int64_t p = 0; p < n_poses; ++p) {
    const int l = pose_lig[p];
    if (p > 0 && l < pose_lig[p - 1]) {
      bad = "pose_lig must be non-decreasing";
      break;
    }
    if (l < 0 || l >= n) {
      bad = "pose ligand index out of range";
      break;
    }
    if (count[l]++ == 0) {
      first[l] = static_cast<int>(p);
      tb[l] = toff;
    }
    toff += L->n_tors[l];
  }
  if (bad) {
    cudaStreamSynchronize(st);  // the issued pack drains before its buffers are reused
    return fail(h, VS_ERR_INVALID_ARGUMENT, bad);
  }
  if (n_tors_values >= 0 && toff != n_tors_values) {  // check_counts, dock.cpp:219-230
    cudaStreamSynchronize(st);  // the issued pack drains before its buffers are reused
    return fail(h, VS_ERR_ATOM_COUNT, "poses need " + std::to_string(toff) +
                                          " torsion values, got " + std::to_string(n_tors_values));
  }
  VS_CUDA(h, up(rb[2], tors, static_cast<size_t>(toff) * 4));
  VS_CUDA(h, up(rb[3], first.data(), n * 4ul));
  VS_CUDA(h, up(rb[4], count.data(), n * 4ul));
  VS_CUDA(h, up(rb[5], tb.data(), n * 8ul));
  rc = pack_finish(h, P, st, pp);
  if (rc) return rc;
  std::vector<int> ligs;
  std::vector<std::pair<int, int>> segs;
  class_lists(P, [&](int l) { return count[l] > 0; }, ligs, segs);
  const auto r2 = clk::now();
  VS_CUDA(h, up(rb[6], ligs.data(), ligs.size() * 4));
  VS_CUDA(h, rb[7].ensure(std::max<size_t>(np, 1) * 4));
  VS_CUDA(h, rb[8].ensure(std::max<size_t>(np, 1) * 4));
  PoseSrc src{};
  src.first = rb[3].as<const int>();
  src.count = rb[4].as<const int>();
  src.tb = rb[5].as<const long>();
  src.t3 = rb[0].as<const float>();
  src.q4 = rb[1].as<const float>();
  src.tors = rb[2].as<const float>();
  src.geo = rb[7].as<float>();
  src.resc = rb[8].as<float>();
  rc = rescore_launch(h, P, rb[6].as<int>(), segs, src, rb[9], st);
  if (rc) return rc;
  if (np) {
    if (geo) VS_CUDA(h, cudaMemcpyAsync(geo, rb[7].p, np * 4, cudaMemcpyDeviceToHost, st));
    if (resc) VS_CUDA(h, cudaMemcpyAsync(resc, rb[8].p, np * 4, cudaMemcpyDeviceToHost, st));
  }
  VS_CUDA(h, cudaStreamSynchronize(st));
  float ms = 0.0f;
  VS_CUDA(h, cudaEventElapsedTime(&ms, h->rev0, h->rev1));
  h->rescore_ms = ms;
  if (const char* ev = std::getenv("VSCREEN_UPLOAD_TIMING"); ev && ev[0] == '1') {
    auto d = [](clk::time_point x, clk::time_point y) {
      return std::chrono::duration<double, std::milli>(y - x).count();
    };
    std::fprintf(stderr, "vs_rescore: check + device pack %.2f ms, ranges + lists %.2f ms, "
                 "H2D + kernels + D2H %.2f ms (kernels %.2f)\n", d(r0, r1), d(r1, r2),
                 d(r2, clk::now()), h->rescore_ms);
  }
  return VS_OK;
}

// the same for poses already in device memory, against the resident
// library (vs_upload_library); everything stays on `stream`
int vs_rescore_device(vs_handle* h, int64_t n_poses, const int32_t* pose_lig, const float* t,
                      const float* q, const float* tors, float* geo, float* resc, void* stream) {
  cudaSetDevice(h->device);
  if (!h->has_pocket) return fail(h, VS_ERR_STATE, "no pocket");
  if (!h->has_lib) return fail(h, VS_ERR_STATE, "no resident library");
  if (n_poses < 0 || n_poses > INT32_MAX)
    return fail(h, VS_ERR_CAPACITY, "n_poses must be in [0, 2^31)");
  const Packed& P = h->libs[h->cur];
  if (!P.on_device) return fail(h, VS_ERR_STATE, "library not packed on the device");
  cudaStream_t st = pick(h, stream);
  VS_CUDA(h, after_prev(h, st));
  DBuf* rb = h->rbuf;
  const int n = P.n;
  const size_t tmp = pose_ranges_temp_bytes(n_poses);
  VS_CUDA(h, rb[3].ensure(std::max(n, 1) * 4ul));
  VS_CUDA(h, rb[4].ensure(std::max(n, 1) * 4ul));
  VS_CUDA(h, rb[5].ensure(std::max(n, 1) * 8ul));
  VS_CUDA(h, rb[10].ensure(2 * (static_cast<size_t>(n_poses) + 1) * 8));
  VS_CUDA(h, rb[11].ensure(tmp));
  VS_CUDA(h, launch_pose_ranges(st, pose_lig, n_poses, P.dev(), rb[3].as<int>(), rb[4].as<int>(),
                                rb[10].as<long>(), rb[5].as<long>(), n, rb[11].p, tmp));
  h->launches += 3;
  // every ligand of each class is a work item (no host knowledge of the
  // poses); ligands without poses return at once
  if (h->lib_lists_n != n) {
    std::vector<int> ligs;
    class_lists(P, [](int) { return true; }, ligs, h->lib_segs);
    VS_CUDA(h, h->d_lib_lists.ensure(std::max<size_t>(ligs.size(), 1) * 4));
    VS_CUDA(h, cudaMemcpyAsync(h->d_lib_lists.p, ligs.data(), ligs.size() * 4,
                               cudaMemcpyHostToDevice, st));
    VS_CUDA(h, cudaStreamSynchronize(st));
    h->lib_lists_n = n;
  }
  PoseSrc src{};
  src.first = rb[3].as<const int>();
  src.count = rb[4].as<const int>();
  src.tb = rb[5].as<const long>();
  src.t3 = t;
  src.q4 = q;
  src.tors = tors;
  src.geo = geo;
  src.resc = resc;
  const int rc = rescore_launch(h, P, h->d_lib_lists.as<int>(), h->lib_segs, src, rb[9], st);
  if (rc) return rc;
  VS_CUDA(h, mark_done(h, st));
  return VS_OK;
}

// the survivors of the last vs_dock re-scored in place against the current
// pocket (e.g. finer maps): geo / resc [n * keep_top] (device), slot
// l * keep_top + k for k < n_surv[l]
int vs_rescore_survivors(vs_handle* h, float* geo, float* resc, void* stream) {
  cudaSetDevice(h->device);
  if (!h->has_pocket) return fail(h, VS_ERR_STATE, "no pocket");
  if (!h->has_results || !h->has_lib || h->res_n != h->libs[h->cur].n)
    return fail(h, VS_ERR_STATE, "no dock results on the resident library");
  const Packed& P = h->libs[h->cur];
  if (!P.on_device) return fail(h, VS_ERR_STATE, "library not packed on the device");
  cudaStream_t st = pick(h, stream);
  VS_CUDA(h, after_prev(h, st));
  if (h->lib_lists_n != P.n) {
    std::vector<int> ligs;
    class_lists(P, [](int) { return true; }, ligs, h->lib_segs);
    VS_CUDA(h, h->d_lib_lists.ensure(std::max<size_t>(ligs.size(), 1) * 4));
    VS_CUDA(h, cudaMemcpyAsync(h->d_lib_lists.p, ligs.data(), ligs.size() * 4,
                               cudaMemcpyHostToDevice, st));
    VS_CUDA(h, cudaStreamSynchronize(st));
    h->lib_lists_n = P.n;
  }
  PoseSrc src{};
  src.surv = h->d_surv.as<const PoseOut>();
  src.surv_tors = h->d_surv_tors.as<const float>();
  src.n_surv = h->d_nsurv.as<const int>();
  src.keep_top = h->last_prm.keep_top;
  src.geo = geo;
  src.resc = resc;
  const int rc = rescore_launch(h, P, h->d_lib_lists.as<int>(), h->lib_segs, src, h->rbuf[9], st);
  if (rc) return rc;
  VS_CUDA(h, mark_done(h, st));
  return VS_OK;
}

}  // extern "C"
