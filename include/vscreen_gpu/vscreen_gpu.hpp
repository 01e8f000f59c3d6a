// vscreen_gpu.hpp — header-only C++ drop-in for the reference dock API
// (proj/include/vscreen/dock.hpp, batcher.hpp, pipeline.hpp) on top of the
// C-ABI in capi.h.  Same function names, argument meaning and exception
// types (in namespace vscreen_gpu), so a caller of vscreen::dock::dock /
// geometric_score / rescore / filter_poses / rank_ligands switches by
// changing the include and namespace.
//
//   #include <vscreen_gpu/vscreen_gpu.hpp>
//   vscreen_gpu::Device gpu(0);
//   auto poses = vscreen_gpu::dock::dock(gpu, conf, topo, pocket, 30, 1.0, seed);
//
// Link with paper_2304_09953_b200/libvscreen_gpu.so.
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "capi.h"

namespace vscreen_gpu {

struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
};
struct Quat {
  double w = 1.0, x = 0.0, y = 0.0, z = 0.0;
};

// ------------------------------------------------------------ exceptions --
class AtomCountMismatch : public std::runtime_error {  // dock.hpp:48-51
 public:
  using std::runtime_error::runtime_error;
};
class LengthMismatch : public std::runtime_error {  // dock.hpp:53-56
 public:
  using std::runtime_error::runtime_error;
};
class EmptyBounds : public std::runtime_error {  // dock.hpp:58-61
 public:
  EmptyBounds() : std::runtime_error("pocket bounds box is empty") {}
};
class OutOfRange : public std::runtime_error {  // batcher.hpp:42-45
 public:
  using std::runtime_error::runtime_error;
};
class ItemTooLarge : public std::runtime_error {  // batcher.hpp:47-50
 public:
  using std::runtime_error::runtime_error;
};
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void check(int rc, const vs_handle* h = nullptr) {
  if (rc >= 0) return;
  const std::string msg = h ? vs_last_error(h) : std::string("vscreen_gpu status ") + std::to_string(rc);
  switch (rc) {
    case VS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case VS_ERR_ATOM_COUNT: throw AtomCountMismatch(msg);
    case VS_ERR_EMPTY_BOUNDS: throw EmptyBounds();
    case VS_ERR_LENGTH: throw LengthMismatch(msg);
    case VS_ERR_OUT_OF_RANGE: throw OutOfRange(msg);
    case VS_ERR_ITEM_TOO_LARGE: throw ItemTooLarge(msg);
    case VS_ERR_CUDA:
    case VS_ERR_NO_DEVICE: throw DeviceError(msg);
    default: throw std::runtime_error(msg);
  }
}

// One GPU (vs_handle), owned.
class Device {
 public:
  explicit Device(int device = 0) { check(vs_create(device, &h_)); }
  ~Device() { vs_destroy(h_); }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  vs_handle* get() const { return h_; }

 private:
  vs_handle* h_ = nullptr;
};

namespace dock {

enum class SiteKind { Steric, HBond, Lipophilic };  // dock.hpp:16

struct Site {  // dock.hpp:18-23
  Vec3 center;
  double weight = 1.0;
  double sigma = 1.0;
  SiteKind kind = SiteKind::Steric;
};

struct Box {  // dock.hpp:25-28
  Vec3 lo, hi;
  bool empty() const { return hi.x <= lo.x || hi.y <= lo.y || hi.z <= lo.z; }
};

struct Pocket {  // dock.hpp:32-37
  std::vector<Site> sites;
  Box bounds;
  double clash_radius = 0.8;
  double clash_penalty = 1.0;
};

struct Pose {  // dock.hpp:39-46
  std::string ligand_id;
  Vec3 translation;
  Quat rotation;
  std::vector<double> torsions;
  double geometric_score = 0.0;
  std::optional<double> rescore;
};

struct TorsionTopology {  // dock.hpp:65-71
  struct Axis {
    int a = 0, b = 0;
    std::vector<int> moving;
  };
  std::vector<Axis> axes;
};

struct Conformer {  // chem.hpp:78-81 (+ element class per atom for rescore)
  std::string ligand_id;
  std::vector<Vec3> coords;
  std::vector<int32_t> atom_class;  // 1 C, 2 N/O, 0 other (dock.cpp:309); empty = 0
};

// Sweep-v1 knobs beyond dock()'s own arguments (docs/SWEEP_V1.md).
struct SweepKnobs {
  int rotations = 256;
  int flex_angles = 16;
  int flex_passes = 2;
  uint64_t rotation_seed = 0x5EED;
  int polish = 1;  // 0 off, 1 rigid compass, 2 + fine torsion pass (SWEEP_V1.md §3.5)
};

namespace detail {

struct FlatLibrary {
  std::vector<int32_t> n_atoms, n_tors, cls, axis_a, axis_b, mcount, moving;
  std::vector<double> coords;
  std::vector<uint64_t> seeds;
  std::vector<uint32_t> id_rank;
  vs_library view() {
    vs_library L{};
    L.n_ligands = static_cast<int32_t>(n_atoms.size());
    L.n_atoms = n_atoms.data();
    L.n_tors = n_tors.data();
    L.rot_bonds = n_tors.data();
    L.coords = coords.data();
    L.atom_class = cls.data();
    L.axis_a = axis_a.data();
    L.axis_b = axis_b.data();
    L.moving_count = mcount.data();
    L.moving = moving.data();
    L.seeds = seeds.data();
    L.id_rank = id_rank.data();
    return L;
  }
};

inline FlatLibrary one(const Conformer& conf, const TorsionTopology& topo, uint64_t seed) {
  FlatLibrary f;
  f.n_atoms.push_back(static_cast<int32_t>(conf.coords.size()));
  f.n_tors.push_back(static_cast<int32_t>(topo.axes.size()));
  for (std::size_t i = 0; i < conf.coords.size(); ++i) {
    f.coords.insert(f.coords.end(), {conf.coords[i].x, conf.coords[i].y, conf.coords[i].z});
    f.cls.push_back(i < conf.atom_class.size() ? conf.atom_class[i] : 0);
  }
  for (const auto& ax : topo.axes) {
    f.axis_a.push_back(ax.a);
    f.axis_b.push_back(ax.b);
    f.mcount.push_back(static_cast<int32_t>(ax.moving.size()));
    f.moving.insert(f.moving.end(), ax.moving.begin(), ax.moving.end());
  }
  f.seeds.push_back(seed);
  f.id_rank.push_back(0);
  // non-null pointers for empty arrays
  for (auto* v : {&f.axis_a, &f.axis_b, &f.mcount, &f.moving})
    if (v->empty()) v->reserve(1);
  return f;
}

inline void set_pocket(Device& dev, const Pocket& p) {
  std::vector<vs_site> sites;
  for (const Site& s : p.sites)
    sites.push_back(vs_site{{s.center.x, s.center.y, s.center.z}, s.weight, s.sigma,
                            static_cast<int32_t>(s.kind), 0});
  vs_pocket vp{};
  vp.sites = sites.data();
  vp.n_sites = static_cast<int32_t>(sites.size());
  vp.lo[0] = p.bounds.lo.x; vp.lo[1] = p.bounds.lo.y; vp.lo[2] = p.bounds.lo.z;
  vp.hi[0] = p.bounds.hi.x; vp.hi[1] = p.bounds.hi.y; vp.hi[2] = p.bounds.hi.z;
  vp.clash_radius = p.clash_radius;
  vp.clash_penalty = p.clash_penalty;
  check(vs_set_pocket(dev.get(), &vp, 0.0, 0.0), dev.get());
}

inline void check_counts(const Conformer& conf, const TorsionTopology& topo, const Pose& pose) {
  if (pose.torsions.size() != topo.axes.size())  // dock.cpp:219-230
    throw AtomCountMismatch("pose has " + std::to_string(pose.torsions.size()) +
                            " torsions, topology has " + std::to_string(topo.axes.size()));
  for (const auto& ax : topo.axes)
    if (ax.a >= static_cast<int>(conf.coords.size()) || ax.b >= static_cast<int>(conf.coords.size()))
      throw AtomCountMismatch("torsion topology does not fit conformer");
}

inline std::pair<double, double> score_pose(Device& dev, const Conformer& conf,
                                            const TorsionTopology& topo, const Pose& pose,
                                            const Pocket& pocket) {
  check_counts(conf, topo, pose);
  set_pocket(dev, pocket);
  FlatLibrary f = one(conf, topo, 0);
  vs_library L = f.view();
  const int32_t lig = 0;
  const float t[3] = {static_cast<float>(pose.translation.x), static_cast<float>(pose.translation.y),
                      static_cast<float>(pose.translation.z)};
  const float q[4] = {static_cast<float>(pose.rotation.w), static_cast<float>(pose.rotation.x),
                      static_cast<float>(pose.rotation.y), static_cast<float>(pose.rotation.z)};
  std::vector<float> th(pose.torsions.begin(), pose.torsions.end());
  th.push_back(0.0f);
  float geo = 0.0f, resc = 0.0f;
  check(vs_rescore(dev.get(), &L, 1, &lig, t, q, th.data(), &geo, &resc), dev.get());
  return {geo, resc};
}

}  // namespace detail

// geometric_score (dock.hpp:80-81) on the GPU, canonical FP32 score.
inline double geometric_score(Device& dev, const Conformer& conf, const TorsionTopology& topo,
                              const Pose& pose, const Pocket& pocket) {
  return detail::score_pose(dev, conf, topo, pose, pocket).first;
}

struct ScoreGradient {  // dock.hpp:86-91
  double score = 0.0;
  Vec3 translation;
  std::array<double, 4> rotation{};  // d/d(w, x, y, z)
  std::vector<double> torsions;
};

// score_gradient (dock.hpp:93-94) on the GPU, FP64: analytic translation /
// rotation derivatives, central differences (h = 1e-5) for torsions.
inline ScoreGradient score_gradient(Device& dev, const Conformer& conf,
                                    const TorsionTopology& topo, const Pose& pose,
                                    const Pocket& pocket) {
  detail::check_counts(conf, topo, pose);
  if (pocket.bounds.empty()) throw EmptyBounds();
  detail::set_pocket(dev, pocket);
  detail::FlatLibrary f = detail::one(conf, topo, 0);
  vs_library L = f.view();
  const int32_t lig = 0;
  const double t[3] = {pose.translation.x, pose.translation.y, pose.translation.z};
  const double q[4] = {pose.rotation.w, pose.rotation.x, pose.rotation.y, pose.rotation.z};
  std::vector<double> th(pose.torsions.begin(), pose.torsions.end());
  th.push_back(0.0);
  ScoreGradient g;
  double gt[3], gq[4];
  std::vector<double> gth(th.size(), 0.0);
  check(vs_score_gradient(dev.get(), &L, 1, &lig, t, q, th.data(), &g.score, gt, gq,
                          gth.data()),
        dev.get());
  g.translation = {gt[0], gt[1], gt[2]};
  g.rotation = {gq[0], gq[1], gq[2], gq[3]};
  g.torsions.assign(gth.begin(), gth.begin() + static_cast<long>(pose.torsions.size()));
  return g;
}

// rescore (dock.hpp:98-99); the element classes travel in conf.atom_class.
inline double rescore(Device& dev, const Conformer& conf, const TorsionTopology& topo,
                      const Pose& pose, const Pocket& pocket) {
  return detail::score_pose(dev, conf, topo, pose, pocket).second;
}

// dock (dock.hpp:107-109) with the sweep-v1 generator; max_steps (the
// reference's ascent length) has no meaning for sweep-v1.
inline std::vector<Pose> dock(Device& dev, const Conformer& conf, const TorsionTopology& topo,
                              const Pocket& pocket, int restarts, double diversity_delta,
                              uint64_t seed, int max_steps = 500, SweepKnobs knobs = {}) {
  (void)max_steps;
  if (pocket.bounds.empty()) throw EmptyBounds();
  if (restarts < 1) throw std::invalid_argument("restarts must be >= 1");
  if (diversity_delta < 0.0) throw std::invalid_argument("diversity_delta must be >= 0");
  if (conf.coords.empty()) throw AtomCountMismatch("conformer has no atoms");
  detail::set_pocket(dev, pocket);
  detail::FlatLibrary f = detail::one(conf, topo, seed);
  vs_library L = f.view();
  vs_dock_params prm{};
  prm.restarts = restarts;
  prm.rotations = knobs.rotations;
  prm.flex_angles = knobs.flex_angles;
  prm.flex_passes = knobs.flex_passes;
  prm.diversity_delta = diversity_delta;
  prm.keep_top = 0;
  prm.write_all_poses = 1;
  prm.min_score = -1e30;
  prm.rotation_seed = knobs.rotation_seed;
  prm.polish = knobs.polish;
  const std::size_t T = topo.axes.size();
  float best = 0.0f;
  int32_t n_kept = 0, n_surv = 0;
  std::vector<vs_pose> all(static_cast<std::size_t>(restarts));
  std::vector<float> all_tors(T * restarts + 1);
  uint64_t key = 0;
  vs_results r{};
  r.best = &best;
  r.n_kept = &n_kept;
  r.n_surv = &n_surv;
  r.all = all.data();
  r.all_tors = all_tors.data();
  r.keys = &key;
  check(vs_dock_host(dev.get(), &L, nullptr, 0, &prm, &r), dev.get());
  std::vector<Pose> out;
  for (int k = 0; k < n_kept; ++k) {
    Pose p;
    p.ligand_id = conf.ligand_id;
    p.translation = {all[k].t[0], all[k].t[1], all[k].t[2]};
    p.rotation = {all[k].q[0], all[k].q[1], all[k].q[2], all[k].q[3]};
    p.torsions.assign(all_tors.begin() + k * T, all_tors.begin() + (k + 1) * T);
    p.geometric_score = all[k].score;
    out.push_back(std::move(p));
  }
  return out;
}

// filter_poses (dock.hpp:113-114)
inline std::vector<Pose> filter_poses(const std::vector<Pose>& poses, std::size_t keep_top,
                                      double min_score) {
  std::vector<double> s;
  for (const Pose& p : poses) s.push_back(p.geometric_score);
  std::vector<int32_t> idx(poses.size() + 1);
  const int n = vs_filter_poses(s.data(), static_cast<int32_t>(s.size()),
                                static_cast<int64_t>(keep_top > (1ull << 62) ? (1ull << 62) : keep_top),
                                min_score, idx.data());
  std::vector<Pose> out;
  for (int i = 0; i < n; ++i) out.push_back(poses[idx[i]]);
  return out;
}

}  // namespace dock

namespace pipeline {

// rank_ligands (pipeline.hpp:108-110)
inline std::vector<std::pair<std::string, double>> rank_ligands(
    const std::map<std::string, double>& scores) {
  std::string blob;
  std::vector<double> s;
  std::vector<std::string> ids;
  for (const auto& [id, v] : scores) {
    blob += id;
    blob.push_back('\0');
    s.push_back(v);
    ids.push_back(id);
  }
  std::vector<int32_t> order(ids.size() + 1);
  const int n = vs_rank_ligands(blob.c_str(), s.data(), static_cast<int32_t>(ids.size()),
                                order.data());
  std::vector<std::pair<std::string, double>> out;
  for (int i = 0; i < n; ++i) out.emplace_back(ids[order[i]], s[order[i]]);
  return out;
}

}  // namespace pipeline
}  // namespace vscreen_gpu
