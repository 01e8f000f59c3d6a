// dock API of the drop-in (include/vscreen/dock.hpp) over the C-ABI.
//
// Every scoring and docking call goes to the GPU through capi.h: one
// vs_handle per calling thread (the reference calls dock() concurrently from
// its std::thread pool, pipeline.cpp:482-486), the pocket uploaded once per
// distinct pocket, the conformer packed as a one-ligand vs_library.  Status
// codes map back onto the reference's exception types (dock.cpp:219-230,
// 321-324, 394-395, 414, 441, 448).  Host-side: torsion_topology (graph
// rule, dock.cpp:234-270), apply_pose / rmsd / pose_rmsd (FP64 bookkeeping,
// dock.cpp:52-67, 392-406), filter_poses (dock.cpp:373-390) and the JSON
// I/O, written with the same JSON library (nlohmann 3.11.3) and call
// pattern as dock.cpp:432-489 so the bytes match.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <fstream>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "../../../include/vscreen_gpu/capi.h"
#include "../vs_ingest.h"
#include "vscreen/dock.hpp"

namespace vscreen::chem {
vs::Graph to_ingest(const MolecularGraph& m);  // vs_dropin_chem.cpp
}

namespace vscreen::dock {

namespace {

[[noreturn]] void raise(int rc, const vs_handle* h) {
  const std::string msg = h ? vs_last_error(h) : ("vscreen_gpu status " + std::to_string(rc));
  switch (rc) {
    case VS_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case VS_ERR_ATOM_COUNT: throw AtomCountMismatch(msg);
    case VS_ERR_EMPTY_BOUNDS: throw EmptyBounds();
    case VS_ERR_LENGTH: throw LengthMismatch(msg);
    default: throw std::runtime_error("vscreen drop-in: " + msg);
  }
}

void check(int rc, const vs_handle* h) {
  if (rc < 0) raise(rc, h);
}

// the calling thread's GPU and the pocket it holds
struct Context {
  vs_handle* h = nullptr;
  bool has_pocket = false;
  Pocket pocket;
  double spacing = 0.0;
  ~Context() {
    if (h) vs_destroy(h);
  }
};
thread_local Context g_ctx;

bool same_pocket(const Pocket& a, const Pocket& b) {
  if (a.sites.size() != b.sites.size() || a.clash_radius != b.clash_radius ||
      a.clash_penalty != b.clash_penalty)
    return false;
  auto eq = [](const Vec3& u, const Vec3& v) { return u.x == v.x && u.y == v.y && u.z == v.z; };
  if (!eq(a.bounds.lo, b.bounds.lo) || !eq(a.bounds.hi, b.bounds.hi)) return false;
  for (std::size_t i = 0; i < a.sites.size(); ++i) {
    const Site &s = a.sites[i], &t = b.sites[i];
    if (!eq(s.center, t.center) || s.weight != t.weight || s.sigma != t.sigma || s.kind != t.kind)
      return false;
  }
  return true;
}

// the device handle of this thread with `pocket` resident.  The sweep runs
// on the analytic field by default (the reference's field, 1e-5 parity per
// pose); VSCREEN_GRID_SPACING > 0 selects grid maps.
vs_handle* device_with(const Pocket& pocket) {
  Context& c = g_ctx;
  if (!c.h) {
    const char* d = std::getenv("VSCREEN_DEVICE");
    const int rc = vs_create(d ? std::atoi(d) : 0, &c.h);
    if (rc != VS_OK) {
      c.h = nullptr;
      throw std::runtime_error("vscreen drop-in: no CUDA device (status " + std::to_string(rc) +
                               "); the dock-and-score path has no CPU fallback");
    }
  }
  const char* gs = std::getenv("VSCREEN_GRID_SPACING");
  const double spacing = gs ? std::atof(gs) : 0.0;
  if (!c.has_pocket || spacing != c.spacing || !same_pocket(pocket, c.pocket)) {
    std::vector<vs_site> sites(pocket.sites.size());
    for (std::size_t i = 0; i < sites.size(); ++i) {
      const Site& s = pocket.sites[i];
      sites[i] = vs_site{{s.center.x, s.center.y, s.center.z}, s.weight, s.sigma,
                         static_cast<int32_t>(s.kind), 0};
    }
    vs_pocket vp{};
    vp.sites = sites.data();
    vp.n_sites = static_cast<int32_t>(sites.size());
    const Vec3 &lo = pocket.bounds.lo, &hi = pocket.bounds.hi;
    vp.lo[0] = lo.x, vp.lo[1] = lo.y, vp.lo[2] = lo.z;
    vp.hi[0] = hi.x, vp.hi[1] = hi.y, vp.hi[2] = hi.z;
    vp.clash_radius = pocket.clash_radius;
    vp.clash_penalty = pocket.clash_penalty;
    c.has_pocket = false;
    check(vs_set_pocket(c.h, &vp, spacing, 2.0), c.h);
    c.pocket = pocket;
    c.spacing = spacing;
    c.has_pocket = true;
  }
  return c.h;
}

// one conformer + topology as a vs_library (arrays owned here)
struct OneLigand {
  std::vector<int32_t> n_atoms, n_tors, axis_a, axis_b, moving_count, moving, atom_class;
  std::vector<double> coords;
  uint64_t seed = 0;
  uint32_t id_rank = 0;
  vs_library lib{};

  OneLigand(const chem::Conformer& conf, const TorsionTopology& topo, uint64_t s,
            const chem::MolecularGraph* g = nullptr)
      : seed(s) {
    n_atoms = {static_cast<int32_t>(conf.coords.size())};
    n_tors = {static_cast<int32_t>(topo.axes.size())};
    for (const Vec3& v : conf.coords) coords.insert(coords.end(), {v.x, v.y, v.z});
    for (const auto& ax : topo.axes) {
      axis_a.push_back(ax.a);
      axis_b.push_back(ax.b);
      moving_count.push_back(static_cast<int32_t>(ax.moving.size()));
      moving.insert(moving.end(), ax.moving.begin(), ax.moving.end());
    }
    atom_class.assign(conf.coords.size(), 0);
    if (g)
      for (std::size_t i = 0; i < g->atoms.size() && i < atom_class.size(); ++i)
        atom_class[i] = vs::element_class(g->atoms[i].element);
    lib.n_ligands = 1;
    lib.n_atoms = n_atoms.data();
    lib.n_tors = n_tors.data();
    lib.rot_bonds = n_tors.data();
    lib.coords = coords.data();
    lib.atom_class = atom_class.data();
    lib.axis_a = axis_a.empty() ? nullptr : axis_a.data();
    lib.axis_b = axis_b.empty() ? nullptr : axis_b.data();
    lib.moving_count = moving_count.empty() ? nullptr : moving_count.data();
    lib.moving = moving.empty() ? nullptr : moving.data();
    lib.seeds = &seed;
    lib.id_rank = &id_rank;
  }
};

// dock.cpp:219-230
void check_counts(const chem::Conformer& conf, const TorsionTopology& topo, const Pose& pose) {
  if (pose.torsions.size() != topo.axes.size())
    throw AtomCountMismatch("pose has " + std::to_string(pose.torsions.size()) +
                            " torsions, topology has " + std::to_string(topo.axes.size()));
  const int n = static_cast<int>(conf.coords.size());
  for (const auto& ax : topo.axes)
    if (ax.a >= n || ax.b >= n) throw AtomCountMismatch("torsion topology does not fit conformer");
}

// FP64 geometric score (and rescore when g != nullptr) of one pose on the GPU
double score_one(const chem::Conformer& conf, const TorsionTopology& topo, const Pose& pose,
                 const Pocket& pocket, const chem::MolecularGraph* g) {
  check_counts(conf, topo, pose);
  if (conf.coords.empty()) return 0.0;  // the sums over atoms and pairs are empty
  vs_handle* h = device_with(pocket);
  OneLigand L(conf, topo, 0, g);
  const int32_t pl = 0;
  const double t[3] = {pose.translation.x, pose.translation.y, pose.translation.z};
  const double q[4] = {pose.rotation.w, pose.rotation.x, pose.rotation.y, pose.rotation.z};
  const double zero = 0.0;
  double geo = 0.0, resc = 0.0;
  check(vs_score64(h, &L.lib, 1, &pl, t, q, pose.torsions.empty() ? &zero : pose.torsions.data(),
                   &geo, g ? &resc : nullptr),
        h);
  return g ? resc : geo;
}

const char* kind_name(SiteKind k) {
  switch (k) {
    case SiteKind::Steric: return "steric";
    case SiteKind::HBond: return "hbond";
    case SiteKind::Lipophilic: return "lipophilic";
  }
  return "steric";
}

SiteKind kind_of(const std::string& s) {
  if (s == "steric") return SiteKind::Steric;
  if (s == "hbond") return SiteKind::HBond;
  if (s == "lipophilic") return SiteKind::Lipophilic;
  throw std::runtime_error("unknown site kind: " + s);
}

Vec3 vec_of(const nlohmann::json& a) {
  return Vec3{a.at(0).get<double>(), a.at(1).get<double>(), a.at(2).get<double>()};
}

}  // namespace

TorsionTopology torsion_topology(const chem::MolecularGraph& g) {
  const vs::Topology t = vs::torsion_axes(chem::to_ingest(g));
  TorsionTopology out;
  out.axes.reserve(t.axes.size());
  for (const vs::Axis& a : t.axes) out.axes.push_back(TorsionTopology::Axis{a.a, a.b, a.moving});
  return out;
}

std::vector<Vec3> apply_pose(const chem::Conformer& conf, const TorsionTopology& topo,
                             const Pose& pose) {
  check_counts(conf, topo, pose);
  std::vector<Vec3> x = conf.coords;
  for (std::size_t j = 0; j < topo.axes.size(); ++j) {
    const auto& ax = topo.axes[j];
    const Vec3 o = x[static_cast<std::size_t>(ax.a)];
    const Vec3 dir = (x[static_cast<std::size_t>(ax.b)] - o).normalized();
    const Quat r = Quat::from_axis_angle(dir, pose.torsions[j]);
    for (int m : ax.moving) x[static_cast<std::size_t>(m)] = o + r.rotate(x[static_cast<std::size_t>(m)] - o);
  }
  const Quat q = pose.rotation.normalized();
  for (Vec3& v : x) v = q.rotate(v) + pose.translation;
  return x;
}

double geometric_score(const chem::Conformer& conf, const TorsionTopology& topo,
                       const Pose& pose, const Pocket& pocket) {
  return score_one(conf, topo, pose, pocket, nullptr);
}

ScoreGradient score_gradient(const chem::Conformer& conf, const TorsionTopology& topo,
                             const Pose& pose, const Pocket& pocket) {
  check_counts(conf, topo, pose);
  ScoreGradient out;
  out.torsions.assign(topo.axes.size(), 0.0);
  if (conf.coords.empty()) return out;
  vs_handle* h = device_with(pocket);
  OneLigand L(conf, topo, 0);
  const int32_t pl = 0;
  const double t[3] = {pose.translation.x, pose.translation.y, pose.translation.z};
  const double q[4] = {pose.rotation.w, pose.rotation.x, pose.rotation.y, pose.rotation.z};
  double gt[3], gq[4], zero = 0.0;
  check(vs_score_gradient(h, &L.lib, 1, &pl, t, q,
                          pose.torsions.empty() ? &zero : pose.torsions.data(), &out.score, gt,
                          gq, out.torsions.empty() ? &zero : out.torsions.data()),
        h);
  out.translation = Vec3{gt[0], gt[1], gt[2]};
  out.rotation = {gq[0], gq[1], gq[2], gq[3]};
  return out;
}

double rescore(const chem::MolecularGraph& g, const chem::Conformer& conf,
               const TorsionTopology& topo, const Pose& pose, const Pocket& pocket) {
  if (g.atom_count() != static_cast<int>(conf.coords.size()))
    throw AtomCountMismatch("graph and conformer disagree on atom count");
  return score_one(conf, topo, pose, pocket, &g);
}

std::vector<Pose> dock(const chem::Conformer& conf, const TorsionTopology& topo,
                       const Pocket& pocket, int restarts, double diversity_delta,
                       std::uint64_t seed, int max_steps) {
  if (pocket.bounds.empty()) throw EmptyBounds();
  if (restarts < 1) throw std::invalid_argument("restarts must be >= 1");
  if (diversity_delta < 0.0) throw std::invalid_argument("diversity_delta must be >= 0");
  if (conf.coords.empty()) throw AtomCountMismatch("conformer has no atoms");
  vs_handle* h = device_with(pocket);
  OneLigand L(conf, topo, seed);
  vs_dock_params prm{};
  prm.restarts = restarts;
  prm.rotations = 256;
  prm.flex_angles = 16;
  prm.flex_passes = 2;
  prm.diversity_delta = diversity_delta;
  prm.keep_top = restarts;
  prm.min_score = -1e300;
  prm.rotation_seed = 0x5EED;
  prm.polish = 1;
  const std::size_t R = static_cast<std::size_t>(restarts), T = topo.axes.size();
  int32_t n_poses = 0;
  std::vector<double> t(3 * R), q(4 * R), th(std::max<std::size_t>(T * R, 1)), sc(R);
  vs_refined out{&n_poses, t.data(), q.data(), th.data(), sc.data(), nullptr};
  // a ligand outside every size class would be dropped: one class holding it
  const vs_size_class all{1, std::max(2, static_cast<int>(conf.coords.size()) + 1), 0,
                          static_cast<int>(T) + 1};
  check(vs_dock_refined_host(h, &L.lib, &all, 1, &prm, std::max(max_steps, 0), &out), h);
  std::vector<Pose> poses(static_cast<std::size_t>(std::max(n_poses, 0)));
  for (std::size_t r = 0; r < poses.size(); ++r) {
    Pose& p = poses[r];
    p.ligand_id = conf.ligand_id;
    p.translation = Vec3{t[3 * r], t[3 * r + 1], t[3 * r + 2]};
    p.rotation = Quat{q[4 * r], q[4 * r + 1], q[4 * r + 2], q[4 * r + 3]};
    p.torsions.assign(th.begin() + static_cast<std::ptrdiff_t>(r * T),
                      th.begin() + static_cast<std::ptrdiff_t>((r + 1) * T));
    p.geometric_score = sc[r];
  }
  return poses;
}

std::vector<Pose> filter_poses(const std::vector<Pose>& poses, std::size_t keep_top,
                               double min_score) {
  std::vector<std::size_t> idx;
  for (std::size_t i = 0; i < poses.size(); ++i)
    if (poses[i].geometric_score >= min_score) idx.push_back(i);
  if (idx.size() > keep_top) {
    std::stable_sort(idx.begin(), idx.end(), [&](std::size_t a, std::size_t b) {
      return poses[a].geometric_score > poses[b].geometric_score;
    });
    idx.resize(keep_top);
    std::sort(idx.begin(), idx.end());  // survivors back in input order
  }
  std::vector<Pose> out;
  out.reserve(idx.size());
  for (std::size_t i : idx) out.push_back(poses[i]);
  return out;
}

double rmsd(std::span<const Vec3> a, std::span<const Vec3> b) {
  if (a.size() != b.size())
    throw LengthMismatch("coordinate sets have different lengths: " + std::to_string(a.size()) +
                         " vs " + std::to_string(b.size()));
  if (a.empty()) return 0.0;
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += (a[i] - b[i]).norm2();
  return std::sqrt(s / static_cast<double>(a.size()));
}

double pose_rmsd(const chem::Conformer& conf, const TorsionTopology& topo, const Pose& a,
                 const Pose& b) {
  const std::vector<Vec3> xa = apply_pose(conf, topo, a), xb = apply_pose(conf, topo, b);
  return rmsd(xa, xb);
}

Pocket parse_pocket_json(const std::string& text) {
  const nlohmann::json j = nlohmann::json::parse(text);
  Pocket p;
  for (const auto& js : j.at("sites")) {
    Site s;
    s.center = vec_of(js.at("center"));
    s.weight = js.at("weight").get<double>();
    s.sigma = js.at("sigma").get<double>();
    s.kind = kind_of(js.at("kind").get<std::string>());
    if (!(s.sigma > 0.0)) throw std::runtime_error("site sigma must be > 0");
    p.sites.push_back(s);
  }
  const auto& b = j.at("bounds");
  p.bounds = Box{vec_of(b.at("min")), vec_of(b.at("max"))};
  p.clash_radius = j.at("clash_radius").get<double>();
  p.clash_penalty = j.at("clash_penalty").get<double>();
  if (p.clash_penalty < 0.0) throw std::runtime_error("clash_penalty must be >= 0");
  return p;
}

Pocket load_pocket_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open pocket file: " + path);
  std::stringstream text;
  text << in.rdbuf();
  return parse_pocket_json(text.str());
}

std::string pocket_to_json(const Pocket& pocket) {
  using J = nlohmann::ordered_json;
  J sites = J::array();
  for (const Site& s : pocket.sites)
    sites.push_back(J{{"center", {s.center.x, s.center.y, s.center.z}},
                      {"weight", s.weight},
                      {"sigma", s.sigma},
                      {"kind", kind_name(s.kind)}});
  const Vec3 &lo = pocket.bounds.lo, &hi = pocket.bounds.hi;
  J j;
  j["sites"] = std::move(sites);
  j["bounds"] = J{{"min", {lo.x, lo.y, lo.z}}, {"max", {hi.x, hi.y, hi.z}}};
  j["clash_radius"] = pocket.clash_radius;
  j["clash_penalty"] = pocket.clash_penalty;
  return j.dump(2);
}

std::string pose_to_json(const Pose& pose) {
  nlohmann::ordered_json j;
  j["ligand"] = pose.ligand_id;
  j["translation"] = {pose.translation.x, pose.translation.y, pose.translation.z};
  j["rotation"] = {pose.rotation.w, pose.rotation.x, pose.rotation.y, pose.rotation.z};
  j["torsions"] = pose.torsions;
  j["geometric_score"] = pose.geometric_score;
  j["rescore"] = pose.rescore ? nlohmann::ordered_json(*pose.rescore) : nlohmann::ordered_json();
  return j.dump();
}

}  // namespace vscreen::dock
