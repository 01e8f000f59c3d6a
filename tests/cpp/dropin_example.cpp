// Compile-and-run check of the C++ drop-in: a reference caller's code
// (include/vscreen/*.hpp, the reference's own API) linked to
// libvscreen_core.so, plus the library-scale C-ABI path (capi.h) for a
// batch: pack -> dock on the GPU -> device top-k.  Host-side functions run
// on the CPU; GPU entry points throw without a device (no CPU fallback).
#include <cmath>
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "vscreen/batcher.hpp"
#include "vscreen/chem.hpp"
#include "vscreen/dock.hpp"
#include "vscreen/pipeline.hpp"
#include "vscreen_gpu/capi.h"

using namespace vscreen;

int main() {
  // host: rank_ligands (test_pipeline.cpp:89-101), filter_poses, batcher
  auto ranked = pipeline::rank_ligands({{"a", 1.0}, {"b", 3.0}, {"c", 2.0}});
  if (ranked.size() != 3 || ranked[0].first != "b" || ranked[2].first != "a") return 1;
  std::vector<dock::Pose> poses(3);
  poses[0].geometric_score = 1;
  poses[1].geometric_score = 5;
  poses[2].geometric_score = 3;
  auto kept = dock::filter_poses(poses, 2, -1e300);
  if (kept.size() != 2 || kept[0].geometric_score != 5 || kept[1].geometric_score != 3) return 2;
  chem::Ligand lig = chem::make_ligand("L1", "CCOc1ccccc1");
  if (batcher::size_class(lig, batcher::default_classes()) != 0) return 3;
  try {
    dock::Pocket p;
    p.bounds = {{-5, -5, -5}, {5, 5, 5}};
    p.clash_radius = 0.7;
    p.clash_penalty = 0.5;
    p.sites = {{{1.0, 0.5, -0.5}, 1.0, 1.0, dock::SiteKind::Steric}};
    chem::Conformer c;
    c.coords = {{0, 0, 0}};
    dock::TorsionTopology none;
    dock::Pose at;
    at.translation = {1.0, 0.5, -0.5};
    const double s = dock::geometric_score(c, none, at, p);  // test_dock.cpp:45-47
    if (std::fabs(s - 1.0) > 1e-9) return 4;
    auto docked = dock::dock(c, none, p, 4, 1.0, 42);
    if (docked.empty() || distance(docked[0].translation, p.sites[0].center) > 1e-4) return 5;
    // a flexible ligand through the same entry point
    chem::Conformer conf = chem::embed_3d(lig.graph, 7, lig.id);
    dock::TorsionTopology topo = dock::torsion_topology(lig.graph);
    auto flex = dock::dock(conf, topo, p, 8, 1.0, 9);
    if (flex.empty()) return 6;
    std::printf("gpu ok %.6f %zu %zu\n", s, docked.size(), flex.size());

    // library scale through the C-ABI: 64 ligands, one launch sequence
    std::vector<int32_t> na, nt, aa, ab, mc, mv, cls;
    std::vector<double> xyz;
    std::vector<uint64_t> seeds;
    std::vector<uint32_t> idr;
    const char* smis[4] = {"CCO", "CCCN", "c1ccccc1O", "CC(C)CC(=O)N"};
    for (int i = 0; i < 64; ++i) {
      chem::Ligand l = chem::make_ligand("M" + std::to_string(i), smis[i % 4]);
      chem::Conformer cf = chem::embed_3d(l.graph, static_cast<uint64_t>(i));
      dock::TorsionTopology tp = dock::torsion_topology(l.graph);
      na.push_back(l.heavy_atoms);
      nt.push_back(static_cast<int32_t>(tp.axes.size()));
      for (const Vec3& v : cf.coords) xyz.insert(xyz.end(), {v.x, v.y, v.z});
      for (const chem::Atom& a : l.graph.atoms)
        cls.push_back(a.element == "C" ? 1 : (a.element == "N" || a.element == "O") ? 2 : 0);
      for (const auto& ax : tp.axes) {
        aa.push_back(ax.a);
        ab.push_back(ax.b);
        mc.push_back(static_cast<int32_t>(ax.moving.size()));
        mv.insert(mv.end(), ax.moving.begin(), ax.moving.end());
      }
      seeds.push_back(1000 + i);
      idr.push_back(static_cast<uint32_t>(i));
    }
    vs_library L{};
    L.n_ligands = 64;
    L.n_atoms = na.data();
    L.n_tors = nt.data();
    L.coords = xyz.data();
    L.atom_class = cls.data();
    L.axis_a = aa.data();
    L.axis_b = ab.data();
    L.moving_count = mc.data();
    L.moving = mv.data();
    L.seeds = seeds.data();
    L.id_rank = idr.data();
    vs_handle* h = nullptr;
    if (vs_create(0, &h) != VS_OK) return 7;
    vs_site site{{1.0, 0.5, -0.5}, 1.0, 1.0, 0, 0};
    vs_pocket vp{&site, 1, 0, {-5, -5, -5}, {5, 5, 5}, 0.7, 0.5};
    vs_dock_params prm{8, 64, 16, 1, 1.0, 4, 0, -1e30, 0x5EED, 1, 0};
    uint64_t top[8];
    if (vs_set_pocket(h, &vp, 0.4, 2.0) != VS_OK || vs_upload_library(h, &L, nullptr, 0) != VS_OK ||
        vs_dock(h, &prm, nullptr) != VS_OK || vs_topk(h, 8, top) != VS_OK) {
      std::printf("c-abi error: %s\n", vs_last_error(h));
      return 8;
    }
    std::printf("batch ok best %.4f id_rank %u\n", vs_key_score(top[0]), vs_key_id_rank(top[0]));
    vs_destroy(h);
  } catch (const std::runtime_error& e) {
    std::printf("no device: %s\n", e.what());
  }
  std::printf("dropin ok\n");
  return 0;
}
