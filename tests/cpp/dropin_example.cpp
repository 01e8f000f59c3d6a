// Compile-and-run check of the header-only C++ drop-in (vscreen_gpu.hpp):
// host-side functions run on the CPU; GPU entry points throw DeviceError
// without a device, or run when one is present.
#include <cmath>
#include <cstdio>
#include <map>
#include <string>

#include <vscreen_gpu/vscreen_gpu.hpp>

int main() {
  namespace vg = vscreen_gpu;
  // rank_ligands known answer (test_pipeline.cpp:89-101)
  auto ranked = vg::pipeline::rank_ligands({{"a", 1.0}, {"b", 3.0}, {"c", 2.0}});
  if (ranked.size() != 3 || ranked[0].first != "b" || ranked[2].first != "a") return 1;
  std::vector<vg::dock::Pose> poses(3);
  poses[0].geometric_score = 1;
  poses[1].geometric_score = 5;
  poses[2].geometric_score = 3;
  auto kept = vg::dock::filter_poses(poses, 2, -1e300);
  if (kept.size() != 2 || kept[0].geometric_score != 5 || kept[1].geometric_score != 3) return 2;
  try {
    vg::Device dev(0);
    vg::dock::Pocket p;
    p.bounds = {{-5, -5, -5}, {5, 5, 5}};
    p.clash_radius = 0.7;
    p.clash_penalty = 0.5;
    p.sites = {{{1.0, 0.5, -0.5}, 1.0, 1.0, vg::dock::SiteKind::Steric}};
    vg::dock::Conformer c;
    c.coords = {{0, 0, 0}};
    vg::dock::TorsionTopology topo;
    vg::dock::Pose at;
    at.translation = {1.0, 0.5, -0.5};
    const double s = vg::dock::geometric_score(dev, c, topo, at, p);  // test_dock.cpp:45-47
    if (std::fabs(s - 1.0) > 1e-6) return 3;
    auto docked = vg::dock::dock(dev, c, topo, p, 4, 1.0, 42);
    if (docked.empty()) return 4;
    // at the site centre the steric gradient vanishes (test_dock.cpp:62-80)
    const auto gr = vg::dock::score_gradient(dev, c, topo, at, p);
    if (std::fabs(gr.score - s) > 1e-9 || std::fabs(gr.translation.x) > 1e-9) return 5;
    std::printf("gpu ok %.6f %zu\n", s, docked.size());
  } catch (const vg::DeviceError& e) {
    std::printf("no device: %s\n", e.what());
  }
  std::printf("dropin ok\n");
  return 0;
}
