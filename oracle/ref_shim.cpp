// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// extern "C" shim over the UNMODIFIED reference library (compiled in place
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets
// the pytest suite and bench.py's reference arm call the reference's own
// dock/score/batcher/rank functions through ctypes.  Only tests/, smoke() and
// bench.py (cpu_baseline / --impl reference legs) may load this library.
//
// Every entry point wraps exactly one reference function (cited) and turns
// C++ exceptions into negative status codes:
//   -1 generic std::exception, -2 AtomCountMismatch, -3 LengthMismatch,
//   -4 EmptyBounds, -5 std::invalid_argument, -6 OutOfRange, -7 ItemTooLarge,
//   -8 ParseError, -9 buffer too small.
#include <cstdint>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <thread>
#include <atomic>

#include <json.hpp>
#include <vector>

#include "smiles_corpus.hpp"  // proj/tools/smiles_corpus.hpp (reference corpus sampler)
#include "vscreen/batcher.hpp"
#include "vscreen/codec.hpp"
#include "vscreen/chem.hpp"
#include "vscreen/dock.hpp"
#include "vscreen/pipeline.hpp"
#include "vscreen/rng.hpp"

using namespace vscreen;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const dock::AtomCountMismatch& e) {
    g_err = e.what();
    return -2;
  } catch (const dock::LengthMismatch& e) {
    g_err = e.what();
    return -3;
  } catch (const dock::EmptyBounds& e) {
    g_err = e.what();
    return -4;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -5;
  } catch (const batcher::OutOfRange& e) {
    g_err = e.what();
    return -6;
  } catch (const batcher::ItemTooLarge& e) {
    g_err = e.what();
    return -7;
  } catch (const chem::ParseError& e) {
    g_err = e.what();
    return -8;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

struct RefLigand {
  chem::Ligand lig;  // graph + descriptors (make_ligand, chem.cpp:333)
  chem::Conformer conf;
  dock::TorsionTopology topo;
};

dock::Pose make_pose(const double* t, const double* q, const double* tors, int nt) {
  dock::Pose p;
  p.translation = {t[0], t[1], t[2]};
  p.rotation = {q[0], q[1], q[2], q[3]};
  p.torsions.assign(tors, tors + nt);
  return p;
}

}  // namespace

extern "C" {

const char* vsref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- ligands --
// make_ligand (chem.cpp:333) + embed_3d (chem.cpp:406) + torsion_topology
// (dock.cpp:234).  iterations < 0 skips the embedding (coords all zero).
int vsref_ligand_new(const char* smiles, const char* id, std::uint64_t embed_seed,
                     int iterations, void** out) {
  return guarded([&] {
    auto* L = new RefLigand;
    try {
      L->lig = chem::make_ligand(id ? id : "", smiles);
      if (iterations >= 0) {
        L->conf = chem::embed_3d(L->lig.graph, embed_seed, L->lig.id, iterations);
      } else {
        L->conf.ligand_id = L->lig.id;
        L->conf.coords.assign(L->lig.graph.atoms.size(), Vec3{});
      }
      L->topo = dock::torsion_topology(L->lig.graph);
    } catch (...) {
      delete L;
      throw;
    }
    *out = L;
    return 0;
  });
}

void vsref_ligand_free(void* h) { delete static_cast<RefLigand*>(h); }

int vsref_ligand_info(void* h, int* n_atoms, int* n_tors, int* rot_bonds, int* moving_total) {
  auto* L = static_cast<RefLigand*>(h);
  *n_atoms = L->lig.heavy_atoms;
  *n_tors = static_cast<int>(L->topo.axes.size());
  *rot_bonds = L->lig.rotatable_bonds;
  int mv = 0;
  for (const auto& ax : L->topo.axes) mv += static_cast<int>(ax.moving.size());
  *moving_total = mv;
  return 0;
}

void vsref_ligand_coords(void* h, double* out) {
  auto* L = static_cast<RefLigand*>(h);
  for (std::size_t i = 0; i < L->conf.coords.size(); ++i) {
    out[3 * i] = L->conf.coords[i].x;
    out[3 * i + 1] = L->conf.coords[i].y;
    out[3 * i + 2] = L->conf.coords[i].z;
  }
}

void vsref_ligand_set_coords(void* h, const double* in) {
  auto* L = static_cast<RefLigand*>(h);
  for (std::size_t i = 0; i < L->conf.coords.size(); ++i) {
    L->conf.coords[i] = {in[3 * i], in[3 * i + 1], in[3 * i + 2]};
  }
}

// element class per atom: 1 = "C", 2 = "N" or "O", 0 = other (the matching
// rule of rescore, dock.cpp:309)
void vsref_ligand_classes(void* h, std::int32_t* out) {
  auto* L = static_cast<RefLigand*>(h);
  for (std::size_t i = 0; i < L->lig.graph.atoms.size(); ++i) {
    const std::string& el = L->lig.graph.atoms[i].element;
    out[i] = el == "C" ? 1 : (el == "N" || el == "O") ? 2 : 0;
  }
}

// bonds (a, b, order) in graph order and ring flags
int vsref_ligand_bonds(void* h, std::int32_t* out, int cap) {
  auto* L = static_cast<RefLigand*>(h);
  const auto& g = L->lig.graph;
  if (static_cast<int>(g.bonds.size()) > cap) return -9;
  for (std::size_t e = 0; e < g.bonds.size(); ++e) {
    out[4 * e] = g.bonds[e].a;
    out[4 * e + 1] = g.bonds[e].b;
    out[4 * e + 2] = static_cast<int>(g.bonds[e].order);
    out[4 * e + 3] = g.ring_bond_flags.size() == g.bonds.size() ? (g.ring_bond_flags[e] ? 1 : 0) : -1;
  }
  return static_cast<int>(g.bonds.size());
}

// axes: a[T], b[T], moving counts[T], moving indices flattened
void vsref_ligand_axes(void* h, std::int32_t* a, std::int32_t* b, std::int32_t* cnt,
                       std::int32_t* moving) {
  auto* L = static_cast<RefLigand*>(h);
  int k = 0;
  for (std::size_t j = 0; j < L->topo.axes.size(); ++j) {
    const auto& ax = L->topo.axes[j];
    a[j] = ax.a;
    b[j] = ax.b;
    cnt[j] = static_cast<int>(ax.moving.size());
    for (int m : ax.moving) moving[k++] = m;
  }
}

// ----------------------------------------------------------------- pocket --
int vsref_pocket_parse(const char* json, void** out) {
  return guarded([&] {
    *out = new dock::Pocket(dock::parse_pocket_json(json));  // dock.cpp:432
    return 0;
  });
}

void vsref_pocket_free(void* p) { delete static_cast<dock::Pocket*>(p); }

// ---------------------------------------------------------------- scoring --
// geometric_score (dock.cpp:278)
int vsref_geometric_score(void* h, void* pk, const double* t, const double* q,
                          const double* tors, int nt, double* out) {
  return guarded([&] {
    auto* L = static_cast<RefLigand*>(h);
    *out = dock::geometric_score(L->conf, L->topo, make_pose(t, q, tors, nt),
                                 *static_cast<dock::Pocket*>(pk));
    return 0;
  });
}

// score_gradient (dock.cpp:284): out = score, gt[3], gq[4], gtor[nt]
int vsref_score_gradient(void* h, void* pk, const double* t, const double* q,
                         const double* tors, int nt, double* out) {
  return guarded([&] {
    auto* L = static_cast<RefLigand*>(h);
    const dock::ScoreGradient g = dock::score_gradient(L->conf, L->topo, make_pose(t, q, tors, nt),
                                                       *static_cast<dock::Pocket*>(pk));
    out[0] = g.score;
    out[1] = g.translation.x;
    out[2] = g.translation.y;
    out[3] = g.translation.z;
    for (int k = 0; k < 4; ++k) out[4 + k] = g.rotation[k];
    for (int j = 0; j < nt; ++j) out[8 + j] = g.torsions[j];
    return 0;
  });
}

// rescore (dock.cpp:297)
int vsref_rescore(void* h, void* pk, const double* t, const double* q, const double* tors,
                  int nt, double* out) {
  return guarded([&] {
    auto* L = static_cast<RefLigand*>(h);
    *out = dock::rescore(L->lig.graph, L->conf, L->topo, make_pose(t, q, tors, nt),
                         *static_cast<dock::Pocket*>(pk));
    return 0;
  });
}

// apply_pose (dock.cpp:272)
int vsref_apply_pose(void* h, const double* t, const double* q, const double* tors, int nt,
                     double* out) {
  return guarded([&] {
    auto* L = static_cast<RefLigand*>(h);
    auto x = dock::apply_pose(L->conf, L->topo, make_pose(t, q, tors, nt));
    for (std::size_t i = 0; i < x.size(); ++i) {
      out[3 * i] = x[i].x;
      out[3 * i + 1] = x[i].y;
      out[3 * i + 2] = x[i].z;
    }
    return 0;
  });
}

// rmsd (dock.cpp:392)
int vsref_rmsd(const double* a, int na, const double* b, int nb, double* out) {
  return guarded([&] {
    std::vector<Vec3> va(na), vb(nb);
    for (int i = 0; i < na; ++i) va[i] = {a[3 * i], a[3 * i + 1], a[3 * i + 2]};
    for (int i = 0; i < nb; ++i) vb[i] = {b[3 * i], b[3 * i + 1], b[3 * i + 2]};
    *out = dock::rmsd(va, vb);
    return 0;
  });
}

// dock (dock.cpp:318).  Record per pose: t[3] q[4] geometric_score rescore
// torsions[T]  (stride 9 + T doubles).  Returns the number of poses.
int vsref_dock(void* h, void* pk, int restarts, double delta, std::uint64_t seed,
               int max_steps, int with_rescore, double* out, int cap) {
  return guarded([&] {
    auto* L = static_cast<RefLigand*>(h);
    const auto& pocket = *static_cast<dock::Pocket*>(pk);
    auto poses = dock::dock(L->conf, L->topo, pocket, restarts, delta, seed, max_steps);
    if (static_cast<int>(poses.size()) > cap) return -9;
    const std::size_t T = L->topo.axes.size();
    for (std::size_t i = 0; i < poses.size(); ++i) {
      double* r = out + i * (9 + T);
      const auto& p = poses[i];
      r[0] = p.translation.x; r[1] = p.translation.y; r[2] = p.translation.z;
      r[3] = p.rotation.w; r[4] = p.rotation.x; r[5] = p.rotation.y; r[6] = p.rotation.z;
      r[7] = p.geometric_score;
      r[8] = with_rescore ? dock::rescore(L->lig.graph, L->conf, L->topo, p, pocket) : 0.0;
      for (std::size_t j = 0; j < T; ++j) r[9 + j] = p.torsions[j];
    }
    return static_cast<int>(poses.size());
  });
}

// The reference's CPU path for one ligand as run_campaign drives it
// (pipeline.cpp:482-515): dock -> rescore -> filter_poses -> best = max
// rescore.  Returns 1 and writes *best when a pose survives, 0 when the
// ligand is dropped.
int vsref_dock_best(void* h, void* pk, int restarts, double delta, std::uint64_t seed,
                    int max_steps, int keep_top, double min_score, double* best) {
  return guarded([&] {
    auto* L = static_cast<RefLigand*>(h);
    const auto& pocket = *static_cast<dock::Pocket*>(pk);
    auto poses = dock::dock(L->conf, L->topo, pocket, restarts, delta, seed, max_steps);
    for (auto& p : poses) p.rescore = dock::rescore(L->lig.graph, L->conf, L->topo, p, pocket);
    poses = dock::filter_poses(poses, static_cast<std::size_t>(keep_top), min_score);
    if (poses.empty()) return 0;
    double b = -1e308;
    for (const auto& p : poses) b = std::max(b, p.rescore.value_or(0.0));
    *best = b;
    return 1;
  });
}

// Multi-threaded driver of vsref_dock_best over many ligands, mirroring the
// reference parallel_for (pipeline.cpp:29-55): atomic work counter, indexed
// writes.  kept[i] = 1/0, best[i] = score.
int vsref_dock_best_many(void** ligs, int n, void* pk, int restarts, double delta,
                         const std::uint64_t* seeds, int max_steps, int keep_top,
                         double min_score, int threads, std::int32_t* kept, double* best) {
  std::atomic<int> next{0};
  std::atomic<int> status{0};
  auto work = [&] {
    for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1)) {
      int rc = vsref_dock_best(ligs[i], pk, restarts, delta, seeds[i], max_steps, keep_top,
                               min_score, &best[i]);
      if (rc < 0) status = rc;
      kept[i] = rc > 0 ? 1 : 0;
    }
  };
  if (threads <= 1) {
    work();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
  }
  return status.load();
}

// filter_poses (dock.cpp:373) on bare scores; writes surviving input indices.
int vsref_filter_poses(const double* scores, int n, long keep_top, double min_score,
                       std::int32_t* out_idx) {
  std::vector<dock::Pose> poses(n);
  for (int i = 0; i < n; ++i) {
    poses[i].geometric_score = scores[i];
    poses[i].ligand_id = std::to_string(i);
  }
  auto kept = dock::filter_poses(poses, static_cast<std::size_t>(keep_top), min_score);
  for (std::size_t i = 0; i < kept.size(); ++i) out_idx[i] = std::stoi(kept[i].ligand_id);
  return static_cast<int>(kept.size());
}

// rank_ligands (pipeline.cpp:243).  ids are NUL-separated; out_order gets
// the input index of each ranked entry.
int vsref_rank_ligands(const char* ids_blob, const double* scores, int n,
                       std::int32_t* out_order) {
  std::map<std::string, double> m;
  std::map<std::string, int> idx;
  const char* p = ids_blob;
  for (int i = 0; i < n; ++i) {
    std::string id(p);
    p += id.size() + 1;
    m[id] = scores[i];
    idx[id] = i;
  }
  auto ranked = pipeline::rank_ligands(m);
  for (std::size_t i = 0; i < ranked.size(); ++i) out_order[i] = idx[ranked[i].first];
  return static_cast<int>(ranked.size());
}

// ---------------------------------------------------------------- batcher --
// classes: flat [atom_lo, atom_hi, rot_lo, rot_hi] x nc
int vsref_size_class(int atoms, int rot, const std::int32_t* classes, int nc) {
  return guarded([&] {
    std::vector<batcher::SizeClass> cls(nc);
    for (int i = 0; i < nc; ++i) {
      cls[i] = {classes[4 * i], classes[4 * i + 1], classes[4 * i + 2], classes[4 * i + 3]};
    }
    chem::Ligand l;
    l.id = "L";
    l.heavy_atoms = atoms;
    l.rotatable_bonds = rot;
    return static_cast<int>(batcher::size_class(l, cls));  // batcher.cpp:19
  });
}

int vsref_target_batch_size(double cap, double fixed, double per_atom, double per_rot,
                            int atom_hi, int rot_hi, long* out) {
  return guarded([&] {
    batcher::DeviceModel dev;
    dev.memory_capacity = cap;
    dev.mem_fixed = fixed;
    dev.mem_per_atom = per_atom;
    dev.mem_per_rotbond = per_rot;
    *out = batcher::target_batch_size({0, atom_hi, 0, rot_hi}, dev);  // batcher.cpp:28
    return 0;
  });
}

double vsref_simulate_throughput(long n, double overhead, double service) {
  batcher::DeviceModel dev;
  dev.launch_overhead = overhead;
  dev.service_time_per_class = {service};
  return batcher::simulate_throughput(n, 0, dev);  // batcher.cpp:40
}

// The dock-stage bucket replay of run_campaign (pipeline.cpp:439-461) with
// the reference BatchQueue.  Inputs: per-ligand (atoms, rot); ids are the
// decimal ligand index.  Outputs: in_range[i] (1/0), batch_cls[b],
// batch_len[b], batch_members (flattened ligand indices).  Returns #batches.
int vsref_bucket_replay(const std::int32_t* atoms, const std::int32_t* rot, int n,
                        const std::int32_t* classes, int nc, double cap, double fixed,
                        double per_atom, double per_rot, std::int32_t* in_range,
                        std::int32_t* batch_cls, std::int32_t* batch_len,
                        std::int32_t* batch_members) {
  return guarded([&] {
    std::vector<batcher::SizeClass> cls(nc);
    for (int i = 0; i < nc; ++i) {
      cls[i] = {classes[4 * i], classes[4 * i + 1], classes[4 * i + 2], classes[4 * i + 3]};
    }
    batcher::DeviceModel dev;
    dev.memory_capacity = cap;
    dev.mem_fixed = fixed;
    dev.mem_per_atom = per_atom;
    dev.mem_per_rotbond = per_rot;
    batcher::BatchQueue queue(cls, dev);
    std::vector<batcher::Batch> batches;
    double now = 0.0;
    for (int i = 0; i < n; ++i) {
      chem::Ligand l;
      l.id = std::to_string(i);
      l.heavy_atoms = atoms[i];
      l.rotatable_bonds = rot[i];
      std::size_t c;
      try {
        c = batcher::size_class(l, cls);
      } catch (const batcher::OutOfRange&) {
        in_range[i] = 0;
        continue;
      }
      in_range[i] = 1;
      now += 0.001;
      for (auto& b : queue.flush_aged(now)) batches.push_back(std::move(b));
      if (auto b = queue.enqueue(l.id, c, now)) batches.push_back(std::move(*b));
    }
    for (auto& b : queue.flush_all()) batches.push_back(std::move(b));
    int k = 0;
    for (std::size_t bi = 0; bi < batches.size(); ++bi) {
      batch_cls[bi] = static_cast<int>(batches[bi].cls);
      batch_len[bi] = static_cast<int>(batches[bi].ligand_ids.size());
      for (const auto& id : batches[bi].ligand_ids) batch_members[k++] = std::stoi(id);
    }
    return static_cast<int>(batches.size());
  });
}

// -------------------------------------------------------------------- rng --
// Rng(seed).split(path[0]).split(path[1])... then n x next_u64 (rng.hpp:14-21)
void vsref_rng_u64(std::uint64_t seed, const std::uint64_t* path, int depth, int n,
                   std::uint64_t* out) {
  Rng r(seed);
  for (int d = 0; d < depth; ++d) r = r.split(path[d]);
  for (int i = 0; i < n; ++i) out[i] = r.next_u64();
}

// kinds: 0 next_double, 1 uniform(lo, hi), 2 normal (rng.hpp:24-41)
void vsref_rng_draws(std::uint64_t seed, const std::uint64_t* path, int depth,
                     const std::int32_t* kinds, const double* lo, const double* hi, int n,
                     double* out) {
  Rng r(seed);
  for (int d = 0; d < depth; ++d) r = r.split(path[d]);
  for (int i = 0; i < n; ++i) {
    switch (kinds[i]) {
      case 0: out[i] = r.next_double(); break;
      case 1: out[i] = r.uniform(lo[i], hi[i]); break;
      default: out[i] = r.normal(); break;
    }
  }
}

// The start draws of dock() (dock.cpp:343-354) for every (ligand, restart,
// attempt < attempts), with the reference's own Rng and Quat: rows of
// `stride` floats t[3], q[4] (w, x, y, z; normalized() or identity as
// dock.cpp:351), theta[T], each the FP32 cast of the reference FP64 value.
void vsref_start_draws(const std::uint64_t* seeds, const std::int32_t* n_tors, int n,
                       int restarts, int attempts, const double* lo, const double* hi,
                       int stride, float* out) {
  for (int i = 0; i < n; ++i) {
    Rng root(seeds[i]);
    for (int r = 0; r < restarts; ++r) {
      Rng rng = root.split(static_cast<std::uint64_t>(r));
      for (int a = 0; a < attempts; ++a) {
        float* o = out + ((static_cast<std::size_t>(i) * restarts + r) * attempts + a) * stride;
        const double tx = rng.uniform(lo[0], hi[0]);
        const double ty = rng.uniform(lo[1], hi[1]);
        const double tz = rng.uniform(lo[2], hi[2]);
        Quat q{rng.normal(), rng.normal(), rng.normal(), rng.normal()};
        q = q.norm() > 1e-12 ? q.normalized() : Quat{};
        o[0] = static_cast<float>(tx);
        o[1] = static_cast<float>(ty);
        o[2] = static_cast<float>(tz);
        o[3] = static_cast<float>(q.w);
        o[4] = static_cast<float>(q.x);
        o[5] = static_cast<float>(q.y);
        o[6] = static_cast<float>(q.z);
        for (int j = 0; j < n_tors[i]; ++j)
          o[7 + j] = static_cast<float>(rng.uniform(-3.14159265358979323846, 3.14159265358979323846));
      }
    }
  }
}

// chem::parse_smiles (chem.cpp:109-264): 0 = parsed (atoms / bonds
// counts out), 1 = ParseError (kind, 1-based position out)
int vsref_parse_check(const char* smiles, int* kind, long* pos, int* n_atoms, int* n_bonds) {
  try {
    const chem::MolecularGraph g = chem::parse_smiles(smiles);
    *n_atoms = g.atom_count();
    *n_bonds = static_cast<int>(g.bonds.size());
    return 0;
  } catch (const chem::ParseError& e) {
    *kind = static_cast<int>(e.kind());
    *pos = static_cast<long>(e.position());
    return 1;
  }
}

// dock::pocket_to_json(parse_pocket_json(text)) (dock.cpp:432-474): bytes
// out (NUL-terminated); the length, or -9 when cap is too small
int vsref_pocket_json(const char* text, char* out, int cap) {
  return guarded([&] {
    const std::string s = dock::pocket_to_json(dock::parse_pocket_json(text));
    if (static_cast<int>(s.size()) + 1 > cap) return -9;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return static_cast<int>(s.size());
  });
}

// dock::pose_to_json (dock.cpp:476-489) of the given pose
int vsref_pose_json(const char* ligand, const double* t, const double* q, const double* tors,
                    int n_tors, double geo, int has_rescore, double rescore, char* out, int cap) {
  dock::Pose p;
  p.ligand_id = ligand;
  p.translation = {t[0], t[1], t[2]};
  p.rotation = {q[0], q[1], q[2], q[3]};
  p.torsions.assign(tors, tors + n_tors);
  p.geometric_score = geo;
  if (has_rescore) p.rescore = rescore;
  const std::string s = dock::pose_to_json(p);
  if (static_cast<int>(s.size()) + 1 > cap) return -9;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

// pipeline::CampaignReport::to_json / results_tsv (pipeline.cpp:269-313) of a
// report given as a JSON spec {stages: [[name, in, out, sim, tasks]], ranked:
// [[id, score, delta_g|null]], pairs: [[id, a, b, est, sem, reps, met]],
// trace_path}; which = 0 report JSON, 1 TSV
int vsref_report_bytes(const char* spec, int which, char* out, int cap) {
  return guarded([&] {
    const nlohmann::json j = nlohmann::json::parse(spec);
    pipeline::CampaignReport r;
    for (const auto& s : j.at("stages"))
      r.stages.push_back({s.at(0).get<std::string>(), s.at(1).get<std::size_t>(),
                          s.at(2).get<std::size_t>(), s.at(3).get<double>(),
                          s.at(4).get<std::size_t>()});
    for (const auto& x : j.at("ranked")) {
      pipeline::RankedLigand rl{x.at(0).get<std::string>(), x.at(1).get<double>(), std::nullopt};
      if (!x.at(2).is_null()) rl.delta_g = x.at(2).get<double>();
      r.ranked.push_back(rl);
    }
    for (const auto& p : j.at("pairs")) {
      pipeline::PairResult pr;
      pr.pair_id = p.at(0).get<std::string>();
      pr.ligand_a = p.at(1).get<std::string>();
      pr.ligand_b = p.at(2).get<std::string>();
      pr.result.estimate = p.at(3).get<double>();
      pr.result.sem = p.at(4).get<double>();
      pr.result.replicas = p.at(5).get<int>();
      pr.result.target_met = p.at(6).get<bool>();
      r.pairs.push_back(pr);
    }
    r.trace_path = j.at("trace_path").get<std::string>();
    const std::string s = which == 0 ? r.to_json() : r.results_tsv();
    if (static_cast<int>(s.size()) + 1 > cap) return -9;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return static_cast<int>(s.size());
  });
}

// codec::compress_stream / decompress_stream (codec.cpp:254-289) with a
// dictionary file: text <-> SMZC bytes; the length, or -9 when cap is small
int vsref_smzc_compress(const char* text, long n, const char* dict_path, char* out, long cap) {
  return guarded([&] {
    const codec::Dictionary d = codec::load_dictionary_file(dict_path);
    std::istringstream in(std::string(text, static_cast<size_t>(n)));
    std::ostringstream o;
    codec::compress_stream(in, o, d);
    const std::string s = o.str();
    if (static_cast<long>(s.size()) > cap) return -9;
    std::memcpy(out, s.data(), s.size());
    return static_cast<int>(s.size());
  });
}
int vsref_smzc_decompress(const char* data, long n, const char* dict_path, char* out, long cap) {
  return guarded([&] {
    const codec::Dictionary d = codec::load_dictionary_file(dict_path);
    std::istringstream in(std::string(data, static_cast<size_t>(n)));
    std::ostringstream o;
    codec::decompress_stream(in, o, d);
    const std::string s = o.str();
    if (static_cast<long>(s.size()) > cap) return -9;
    std::memcpy(out, s.data(), s.size());
    return static_cast<int>(s.size());
  });
}
// codec::train_dictionary + save_dictionary (codec.cpp:82-130, 174-186)
int vsref_train_dictionary(const char* text, long n, int max_entries, char* out, long cap) {
  return guarded([&] {
    std::vector<std::string> corpus;
    std::istringstream in(std::string(text, static_cast<size_t>(n)));
    for (std::string line; std::getline(in, line);) corpus.push_back(line);
    const codec::Dictionary d = codec::train_dictionary(corpus, static_cast<size_t>(max_entries));
    std::ostringstream o;
    codec::save_dictionary(d, o);
    const std::string s = o.str();
    if (static_cast<long>(s.size()) > cap) return -9;
    std::memcpy(out, s.data(), s.size());
    return static_cast<int>(s.size());
  });
}

// pipeline::run_campaign (pipeline.cpp:357-590) on a config file, with its
// trace / report / TSV paths redirected; returns the report's stage count
int vsref_run_campaign(const char* cfg_path, const char* trace_path, const char* report_path,
                       const char* tsv_path) {
  return guarded([&] {
    pipeline::CampaignConfig cfg = pipeline::load_config_file(cfg_path);
    cfg.trace_path = trace_path;
    cfg.report_path = report_path;
    cfg.results_tsv_path = tsv_path;
    const pipeline::CampaignReport rep = pipeline::run_campaign(cfg);
    return static_cast<int>(rep.stages.size());
  });
}

// codec::load_dictionary_file (codec.cpp:217-221): entries NUL-separated;
// the total length, or -9 when cap is small
int vsref_dictionary_entries(const char* path, char* out, long cap) {
  return guarded([&] {
    const codec::Dictionary d = codec::load_dictionary_file(path);
    std::string s;
    for (const auto& e : d.entries) {
      s += e;
      s.push_back('\0');
    }
    if (static_cast<long>(s.size()) > cap) return -9;
    std::memcpy(out, s.data(), s.size());
    return static_cast<int>(s.size());
  });
}

// ----------------------------------------------------------------- corpus --
// corpus::random_smiles(Rng(seed).split(i)) (tools/smiles_corpus.hpp:13,51)
int vsref_random_smiles(std::uint64_t seed, std::uint64_t i, char* out, int cap) {
  Rng root(seed);
  Rng r = root.split(i);
  std::string s = corpus::random_smiles(r);
  if (static_cast<int>(s.size()) + 1 > cap) return -9;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

}  // extern "C"
