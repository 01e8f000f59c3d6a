// Host-side C-ABI entry points (capi.h "host-side" section): RNG, ligand
// ingest, batcher, filter, rank.  Pure C++ on the CPU; no CUDA.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <exception>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vscreen_gpu/capi.h"
#include "vs_ingest.h"
#include "vs_rng.h"

using namespace vs;

namespace {

std::vector<std::string> split_blob(const char* blob, int n) {
  std::vector<std::string> out;
  out.reserve(static_cast<std::size_t>(n));
  const char* p = blob;
  for (int i = 0; i < n; ++i) {
    out.emplace_back(p);
    p += out.back().size() + 1;
  }
  return out;
}

struct BuiltLigand {
  int status = 0;
  int rot = 0;
  std::vector<double> coords;
  std::vector<int> cls;
  std::vector<int> bonds;  // (a, b) pairs, kept for the device spring relaxation
  std::uint64_t seed = 0;  // embed seed (VS_EMBED_DEVICE: the placement runs on the device)
  bool place = false;      // built with VS_EMBED_DEVICE
  Topology topo;
};

BuiltLigand build_one(const std::string& smiles, std::uint64_t seed, int iterations) {
  BuiltLigand b;
  try {
    Graph g = parse_smiles(smiles);
    b.rot = rotatable_bond_count(g);
    b.topo = torsion_axes(g);
    b.cls.resize(g.elements.size());
    for (std::size_t i = 0; i < g.elements.size(); ++i) b.cls[i] = element_class(g.elements[i]);
    if (iterations >= 0) {
      b.coords = embed(g, seed, iterations);
    } else if (iterations == VS_EMBED_PLACE_ONLY || iterations == VS_EMBED_DEVICE) {
      if (iterations == VS_EMBED_PLACE_ONLY) {
        b.coords = embed_place(g, seed);
      } else {
        require_connected(g);
        b.coords.assign(3 * g.elements.size(), 0.0);
        b.seed = seed;
        b.place = true;
      }
      b.bonds.reserve(2 * g.bonds.size());
      for (const auto& e : g.bonds) {
        b.bonds.push_back(e.a);
        b.bonds.push_back(e.b);
      }
    } else {
      b.coords.assign(3 * g.elements.size(), 0.0);
    }
  } catch (const ParseFailure&) {
    b.status = VS_ERR_PARSE;
  } catch (const std::exception&) {
    b.status = VS_ERR_DISCONNECTED;
  }
  return b;
}

}  // namespace

struct vs_libbuild {
  std::vector<BuiltLigand> ligs;
};

extern "C" {

int vs_rng_u64(uint64_t seed, const uint64_t* path, int32_t depth, int32_t n, uint64_t* out) {
  HostRng r(seed);
  for (int d = 0; d < depth; ++d) r = r.split(path[d]);
  for (int i = 0; i < n; ++i) out[i] = r.next_u64();
  return VS_OK;
}

int vs_random_smiles(uint64_t seed, uint64_t i, char* out, int32_t cap) {
  const std::string s = random_smiles(seed, i);
  if (static_cast<int>(s.size()) + 1 > cap) return VS_ERR_CAPACITY;
  std::memcpy(out, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

int vs_ligand_build(const char* smiles, uint64_t embed_seed, int32_t iterations,
                    vs_ligand_buf* o) {
  Graph g;
  try {
    g = parse_smiles(smiles);
  } catch (const ParseFailure& e) {
    o->parse_kind = e.kind;
    o->parse_pos = static_cast<int32_t>(e.pos);
    return VS_ERR_PARSE;
  }
  const Topology t = torsion_axes(g);
  const int n = static_cast<int>(g.elements.size());
  int mv = 0;
  for (const auto& a : t.axes) mv += static_cast<int>(a.moving.size());
  o->n_atoms = n;
  o->n_bonds = static_cast<int>(g.bonds.size());
  o->n_tors = static_cast<int>(t.axes.size());
  o->n_moving = mv;
  o->rot_bonds = rotatable_bond_count(g);
  if (n > o->cap_atoms || o->n_bonds > o->cap_bonds || o->n_tors > o->cap_tors ||
      mv > o->cap_moving)
    return VS_ERR_CAPACITY;
  std::vector<double> xyz;
  try {
    xyz = iterations >= 0 ? embed(g, embed_seed, iterations) : std::vector<double>(3 * n, 0.0);
  } catch (const std::exception&) {
    return VS_ERR_DISCONNECTED;
  }
  for (int i = 0; i < n; ++i) {
    for (int c = 0; c < 3; ++c) o->coords[3 * i + c] = xyz[3 * i + c];
    o->atom_class[i] = element_class(g.elements[i]);
    std::memset(o->elements + 3 * i, 0, 3);
    std::memcpy(o->elements + 3 * i, g.elements[i].c_str(), std::min<std::size_t>(2, g.elements[i].size()));
    o->aromatic[i] = g.aromatic[i] ? 1 : 0;
  }
  for (int e = 0; e < o->n_bonds; ++e) {
    o->bonds[3 * e] = g.bonds[e].a;
    o->bonds[3 * e + 1] = g.bonds[e].b;
    o->bonds[3 * e + 2] = g.bonds[e].order;
    o->ring[e] = g.ring[e] ? 1 : 0;
  }
  int k = 0;
  for (int j = 0; j < o->n_tors; ++j) {
    o->axis_a[j] = t.axes[j].a;
    o->axis_b[j] = t.axes[j].b;
    o->moving_count[j] = static_cast<int>(t.axes[j].moving.size());
    for (int m : t.axes[j].moving) o->moving[k++] = m;
  }
  return VS_OK;
}

int vs_libbuild_run(const char* blob, int32_t n, const uint64_t* seeds, int32_t iterations,
                    int32_t threads, vs_libbuild** out) {
  auto* b = new vs_libbuild;
  b->ligs.resize(static_cast<std::size_t>(n));
  const auto smiles = split_blob(blob, n);
  std::atomic<int> next{0};
  auto work = [&] {
    for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1))
      b->ligs[i] = build_one(smiles[i], seeds[i], iterations);
  };
  const int nt = std::max(1, std::min<int>(threads, n));
  if (nt == 1) {
    work();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
  }
  *out = b;
  return VS_OK;
}

int vs_libbuild_sizes(const vs_libbuild* b, int64_t* atoms, int64_t* tors, int64_t* moving) {
  int64_t a = 0, t = 0, m = 0;
  for (const auto& l : b->ligs) {
    if (l.status) continue;
    a += static_cast<int64_t>(l.cls.size());
    t += static_cast<int64_t>(l.topo.axes.size());
    for (const auto& ax : l.topo.axes) m += static_cast<int64_t>(ax.moving.size());
  }
  *atoms = a;
  *tors = t;
  *moving = m;
  return VS_OK;
}

// Failed ligands contribute zero atoms/torsions and a non-zero status.
int vs_libbuild_fetch(const vs_libbuild* b, int32_t* status, int32_t* n_atoms, int32_t* n_tors,
                      int32_t* rot_bonds, double* coords, int32_t* atom_class, int32_t* axis_a,
                      int32_t* axis_b, int32_t* moving_count, int32_t* moving) {
  std::size_t ao = 0, to = 0, mo = 0;
  for (std::size_t i = 0; i < b->ligs.size(); ++i) {
    const auto& l = b->ligs[i];
    status[i] = l.status;
    if (l.status) {
      n_atoms[i] = n_tors[i] = rot_bonds[i] = 0;
      continue;
    }
    n_atoms[i] = static_cast<int32_t>(l.cls.size());
    n_tors[i] = static_cast<int32_t>(l.topo.axes.size());
    rot_bonds[i] = l.rot;
    std::memcpy(coords + 3 * ao, l.coords.data(), l.coords.size() * sizeof(double));
    std::memcpy(atom_class + ao, l.cls.data(), l.cls.size() * sizeof(int32_t));
    ao += l.cls.size();
    for (const auto& ax : l.topo.axes) {
      axis_a[to] = ax.a;
      axis_b[to] = ax.b;
      moving_count[to] = static_cast<int32_t>(ax.moving.size());
      ++to;
      for (int m : ax.moving) moving[mo++] = m;
    }
  }
  return VS_OK;
}

void vs_libbuild_free(vs_libbuild* b) { delete b; }

}  // extern "C"

namespace vs {
int relax_on_device(vs_handle* h, int n, const int64_t* atom_off, const int32_t* n_atoms,
                    double* coords, const int64_t* bond_off, const int32_t* n_bonds,
                    const int32_t* bonds, int iterations, const uint64_t* place_seeds);
void* relax_host_buffer(vs_handle* h, size_t bytes);
}

extern "C" {

namespace {
// the device half of embed_3d for the ligands built with `mode`
// (VS_EMBED_PLACE_ONLY: spring relaxation; VS_EMBED_DEVICE: BFS placement +
// relaxation); coordinates updated in place
int embed_on_device(vs_handle* h, vs_libbuild* b, int32_t iterations, bool place) {
  const int n = static_cast<int>(b->ligs.size());
  std::vector<int64_t> aoff(n + 1, 0), boff(n + 1, 0);
  std::vector<int32_t> na(n, 0), nb(n, 0);
  std::vector<uint64_t> seeds(place ? std::max(n, 1) : 0, 0);
  for (int i = 0; i < n; ++i) {
    const auto& l = b->ligs[i];
    const bool use = l.status == 0 && l.place == place && !l.bonds.empty();
    na[i] = use ? static_cast<int32_t>(l.coords.size() / 3) : 0;
    nb[i] = use ? static_cast<int32_t>(l.bonds.size() / 2) : 0;
    aoff[i + 1] = aoff[i] + na[i];
    boff[i + 1] = boff[i] + nb[i];
    if (place) seeds[i] = l.seed;
  }
  // one pinned block: xyz (FP64) then the bonds, filled straight from the
  // per-ligand vectors
  const size_t xyz_n = static_cast<size_t>(3 * std::max<int64_t>(aoff[n], 1));
  const size_t bd_n = static_cast<size_t>(2 * std::max<int64_t>(boff[n], 1));
  unsigned char* pin = static_cast<unsigned char*>(
      relax_host_buffer(h, xyz_n * sizeof(double) + bd_n * sizeof(int32_t)));
  if (!pin) return VS_ERR_CUDA;
  double* xyz = reinterpret_cast<double*>(pin);
  int32_t* bd = reinterpret_cast<int32_t*>(pin + xyz_n * sizeof(double));
  for (int i = 0; i < n; ++i) {
    if (!na[i]) continue;
    const auto& l = b->ligs[i];
    std::memcpy(xyz + 3 * aoff[i], l.coords.data(), l.coords.size() * sizeof(double));
    std::memcpy(bd + 2 * boff[i], l.bonds.data(), l.bonds.size() * sizeof(int32_t));
  }
  const int rc = relax_on_device(h, n, aoff.data(), na.data(), xyz, boff.data(), nb.data(), bd,
                                 iterations, place ? seeds.data() : nullptr);
  if (rc) return rc;
  for (int i = 0; i < n; ++i) {
    if (!na[i]) continue;
    auto& l = b->ligs[i];
    std::memcpy(l.coords.data(), xyz + 3 * aoff[i], l.coords.size() * sizeof(double));
    l.bonds.clear();
    l.bonds.shrink_to_fit();
    l.place = false;
  }
  return VS_OK;
}
}  // namespace

// Spring relaxation (chem.cpp:355-392, 434-445) of every ligand built with
// iterations = VS_EMBED_PLACE_ONLY, on the device; coordinates updated in place.
int vs_libbuild_relax(vs_handle* h, vs_libbuild* b, int32_t iterations) {
  return embed_on_device(h, b, iterations, false);
}

// The whole embed_3d (chem.cpp:404-446: BFS placement with the Rng jitter,
// then the relaxation) of every ligand built with VS_EMBED_DEVICE.
int vs_libbuild_embed(vs_handle* h, vs_libbuild* b, int32_t iterations) {
  return embed_on_device(h, b, iterations, true);
}

// Scan corpus::random_smiles(Rng(seed).split(i)) for i = 0, 1, ... and keep
// the first n_want whose heavy atoms lie in [atom_lo, atom_hi] and torsion
// axes in [tors_lo, tors_hi] (the C1-C4 library filters).
int vs_corpus_select(uint64_t seed, int64_t n_want, int32_t atom_lo, int32_t atom_hi,
                     int32_t tors_lo, int32_t tors_hi, int64_t max_scan, int32_t threads,
                     int64_t* out_index) {
  const int nt = std::max(1, threads);
  const int64_t chunk = 4096;
  int64_t found = 0;
  std::vector<char> ok(static_cast<std::size_t>(chunk));
  for (int64_t base = 0; base < max_scan && found < n_want; base += chunk) {
    std::atomic<int64_t> next{0};
    auto work = [&] {
      for (int64_t k = next.fetch_add(1); k < chunk; k = next.fetch_add(1)) {
        ok[k] = 0;
        try {
          const Graph g = parse_smiles(random_smiles(seed, static_cast<uint64_t>(base + k)));
          const int n = static_cast<int>(g.elements.size());
          const int t = static_cast<int>(torsion_axes(g).axes.size());
          ok[k] = (n >= atom_lo && n <= atom_hi && t >= tors_lo && t <= tors_hi) ? 1 : 0;
        } catch (const std::exception&) {
        }
      }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
    for (int64_t k = 0; k < chunk && found < n_want && base + k < max_scan; ++k)
      if (ok[k]) out_index[found++] = base + k;
  }
  return static_cast<int>(found);
}

// C4 population: concatenate consecutive corpus entries until the graph has
// >= atom_lo heavy atoms; keep the string when atoms <= atom_hi and the
// torsion axes lie in [tors_lo, tors_hi].  Writes [first entry, count) per
// accepted ligand; returns how many were found.
int vs_flexible_select(uint64_t seed, int32_t n_want, int32_t atom_lo, int32_t atom_hi,
                       int32_t tors_lo, int32_t tors_hi, int64_t max_scan, int64_t* first,
                       int32_t* count) {
  // The corpus index space is cut into fixed chunks of kChunk entries; each
  // chunk is scanned on its own from its first entry (a candidate may read
  // past the chunk end), so the selection is independent of the thread
  // count.  Within a chunk: entries are appended while the summed per-entry
  // heavy-atom count is < atom_lo (an entry that does not parse rejects the
  // candidate, the next one starts after it); the concatenation is parsed
  // once, and kept when its atoms and torsion axes fall inside the bounds.
  constexpr int64_t kChunk = 16384;
  const int64_t n_chunks = (max_scan + kChunk - 1) / kChunk;
  if (n_want <= 0 || n_chunks <= 0) return 0;
  std::vector<std::vector<std::pair<int64_t, int32_t>>> got(static_cast<std::size_t>(n_chunks));
  std::vector<char> done(static_cast<std::size_t>(n_chunks), 0);
  std::atomic<int64_t> next{0};
  std::atomic<bool> enough{false};
  std::mutex mu;
  int64_t prefix = 0, prefix_found = 0;  // completed chunk prefix (under mu)
  auto scan = [&](int64_t c) {
    std::vector<std::pair<int64_t, int32_t>> out;
    const int64_t end = std::min(max_scan, (c + 1) * kChunk);
    int64_t i = c * kChunk;
    while (i < end) {
      const int64_t start = i;
      std::string s;
      int na = 0;
      bool ok = true;
      while (na < atom_lo && i < max_scan) {
        const std::string e = random_smiles(seed, static_cast<uint64_t>(i++));
        try {
          na += static_cast<int>(parse_smiles(e).elements.size());
        } catch (const std::exception&) {
          ok = false;
          break;
        }
        s += e;
      }
      if (!ok || na < atom_lo || na > atom_hi) continue;
      try {
        const Graph g = parse_smiles(s);
        const int n2 = static_cast<int>(g.elements.size());
        const int nt = static_cast<int>(torsion_axes(g).axes.size());
        if (n2 >= atom_lo && n2 <= atom_hi && nt >= tors_lo && nt <= tors_hi)
          out.emplace_back(start, static_cast<int32_t>(i - start));
      } catch (const std::exception&) {
      }
    }
    std::lock_guard<std::mutex> lk(mu);
    got[static_cast<std::size_t>(c)] = std::move(out);
    done[static_cast<std::size_t>(c)] = 1;
    while (prefix < n_chunks && done[static_cast<std::size_t>(prefix)]) {
      prefix_found += static_cast<int64_t>(got[static_cast<std::size_t>(prefix)].size());
      ++prefix;
    }
    if (prefix_found >= n_want) enough = true;
  };
  auto work = [&] {
    while (!enough) {
      const int64_t c = next.fetch_add(1);
      if (c >= n_chunks) break;
      scan(c);
    }
  };
  const int nt = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()),
                                           static_cast<int>(std::min<int64_t>(n_chunks, 256))));
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) pool.emplace_back(work);
  for (auto& th : pool) th.join();
  int found = 0;
  for (int64_t c = 0; c < prefix && found < n_want; ++c)
    for (const auto& fc : got[static_cast<std::size_t>(c)]) {
      if (found >= n_want) break;
      first[found] = fc.first;
      count[found] = fc.second;
      ++found;
    }
  return found;
}

// vs_libbuild_run over corpus entries given by index (SMILES generated here).
int vs_libbuild_corpus(uint64_t seed, const int64_t* index, int32_t n, const uint64_t* embed_seeds,
                       int32_t iterations, int32_t threads, vs_libbuild** out) {
  auto* b = new vs_libbuild;
  b->ligs.resize(static_cast<std::size_t>(n));
  std::atomic<int> next{0};
  auto work = [&] {
    for (int i = next.fetch_add(1); i < n; i = next.fetch_add(1))
      b->ligs[i] = build_one(random_smiles(seed, static_cast<uint64_t>(index[i])), embed_seeds[i],
                             iterations);
  };
  const int nt = std::max(1, std::min<int>(threads, n));
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) pool.emplace_back(work);
  for (auto& th : pool) th.join();
  *out = b;
  return VS_OK;
}

// ---------------------------------------------------------------- batcher --
int vs_default_classes(vs_size_class* out, int32_t cap) {
  static const int atoms[4] = {1, 20, 40, 80};  // batcher.cpp:9-10
  static const int rots[3] = {0, 4, 12};
  if (cap < 6) return VS_ERR_CAPACITY;
  int k = 0;
  for (int ai = 0; ai < 3; ++ai)
    for (int ri = 0; ri < 2; ++ri) out[k++] = {atoms[ai], atoms[ai + 1], rots[ri], rots[ri + 1]};
  return k;
}

int vs_size_class_of(int32_t atoms, int32_t rot, const vs_size_class* c, int32_t n) {
  for (int i = 0; i < n; ++i) {
    if (atoms >= c[i].atom_lo && atoms < c[i].atom_hi && rot >= c[i].rot_lo && rot < c[i].rot_hi)
      return i;
  }
  return VS_ERR_OUT_OF_RANGE;
}

int vs_target_batch_size(const vs_size_class* cls, double cap, double fixed, double per_atom,
                         double per_rot, int64_t* out) {
  const double item = per_atom * cls->atom_hi + per_rot * cls->rot_hi;
  const double budget = cap - fixed;
  if (item > budget) return VS_ERR_ITEM_TOO_LARGE;
  if (item <= 0.0) {
    *out = 1;
    return VS_OK;
  }
  const auto n = static_cast<int64_t>(std::floor(budget / item));
  *out = n < 1 ? 1 : n;
  return VS_OK;
}

double vs_simulate_throughput(int64_t n_items, double overhead, double service) {
  const double n = static_cast<double>(n_items);
  return n / (overhead + n * service);
}

int vs_bucket_replay(const int32_t* atoms, const int32_t* rot, int32_t n,
                     const vs_size_class* classes, int32_t nc, double cap, double fixed,
                     double per_atom, double per_rot, double max_age, int32_t* in_range,
                     int32_t* batch_cls, int32_t* batch_len, int32_t* members) {
  std::vector<int64_t> target(static_cast<std::size_t>(nc));
  for (int c = 0; c < nc; ++c) {
    const int rc = vs_target_batch_size(&classes[c], cap, fixed, per_atom, per_rot, &target[c]);
    if (rc) return rc;
  }
  struct Pending {
    std::vector<int> ids;
    std::vector<double> t;
    std::size_t head = 0;
  };
  std::vector<Pending> buf(static_cast<std::size_t>(nc));
  int nb = 0, nm = 0;
  auto emit = [&](int c) {
    batch_cls[nb] = c;
    batch_len[nb] = static_cast<int32_t>(buf[c].ids.size());
    for (int id : buf[c].ids) members[nm++] = id;
    ++nb;
    buf[c].ids.clear();
    buf[c].t.clear();
  };
  double now = 0.0;
  for (int i = 0; i < n; ++i) {
    const int c = vs_size_class_of(atoms[i], rot[i], classes, nc);
    if (c < 0) {
      in_range[i] = 0;
      continue;
    }
    in_range[i] = 1;
    now += 0.001;  // pipeline.cpp:453
    for (int k = 0; k < nc; ++k) {  // flush_aged (batcher.cpp:69-77)
      if (!buf[k].ids.empty() && now - buf[k].t.front() > max_age) emit(k);
    }
    buf[c].ids.push_back(i);  // enqueue (batcher.cpp:59-67)
    buf[c].t.push_back(now);
    if (static_cast<int64_t>(buf[c].ids.size()) >= target[c]) emit(c);
  }
  for (int k = 0; k < nc; ++k)
    if (!buf[k].ids.empty()) emit(k);
  return nb;
}

int vs_campaign_seeds(uint64_t master, int32_t stage, const int32_t* in_range, int32_t n,
                      uint64_t* out) {
  const HostRng st = HostRng(master).split(static_cast<std::uint64_t>(stage));
  std::uint64_t idx = 0;
  for (int i = 0; i < n; ++i) {
    if (in_range && !in_range[i]) {
      out[i] = 0;
      continue;
    }
    HostRng r = st.split(idx++);
    out[i] = r.next_u64();
  }
  return VS_OK;
}

int vs_topk_merge_host(const uint64_t* keys, int64_t n, int32_t k, uint64_t* out) {
  if (k < 0 || n < 0) return VS_ERR_INVALID_ARGUMENT;
  // keys are unique per ligand (id_rank in the low word), so the k smallest
  // are a set; dropped ligands (~0) sort last
  std::vector<uint64_t> v(keys, keys + n);
  const size_t m = std::min<size_t>(static_cast<size_t>(k), v.size());
  std::partial_sort(v.begin(), v.begin() + static_cast<std::ptrdiff_t>(m), v.end());
  for (size_t i = 0; i < static_cast<size_t>(k); ++i) out[i] = i < m ? v[i] : ~0ull;
  return VS_OK;
}

int vs_filter_poses(const double* scores, int32_t n, int64_t keep_top, double min_score,
                    int32_t* out_idx) {
  std::vector<int32_t> idx;
  for (int i = 0; i < n; ++i)
    if (scores[i] >= min_score) idx.push_back(i);
  if (static_cast<int64_t>(idx.size()) > keep_top) {
    std::stable_sort(idx.begin(), idx.end(),
                     [&](int32_t a, int32_t b) { return scores[a] > scores[b]; });
    idx.resize(static_cast<std::size_t>(keep_top));
    std::sort(idx.begin(), idx.end());
  }
  std::copy(idx.begin(), idx.end(), out_idx);
  return static_cast<int>(idx.size());
}

int vs_id_ranks(const char* blob, int32_t n, uint32_t* out_rank) {
  const auto ids = split_blob(blob, n);
  std::vector<int32_t> ord(static_cast<std::size_t>(n));
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return ids[a] < ids[b]; });
  for (int r = 0; r < n; ++r) out_rank[ord[r]] = static_cast<uint32_t>(r);
  return VS_OK;
}

// rank_ligands: std::map iteration (bytewise id order; a repeated id keeps
// its last score, as map operator[] does) then stable sort by score desc.
int vs_rank_ligands(const char* blob, const double* scores, int32_t n, int32_t* out_order) {
  const auto ids = split_blob(blob, n);
  std::vector<int32_t> ord(static_cast<std::size_t>(n));
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) { return ids[a] < ids[b]; });
  std::vector<int32_t> uniq;
  for (std::size_t k = 0; k < ord.size(); ++k) {
    if (k + 1 < ord.size() && ids[ord[k]] == ids[ord[k + 1]]) continue;  // last one wins
    uniq.push_back(ord[k]);
  }
  std::stable_sort(uniq.begin(), uniq.end(),
                   [&](int32_t a, int32_t b) { return scores[a] > scores[b]; });
  std::copy(uniq.begin(), uniq.end(), out_order);
  return static_cast<int>(uniq.size());
}

}  // extern "C"
