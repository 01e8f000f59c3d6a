// Ligand ingest on the host: the path's upstream inputs (SURVEY §8 rows A7,
// A21 and "next" rows f1/f2), restated so the framework can load libraries
// and synthesise benchmark inputs without the reference.
//
//   parse            restricted SMILES grammar      (chem.cpp:109-264)
//   ring flags       bridge test                    (chem.cpp:266-317)
//   rotatable bonds  single, acyclic, deg >= 2      (chem.cpp:319-331)
//   torsion axes     bond order, b-side moving set  (dock.cpp:234-270)
//   embed            BFS tetrahedral + springs      (chem.cpp:343-446)
//   corpus           drug-like sampler              (tools/smiles_corpus.hpp:13-60)
//   library text     SMILES<TAB>ID records          (chem.cpp:448-476)
//
// The embedding is FP64 with the reference's operation order, so the same
// (SMILES, seed) yields bit-identical coordinates (tests/test_ingest.py).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "vs_ingest.h"
#include "vs_rng.h"

namespace vs {

namespace {

struct RingOpen {
  int atom = -1;
  int order = 0;  // 0 = unspecified
  std::size_t pos = 0;
};

int bond_char_order(char c) {
  return c == '-' ? 1 : c == '=' ? 2 : c == '#' ? 3 : 0;
}

}  // namespace

ParseFailure::ParseFailure(int kind, std::size_t pos, const std::string& msg)
    : std::runtime_error(msg), kind(kind), pos(pos) {}

// ----------------------------------------------------------------- parse --
Graph parse_smiles(const std::string& text) {
  Graph g;
  if (text.empty()) throw ParseFailure(kUnknownToken, 1, "empty input");
  int prev = -1;
  int pending = 0;
  std::size_t pending_pos = 0;
  std::vector<std::pair<int, std::size_t>> branches;
  std::array<RingOpen, 100> rings{};

  auto connect = [&](int a, int b, int order, std::size_t pos) {
    if (a == b) throw ParseFailure(kUnclosedRingBond, pos, "ring bond to the same atom");
    for (const auto& e : g.bonds) {
      if ((e.a == a && e.b == b) || (e.a == b && e.b == a))
        throw ParseFailure(kUnclosedRingBond, pos, "duplicate bond");
    }
    g.bonds.push_back({a, b, order});
  };
  auto atom = [&](const char* el, bool aromatic, std::size_t pos) {
    const int idx = static_cast<int>(g.elements.size());
    g.elements.emplace_back(el);
    g.aromatic.push_back(aromatic);
    if (prev >= 0) {
      const int order = pending ? pending : (aromatic && g.aromatic[prev]) ? 4 : 1;
      connect(prev, idx, order, pos);
    } else if (pending) {
      throw ParseFailure(kUnknownToken, pending_pos, "bond before any atom");
    }
    pending = 0;
    prev = idx;
  };
  auto ring = [&](int num, std::size_t pos) {
    if (prev < 0) throw ParseFailure(kUnknownToken, pos, "ring closure before any atom");
    RingOpen& r = rings[static_cast<std::size_t>(num)];
    if (r.atom < 0) {
      r = {prev, pending, pos};
      pending = 0;
      return;
    }
    if (r.order && pending && r.order != pending)
      throw ParseFailure(kUnclosedRingBond, pos, "conflicting ring bond orders");
    int order = pending ? pending
                : r.order ? r.order
                : (g.aromatic[r.atom] && g.aromatic[prev]) ? 4
                                                           : 1;
    connect(r.atom, prev, order, pos);
    r = RingOpen{};
    pending = 0;
  };

  const std::size_t n = text.size();
  for (std::size_t i = 0; i < n;) {
    const char c = text[i];
    const std::size_t pos = i + 1;
    const char nx = i + 1 < n ? text[i + 1] : '\0';
    if (c == 'C' && nx == 'l') {
      atom("Cl", false, pos);
      i += 2;
      continue;
    }
    if (c == 'B' && nx == 'r') {
      atom("Br", false, pos);
      i += 2;
      continue;
    }
    if (std::strchr("BCNOPSFI", c) && c != '\0') {
      const char el[2] = {c, '\0'};
      atom(el, false, pos);
      ++i;
      continue;
    }
    if (std::strchr("bcnops", c) && c != '\0') {
      const char el[2] = {static_cast<char>(c - 'a' + 'A'), '\0'};
      atom(el, true, pos);
      ++i;
      continue;
    }
    if (const int bo = bond_char_order(c)) {
      if (pending) throw ParseFailure(kUnknownToken, pos, "two bond symbols in a row");
      if (prev < 0) throw ParseFailure(kUnknownToken, pos, "bond before any atom");
      pending = bo;
      pending_pos = pos;
      ++i;
      continue;
    }
    switch (c) {
      case '(':
        if (prev < 0) throw ParseFailure(kUnbalancedBranch, pos, "branch before any atom");
        if (pending) throw ParseFailure(kUnknownToken, pos, "bond before branch open");
        branches.emplace_back(prev, pos);
        ++i;
        continue;
      case ')':
        if (branches.empty()) throw ParseFailure(kUnbalancedBranch, pos, "unmatched ')'");
        if (pending) throw ParseFailure(kUnknownToken, pos, "dangling bond before ')'");
        prev = branches.back().first;
        branches.pop_back();
        ++i;
        continue;
      case '%': {
        const bool ok = i + 2 < n && std::isdigit(static_cast<unsigned char>(text[i + 1])) &&
                        std::isdigit(static_cast<unsigned char>(text[i + 2]));
        if (!ok) throw ParseFailure(kUnknownToken, pos, "'%' needs two digits");
        const int num = (text[i + 1] - '0') * 10 + (text[i + 2] - '0');
        if (num < 10) throw ParseFailure(kUnknownToken, pos, "'%' ring numbers start at 10");
        ring(num, pos);
        i += 3;
        continue;
      }
      default:
        break;
    }
    if (c >= '1' && c <= '9') {
      ring(c - '0', pos);
      ++i;
      continue;
    }
    throw ParseFailure(kUnknownToken, pos, std::string("unexpected character '") + c + "'");
  }
  if (pending) throw ParseFailure(kUnknownToken, pending_pos, "dangling bond at end of input");
  if (!branches.empty()) throw ParseFailure(kUnbalancedBranch, branches.front().second, "unclosed '('");
  for (const RingOpen& r : rings) {
    if (r.atom >= 0) throw ParseFailure(kUnclosedRingBond, r.pos, "unclosed ring bond");
  }
  g.ring = ring_bond_flags(g);
  return g;
}

// A bond lies on a cycle iff removing it keeps its endpoints connected
// (chem.cpp:266-317 finds the same set with Tarjan's bridge DFS).
std::vector<bool> ring_bond_flags(const Graph& g) {
  const int n = static_cast<int>(g.elements.size());
  const int m = static_cast<int>(g.bonds.size());
  std::vector<bool> ring(static_cast<std::size_t>(m), false);
  if (n == 0 || m == 0) return ring;
  std::vector<std::vector<std::pair<int, int>>> adj(static_cast<std::size_t>(n));
  for (int e = 0; e < m; ++e) {
    adj[g.bonds[e].a].push_back({g.bonds[e].b, e});
    adj[g.bonds[e].b].push_back({g.bonds[e].a, e});
  }
  std::vector<int> seen(static_cast<std::size_t>(n), -1);
  std::vector<int> stack;
  for (int e = 0; e < m; ++e) {
    // reachability from a to b avoiding bond e
    const int src = g.bonds[e].a, dst = g.bonds[e].b;
    stack.assign(1, src);
    seen[src] = e;
    bool found = false;
    while (!stack.empty() && !found) {
      const int v = stack.back();
      stack.pop_back();
      for (const auto& [w, f] : adj[v]) {
        if (f == e || seen[w] == e) continue;
        if (w == dst) {
          found = true;
          break;
        }
        seen[w] = e;
        stack.push_back(w);
      }
    }
    ring[static_cast<std::size_t>(e)] = found;
  }
  return ring;
}

std::vector<int> degrees(const Graph& g) {
  std::vector<int> d(g.elements.size(), 0);
  for (const auto& b : g.bonds) {
    ++d[b.a];
    ++d[b.b];
  }
  return d;
}

int rotatable_bond_count(const Graph& g) {
  const auto deg = degrees(g);
  int count = 0;
  for (std::size_t e = 0; e < g.bonds.size(); ++e) {
    const auto& b = g.bonds[e];
    if (b.order == 1 && !g.ring[e] && deg[b.a] >= 2 && deg[b.b] >= 2) ++count;
  }
  return count;
}

Topology torsion_axes(const Graph& g) {
  Topology t;
  const auto deg = degrees(g);
  const std::size_t n = g.elements.size();
  std::vector<std::vector<int>> adj(n);
  for (const auto& b : g.bonds) {
    adj[b.a].push_back(b.b);
    adj[b.b].push_back(b.a);
  }
  std::vector<char> seen(n);
  for (std::size_t e = 0; e < g.bonds.size(); ++e) {
    const auto& b = g.bonds[e];
    if (b.order != 1 || g.ring[e] || deg[b.a] < 2 || deg[b.b] < 2) continue;
    Axis ax;
    ax.a = b.a;
    ax.b = b.b;
    std::fill(seen.begin(), seen.end(), 0);
    seen[b.a] = seen[b.b] = 1;
    std::vector<int> todo{b.b};
    while (!todo.empty()) {
      const int v = todo.back();
      todo.pop_back();
      for (int w : adj[v]) {
        if (seen[w]) continue;
        seen[w] = 1;
        ax.moving.push_back(w);
        todo.push_back(w);
      }
    }
    std::sort(ax.moving.begin(), ax.moving.end());
    t.axes.push_back(std::move(ax));
  }
  return t;
}

// ----------------------------------------------------------------- embed --
namespace {

struct V3 {
  double x, y, z;
};
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator*(V3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }
inline double norm(V3 a) { return std::sqrt(a.x * a.x + a.y * a.y + a.z * a.z); }

void springs(const Graph& g, std::vector<V3>& pos, int iterations) {
  const std::size_t n = pos.size();
  std::vector<char> bonded(n * n, 0);
  for (const auto& b : g.bonds) bonded[b.a * n + b.b] = bonded[b.b * n + b.a] = 1;
  std::vector<V3> grad(n);
  for (int it = 0; it < iterations; ++it) {
    std::fill(grad.begin(), grad.end(), V3{0, 0, 0});
    for (const auto& b : g.bonds) {  // bonded rest length 1.5
      const V3 d = pos[b.a] - pos[b.b];
      const double len = norm(d);
      if (len < 1e-12) continue;
      const V3 dg = d * (2.0 * (len - 1.5) / len);
      grad[b.a] = grad[b.a] + dg;
      grad[b.b] = grad[b.b] - dg;
    }
    for (std::size_t a = 0; a < n; ++a) {  // non-bonded repulsion below 1.0
      for (std::size_t b = a + 1; b < n; ++b) {
        if (bonded[a * n + b]) continue;
        const V3 d = pos[a] - pos[b];
        const double len = norm(d);
        if (len >= 1.0 || len < 1e-12) continue;
        const V3 dg = d * (-2.0 * (1.0 - len) / len);
        grad[a] = grad[a] + dg;
        grad[b] = grad[b] - dg;
      }
    }
    for (std::size_t a = 0; a < n; ++a) {
      V3 st = grad[a] * (-0.05);
      const double sn = norm(st);
      if (sn > 0.2) st = st * (0.2 / sn);
      pos[a] = pos[a] + st;
    }
  }
}

double closest_pair(const std::vector<V3>& pos) {
  double best = std::numeric_limits<double>::infinity();
  for (std::size_t a = 0; a < pos.size(); ++a)
    for (std::size_t b = a + 1; b < pos.size(); ++b) best = std::min(best, norm(pos[a] - pos[b]));
  return best;
}

}  // namespace

// BFS tetrahedral placement with RNG jitter (chem.cpp:406-432): the embed
// before the spring relaxation; throws on a disconnected graph.
std::vector<double> embed_place(const Graph& g, std::uint64_t seed) {
  return embed(g, seed, -1);
}

std::vector<double> embed(const Graph& g, std::uint64_t seed, int iterations) {
  const std::size_t n = g.elements.size();
  std::vector<V3> pos(n, V3{0, 0, 0});
  if (n == 0) return {};
  std::vector<std::vector<int>> adj(n);
  for (const auto& b : g.bonds) {
    adj[b.a].push_back(b.b);
    adj[b.b].push_back(b.a);
  }
  {  // connectivity (chem.cpp:408)
    std::vector<char> vis(n, 0);
    std::vector<int> st{0};
    vis[0] = 1;
    std::size_t cnt = 1;
    while (!st.empty()) {
      const int v = st.back();
      st.pop_back();
      for (int w : adj[v])
        if (!vis[w]) {
          vis[w] = 1;
          ++cnt;
          st.push_back(w);
        }
    }
    if (cnt != n) throw std::runtime_error("graph is not connected");
  }
  const double s3 = std::sqrt(3.0);
  const V3 tetra[4] = {{1 / s3, 1 / s3, 1 / s3},
                       {1 / s3, -1 / s3, -1 / s3},
                       {-1 / s3, 1 / s3, -1 / s3},
                       {-1 / s3, -1 / s3, 1 / s3}};
  HostRng rng = HostRng(seed).split(0x3d);
  std::vector<char> placed(n, 0);
  std::vector<int> children(n, 0);
  std::vector<int> bfs{0};
  placed[0] = 1;
  for (std::size_t qi = 0; qi < bfs.size(); ++qi) {
    const int v = bfs[qi];
    for (int w : adj[v]) {
      if (placed[w]) continue;
      const V3 dir = tetra[children[v] % 4];
      V3 jit;
      jit.x = rng.normal();
      jit.y = rng.normal();
      jit.z = rng.normal();
      pos[w] = (pos[v] + dir * 1.5) + jit * 0.05;
      ++children[v];
      placed[w] = 1;
      bfs.push_back(w);
    }
  }
  if (iterations >= 0) {  // iterations < 0: placement only (embed_place)
    springs(g, pos, iterations);
    for (int round = 0; round < 20 && n > 1 && closest_pair(pos) < 0.5; ++round)
      springs(g, pos, 50);
  }
  std::vector<double> out(3 * n);
  for (std::size_t i = 0; i < n; ++i) {
    out[3 * i] = pos[i].x;
    out[3 * i + 1] = pos[i].y;
    out[3 * i + 2] = pos[i].z;
  }
  return out;
}

int element_class(const std::string& el) {
  if (el == "C") return 1;
  if (el == "N" || el == "O") return 2;
  return 0;
}

// ---------------------------------------------------------------- corpus --
std::string random_smiles(std::uint64_t seed, std::uint64_t index) {
  static const char* const kInline[] = {
      "C",        "CC",       "CCC",      "CCCC",    "N",        "O",
      "S",        "P",        "B",        "CN",      "CO",       "CS",
      "C=C",      "C#N",      "C#C",      "C=N",     "c1ccccc1", "c1ccncc1",
      "c1cnccc1", "c1ccsc1",  "c1ccoc1",  "c1cncnc1", "C1CCCCC1", "C1CCNCC1",
      "C1CCOCC1", "C1CCCC1",  "C1CCC1",   "C1CC1",   "C=O",      "CCl",
      "CBr",      "CF",       "CI",       "OCC",     "NC",       "SC",
      "NCC",      "OCO",      "NCN",      "CC=O",    "CCN",      "CCO",
      "C=CC",     "CC#N",     "SCC",      "NCO"};
  static const char* const kBranch[] = {"C",   "CC",  "CCC", "O",   "N",   "S",   "=O",
                                        "=C",  "=N",  "#N",  "Cl",  "Br",  "F",   "I",
                                        "OC",  "NC",  "CN",  "CO",  "C=O", "CCl", "OCC",
                                        "C#N", "NCC", "CCO", "CF",  "SC"};
  static const char kChain[] = {'C', 'C', 'C', 'N', 'O', 'S'};
  constexpr std::uint64_t nInline = sizeof(kInline) / sizeof(kInline[0]);
  constexpr std::uint64_t nBranch = sizeof(kBranch) / sizeof(kBranch[0]);
  HostRng rng = HostRng(seed).split(index);
  std::string s = kInline[rng.next_below(nInline)];
  const std::uint64_t units = 1 + rng.next_below(6);
  for (std::uint64_t u = 0; u < units; ++u) {
    const double roll = rng.next_double();
    if (roll < 0.3) {
      s += '(';
      s += kBranch[rng.next_below(nBranch)];
      s += ')';
    } else if (roll < 0.45) {
      const std::uint64_t len = 2 + rng.next_below(6);
      for (std::uint64_t k = 0; k < len; ++k) s += kChain[rng.next_below(6)];
    } else {
      s += kInline[rng.next_below(nInline)];
    }
  }
  return s;
}

}  // namespace vs
