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

ParseFailure::ParseFailure(int kind, std::size_t pos, const std::string& msg)
    : std::runtime_error(msg), kind(kind), pos(pos) {}

// ----------------------------------------------------------------- parse --
// The contract (chem.cpp:109-264): the organic-subset grammar, implicit
// bond orders (aromatic-aromatic -> aromatic, else single), and which error
// kind and 1-based position each malformed input reports, in text order.
// Built here as a streaming lexer (one token per call, so a lexical error
// never pre-empts an earlier structural one) driving a small graph-builder
// state machine.
namespace {

enum class Tok { Atom, Bond, Open, Close, Ring, End };

struct Token {
  Tok kind = Tok::End;
  std::size_t pos = 0;  // 1-based offset of the token's first byte
  char sym[3] = {0, 0, 0};
  bool aromatic = false;
  int value = 0;  // bond order, or ring-closure number
};

class Lexer {
 public:
  explicit Lexer(const std::string& s) : s_(s) {}

  Token next() {
    Token t;
    t.pos = i_ + 1;
    if (i_ >= s_.size()) return t;
    const char c = s_[i_];
    const char d = i_ + 1 < s_.size() ? s_[i_ + 1] : '\0';
    if ((c == 'C' && d == 'l') || (c == 'B' && d == 'r')) {  // two-letter halogens first
      t.kind = Tok::Atom;
      t.sym[0] = c;
      t.sym[1] = d;
      i_ += 2;
      return t;
    }
    switch (c) {
      case 'B': case 'C': case 'N': case 'O': case 'P': case 'S': case 'F': case 'I':
        t.kind = Tok::Atom;
        t.sym[0] = c;
        break;
      case 'b': case 'c': case 'n': case 'o': case 'p': case 's':
        t.kind = Tok::Atom;
        t.sym[0] = static_cast<char>(c - 32);  // stored uppercase (chem.cpp:197)
        t.aromatic = true;
        break;
      case '-': t.kind = Tok::Bond; t.value = 1; break;
      case '=': t.kind = Tok::Bond; t.value = 2; break;
      case '#': t.kind = Tok::Bond; t.value = 3; break;
      case '(': t.kind = Tok::Open; break;
      case ')': t.kind = Tok::Close; break;
      case '%': {
        const bool two = i_ + 2 < s_.size() && digit(s_[i_ + 1]) && digit(s_[i_ + 2]);
        if (!two) throw ParseFailure(kUnknownToken, t.pos, "'%' must be followed by two digits");
        t.value = 10 * (s_[i_ + 1] - '0') + (s_[i_ + 2] - '0');
        if (t.value < 10)
          throw ParseFailure(kUnknownToken, t.pos, "two-digit ring label below 10");
        t.kind = Tok::Ring;
        i_ += 3;
        return t;
      }
      default:
        if (c >= '1' && c <= '9') {
          t.kind = Tok::Ring;
          t.value = c - '0';
          break;
        }
        throw ParseFailure(kUnknownToken, t.pos, std::string("character '") + c + "' not in the grammar");
    }
    ++i_;
    return t;
  }

 private:
  static bool digit(char c) { return c >= '0' && c <= '9'; }
  const std::string& s_;
  std::size_t i_ = 0;
};

class GraphBuilder {
 public:
  explicit GraphBuilder(Graph& g) : g_(g) { open_.fill(Label{}); }

  void atom(const Token& t) {
    const int id = static_cast<int>(g_.elements.size());
    g_.elements.emplace_back(t.sym);
    g_.aromatic.push_back(t.aromatic);
    if (anchor_ < 0) {
      if (bond_) throw ParseFailure(kUnknownToken, bond_pos_, "bond symbol with no atom before it");
    } else {
      add_bond(anchor_, id, bond_ ? bond_ : implicit(anchor_, id), t.pos);
    }
    bond_ = 0;
    anchor_ = id;
  }

  void bond(const Token& t) {
    if (bond_) throw ParseFailure(kUnknownToken, t.pos, "consecutive bond symbols");
    if (anchor_ < 0) throw ParseFailure(kUnknownToken, t.pos, "bond symbol with no atom before it");
    bond_ = t.value;
    bond_pos_ = t.pos;
  }

  void open(const Token& t) {
    if (anchor_ < 0) throw ParseFailure(kUnbalancedBranch, t.pos, "branch with no atom before it");
    if (bond_) throw ParseFailure(kUnknownToken, t.pos, "bond symbol in front of '('");
    branches_.push_back({anchor_, t.pos});
  }

  void close(const Token& t) {
    if (branches_.empty()) throw ParseFailure(kUnbalancedBranch, t.pos, "')' without a matching '('");
    if (bond_) throw ParseFailure(kUnknownToken, t.pos, "bond symbol in front of ')'");
    anchor_ = branches_.back().atom;
    branches_.pop_back();
  }

  void ring(const Token& t) {
    if (anchor_ < 0) throw ParseFailure(kUnknownToken, t.pos, "ring label with no atom before it");
    Label& l = open_[static_cast<std::size_t>(t.value)];
    if (l.atom < 0) {  // opens the label
      l = Label{anchor_, bond_, t.pos};
      bond_ = 0;
      return;
    }
    if (l.order && bond_ && l.order != bond_)
      throw ParseFailure(kUnclosedRingBond, t.pos, "ring label closed with another bond order");
    const int order = bond_ ? bond_ : l.order ? l.order : implicit(l.atom, anchor_);
    add_bond(l.atom, anchor_, order, t.pos);
    l = Label{};
    bond_ = 0;
  }

  void finish() {
    if (bond_) throw ParseFailure(kUnknownToken, bond_pos_, "input ends after a bond symbol");
    if (!branches_.empty())
      throw ParseFailure(kUnbalancedBranch, branches_.front().pos, "'(' never closed");
    for (const Label& l : open_)
      if (l.atom >= 0) throw ParseFailure(kUnclosedRingBond, l.pos, "ring label never closed");
  }

 private:
  struct Label {
    int atom = -1;
    int order = 0;  // 0: not given at the opening
    std::size_t pos = 0;
  };
  struct Branch {
    int atom;
    std::size_t pos;
  };

  int implicit(int a, int b) const { return g_.aromatic[a] && g_.aromatic[b] ? 4 : 1; }

  void add_bond(int a, int b, int order, std::size_t pos) {
    if (a == b) throw ParseFailure(kUnclosedRingBond, pos, "ring label closes on its own atom");
    for (const BondRec& e : g_.bonds)
      if ((e.a == a && e.b == b) || (e.a == b && e.b == a))
        throw ParseFailure(kUnclosedRingBond, pos, "atoms already bonded");
    g_.bonds.push_back(BondRec{a, b, order});
  }

  Graph& g_;
  int anchor_ = -1;  // the atom the next atom / bond / label attaches to
  int bond_ = 0;     // explicit order waiting for its second atom
  std::size_t bond_pos_ = 0;
  std::vector<Branch> branches_;
  std::array<Label, 100> open_;
};

}  // namespace

Graph parse_smiles(const std::string& text) {
  if (text.empty()) throw ParseFailure(kUnknownToken, 1, "empty SMILES");
  Graph g;
  Lexer lex(text);
  GraphBuilder build(g);
  for (Token t = lex.next(); t.kind != Tok::End; t = lex.next()) {
    switch (t.kind) {
      case Tok::Atom: build.atom(t); break;
      case Tok::Bond: build.bond(t); break;
      case Tok::Open: build.open(t); break;
      case Tok::Close: build.close(t); break;
      case Tok::Ring: build.ring(t); break;
      case Tok::End: break;
    }
  }
  build.finish();
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

// Torsion axes (dock.cpp:234-270): in bond order, every single non-ring
// bond whose atoms both have degree >= 2; moving = the atoms on b's side of
// the bond, b itself excluded, ascending.  One DFS forest gives every atom's
// pre-order interval, so each side of a bridge is an interval test: for a
// DFS tree edge parent -> child the child's side is the child's subtree, the
// parent's side the rest of that tree.
Topology torsion_axes(const Graph& g) {
  Topology t;
  const int n = static_cast<int>(g.elements.size());
  const auto deg = degrees(g);
  std::vector<std::vector<int>> adj(static_cast<std::size_t>(n));
  for (const auto& e : g.bonds) {
    adj[e.a].push_back(e.b);
    adj[e.b].push_back(e.a);
  }
  std::vector<int> tin(n, -1), tout(n, -1), root(n, -1), parent(n, -1);
  int clock = 0;
  for (int r = 0; r < n; ++r) {
    if (tin[r] >= 0) continue;
    std::vector<std::pair<int, std::size_t>> st{{r, 0}};  // (atom, next neighbour)
    tin[r] = clock++;
    root[r] = r;
    while (!st.empty()) {
      auto& [v, k] = st.back();
      if (k < adj[v].size()) {
        const int w = adj[v][k++];
        if (tin[w] < 0) {
          tin[w] = clock++;
          root[w] = r;
          parent[w] = v;
          st.push_back({w, 0});
        }
      } else {
        tout[v] = clock;
        st.pop_back();
      }
    }
  }
  auto inside = [&](int x, int v) { return tin[v] <= tin[x] && tin[x] < tout[v]; };
  for (std::size_t e = 0; e < g.bonds.size(); ++e) {
    const BondRec& bd = g.bonds[e];
    if (bd.order != 1 || g.ring[e] || deg[bd.a] < 2 || deg[bd.b] < 2) continue;
    Axis ax;
    ax.a = bd.a;
    ax.b = bd.b;
    // a bridge is a tree edge: b is a's child or a is b's child
    const bool b_below = parent[bd.b] == bd.a;
    for (int x = 0; x < n; ++x) {
      if (x == bd.b || root[x] != root[bd.b]) continue;
      const bool side_b = b_below ? inside(x, bd.b) : !inside(x, bd.a);
      if (side_b) ax.moving.push_back(x);
    }
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

namespace {
std::vector<std::vector<int>> adjacency(const Graph& g) {
  std::vector<std::vector<int>> adj(g.elements.size());
  for (const auto& b : g.bonds) {
    adj[b.a].push_back(b.b);
    adj[b.b].push_back(b.a);
  }
  return adj;
}

void require_connected(const std::vector<std::vector<int>>& adj) {  // chem.cpp:408
  const std::size_t n = adj.size();
  if (n == 0) return;
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
}  // namespace

void require_connected(const Graph& g) { require_connected(adjacency(g)); }

std::vector<double> embed(const Graph& g, std::uint64_t seed, int iterations) {
  const std::size_t n = g.elements.size();
  std::vector<V3> pos(n, V3{0, 0, 0});
  if (n == 0) return {};
  const std::vector<std::vector<int>> adj = adjacency(g);
  require_connected(adj);
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
