// chem API of the drop-in (include/vscreen/chem.hpp) over the host ingest
// (vs_ingest.cpp).  The reference's behaviour it keeps: chem.cpp:109-264
// (parse, ParseError kind / 1-based position), :266-331 (ring flags,
// rotatable bonds: the graph's own ring flags when they match its bonds),
// :333-341 (make_ligand), :406-446 (embed_3d, DisconnectedGraph first),
// :448-476 (library records).
#include <fstream>
#include <istream>
#include <string>
#include <vector>

#include "../vs_ingest.h"
#include "vscreen/chem.hpp"

namespace vscreen::chem {

namespace {

MolecularGraph from_ingest(const vs::Graph& g) {
  MolecularGraph m;
  m.atoms.reserve(g.elements.size());
  for (std::size_t i = 0; i < g.elements.size(); ++i) m.atoms.push_back(Atom{g.elements[i], g.aromatic[i]});
  m.bonds.reserve(g.bonds.size());
  for (const vs::BondRec& b : g.bonds) m.bonds.push_back(Bond{b.a, b.b, static_cast<BondOrder>(b.order)});
  m.ring_bond_flags = g.ring;
  return m;
}

}  // namespace

// also used by the dock drop-in (torsion_topology)
vs::Graph to_ingest(const MolecularGraph& m) {
  vs::Graph g;
  for (const Atom& a : m.atoms) {
    g.elements.push_back(a.element);
    g.aromatic.push_back(a.aromatic);
  }
  for (const Bond& b : m.bonds) g.bonds.push_back(vs::BondRec{b.a, b.b, static_cast<int>(b.order)});
  g.ring = m.ring_bond_flags.size() == m.bonds.size() ? m.ring_bond_flags : vs::ring_bond_flags(g);
  return g;
}

ParseError::ParseError(ParseErrorKind kind, std::size_t position, const std::string& msg)
    : std::runtime_error(msg), kind_(kind), position_(position) {}

std::vector<int> MolecularGraph::degrees() const {
  std::vector<int> d(atoms.size(), 0);
  for (const Bond& b : bonds) {
    ++d[static_cast<std::size_t>(b.a)];
    ++d[static_cast<std::size_t>(b.b)];
  }
  return d;
}

bool MolecularGraph::connected() const {
  const std::size_t n = atoms.size();
  if (n <= 1) return true;
  std::vector<std::vector<int>> adj(n);
  for (const Bond& b : bonds) {
    adj[static_cast<std::size_t>(b.a)].push_back(b.b);
    adj[static_cast<std::size_t>(b.b)].push_back(b.a);
  }
  std::vector<char> seen(n, 0);
  std::vector<int> stack{0};
  seen[0] = 1;
  std::size_t reached = 1;
  while (!stack.empty()) {
    const int v = stack.back();
    stack.pop_back();
    for (int w : adj[static_cast<std::size_t>(v)])
      if (!seen[static_cast<std::size_t>(w)]) {
        seen[static_cast<std::size_t>(w)] = 1;
        ++reached;
        stack.push_back(w);
      }
  }
  return reached == n;
}

MolecularGraph parse_smiles(std::string_view text) {
  try {
    return from_ingest(vs::parse_smiles(std::string(text)));
  } catch (const vs::ParseFailure& e) {
    throw ParseError(static_cast<ParseErrorKind>(e.kind), e.pos, e.what());
  }
}

std::vector<bool> compute_ring_bonds(const MolecularGraph& g) {
  vs::Graph t = to_ingest(g);
  return vs::ring_bond_flags(t);
}

int rotatable_bonds(const MolecularGraph& g) { return vs::rotatable_bond_count(to_ingest(g)); }

Ligand make_ligand(std::string id, std::string smiles) {
  Ligand lig;
  lig.id = std::move(id);
  lig.smiles = std::move(smiles);
  lig.graph = parse_smiles(lig.smiles);
  lig.heavy_atoms = lig.graph.atom_count();
  lig.rotatable_bonds = rotatable_bonds(lig.graph);
  return lig;
}

Conformer embed_3d(const MolecularGraph& g, std::uint64_t seed, std::string ligand_id,
                   int iterations) {
  if (!g.connected()) throw DisconnectedGraph();
  Conformer c;
  c.ligand_id = std::move(ligand_id);
  const std::vector<double> xyz = vs::embed(to_ingest(g), seed, iterations);
  c.coords.resize(static_cast<std::size_t>(g.atom_count()));
  for (std::size_t i = 0; i < c.coords.size(); ++i)
    c.coords[i] = Vec3{xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
  return c;
}

std::vector<LibraryRecord> read_library_records(std::istream& in) {
  std::vector<LibraryRecord> out;
  std::string line;
  for (std::size_t no = 1; std::getline(in, line); ++no) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (line.empty() || line.front() == '#') continue;
    LibraryRecord r;
    r.line_number = no;
    const std::size_t tab = line.find('\t');
    r.smiles = line.substr(0, tab);
    if (tab != std::string::npos) r.id = line.substr(tab + 1);
    if (r.id.empty()) r.id = "L" + std::to_string(no);
    out.push_back(std::move(r));
  }
  return out;
}

std::vector<LibraryRecord> read_library_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw std::runtime_error("cannot open library file: " + path);
  return read_library_records(in);
}

}  // namespace vscreen::chem
