// Host ligand ingest (see vs_ingest.cpp).
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace vs {

enum ParseKind { kUnbalancedBranch = 0, kUnclosedRingBond = 1, kUnknownToken = 2 };

struct ParseFailure : std::runtime_error {
  ParseFailure(int kind, std::size_t pos, const std::string& msg);
  int kind;
  std::size_t pos;  // 1-based byte offset
};

struct BondRec {
  int a, b;
  int order;  // 1 single, 2 double, 3 triple, 4 aromatic (chem.hpp:11)
};

struct Graph {
  std::vector<std::string> elements;  // aromatic atoms stored uppercase
  std::vector<bool> aromatic;
  std::vector<BondRec> bonds;
  std::vector<bool> ring;
};

struct Axis {
  int a = 0, b = 0;
  std::vector<int> moving;
};

struct Topology {
  std::vector<Axis> axes;
};

Graph parse_smiles(const std::string& text);
std::vector<bool> ring_bond_flags(const Graph& g);
std::vector<int> degrees(const Graph& g);
int rotatable_bond_count(const Graph& g);
Topology torsion_axes(const Graph& g);
std::vector<double> embed(const Graph& g, std::uint64_t seed, int iterations);
std::vector<double> embed_place(const Graph& g, std::uint64_t seed);
// embed_3d's DisconnectedGraph check (chem.cpp:408): throws if not connected
void require_connected(const Graph& g);
int element_class(const std::string& el);
std::string random_smiles(std::uint64_t seed, std::uint64_t index);

}  // namespace vs
