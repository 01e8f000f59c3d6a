// JSON I/O of the C++ drop-in (include/vscreen/dock.hpp): reads a pocket
// JSON document on stdin and prints pocket_to_json(parse_pocket_json(..)),
// then "\n--\n" and pose_to_json of a pose given on the command line
// (ligand, t x3, q x4, geo, rescore|none, torsions...).  Host-only.
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <iterator>
#include <string>

#include "vscreen/dock.hpp"

int main(int argc, char** argv) {
  using namespace vscreen;
  std::string text((std::istreambuf_iterator<char>(std::cin)), std::istreambuf_iterator<char>());
  std::cout << dock::pocket_to_json(dock::parse_pocket_json(text)) << "\n--\n";
  if (argc >= 11) {
    dock::Pose p;
    p.ligand_id = argv[1];
    p.translation = {std::strtod(argv[2], nullptr), std::strtod(argv[3], nullptr),
                     std::strtod(argv[4], nullptr)};
    p.rotation = {std::strtod(argv[5], nullptr), std::strtod(argv[6], nullptr),
                  std::strtod(argv[7], nullptr), std::strtod(argv[8], nullptr)};
    p.geometric_score = std::strtod(argv[9], nullptr);
    if (std::string(argv[10]) != "none") p.rescore = std::strtod(argv[10], nullptr);
    for (int i = 11; i < argc; ++i) p.torsions.push_back(std::strtod(argv[i], nullptr));
    std::cout << dock::pose_to_json(p);
  }
  return 0;
}
