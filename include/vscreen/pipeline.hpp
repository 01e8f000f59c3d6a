// vscreen/pipeline.hpp — the ranked-result record of the dock funnel.
//
// The hot-path subset of the reference's pipeline API (proj/include/
// vscreen/pipeline.hpp:79-110): the ranked record and rank_ligands.  The
// campaign driver, its config / report / trace and the FEP stages are the
// reference's other subsystems and are not part of this drop-in (SURVEY
// §2); the GPU ranking is capi.h vs_topk / vs_topk_allgather.
#pragma once

#include <map>
#include <optional>
#include <string>
#include <utility>
#include <vector>

namespace vscreen::pipeline {

struct RankedLigand {
  std::string id;
  double score = 0.0;
  std::optional<double> delta_g;  // only for ligands that reached the FEP stage
};

// descending score, ties by ascending id (bytewise)
std::vector<std::pair<std::string, double>> rank_ligands(
    const std::map<std::string, double>& scores);

}  // namespace vscreen::pipeline
