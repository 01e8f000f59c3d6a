// vscreen/pipeline.hpp — the ranked-result record of the dock funnel.
//
// The hot-path subset of the reference's pipeline API (proj/include/
// vscreen/pipeline.hpp:71-110): the stage and ranked records, the campaign
// report with its deterministic JSON bytes, and rank_ligands.  The campaign
// driver itself and the FEP stages are the reference's other subsystems and
// are not part of this drop-in; the GPU ranking is capi.h
// vs_topk / vs_topk_allgather.
#pragma once

#include <cstddef>
#include <map>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "vscreen/fep.hpp"

namespace vscreen::pipeline {

struct StageStats {
  std::string name;
  std::size_t in = 0;
  std::size_t out = 0;
  double sim_seconds = 0.0;  // simulated cluster time, 0 for inline stages
  std::size_t tasks = 0;     // scheduler tasks the stage submitted
};

struct RankedLigand {
  std::string id;
  double score = 0.0;
  std::optional<double> delta_g;  // only for ligands that reached the FEP stage
};

struct PairResult {
  std::string pair_id;
  std::string ligand_a;
  std::string ligand_b;
  fep::FreeEnergyResult result;
};

struct CampaignReport {
  std::vector<StageStats> stages;
  std::vector<RankedLigand> ranked;
  std::vector<PairResult> pairs;
  std::string trace_path;

  // the reference's report bytes (pipeline.cpp:269-301): ordered JSON, dump(2)
  [[nodiscard]] std::string to_json() const;
  // tab-separated per-pair results (pipeline.cpp:303-313)
  [[nodiscard]] std::string results_tsv() const;
};

// descending score, ties by ascending id (bytewise)
std::vector<std::pair<std::string, double>> rank_ligands(
    const std::map<std::string, double>& scores);

}  // namespace vscreen::pipeline
