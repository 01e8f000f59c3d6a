// CampaignReport of the C++ drop-in (include/vscreen/pipeline.hpp): builds
// the report of tests/test_json_bytes.py's fixed spec and prints to_json(),
// "\n--\n" and results_tsv().  Host-only.
#include <iostream>

#include "vscreen/pipeline.hpp"

int main() {
  using namespace vscreen::pipeline;
  CampaignReport r;
  r.stages = {{"parse", 100, 98, 0.0, 0}, {"dock", 98, 91, 12.345678901234567, 7},
              {"rank", 91, 9, 0.0, 0}};
  r.ranked = {{"L10", 45.25, std::nullopt}, {"L2", -1e-5, 0.1}, {"é\"x", 1e20, -3.5}};
  PairResult p;
  p.pair_id = "P0";
  p.ligand_a = "L10";
  p.ligand_b = "L2";
  p.result.estimate = -1.234567890123;
  p.result.sem = 0.05;
  p.result.replicas = 4;
  p.result.target_met = true;
  r.pairs = {p};
  r.trace_path = "out/campaign_trace.jsonl";
  std::cout << r.to_json() << "\n--\n" << r.results_tsv();
  return 0;
}
