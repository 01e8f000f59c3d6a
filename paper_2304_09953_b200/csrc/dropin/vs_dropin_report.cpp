// Campaign report of the drop-in (include/vscreen/pipeline.hpp): the
// reference's deterministic report bytes (pipeline.cpp:269-301: an ordered
// JSON document dumped with indent 2 by nlohmann 3.11.3, the library the
// reference uses) and its per-pair TSV (pipeline.cpp:303-313).
#include <sstream>
#include <string>

#include <nlohmann/json.hpp>

#include "vscreen/pipeline.hpp"

namespace vscreen::pipeline {

std::string CampaignReport::to_json() const {
  using J = nlohmann::ordered_json;
  J st = J::array(), rk = J::array(), pr = J::array();
  for (const StageStats& s : stages)
    st.push_back(J{{"name", s.name}, {"in", s.in}, {"out", s.out},
                   {"sim_seconds", s.sim_seconds}, {"tasks", s.tasks}});
  for (const RankedLigand& r : ranked) {
    J e{{"id", r.id}, {"score", r.score}};
    e["delta_g"] = r.delta_g ? J(*r.delta_g) : J();
    rk.push_back(std::move(e));
  }
  for (const PairResult& p : pairs)
    pr.push_back(J{{"pair_id", p.pair_id}, {"ligand_a", p.ligand_a}, {"ligand_b", p.ligand_b},
                   {"ddg_kT", p.result.estimate}, {"sem_kT", p.result.sem},
                   {"replicas", p.result.replicas}, {"target_met", p.result.target_met}});
  J j;
  j["stages"] = std::move(st);
  j["ranked"] = std::move(rk);
  j["pairs"] = std::move(pr);
  j["trace_path"] = trace_path;
  return j.dump(2);
}

std::string CampaignReport::results_tsv() const {
  std::ostringstream o;
  o << "pair_id\tligand_a\tligand_b\tddg_kT\tsem_kT\treplicas\tflag\n";
  for (const PairResult& p : pairs) {
    o << p.pair_id << '\t' << p.ligand_a << '\t' << p.ligand_b << '\t';
    o.precision(10);
    o << p.result.estimate << '\t' << p.result.sem << '\t' << p.result.replicas << '\t'
      << (p.result.target_met ? "ok" : "target_not_met") << '\n';
  }
  return o.str();
}

}  // namespace vscreen::pipeline
