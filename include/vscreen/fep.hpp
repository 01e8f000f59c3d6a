// vscreen/fep.hpp — the free-energy result record only.
//
// The FEP / AWH stage of the reference (proj/include/vscreen/fep.hpp) is
// outside the dock-and-score path; the campaign report
// (pipeline.hpp CampaignReport) carries its per-pair result, so the record
// is declared here with the reference's fields (fep.hpp:92-98).
#pragma once

namespace vscreen::fep {

struct FreeEnergyResult {
  double estimate = 0.0;  // kT
  double sem = 0.0;       // kT
  int replicas = 0;
  int bias_history_length = 0;
  bool target_met = false;
};

}  // namespace vscreen::fep
