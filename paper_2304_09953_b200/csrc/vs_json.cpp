// Doubles as the reference's JSON writer prints them.  The reference dumps
// every pose, pocket and report through nlohmann::json 3.11 (dock.cpp:460-489,
// pipeline.cpp:269-301), whose Grisu2 digits are round-trip exact but not
// always the shortest ones; the Python writers (dock.pose_to_json,
// campaign.report_to_json) take their number text from here so the bytes are
// the reference's.  nlohmann 3.11.3 is the copy vendored with cudnn_frontend.
#include <cstdint>
#include <cstring>
#include <string>

#include <nlohmann/json.hpp>

#include "../../include/vscreen_gpu/capi.h"

extern "C" int vs_json_format_doubles(const double* x, int64_t n, char* out, int32_t stride) {
  if (n < 0 || stride < 2 || (n > 0 && (!x || !out))) return VS_ERR_INVALID_ARGUMENT;
  for (int64_t i = 0; i < n; ++i) {
    const std::string s = nlohmann::json(x[i]).dump();
    if (static_cast<int64_t>(s.size()) >= stride) return VS_ERR_CAPACITY;
    char* o = out + i * stride;
    std::memcpy(o, s.data(), s.size());
    o[s.size()] = '\0';
  }
  return VS_OK;
}
