// The codec read side of the C++ drop-in (include/vscreen/codec.hpp) as a
// reference caller uses it (pipeline.cpp:384-396): usage codec_read <golden dir>
// <campaign dir>; prints "codec ok" when every check holds.
#include <cstdio>
#include <fstream>
#include <iterator>
#include <sstream>
#include <string>
#include <vector>

#include "vscreen/codec.hpp"

using namespace vscreen::codec;

static std::string slurp(const std::string& p) {
  std::ifstream f(p, std::ios::binary);
  return std::string((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}

#define CHECK(c)                                                  \
  do {                                                            \
    if (!(c)) {                                                   \
      std::printf("FAILED %s (line %d)\n", #c, __LINE__);          \
      return 1;                                                   \
    }                                                             \
  } while (0)

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const std::string codec_dir = argv[1], camp = argv[2];
  // pipeline.cpp:390-396
  const Dictionary dict = load_dictionary_file(camp + "/smiles.dict");
  std::ifstream in(codec_dir + "/library_100.smzc", std::ios::binary);
  std::ostringstream text;
  decompress_stream(in, text, dict);
  CHECK(text.str() == slurp(camp + "/sample_library_100.smi"));
  // the hash in the file is dictionary_sha256 of the dictionary
  const std::string packed = slurp(codec_dir + "/library_100.smzc");
  const auto h = dictionary_sha256(dict);
  CHECK(packed.compare(4, 32, std::string(h.begin(), h.end())) == 0);
  // a different dictionary: BadFormat with the reference's message
  const Dictionary other = load_dictionary_file(codec_dir + "/trained.dict");
  std::istringstream pin(packed);
  std::ostringstream o2;
  try {
    decompress_stream(pin, o2, other);
    CHECK(false);
  } catch (const BadFormat& e) {
    CHECK(std::string(e.what()) ==
          "dictionary hash mismatch: file was written with a different dictionary");
  }
  // decompress_line known answers (test_codec.cpp:92-108)
  Dictionary d;
  d.entries = {"CC"};
  const std::vector<std::uint8_t> data = {0x80, 'O'};
  CHECK(decompress_line(data, d) == "CCO");
  Dictionary empty;
  const std::vector<std::uint8_t> bad = {0x90};
  try {
    decompress_line(bad, empty);
    CHECK(false);
  } catch (const UnknownCode& e) {
    CHECK(e.code() == 0x90 && e.offset() == 0);
  }
  // load_dictionary checks
  std::istringstream bd(std::string("SMZ1\x01\x01", 6) + "C");
  try {
    load_dictionary(bd);
    CHECK(false);
  } catch (const BadFormat& e) {
    CHECK(std::string(e.what()) == "dictionary entry length out of range");
  }
  // an unknown code in a stream: UnknownCode (record offset)
  std::string s = "SMZC" + std::string(h.begin(), h.end());
  s += std::string("\x02", 1) + "C" + std::string(1, static_cast<char>(0x80 + dict.size()));
  std::istringstream ps(s);
  std::ostringstream o3;
  try {
    decompress_stream(ps, o3, dict);
    CHECK(false);
  } catch (const UnknownCode& e) {
    CHECK(e.code() == 0x80 + dict.size() && e.offset() == 1);
  }
  std::printf("codec ok\n");
  return 0;
}
