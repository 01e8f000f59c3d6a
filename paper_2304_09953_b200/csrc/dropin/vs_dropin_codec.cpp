// The codec's read side for the C++ drop-in (include/vscreen/codec.hpp):
// SMZ1 parsing from a stream with the reference's checks and messages
// (codec.cpp:188-221), dictionary_sha256 and decompress_stream over the
// native decoder (capi.h vs_sha256, vs_smzc_decompress), decompress_line.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <istream>
#include <iterator>
#include <ostream>
#include <sstream>
#include <thread>

#include "vscreen/codec.hpp"
#include "vscreen_gpu/capi.h"

namespace vscreen::codec {

namespace {
std::string unknown_text(std::uint8_t code, std::size_t offset) {
  std::ostringstream os;
  os << "unknown code byte 0x" << std::hex << static_cast<int>(code) << " at offset " << std::dec
     << offset;
  return os.str();
}

std::string smz1_bytes(const Dictionary& d) {
  std::ostringstream o;
  save_dictionary(d, o);
  return o.str();
}
}  // namespace

UnknownCode::UnknownCode(std::uint8_t code, std::size_t offset)
    : std::runtime_error(unknown_text(code, offset)), code_(code), offset_(offset) {}

std::string decompress_line(std::span<const std::uint8_t> data, const Dictionary& d) {
  std::string out;
  out.reserve(data.size() * 2);
  for (std::size_t i = 0; i < data.size(); ++i) {
    const std::uint8_t b = data[i];
    if (b < 0x80) {
      out.push_back(static_cast<char>(b));
    } else if (static_cast<std::size_t>(b - 0x80) < d.entries.size()) {
      out += d.entries[b - 0x80];
    } else {
      throw UnknownCode(b, i);
    }
  }
  return out;
}

void save_dictionary(const Dictionary& d, std::ostream& out) {
  if (d.entries.size() > Dictionary::kMaxEntries) throw BadFormat("dictionary has too many entries");
  out.write("SMZ1", 4);
  out.put(static_cast<char>(static_cast<std::uint8_t>(d.entries.size())));
  for (const std::string& e : d.entries) {
    out.put(static_cast<char>(static_cast<std::uint8_t>(e.size())));
    out.write(e.data(), static_cast<std::streamsize>(e.size()));
  }
}

// the stream is consumed exactly up to the end of the dictionary
Dictionary load_dictionary(std::istream& in) {
  char magic[4];
  if (!in.read(magic, 4) || std::memcmp(magic, "SMZ1", 4) != 0)
    throw BadFormat("bad dictionary magic (want SMZ1)");
  const int count = in.get();
  if (count == std::char_traits<char>::eof()) throw BadFormat("truncated dictionary header");
  if (static_cast<std::size_t>(count) > Dictionary::kMaxEntries)
    throw BadFormat("dictionary entry count exceeds 128");
  Dictionary d;
  for (int i = 0; i < count; ++i) {
    const int len = in.get();
    if (len == std::char_traits<char>::eof()) throw BadFormat("truncated dictionary entry");
    if (len < static_cast<int>(Dictionary::kMinEntryLen) ||
        len > static_cast<int>(Dictionary::kMaxEntryLen))
      throw BadFormat("dictionary entry length out of range");
    std::string e(static_cast<std::size_t>(len), '\0');
    if (!in.read(e.data(), len)) throw BadFormat("truncated dictionary entry");
    for (char c : e)
      if (c < 0x20 || c > 0x7e) throw BadFormat("dictionary entry is not printable ASCII");
    for (const std::string& x : d.entries)
      if (x == e) throw BadFormat("duplicate dictionary entry");
    d.entries.push_back(std::move(e));
  }
  return d;
}

Dictionary load_dictionary_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw BadFormat("cannot open dictionary: " + path);
  return load_dictionary(in);
}

std::array<std::uint8_t, 32> dictionary_sha256(const Dictionary& d) {
  const std::string b = smz1_bytes(d);
  std::array<std::uint8_t, 32> out{};
  vs_sha256(reinterpret_cast<const std::uint8_t*>(b.data()), static_cast<int64_t>(b.size()),
            out.data());
  return out;
}

// The whole remaining stream is decoded by the native multithreaded decoder;
// on an error nothing is written (the reference has written the records
// before the bad one).
void decompress_stream(std::istream& in, std::ostream& out, const Dictionary& d) {
  const std::string data((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  const std::string dict = smz1_bytes(d);
  const auto* db = reinterpret_cast<const std::uint8_t*>(dict.data());
  const auto* xb = reinterpret_cast<const std::uint8_t*>(data.data());
  const auto th = static_cast<int32_t>(std::max(1u, std::thread::hardware_concurrency()));
  int64_t need = 0;
  int rc = vs_smzc_decompress(db, static_cast<int64_t>(dict.size()), xb,
                              static_cast<int64_t>(data.size()), th, nullptr, 0, &need);
  std::string text;
  if (rc == VS_OK) {
    text.resize(static_cast<std::size_t>(need));
    rc = vs_smzc_decompress(db, static_cast<int64_t>(dict.size()), xb,
                            static_cast<int64_t>(data.size()), th, text.data(), need, &need);
  }
  if (rc != VS_OK) {
    const std::string msg = vs_codec_last_error();
    unsigned code = 0;
    unsigned long long off = 0;
    if (std::sscanf(msg.c_str(), "unknown code byte 0x%x at offset %llu", &code, &off) == 2)
      throw UnknownCode(static_cast<std::uint8_t>(code), static_cast<std::size_t>(off));
    throw BadFormat(msg);
  }
  out.write(text.data(), static_cast<std::streamsize>(text.size()));
}

}  // namespace vscreen::codec
