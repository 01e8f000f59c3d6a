#pragma once
// Drop-in for the read side of the reference codec (proj/include/vscreen/
// codec.hpp:14-79): the SMZ1 dictionary loader, dictionary_sha256,
// decompress_line and decompress_stream, implemented over the native SMZC
// decoder of libvscreen_gpu.so (capi.h vs_smzc_decompress).  The write side
// (train_dictionary, compress_line, compress_stream, save_dictionary_file)
// belongs to the library build tools, outside the dock-and-score path, and is
// not declared here.

#include <array>
#include <cstdint>
#include <iosfwd>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace vscreen::codec {

class UnknownCode : public std::runtime_error {
 public:
  UnknownCode(std::uint8_t code, std::size_t offset);
  [[nodiscard]] std::uint8_t code() const { return code_; }
  [[nodiscard]] std::size_t offset() const { return offset_; }

 private:
  std::uint8_t code_;
  std::size_t offset_;
};

class BadFormat : public std::runtime_error {
 public:
  explicit BadFormat(const std::string& msg) : std::runtime_error(msg) {}
};

struct Dictionary {
  static constexpr std::size_t kMaxEntries = 128;
  static constexpr std::size_t kMinEntryLen = 2;
  static constexpr std::size_t kMaxEntryLen = 8;

  std::vector<std::string> entries;  // entries[i] <-> code byte 0x80 + i
  std::uint32_t version = 1;

  [[nodiscard]] std::size_t size() const { return entries.size(); }
};

std::string decompress_line(std::span<const std::uint8_t> data, const Dictionary& d);

void save_dictionary(const Dictionary& d, std::ostream& out);
Dictionary load_dictionary(std::istream& in);
Dictionary load_dictionary_file(const std::string& path);

std::array<std::uint8_t, 32> dictionary_sha256(const Dictionary& d);

void decompress_stream(std::istream& in, std::ostream& out, const Dictionary& d);

}  // namespace vscreen::codec
