// SMZC library decompression for the ingest feed: the
// reference's compressed-library format (codec.hpp:41-79, codec.cpp:147-161,
// 195-289) decoded on all host threads.
//
//   dictionary  "SMZ1", count byte, per entry a length byte (2..8) + bytes
//               (printable ASCII, no duplicates); entry i <-> code 0x80 + i
//   library     "SMZC", SHA-256 of the serialized dictionary (32 bytes),
//               then per line a LEB128 byte length + payload; payload bytes
//               < 0x80 are literals, >= 0x80 dictionary codes
//
// The record boundaries are one sequential varint walk (cheap: a header per
// line); the records then expand in parallel into per-thread spans that are
// laid out by a prefix sum, so the output is the reference's byte for byte
// (each record + '\n').  SHA-256 is implemented here (FIPS 180-4) so the
// library needs no crypto dependency.
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/vscreen_gpu/capi.h"

namespace {

// ---------------------------------------------------------------- SHA-256
struct Sha256 {
  uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                   0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
  static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }
  void block(const uint8_t* p) {
    static const uint32_t k[64] = {
        0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u,
        0xab1c5ed5u, 0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu,
        0x9bdc06a7u, 0xc19bf174u, 0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu,
        0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau, 0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u,
        0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u, 0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu,
        0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u, 0xa2bfe8a1u, 0xa81a664bu,
        0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u, 0x19a4c116u,
        0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
        0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u,
        0xc67178f2u};
    uint32_t w[64];
    for (int i = 0; i < 16; ++i)
      w[i] = (uint32_t(p[4 * i]) << 24) | (uint32_t(p[4 * i + 1]) << 16) |
             (uint32_t(p[4 * i + 2]) << 8) | uint32_t(p[4 * i + 3]);
    for (int i = 16; i < 64; ++i) {
      const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int i = 0; i < 64; ++i) {
      const uint32_t t1 = hh + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) +
                          k[i] + w[i];
      const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      hh = g;
      g = f;
      f = e;
      e = d + t1;
      d = c;
      c = b;
      b = a;
      a = t1 + t2;
    }
    h[0] += a, h[1] += b, h[2] += c, h[3] += d, h[4] += e, h[5] += f, h[6] += g, h[7] += hh;
  }
  std::array<uint8_t, 32> digest(const uint8_t* data, size_t n) {
    size_t i = 0;
    for (; i + 64 <= n; i += 64) block(data + i);
    uint8_t tail[128] = {0};
    const size_t r = n - i;
    std::memcpy(tail, data + i, r);
    tail[r] = 0x80;
    const size_t tl = r + 9 <= 64 ? 64 : 128;
    const uint64_t bits = static_cast<uint64_t>(n) * 8;
    for (int b = 0; b < 8; ++b) tail[tl - 1 - b] = static_cast<uint8_t>(bits >> (8 * b));
    block(tail);
    if (tl == 128) block(tail + 64);
    std::array<uint8_t, 32> out{};
    for (int j = 0; j < 8; ++j)
      for (int b = 0; b < 4; ++b) out[4 * j + b] = static_cast<uint8_t>(h[j] >> (24 - 8 * b));
    return out;
  }
};

struct Dict {
  std::vector<std::string> entries;
  std::vector<uint8_t> bytes;  // serialized as the file holds it (hashed)
};

// SMZ1 (codec.cpp:195-226); status + message
int parse_dict(const uint8_t* p, int64_t n, Dict& d, std::string& msg) {
  if (n < 4 || std::memcmp(p, "SMZ1", 4) != 0) return msg = "bad dictionary magic (want SMZ1)", VS_ERR_FORMAT;
  if (n < 5) return msg = "truncated dictionary header", VS_ERR_FORMAT;
  const int count = p[4];
  if (count > 128) return msg = "dictionary entry count exceeds 128", VS_ERR_FORMAT;
  int64_t o = 5;
  for (int i = 0; i < count; ++i) {
    if (o >= n) return msg = "truncated dictionary entry", VS_ERR_FORMAT;
    const int len = p[o++];
    if (len < 2 || len > 8) return msg = "dictionary entry length out of range", VS_ERR_FORMAT;
    if (o + len > n) return msg = "truncated dictionary entry", VS_ERR_FORMAT;
    std::string e(reinterpret_cast<const char*>(p + o), static_cast<size_t>(len));
    o += len;
    for (char c : e)
      if (c < 0x20 || c > 0x7e) return msg = "dictionary entry is not printable ASCII", VS_ERR_FORMAT;
    for (const auto& x : d.entries)
      if (x == e) return msg = "duplicate dictionary entry", VS_ERR_FORMAT;
    d.entries.push_back(std::move(e));
  }
  // the hash covers the serialized dictionary (save_dictionary's bytes),
  // which is the consumed prefix
  d.bytes.assign(p, p + o);
  return VS_OK;
}

thread_local std::string g_codec_err;

}  // namespace

extern "C" {

const char* vs_codec_last_error(void) { return g_codec_err.c_str(); }

int vs_sha256(const uint8_t* data, int64_t len, uint8_t* out32) {
  if (len < 0 || !out32 || (len > 0 && !data)) return VS_ERR_INVALID_ARGUMENT;
  Sha256 sha;
  const auto d = sha.digest(data, static_cast<size_t>(len));
  std::memcpy(out32, d.data(), 32);
  return VS_OK;
}

int vs_smz1_check(const uint8_t* dict, int64_t dict_len, int32_t* n_entries) {
  Dict d;
  std::string msg;
  const int rc = parse_dict(dict, dict_len, d, msg);
  if (rc) return g_codec_err = msg, rc;
  if (n_entries) *n_entries = static_cast<int32_t>(d.entries.size());
  return VS_OK;
}

int vs_smzc_decompress(const uint8_t* dict, int64_t dict_len, const uint8_t* data, int64_t len,
                       int32_t threads, char* out, int64_t cap, int64_t* out_len) {
  Dict d;
  std::string msg;
  int rc = parse_dict(dict, dict_len, d, msg);
  if (rc) return g_codec_err = msg, rc;
  if (len < 4 || std::memcmp(data, "SMZC", 4) != 0)
    return g_codec_err = "bad compressed-library magic (want SMZC)", VS_ERR_FORMAT;
  if (len < 36) return g_codec_err = "truncated dictionary hash", VS_ERR_FORMAT;
  Sha256 sha;
  const auto want = sha.digest(d.bytes.data(), d.bytes.size());
  if (std::memcmp(want.data(), data + 4, 32) != 0)
    return g_codec_err = "dictionary hash mismatch: file was written with a different dictionary",
           VS_ERR_FORMAT;
  // record boundaries: the sequential varint walk. A framing error ends the
  // walk; it is reported only if no earlier record has an unknown code, the
  // order in which decompress_stream (codec.cpp:275-289) meets them.
  std::vector<int64_t> rec_off, rec_len;
  const char* tail_err = nullptr;
  int64_t o = 36;
  while (o < len && !tail_err) {
    uint64_t v = 0;
    int shift = 0;
    while (true) {
      if (o >= len) {
        tail_err = "truncated varint";
        break;
      }
      const uint8_t c = data[o++];
      v |= static_cast<uint64_t>(c & 0x7f) << shift;
      if (!(c & 0x80)) break;
      shift += 7;
      if (shift > 63) {
        tail_err = "varint overflow";
        break;
      }
    }
    if (tail_err) break;
    if (static_cast<uint64_t>(len - o) < v) {
      tail_err = "truncated record payload";
      break;
    }
    rec_off.push_back(o);
    rec_len.push_back(static_cast<int64_t>(v));
    o += static_cast<int64_t>(v);
  }
  const size_t nr = rec_off.size();
  // per record: expanded size (+ '\n'), the first unknown code
  std::vector<int64_t> size(nr + 1, 0);
  std::vector<int64_t> bad(nr, -1);
  std::array<int, 128> elen{};
  for (size_t i = 0; i < d.entries.size(); ++i) elen[i] = static_cast<int>(d.entries[i].size());
  const int ne = static_cast<int>(d.entries.size());
  const int nth = std::max(1, std::min<int>(threads > 0 ? threads : 1, 64));
  auto pass = [&](int t, bool write, const int64_t* at) {
    const size_t lo = nr * t / nth, hi = nr * (t + 1) / nth;
    for (size_t r = lo; r < hi; ++r) {
      const uint8_t* p = data + rec_off[r];
      if (!write) {
        int64_t s = 1;
        for (int64_t k = 0; k < rec_len[r]; ++k) {
          const uint8_t b = p[k];
          if (b < 0x80) {
            ++s;
          } else if (b - 0x80 < ne) {
            s += elen[b - 0x80];
          } else {
            bad[r] = k;
            break;
          }
        }
        size[r] = s;
      } else {
        char* dst = out + at[r];
        for (int64_t k = 0; k < rec_len[r]; ++k) {
          const uint8_t b = p[k];
          if (b < 0x80) {
            *dst++ = static_cast<char>(b);
          } else {
            const std::string& e = d.entries[b - 0x80];
            std::memcpy(dst, e.data(), e.size());
            dst += e.size();
          }
        }
        *dst = '\n';
      }
    }
  };
  auto run = [&](bool write, const int64_t* at) {
    if (nth == 1 || nr < 4096) {
      for (int t = 0; t < nth; ++t) pass(t, write, at);
      return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < nth; ++t) pool.emplace_back(pass, t, write, at);
    for (auto& th : pool) th.join();
  };
  run(false, nullptr);
  for (size_t r = 0; r < nr; ++r)
    if (bad[r] >= 0) {
      const uint8_t code = data[rec_off[r] + bad[r]];
      char buf[96];
      std::snprintf(buf, sizeof buf, "unknown code byte 0x%x at offset %lld", code,
                    static_cast<long long>(bad[r]));
      return g_codec_err = buf, VS_ERR_FORMAT;
    }
  if (tail_err) return g_codec_err = tail_err, VS_ERR_FORMAT;
  std::vector<int64_t> at(nr + 1, 0);
  for (size_t r = 0; r < nr; ++r) at[r + 1] = at[r] + size[r];
  if (out_len) *out_len = at[nr];
  if (!out) return VS_OK;  // size query
  if (cap < at[nr]) return g_codec_err = "output buffer too small", VS_ERR_CAPACITY;
  run(true, at.data());
  return VS_OK;
}

}  // extern "C"
