// frag core types for the B200 build — a fresh, header-only definition of the
// reference's common surface (/root/reference/proj/include/frag/common.hpp:12-147),
// including the out-of-line bodies the reference declares but does not ship
// (Hash128::hex/from_hex, hash_*, fnv1a, format_float, byte tokenizer).
//
//   Token / Pos                common.hpp:14-15
//   ContractError / StoreError / FormatError{Kind}   common.hpp:17-40
//   Rng (splitmix64 + Box-Muller, bit-exact with the reference; pinned by
//        tests/golden/rng_kat.json generated from the reference header)  common.hpp:45-100
//   Hash128 / ChunkId / PrefixKey / Hash128Hasher    common.hpp:102-132
//   fnv1a, format_float, tokenize_bytes              common.hpp:134-145
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace frag {

using Token = int32_t;
using Pos = int32_t;  // 1-based token position

struct ContractError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StoreError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct FormatError : std::runtime_error {
  enum class Kind { BadMagic, BadVersion, Truncated, Malformed, Io };
  FormatError(Kind k, const std::string& msg) : std::runtime_error(msg), kind_(k) {}
  Kind kind() const noexcept { return kind_; }

 private:
  Kind kind_;
};

namespace detail {
inline uint64_t mix64(uint64_t z) noexcept {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
}  // namespace detail

// splitmix64 generator; the n-th draw is mix64(seed + n * gamma) (n >= 1), which
// is what lets the GPU weight initialiser evaluate the stream in parallel.
class Rng {
 public:
  static constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
  explicit Rng(uint64_t seed) : s_(seed) {}
  uint64_t next_u64() noexcept { return detail::mix64(s_ += kGamma); }
  uint32_t next_u32() noexcept { return static_cast<uint32_t>(next_u64() >> 32); }
  double next_double() noexcept { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  float next_float() noexcept { return static_cast<float>(next_double()); }
  uint64_t below(uint64_t n) {  // unbiased rejection
    if (n == 0) throw ContractError("Rng::below: n must be positive");
    const uint64_t lim = (0 - n) % n;
    uint64_t r;
    do r = next_u64();
    while (r < lim);
    return r % n;
  }
  int64_t range(int64_t lo, int64_t hi) {
    if (hi < lo) throw ContractError("Rng::range: hi < lo");
    return lo + static_cast<int64_t>(below(static_cast<uint64_t>(hi - lo) + 1));
  }
  double normal() {  // Box-Muller, cos first, sin cached
    if (cached_) {
      cached_ = false;
      return cache_;
    }
    double u1;
    do u1 = next_double();
    while (u1 <= 0.0);
    const double u2 = next_double();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double t = 6.283185307179586477 * u2;
    cache_ = r * std::sin(t);
    cached_ = true;
    return r * std::cos(t);
  }
  float normal_f(float sigma) { return static_cast<float>(normal()) * sigma; }

 private:
  uint64_t s_;
  bool cached_ = false;
  double cache_ = 0.0;
};

struct Hash128 {
  std::array<uint8_t, 16> bytes{};
  auto operator<=>(const Hash128&) const = default;
  bool is_zero() const noexcept {
    for (auto b : bytes)
      if (b) return false;
    return true;
  }
  std::string hex() const {
    static const char* d = "0123456789abcdef";
    std::string s(32, '0');
    for (int i = 0; i < 16; ++i) s[2 * i] = d[bytes[i] >> 4], s[2 * i + 1] = d[bytes[i] & 15];
    return s;
  }
  static Hash128 from_hex(const std::string& s) {
    if (s.size() != 32) throw FormatError(FormatError::Kind::Malformed, "Hash128::from_hex: need 32 hex digits");
    auto v = [&](char c) -> int {
      if (c >= '0' && c <= '9') return c - '0';
      if (c >= 'a' && c <= 'f') return c - 'a' + 10;
      if (c >= 'A' && c <= 'F') return c - 'A' + 10;
      throw FormatError(FormatError::Kind::Malformed, "Hash128::from_hex: bad digit");
    };
    Hash128 h;
    for (int i = 0; i < 16; ++i) h.bytes[i] = static_cast<uint8_t>(v(s[2 * i]) * 16 + v(s[2 * i + 1]));
    return h;
  }
};
using ChunkId = Hash128;
using PrefixKey = Hash128;

struct Hash128Hasher {
  size_t operator()(const Hash128& h) const noexcept {
    uint64_t v;
    std::memcpy(&v, h.bytes.data(), 8);
    return static_cast<size_t>(v);
  }
};

namespace detail {
// Two independent splitmix-mixed lanes over (index, 32-bit word); identical to
// libfrag's frag_hash_tokens (paper_2601_12904_b200/csrc/store.cpp) for tokens.
inline Hash128 hash_words(const uint32_t* w, size_t n, uint64_t salt) {
  uint64_t a = 0x243f6a8885a308d3ULL ^ salt;
  uint64_t b = 0x13198a2e03707344ULL ^ mix64(salt + 1);
  for (size_t i = 0; i < n; ++i) {
    const uint64_t u = w[i];
    a = mix64(a + Rng::kGamma * (u + 1) + static_cast<uint64_t>(i));
    b = mix64(b ^ (u * 0xd1b54a32d192ed03ULL + 0x8cb92ba72f3d8dd7ULL * static_cast<uint64_t>(i + 1)));
  }
  a = mix64(a ^ static_cast<uint64_t>(n));
  b = mix64(b + static_cast<uint64_t>(n) * Rng::kGamma);
  Hash128 h;
  std::memcpy(h.bytes.data(), &a, 8);
  std::memcpy(h.bytes.data() + 8, &b, 8);
  return h;
}
}  // namespace detail

inline Hash128 hash_tokens(std::span<const Token> t, uint64_t salt = 0) {
  return detail::hash_words(reinterpret_cast<const uint32_t*>(t.data()), t.size(), salt);
}
inline Hash128 hash_bytes(std::span<const uint8_t> data, uint64_t salt = 0) {
  std::vector<uint32_t> w(data.begin(), data.end());
  return detail::hash_words(w.data(), w.size(), salt ^ 0x5bd1e9955bd1e995ULL);
}
inline Hash128 hash_string(const std::string& s, uint64_t salt = 0) {
  return hash_bytes({reinterpret_cast<const uint8_t*>(s.data()), s.size()}, salt);
}
// Order-sensitive rolling combine: key' = H(key || next).
inline Hash128 hash_combine(const Hash128& key, const Hash128& next) {
  uint32_t w[8];
  std::memcpy(w, key.bytes.data(), 16);
  std::memcpy(w + 4, next.bytes.data(), 16);
  return detail::hash_words(w, 8, 0x2545f4914f6cdd1dULL);
}

inline uint64_t fnv1a(std::span<const uint8_t> data) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (uint8_t b : data) h = (h ^ b) * 0x100000001b3ULL;
  return h;
}
inline std::span<const uint8_t> as_bytes_span(const std::vector<float>& v) {
  return {reinterpret_cast<const uint8_t*>(v.data()), v.size() * sizeof(float)};
}
// Replay-stable float text: shortest round-trip form ("%.9g" for float range, "%.17g" otherwise).
inline std::string format_float(double v) {
  char buf[40];
  if (std::isnan(v)) return "nan";
  if (std::isinf(v)) return v > 0 ? "inf" : "-inf";
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}
// Byte-level tokenizer (vocab 256).
inline std::vector<Token> tokenize_bytes(const std::string& text) {
  return std::vector<Token>(reinterpret_cast<const uint8_t*>(text.data()),
                            reinterpret_cast<const uint8_t*>(text.data()) + text.size());
}
inline std::string detokenize_bytes(std::span<const Token> tokens) {
  std::string s;
  s.reserve(tokens.size());
  for (Token t : tokens) {
    if (t < 0 || t > 255) throw ContractError("detokenize_bytes: token outside byte vocabulary");
    s.push_back(static_cast<char>(t));
  }
  return s;
}

}  // namespace frag
