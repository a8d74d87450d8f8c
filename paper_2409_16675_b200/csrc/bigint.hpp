// Minimal host-side unsigned big integer for context constants
// (q = prod q_i, floor(q/t), (q-1)/2, mixed-radix weights ...).
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

namespace ctb {

struct BigU {
  std::vector<uint32_t> w;  // little-endian 32-bit words, no leading zeros
  BigU() {}
  explicit BigU(uint64_t v) { while (v) { w.push_back((uint32_t)v); v >>= 32; } }
  void trim() { while (!w.empty() && w.back() == 0) w.pop_back(); }
  bool is_zero() const { return w.empty(); }
  BigU& mul_small(uint64_t m) {
    unsigned __int128 carry = 0;
    for (auto& x : w) {
      unsigned __int128 t = (unsigned __int128)x * m + carry;
      x = (uint32_t)t;
      carry = t >> 32;
    }
    while (carry) { w.push_back((uint32_t)carry); carry >>= 32; }
    trim();
    return *this;
  }
  BigU& add_small(uint64_t a) {
    unsigned __int128 carry = a;
    for (size_t i = 0; carry && i < w.size(); ++i) {
      unsigned __int128 t = (unsigned __int128)w[i] + carry;
      w[i] = (uint32_t)t;
      carry = t >> 32;
    }
    while (carry) { w.push_back((uint32_t)carry); carry >>= 32; }
    return *this;
  }
  // floor-divide by m (< 2^63), returns remainder
  uint64_t divmod_small(uint64_t m) {
    unsigned __int128 rem = 0;
    for (size_t i = w.size(); i-- > 0;) {
      unsigned __int128 cur = (rem << 32) | w[i];
      w[i] = (uint32_t)(cur / m);
      rem = cur % m;
    }
    trim();
    return (uint64_t)rem;
  }
  uint64_t mod_small(uint64_t m) const { BigU c = *this; return c.divmod_small(m); }
  BigU& shr1() {
    for (size_t i = 0; i < w.size(); ++i) {
      w[i] >>= 1;
      if (i + 1 < w.size()) w[i] |= (w[i + 1] & 1u) << 31;
    }
    trim();
    return *this;
  }
  static int cmp(const BigU& a, const BigU& b) {
    if (a.w.size() != b.w.size()) return a.w.size() < b.w.size() ? -1 : 1;
    for (size_t i = a.w.size(); i-- > 0;)
      if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
  }
  static BigU add(const BigU& a, const BigU& b) {
    BigU r; r.w.resize(std::max(a.w.size(), b.w.size()) + 1, 0);
    uint64_t c = 0;
    for (size_t i = 0; i < r.w.size(); ++i) {
      uint64_t s = c + (i < a.w.size() ? a.w[i] : 0) + (i < b.w.size() ? b.w[i] : 0);
      r.w[i] = (uint32_t)s; c = s >> 32;
    }
    r.trim();
    return r;
  }
  // a - b, requires a >= b
  static BigU sub(const BigU& a, const BigU& b) {
    BigU r; r.w.resize(a.w.size(), 0);
    int64_t br = 0;
    for (size_t i = 0; i < a.w.size(); ++i) {
      int64_t s = (int64_t)a.w[i] - (i < b.w.size() ? b.w[i] : 0) - br;
      br = s < 0; if (s < 0) s += (1ll << 32);
      r.w[i] = (uint32_t)s;
    }
    r.trim();
    return r;
  }
  static BigU mul(const BigU& a, const BigU& b) {
    BigU r; r.w.assign(a.w.size() + b.w.size() + 1, 0);
    for (size_t i = 0; i < a.w.size(); ++i) {
      uint64_t c = 0;
      for (size_t j = 0; j < b.w.size(); ++j) {
        uint64_t t = (uint64_t)a.w[i] * b.w[j] + r.w[i + j] + c;
        r.w[i + j] = (uint32_t)t; c = t >> 32;
      }
      size_t k = i + b.w.size();
      while (c) { uint64_t t = (uint64_t)r.w[k] + c; r.w[k] = (uint32_t)t; c = t >> 32; ++k; }
    }
    r.trim();
    return r;
  }
  size_t bit_length() const {
    if (w.empty()) return 0;
    size_t b = 32 * (w.size() - 1);
    uint32_t top = w.back();
    while (top) { ++b; top >>= 1; }
    return b;
  }
  uint64_t word64(size_t k) const {
    uint64_t lo = 2 * k < w.size() ? w[2 * k] : 0, hi = 2 * k + 1 < w.size() ? w[2 * k + 1] : 0;
    return lo | (hi << 32);
  }
};

// floor(a / b) for big a and b (schoolbook via binary long division; host-only, tiny sizes)
inline BigU big_div(const BigU& a, const BigU& b, BigU* rem = nullptr) {
  BigU q, r;
  for (size_t i = a.bit_length(); i-- > 0;) {
    r.mul_small(2);
    if ((a.w[i / 32] >> (i % 32)) & 1u) r.add_small(1);
    q.mul_small(2);
    if (BigU::cmp(r, b) >= 0) { r = BigU::sub(r, b); q.add_small(1); }
  }
  if (rem) *rem = r;
  return q;
}

}  // namespace ctb
