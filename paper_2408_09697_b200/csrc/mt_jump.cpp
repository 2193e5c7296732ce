// Jump-ahead for libstdc++'s std::mt19937_64, so that one long stream (a dense feature
// type of gen_synthetic, harness.cpp:153-162: one engine output per value) can be
// produced in parallel chunks that are bit-identical to the serial stream.
//
// The engine's word sequence satisfies w[n+312] = w[n+156] ^ twist(w[n], w[n+1]) (the
// recurrence of random.tcc:399-431); its 312-word windows V_n = (w_n .. w_{n+311}) evolve
// by a linear map T over GF(2). On windows that are images of T (all V_n, n >= 0: the low
// 31 bits of the oldest word never feed forward) T satisfies its characteristic
// polynomial phi of degree 19937, so T^J V = (t^J mod phi)(T) V. phi is recovered once by
// Berlekamp-Massey from 2 x 19937 output bits; t^J mod phi by square-and-multiply; the
// polynomial is applied to a window by Horner's rule (19937 window steps and XORs). An
// engine whose next output is w_m is the window V_{m-312} streamed into
// std::mt19937_64 with index 312 (operator>>, random.tcc:513-515).
#include <cstdint>
#include <map>
#include <mutex>
#include <random>
#include <sstream>
#include <stdexcept>
#include <vector>

#include "host.hpp"

namespace hetgpu {

namespace {

constexpr int kN = 312, kM = 156, kDeg = 19937;
constexpr std::uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL, kA = 0xB5026F5AA96619E9ULL;

std::uint64_t next_word(std::uint64_t w0, std::uint64_t w1, std::uint64_t w156) {
  const std::uint64_t y = (w0 & kUpper) | (w1 & kLower);
  return w156 ^ (y >> 1) ^ ((y & 1ULL) ? kA : 0ULL);
}

// GF(2) polynomial as a bit vector (bit i = coefficient of t^i)
struct Poly {
  std::vector<std::uint64_t> w;
  explicit Poly(std::size_t bits = 0) : w((bits + 63) / 64, 0) {}
  bool get(std::size_t i) const { return i / 64 < w.size() && ((w[i / 64] >> (i % 64)) & 1ULL); }
  void flip(std::size_t i) { w[i / 64] ^= 1ULL << (i % 64); }
  int degree() const {
    for (std::size_t k = w.size(); k-- > 0;)
      if (w[k]) return static_cast<int>(k * 64 + 63 - __builtin_clzll(w[k]));
    return -1;
  }
};

// a ^= b << s
void xor_shifted(std::vector<std::uint64_t>& a, const std::vector<std::uint64_t>& b, std::size_t s) {
  const std::size_t ws = s / 64, bs = s % 64;
  for (std::size_t k = 0; k < b.size(); ++k) {
    if (!b[k]) continue;
    if (k + ws < a.size()) a[k + ws] ^= b[k] << bs;
    if (bs && k + ws + 1 < a.size()) a[k + ws + 1] ^= b[k] >> (64 - bs);
  }
}

// r mod phi (phi monic of degree kDeg)
void reduce(Poly& r, const Poly& phi) {
  for (int d = r.degree(); d >= kDeg; d = r.degree()) xor_shifted(r.w, phi.w, static_cast<std::size_t>(d - kDeg));
}

// t^e mod phi
Poly pow_t(std::uint64_t e, const Poly& phi) {
  Poly r(kDeg + 64);
  r.flip(0);
  for (int bit = 63; bit >= 0; --bit) {
    // square: coefficient i -> 2i
    Poly sq(2 * kDeg + 128);
    for (int i = r.degree(); i >= 0; --i)
      if (r.get(static_cast<std::size_t>(i))) sq.flip(2 * static_cast<std::size_t>(i));
    reduce(sq, phi);
    r = sq;
    if ((e >> bit) & 1ULL) {
      Poly t1(2 * kDeg + 128);
      xor_shifted(t1.w, r.w, 1);
      reduce(t1, phi);
      r = t1;
    }
  }
  r.w.resize((kDeg + 63) / 64 + 1);
  return r;
}

// characteristic polynomial of T from the low bit of 2 x kDeg words (Berlekamp-Massey)
Poly characteristic() {
  std::mt19937_64 eng(0x5eed1234abcdULL);
  const int n_bits = 2 * kDeg;
  std::vector<std::uint8_t> s(n_bits);
  for (int i = 0; i < n_bits; ++i) s[i] = static_cast<std::uint8_t>(eng() & 1ULL);  // temper is linear
  const std::size_t bits = static_cast<std::size_t>(n_bits) + 128;
  Poly C(bits), B(bits), rs(bits);  // rs bit i = s[n - i]
  C.flip(0);
  B.flip(0);
  int L = 0, m = 1;
  for (int n = 0; n < n_bits; ++n) {
    std::uint64_t acc = 0;
    for (std::size_t k = 0; k < C.w.size(); ++k) acc ^= C.w[k] & rs.w[k];
    const int d = (s[n] ^ __builtin_parityll(acc)) & 1;
    if (d) {
      if (2 * L <= n) {
        const Poly Tmp = C;
        xor_shifted(C.w, B.w, static_cast<std::size_t>(m));
        L = n + 1 - L;
        B = Tmp;
        m = 1;
      } else {
        xor_shifted(C.w, B.w, static_cast<std::size_t>(m));
        ++m;
      }
    } else {
      ++m;
    }
    // shift rs by one (bit i -> i+1) and put s[n] at bit 1
    for (std::size_t k = rs.w.size(); k-- > 0;) rs.w[k] = (rs.w[k] << 1) | (k ? rs.w[k - 1] >> 63 : 0ULL);
    if (s[n]) rs.w[0] |= 2ULL;
  }
  if (L != kDeg) throw std::runtime_error("mt19937_64 jump: unexpected linear complexity " + std::to_string(L));
  Poly phi(kDeg + 64);  // phi_i = C_{L - i}
  for (int i = 0; i <= L; ++i)
    if (C.get(static_cast<std::size_t>(L - i))) phi.flip(static_cast<std::size_t>(i));
  return phi;
}

const Poly& phi() {
  static Poly p;
  static std::once_flag once;
  std::call_once(once, [] { p = characteristic(); });
  return p;
}

// g(T) V for a window V (positional words w_n .. w_{n+311}), Horner's rule
std::vector<std::uint64_t> apply_poly(const Poly& g, const std::vector<std::uint64_t>& v) {
  std::vector<std::uint64_t> buf(kN, 0);  // R as a circular window, logical k at (h + k) % kN
  int h = 0;
  for (int i = g.degree(); i >= 0; --i) {
    // R = T(R): append the next word, drop the oldest
    const std::uint64_t nw = next_word(buf[h], buf[(h + 1) % kN], buf[(h + kM) % kN]);
    buf[h] = nw;
    h = (h + 1) % kN;
    if (g.get(static_cast<std::size_t>(i)))
      for (int k = 0; k < kN; ++k) buf[(h + k) % kN] ^= v[k];
  }
  std::vector<std::uint64_t> out(kN);
  for (int k = 0; k < kN; ++k) out[k] = buf[(h + k) % kN];
  return out;
}

std::mt19937_64 engine_from_window(const std::vector<std::uint64_t>& v) {
  std::ostringstream os;
  for (int k = 0; k < kN; ++k) os << v[k] << ' ';
  os << kN;
  std::istringstream is(os.str());
  std::mt19937_64 e;
  is >> e;
  return e;
}

}  // namespace

// Engines whose next outputs are outputs starts[c] (ascending) of std::mt19937_64(seed):
// the stream split into chunks that can be generated concurrently.
std::vector<std::mt19937_64> mt64_jump_engines(std::uint64_t seed, const std::vector<std::uint64_t>& starts) {
  std::vector<std::mt19937_64> out;
  std::map<std::uint64_t, Poly> jumps;  // t^d mod phi per distinct step d (equal chunks: two)
  // V_0: the first 312 outputs' words (untempered), via a copy of the engine's state
  std::vector<std::uint64_t> v0(kN);
  {
    std::mt19937_64 e(seed);
    e();  // twist: the buffer now holds V_0 with index 1
    std::ostringstream os;
    os << e;
    std::istringstream is(os.str());
    for (int k = 0; k < kN; ++k) is >> v0[k];
  }
  std::vector<std::uint64_t> cur = v0;  // window V_{at}
  std::uint64_t at = 0;
  for (std::uint64_t m : starts) {
    if (m < static_cast<std::uint64_t>(kN)) {  // near the start: plain discard
      std::mt19937_64 e(seed);
      e.discard(m);
      out.push_back(e);
      continue;
    }
    const std::uint64_t target = m - kN;  // the engine's buffer is V_{m-312}
    if (target < at) throw std::invalid_argument("mt19937_64 jump: chunk starts must ascend");
    if (target > at) {
      auto it = jumps.find(target - at);
      if (it == jumps.end()) it = jumps.emplace(target - at, pow_t(target - at, phi())).first;
      cur = apply_poly(it->second, cur);
      at = target;
    }
    out.push_back(engine_from_window(cur));
  }
  return out;
}

}  // namespace hetgpu
