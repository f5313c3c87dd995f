// SPDX-License-Identifier: Apache-2.0
//
// Host-side number theory for building device tables: primality, the
// smallest-generator primitive 2N-th root (same root as find_ntt_root,
// henet/modmath.hpp:195-222, because the smallest generator is unique), and
// the bit-reversed psi power tables of NttTables (henet/modmath.hpp:312-325).
#pragma once

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

namespace hg {
namespace nt {

using u64 = uint64_t;
using u128 = unsigned __int128;

inline u64 mulmod(u64 a, u64 b, u64 m) { return static_cast<u64>(static_cast<u128>(a) * b % m); }

inline u64 powmod(u64 b, u64 e, u64 m) {
  u64 r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = mulmod(r, b, m);
    b = mulmod(b, b, m);
    e >>= 1;
  }
  return r;
}

inline bool is_prime(u64 n) {
  if (n < 2) return false;
  static const u64 small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (u64 p : small) {
    if (n % p == 0) return n == p;
  }
  u64 d = n - 1;
  int r = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++r;
  }
  for (u64 a : small) {
    u64 x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool composite = true;
    for (int i = 1; i < r; ++i) {
      x = mulmod(x, x, n);
      if (x == n - 1) {
        composite = false;
        break;
      }
    }
    if (composite) return false;
  }
  return true;
}

inline u64 rho(u64 n) {
  if ((n & 1) == 0) return 2;
  for (u64 c = 1;; ++c) {
    u64 x = 2, y = 2, d = 1;
    auto f = [&](u64 v) { return static_cast<u64>((static_cast<u128>(v) * v + c) % n); };
    while (d == 1) {
      x = f(x);
      y = f(f(y));
      d = std::gcd(x > y ? x - y : y - x, n);
    }
    if (d != n) return d;
  }
}

inline void factor(u64 n, std::vector<u64>& out) {
  for (u64 p = 2; p < 1000 && p * p <= n; ++p) {
    if (n % p == 0) {
      out.push_back(p);
      while (n % p == 0) n /= p;
    }
  }
  if (n == 1) return;
  if (is_prime(n)) {
    out.push_back(n);
    return;
  }
  u64 d = rho(n);
  factor(d, out);
  factor(n / d, out);
}

// Smallest primitive root g of prime q, then psi = g^((q-1)/2N).
inline u64 primitive_2n_root(u64 q, u64 n) {
  std::vector<u64> f;
  factor(q - 1, f);
  std::sort(f.begin(), f.end());
  f.erase(std::unique(f.begin(), f.end()), f.end());
  for (u64 g = 2; g < q; ++g) {
    bool prim = true;
    for (u64 p : f) {
      if (powmod(g, (q - 1) / p, q) == 1) {
        prim = false;
        break;
      }
    }
    if (prim) return powmod(g, (q - 1) / (2 * n), q);
  }
  return 0;
}

inline uint32_t bit_reverse(uint32_t v, uint32_t bits) {
  uint32_t r = 0;
  for (uint32_t i = 0; i < bits; ++i) r = (r << 1) | ((v >> i) & 1);
  return r;
}

inline uint32_t shoup(u64 w, u64 q) { return static_cast<uint32_t>((static_cast<u128>(w) << 32) / q); }

inline u64 inv(u64 a, u64 q) { return powmod(a % q, q - 2, q); }

}  // namespace nt
}  // namespace hg
