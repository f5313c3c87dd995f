/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference algorithms
 * on the hot path (see henet_oracle.h).  Each function cites the reference
 * file:line it follows (paths relative to /root/reference/proj/include).
 * Compiled with -ffp-contract=off so the floating-point encode path rounds
 * every operation exactly as the reference's x86-64 build does.
 */
#include "henet_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef uint32_t u32;
typedef int64_t i64;
typedef unsigned __int128 u128;
typedef __int128 i128;

#define MAXB 32

typedef struct {
  u64 value;
  int bit_width;
  u64 r128_lo, r128_hi, r64; /* floor(2^128/q), floor(2^64/q) -- henet/modmath.hpp:91-115 */
} prime_t;

typedef struct {
  u64* root_powers; /* psi^bitrev(i) */
  u64* inv_root_powers;
  u64 degree_inv;
  u64 psi;
} ntt_t;

struct oc_ctx {
  u32 n, logn, L;
  int has_special;
  double scale;
  prime_t p[MAXB];
  ntt_t t[MAXB];
  long double qprod[MAXB + 1];
  double* dft_re; /* dft_roots_, henet/fft.hpp:34-38 */
  double* dft_im;
  double* tw_re; /* twist_, henet/fft.hpp:39-43 */
  double* tw_im;
  u32* bitrev;
};

/* ---------------------------------------------------------------------------
 * Word arithmetic (henet/common.hpp:50-65, henet/modmath.hpp:122-188)
 * ------------------------------------------------------------------------- */
static u64 mul_hw64(u64 a, u64 b) { return (u64)(((u128)a * b) >> 64); }

u64 oc_barrett_reduce_128_p(u64 z_lo, u64 z_hi, const prime_t* q) {
  u64 r0 = q->r128_lo, r1 = q->r128_hi;
  u64 carry = mul_hw64(z_lo, r0);
  u128 p = (u128)z_lo * r1;
  u64 prod_lo = (u64)p, prod_hi = (u64)(p >> 64);
  u64 tmp1 = prod_lo + carry;
  u64 tmp3 = prod_hi + (tmp1 < prod_lo);
  p = (u128)z_hi * r0;
  prod_lo = (u64)p;
  prod_hi = (u64)(p >> 64);
  u64 s = tmp1 + prod_lo;
  carry = prod_hi + (s < tmp1);
  tmp1 = z_hi * r1 + tmp3 + carry;
  tmp3 = z_lo - tmp1 * q->value;
  return tmp3 >= q->value ? tmp3 - q->value : tmp3;
}

static u64 barrett_reduce_64_p(u64 z, const prime_t* q) {
  u64 c = mul_hw64(z, q->r64);
  c = z - c * q->value;
  return c >= q->value ? c - q->value : c;
}

static void prime_init(prime_t* q, u64 v) {
  q->value = v;
  q->bit_width = 64 - __builtin_clzll(v);
  u64 d1 = (u64)(((u128)1 << 64) / v);
  u64 r1 = (u64)(((u128)1 << 64) % v);
  q->r128_hi = d1;
  q->r128_lo = (u64)(((u128)r1 << 64) / v);
  q->r64 = d1;
}

uint64_t oc_barrett_reduce_128(uint64_t lo, uint64_t hi, uint64_t qv) {
  prime_t q;
  prime_init(&q, qv);
  return oc_barrett_reduce_128_p(lo, hi, &q);
}

uint64_t oc_barrett_reduce_64(uint64_t z, uint64_t qv) {
  prime_t q;
  prime_init(&q, qv);
  return barrett_reduce_64_p(z, &q);
}

static inline u64 mod_add(u64 a, u64 b, const prime_t* q) {
  u64 s = a + b;
  return s >= q->value ? s - q->value : s;
}
static inline u64 mod_sub(u64 a, u64 b, const prime_t* q) { return a >= b ? a - b : a + q->value - b; }
static inline u64 mod_mul(u64 a, u64 b, const prime_t* q) {
  if (q->bit_width <= 32) return barrett_reduce_64_p(a * b, q);
  u128 z = (u128)a * b;
  return oc_barrett_reduce_128_p((u64)z, (u64)(z >> 64), q);
}
static u64 mod_pow(u64 b, u64 e, const prime_t* q) {
  u64 r = 1 % q->value;
  b %= q->value;
  while (e) {
    if (e & 1) r = mod_mul(r, b, q);
    b = mod_mul(b, b, q);
    e >>= 1;
  }
  return r;
}
static u64 mod_inv(u64 a, const prime_t* q) { return mod_pow(a, q->value - 2, q); }
static u64 mod_from_signed(i64 v, const prime_t* q) {
  i64 r = v % (i64)q->value;
  if (r < 0) r += (i64)q->value;
  return (u64)r;
}

/* ---------------------------------------------------------------------------
 * Primitive root (henet/modmath.hpp:29-97, 195-222): smallest generator g,
 * psi = g^((q-1)/2N).
 * ------------------------------------------------------------------------- */
static u64 powm(u64 b, u64 e, u64 m) {
  u64 r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = (u64)((u128)r * b % m);
    b = (u64)((u128)b * b % m);
    e >>= 1;
  }
  return r;
}
static int is_prime(u64 n) {
  static const u64 sp[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i)
    if (n % sp[i] == 0) return n == sp[i];
  u64 d = n - 1;
  int r = 0;
  while (!(d & 1)) {
    d >>= 1;
    ++r;
  }
  for (int i = 0; i < 12; ++i) {
    u64 x = powm(sp[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int wit = 1;
    for (int k = 1; k < r; ++k) {
      x = (u64)((u128)x * x % n);
      if (x == n - 1) {
        wit = 0;
        break;
      }
    }
    if (wit) return 0;
  }
  return 1;
}
static u64 gcd64(u64 a, u64 b) {
  while (b) {
    u64 t = a % b;
    a = b;
    b = t;
  }
  return a;
}
static u64 rho(u64 n) {
  if (!(n & 1)) return 2;
  for (u64 c = 1;; ++c) {
    u64 x = 2, y = 2, d = 1;
    while (d == 1) {
      x = (u64)(((u128)x * x + c) % n);
      y = (u64)(((u128)y * y + c) % n);
      y = (u64)(((u128)y * y + c) % n);
      d = gcd64(x > y ? x - y : y - x, n);
    }
    if (d != n) return d;
  }
}
static void factorize(u64 n, u64* f, int* nf) {
  if (n == 1) return;
  if (is_prime(n)) {
    for (int i = 0; i < *nf; ++i)
      if (f[i] == n) return;
    f[(*nf)++] = n;
    return;
  }
  u64 d = rho(n);
  factorize(d, f, nf);
  factorize(n / d, f, nf);
}
static u64 find_ntt_root(const prime_t* q, u32 n) {
  u64 f[64];
  int nf = 0;
  factorize(q->value - 1, f, &nf);
  for (u64 g = 2; g < q->value; ++g) {
    int prim = 1;
    for (int i = 0; i < nf; ++i)
      if (mod_pow(g, (q->value - 1) / f[i], q) == 1) {
        prim = 0;
        break;
      }
    if (prim) return mod_pow(g, (q->value - 1) / (2ull * n), q);
  }
  return 0;
}

static u32 bit_reverse(u32 v, u32 bits) {
  u32 r = 0;
  for (u32 i = 0; i < bits; ++i) r = (r << 1) | ((v >> i) & 1);
  return r;
}

/* NttTables (henet/modmath.hpp:303-334) */
static void ntt_init(ntt_t* t, const prime_t* q, u32 n, u32 logn) {
  t->psi = find_ntt_root(q, n);
  u64 psi_inv = mod_inv(t->psi, q);
  t->root_powers = malloc(sizeof(u64) * n);
  t->inv_root_powers = malloc(sizeof(u64) * n);
  for (u32 i = 0; i < n; ++i) {
    u32 rev = bit_reverse(i, logn);
    t->root_powers[i] = mod_pow(t->psi, rev, q);
    t->inv_root_powers[i] = mod_pow(psi_inv, rev, q);
  }
  t->degree_inv = mod_inv(n % q->value, q);
}

/* ntt_forward_limb (henet/modmath.hpp:338-355) */
static void ntt_fwd(const oc_ctx* c, u32 b, u64* a) {
  const prime_t* q = &c->p[b];
  const u64* rp = c->t[b].root_powers;
  u32 n = c->n, t = n;
  for (u32 m = 1; m < n; m <<= 1) {
    t >>= 1;
    for (u32 i = 0; i < m; ++i) {
      u64 w = rp[m + i];
      u32 j1 = 2 * i * t;
      for (u32 j = j1; j < j1 + t; ++j) {
        u64 u = a[j];
        u64 v = mod_mul(a[j + t], w, q);
        a[j] = mod_add(u, v, q);
        a[j + t] = mod_sub(u, v, q);
      }
    }
  }
}

/* ntt_inverse_limb (henet/modmath.hpp:357-377) */
static void ntt_inv(const oc_ctx* c, u32 b, u64* a) {
  const prime_t* q = &c->p[b];
  const u64* ip = c->t[b].inv_root_powers;
  u32 n = c->n, t = 1;
  for (u32 m = n >> 1; m >= 1; m >>= 1) {
    for (u32 i = 0; i < m; ++i) {
      u64 w = ip[m + i];
      u32 j1 = 2 * i * t;
      for (u32 j = j1; j < j1 + t; ++j) {
        u64 u = a[j], v = a[j + t];
        a[j] = mod_add(u, v, q);
        a[j + t] = mod_mul(mod_sub(u, v, q), w, q);
      }
    }
    t <<= 1;
  }
  for (u32 j = 0; j < n; ++j) a[j] = mod_mul(a[j], c->t[b].degree_inv, q);
}

void oc_ntt_forward(const oc_ctx* c, uint32_t b, uint64_t* limb) { ntt_fwd(c, b, limb); }
void oc_ntt_inverse(const oc_ctx* c, uint32_t b, uint64_t* limb) { ntt_inv(c, b, limb); }

/* ---------------------------------------------------------------------------
 * Context (henet/params.hpp:112-129, henet/fft.hpp:30-50)
 * ------------------------------------------------------------------------- */
oc_ctx* oc_ctx_create(uint32_t n, const uint64_t* chain, uint32_t L, uint64_t special, double scale) {
  if (L + 1 > MAXB) return NULL;
  oc_ctx* c = calloc(1, sizeof(oc_ctx));
  c->n = n;
  c->logn = 0;
  while ((1u << c->logn) < n) ++c->logn;
  c->L = L;
  c->has_special = special != 0;
  c->scale = scale;
  for (u32 i = 0; i < L; ++i) prime_init(&c->p[i], chain[i]);
  if (special) prime_init(&c->p[L], special);
  for (u32 i = 0; i < L + (special ? 1 : 0); ++i) ntt_init(&c->t[i], &c->p[i], n, c->logn);
  long double acc = 1.0L;
  c->qprod[0] = acc;
  for (u32 i = 0; i < L; ++i) {
    acc *= (long double)chain[i];
    c->qprod[i + 1] = acc;
  }
  const double pi = acos(-1.0);
  c->dft_re = malloc(sizeof(double) * n / 2);
  c->dft_im = malloc(sizeof(double) * n / 2);
  for (u32 k = 0; k < n / 2; ++k) {
    double ang = -2.0 * pi * k / n;
    c->dft_re[k] = cos(ang);
    c->dft_im[k] = sin(ang);
  }
  c->tw_re = malloc(sizeof(double) * n);
  c->tw_im = malloc(sizeof(double) * n);
  for (u32 k = 0; k < n; ++k) {
    double ang = pi * k / n;
    c->tw_re[k] = cos(ang);
    c->tw_im[k] = sin(ang);
  }
  c->bitrev = malloc(sizeof(u32) * n);
  for (u32 i = 0; i < n; ++i) c->bitrev[i] = bit_reverse(i, c->logn);
  return c;
}

void oc_ctx_destroy(oc_ctx* c) {
  if (!c) return;
  for (u32 i = 0; i < c->L + (c->has_special ? 1 : 0); ++i) {
    free(c->t[i].root_powers);
    free(c->t[i].inv_root_powers);
  }
  free(c->dft_re);
  free(c->dft_im);
  free(c->tw_re);
  free(c->tw_im);
  free(c->bitrev);
  free(c);
}

uint64_t oc_ntt_root(const oc_ctx* c, uint32_t b) { return c->t[b].psi; }

/* ---------------------------------------------------------------------------
 * Embedding FFT (henet/fft.hpp:57-105).  Complex products are written out as
 * (ac - bd) + (ad + bc)i, the order GCC emits for std::complex<double>.
 * ------------------------------------------------------------------------- */
typedef struct {
  double re, im;
} cplx;
static inline cplx cmul(cplx x, cplx w) {
  cplx r;
  r.re = x.re * w.re - x.im * w.im;
  r.im = x.re * w.im + x.im * w.re;
  return r;
}

static void dft_inplace(const oc_ctx* c, cplx* a) {
  u32 n = c->n;
  for (u32 i = 0; i < n; ++i) {
    u32 r = c->bitrev[i];
    if (i < r) {
      cplx t = a[i];
      a[i] = a[r];
      a[r] = t;
    }
  }
  for (u32 len = 2; len <= n; len <<= 1) {
    u32 step = n / len;
    for (u32 base = 0; base < n; base += len) {
      for (u32 k = 0; k < len / 2; ++k) {
        cplx w = {c->dft_re[k * step], c->dft_im[k * step]};
        cplx u = a[base + k];
        cplx v = cmul(a[base + k + len / 2], w);
        a[base + k].re = u.re + v.re;
        a[base + k].im = u.im + v.im;
        a[base + k + len / 2].re = u.re - v.re;
        a[base + k + len / 2].im = u.im - v.im;
      }
    }
  }
}

/* ---------------------------------------------------------------------------
 * Encoding (henet/encoding.hpp:122-197)
 * ------------------------------------------------------------------------- */
static u64 residue_from_i128(i128 x, const prime_t* q) {
  i128 r = x % (i128)q->value;
  if (r < 0) r += (i128)q->value;
  return (u64)r;
}

int oc_encode_scalar(const oc_ctx* c, double value, uint32_t level, double scale, uint64_t* out) {
  if (level < 1 || level > c->L || !(scale > 0.0)) return 1;
  long double scaled = (long double)value * (long double)scale;
  if (!((scaled < 0.0L ? -scaled : scaled) < c->qprod[level])) return 1;
  if (!(fabs((double)scaled) < ldexp(1.0, 100))) return 1;
  i128 x = (i128)roundl(scaled);
  for (u32 i = 0; i < level; ++i) out[i] = residue_from_i128(x, &c->p[i]);
  return 0;
}

int oc_encode_vector(const oc_ctx* c, const double* re_im, uint32_t ns, uint32_t level, double scale,
                     uint64_t* out) {
  u32 n = c->n;
  if (level < 1 || level > c->L || !(scale > 0.0) || ns > n / 2) return 1;
  cplx* e = calloc(n, sizeof(cplx));
  for (u32 j = 0; j < ns; ++j) {
    e[j].re = re_im[2 * j];
    e[j].im = re_im[2 * j + 1];
    e[n - 1 - j].re = re_im[2 * j];
    e[n - 1 - j].im = -re_im[2 * j + 1];
  }
  dft_inplace(c, e);
  const double inv_n = 1.0 / (double)n;
  i128* rounded = malloc(sizeof(i128) * n);
  long double max_scaled = 0.0L;
  int err = 0;
  for (u32 k = 0; k < n; ++k) {
    cplx tw = {c->tw_re[k], -c->tw_im[k]};
    cplx v = cmul(e[k], tw);
    double coeff = v.re * inv_n;
    long double scaled = (long double)coeff * (long double)scale;
    long double a = scaled < 0.0L ? -scaled : scaled;
    if (a > max_scaled) max_scaled = a;
    if (!(fabs((double)scaled) < ldexp(1.0, 100))) {
      err = 1;
      break;
    }
    rounded[k] = (i128)roundl(scaled);
  }
  if (!err && !(max_scaled < c->qprod[level] / 2.0L)) err = 1;
  if (!err) {
    for (u32 i = 0; i < level; ++i) {
      u64* limb = out + (size_t)i * n;
      for (u32 k = 0; k < n; ++k) limb[k] = residue_from_i128(rounded[k], &c->p[i]);
      ntt_fwd(c, i, limb);
    }
  }
  free(e);
  free(rounded);
  return err;
}

/* decode_slots (henet/encoding.hpp:223-267) with a small multi-word integer. */
#define WMAX 12
typedef struct {
  u64 w[WMAX];
  int n;
} wide_t;
static void w_set(wide_t* a, u64 v) {
  memset(a, 0, sizeof(*a));
  a->w[0] = v;
  a->n = 1;
}
static void w_mul_small(wide_t* a, u64 m) {
  u64 carry = 0;
  for (int i = 0; i < a->n; ++i) {
    u128 z = (u128)a->w[i] * m + carry;
    a->w[i] = (u64)z;
    carry = (u64)(z >> 64);
  }
  if (carry) a->w[a->n++] = carry;
}
static void w_add(wide_t* a, const wide_t* b) {
  int n = a->n > b->n ? a->n : b->n;
  u64 carry = 0;
  for (int i = 0; i < n; ++i) {
    u64 x = i < a->n ? a->w[i] : 0, y = i < b->n ? b->w[i] : 0;
    u128 s = (u128)x + y + carry;
    a->w[i] = (u64)s;
    carry = (u64)(s >> 64);
  }
  a->n = n;
  if (carry) a->w[a->n++] = carry;
}
static void w_trim(wide_t* a) {
  while (a->n > 1 && a->w[a->n - 1] == 0) --a->n;
}
static void w_sub(wide_t* a, const wide_t* b) { /* a >= b */
  u64 borrow = 0;
  for (int i = 0; i < a->n; ++i) {
    u64 y = i < b->n ? b->w[i] : 0;
    u128 need = (u128)y + borrow;
    if ((u128)a->w[i] >= need) {
      a->w[i] = (u64)((u128)a->w[i] - need);
      borrow = 0;
    } else {
      a->w[i] = (u64)(((u128)1 << 64) + a->w[i] - need);
      borrow = 1;
    }
  }
  w_trim(a);
}
static int w_cmp(const wide_t* a, const wide_t* b) {
  int n = a->n > b->n ? a->n : b->n;
  for (int i = n - 1; i >= 0; --i) {
    u64 x = i < a->n ? a->w[i] : 0, y = i < b->n ? b->w[i] : 0;
    if (x != y) return x < y ? -1 : 1;
  }
  return 0;
}
static void w_shr1(wide_t* a) {
  for (int i = 0; i < a->n; ++i) {
    u64 nx = i + 1 < a->n ? a->w[i + 1] : 0;
    a->w[i] = (a->w[i] >> 1) | (nx << 63);
  }
  w_trim(a);
}
static u64 w_mod(const wide_t* a, const prime_t* q) {
  u64 r = 0;
  for (int i = a->n - 1; i >= 0; --i) r = oc_barrett_reduce_128_p(a->w[i], r, q);
  return r;
}
static long double w_ld(const wide_t* a) {
  long double v = 0.0L;
  for (int i = a->n - 1; i >= 0; --i) v = v * 18446744073709551616.0L + (long double)a->w[i];
  return v;
}

void oc_decode(const oc_ctx* c, const uint64_t* words, uint32_t level, double scale, double* out_re_im) {
  u32 n = c->n;
  u64* poly = malloc(sizeof(u64) * n * level);
  memcpy(poly, words, sizeof(u64) * n * level);
  for (u32 i = 0; i < level; ++i) ntt_inv(c, i, poly + (size_t)i * n);
  wide_t big_q, q_half, q_over_p[MAXB];
  u64 inv[MAXB];
  w_set(&big_q, 1);
  for (u32 i = 0; i < level; ++i) w_mul_small(&big_q, c->p[i].value);
  q_half = big_q;
  w_shr1(&q_half);
  for (u32 i = 0; i < level; ++i) {
    w_set(&q_over_p[i], 1);
    for (u32 j = 0; j < level; ++j)
      if (j != i) w_mul_small(&q_over_p[i], c->p[j].value);
    inv[i] = mod_inv(w_mod(&q_over_p[i], &c->p[i]), &c->p[i]);
  }
  double* coeffs = malloc(sizeof(double) * n);
  const long double inv_scale = 1.0L / (long double)scale;
  for (u32 k = 0; k < n; ++k) {
    wide_t acc;
    w_set(&acc, 0);
    for (u32 i = 0; i < level; ++i) {
      u64 y = mod_mul(poly[(size_t)i * n + k], inv[i], &c->p[i]);
      wide_t term = q_over_p[i];
      w_mul_small(&term, y);
      w_add(&acc, &term);
    }
    while (w_cmp(&acc, &big_q) >= 0) w_sub(&acc, &big_q);
    if (w_cmp(&acc, &q_half) > 0) {
      wide_t neg = big_q;
      w_sub(&neg, &acc);
      coeffs[k] = (double)(-w_ld(&neg) * inv_scale);
    } else {
      coeffs[k] = (double)(w_ld(&acc) * inv_scale);
    }
  }
  /* coeffs_to_slots (henet/fft.hpp:77-85) */
  cplx* y = malloc(sizeof(cplx) * n);
  for (u32 k = 0; k < n; ++k) {
    y[k].re = c->tw_re[k] * coeffs[k];
    y[k].im = -(c->tw_im[k] * coeffs[k]);
  }
  dft_inplace(c, y);
  for (u32 j = 0; j < n / 2; ++j) {
    out_re_im[2 * j] = y[j].re;
    out_re_im[2 * j + 1] = -y[j].im;
  }
  free(y);
  free(coeffs);
  free(poly);
}

/* ---------------------------------------------------------------------------
 * Ciphertext operations (henet/ckks.hpp:88-154, 281-524)
 * ------------------------------------------------------------------------- */
void oc_add_ct_ct(const oc_ctx* c, const uint64_t* a, const uint64_t* b, uint32_t polys, uint32_t level,
                  uint64_t* out) {
  u32 n = c->n;
  for (u32 k = 0; k < polys; ++k)
    for (u32 i = 0; i < level; ++i) {
      size_t o = ((size_t)k * level + i) * n;
      for (u32 j = 0; j < n; ++j) out[o + j] = mod_add(a[o + j], b[o + j], &c->p[i]);
    }
}

/* mul_ct_pt_scalar_inplace (henet/ckks.hpp:363-385) */
void oc_mul_ct_pt_scalar(const oc_ctx* c, const uint64_t* ct, uint32_t polys, uint32_t level,
                         const uint64_t* res, uint64_t* out) {
  u32 n = c->n;
  for (u32 k = 0; k < polys; ++k)
    for (u32 i = 0; i < level; ++i) {
      const prime_t* q = &c->p[i];
      size_t o = ((size_t)k * level + i) * n;
      if (q->bit_width <= 32) {
        for (u32 j = 0; j < n; ++j) out[o + j] = barrett_reduce_64_p(ct[o + j] * res[i], q);
      } else {
        for (u32 j = 0; j < n; ++j) {
          u128 z = (u128)ct[o + j] * res[i];
          out[o + j] = oc_barrett_reduce_128_p((u64)z, (u64)(z >> 64), q);
        }
      }
    }
}

void oc_add_ct_pt_vector(const oc_ctx* c, const uint64_t* ct, uint32_t polys, uint32_t level, const uint64_t* pt,
                         uint64_t* out) {
  u32 n = c->n;
  memcpy(out, ct, sizeof(u64) * polys * level * n);
  for (u32 i = 0; i < level; ++i)
    for (u32 j = 0; j < n; ++j) out[(size_t)i * n + j] = mod_add(ct[(size_t)i * n + j], pt[(size_t)i * n + j], &c->p[i]);
}

static void mul_elem(const oc_ctx* c, const u64* a, const u64* b, u32 limbs, u64* out) {
  u32 n = c->n;
  for (u32 i = 0; i < limbs; ++i)
    for (u32 j = 0; j < n; ++j) out[(size_t)i * n + j] = mod_mul(a[(size_t)i * n + j], b[(size_t)i * n + j], &c->p[i]);
}

void oc_square(const oc_ctx* c, const uint64_t* ct, uint32_t level, uint64_t* out3) {
  size_t pw = (size_t)level * c->n;
  mul_elem(c, ct, ct, level, out3);
  mul_elem(c, ct, ct + pw, level, out3 + pw);
  for (u32 i = 0; i < level; ++i)
    for (u32 j = 0; j < c->n; ++j) {
      size_t o = pw + (size_t)i * c->n + j;
      out3[o] = mod_add(out3[o], out3[o], &c->p[i]);
    }
  mul_elem(c, ct + pw, ct + pw, level, out3 + 2 * pw);
}

void oc_mul_ct_ct(const oc_ctx* c, const uint64_t* a, const uint64_t* b, uint32_t level, uint64_t* out3) {
  size_t pw = (size_t)level * c->n;
  u64* tmp = malloc(sizeof(u64) * pw);
  mul_elem(c, a, b, level, out3);
  mul_elem(c, a, b + pw, level, out3 + pw);
  mul_elem(c, a + pw, b, level, tmp);
  for (u32 i = 0; i < level; ++i)
    for (u32 j = 0; j < c->n; ++j) {
      size_t o = (size_t)i * c->n + j;
      out3[pw + o] = mod_add(out3[pw + o], tmp[o], &c->p[i]);
    }
  mul_elem(c, a + pw, b + pw, level, out3 + 2 * pw);
  free(tmp);
}

/* divide_round_last (henet/ckks.hpp:132-154); `moduli` given as basis indices. */
static void divide_round_last(const oc_ctx* c, u64* x, const u32* bidx, u32 lvl) {
  u32 n = c->n, last = lvl - 1;
  const prime_t* p = &c->p[bidx[last]];
  u64 half = p->value >> 1;
  u64* rl = x + (size_t)last * n;
  for (u32 j = 0; j < n; ++j) rl[j] = mod_add(rl[j], half, p);
  for (u32 i = 0; i < last; ++i) {
    const prime_t* q = &c->p[bidx[i]];
    u64 half_mod = oc_barrett_reduce_128_p(half, 0, q);
    u64 p_inv = mod_inv(oc_barrett_reduce_128_p(p->value, 0, q), q);
    u64* li = x + (size_t)i * n;
    for (u32 j = 0; j < n; ++j) {
      u64 r = oc_barrett_reduce_128_p(rl[j], 0, q);
      u64 y = mod_sub(mod_add(li[j], half_mod, q), r, q);
      li[j] = mod_mul(y, p_inv, q);
    }
  }
}

/* relinearize (henet/ckks.hpp:442-499) */
void oc_relinearize(const oc_ctx* c, const uint64_t* ct3, uint32_t level, const uint64_t* rk, uint64_t* out2) {
  u32 n = c->n, L = c->L, ext = level + 1;
  size_t pw = (size_t)level * n;
  u64* c2 = malloc(sizeof(u64) * pw);
  memcpy(c2, ct3 + 2 * pw, sizeof(u64) * pw);
  for (u32 i = 0; i < level; ++i) ntt_inv(c, i, c2 + (size_t)i * n);
  u64* acc[2];
  acc[0] = calloc((size_t)ext * n, sizeof(u64));
  acc[1] = calloc((size_t)ext * n, sizeof(u64));
  u64* tmp = malloc(sizeof(u64) * n);
  u32 bidx[MAXB];
  for (u32 t = 0; t < level; ++t) bidx[t] = t;
  bidx[level] = L; /* special */
  for (u32 j = 0; j < level; ++j) {
    const u64* digit = c2 + (size_t)j * n;
    for (u32 t = 0; t < ext; ++t) {
      const prime_t* q = &c->p[bidx[t]];
      for (u32 k = 0; k < n; ++k) tmp[k] = digit[k] < q->value ? digit[k] : oc_barrett_reduce_128_p(digit[k], 0, q);
      ntt_fwd(c, bidx[t], tmp);
      u32 key_idx = t == level ? L : t;
      const u64* k0 = rk + (((size_t)j * 2 + 0) * (L + 1) + key_idx) * n;
      const u64* k1 = rk + (((size_t)j * 2 + 1) * (L + 1) + key_idx) * n;
      u64* a0 = acc[0] + (size_t)t * n;
      u64* a1 = acc[1] + (size_t)t * n;
      for (u32 k = 0; k < n; ++k) {
        a0[k] = mod_add(a0[k], mod_mul(tmp[k], k0[k], q), q);
        a1[k] = mod_add(a1[k], mod_mul(tmp[k], k1[k], q), q);
      }
    }
  }
  for (int a = 0; a < 2; ++a) {
    for (u32 i = 0; i < ext; ++i) ntt_inv(c, bidx[i], acc[a] + (size_t)i * n);
    divide_round_last(c, acc[a], bidx, ext);
    for (u32 i = 0; i < level; ++i) ntt_fwd(c, i, acc[a] + (size_t)i * n);
    for (u32 i = 0; i < level; ++i)
      for (u32 k = 0; k < n; ++k) {
        size_t o = (size_t)i * n + k;
        out2[a * pw + o] = mod_add(acc[a][o], ct3[a * pw + o], &c->p[i]);
      }
  }
  free(c2);
  free(acc[0]);
  free(acc[1]);
  free(tmp);
}

/* rescale (henet/ckks.hpp:504-519) */
int oc_rescale(const oc_ctx* c, const uint64_t* ct, uint32_t polys, uint32_t level, uint32_t target, uint64_t* out) {
  if (level < 2 || target < 1 || target >= level) return 1;
  u32 n = c->n;
  u64* cur = malloc(sizeof(u64) * polys * level * n);
  memcpy(cur, ct, sizeof(u64) * polys * level * n);
  u32 bidx[MAXB];
  for (u32 i = 0; i < MAXB; ++i) bidx[i] = i;
  u32 lvl = level;
  while (lvl > target) {
    u64* nxt = malloc(sizeof(u64) * polys * (lvl - 1) * n);
    for (u32 k = 0; k < polys; ++k) {
      u64* p = cur + (size_t)k * lvl * n;
      for (u32 i = 0; i < lvl; ++i) ntt_inv(c, i, p + (size_t)i * n);
      divide_round_last(c, p, bidx, lvl);
      for (u32 i = 0; i + 1 < lvl; ++i) ntt_fwd(c, i, p + (size_t)i * n);
      memcpy(nxt + (size_t)k * (lvl - 1) * n, p, sizeof(u64) * (lvl - 1) * n);
    }
    free(cur);
    cur = nxt;
    --lvl;
  }
  memcpy(out, cur, sizeof(u64) * polys * target * n);
  free(cur);
  return 0;
}

/* ---------------------------------------------------------------------------
 * ChaCha20 stream and samplers (henet/rng.hpp:21-125)
 * ------------------------------------------------------------------------- */
typedef struct {
  u32 state[16], block[16];
  int pos;
} chacha_t;
static inline u32 rotl(u32 x, int n) { return (x << n) | (x >> (32 - n)); }
#define QR(a, b, c, d) \
  a += b; d ^= a; d = rotl(d, 16); \
  c += d; b ^= c; b = rotl(b, 12); \
  a += b; d ^= a; d = rotl(d, 8);  \
  c += d; b ^= c; b = rotl(b, 7);
static void cc_refill(chacha_t* r) {
  u32 x[16];
  memcpy(x, r->state, sizeof(x));
  for (int i = 0; i < 10; ++i) {
    QR(x[0], x[4], x[8], x[12]) QR(x[1], x[5], x[9], x[13]) QR(x[2], x[6], x[10], x[14])
    QR(x[3], x[7], x[11], x[15]) QR(x[0], x[5], x[10], x[15]) QR(x[1], x[6], x[11], x[12])
    QR(x[2], x[7], x[8], x[13]) QR(x[3], x[4], x[9], x[14])
  }
  for (int i = 0; i < 16; ++i) r->block[i] = x[i] + r->state[i];
  if (++r->state[12] == 0) ++r->state[13];
  r->pos = 0;
}
static void cc_init(chacha_t* r, u64 seed, u64 stream) {
  r->state[0] = 0x61707865;
  r->state[1] = 0x3320646e;
  r->state[2] = 0x79622d32;
  r->state[3] = 0x6b206574;
  r->state[4] = (u32)seed;
  r->state[5] = (u32)(seed >> 32);
  r->state[6] = (u32)stream;
  r->state[7] = (u32)(stream >> 32);
  r->state[8] = (u32)(seed ^ 0x9e3779b97f4a7c15ULL);
  r->state[9] = (u32)((seed ^ 0x9e3779b97f4a7c15ULL) >> 32);
  r->state[10] = (u32)(stream ^ 0xbf58476d1ce4e5b9ULL);
  r->state[11] = (u32)((stream ^ 0xbf58476d1ce4e5b9ULL) >> 32);
  r->state[12] = 0;
  r->state[13] = 0;
  r->state[14] = 0x68650000u;
  r->state[15] = 0;
  cc_refill(r);
}
static u64 cc_u64(chacha_t* r) {
  if (r->pos + 2 > 16) cc_refill(r);
  u64 lo = r->block[r->pos], hi = r->block[r->pos + 1];
  r->pos += 2;
  return lo | (hi << 32);
}
static double cc_double(chacha_t* r) { return (double)(cc_u64(r) >> 11) * 0x1.0p-53; }
static u64 cc_below(chacha_t* r, u64 bound) {
  u64 threshold = (0 - bound) % bound;
  for (;;) {
    u64 x = cc_u64(r);
    if (x >= threshold) return x % bound;
  }
}
uint64_t oc_derive_seed(uint64_t seed, uint64_t tag) {
  u64 z = seed + 0x9e3779b97f4a7c15ULL * (tag + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static i64 sample_ternary(chacha_t* r) { return (i64)cc_below(r, 3) - 1; }
static i64 sample_gaussian(chacha_t* r, double sigma) {
  double u1 = cc_double(r), u2 = cc_double(r);
  while (u1 <= 0.0) u1 = cc_double(r);
  double g = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
  double v = g * sigma, cap = 6.0 * sigma;
  if (v > cap) v = cap;
  if (v < -cap) v = -cap;
  return (i64)llround(v);
}

/* lift_signed / sample_uniform / sample_error (henet/ckks.hpp:58-86), limbs over the full basis */
static void lift_signed(const oc_ctx* c, const i64* v, u32 limbs, u64* out) {
  u32 n = c->n;
  for (u32 i = 0; i < limbs; ++i) {
    for (u32 k = 0; k < n; ++k) out[(size_t)i * n + k] = mod_from_signed(v[k], &c->p[i]);
    ntt_fwd(c, i, out + (size_t)i * n);
  }
}
static void sample_uniform(const oc_ctx* c, chacha_t* r, u32 limbs, u64* out) {
  for (u32 i = 0; i < limbs; ++i)
    for (u32 k = 0; k < c->n; ++k) out[(size_t)i * c->n + k] = cc_below(r, c->p[i].value);
}
static void sample_error(const oc_ctx* c, chacha_t* r, u32 limbs, u64* out) {
  i64* e = malloc(sizeof(i64) * c->n);
  for (u32 k = 0; k < c->n; ++k) e[k] = sample_gaussian(r, 3.2);
  lift_signed(c, e, limbs, out);
  free(e);
}

/* keygen (henet/ckks.hpp:186-222) */
void oc_keygen(const oc_ctx* c, uint64_t seed, uint64_t* sk, uint64_t* rk) {
  u32 n = c->n, L = c->L, full = L + (c->has_special ? 1 : 0);
  chacha_t r;
  cc_init(&r, seed, 0);
  i64* s = malloc(sizeof(i64) * n);
  for (u32 k = 0; k < n; ++k) s[k] = sample_ternary(&r);
  lift_signed(c, s, full, sk);
  free(s);
  if (!rk || !c->has_special) return;
  size_t fw = (size_t)full * n;
  u64* s_sq = malloc(sizeof(u64) * fw);
  mul_elem(c, sk, sk, full, s_sq);
  u64* a = malloc(sizeof(u64) * fw);
  u64* as = malloc(sizeof(u64) * fw);
  for (u32 j = 0; j < L; ++j) {
    u64* c0 = rk + ((size_t)j * 2 + 0) * fw;
    u64* c1 = rk + ((size_t)j * 2 + 1) * fw;
    sample_uniform(c, &r, full, a);
    sample_error(c, &r, full, c0);
    mul_elem(c, a, sk, full, as);
    for (u32 i = 0; i < full; ++i)
      for (u32 k = 0; k < n; ++k) {
        size_t o = (size_t)i * n + k;
        c0[o] = mod_sub(c0[o], as[o], &c->p[i]);
      }
    const prime_t* qj = &c->p[j];
    u64 p_mod = oc_barrett_reduce_128_p(c->p[L].value, 0, qj);
    for (u32 k = 0; k < n; ++k) {
      size_t o = (size_t)j * n + k;
      c0[o] = mod_add(c0[o], mod_mul(p_mod, s_sq[o], qj), qj);
    }
    memcpy(c1, a, sizeof(u64) * fw);
  }
  free(s_sq);
  free(a);
  free(as);
}

/* encrypt_batch (henet/ckks.hpp:229-254, encoding.hpp:72-87) */
int oc_encrypt_batch(const oc_ctx* c, const uint64_t* sk, const double* values, uint32_t count, int packing,
                     uint64_t seed, uint64_t* out) {
  u32 n = c->n, L = c->L;
  u32 ns = packing ? count / 2 : count;
  double* slots = calloc(2 * (size_t)(ns ? ns : 1), sizeof(double));
  for (u32 j = 0; j < ns; ++j) {
    slots[2 * j] = values[j];
    slots[2 * j + 1] = packing ? values[j + ns] : 0.0;
  }
  size_t pw = (size_t)L * n;
  u64* pt = malloc(sizeof(u64) * pw);
  int err = oc_encode_vector(c, slots, ns, L, c->scale, pt);
  free(slots);
  if (err) {
    free(pt);
    return err;
  }
  chacha_t r;
  cc_init(&r, seed, 1);
  u64* a = out + pw;
  u64* c0 = out;
  sample_uniform(c, &r, L, a);
  sample_error(c, &r, L, c0);
  u64* as = malloc(sizeof(u64) * pw);
  mul_elem(c, a, sk, L, as);
  for (u32 i = 0; i < L; ++i)
    for (u32 k = 0; k < n; ++k) {
      size_t o = (size_t)i * n + k;
      c0[o] = mod_add(mod_sub(c0[o], as[o], &c->p[i]), pt[o], &c->p[i]);
    }
  free(as);
  free(pt);
  return 0;
}

void oc_decrypt(const oc_ctx* c, const uint64_t* sk, const uint64_t* ct, uint32_t polys, uint32_t level,
                double scale, double* out_re_im) {
  u32 n = c->n;
  size_t pw = (size_t)level * n;
  u64* m = malloc(sizeof(u64) * pw);
  u64* t = malloc(sizeof(u64) * pw);
  memcpy(m, ct, sizeof(u64) * pw);
  mul_elem(c, ct + pw, sk, level, t);
  for (size_t o = 0; o < pw; ++o) m[o] = mod_add(m[o], t[o], &c->p[o / n]);
  if (polys == 3) {
    u64* s2 = malloc(sizeof(u64) * pw);
    mul_elem(c, sk, sk, level, s2);
    mul_elem(c, ct + 2 * pw, s2, level, t);
    for (size_t o = 0; o < pw; ++o) m[o] = mod_add(m[o], t[o], &c->p[o / n]);
    free(s2);
  }
  oc_decode(c, m, level, scale, out_re_im);
  free(m);
  free(t);
}

/* ---------------------------------------------------------------------------
 * Graph layers (henet/graph.hpp:905-1008)
 * ------------------------------------------------------------------------- */
static int bias_plaintext(const oc_ctx* c, double b, int packing, u32 level, double acc_scale, u64* pt) {
  u32 n = c->n;
  if (packing == 0) { /* expand_scalar(encode_scalar(...)), henet/encoding.hpp:210-219, 275-280 */
    u64 res[MAXB];
    if (oc_encode_scalar(c, b, level, acc_scale, res)) return 1;
    for (u32 i = 0; i < level; ++i)
      for (u32 k = 0; k < n; ++k) pt[(size_t)i * n + k] = res[i];
    return 0;
  }
  double* slots = malloc(sizeof(double) * n); /* n/2 complex (b, b) */
  for (u32 j = 0; j < n / 2; ++j) {
    slots[2 * j] = b;
    slots[2 * j + 1] = b;
  }
  int e = oc_encode_vector(c, slots, n / 2, level, acc_scale, pt);
  free(slots);
  return e;
}

/* one mac_output: taps (in_idx, weight) in ascending order */
static int mac_output(const oc_ctx* c, const u64* x, const u32* tap_in, const float* tap_w, u32 ntaps, u32 level,
                      double x_scale, int has_bias, double bias, int packing, int rescale, u64* out) {
  u32 n = c->n;
  size_t cw = 2 * (size_t)level * n;
  u64* acc = malloc(sizeof(u64) * cw);
  u64* term = malloc(sizeof(u64) * cw);
  u64 res[MAXB];
  int err = 0;
  for (u32 t = 0; t < ntaps && !err; ++t) {
    if (oc_encode_scalar(c, (double)tap_w[t], level, c->scale, res)) {
      err = 1;
      break;
    }
    oc_mul_ct_pt_scalar(c, x + (size_t)tap_in[t] * cw, 2, level, res, t == 0 ? acc : term);
    if (t) oc_add_ct_ct(c, acc, term, 2, level, acc);
  }
  if (!err && has_bias) {
    u64* pt = malloc(sizeof(u64) * level * n);
    err = bias_plaintext(c, bias, packing, level, x_scale * c->scale, pt);
    if (!err) oc_add_ct_pt_vector(c, acc, 2, level, pt, acc);
    free(pt);
  }
  if (!err) {
    if (rescale) err = oc_rescale(c, acc, 2, level, level - 1, out);
    else memcpy(out, acc, sizeof(u64) * cw);
  }
  free(acc);
  free(term);
  return err;
}

int oc_dense(const oc_ctx* c, const uint64_t* x, uint32_t K, uint32_t M, uint32_t level, double x_scale,
             const float* w, const float* bias, int packing, int rescale, const uint32_t* outputs,
             uint32_t n_outputs, uint64_t* out) {
  u32 cnt = outputs ? n_outputs : M;
  u32 lo = rescale ? level - 1 : level;
  size_t ow = 2 * (size_t)lo * c->n;
  int err = 0;
#pragma omp parallel for schedule(dynamic) reduction(| : err)
  for (u32 o = 0; o < cnt; ++o) {
    u32 j = outputs ? outputs[o] : o;
    u32* tin = malloc(sizeof(u32) * K);
    float* tw = malloc(sizeof(float) * K);
    for (u32 i = 0; i < K; ++i) {
      tin[i] = i;
      tw[i] = w[(size_t)i * M + j];
    }
    err |= mac_output(c, x, tin, tw, K, level, x_scale, bias != NULL, bias ? bias[j] : 0.0, packing, rescale,
                      out + (size_t)o * ow);
    free(tin);
    free(tw);
  }
  return err;
}

/* oc_dense for large K without a bias (the c5b shape): the same residues as mac_output's
 * per-tap mul_ct_pt_scalar + add_ct_ct chain (henet/graph.hpp:905-933), computed as one
 * 128-bit sum of the products per residue and a single Barrett128 at the end:
 * sum_i (a_i b_i mod p) mod p == (sum_i a_i b_i) mod p, and K < 2^48 terms of < 2^80 fit
 * in 128 bits.  Blocked over residues so x streams through memory once for all outputs.
 * tests/test_oracle_golden.py checks it against oc_dense. */
int oc_dense_lazy(const oc_ctx* c, const uint64_t* x, uint32_t K, uint32_t M, uint32_t level,
                  const float* w, int rescale, uint64_t* out) {
  const u32 n = c->n;
  const size_t cw = 2 * (size_t)level * n;
  u64* wres = malloc(sizeof(u64) * (size_t)K * M * level); /* [limb][k][m] */
  u64* acc = malloc(sizeof(u64) * (size_t)M * cw);         /* canonical sums, [m][poly][limb][N] */
  int err = 0;
  for (u32 k = 0; k < K && !err; ++k)
    for (u32 m = 0; m < M && !err; ++m) {
      u64 r[MAXB];
      if (oc_encode_scalar(c, (double)w[(size_t)k * M + m], level, c->scale, r)) err = 1;
      for (u32 i = 0; i < level; ++i) wres[((size_t)i * K + k) * M + m] = r[i];
    }
  if (err) {
    free(wres);
    free(acc);
    return 1;
  }
  enum { RB = 64 };
  const size_t nblk = cw / RB;
#pragma omp parallel
  {
    u128* s = malloc(sizeof(u128) * (size_t)M * RB);
#pragma omp for schedule(dynamic)
    for (size_t b = 0; b < nblk; ++b) {
      const size_t r0 = b * RB;
      const u32 limb = (u32)((r0 / n) % level);
      const u64* wl = wres + (size_t)limb * K * M;
      memset(s, 0, sizeof(u128) * (size_t)M * RB);
      for (u32 k = 0; k < K; ++k) {
        const u64* xk = x + (size_t)k * cw + r0;
        const u64* wk = wl + (size_t)k * M;
        for (u32 m = 0; m < M; ++m) {
          const u64 wv = wk[m];
          u128* sm = s + (size_t)m * RB;
          for (u32 t = 0; t < RB; ++t) sm[t] += (u128)xk[t] * wv;
        }
      }
      const prime_t* q = &c->p[limb];
      for (u32 m = 0; m < M; ++m)
        for (u32 t = 0; t < RB; ++t) {
          const u128 z = s[(size_t)m * RB + t];
          acc[(size_t)m * cw + r0 + t] = oc_barrett_reduce_128_p((u64)z, (u64)(z >> 64), q);
        }
    }
    free(s);
  }
  const u32 lo = rescale ? level - 1 : level;
  const size_t ow = 2 * (size_t)lo * n;
#pragma omp parallel for schedule(dynamic) reduction(| : err)
  for (u32 m = 0; m < M; ++m) {
    if (rescale) err |= oc_rescale(c, acc + (size_t)m * cw, 2, level, level - 1, out + (size_t)m * ow);
    else memcpy(out + (size_t)m * ow, acc + (size_t)m * cw, sizeof(u64) * cw);
  }
  free(wres);
  free(acc);
  return err;
}

int oc_conv(const oc_ctx* c, const uint64_t* x, uint32_t C, uint32_t IH, uint32_t IW, uint32_t F, uint32_t win,
            uint32_t stride, uint32_t pad_top, uint32_t pad_left, uint32_t OH, uint32_t OW, uint32_t level,
            double x_scale, const float* w, const float* bias, int packing, int rescale, const uint32_t* outputs,
            uint32_t n_outputs, uint64_t* out) {
  u32 total = F * OH * OW;
  u32 cnt = outputs ? n_outputs : total;
  u32 lo = rescale ? level - 1 : level;
  size_t ow = 2 * (size_t)lo * c->n;
  int err = 0;
#pragma omp parallel for schedule(dynamic) reduction(| : err)
  for (u32 o = 0; o < cnt; ++o) {
    u32 e = outputs ? outputs[o] : o;
    u32 f = e / (OH * OW), y = (e / OW) % OH, xo = e % OW;
    u32* tin = malloc(sizeof(u32) * C * win * win);
    float* tw = malloc(sizeof(float) * C * win * win);
    u32 nt = 0;
    for (u32 ch = 0; ch < C; ++ch)
      for (u32 ky = 0; ky < win; ++ky)
        for (u32 kx = 0; kx < win; ++kx) {
          i64 iy = (i64)y * stride + ky - pad_top;
          i64 ix = (i64)xo * stride + kx - pad_left;
          if (iy < 0 || iy >= IH || ix < 0 || ix >= IW) continue;
          tin[nt] = (u32)(((size_t)ch * IH + iy) * IW + ix);
          tw[nt] = w[(((size_t)f * C + ch) * win + ky) * win + kx];
          ++nt;
        }
    err |= mac_output(c, x, tin, tw, nt, level, x_scale, bias != NULL, bias ? bias[f] : 0.0, packing, rescale,
                      out + (size_t)o * ow);
    free(tin);
    free(tw);
  }
  return err;
}

void oc_square_layer(const oc_ctx* c, const uint64_t* x, uint64_t count, uint32_t level, const uint64_t* rk,
                     int rescale, uint64_t* out) {
  size_t cw = 2 * (size_t)level * c->n;
  u32 lo = rescale ? level - 1 : level;
  size_t ow = 2 * (size_t)lo * c->n;
#pragma omp parallel for schedule(dynamic)
  for (u64 e = 0; e < count; ++e) {
    u64* sq = malloc(sizeof(u64) * 3 * level * c->n);
    u64* rl = malloc(sizeof(u64) * cw);
    oc_square(c, x + e * cw, level, sq);
    oc_relinearize(c, sq, level, rk, rl);
    if (rescale) oc_rescale(c, rl, 2, level, level - 1, out + e * ow);
    else memcpy(out + e * ow, rl, sizeof(u64) * cw);
    free(sq);
    free(rl);
  }
}
