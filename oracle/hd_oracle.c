/*
 * oracle/hd_oracle.c -- CPU ORACLE (TEST INFRASTRUCTURE ONLY; see hd_oracle.h).
 *
 * Plain C11, single-threaded, no blocking/fusion/reordering beyond what the
 * paper's algorithm or the operation's definition states.  Compile with
 * -ffp-contract=off (no FMA) so the floating-point encoder is the pinned
 * operation order of DESIGN.md R15.
 *
 * Parity pins for every function live in tests/test_oracle_*.py ("not gpu").
 */
#define _GNU_SOURCE
#include "hd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------------ */
/* Modular arithmetic: the plain definitions.                               */
/* ------------------------------------------------------------------------ */
static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)(((u128)a * b) % m); }
static uint64_t addmod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)(((u128)a + b) % m); }
static uint64_t submod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)(((u128)a + m - b) % m); }
static uint64_t powmod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = mulmod(r, b, m);
    b = mulmod(b, b, m);
    e >>= 1;
  }
  return r;
}
/* inverse by Fermat (m prime) */
static uint64_t invmod(uint64_t a, uint64_t m) { return powmod(a, m - 2, m); }
/* signed integer -> residue in [0, m) */
static uint64_t smod(int64_t x, uint64_t m) {
  if (x >= 0) return (uint64_t)x % m;
  uint64_t r = (uint64_t)(-(x + 1)) % m; /* -(x+1) >= 0, avoids INT64_MIN overflow */
  r = (r + 1) % m;                        /* |x| mod m */
  return r == 0 ? 0 : m - r;
}
/* centred representative of x in [0,q): (-q/2, q/2]  (R12) */
static int64_t centre(uint64_t x, uint64_t q) {
  if (x > q / 2) return -(int64_t)(q - x);
  return (int64_t)x;
}
static uint32_t bitrev(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; i++) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

/* ------------------------------------------------------------------------ */
/* Parameters (R5, R13).                                                    */
/* ------------------------------------------------------------------------ */
int or_is_prime(uint64_t x) {
  static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (x < 2) return 0;
  for (int i = 0; i < 12; i++) {
    if (x % bases[i] == 0) return x == bases[i];
  }
  uint64_t d = x - 1;
  int s = 0;
  while ((d & 1) == 0) { d >>= 1; s++; }
  for (int i = 0; i < 12; i++) {
    uint64_t y = powmod(bases[i], d, x);
    if (y == 1 || y == x - 1) continue;
    int composite = 1;
    for (int r = 1; r < s; r++) {
      y = mulmod(y, y, x);
      if (y == x - 1) { composite = 0; break; }
    }
    if (composite) return 0;
  }
  return 1;
}

/* Largest prime c < below with c = 1 (mod two_n); candidates 2n*k+1, k descending. */
static uint64_t prev_ntt_prime(uint64_t below, uint64_t two_n) {
  uint64_t k = (below - 2) / two_n;
  for (; k > 0; k--) {
    uint64_t c = two_n * k + 1;
    if (c < below && or_is_prime(c)) return c;
  }
  return 0;
}

/* Numerically smallest primitive 2n-th root of unity mod m (R13). */
static uint64_t min_root(uint64_t m, uint64_t n) {
  uint64_t y = 0;
  for (uint64_t x = 2; x < m; x++) {
    y = powmod(x, (m - 1) / (2 * n), m);
    if (powmod(y, n, m) == m - 1) break; /* order exactly 2n */
  }
  uint64_t y2 = mulmod(y, y, m), cur = y, best = y;
  for (uint64_t t = 1; t < n; t++) {
    cur = mulmod(cur, y2, m); /* y^(2t+1): every primitive 2n-th root */
    if (cur < best) best = cur;
  }
  return best;
}

int or_params_init(or_params *p, int32_t log_n, int32_t L, uint64_t seed) {
  return or_params_init_ex(p, log_n, L, 1, 1, seed);
}

int32_t or_num_digits(const or_params *p, int32_t ell) { return (ell + p->alpha - 1) / p->alpha; }

int or_params_init_ex(or_params *p, int32_t log_n, int32_t L, int32_t K_sp, int32_t alpha, uint64_t seed) {
  if (!p || log_n < 2 || log_n > 17 || L < 2 || K_sp < 1 || alpha < 1 || alpha > L || L + K_sp > OR_MAXMOD)
    return OR_E_PARAMS;
  memset(p, 0, sizeof(*p));
  p->K_sp = K_sp;
  p->alpha = alpha;
  p->log_n = log_n;
  p->n = 1 << log_n;
  p->num_slots = p->n / 2;
  p->L = L;
  p->q0_bits = 60;
  p->scale_bits = 45;
  p->special_bits = 60;
  p->seed = seed;
  uint64_t two_n = 2 * (uint64_t)p->n;
  p->mod[0] = prev_ntt_prime((uint64_t)1 << p->q0_bits, two_n);
  /* special primes: the next NTT primes below q0, descending (K = 1: P, R5) */
  for (int k = 0; k < K_sp; k++) p->mod[L + k] = prev_ntt_prime(k ? p->mod[L + k - 1] : p->mod[0], two_n);
  uint64_t below = (uint64_t)1 << p->scale_bits;
  for (int i = 1; i < L; i++) {
    p->mod[i] = prev_ntt_prime(below, two_n);
    below = p->mod[i];
  }
  for (int i = 0; i < L + K_sp; i++) {
    if (p->mod[i] == 0) return OR_E_PARAMS;
    p->psi[i] = min_root(p->mod[i], (uint64_t)p->n);
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* NTT (R13).  Definition: a^[i] = sum_j a_j psi^{(2 br(i)+1) j} mod m.      */
/* ------------------------------------------------------------------------ */
int or_ntt_definition(const or_params *p, int32_t l, const uint64_t *a, uint64_t *out) {
  if (l < 0 || l >= p->L + p->K_sp) return OR_E_ARG;
  uint64_t m = p->mod[l];
  int n = p->n;
  for (int i = 0; i < n; i++) {
    uint64_t w = powmod(p->psi[l], 2 * (uint64_t)bitrev((uint32_t)i, p->log_n) + 1, m);
    uint64_t acc = 0, pw = 1;
    for (int j = 0; j < n; j++) {
      acc = addmod(acc, mulmod(a[j], pw, m), m);
      pw = mulmod(pw, w, m);
    }
    out[i] = acc;
  }
  return OR_OK;
}

/* psi_rev[k] = psi^{br(k)} (or psi^{-br(k)}), k in [0, n) */
static uint64_t *psi_rev_table(const or_params *p, int32_t l, int inverse) {
  int n = p->n;
  uint64_t m = p->mod[l];
  uint64_t base = inverse ? invmod(p->psi[l], m) : p->psi[l];
  uint64_t *pw = malloc(sizeof(uint64_t) * n), *rev = malloc(sizeof(uint64_t) * n);
  pw[0] = 1;
  for (int k = 1; k < n; k++) pw[k] = mulmod(pw[k - 1], base, m);
  for (int k = 0; k < n; k++) rev[k] = pw[bitrev((uint32_t)k, p->log_n)];
  free(pw);
  return rev;
}

/* Cooley-Tukey, natural order in, bit-reversed evaluation order out. */
int or_ntt_forward(const or_params *p, int32_t l, uint64_t *a) {
  if (l < 0 || l >= p->L + p->K_sp) return OR_E_ARG;
  uint64_t m = p->mod[l];
  int n = p->n;
  uint64_t *S = psi_rev_table(p, l, 0);
  int t = n;
  for (int mm = 1; mm < n; mm <<= 1) {
    t >>= 1;
    for (int i = 0; i < mm; i++) {
      uint64_t w = S[mm + i];
      for (int j = 2 * i * t; j < 2 * i * t + t; j++) {
        uint64_t U = a[j], V = mulmod(a[j + t], w, m);
        a[j] = addmod(U, V, m);
        a[j + t] = submod(U, V, m);
      }
    }
  }
  free(S);
  return OR_OK;
}

/* Gentleman-Sande inverse of the above, then multiply by n^{-1}. */
int or_ntt_inverse(const or_params *p, int32_t l, uint64_t *a) {
  if (l < 0 || l >= p->L + p->K_sp) return OR_E_ARG;
  uint64_t m = p->mod[l];
  int n = p->n;
  uint64_t *S = psi_rev_table(p, l, 1);
  int t = 1;
  for (int mm = n / 2; mm >= 1; mm >>= 1) {
    for (int i = 0; i < mm; i++) {
      uint64_t w = S[mm + i];
      for (int j = 2 * i * t; j < 2 * i * t + t; j++) {
        uint64_t U = a[j], V = a[j + t];
        a[j] = addmod(U, V, m);
        a[j + t] = mulmod(submod(U, V, m), w, m);
      }
    }
    t <<= 1;
  }
  uint64_t ninv = invmod((uint64_t)n, m);
  for (int j = 0; j < n; j++) a[j] = mulmod(a[j], ninv, m);
  free(S);
  return OR_OK;
}

/* Schoolbook product in Z_m[X]/(X^n+1): the textbook definition. */
int or_negacyclic_schoolbook(const uint64_t *a, const uint64_t *b, int32_t n, uint64_t m,
                             uint64_t *out) {
  for (int k = 0; k < n; k++) out[k] = 0;
  for (int i = 0; i < n; i++)
    for (int j = 0; j < n; j++) {
      uint64_t prod = mulmod(a[i], b[j], m);
      int k = i + j;
      if (k < n) out[k] = addmod(out[k], prod, m);
      else out[k - n] = submod(out[k - n], prod, m); /* X^n = -1 */
    }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Randomness (R14): Philox4x32-10, counter (j, l, obj, tag<<16|sub).        */
/* ------------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; r++) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

enum { TAG_SECRET = 1, TAG_KEY_A = 2, TAG_KEY_E = 3, TAG_ENC_A = 4, TAG_ENC_E = 5,
       /* encrypted-database mode (NEXT-1, R26) */
       TAG_PK_A = 6, TAG_PK_E = 7, TAG_PKE_V = 8, TAG_PKE_E = 9, TAG_RLK_A = 10, TAG_RLK_E = 11 };

static void draw(uint64_t seed, uint32_t j, uint32_t l, uint32_t obj, uint32_t tag, uint32_t sub,
                 uint64_t *w0, uint64_t *w1) {
  uint32_t ctr[4] = {j, l, obj, (tag << 16) | sub};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t o[4];
  or_philox4x32_10(ctr, key, o);
  *w0 = (uint64_t)o[0] | ((uint64_t)o[1] << 32);
  *w1 = (uint64_t)o[2] | ((uint64_t)o[3] << 32);
}
static uint64_t draw_uniform(uint64_t seed, uint32_t j, uint32_t l, uint32_t obj, uint32_t tag,
                             uint32_t sub, uint64_t m) {
  uint64_t w0, w1;
  draw(seed, j, l, obj, tag, sub, &w0, &w1);
  return (uint64_t)((((u128)w0 << 64) | w1) % m);
}
static int64_t draw_cbd21(uint64_t seed, uint32_t j, uint32_t obj, uint32_t tag, uint32_t sub) {
  uint64_t w0, w1;
  draw(seed, j, 0, obj, tag, sub, &w0, &w1);
  return (int64_t)__builtin_popcountll(w0 & 0x1FFFFFull) -
         (int64_t)__builtin_popcountll((w0 >> 21) & 0x1FFFFFull);
}
static int64_t draw_ternary(uint64_t seed, uint32_t j, uint32_t obj, uint32_t tag) {
  uint64_t w0, w1;
  draw(seed, j, 0, obj, tag, 0, &w0, &w1);
  return (int64_t)(w0 % 3) - 1;
}

/* ------------------------------------------------------------------------ */
/* Galois automorphisms (R7).                                        */
/* ------------------------------------------------------------------------ */
uint64_t or_galois_elt(const or_params *p, int64_t step) {
  uint64_t two_n = 2 * (uint64_t)p->n;
  int64_t r = step % p->num_slots;
  if (r < 0) r += p->num_slots;
  return powmod(5, (uint64_t)r, two_n);
}

/* sigma_g on coefficients: X^j -> X^{jg mod 2n}, X^n = -1 (the definition). */
int or_automorph_coeff(const or_params *p, uint64_t g, const int64_t *a, int64_t *out) {
  int n = p->n;
  uint64_t two_n = 2 * (uint64_t)n;
  for (int j = 0; j < n; j++) {
    uint64_t idx = ((uint64_t)j * g) % two_n;
    if (idx < (uint64_t)n) out[idx] = a[j];
    else out[idx - n] = -a[j];
  }
  return OR_OK;
}

/* sigma_g in the NTT domain: out[i] = a[pi_g(i)],
 * pi_g(i) = br(((g (2 br(i)+1)) mod 2n - 1) / 2).  Pinned against
 * or_automorph_coeff by tests/test_oracle_ring.py. */
int or_automorph_ntt(const or_params *p, uint64_t g, const uint64_t *a, uint64_t *out) {
  int n = p->n;
  uint64_t two_n = 2 * (uint64_t)n;
  for (int i = 0; i < n; i++) {
    uint64_t e = (g * (2 * (uint64_t)bitrev((uint32_t)i, p->log_n) + 1)) % two_n;
    uint32_t src = bitrev((uint32_t)((e - 1) / 2), p->log_n);
    out[i] = a[src];
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* CKKS encoding (R15): pinned special inverse FFT.              */
/* xi^t = (cos(2 pi t / 2n), sin(2 pi t / 2n)); complex multiply without FMA. */
/* ------------------------------------------------------------------------ */
static void xi(const or_params *p, uint64_t t, double *re, double *im) {
  double ang = (2.0 * 3.141592653589793 * (double)t) / (double)(2 * (uint64_t)p->n);
  *re = cos(ang);
  *im = sin(ang);
}

static void bitrev_permute(double *re, double *im, int size) {
  int bits = 0;
  while ((1 << bits) < size) bits++;
  for (int i = 0; i < size; i++) {
    int r = (int)bitrev((uint32_t)i, bits);
    if (r > i) {
      double t = re[i]; re[i] = re[r]; re[r] = t;
      t = im[i]; im[i] = im[r]; im[r] = t;
    }
  }
}

/* Special inverse FFT (canonical-embedding inverse over slots zeta^{5^j}). */
static void fft_special_inv(const or_params *p, double *re, double *im) {
  int size = p->num_slots;
  uint64_t M = 2 * (uint64_t)p->n;
  for (int len = size; len >= 2; len >>= 1) {
    int lenh = len >> 1;
    uint64_t lenq = (uint64_t)len << 2;
    for (int i = 0; i < size; i += len) {
      for (int j = 0; j < lenh; j++) {
        uint64_t rot = powmod(5, (uint64_t)j, M);
        uint64_t idx = (lenq - (rot % lenq)) * (M / lenq);
        double wr, wi;
        xi(p, idx, &wr, &wi);
        double ur = re[i + j] + re[i + j + lenh], ui = im[i + j] + im[i + j + lenh];
        double vr = re[i + j] - re[i + j + lenh], vi = im[i + j] - im[i + j + lenh];
        double tr = vr * wr - vi * wi;
        double ti = vr * wi + vi * wr;
        re[i + j] = ur; im[i + j] = ui;
        re[i + j + lenh] = tr; im[i + j + lenh] = ti;
      }
    }
  }
  bitrev_permute(re, im, size);
  for (int i = 0; i < size; i++) {
    re[i] = re[i] / (double)size;
    im[i] = im[i] / (double)size;
  }
}

/* Special forward FFT (decode). */
static void fft_special(const or_params *p, double *re, double *im) {
  int size = p->num_slots;
  uint64_t M = 2 * (uint64_t)p->n;
  bitrev_permute(re, im, size);
  for (int len = 2; len <= size; len <<= 1) {
    int lenh = len >> 1;
    uint64_t lenq = (uint64_t)len << 2;
    for (int i = 0; i < size; i += len) {
      for (int j = 0; j < lenh; j++) {
        uint64_t rot = powmod(5, (uint64_t)j, M);
        uint64_t idx = (rot % lenq) * (M / lenq);
        double wr, wi;
        xi(p, idx, &wr, &wi);
        double ur = re[i + j], ui = im[i + j];
        double xr = re[i + j + lenh], xim = im[i + j + lenh];
        double vr = xr * wr - xim * wi;
        double vi = xr * wi + xim * wr;
        re[i + j] = ur + vr; im[i + j] = ui + vi;
        re[i + j + lenh] = ur - vr; im[i + j + lenh] = ui - vi;
      }
    }
  }
}

/* Integer coefficients coef_k = llrint(x_k * delta) (round-half-even). */
int or_encode_coeffs(const or_params *p, const double *z, double delta, int64_t *coef) {
  int ns = p->num_slots;
  double *re = malloc(sizeof(double) * ns), *im = malloc(sizeof(double) * ns);
  for (int i = 0; i < ns; i++) { re[i] = z[i]; im[i] = 0.0; }
  fft_special_inv(p, re, im);
  int rc = OR_OK;
  for (int i = 0; i < ns; i++) {
    double a = re[i] * delta, b = im[i] * delta;
    if (!(fabs(a) < 4611686018427387904.0) || !(fabs(b) < 4611686018427387904.0)) rc = OR_E_RANGE;
    coef[i] = llrint(a);
    coef[i + ns] = llrint(b);
  }
  free(re);
  free(im);
  return rc;
}

int or_encode(const or_params *p, const double *z, double delta, int32_t nlimbs, uint64_t *pt) {
  if (nlimbs < 1 || nlimbs > p->L) return OR_E_ARG;
  int n = p->n;
  int64_t *coef = malloc(sizeof(int64_t) * n);
  int rc = or_encode_coeffs(p, z, delta, coef);
  if (rc == OR_OK) {
    for (int l = 0; l < nlimbs; l++) {
      for (int j = 0; j < n; j++) pt[(size_t)l * n + j] = smod(coef[j], p->mod[l]);
      or_ntt_forward(p, l, pt + (size_t)l * n);
    }
  }
  free(coef);
  return rc;
}

/* Centred CRT of one coefficient over q_0..q_{nlimbs-1} (Garner), as double. */
static double crt_centred(const or_params *p, const uint64_t *x, int nlimbs) {
  /* mixed-radix digits v_i */
  uint64_t v[OR_MAXMOD];
  for (int i = 0; i < nlimbs; i++) {
    uint64_t qi = p->mod[i];
    uint64_t t = x[i] % qi;
    for (int k = 0; k < i; k++) t = mulmod(submod(t, v[k] % qi, qi), invmod(p->mod[k] % qi, qi), qi);
    v[i] = t;
  }
  /* X = sum v_i prod_{k<i} q_k and Q = prod q_k as little-endian 64-bit words */
  uint64_t X[OR_MAXMOD + 1] = {0}, Q[OR_MAXMOD + 1] = {0}, W[OR_MAXMOD + 1] = {0};
  int words = nlimbs + 1;
  W[0] = 1;
  for (int i = 0; i < nlimbs; i++) {
    u128 carry = 0; /* X += v_i * W */
    for (int w = 0; w < words; w++) {
      u128 s = (u128)v[i] * W[w] + X[w] + carry;
      X[w] = (uint64_t)s;
      carry = s >> 64;
    }
    carry = 0; /* W *= q_i */
    for (int w = 0; w < words; w++) {
      u128 s = (u128)W[w] * p->mod[i] + carry;
      W[w] = (uint64_t)s;
      carry = s >> 64;
    }
  }
  memcpy(Q, W, sizeof(Q));
  /* negative iff 2X > Q */
  uint64_t X2[OR_MAXMOD + 1];
  uint64_t c = 0;
  for (int w = 0; w < words; w++) {
    X2[w] = (X[w] << 1) | c;
    c = X[w] >> 63;
  }
  int gt = 0;
  for (int w = words - 1; w >= 0; w--) {
    if (X2[w] != Q[w]) { gt = X2[w] > Q[w]; break; }
  }
  uint64_t mag[OR_MAXMOD + 1];
  if (gt) { /* mag = Q - X */
    u128 borrow = 0;
    for (int w = 0; w < words; w++) {
      u128 d = (u128)Q[w] - X[w] - borrow;
      mag[w] = (uint64_t)d;
      borrow = (d >> 64) ? 1 : 0;
    }
  } else {
    memcpy(mag, X, sizeof(mag));
  }
  long double r = 0.0L;
  for (int w = words - 1; w >= 0; w--) r = r * 18446744073709551616.0L + (long double)mag[w];
  return gt ? -(double)r : (double)r;
}

int or_decode(const or_params *p, const uint64_t *pt, int32_t nlimbs, double delta, double *z) {
  if (nlimbs < 1 || nlimbs > p->L) return OR_E_ARG;
  int n = p->n, ns = p->num_slots;
  uint64_t *c = malloc(sizeof(uint64_t) * (size_t)n * nlimbs);
  memcpy(c, pt, sizeof(uint64_t) * (size_t)n * nlimbs);
  for (int l = 0; l < nlimbs; l++) or_ntt_inverse(p, l, c + (size_t)l * n);
  double *re = malloc(sizeof(double) * ns), *im = malloc(sizeof(double) * ns);
  uint64_t x[OR_MAXMOD];
  for (int k = 0; k < ns; k++) {
    for (int l = 0; l < nlimbs; l++) x[l] = c[(size_t)l * n + k];
    re[k] = crt_centred(p, x, nlimbs) / delta;
    for (int l = 0; l < nlimbs; l++) x[l] = c[(size_t)l * n + k + ns];
    im[k] = crt_centred(p, x, nlimbs) / delta;
  }
  fft_special(p, re, im);
  for (int k = 0; k < ns; k++) z[k] = re[k];
  free(c); free(re); free(im);
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Secret key, rotation keys, encryption.   */
/* ------------------------------------------------------------------------ */
int or_secret_key(const or_params *p, int64_t *s_coeff, uint64_t *s_ntt) {
  int n = p->n;
  for (int j = 0; j < n; j++) s_coeff[j] = draw_ternary(p->seed, (uint32_t)j, 0, TAG_SECRET);
  for (int l = 0; l < p->L + p->K_sp; l++) {
    uint64_t *row = s_ntt + (size_t)l * n;
    for (int j = 0; j < n; j++) row[j] = smod(s_coeff[j], p->mod[l]);
    or_ntt_forward(p, l, row);
  }
  return OR_OK;
}

/* P = prod_k p_k mod m */
static uint64_t P_mod(const or_params *p, uint64_t m) {
  uint64_t r = 1 % m;
  for (int k = 0; k < p->K_sp; k++) r = mulmod(r, p->mod[p->L + k] % m, m);
  return r;
}

/* Hybrid key-switching key (R11, R31) from s' to s (s' in NTT form over all L+K moduli):
 * b_d = -a_d s + e_d + [l in I_d] (P mod q_l) s' for digit d = limbs I_d = [d alpha,
 * (d+1) alpha) (alpha = K = 1: [l == d] (P mod q_d) s'); draws keyed by (obj, tag_a, tag_e),
 * a at modulus index l in [q_0..q_{L-1}, p_0..p_{K-1}] (R14), sub = digit. */
static void switch_key(const or_params *p, const uint64_t *s_ntt, const uint64_t *sp_ntt, uint32_t obj,
                       uint32_t tag_a, uint32_t tag_e, uint64_t *key) {
  int n = p->n, L = p->L, M = p->L + p->K_sp, beta = or_num_digits(p, L);
  uint64_t *e_ntt = malloc(sizeof(uint64_t) * n);
  for (int d = 0; d < beta; d++) {
    for (int l = 0; l < M; l++) {
      uint64_t m = p->mod[l];
      for (int j = 0; j < n; j++)
        e_ntt[j] = smod(draw_cbd21(p->seed, (uint32_t)j, obj, tag_e, (uint32_t)d), m);
      or_ntt_forward(p, l, e_ntt);
      uint64_t *kb = key + (((size_t)d * 2 + 0) * M + l) * n;
      uint64_t *ka = key + (((size_t)d * 2 + 1) * M + l) * n;
      uint64_t gad = (l < L && l / p->alpha == d) ? P_mod(p, m) : 0; /* (P mod q_l) on digit d's limbs */
      for (int j = 0; j < n; j++) {
        uint64_t a = draw_uniform(p->seed, (uint32_t)j, (uint32_t)l, obj, tag_a, (uint32_t)d, m);
        uint64_t b = submod(e_ntt[j], mulmod(a, s_ntt[(size_t)l * n + j], m), m);
        b = addmod(b, mulmod(gad, sp_ntt[(size_t)l * n + j], m), m);
        ka[j] = a;
        kb[j] = b;
      }
    }
  }
  free(e_ntt);
}

int or_rotation_key(const or_params *p, const uint64_t *s_ntt, int64_t step, uint64_t *key) {
  int n = p->n, L = p->L;
  if (step <= 0 || step >= p->num_slots) return OR_E_ARG;
  uint64_t g = or_galois_elt(p, step);
  /* s' = sigma_g(s) from the coefficient-domain definition */
  int64_t *s = malloc(sizeof(int64_t) * n), *sp = malloc(sizeof(int64_t) * n);
  uint64_t *sp_ntt = malloc(sizeof(uint64_t) * (size_t)(L + p->K_sp) * n);
  for (int j = 0; j < n; j++) s[j] = draw_ternary(p->seed, (uint32_t)j, 0, TAG_SECRET);
  or_automorph_coeff(p, g, s, sp);
  for (int l = 0; l < L + p->K_sp; l++) {
    uint64_t *row = sp_ntt + (size_t)l * n;
    for (int j = 0; j < n; j++) row[j] = smod(sp[j], p->mod[l]);
    or_ntt_forward(p, l, row);
  }
  switch_key(p, s_ntt, sp_ntt, (uint32_t)step, TAG_KEY_A, TAG_KEY_E, key);
  free(s); free(sp); free(sp_ntt);
  return OR_OK;
}

/* Relinearisation key (encrypted-database mode): switching key from s^2 to s;
 * s^2 in NTT form is the pointwise square of s_ntt (the negacyclic product). */
int or_relin_key(const or_params *p, const uint64_t *s_ntt, uint64_t *key) {
  int n = p->n, L = p->L;
  uint64_t *s2 = malloc(sizeof(uint64_t) * (size_t)(L + p->K_sp) * n);
  for (int l = 0; l < L + p->K_sp; l++)
    for (int j = 0; j < n; j++) {
      size_t o = (size_t)l * n + j;
      s2[o] = mulmod(s_ntt[o], s_ntt[o], p->mod[l]);
    }
  switch_key(p, s_ntt, s2, 0, TAG_RLK_A, TAG_RLK_E, key);
  free(s2);
  return OR_OK;
}

/* Public key (R26): pk = (b, a) over the L ciphertext moduli, b = -a s + e. */
int or_public_key(const or_params *p, const uint64_t *s_ntt, uint64_t *pk /* [2][L][n] */) {
  int n = p->n, L = p->L;
  uint64_t *e_ntt = malloc(sizeof(uint64_t) * n);
  for (int l = 0; l < L; l++) {
    uint64_t m = p->mod[l];
    for (int j = 0; j < n; j++) e_ntt[j] = smod(draw_cbd21(p->seed, (uint32_t)j, 0, TAG_PK_E, 0), m);
    or_ntt_forward(p, l, e_ntt);
    uint64_t *b = pk + (size_t)l * n, *a = pk + ((size_t)L + l) * n;
    for (int j = 0; j < n; j++) {
      a[j] = draw_uniform(p->seed, (uint32_t)j, (uint32_t)l, 0, TAG_PK_A, 0, m);
      b[j] = submod(e_ntt[j], mulmod(a[j], s_ntt[(size_t)l * n + j], m), m);
    }
  }
  free(e_ntt);
  return OR_OK;
}

/* Public-key encryption (R26): c = (v b + e0 + pt, v a + e1), v ternary, e0/e1 CBD(21),
 * drawn in the coefficient domain with Philox key enc_seed and object id obj. */
int or_encrypt_pk(const or_params *p, const uint64_t *pk, const uint64_t *pt, int32_t nlimbs, uint64_t enc_seed,
                  uint32_t obj, uint64_t *ct) {
  int n = p->n, L = p->L;
  if (nlimbs < 1 || nlimbs > L) return OR_E_ARG;
  uint64_t *v = malloc(sizeof(uint64_t) * n), *e0 = malloc(sizeof(uint64_t) * n), *e1 = malloc(sizeof(uint64_t) * n);
  for (int l = 0; l < nlimbs; l++) {
    uint64_t m = p->mod[l];
    for (int j = 0; j < n; j++) {
      v[j] = smod(draw_ternary(enc_seed, (uint32_t)j, obj, TAG_PKE_V), m);
      e0[j] = smod(draw_cbd21(enc_seed, (uint32_t)j, obj, TAG_PKE_E, 0), m);
      e1[j] = smod(draw_cbd21(enc_seed, (uint32_t)j, obj, TAG_PKE_E, 1), m);
    }
    or_ntt_forward(p, l, v);
    or_ntt_forward(p, l, e0);
    or_ntt_forward(p, l, e1);
    const uint64_t *b = pk + (size_t)l * n, *a = pk + ((size_t)L + l) * n;
    uint64_t *c0 = ct + (size_t)l * n, *c1 = ct + ((size_t)nlimbs + l) * n;
    for (int j = 0; j < n; j++) {
      c0[j] = addmod(addmod(mulmod(v[j], b[j], m), e0[j], m), pt[(size_t)l * n + j], m);
      c1[j] = addmod(mulmod(v[j], a[j], m), e1[j], m);
    }
  }
  free(v); free(e0); free(e1);
  return OR_OK;
}

/* Symmetric encryption c = (-a s + e + pt, a). */
int or_encrypt(const or_params *p, const uint64_t *s_ntt, const uint64_t *pt, int32_t nlimbs,
               uint64_t enc_seed, uint64_t *ct) {
  int n = p->n;
  if (nlimbs < 1 || nlimbs > p->L) return OR_E_ARG;
  uint64_t *e_ntt = malloc(sizeof(uint64_t) * n);
  for (int l = 0; l < nlimbs; l++) {
    uint64_t m = p->mod[l];
    for (int j = 0; j < n; j++) e_ntt[j] = smod(draw_cbd21(enc_seed, (uint32_t)j, 0, TAG_ENC_E, 0), m);
    or_ntt_forward(p, l, e_ntt);
    uint64_t *c0 = ct + (size_t)l * n, *c1 = ct + ((size_t)nlimbs + l) * n;
    for (int j = 0; j < n; j++) {
      uint64_t a = draw_uniform(enc_seed, (uint32_t)j, (uint32_t)l, 0, TAG_ENC_A, 0, m);
      uint64_t v = submod(e_ntt[j], mulmod(a, s_ntt[(size_t)l * n + j], m), m);
      c0[j] = addmod(v, pt[(size_t)l * n + j], m);
      c1[j] = a;
    }
  }
  free(e_ntt);
  return OR_OK;
}

int or_decrypt(const or_params *p, const uint64_t *s_ntt, const uint64_t *ct, int32_t nlimbs,
               uint64_t *pt) {
  int n = p->n;
  for (int l = 0; l < nlimbs; l++) {
    uint64_t m = p->mod[l];
    const uint64_t *c0 = ct + (size_t)l * n, *c1 = ct + ((size_t)nlimbs + l) * n;
    for (int j = 0; j < n; j++)
      pt[(size_t)l * n + j] = addmod(c0[j], mulmod(c1[j], s_ntt[(size_t)l * n + j], m), m);
  }
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Key switching (P:L479-496 hoisting; R11, R12, R31).                       */
/* ext modulus index e in [0, ell+K): e < ell -> q_e, e >= ell -> p_{e-ell}.  */
/* ------------------------------------------------------------------------ */
static int ext_mod_index(const or_params *p, int ell, int e) { return e < ell ? e : p->L + (e - ell); }

/* Fast basis conversion with centred digits (R12, R31): the residues x_i (coefficient
 * form) of one integer X modulo the basis B = {b_i}, i < cnt, map to
 *   sum_i y_i (B / b_i) mod m,   y_i = centred([x_i (B / b_i)^{-1}]_{b_i}),
 * an integer congruent to X mod B with |.| <= cnt B / 2.  For one modulus (cnt = 1) this is
 * the centred lift of x_0 (the alpha = K = 1 case of R12). */
static void basis_convert(const or_params *p, const uint64_t *const *x, const int *bidx, int cnt, int mi,
                          uint64_t *out) {
  int n = p->n;
  uint64_t m = p->mod[mi];
  for (int j = 0; j < n; j++) out[j] = 0;
  for (int i = 0; i < cnt; i++) {
    uint64_t b = p->mod[bidx[i]], hat_b = 1, hat_m = 1 % m; /* B / b_i mod b_i and mod m */
    for (int k = 0; k < cnt; k++) {
      if (k == i) continue;
      hat_b = mulmod(hat_b, p->mod[bidx[k]] % b, b);
      hat_m = mulmod(hat_m, p->mod[bidx[k]] % m, m);
    }
    uint64_t inv = invmod(hat_b, b);
    for (int j = 0; j < n; j++) {
      int64_t y = centre(mulmod(x[i][j], inv, b), b);
      out[j] = addmod(out[j], mulmod(smod(y, m), hat_m, m), m);
    }
  }
}

/* ModUp ("EvalFastRotationPrecompute"): digit d = limbs I_d = [d alpha,
 * min((d+1) alpha, ell)) of c1, INTT, fast-basis-converted (centred) into every modulus of
 * Q_ell u P, NTT.  Rows of the digit's own limbs equal c1 (the conversion is exact there).
 * dig: [beta(ell)][ell+K][n]. */
int or_modup(const or_params *p, const uint64_t *c1, int32_t ell, uint64_t *dig) {
  int n = p->n, ext = ell + p->K_sp, beta = or_num_digits(p, ell);
  if (ell < 1 || ell > p->L) return OR_E_ARG;
  uint64_t *x = malloc(sizeof(uint64_t) * (size_t)p->alpha * n);
  const uint64_t *xr[OR_MAXMOD];
  int bidx[OR_MAXMOD];
  for (int d = 0; d < beta; d++) {
    int lo = d * p->alpha, hi = lo + p->alpha < ell ? lo + p->alpha : ell, cnt = hi - lo;
    for (int i = 0; i < cnt; i++) {
      memcpy(x + (size_t)i * n, c1 + (size_t)(lo + i) * n, sizeof(uint64_t) * n);
      or_ntt_inverse(p, lo + i, x + (size_t)i * n);
      xr[i] = x + (size_t)i * n;
      bidx[i] = lo + i;
    }
    for (int e = 0; e < ext; e++) {
      uint64_t *row = dig + ((size_t)d * ext + e) * n;
      int mi = ext_mod_index(p, ell, e);
      if (e >= lo && e < hi) {
        memcpy(row, c1 + (size_t)e * n, sizeof(uint64_t) * n);
        continue;
      }
      basis_convert(p, xr, bidx, cnt, mi, row);
      or_ntt_forward(p, mi, row);
    }
  }
  free(x);
  return OR_OK;
}

/* ModDown: u'[q] = (u[q] - NTT_q(Conv_{P->q}(INTT_P(u[P])))) * P^{-1} mod q, the conversion
 * of the K special residues centred as in ModUp (K = 1: the centred lift of INTT_P(u[P])).
 * u: (ell+K) x n. */
static void moddown(const or_params *p, uint64_t *u, int ell, uint64_t *out) {
  int n = p->n, K = p->K_sp;
  uint64_t *y = malloc(sizeof(uint64_t) * (size_t)K * n), *t = malloc(sizeof(uint64_t) * n);
  const uint64_t *yr[OR_MAXMOD];
  int bidx[OR_MAXMOD];
  for (int k = 0; k < K; k++) {
    memcpy(y + (size_t)k * n, u + (size_t)(ell + k) * n, sizeof(uint64_t) * n);
    or_ntt_inverse(p, p->L + k, y + (size_t)k * n);
    yr[k] = y + (size_t)k * n;
    bidx[k] = p->L + k;
  }
  for (int l = 0; l < ell; l++) {
    uint64_t q = p->mod[l];
    basis_convert(p, yr, bidx, K, l, t);
    or_ntt_forward(p, l, t);
    uint64_t pinv = invmod(P_mod(p, q), q);
    for (int j = 0; j < n; j++) out[(size_t)l * n + j] = mulmod(submod(u[(size_t)l * n + j], t[j], q), pinv, q);
  }
  free(y); free(t);
}

int or_basis_convert(const or_params *p, const uint64_t *x, const int32_t *bidx, int32_t cnt, int32_t mi,
                     uint64_t *out) {
  const uint64_t *xr[OR_MAXMOD];
  int bi[OR_MAXMOD];
  if (cnt < 1 || cnt > OR_MAXMOD || mi < 0 || mi >= p->L + p->K_sp) return OR_E_ARG;
  for (int i = 0; i < cnt; i++) {
    if (bidx[i] < 0 || bidx[i] >= p->L + p->K_sp) return OR_E_ARG;
    xr[i] = x + (size_t)i * p->n;
    bi[i] = bidx[i];
  }
  basis_convert(p, xr, bi, cnt, mi, out);
  return OR_OK;
}

int or_moddown(const or_params *p, const uint64_t *u, int32_t ell, uint64_t *out) {
  if (ell < 1 || ell > p->L) return OR_E_ARG;
  size_t sz = sizeof(uint64_t) * (size_t)(ell + p->K_sp) * p->n;
  uint64_t *w = malloc(sz);
  memcpy(w, u, sz);
  moddown(p, w, ell, out);
  free(w);
  return OR_OK;
}

/* Key inner product in the extended basis: u[pp][e] += sum_d pi_g(dig_d)[e] * key[d][pp][e]
 * (u: 2 x (ell+K) x n, accumulated, so several rotations can share one ModDown). */
static void kip_accumulate(const or_params *p, const uint64_t *dig, int32_t ell, const uint64_t *key,
                           uint64_t g, uint64_t *u) {
  int n = p->n, M = p->L + p->K_sp, ext = ell + p->K_sp, beta = or_num_digits(p, ell);
  uint64_t *perm = malloc(sizeof(uint64_t) * n);
  for (int d = 0; d < beta; d++) {
    for (int e = 0; e < ext; e++) {
      int mi = ext_mod_index(p, ell, e);
      uint64_t m = p->mod[mi];
      or_automorph_ntt(p, g, dig + ((size_t)d * ext + e) * n, perm);
      for (int pp = 0; pp < 2; pp++) {
        const uint64_t *k = key + (((size_t)d * 2 + pp) * M + mi) * n;
        uint64_t *acc = u + ((size_t)pp * ext + e) * n;
        for (int j = 0; j < n; j++) acc[j] = addmod(acc[j], mulmod(perm[j], k[j], m), m);
      }
    }
  }
  free(perm);
}

/* "EvalFastRotation": permute digits by pi_g in the NTT domain, key inner
 * product over Q_ell u P, ModDown, add pi_g(c0). */
int or_rotate_hoisted(const or_params *p, const uint64_t *ct, const uint64_t *dig, int32_t ell,
                      const uint64_t *key, int64_t step, uint64_t *out) {
  int n = p->n, L = p->L, ext = ell + p->K_sp;
  if (ell < 1 || ell > L) return OR_E_ARG;
  uint64_t g = or_galois_elt(p, step);
  uint64_t *u = calloc((size_t)2 * ext * n, sizeof(uint64_t));
  uint64_t *perm = malloc(sizeof(uint64_t) * n);
  kip_accumulate(p, dig, ell, key, g, u);
  uint64_t *u0 = malloc(sizeof(uint64_t) * (size_t)ell * n), *u1 = malloc(sizeof(uint64_t) * (size_t)ell * n);
  moddown(p, u, ell, u0);
  moddown(p, u + (size_t)ext * n, ell, u1);
  for (int l = 0; l < ell; l++) {
    uint64_t q = p->mod[l];
    or_automorph_ntt(p, g, ct + (size_t)l * n, perm);
    for (int j = 0; j < n; j++) {
      out[(size_t)l * n + j] = addmod(perm[j], u0[(size_t)l * n + j], q);
      out[((size_t)ell + l) * n + j] = u1[(size_t)l * n + j];
    }
  }
  free(u); free(perm); free(u0); free(u1);
  return OR_OK;
}

static size_t dig_elems(const or_params *p, int ell) {
  return (size_t)or_num_digits(p, ell) * (ell + p->K_sp) * p->n;
}

int or_rotate(const or_params *p, const uint64_t *ct, int32_t ell, const uint64_t *key,
              int64_t step, uint64_t *out) {
  int n = p->n;
  uint64_t *dig = malloc(sizeof(uint64_t) * dig_elems(p, ell));
  int rc = or_modup(p, ct + (size_t)ell * n, ell, dig);
  if (rc == OR_OK) rc = or_rotate_hoisted(p, ct, dig, ell, key, step, out);
  free(dig);
  return rc;
}

/* Rescale: drop q_{ell-1} with the centred lift (R12). */
int or_rescale(const or_params *p, const uint64_t *ct, int32_t ell, uint64_t *out) {
  int n = p->n;
  if (ell < 2 || ell > p->L) return OR_E_ARG;
  uint64_t ql = p->mod[ell - 1];
  uint64_t *y = malloc(sizeof(uint64_t) * n), *t = malloc(sizeof(uint64_t) * n);
  for (int pp = 0; pp < 2; pp++) {
    memcpy(y, ct + ((size_t)pp * ell + ell - 1) * n, sizeof(uint64_t) * n);
    or_ntt_inverse(p, ell - 1, y);
    for (int l = 0; l < ell - 1; l++) {
      uint64_t q = p->mod[l];
      for (int j = 0; j < n; j++) t[j] = smod(centre(y[j], ql), q);
      or_ntt_forward(p, l, t);
      uint64_t inv = invmod(ql % q, q);
      const uint64_t *src = ct + ((size_t)pp * ell + l) * n;
      uint64_t *dst = out + ((size_t)pp * (ell - 1) + l) * n;
      for (int j = 0; j < n; j++) dst[j] = mulmod(submod(src[j], t[j], q), inv, q);
    }
  }
  free(y); free(t);
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Enrollment (Alg. enroller_bsgs) and the query.        */
/* ------------------------------------------------------------------------ */
/* Step 1: L2 normalisation, sequential double sum (R16). */
int or_normalize(const float *v, int32_t dim, double *u) {
  double s = 0.0;
  for (int i = 0; i < dim; i++) {
    double x = (double)v[i];
    s = s + x * x;
  }
  if (s == 0.0) return OR_E_ZERO_VECTOR;
  double nrm = sqrt(s);
  for (int i = 0; i < dim; i++) u[i] = (double)v[i] / nrm;
  return OR_OK;
}

static int layout_check(const or_params *p, int32_t dim, int32_t n1) {
  int ns = p->num_slots;
  if (dim < 2 || n1 < 1) return OR_E_ARG;
  if ((dim & (dim - 1)) != 0) return OR_E_LAYOUT; /* R19 */
  int N = dim < ns ? dim : ns;
  if (ns % (2 * N) != 0) return OR_E_LAYOUT;       /* M even (R19) */
  return OR_OK;
}

/* Query slots: numSlots/N replicated copies, period N over ALL slots (R8). */
int or_query_slots(const or_params *p, const float *q, int32_t dim, double *z) {
  int rc = layout_check(p, dim, 1);
  if (rc) return rc;
  double *u = malloc(sizeof(double) * dim);
  rc = or_normalize(q, dim, u);
  if (rc == OR_OK)
    for (int j = 0; j < p->num_slots; j++) z[j] = u[j % dim];
  free(u);
  return rc;
}

/* Step 1 for a slice of rows: U[r] = Normalize(vecs[r]). */
int or_normalize_rows(const float *vecs, int64_t rows, int32_t dim, double *U) {
  for (int64_t r = 0; r < rows; r++) {
    int rc = or_normalize(vecs + (size_t)r * dim, dim, U + (size_t)r * dim);
    if (rc) return rc;
  }
  return OR_OK;
}

/* Slot vector of aggregate `agg`, diagonal k: Steps 2-5 of Alg. enroller_bsgs,
 * literally (temporary M-block plaintext of the pair, then the stride-2N
 * A/B replication); aggregate = output ciphertext (R4).
 * U holds the Step-1-normalised rows [u_first, u_first + u_count) of the
 * database; a row the step needs outside that slice is an OR_E_ARG. */
int or_enroll_slots(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                    int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg, int32_t k,
                    double *z) {
  int rc = layout_check(p, dim, n1);
  if (rc) return rc;
  int ns = p->num_slots;
  /* Step 2 */
  int N = dim < ns ? dim : ns;
  int M = ns / N;
  /* Step 3 */
  int64_t G = (num_vectors + N - 1) / N;
  int64_t A = (2 * G + M - 1) / M;
  if (agg < 0 || agg >= A || k < 0 || k >= N) return OR_E_ARG;
  int64_t a = agg - (agg % 2); /* pair start: "for a = 0 to A-1 step 2" */
  int64_t g0 = a * (M / 2);
  int64_t g1 = g0 + M < G ? g0 + M : G;
  int64_t W = g1 - g0;
  /* giant-step index of diagonal k (floor, R3) */
  int k_signed = k < N / 2 ? k : k - N;
  int j = (int)floor((double)k_signed / (double)n1);
  int shiftN = ((n1 * j) % N + N) % N;
  double *tmp = calloc((size_t)ns, sizeof(double));
  for (int64_t b = 0; b < W; b++) {
    int64_t g = g0 + b, offset = b * N;
    for (int t = 0; t < N; t++) {
      int src = (t - shiftN + N) % N;
      /* Step 4: diagonal_g[k][src] = group_g[src][(src + k) mod N],
       * zero when row src of group g is beyond the database (|group_g| < N). */
      int64_t v = g * N + src;
      double val = 0.0;
      if (v < num_vectors) {
        if (v < u_first || v >= u_first + u_count) { free(tmp); return OR_E_ARG; }
        val = U[(size_t)(v - u_first) * dim + (src + k) % N];
      }
      tmp[offset + t] = val;
    }
  }
  /* replicate with stride 2N into plaintextA / plaintextB */
  for (int i = 0; i < ns; i++) z[i] = 0.0;
  for (int b = 0; b < M / 2; b++)
    for (int t = 0; t < N; t++) {
      if (agg == a) z[b * 2 * N + t] = tmp[b * N + t];
      else z[b * 2 * N + t] = tmp[b * N + t + ns / 2];
    }
  free(tmp);
  return OR_OK;
}

/* Diagonal plaintexts D[agg][k], k in [0, N): Encode at scale q_{L-1} over L
 * limbs (pt mode, R1; encoding R15).  Dagg = N x pt(L). */
int or_enroll_aggregate(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                        int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg,
                        uint64_t *Dagg) {
  int ns = p->num_slots;
  int N = dim < ns ? dim : ns;
  double *z = malloc(sizeof(double) * ns);
  int rc = OR_OK;
  for (int k = 0; k < N && rc == OR_OK; k++) {
    rc = or_enroll_slots(p, U, u_first, u_count, num_vectors, dim, n1, agg, k, z);
    if (rc == OR_OK)
      rc = or_encode(p, z, (double)p->mod[p->L - 1], p->L, Dagg + (size_t)k * p->L * p->n);
  }
  free(z);
  return rc;
}

/* Encrypted-database enrollment (NEXT-1, R26): the diagonal plaintexts of
 * or_enroll_aggregate, each encrypted under the public key with object id
 * agg * N + k (the enroller ships encrypted diagonals). */
int or_enroll_aggregate_encrypted(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                                  int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg,
                                  const uint64_t *pk, uint64_t enc_seed, uint64_t *Dct /* N x ct(L) */) {
  int ns = p->num_slots, L = p->L, n = p->n;
  int N = dim < ns ? dim : ns;
  uint64_t *Dagg = malloc(sizeof(uint64_t) * (size_t)N * L * n);
  int rc = or_enroll_aggregate(p, U, u_first, u_count, num_vectors, dim, n1, agg, Dagg);
  for (int k = 0; k < N && rc == OR_OK; k++)
    rc = or_encrypt_pk(p, pk, Dagg + (size_t)k * L * n, L, enc_seed, (uint32_t)(agg * N + k),
                       Dct + (size_t)k * 2 * L * n);
  free(Dagg);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* Flat pre-rotated layout (NEXT-2, R27: BSGS-RTX-TBE). */
/* ------------------------------------------------------------------------ */
/* Slot vector of pre-rotated diagonal k of aggregate agg in the flat HyDia packing
 * (Eq. equ:diag P:L332-336): M = numSlots/N groups per ciphertext, no gaps,
 *   diag_k[b N + t] = group_{agg M + b}[t][(t + k) mod N]   (0 beyond the database),
 * and the enroller's plaintext pre-rotation (Eq. eq:prerotation):
 *   diag'_k = Rot_{-j n1}(diag_k),  j = floor(k / n1),  i.e. diag'_k[s] = diag_k[s - j n1]. */
static int flat_slots(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                      int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg, int32_t k, int prerotate,
                      double *z);
int or_enroll_slots_flat(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                         int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg, int32_t k, double *z) {
  return flat_slots(p, U, u_first, u_count, num_vectors, dim, n1, agg, k, 1, z);
}
static int flat_slots(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                      int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg, int32_t k, int prerotate,
                      double *z) {
  int ns = p->num_slots;
  if (dim < 2 || n1 < 1 || (dim & (dim - 1)) != 0 || ns % dim != 0) return OR_E_LAYOUT;
  int N = dim, M = ns / N;
  int64_t G = (num_vectors + N - 1) / N, A = (G + M - 1) / M;
  if (agg < 0 || agg >= A || k < 0 || k >= N) return OR_E_ARG;
  double *diag = calloc((size_t)ns, sizeof(double));
  for (int b = 0; b < M; b++)
    for (int t = 0; t < N; t++) {
      int64_t v = (agg * M + b) * N + t;
      if (v >= num_vectors) continue;
      if (v < u_first || v >= u_first + u_count) { free(diag); return OR_E_ARG; }
      diag[b * N + t] = U[(size_t)(v - u_first) * dim + (t + k) % N];
    }
  int sh = prerotate ? (k / n1) * n1 : 0; /* Rot_{-j n1} */
  for (int s = 0; s < ns; s++) z[s] = diag[((s - sh) % ns + ns) % ns];
  free(diag);
  return OR_OK;
}

int or_enroll_aggregate_flat(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                             int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg, uint64_t *Dagg) {
  int ns = p->num_slots;
  double *z = malloc(sizeof(double) * ns);
  int rc = OR_OK;
  for (int k = 0; k < dim && rc == OR_OK; k++) {
    rc = or_enroll_slots_flat(p, U, u_first, u_count, num_vectors, dim, n1, agg, k, z);
    if (rc == OR_OK) rc = or_encode(p, z, (double)p->mod[p->L - 1], p->L, Dagg + (size_t)k * p->L * p->n);
  }
  free(z);
  return rc;
}

/* BSGS-RTX-TBS: the enroller encrypts the plain flat (HyDia) diagonals; the
 * server pre-rotates them homomorphically, diag'_k = Rot_{-j n1}(Dct_k) for j = floor(k/n1)
 * >= 1, with the negative giant-step keys numSlots - j n1 (or_prerotate_tbs). */
int or_enroll_aggregate_flat_tbs(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                                 int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg, const uint64_t *pk,
                                 uint64_t enc_seed, uint64_t *Dct) {
  int ns = p->num_slots, L = p->L, n = p->n;
  double *z = malloc(sizeof(double) * ns);
  uint64_t *pt = malloc(sizeof(uint64_t) * (size_t)L * n);
  int rc = OR_OK;
  for (int k = 0; k < dim && rc == OR_OK; k++) {
    rc = flat_slots(p, U, u_first, u_count, num_vectors, dim, n1, agg, k, 0, z);
    if (rc == OR_OK) rc = or_encode(p, z, (double)p->mod[L - 1], L, pt);
    if (rc == OR_OK)
      rc = or_encrypt_pk(p, pk, pt, L, enc_seed, (uint32_t)(agg * dim + k), Dct + (size_t)k * 2 * L * n);
  }
  free(z); free(pt);
  return rc;
}

static const uint64_t *find_key(const or_params *p, const int32_t *steps, int32_t nkeys,
                                const uint64_t *keys, int64_t step);
int or_prerotate_tbs(const or_params *p, uint64_t *Dct, int32_t dim, int32_t n1, const int32_t *steps,
                     int32_t nkeys, const uint64_t *keys) {
  int ns = p->num_slots, L = p->L, n = p->n;
  size_t ct = (size_t)2 * L * n;
  uint64_t *tmp = malloc(sizeof(uint64_t) * ct);
  int rc = OR_OK;
  for (int k = n1; k < dim && rc == OR_OK; k++) {
    int step = ns - (k / n1) * n1;
    const uint64_t *key = find_key(p, steps, nkeys, keys, step);
    if (!key) { rc = OR_E_MISSING_KEY; break; }
    rc = or_rotate(p, Dct + (size_t)k * ct, L, key, step, tmp);
    if (rc == OR_OK) memcpy(Dct + (size_t)k * ct, tmp, sizeof(uint64_t) * ct);
  }
  free(tmp);
  return rc;
}

/* BSGS-RTX-TBE as in the paper: the enroller pre-rotates each flat diagonal
 * plaintext and then encrypts it under the public key (object id agg N + k, R26). */
int or_enroll_aggregate_flat_encrypted(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                                       int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg,
                                       const uint64_t *pk, uint64_t enc_seed, uint64_t *Dct) {
  int L = p->L, n = p->n;
  uint64_t *Dagg = malloc(sizeof(uint64_t) * (size_t)dim * L * n);
  int rc = or_enroll_aggregate_flat(p, U, u_first, u_count, num_vectors, dim, n1, agg, Dagg);
  for (int k = 0; k < dim && rc == OR_OK; k++)
    rc = or_encrypt_pk(p, pk, Dagg + (size_t)k * L * n, L, enc_seed, (uint32_t)(agg * dim + k),
                       Dct + (size_t)k * 2 * L * n);
  free(Dagg);
  return rc;
}

/* Keys of the flat schedule: baby {1..n1-1}, giant {j n1 : 1 <= j < ceil(N/n1)}. */
int or_rotation_steps_flat(const or_params *p, int32_t N, int32_t n1, int32_t *steps, int32_t cap,
                           int32_t *count) {
  int ns = p->num_slots, c = 0;
  char *used = calloc((size_t)ns, 1);
  for (int i = 1; i < n1 && i < ns; i++) used[i] = 1;
  for (int j = 1; j * n1 < N; j++) used[(j * n1) % ns] = 1;
  for (int s = 1; s < ns; s++)
    if (used[s]) {
      if (c < cap) steps[c] = s;
      c++;
    }
  free(used);
  *count = c;
  return c <= cap ? OR_OK : OR_E_ARG;
}

/* Decrypt + decode a flat-layout output: score(v) = slot (floor(v/N) mod M) N + (v mod N)
 * of output floor(v / (M N)). */
int or_decrypt_scores_flat(const or_params *p, const uint64_t *s_ntt, const uint64_t *out_ct, int32_t N,
                           int64_t agg, int64_t num_vectors, double *scores /* M N */) {
  int n = p->n, ell = p->L - 1, ns = p->num_slots, M = ns / N;
  uint64_t *pt = malloc(sizeof(uint64_t) * (size_t)ell * n);
  double *z = malloc(sizeof(double) * ns);
  or_decrypt(p, s_ntt, out_ct, ell, pt);
  or_decode(p, pt, ell, ldexp(1.0, p->scale_bits), z);
  for (int b = 0; b < M; b++)
    for (int t = 0; t < N; t++) {
      int64_t v = (agg * M + b) * N + t;
      scores[(size_t)b * N + t] = v < num_vectors ? z[b * N + t] : 0.0;
    }
  free(pt); free(z);
  return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Scan (Alg. sender-bsgs).                                      */
/* ------------------------------------------------------------------------ */
static int floordiv(int a, int b) { return (int)floor((double)a / (double)b); }

/* giantSteps (R6): j in [floor(-(N/2)/n1), floor((N/2-1)/n1)]. */
int or_giant_range(int32_t N, int32_t n1, int32_t *j_min, int32_t *j_max) {
  *j_min = floordiv(-(N / 2), n1);
  *j_max = floordiv(N / 2 - 1, n1);
  return OR_OK;
}
/* preRot = ((n1 j) mod N + N) mod N */
int32_t or_pre_rot(int32_t N, int32_t n1, int32_t j) { return ((n1 * j) % N + N) % N; }

/* Rotation-key set of the fold schedule (R2): baby {1..n1-1}, giant {preRot(j) != 0},
 * fold {numSlots - N}; sorted ascending, unique. */
int or_rotation_steps(const or_params *p, int32_t N, int32_t n1, int32_t *steps, int32_t cap,
                      int32_t *count) {
  int ns = p->num_slots;
  char *used = calloc((size_t)ns, 1);
  for (int i = 1; i < n1; i++) used[i % ns] = 1;
  int jmin, jmax;
  or_giant_range(N, n1, &jmin, &jmax);
  for (int j = jmin; j <= jmax; j++) {
    int s = or_pre_rot(N, n1, j);
    if (s) used[s] = 1;
  }
  used[ns - N] = 1;
  int c = 0;
  for (int s = 1; s < ns; s++)
    if (used[s]) {
      if (c < cap) steps[c] = s;
      c++;
    }
  free(used);
  *count = c;
  return c <= cap ? OR_OK : OR_E_ARG;
}

static const uint64_t *find_key(const or_params *p, const int32_t *steps, int32_t nkeys,
                                const uint64_t *keys, int64_t step) {
  size_t ksz = (size_t)or_num_digits(p, p->L) * 2 * (p->L + p->K_sp) * p->n;
  for (int i = 0; i < nkeys; i++)
    if (steps[i] == step) return keys + ksz * i;
  return NULL;
}

/* Step 1: r[i] = Rot_i(ct) for i in [0, n1), hoisted. */
int or_baby_steps(const or_params *p, const uint64_t *q_ct, int32_t n1, const int32_t *steps,
                  int32_t nkeys, const uint64_t *keys, uint64_t *r) {
  int n = p->n, L = p->L;
  size_t ctsz = (size_t)2 * L * n;
  uint64_t *dig = malloc(sizeof(uint64_t) * dig_elems(p, L));
  or_modup(p, q_ct + (size_t)L * n, L, dig); /* preV */
  memcpy(r, q_ct, sizeof(uint64_t) * ctsz);  /* r[0] = ct */
  int rc = OR_OK;
  for (int i = 1; i < n1 && rc == OR_OK; i++) {
    const uint64_t *key = find_key(p, steps, nkeys, keys, i);
    if (!key) { rc = OR_E_MISSING_KEY; break; }
    rc = or_rotate_hoisted(p, q_ct, dig, L, key, i, r + ctsz * i);
  }
  free(dig);
  return rc;
}

/* Steps 2a-2b: S_j = sum_{i=i_lo}^{i_hi} r[i] (.) diagonal k(j,i). */
int or_giant_sum(const or_params *p, const uint64_t *r, int32_t n1, int32_t N,
                 const uint64_t *Dagg, int32_t j, uint64_t *S) {
  int n = p->n, L = p->L;
  size_t ctsz = (size_t)2 * L * n, ptsz = (size_t)L * n;
  int i_lo = 0 > -j * n1 - N / 2 ? 0 : -j * n1 - N / 2;
  int i_hi = n1 - 1 < N / 2 - 1 - j * n1 ? n1 - 1 : N / 2 - 1 - j * n1;
  memset(S, 0, sizeof(uint64_t) * ctsz);
  if (i_lo > i_hi) return OR_E_RANGE; /* skipped giant step */
  for (int i = i_lo; i <= i_hi; i++) {
    int k_signed = j * n1 + i;
    int k = ((k_signed % N) + N) % N;
    const uint64_t *diag = Dagg + ptsz * k;
    for (int pp = 0; pp < 2; pp++)
      for (int l = 0; l < L; l++) {
        uint64_t q = p->mod[l];
        const uint64_t *ri = r + ctsz * i + ((size_t)pp * L + l) * n;
        uint64_t *acc = S + ((size_t)pp * L + l) * n;
        const uint64_t *dl = diag + (size_t)l * n;
        for (int t = 0; t < n; t++) acc[t] = addmod(acc[t], mulmod(ri[t], dl[t], q), q);
      }
  }
  return OR_OK;
}

/* Encrypted diagonals (NEXT-1): S_j = sum_i EvalMultNoRelin(r[i], Dct_k),
 * the degree-2 tensor (r0 + r1 s)(D0 + D1 s) = d0 + d1 s + d2 s^2 accumulated as
 * d0 += r0 D0, d1 += r0 D1 + r1 D0, d2 += r1 D1.  S: [3][L][n]. */
static int giant_sum_ct_range(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dct,
                              int32_t j, int32_t i_lo, int32_t i_hi, uint64_t *S);
int or_giant_sum_ct(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dct,
                    int32_t j, uint64_t *S) {
  int i_lo = 0 > -j * n1 - N / 2 ? 0 : -j * n1 - N / 2;
  int i_hi = n1 - 1 < N / 2 - 1 - j * n1 ? n1 - 1 : N / 2 - 1 - j * n1;
  return giant_sum_ct_range(p, r, n1, N, Dct, j, i_lo, i_hi, S);
}
/* Flat layout (R27): diagonals j n1 + i, i < n1, below N. */
int or_giant_sum_ct_flat(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dct,
                         int32_t j, uint64_t *S) {
  if (j < 0 || j * n1 >= N) {
    memset(S, 0, sizeof(uint64_t) * 3 * p->L * p->n);
    return OR_E_RANGE;
  }
  int i_hi = n1 - 1 < N - 1 - j * n1 ? n1 - 1 : N - 1 - j * n1;
  return giant_sum_ct_range(p, r, n1, N, Dct, j, 0, i_hi, S);
}
static int giant_sum_ct_range(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dct,
                              int32_t j, int32_t i_lo, int32_t i_hi, uint64_t *S) {
  int n = p->n, L = p->L;
  size_t ctsz = (size_t)2 * L * n;
  memset(S, 0, sizeof(uint64_t) * 3 * L * n);
  if (i_lo > i_hi) return OR_E_RANGE;
  for (int i = i_lo; i <= i_hi; i++) {
    int k = (((j * n1 + i) % N) + N) % N;
    const uint64_t *D = Dct + ctsz * k, *ri = r + ctsz * i;
    for (int l = 0; l < L; l++) {
      uint64_t q = p->mod[l];
      const uint64_t *r0 = ri + (size_t)l * n, *r1 = ri + ((size_t)L + l) * n;
      const uint64_t *D0 = D + (size_t)l * n, *D1 = D + ((size_t)L + l) * n;
      uint64_t *d0 = S + (size_t)l * n, *d1 = S + ((size_t)L + l) * n, *d2 = S + ((size_t)2 * L + l) * n;
      for (int t = 0; t < n; t++) {
        d0[t] = addmod(d0[t], mulmod(r0[t], D0[t], q), q);
        d1[t] = addmod(d1[t], addmod(mulmod(r0[t], D1[t], q), mulmod(r1[t], D0[t], q), q), q);
        d2[t] = addmod(d2[t], mulmod(r1[t], D1[t], q), q);
      }
    }
  }
  return OR_OK;
}

/* Relinearize: (d0, d1, d2) -> (d0, d1) + KeySwitch_{s^2 -> s}(d2): ModUp of
 * d2, key inner product with the relinearisation key (no automorphism), ModDown. */
int or_relinearize(const or_params *p, const uint64_t *S3, int32_t ell, const uint64_t *rlk, uint64_t *out) {
  int n = p->n;
  if (ell < 1 || ell > p->L) return OR_E_ARG;
  size_t ext = (size_t)(ell + p->K_sp) * n;
  uint64_t *dig = malloc(sizeof(uint64_t) * dig_elems(p, ell));
  uint64_t *u = calloc(2 * ext, sizeof(uint64_t));
  uint64_t *u0 = malloc(sizeof(uint64_t) * (size_t)ell * n), *u1 = malloc(sizeof(uint64_t) * (size_t)ell * n);
  or_modup(p, S3 + (size_t)2 * ell * n, ell, dig);
  kip_accumulate(p, dig, ell, rlk, 1, u);
  moddown(p, u, ell, u0);
  moddown(p, u + ext, ell, u1);
  for (int l = 0; l < ell; l++) {
    uint64_t q = p->mod[l];
    for (int t = 0; t < n; t++) {
      size_t o = (size_t)l * n + t;
      out[o] = addmod(S3[o], u0[o], q);
      out[(size_t)ell * n + o] = addmod(S3[(size_t)ell * n + o], u1[o], q);
    }
  }
  free(dig); free(u); free(u0); free(u1);
  return OR_OK;
}

/* One aggregate: steps 2a-2f with the fold reading (R2):
 * y = sum_j Rot_{preRot(j)}(Rescale(S_j)); out = y + Rot_{numSlots-N}(y). */
int or_scan_aggregate(const or_params *p, const uint64_t *r, int32_t n1, int32_t N,
                      const uint64_t *Dagg, const int32_t *steps, int32_t nkeys,
                      const uint64_t *keys, uint64_t *out, uint64_t *y_out) {
  int n = p->n, L = p->L, ell = L - 1;
  size_t ctL = (size_t)2 * L * n, ct1 = (size_t)2 * ell * n;
  uint64_t *S = malloc(sizeof(uint64_t) * ctL), *Sp = malloc(sizeof(uint64_t) * ct1);
  uint64_t *T = malloc(sizeof(uint64_t) * ct1), *y = calloc(ct1, sizeof(uint64_t));
  int jmin, jmax, rc = OR_OK;
  or_giant_range(N, n1, &jmin, &jmax);
  for (int j = jmin; j <= jmax && rc == OR_OK; j++) {
    if (or_giant_sum(p, r, n1, N, Dagg, j, S) != OR_OK) continue; /* empty range */
    or_rescale(p, S, L, Sp);                                      /* Step 2c */
    int s = or_pre_rot(N, n1, j);                                 /* Step 2d */
    if (s != 0) {
      const uint64_t *key = find_key(p, steps, nkeys, keys, s);
      if (!key) { rc = OR_E_MISSING_KEY; break; }
      or_rotate(p, Sp, ell, key, s, T);
    } else {
      memcpy(T, Sp, sizeof(uint64_t) * ct1);
    }
    for (int pp = 0; pp < 2; pp++) /* Step 2e */
      for (int l = 0; l < ell; l++)
        for (int t = 0; t < n; t++) {
          size_t o = ((size_t)pp * ell + l) * n + t;
          y[o] = addmod(y[o], T[o], p->mod[l]);
        }
  }
  if (rc == OR_OK) {
    int fold = p->num_slots - N; /* Rot_{-N} (R2, App. A.4 of SURVEY) */
    const uint64_t *key = find_key(p, steps, nkeys, keys, fold);
    if (!key) rc = OR_E_MISSING_KEY;
    else {
      or_rotate(p, y, ell, key, fold, T);
      for (int pp = 0; pp < 2; pp++)
        for (int l = 0; l < ell; l++)
          for (int t = 0; t < n; t++) {
            size_t o = ((size_t)pp * ell + l) * n + t;
            out[o] = addmod(y[o], T[o], p->mod[l]);
          }
      if (y_out) memcpy(y_out, y, sizeof(uint64_t) * ct1);
    }
  }
  free(S); free(Sp); free(T); free(y);
  return rc;
}

/* One aggregate with the giant-step rotations accumulated in the extended basis
 * Q_ell u {P} and ONE ModDown per aggregate (R23; "double hoisting",
 * P:L498-506): with T_j = Rescale(S_j) and s_j = preRot(j),
 *   y_ext = sum_{s_j = 0} P T_j  +  sum_{s_j != 0} ( KIP_{s_j}(pi_{s_j}(ModUp(T_j.c1)))
 *                                                    + (P pi_{s_j}(T_j.c0), 0) ),
 *   y = ModDown(y_ext),  out = y + Rot_{numSlots-N}(y)          (fold as in R2).
 * Each term ModDown'ed alone is exactly the eager rotation (ModDown(P x + a) =
 * x + ModDown(a)), so the sum differs from or_scan_aggregate only by the rounding of
 * the single ModDown. */
static int scan_hoisted(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dagg,
                        const uint64_t *Dct, const uint64_t *rlk, int flat, const int32_t *steps, int32_t nkeys,
                        const uint64_t *keys, uint64_t *out, uint64_t *y_out);

int or_scan_aggregate_hoisted(const or_params *p, const uint64_t *r, int32_t n1, int32_t N,
                              const uint64_t *Dagg, const int32_t *steps, int32_t nkeys,
                              const uint64_t *keys, uint64_t *out, uint64_t *y_out) {
  return scan_hoisted(p, r, n1, N, Dagg, NULL, NULL, 0, steps, nkeys, keys, out, y_out);
}

/* Encrypted-database scan (NEXT-1): Alg. sender-bsgs as written, S_j = Relinearize(
 * sum_i EvalMultNoRelin(r[i], Dct_k)), then the schedule of
 * or_scan_aggregate_hoisted (rescale, giant rotations in Q u {P}, fold). */
int or_scan_aggregate_ct(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dct,
                         const uint64_t *rlk, const int32_t *steps, int32_t nkeys, const uint64_t *keys,
                         uint64_t *out, uint64_t *y_out) {
  return scan_hoisted(p, r, n1, N, NULL, Dct, rlk, 0, steps, nkeys, keys, out, y_out);
}

/* Flat pre-rotated layout (NEXT-2, R27): for j = 0 .. ceil(N/n1)-1,
 *   S_j = sum_{i < n1, j n1 + i < N} r[i] (.) diag'_{j n1 + i},
 * rescale, y = sum_j Rot_{j n1}(S'_j) accumulated in Q u {P} as in R23 (the giant
 * rotation re-aligns the baby component; Rot_{j n1} Rot_{-j n1} = id),
 * and out = y: no fold (no gaps). */
int or_scan_aggregate_flat(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dagg,
                           const int32_t *steps, int32_t nkeys, const uint64_t *keys, uint64_t *out) {
  return scan_hoisted(p, r, n1, N, Dagg, NULL, NULL, 1, steps, nkeys, keys, out, NULL);
}

/* Encrypted flat scan (BSGS-RTX-TBE with encrypted diagonals, the paper's GPU setting):
 * S_j = Relinearize(sum_i r[i] (x) Dct'_{j n1 + i}), then as or_scan_aggregate_flat. */
int or_scan_aggregate_flat_ct(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dct,
                              const uint64_t *rlk, const int32_t *steps, int32_t nkeys, const uint64_t *keys,
                              uint64_t *out) {
  return scan_hoisted(p, r, n1, N, NULL, Dct, rlk, 1, steps, nkeys, keys, out, NULL);
}

/* S_j of the flat layout (diagonals j n1 + i, i < n1, below N); OR_E_RANGE if empty. */
int or_giant_sum_flat(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dagg,
                      int32_t j, uint64_t *S) {
  int n = p->n, L = p->L;
  size_t ctsz = (size_t)2 * L * n, ptsz = (size_t)L * n;
  memset(S, 0, sizeof(uint64_t) * ctsz);
  if (j < 0 || j * n1 >= N) return OR_E_RANGE;
  for (int i = 0; i < n1 && j * n1 + i < N; i++) {
    const uint64_t *diag = Dagg + ptsz * (size_t)(j * n1 + i);
    for (int pp = 0; pp < 2; pp++)
      for (int l = 0; l < L; l++) {
        uint64_t q = p->mod[l];
        const uint64_t *ri = r + ctsz * i + ((size_t)pp * L + l) * n;
        uint64_t *acc = S + ((size_t)pp * L + l) * n;
        const uint64_t *dl = diag + (size_t)l * n;
        for (int t = 0; t < n; t++) acc[t] = addmod(acc[t], mulmod(ri[t], dl[t], q), q);
      }
  }
  return OR_OK;
}

static int scan_hoisted(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dagg,
                        const uint64_t *Dct, const uint64_t *rlk, int flat, const int32_t *steps, int32_t nkeys,
                        const uint64_t *keys, uint64_t *out, uint64_t *y_out) {
  int n = p->n, L = p->L, ell = L - 1;
  size_t ctL = (size_t)2 * L * n, ct1 = (size_t)2 * ell * n, ext = (size_t)(ell + p->K_sp) * n;
  uint64_t *S = malloc(sizeof(uint64_t) * ctL), *Sp = malloc(sizeof(uint64_t) * ct1);
  uint64_t *T = malloc(sizeof(uint64_t) * ct1), *y = malloc(sizeof(uint64_t) * ct1);
  uint64_t *yx = calloc(2 * ext, sizeof(uint64_t)); /* [pp][e][t], e >= ell: p_{e-ell} */
  uint64_t *dig = malloc(sizeof(uint64_t) * dig_elems(p, ell));
  uint64_t *perm = malloc(sizeof(uint64_t) * n);
  uint64_t *S3 = Dct ? malloc(sizeof(uint64_t) * (size_t)3 * L * n) : NULL;
  int jmin, jmax, rc = OR_OK;
  if (flat) {
    jmin = 0;
    jmax = (N + n1 - 1) / n1 - 1;
  } else {
    or_giant_range(N, n1, &jmin, &jmax);
  }
  for (int j = jmin; j <= jmax && rc == OR_OK; j++) {
    if (flat && Dct) {
      if (or_giant_sum_ct_flat(p, r, n1, N, Dct, j, S3) != OR_OK) continue;
      or_relinearize(p, S3, L, rlk, S);
    } else if (flat) {
      if (or_giant_sum_flat(p, r, n1, N, Dagg, j, S) != OR_OK) continue;
    } else if (Dct) {
      if (or_giant_sum_ct(p, r, n1, N, Dct, j, S3) != OR_OK) continue; /* empty range */
      or_relinearize(p, S3, L, rlk, S);                                  /* Step 2c */
    } else if (or_giant_sum(p, r, n1, N, Dagg, j, S) != OR_OK) {
      continue; /* empty range */
    }
    or_rescale(p, S, L, Sp);                                      /* Step 2c */
    int s = flat ? (j * n1) % p->num_slots : or_pre_rot(N, n1, j); /* Step 2d */
    if (s == 0) { /* y_ext += P T_j (P limbs += 0) */
      for (int pp = 0; pp < 2; pp++)
        for (int l = 0; l < ell; l++) {
          uint64_t q = p->mod[l];
          for (int t = 0; t < n; t++) {
            size_t o = (size_t)pp * ext + (size_t)l * n + t;
            yx[o] = addmod(yx[o], mulmod(P_mod(p, q), Sp[((size_t)pp * ell + l) * n + t], q), q);
          }
        }
      continue;
    }
    const uint64_t *key = find_key(p, steps, nkeys, keys, s);
    if (!key) { rc = OR_E_MISSING_KEY; break; }
    uint64_t g = or_galois_elt(p, s);
    or_modup(p, Sp + (size_t)ell * n, ell, dig);
    kip_accumulate(p, dig, ell, key, g, yx);
    for (int l = 0; l < ell; l++) { /* + (P pi_g(T_j.c0), 0) */
      uint64_t q = p->mod[l];
      or_automorph_ntt(p, g, Sp + (size_t)l * n, perm);
      for (int t = 0; t < n; t++) {
        size_t o = (size_t)l * n + t;
        yx[o] = addmod(yx[o], mulmod(P_mod(p, q), perm[t], q), q);
      }
    }
  }
  if (rc == OR_OK && flat) { /* no fold: out = y */
    moddown(p, yx, ell, out);
    moddown(p, yx + ext, ell, out + (size_t)ell * n);
  } else if (rc == OR_OK) {
    moddown(p, yx, ell, y);                      /* c0 */
    moddown(p, yx + ext, ell, y + (size_t)ell * n); /* c1 */
    int fold = p->num_slots - N;
    const uint64_t *key = find_key(p, steps, nkeys, keys, fold);
    if (!key) rc = OR_E_MISSING_KEY;
    else {
      or_rotate(p, y, ell, key, fold, T);
      for (int pp = 0; pp < 2; pp++)
        for (int l = 0; l < ell; l++)
          for (int t = 0; t < n; t++) {
            size_t o = ((size_t)pp * ell + l) * n + t;
            out[o] = addmod(y[o], T[o], p->mod[l]);
          }
      if (y_out) memcpy(y_out, y, sizeof(uint64_t) * ct1);
    }
  }
  free(S); free(Sp); free(T); free(y); free(yx); free(dig); free(perm); free(S3);
  return rc;
}

/* Decrypt + decode out_agg and read vector scores (R4):
 * score(v) = slot (floor(v/N) mod M/2) * 2N + (v mod N). */
int or_decrypt_scores(const or_params *p, const uint64_t *s_ntt, const uint64_t *out_ct,
                      int32_t N, int64_t agg, int64_t num_vectors, double *scores) {
  int n = p->n, ell = p->L - 1, ns = p->num_slots, M = ns / N;
  uint64_t *pt = malloc(sizeof(uint64_t) * (size_t)ell * n);
  double *z = malloc(sizeof(double) * ns);
  or_decrypt(p, s_ntt, out_ct, ell, pt);
  or_decode(p, pt, ell, ldexp(1.0, p->scale_bits), z);
  for (int b = 0; b < M / 2; b++)
    for (int t = 0; t < N; t++) {
      int64_t v = (agg * (M / 2) + b) * N + t;
      scores[(size_t)b * N + t] = v < num_vectors ? z[b * 2 * N + t] : 0.0;
    }
  free(pt); free(z);
  return OR_OK;
}

/* ======================================================================== */
/* Encrypted comparison and scenario tail (NEXT-3; reading R29 of DESIGN.md) */
/* ======================================================================== */
/* Degree of the Chebyshev series from the comparison depth budget kappa: the
 * paper's Paterson-Stockmeyer-aware lookup table: 7 -> 5, 8 -> 13,
 * 9 -> 27, 10 -> 59.  Other kappa: 0 (unsupported). */
int32_t or_cheb_degree(int32_t kappa) {
  switch (kappa) {
    case 7: return 5;
    case 8: return 13;
    case 9: return 27;
    case 10: return 59;
    default: return 0;
  }
}

/* PS split: d1, d2 minimising d1 + d2 subject to d1 * 2^(d2-1) >= n;
 * ties go to the smallest d2 (R29: n = 13 -> (2, 4) as the paper states). */
int or_ps_split(int32_t n, int32_t *d1, int32_t *d2) {
  if (n < 1) return OR_E_ARG;
  int best = 1 << 30, b1 = 0, b2 = 0;
  for (int g = 1; g <= 31; g++)
    for (int b = 1; b <= n; b++) {
      if ((long long)b << (g - 1) < n) continue;
      if (b + g < best || (b + g == best && g < b2)) { best = b + g; b1 = b; b2 = g; }
      break; /* larger b only grows b + g */
    }
  *d1 = b1; *d2 = b2;
  return OR_OK;
}

/* Chebyshev coefficients ("computed offline via DCT-based interpolation";
 * R29): the degree-n interpolant of f(x) = 1/2 (sign(x - delta) + 1) (Eq. eq:cheb-sign,
 * sign(0) = +1 so f = 1 for x >= delta) at the n + 1 Chebyshev nodes of the first kind
 * x_k = cos(pi (k + 1/2) / (n + 1)):
 *   c_i = 2/(n+1) sum_k f(x_k) cos(pi i (k + 1/2) / (n + 1)),   c_0 halved.
 * Interpolating f directly folds the 1/2 and the Alg.'s final "+1" into the series. */
int or_cheb_coeffs(double delta, int32_t n, double *c) {
  if (n < 1) return OR_E_ARG;
  const double pi = 3.14159265358979323846;
  for (int i = 0; i <= n; i++) {
    double s = 0.0;
    for (int k = 0; k <= n; k++) {
      double xk = cos(pi * ((double)k + 0.5) / (double)(n + 1));
      double fk = xk >= delta ? 1.0 : 0.0;
      s = s + fk * cos(pi * (double)i * ((double)k + 0.5) / (double)(n + 1));
    }
    c[i] = 2.0 * s / (double)(n + 1);
  }
  c[0] = c[0] / 2.0;
  return OR_OK;
}

/* Set when a product or a scalar multiplication is asked for at one limb (no level left). */
static int g_cheb_range_err;

/* A ciphertext in the comparison: [2][ell][n] residues plus its scale (R29). */
typedef struct {
  uint64_t *d;
  int ell;
  double scale;
} or_cct;

static or_cct cct_new(const or_params *p, int ell, double scale) {
  or_cct r;
  r.d = calloc((size_t)2 * ell * p->n, sizeof(uint64_t));
  r.ell = ell;
  r.scale = scale;
  return r;
}
static void cct_free(or_cct *a) { free(a->d); a->d = NULL; }

/* MatchLevel: keep limbs q_0..q_{ell-1} of both polynomials (exact
 * modular reduction; the scale is unchanged). */
static or_cct cct_drop(const or_params *p, const or_cct *a, int ell) {
  or_cct r = cct_new(p, ell, a->scale);
  int n = p->n;
  for (int pp = 0; pp < 2; pp++)
    memcpy(r.d + (size_t)pp * ell * n, a->d + (size_t)pp * a->ell * n, sizeof(uint64_t) * (size_t)ell * n);
  return r;
}

/* Relinearize + Rescale in one rounding (R29): X = P (d0, d1) + KIP(ModUp(d2), rlk) exactly over
 * Q_ell u {P}; out = (X - [X mod P q_{ell-1}]) / (P q_{ell-1}) over q_0..q_{ell-2}, with the
 * remainder from the CRT of X's P and q_{ell-1} residues in the coefficient domain, centred in
 * (-P q/2, P q/2] (R12).  Identical to Rescale(Relinearize(.)) bit for bit: with r = [X]_P and
 * s = [(X - r)/P]_q (the two centred lifts of the two-stage path), r + P s lies in
 * [-(Pq-1)/2, (Pq-1)/2], so it IS [X]_{Pq} (mixed radix).  Not used by the oracle's own
 * schedule; it pins the identity the CUDA path's fused relinearise-rescale relies on. */
int or_relin_rescale(const or_params *p, const uint64_t *S3, int32_t ell, const uint64_t *rlk, uint64_t *out) {
  int n = p->n, L = p->L;
  if (ell < 2 || ell > L) return OR_E_ARG;
  if (p->K_sp != 1 || p->alpha != 1) return OR_E_PARAMS; /* the two-modulus CRT identity needs one P */
  size_t ext = (size_t)(ell + 1) * n;
  uint64_t *dig = malloc(sizeof(uint64_t) * (size_t)ell * (ell + 1) * n);
  uint64_t *u = calloc(2 * ext, sizeof(uint64_t));
  or_modup(p, S3 + (size_t)2 * ell * n, ell, dig);
  kip_accumulate(p, dig, ell, rlk, 1, u);
  const uint64_t P = p->mod[L], qt = p->mod[ell - 1];
  const u128 PQ = (u128)P * qt;
  const uint64_t qinvP = invmod(qt % P, P);
  uint64_t *X = malloc(sizeof(uint64_t) * (size_t)ell * n), *xq = malloc(sizeof(uint64_t) * n),
           *xP = malloc(sizeof(uint64_t) * n), *V = malloc(sizeof(uint64_t) * (size_t)ell * n);
  for (int pp = 0; pp < 2; pp++) {
    const uint64_t *up = u + (size_t)pp * ext, *dp = S3 + (size_t)pp * ell * n;
    for (int l = 0; l < ell; l++) {
      uint64_t q = p->mod[l], Pq = P % q;
      for (int j = 0; j < n; j++)
        X[(size_t)l * n + j] = addmod(up[(size_t)l * n + j], mulmod(Pq, dp[(size_t)l * n + j], q), q);
    }
    memcpy(xq, X + (size_t)(ell - 1) * n, sizeof(uint64_t) * n);
    or_ntt_inverse(p, ell - 1, xq);
    memcpy(xP, up + (size_t)ell * n, sizeof(uint64_t) * n);
    or_ntt_inverse(p, L, xP);
    for (int j = 0; j < n; j++) {
      uint64_t k = mulmod(submod(xP[j], xq[j] % P, P), qinvP, P);
      u128 v = (u128)xq[j] + (u128)qt * k; /* [X mod P q] in [0, P q) */
      int neg = v > PQ / 2;
      u128 mag = neg ? PQ - v : v;
      for (int l = 0; l < ell - 1; l++) {
        uint64_t q = p->mod[l], r = (uint64_t)(mag % q);
        V[(size_t)l * n + j] = neg ? (q - r) % q : r;
      }
    }
    for (int l = 0; l < ell - 1; l++) {
      uint64_t q = p->mod[l];
      uint64_t w = invmod((uint64_t)(PQ % q), q);
      or_ntt_forward(p, l, V + (size_t)l * n);
      for (int j = 0; j < n; j++)
        out[((size_t)pp * (ell - 1) + l) * n + j] = mulmod(submod(X[(size_t)l * n + j], V[(size_t)l * n + j], q), w, q);
    }
  }
  free(dig); free(u); free(X); free(xq); free(xP); free(V);
  return OR_OK;
}

/* Ciphertext product: MatchLevel, tensor (d0, d1, d2) = (a0 b0, a0 b1 + a1 b0, a1 b1),
 * Relinearize, Rescale (invariant (i) of P:L792-793: every product is
 * rescaled at once).  scale = s_a s_b / q_{ell-1}. */
static or_cct cct_mul(const or_params *p, const or_cct *a0, const or_cct *b0, const uint64_t *rlk) {
  int ell = a0->ell < b0->ell ? a0->ell : b0->ell, n = p->n;
  if (ell < 2) { g_cheb_range_err = 1; return cct_new(p, 1, a0->scale); }
  or_cct a = cct_drop(p, a0, ell), b = cct_drop(p, b0, ell);
  uint64_t *S3 = malloc(sizeof(uint64_t) * (size_t)3 * ell * n);
  uint64_t *R = malloc(sizeof(uint64_t) * (size_t)2 * ell * n);
  for (int l = 0; l < ell; l++) {
    uint64_t q = p->mod[l];
    for (int t = 0; t < n; t++) {
      size_t o = (size_t)l * n + t, o1 = (size_t)ell * n + o;
      S3[o] = mulmod(a.d[o], b.d[o], q);
      S3[o1] = addmod(mulmod(a.d[o], b.d[o1], q), mulmod(a.d[o1], b.d[o], q), q);
      S3[(size_t)2 * ell * n + o] = mulmod(a.d[o1], b.d[o1], q);
    }
  }
  or_relinearize(p, S3, ell, rlk, R);
  or_cct r = cct_new(p, ell - 1, a.scale * b.scale / (double)p->mod[ell - 1]);
  or_rescale(p, R, ell, r.d);
  free(S3); free(R); cct_free(&a); cct_free(&b);
  return r;
}

/* k * a for a small integer k (exact; scale unchanged). */
static or_cct cct_mul_int(const or_params *p, const or_cct *a, int64_t k) {
  or_cct r = cct_new(p, a->ell, a->scale);
  int n = p->n;
  for (int pp = 0; pp < 2; pp++)
    for (int l = 0; l < a->ell; l++) {
      uint64_t q = p->mod[l], kq = smod(k, q);
      for (int t = 0; t < n; t++) {
        size_t o = ((size_t)pp * a->ell + l) * n + t;
        r.d[o] = mulmod(a->d[o], kq, q);
      }
    }
  return r;
}

/* a + c for a real constant c: the constant polynomial round(c * scale) (R15
 * rounding, half-even) is constant in every NTT slot; added to c0. */
static or_cct cct_add_const(const or_params *p, const or_cct *a, double c) {
  or_cct r = cct_new(p, a->ell, a->scale);
  int n = p->n;
  int64_t v = llrint(c * a->scale);
  memcpy(r.d, a->d, sizeof(uint64_t) * (size_t)2 * a->ell * n);
  for (int l = 0; l < a->ell; l++) {
    uint64_t q = p->mod[l], vq = smod(v, q);
    for (int t = 0; t < n; t++) r.d[(size_t)l * n + t] = addmod(r.d[(size_t)l * n + t], vq, q);
  }
  return r;
}

/* c * a for a real constant c: multiply by C = round(c * q_{ell-1}) and rescale by
 * q_{ell-1}; the message becomes m C / q_{ell-1} ~ c m, the scale is kept (R29). */
static or_cct cct_mul_const(const or_params *p, const or_cct *a, double c) {
  int ell = a->ell, n = p->n;
  if (ell < 2) { g_cheb_range_err = 1; return cct_new(p, 1, a->scale); }
  int64_t C = llrint(c * (double)p->mod[ell - 1]);
  uint64_t *X = malloc(sizeof(uint64_t) * (size_t)2 * ell * n);
  for (int pp = 0; pp < 2; pp++)
    for (int l = 0; l < ell; l++) {
      uint64_t q = p->mod[l], Cq = smod(C, q);
      for (int t = 0; t < n; t++) {
        size_t o = ((size_t)pp * ell + l) * n + t;
        X[o] = mulmod(a->d[o], Cq, q);
      }
    }
  or_cct r = cct_new(p, ell - 1, a->scale);
  or_rescale(p, X, ell, r.d);
  free(X);
  return r;
}

/* a + sgn * b after MatchLevel; the result keeps a's scale (R29). */
static or_cct cct_add(const or_params *p, const or_cct *a0, const or_cct *b0, int sgn) {
  int ell = a0->ell < b0->ell ? a0->ell : b0->ell, n = p->n;
  or_cct a = cct_drop(p, a0, ell), b = cct_drop(p, b0, ell);
  for (int pp = 0; pp < 2; pp++)
    for (int l = 0; l < ell; l++) {
      uint64_t q = p->mod[l];
      for (int t = 0; t < n; t++) {
        size_t o = ((size_t)pp * ell + l) * n + t;
        a.d[o] = sgn > 0 ? addmod(a.d[o], b.d[o], q) : submod(a.d[o], b.d[o], q);
      }
    }
  cct_free(&b);
  return a;
}

/* An intermediate value of the evaluation: a ciphertext, or a plain constant. */
typedef struct {
  int is_ct;
  or_cct ct;
  double k;
} or_val;

typedef struct {
  const or_params *p;
  const uint64_t *rlk;
  int d1, d2;
  or_cct T[64];     /* baby powers T[1..d1] (Step 1) */
  or_cct G[32];     /* giant powers G[j] = T_{d1 2^j} (Step 2) */
  int nG;
} or_ps;

/* 2 a b - c, every product rescaled. */
static or_cct cct_two_ab_minus(const or_params *p, const or_cct *a, const or_cct *b, const or_cct *c_ct,
                               double c_const, const uint64_t *rlk) {
  or_cct ab = cct_mul(p, a, b, rlk);
  or_cct t2 = cct_mul_int(p, &ab, 2);
  cct_free(&ab);
  or_cct r;
  if (c_ct) r = cct_add(p, &t2, c_ct, -1);
  else r = cct_add_const(p, &t2, -c_const);
  cct_free(&t2);
  return r;
}

static or_val val_const(double k) { or_val v; memset(&v, 0, sizeof v); v.k = k; return v; }
static or_val val_ct(or_cct c) { or_val v; memset(&v, 0, sizeof v); v.is_ct = 1; v.ct = c; return v; }

/* MatchLevel ahead of use (R29): a copy of a at min(a.ell, ell) limbs. */
static or_cct cct_at(const or_params *p, const or_cct *a, int ell) {
  return cct_drop(p, a, a->ell < ell ? a->ell : ell);
}

/* Chunk polynomial (Alg. gpu-chebyshev Step 3): Q = c_0 + sum_{i>=1, c_i != 0}
 * c_i T[i], deg < d1, produced at `need` limbs (each T[i] dropped to need + 1 first). */
static or_val ps_chunk(or_ps *S, const double *c, int m, int need) {
  or_val acc = val_const(0.0);
  for (int i = 1; i <= m; i++) {
    if (c[i] == 0.0) continue;
    or_cct Ti = cct_at(S->p, &S->T[i], need + 1);
    or_cct t = cct_mul_const(S->p, &Ti, c[i]);
    cct_free(&Ti);
    if (!acc.is_ct) {
      acc = val_ct(t);
    } else {
      or_cct s = cct_add(S->p, &acc.ct, &t, 1);
      cct_free(&acc.ct); cct_free(&t);
      acc.ct = s;
    }
  }
  if (!acc.is_ct) return val_const(c[0]);
  if (c[0] != 0.0) {
    or_cct s = cct_add_const(S->p, &acc.ct, c[0]);
    cct_free(&acc.ct);
    acc.ct = s;
  }
  return acc;
}

/* Evaluates sum_{i<=m} c_i T_i by Chebyshev-basis division (R29): with k = d1 2^j the
 * largest giant degree <= m, p = q T_k + r where q_0 = c_k, q_i = 2 c_{k+i} and
 * r_{k-i} = c_{k-i} - c_{k+i} (T_k T_i = (T_{k+i} + T_{k-i}) / 2; m < 2k).
 * Levels top-down (R29): the result is wanted at `need` limbs, so the product q T_k is taken
 * at need + 1 limbs (q evaluated for need + 1, T_k dropped to it) and r is evaluated for need. */
static or_val ps_eval(or_ps *S, const double *c0, int m, int need) {
  while (m > 0 && c0[m] == 0.0) m--;
  if (m < S->d1) return ps_chunk(S, c0, m, need);
  int j = 0;
  while (j + 1 < S->nG && (S->d1 << (j + 1)) <= m) j++;
  int k = S->d1 << j;
  double *q = malloc(sizeof(double) * (size_t)(m - k + 1)), *r = malloc(sizeof(double) * (size_t)k);
  q[0] = c0[k];
  for (int i = 1; i <= m - k; i++) q[i] = 2.0 * c0[k + i];
  for (int i = 0; i < k; i++) r[i] = c0[i];
  for (int i = 1; i <= m - k; i++) r[k - i] = r[k - i] - c0[k + i];
  or_val Q = ps_eval(S, q, m - k, need + 1), R = ps_eval(S, r, k - 1, need);
  free(q); free(r);
  or_val P;
  or_cct Gj = cct_at(S->p, &S->G[j], need + 1);
  if (Q.is_ct) {
    P = val_ct(cct_mul(S->p, &Q.ct, &Gj, S->rlk));
    cct_free(&Q.ct);
  } else if (Q.k != 0.0) {
    P = val_ct(cct_mul_const(S->p, &Gj, Q.k));
  } else {
    P = val_const(0.0);
  }
  cct_free(&Gj);
  if (!P.is_ct) return R;
  if (R.is_ct) {
    or_cct s = cct_add(S->p, &P.ct, &R.ct, 1);
    cct_free(&P.ct); cct_free(&R.ct);
    P.ct = s;
  } else if (R.k != 0.0) {
    or_cct s = cct_add_const(S->p, &P.ct, R.k);
    cct_free(&P.ct);
    P.ct = s;
  }
  return P;
}

/* ChebyshevCompare (Alg. gpu-chebyshev; R29).  in: [2][ell][n] at scale
 * `scale` (slots in [-1, 1]); c[0..degree]; rlk: relinearisation key.  out: [2][*ell_out][n]
 * (capacity 2 ell n), *scale_out its scale.  OR_E_RANGE if the levels run out. */
int or_cheb_compare(const or_params *p, const uint64_t *in, int32_t ell, double scale, const double *c,
                    int32_t degree, const uint64_t *rlk, uint64_t *out, int32_t *ell_out, double *scale_out) {
  return or_cheb_compare_at(p, in, ell, scale, c, degree, rlk, 1, out, ell_out, scale_out);
}

/* As or_cheb_compare with the result wanted at `need` limbs (R29): a membership sum over many
 * slots needs the headroom of q_0 q_1 (the sum of 2^20 values near 1 at scale 2^45 exceeds
 * q_0 / 2). */
int or_cheb_compare_at(const or_params *p, const uint64_t *in, int32_t ell, double scale, const double *c,
                       int32_t degree, const uint64_t *rlk, int32_t need, uint64_t *out, int32_t *ell_out,
                       double *scale_out) {
  if (need < 1 || need >= ell) return OR_E_ARG;
  if (ell < 1 || ell > p->L || degree < 1) return OR_E_ARG;
  or_ps S;
  memset(&S, 0, sizeof S);
  S.p = p;
  S.rlk = rlk;
  g_cheb_range_err = 0;
  or_ps_split(degree, &S.d1, &S.d2);
  if (S.d1 >= 64) return OR_E_ARG;
  /* Step 1: baby powers */
  S.T[1] = cct_new(p, ell, scale);
  memcpy(S.T[1].d, in, sizeof(uint64_t) * (size_t)2 * ell * p->n);
  for (int i = 2; i <= S.d1; i++) {
    if ((i & (i - 1)) == 0)
      S.T[i] = cct_two_ab_minus(p, &S.T[i / 2], &S.T[i / 2], NULL, 1.0, rlk);
    else
      S.T[i] = cct_two_ab_minus(p, &S.T[i / 2], &S.T[(i + 1) / 2], &S.T[1], 0.0, rlk);
  }
  /* Step 2: giant powers T_{d1 2^j} by doubling, up to the degree */
  S.G[0] = cct_drop(p, &S.T[S.d1], S.T[S.d1].ell);
  S.nG = 1;
  while ((S.d1 << S.nG) <= degree) {
    S.G[S.nG] = cct_two_ab_minus(p, &S.G[S.nG - 1], &S.G[S.nG - 1], NULL, 1.0, rlk);
    S.nG++;
  }
  /* Step 3: chunks and combination */
  int rc = OR_OK;
  or_val V = ps_eval(&S, c, degree, need); /* the result at `need` limbs (1: q_0 only) */
  if (!V.is_ct) {
    rc = OR_E_ARG; /* constant polynomial: nothing encrypted to return */
  } else if (g_cheb_range_err || V.ct.ell < need) { /* no level left, or below the requested one */
    rc = OR_E_RANGE;
    cct_free(&V.ct);
  } else {
    *ell_out = V.ct.ell;
    *scale_out = V.ct.scale;
    memcpy(out, V.ct.d, sizeof(uint64_t) * (size_t)2 * V.ct.ell * p->n);
    cct_free(&V.ct);
  }
  for (int i = 1; i <= S.d1; i++) cct_free(&S.T[i]);
  for (int j = 0; j < S.nG; j++) cct_free(&S.G[j]);
  return rc;
}

/* Membership tail (Alg. membership, Alg. gpu-bsgs-membership):
 * EvalAddMany of the count comparison ciphertexts ([count][2][ell][n]), then
 * RotateAndSum over numSlots: x <- x + Rot_k(x) for k = 1, 2, 4, ..., numSlots/2
 * (power-of-two keys).  Every slot of out = the sum over all slots. */
int or_membership(const or_params *p, const uint64_t *cts, int32_t count, int32_t ell, const int32_t *steps,
                  int32_t nkeys, const uint64_t *keys, uint64_t *out) {
  int n = p->n;
  size_t ct = (size_t)2 * ell * n;
  if (count < 1 || ell < 1) return OR_E_ARG;
  memcpy(out, cts, sizeof(uint64_t) * ct);
  for (int i = 1; i < count; i++)
    for (int pp = 0; pp < 2; pp++)
      for (int l = 0; l < ell; l++)
        for (int t = 0; t < n; t++) {
          size_t o = ((size_t)pp * ell + l) * n + t;
          out[o] = addmod(out[o], cts[(size_t)i * ct + o], p->mod[l]);
        }
  uint64_t *R = malloc(sizeof(uint64_t) * ct);
  int rc = OR_OK;
  for (int k = 1; k < p->num_slots; k <<= 1) {
    const uint64_t *key = find_key(p, steps, nkeys, keys, k);
    if (!key) { rc = OR_E_MISSING_KEY; break; }
    or_rotate(p, out, ell, key, k, R);
    for (int pp = 0; pp < 2; pp++)
      for (int l = 0; l < ell; l++)
        for (int t = 0; t < n; t++) {
          size_t o = ((size_t)pp * ell + l) * n + t;
          out[o] = addmod(out[o], R[o], p->mod[l]);
        }
  }
  free(R);
  return rc;
}

/* Online database aggregation (Alg. online-aggr Step 2): diag_i summed over the
 * A aggregates, residue by residue.  D: A x N diagonals of dpoly polynomials of L limbs
 * ([a][k][poly][limb][n]); out: N x dpoly x L x n. */
int or_aggregate_diagonals(const or_params *p, const uint64_t *D, int32_t A, int32_t N, int32_t dpoly, uint64_t *out) {
  int n = p->n, L = p->L;
  if (A < 1 || N < 1 || dpoly < 1) return OR_E_ARG;
  size_t per = (size_t)N * dpoly * L * n;
  for (size_t e = 0; e < per; e++) {
    uint64_t q = p->mod[(e / (size_t)n) % (size_t)L], acc = 0;
    for (int a = 0; a < A; a++) acc = addmod(acc, D[(size_t)a * per + e], q);
    out[e] = acc;
  }
  return OR_OK;
}
