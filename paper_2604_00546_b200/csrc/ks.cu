// ks.cu -- hybrid RNS key switching (alpha = 1, one special prime P) and rescale.
//
// Rotation by r (R11): ModUp of c1 (digit d = centred
// INTT of limb d lifted into every other modulus of Q_ell u {P}, then NTT);
// key inner product with the NTT-domain Galois permutation pi_g fused into the
// digit loads; ModDown (centred INTT of the P limb, lift, NTT, (u - .) P^{-1});
// + pi_g(c0).  Rescale drops q_{ell-1} the same way (R12).
//
// Every lift is fused into the load of the forward NTT that follows it, and every
// combine into that NTT's final store (ntt_run): a ModUp is 2 INTT kernels + 2 NTT
// kernels, a ModDown 2 + 2, a rescale 2 + 2, plus the key inner product.
#include "common.cuh"
#include "ks.cuh"

#include <vector>

namespace {
constexpr int TPB = 256;

// Key inner product; x = b * K + k.  Output u[x][p][e][t], e <= ell (e == ell: P).
// Digit d in extended modulus e: e == d -> c1[b][d] itself (NTT form), else the
// lifted digit dig[b][d][slot], slot = e < d ? e : e - 1.  Two coefficients per thread.
// Extended-basis accumulation (R23): with acc.c0 set, u[x][p][e] += sum + (p == 0 &&
// e < ell ? P pi_g(c0_b)[e] : 0), i.e. the rotation before its ModDown, added onto u.
struct KipAcc {
  const uint64_t *c0 = nullptr;  // c0 of ciphertext b at c0 + b * c0_stride ([ell][n])
  size_t c0_stride = 0;
  uint64_t pw[HD_MAXMOD] = {}, pws[HD_MAXMOD] = {};  // P mod q_e and its Shoup companion
};
__global__ void __launch_bounds__(TPB) kip_kernel(const uint64_t *__restrict__ dig, const uint64_t *__restrict__ c1,
                                                  size_t c1_stride, uint64_t *__restrict__ u, int ell, int K, int L,
                                                  int logn, const uint64_t *const *__restrict__ kptr,
                                                  const uint32_t *__restrict__ gal, ModTab mt, KipAcc ka,
                                                  FDiv f_ell1, FDiv f_K) {
  const int n = 1 << logn;
  const uint32_t t = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const uint32_t xe = blockIdx.y;
  const uint32_t x = fdiv_q(xe, f_ell1), e = xe - x * (ell + 1);
  const uint32_t b = fdiv_q(x, f_K), k = x - b * K;
  if (t >= (uint32_t)n) return;
  const int gm = (int)e < ell ? (int)e : L;
  const uint32_t g = gal[k];
  const uint32_t s0 = galois_src(t, g, logn), s1 = galois_src(t + 1, g, logn);
  const uint64_t *key = kptr[k];
  const uint64_t *dg = dig + (size_t)b * ell * ell * n;
  const uint64_t *cb = c1 + (size_t)b * c1_stride;
  uint64_t a0l = 0, a0h = 0, a1l = 0, a1h = 0, b0l = 0, b0h = 0, b1l = 0, b1h = 0;
  // digits in groups of KIP_DG: every load of a group (the Galois-gathered digit words and
  // the key words) is issued before its products (the kernel is load-latency bound)
  constexpr int KIP_DG = 4;
  for (int d0 = 0; d0 < ell; d0 += KIP_DG) {
    uint64_t v0[KIP_DG], v1[KIP_DG];
    ulonglong2 k0[KIP_DG], k1[KIP_DG];
#pragma unroll
    for (int i = 0; i < KIP_DG; i++) {
      const int d = d0 + i;
      if (d < ell) {
        const uint64_t *row = ((int)e == d) ? cb + (size_t)d * n
                                            : dg + ((size_t)d * ell + ((int)e < d ? (int)e : (int)e - 1)) * n;
        v0[i] = row[s0];
        v1[i] = row[s1];
        k0[i] = *reinterpret_cast<const ulonglong2 *>(key + ((size_t)(d * 2 + 0) * (L + 1) + gm) * n + t);
        k1[i] = *reinterpret_cast<const ulonglong2 *>(key + ((size_t)(d * 2 + 1) * (L + 1) + gm) * n + t);
      }
    }
#pragma unroll
    for (int i = 0; i < KIP_DG; i++) {
      if (d0 + i < ell) {
        mac128(a0l, a0h, v0[i], k0[i].x);
        mac128(b0l, b0h, v1[i], k0[i].y);
        mac128(a1l, a1h, v0[i], k1[i].x);
        mac128(b1l, b1h, v1[i], k1[i].y);
      }
    }
  }
  const uint64_t q = mt.q[gm], bar = mt.bar[gm], r64 = mt.r64[gm], r64s = mt.r64s[gm];
  ulonglong2 *o0 = reinterpret_cast<ulonglong2 *>(u + ((size_t)(x * 2 + 0) * (ell + 1) + e) * n + t);
  ulonglong2 *o1 = reinterpret_cast<ulonglong2 *>(u + ((size_t)(x * 2 + 1) * (ell + 1) + e) * n + t);
  ulonglong2 v0 = make_ulonglong2(reduce128(a0h, a0l, q, bar, r64, r64s), reduce128(b0h, b0l, q, bar, r64, r64s));
  ulonglong2 v1 = make_ulonglong2(reduce128(a1h, a1l, q, bar, r64, r64s), reduce128(b1h, b1l, q, bar, r64, r64s));
  if (ka.c0) {
    const ulonglong2 p0 = *o0, p1 = *o1;
    v0 = make_ulonglong2(addmod(v0.x, p0.x, q), addmod(v0.y, p0.y, q));
    v1 = make_ulonglong2(addmod(v1.x, p1.x, q), addmod(v1.y, p1.y, q));
    if ((int)e < ell) {
      const uint64_t *c0r = ka.c0 + (size_t)b * ka.c0_stride + (size_t)e * n;
      v0.x = addmod(v0.x, shoup(c0r[s0], ka.pw[e], ka.pws[e], q), q);
      v0.y = addmod(v0.y, shoup(c0r[s1], ka.pw[e], ka.pws[e], q), q);
    }
  }
  *o0 = v0;
  *o1 = v1;
}

// kip_kernel with ell known at compile time and one coefficient per thread: the ell Galois
// gathers and 2 ell key words of a thread are all loaded before the first product (the
// two-coefficient kernel above holds 78 registers, 3 CTAs per SM, and waits on its gathers).
template <int ELL>
__global__ void __launch_bounds__(TPB) kip1_kernel(const uint64_t *__restrict__ dig, const uint64_t *__restrict__ c1,
                                                   size_t c1_stride, uint64_t *__restrict__ u, int K, int L, int logn,
                                                   const uint64_t *const *__restrict__ kptr,
                                                   const uint32_t *__restrict__ gal, ModTab mt, KipAcc ka, FDiv f_K) {
  const int n = 1 << logn;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t x = blockIdx.y / (ELL + 1), e = blockIdx.y % (ELL + 1);
  const uint32_t b = fdiv_q(x, f_K), k = x - b * K;
  if (t >= (uint32_t)n) return;
  const int gm = (int)e < ELL ? (int)e : L;
  const uint32_t s = galois_src(t, gal[k], logn);
  const uint64_t *key = kptr[k];
  const uint64_t *dg = dig + (size_t)b * ELL * ELL * n;
  const uint64_t *cb = c1 + (size_t)b * c1_stride;
  uint64_t v[ELL], k0[ELL], k1[ELL];
#pragma unroll
  for (int d = 0; d < ELL; d++) {
    const uint64_t *row = ((int)e == d) ? cb + (size_t)d * n
                                        : dg + ((size_t)d * ELL + ((int)e < d ? (int)e : (int)e - 1)) * n;
    v[d] = row[s];
    k0[d] = __ldg(key + ((size_t)(d * 2 + 0) * (L + 1) + gm) * n + t);
    k1[d] = __ldg(key + ((size_t)(d * 2 + 1) * (L + 1) + gm) * n + t);
  }
  uint64_t a0l = 0, a0h = 0, a1l = 0, a1h = 0;
#pragma unroll
  for (int d = 0; d < ELL; d++) {
    mac128(a0l, a0h, v[d], k0[d]);
    mac128(a1l, a1h, v[d], k1[d]);
  }
  const uint64_t q = mt.q[gm], bar = mt.bar[gm], r64 = mt.r64[gm], r64s = mt.r64s[gm];
  uint64_t o0 = reduce128(a0h, a0l, q, bar, r64, r64s), o1 = reduce128(a1h, a1l, q, bar, r64, r64s);
  uint64_t *p0 = u + ((size_t)(x * 2 + 0) * (ELL + 1) + e) * n + t;
  uint64_t *p1 = u + ((size_t)(x * 2 + 1) * (ELL + 1) + e) * n + t;
  if (ka.c0) {
    o0 = addmod(o0, *p0, q);
    o1 = addmod(o1, *p1, q);
    if ((int)e < ELL)
      o0 = addmod(o0, shoup(ka.c0[(size_t)b * ka.c0_stride + (size_t)e * n + s], ka.pw[e], ka.pws[e], q), q);
  }
  *p0 = o0;
  *p1 = o1;
}

// The whole hoisted giant-step sum of R23 in one pass (alpha = K = 1): for every aggregate b,
//   u[b][p][e] = sum_j ( KIP(pi_j(dig_j[b]))[p][e] + [p == 0, e < ell] P pi_j(c0_j[b])[e] )
//              + [e < ell] P T0[b][p][e]
// over the J rotated giant steps j (digits dig_j, sums ct_j at ct_j + b ct_stride, key slot j)
// and the unrotated one T0 (optional).  Written once, instead of J read-modify-write passes
// over u plus one add_pscaled pass.  Two coefficients per thread; 128-bit accumulation of
// the J ell products per output (< 2^128 for J ell < 2^8).
constexpr int GIANT_MAXJ = 8;
struct GiantSet {
  int J = 0;
  const uint64_t *dig[GIANT_MAXJ] = {};  // [B][ell][ell][n] (alpha = 1 slot layout)
  const uint64_t *ct[GIANT_MAXJ] = {};   // S'_j of aggregate b at ct[j] + b ct_stride ([2][ell][n])
  int slot[GIANT_MAXJ] = {};             // key / Galois slot in kptr / gal
  const uint64_t *t0 = nullptr;          // unrotated giant-step sum (or null)
  size_t ct_stride = 0;
};
__global__ void __launch_bounds__(TPB) kip_giant_kernel(uint64_t *__restrict__ u, int ell, int L, int logn,
                                                        const uint64_t *const *__restrict__ kptr,
                                                        const uint32_t *__restrict__ gal, ModTab mt, KipAcc ka,
                                                        GiantSet gs, FDiv f_ell1) {
  const int n = 1 << logn;
  const uint32_t t = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const uint32_t be = blockIdx.y;
  const uint32_t b = fdiv_q(be, f_ell1), e = be - b * (ell + 1);
  if (t >= (uint32_t)n) return;
  const int gm = (int)e < ell ? (int)e : L;
  const uint64_t q = mt.q[gm], bar = mt.bar[gm], r64 = mt.r64[gm], r64s = mt.r64s[gm];
  uint64_t a0l = 0, a0h = 0, a1l = 0, a1h = 0, b0l = 0, b0h = 0, b1l = 0, b1h = 0;
  uint64_t c00 = 0, c01 = 0;  // sum_j pi_j(c0_j)[e] (mod q), p = 0 only
  for (int jj = 0; jj < gs.J; jj++) {
    const uint32_t g = gal[gs.slot[jj]];
    const uint32_t s0 = galois_src(t, g, logn), s1 = galois_src(t + 1, g, logn);
    const uint64_t *key = kptr[gs.slot[jj]];
    const uint64_t *dg = gs.dig[jj] + (size_t)b * ell * ell * n;
    const uint64_t *cb = gs.ct[jj] + (size_t)b * gs.ct_stride;  // c0 rows [0, ell), c1 rows [ell, 2 ell)
    for (int d = 0; d < ell; d++) {
      const uint64_t *row = ((int)e == d) ? cb + (size_t)(ell + d) * n
                                          : dg + ((size_t)d * ell + ((int)e < d ? (int)e : (int)e - 1)) * n;
      const uint64_t v0 = row[s0], v1 = row[s1];
      const ulonglong2 k0 = *reinterpret_cast<const ulonglong2 *>(key + ((size_t)(d * 2 + 0) * (L + 1) + gm) * n + t);
      const ulonglong2 k1 = *reinterpret_cast<const ulonglong2 *>(key + ((size_t)(d * 2 + 1) * (L + 1) + gm) * n + t);
      mac128(a0l, a0h, v0, k0.x);
      mac128(b0l, b0h, v1, k0.y);
      mac128(a1l, a1h, v0, k1.x);
      mac128(b1l, b1h, v1, k1.y);
    }
    if ((int)e < ell) {
      const uint64_t *c0r = cb + (size_t)e * n;
      c00 = addmod(c00, c0r[s0], q);
      c01 = addmod(c01, c0r[s1], q);
    }
  }
  ulonglong2 v0 = make_ulonglong2(reduce128(a0h, a0l, q, bar, r64, r64s), reduce128(b0h, b0l, q, bar, r64, r64s));
  ulonglong2 v1 = make_ulonglong2(reduce128(a1h, a1l, q, bar, r64, r64s), reduce128(b1h, b1l, q, bar, r64, r64s));
  if ((int)e < ell) {
    const uint64_t pw = ka.pw[e], pws = ka.pws[e];
    if (gs.t0) {  // + P T0 (both polys)
      const ulonglong2 x0 = *reinterpret_cast<const ulonglong2 *>(gs.t0 + (size_t)b * gs.ct_stride + (size_t)e * n + t);
      const ulonglong2 x1 =
          *reinterpret_cast<const ulonglong2 *>(gs.t0 + (size_t)b * gs.ct_stride + (size_t)(ell + e) * n + t);
      c00 = addmod(c00, x0.x, q);
      c01 = addmod(c01, x0.y, q);
      v1.x = addmod(v1.x, shoup(x1.x, pw, pws, q), q);
      v1.y = addmod(v1.y, shoup(x1.y, pw, pws, q), q);
    }
    v0.x = addmod(v0.x, shoup(c00, pw, pws, q), q);
    v0.y = addmod(v0.y, shoup(c01, pw, pws, q), q);
  }
  *reinterpret_cast<ulonglong2 *>(u + ((size_t)(b * 2 + 0) * (ell + 1) + e) * n + t) = v0;
  *reinterpret_cast<ulonglong2 *>(u + ((size_t)(b * 2 + 1) * (ell + 1) + e) * n + t) = v1;
}

// The same sum with (J, ell) known at compile time and one coefficient per thread: every
// Galois-gathered digit word and key word of the J rotations is loaded before the first
// product (the gathers are scattered; the generic kernel above waits on each in turn at two
// CTAs per SM and ran at 2.3 TB/s, long_scoreboard 4.5 stalls per issue).
template <int J, int ELL>
__global__ void __launch_bounds__(TPB) kip_giant1_kernel(uint64_t *__restrict__ u, int L, int logn,
                                                         const uint64_t *const *__restrict__ kptr,
                                                         const uint32_t *__restrict__ gal, ModTab mt, KipAcc ka,
                                                         GiantSet gs) {
  const int n = 1 << logn;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t b = blockIdx.y / (ELL + 1), e = blockIdx.y % (ELL + 1);
  if (t >= (uint32_t)n) return;
  const int gm = (int)e < ELL ? (int)e : L;
  const uint64_t q = mt.q[gm], bar = mt.bar[gm], r64 = mt.r64[gm], r64s = mt.r64s[gm];
  uint64_t v[J][ELL], k0[J][ELL], k1[J][ELL], cz[J];
#pragma unroll
  for (int jj = 0; jj < J; jj++) {
    const uint32_t s = galois_src(t, gal[gs.slot[jj]], logn);
    const uint64_t *key = kptr[gs.slot[jj]];
    const uint64_t *dg = gs.dig[jj] + (size_t)b * ELL * ELL * n;
    const uint64_t *cb = gs.ct[jj] + (size_t)b * gs.ct_stride;  // c0 rows [0, ell), c1 rows [ell, 2 ell)
#pragma unroll
    for (int d = 0; d < ELL; d++) {
      const uint64_t *row = ((int)e == d) ? cb + (size_t)(ELL + d) * n
                                          : dg + ((size_t)d * ELL + ((int)e < d ? (int)e : (int)e - 1)) * n;
      v[jj][d] = row[s];
      k0[jj][d] = __ldg(key + ((size_t)(d * 2 + 0) * (L + 1) + gm) * n + t);
      k1[jj][d] = __ldg(key + ((size_t)(d * 2 + 1) * (L + 1) + gm) * n + t);
    }
    cz[jj] = (int)e < ELL ? cb[(size_t)e * n + s] : 0;
  }
  uint64_t a0l = 0, a0h = 0, a1l = 0, a1h = 0, c0 = 0;
#pragma unroll
  for (int jj = 0; jj < J; jj++) {
#pragma unroll
    for (int d = 0; d < ELL; d++) {
      mac128(a0l, a0h, v[jj][d], k0[jj][d]);
      mac128(a1l, a1h, v[jj][d], k1[jj][d]);
    }
    c0 = addmod(c0, cz[jj], q);
  }
  uint64_t o0 = reduce128(a0h, a0l, q, bar, r64, r64s), o1 = reduce128(a1h, a1l, q, bar, r64, r64s);
  if ((int)e < ELL) {
    const uint64_t pw = ka.pw[e], pws = ka.pws[e];
    if (gs.t0) {  // + P T0 (both polys)
      c0 = addmod(c0, gs.t0[(size_t)b * gs.ct_stride + (size_t)e * n + t], q);
      o1 = addmod(o1, shoup(gs.t0[(size_t)b * gs.ct_stride + (size_t)(ELL + e) * n + t], pw, pws, q), q);
    }
    o0 = addmod(o0, shoup(c0, pw, pws, q), q);
  }
  u[((size_t)(b * 2 + 0) * (ELL + 1) + e) * n + t] = o0;
  u[((size_t)(b * 2 + 1) * (ELL + 1) + e) * n + t] = o1;
}

// dst[b][p][e] += P src[b][p][e] for e < ell (the P limb of P src is 0): a giant step
// without rotation, in the extended basis (R23).  dst rows [b][p][ell+1][n], src [b][p][ell][n].
__global__ void add_pscaled_kernel(uint64_t *__restrict__ dst, size_t dst_stride, const uint64_t *__restrict__ src,
                                   size_t src_stride, int ell, int ext, int n, ModTab mt, KipAcc ka) {
  const uint32_t t = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const uint32_t bpl = blockIdx.y;
  const uint32_t l = bpl % ell, bp = bpl / ell, b = bp / 2, p = bp % 2;
  if (t >= (uint32_t)n) return;
  const uint64_t q = mt.q[l];
  ulonglong2 *o = reinterpret_cast<ulonglong2 *>(dst + (size_t)b * dst_stride + ((size_t)p * ext + l) * n + t);
  const ulonglong2 sv =
      *reinterpret_cast<const ulonglong2 *>(src + (size_t)b * src_stride + ((size_t)p * ell + l) * n + t);
  const ulonglong2 dv = *o;
  *o = make_ulonglong2(addmod(dv.x, shoup(sv.x, ka.pw[l], ka.pws[l], q), q),
                       addmod(dv.y, shoup(sv.y, ka.pw[l], ka.pws[l], q), q));
}

// Fused relinearise-rescale (R29): from the coefficient forms of X's q_last and P rows
// (x = u[b][p][ell-1], xP = u[b][p][ell]) the centred remainder v = [X mod P q_last] by CRT,
// v = x + q_last ((xP - x) q_last^{-1} mod P) in [0, P q_last), centred; V[b][p][l] = v mod q_l.
__global__ void crt2_kernel(const uint64_t *__restrict__ u, int ell, int logn, uint32_t total,
                            uint64_t *__restrict__ V, ModTab mt, int Lp, uint64_t qt, uint64_t qinvP,
                            uint64_t qinvPs, uint64_t pq_hi, uint64_t pq_lo) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const uint32_t n = 1u << logn, t = i & (n - 1), bp = i >> logn;  // bp = b * 2 + p
  const uint64_t *row = u + ((size_t)bp * (ell + 1) + ell - 1) * n;
  const uint64_t x = row[t], xP = row[n + t];
  const uint64_t P = mt.q[Lp];
  const uint64_t k = shoup(submod(xP, x, P), qinvP, qinvPs, P);  // x < q_last < P
  uint64_t lo = qt * k, hi = __umul64hi(qt, k);
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, 0;" : "+l"(lo), "+l"(hi) : "l"(x));
  // centred: v > floor(P q / 2)  <=>  2 v > P q  (P q odd)
  const uint64_t h2 = (hi << 1) | (lo >> 63), l2 = lo << 1;
  const bool neg = h2 > pq_hi || (h2 == pq_hi && l2 > pq_lo);
  if (neg) {  // magnitude P q - v
    const uint64_t nl = pq_lo - lo, nh = pq_hi - hi - (pq_lo < lo ? 1 : 0);
    lo = nl;
    hi = nh;
  }
  uint64_t *out = V + (size_t)bp * (ell - 1) * n + t;
  for (int l = 0; l < ell - 1; l++) {
    const uint64_t q = mt.q[l];
    const uint64_t r = reduce128(hi, lo, q, mt.bar[l], mt.r64[l], mt.r64s[l]);
    out[(size_t)l * n] = neg ? (r ? q - r : 0) : r;
  }
}

KipAcc kip_acc(const hd_context *c, int ell, const uint64_t *c0, size_t c0_stride) {
  KipAcc ka;
  ka.c0 = c0;
  ka.c0_stride = c0_stride;
  for (int l = 0; l < ell; l++) {
    ka.pw[l] = ks_P_mod(c, c->mod[l]);
    ka.pws[l] = host_shoup(ka.pw[l], c->mod[l]);
  }
  return ka;
}

// ---- general hybrid key switching (R31: alpha limbs per digit, K special primes) ----------
// Fast basis conversion with centred digits: from the coefficient-form residues x_i of one
// integer modulo the source moduli b_i (i < cnt), out_j = sum_i y_i (B/b_i) mod m_j with
// y_i = centred([x_i (B/b_i)^{-1}]_{b_i}) -- for one source modulus the centred lift (R12).
constexpr int CONV_MAXSRC = 8, CONV_MAXTGT = 24;
struct ConvTab {
  int cnt = 0, ntgt = 0;
  uint8_t src_m[CONV_MAXSRC] = {}, tgt_m[CONV_MAXTGT] = {};
  uint64_t inv[CONV_MAXSRC] = {}, invs[CONV_MAXSRC] = {};
  uint64_t hat[CONV_MAXSRC][CONV_MAXTGT] = {}, hats[CONV_MAXSRC][CONV_MAXTGT] = {};
};
// src rows of group g: src + g src_gs + i n (i < cnt); out rows: out + g out_gs + j n (j < ntgt)
__global__ void __launch_bounds__(TPB) conv_kernel(const uint64_t *__restrict__ src, size_t src_gs,
                                                   uint64_t *__restrict__ out, size_t out_gs, int n, ModTab mt,
                                                   ConvTab ct) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t g = blockIdx.y;
  if (t >= (uint32_t)n) return;
  uint64_t mag[CONV_MAXSRC];
  bool neg[CONV_MAXSRC];
  for (int i = 0; i < ct.cnt; i++) {
    const int bm = ct.src_m[i];
    const uint64_t b = mt.q[bm];
    const uint64_t y = shoup(src[(size_t)g * src_gs + (size_t)i * n + t], ct.inv[i], ct.invs[i], b);
    neg[i] = y > (b >> 1);
    mag[i] = neg[i] ? b - y : y;
  }
  for (int j = 0; j < ct.ntgt; j++) {
    const int m = ct.tgt_m[j];
    const uint64_t q = mt.q[m], bar = mt.bar[m];
    uint64_t acc = 0;
    for (int i = 0; i < ct.cnt; i++) {
      const uint64_t v = shoup(reduce64(mag[i], q, bar), ct.hat[i][j], ct.hats[i][j], q);
      acc = addmod(acc, neg[i] ? (v ? q - v : 0) : v, q);
    }
    out[(size_t)g * out_gs + (size_t)j * n + t] = acc;
  }
}

ConvTab conv_table(const hd_context *c, const std::vector<int> &srcm, const std::vector<int> &tgtm) {
  ConvTab ct;
  ct.cnt = (int)srcm.size();
  ct.ntgt = (int)tgtm.size();
  for (int i = 0; i < ct.cnt; i++) {
    const uint64_t b = c->mod[srcm[i]];
    uint64_t hb = 1 % b;
    for (int k = 0; k < ct.cnt; k++)
      if (k != i) hb = host_mulmod(hb, c->mod[srcm[k]] % b, b);
    ct.src_m[i] = (uint8_t)srcm[i];
    ct.inv[i] = host_powmod(hb, b - 2, b);
    ct.invs[i] = host_shoup(ct.inv[i], b);
    for (int j = 0; j < ct.ntgt; j++) {
      const uint64_t m = c->mod[tgtm[j]];
      uint64_t h = 1 % m;
      for (int k = 0; k < ct.cnt; k++)
        if (k != i) h = host_mulmod(h, c->mod[srcm[k]] % m, m);
      ct.hat[i][j] = h;
      ct.hats[i][j] = host_shoup(h, m);
    }
  }
  for (int j = 0; j < ct.ntgt; j++) ct.tgt_m[j] = (uint8_t)tgtm[j];
  return ct;
}

hd_status conv_run(hd_context *c, const uint64_t *src, size_t src_gs, uint32_t groups, uint64_t *out, size_t out_gs,
                   const ConvTab &ct) {
  if (ct.cnt > CONV_MAXSRC || ct.ntgt > CONV_MAXTGT) return hd_fail(HD_E_PARAMS, "basis conversion too wide");
  conv_kernel<<<dim3((c->n + TPB - 1) / TPB, groups), TPB, 0, c->stream>>>(src, src_gs, out, out_gs, c->n, c->mt, ct);
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

// Key inner product over the general extended basis; x = b * K + k, output u[x][p][e],
// e < ell + Ksp.  dig [b][d][slot][n] (the digit's non-own moduli, NTT form; its own limbs are
// c1's rows c1 + b c1_stride + e n), key [d][p][M][n].
// Accumulate mode as kip_kernel (R23).  Two coefficients per thread.
__global__ void __launch_bounds__(TPB) kipg_kernel(const uint64_t *__restrict__ dig, const uint64_t *__restrict__ c1,
                                                   size_t c1_stride, uint64_t *__restrict__ u, int ell, int ext,
                                                   int beta, int alpha, int K, int L, int M, int logn,
                                                   const uint64_t *const *__restrict__ kptr,
                                                   const uint32_t *__restrict__ gal, ModTab mt, KipAcc ka,
                                                   FDiv f_ext, FDiv f_K) {
  const int n = 1 << logn;
  const uint32_t t = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const uint32_t xe = blockIdx.y;
  const uint32_t x = fdiv_q(xe, f_ext), e = xe - x * ext;
  const uint32_t b = fdiv_q(x, f_K), k = x - b * K;
  if (t >= (uint32_t)n) return;
  const int gm = (int)e < ell ? (int)e : L + ((int)e - ell);
  const uint32_t g = gal[k];
  const uint32_t s0 = galois_src(t, g, logn), s1 = galois_src(t + 1, g, logn);
  const uint64_t *key = kptr[k];
  const uint64_t *dg = dig + (size_t)b * beta * ext * n;
  uint64_t a0l = 0, a0h = 0, a1l = 0, a1h = 0, b0l = 0, b0h = 0, b1l = 0, b1h = 0;
  for (int d = 0; d < beta; d++) {
    // digit d's own limbs [lo, lo + cnt) are c1's rows (the conversion reproduces them exactly,
    // R31); its other moduli sit in slots e (e < lo) and e - cnt (e >= lo + cnt)
    const int lo = d * alpha, cnt = min(alpha, ell - lo);
    const uint64_t *row = ((int)e >= lo && (int)e < lo + cnt)
                              ? c1 + (size_t)b * c1_stride + (size_t)e * n
                              : dg + ((size_t)d * ext + ((int)e < lo ? (int)e : (int)e - cnt)) * n;
    const uint64_t v0 = row[s0], v1 = row[s1];
    const ulonglong2 k0 = *reinterpret_cast<const ulonglong2 *>(key + ((size_t)(d * 2 + 0) * M + gm) * n + t);
    const ulonglong2 k1 = *reinterpret_cast<const ulonglong2 *>(key + ((size_t)(d * 2 + 1) * M + gm) * n + t);
    mac128(a0l, a0h, v0, k0.x);
    mac128(b0l, b0h, v1, k0.y);
    mac128(a1l, a1h, v0, k1.x);
    mac128(b1l, b1h, v1, k1.y);
  }
  const uint64_t q = mt.q[gm], bar = mt.bar[gm], r64 = mt.r64[gm], r64s = mt.r64s[gm];
  ulonglong2 *o0 = reinterpret_cast<ulonglong2 *>(u + ((size_t)(x * 2 + 0) * ext + e) * n + t);
  ulonglong2 *o1 = reinterpret_cast<ulonglong2 *>(u + ((size_t)(x * 2 + 1) * ext + e) * n + t);
  ulonglong2 v0 = make_ulonglong2(reduce128(a0h, a0l, q, bar, r64, r64s), reduce128(b0h, b0l, q, bar, r64, r64s));
  ulonglong2 v1 = make_ulonglong2(reduce128(a1h, a1l, q, bar, r64, r64s), reduce128(b1h, b1l, q, bar, r64, r64s));
  if (ka.c0) {
    const ulonglong2 p0 = *o0, p1 = *o1;
    v0 = make_ulonglong2(addmod(v0.x, p0.x, q), addmod(v0.y, p0.y, q));
    v1 = make_ulonglong2(addmod(v1.x, p1.x, q), addmod(v1.y, p1.y, q));
    if ((int)e < ell) {
      const uint64_t *c0r = ka.c0 + (size_t)b * ka.c0_stride + (size_t)e * n;
      v0.x = addmod(v0.x, shoup(c0r[s0], ka.pw[e], ka.pws[e], q), q);
      v0.y = addmod(v0.y, shoup(c0r[s1], ka.pw[e], ka.pws[e], q), q);
    }
  }
  *o0 = v0;
  *o1 = v1;
}

inline dim3 grid_pairs(int n, uint32_t rows) { return dim3((n / 2 + TPB - 1) / TPB, rows); }

RowMap mods_seq(RowMap rm, uint32_t mdiv, int count, int first = 0) {
  rm.mdiv = mdiv;
  rm.mlen = count;
  for (int i = 0; i < count; i++) rm.midx[i] = (uint8_t)(first + i);
  return rm;
}
}  // namespace

hd_status ks_modup(hd_context *c, const uint64_t *c1, size_t c1_stride, uint32_t B, int ell, uint64_t *dig,
                   uint64_t *tmp) {
  const int n = c->n;
  // 1. INTT of every limb of c1 (out of place, into tmp[b][d]); modulus q_d
  RowMap rt = mods_seq(RowMap{}, 1, ell);
  NttSrc src;
  src.base = c1;
  src.map.gsize = ell;
  src.map.gstride = c1_stride;
  hd_status s = ntt_run(c, tmp, B * ell, rt, true, &src, nullptr);
  if (s) return s;
  if (ks_general(c)) {
    // 2. digit d (limbs [d alpha, min((d+1) alpha, ell))): fast basis conversion with centred
    //    digits into every modulus e of Q_ell u P (own limbs reproduce c1), rows dig[b][d][e]
    //    except the digit's own limbs, which reproduce c1 (the KIP reads c1's rows there): slots
    //    [0, ext - cnt) of dig[b][d] hold the other moduli in order
    const int ext = ell + c->K, beta = ks_beta(c, ell);
    for (int d = 0; d < beta; d++) {
      const int lo = d * c->alpha, cnt = std::min(c->alpha, ell - lo);
      std::vector<int> sm(cnt), tg;
      for (int i = 0; i < cnt; i++) sm[i] = lo + i;
      for (int e = 0; e < ext; e++)
        if (e < lo || e >= lo + cnt) tg.push_back(ks_ext_mod(c, ell, e));
      uint64_t *dd = dig + (size_t)d * ext * n;
      if ((s = conv_run(c, tmp + (size_t)lo * n, (size_t)ell * n, B, dd, (size_t)beta * ext * n, conv_table(c, sm, tg))))
        return s;
      // 3. NTT of the digit's rows: B groups of ext - cnt rows
      RowMap rd{};
      rd.gsize = (uint32_t)tg.size();
      rd.gstride = (uint64_t)beta * ext * n;
      rd.mdiv = 1;
      rd.mlen = (uint32_t)tg.size();
      for (size_t i = 0; i < tg.size(); i++) rd.midx[i] = (uint8_t)tg[i];
      if ((s = ntt_run(c, dd, B * (uint32_t)tg.size(), rd, false, nullptr, nullptr))) return s;
    }
    return HD_OK;
  }
  // 2. rows (b, d, slot) of dig: NTT over ext modulus e = slot < d ? slot : slot + 1 of the
  //    centred lift of tmp[b][d] (source modulus q_d)
  RowMap rd{};
  rd.mdiv = 1;
  rd.mlen = ell * ell;
  for (int d = 0; d < ell; d++)
    for (int sl = 0; sl < ell; sl++) {
      const int e = sl < d ? sl : sl + 1;
      rd.midx[d * ell + sl] = (uint8_t)(e < ell ? e : c->L);
    }
  NttSrc lift;
  lift.base = tmp;
  lift.lift = true;
  lift.map.gsize = ell;  // rows (b, d, *) all read tmp row (b, d)
  lift.map.gstride = n;
  lift.map.s3 = 0;
  lift.map.g2 = 1;
  lift.map.s2 = 0;
  lift.map = mods_seq(lift.map, ell, ell);  // source modulus d = (r / ell) % ell
  return ntt_run(c, dig, B * ell * ell, rd, false, &lift, nullptr);
}

hd_status ks_kip(hd_context *c, const uint64_t *dig, const uint64_t *c1, size_t c1_stride, uint32_t B, uint32_t K,
                 int ell, const uint64_t *const *kptr_dev, const uint32_t *gal_dev, uint64_t *u) {
  if (ks_general(c)) {
    const int ext = ell + c->K;
    kipg_kernel<<<grid_pairs(c->n, B * K * ext), TPB, 0, c->stream>>>(
        dig, c1, c1_stride, u, ell, ext, ks_beta(c, ell), c->alpha, K, c->L, ks_M(c), c->logn, kptr_dev, gal_dev,
        c->mt, KipAcc{}, fdiv_make(ext), fdiv_make(K));
    ++c->launches;
    HD_CUDA(cudaGetLastError());
    return HD_OK;
  }
  const dim3 g1((c->n + TPB - 1) / TPB, B * K * (ell + 1));
  const char *kv = getenv("HD_KIP1");  // A/B knob: 0 keeps the two-coefficient kernel
  if (!(kv && kv[0] == '0') && ell >= 1 && ell <= 4 && B * K * (ell + 1) <= 65535u) {
    auto kern = ell == 1 ? kip1_kernel<1> : ell == 2 ? kip1_kernel<2> : ell == 3 ? kip1_kernel<3> : kip1_kernel<4>;
    kern<<<g1, TPB, 0, c->stream>>>(dig, c1, c1_stride, u, K, c->L, c->logn, kptr_dev, gal_dev, c->mt, KipAcc{},
                                    fdiv_make(K));
    ++c->launches;
    HD_CUDA(cudaGetLastError());
    return HD_OK;
  }
  kip_kernel<<<grid_pairs(c->n, B * K * (ell + 1)), TPB, 0, c->stream>>>(dig, c1, c1_stride, u, ell, K, c->L, c->logn,
                                                                        kptr_dev, gal_dev, c->mt, KipAcc{},
                                                                        fdiv_make(ell + 1), fdiv_make(K));
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status ks_kip_accumulate(hd_context *c, const uint64_t *dig, const uint64_t *ct, size_t ct_stride, uint32_t B,
                            int ell, const uint64_t *const *kptr_dev, const uint32_t *gal_dev, uint64_t *u) {
  if (ks_general(c)) {
    const int ext = ell + c->K;
    kipg_kernel<<<grid_pairs(c->n, B * ext), TPB, 0, c->stream>>>(
        dig, ct + (size_t)ell * c->n, ct_stride, u, ell, ext, ks_beta(c, ell), c->alpha, 1, c->L, ks_M(c), c->logn,
        kptr_dev, gal_dev, c->mt, kip_acc(c, ell, ct, ct_stride), fdiv_make(ext), fdiv_make(1));
    ++c->launches;
    HD_CUDA(cudaGetLastError());
    return HD_OK;
  }
  kip_kernel<<<grid_pairs(c->n, B * (ell + 1)), TPB, 0, c->stream>>>(
      dig, ct + (size_t)ell * c->n, ct_stride, u, ell, 1, c->L, c->logn, kptr_dev, gal_dev, c->mt,
      kip_acc(c, ell, ct, ct_stride), fdiv_make(ell + 1), fdiv_make(1));
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status ks_giant_sum(hd_context *c, uint32_t B, int ell, int J, const uint64_t *const *dig, const uint64_t *const *ct,
                       const int *slot, const uint64_t *t0, size_t ct_stride, const uint64_t *const *kptr_dev,
                       const uint32_t *gal_dev, uint64_t *u) {
  if (ks_general(c) || J > GIANT_MAXJ) return hd_fail(HD_E_PARAMS, "combined giant sum: alpha = K = 1, J <= 8");
  GiantSet gs;
  gs.J = J;
  for (int j = 0; j < J; j++) {
    gs.dig[j] = dig[j];
    gs.ct[j] = ct[j];
    gs.slot[j] = slot[j];
  }
  gs.t0 = t0;
  gs.ct_stride = ct_stride;
  const KipAcc ka = kip_acc(c, ell, nullptr, 0);
  const dim3 g1((c->n + TPB - 1) / TPB, B * (ell + 1));
#define HD_KG(J_, E_)                                                                                          \
  if (J == J_ && ell == E_) {                                                                                  \
    kip_giant1_kernel<J_, E_><<<g1, TPB, 0, c->stream>>>(u, c->L, c->logn, kptr_dev, gal_dev, c->mt, ka, gs); \
    ++c->launches;                                                                                             \
    HD_CUDA(cudaGetLastError());                                                                               \
    return HD_OK;                                                                                              \
  }
  HD_KG(1, 1) HD_KG(1, 2) HD_KG(2, 1) HD_KG(2, 2) HD_KG(3, 1) HD_KG(3, 2) HD_KG(3, 3) HD_KG(1, 3) HD_KG(2, 3)
#undef HD_KG
  kip_giant_kernel<<<grid_pairs(c->n, B * (ell + 1)), TPB, 0, c->stream>>>(u, ell, c->L, c->logn, kptr_dev, gal_dev,
                                                                          c->mt, ka, gs, fdiv_make(ell + 1));
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status ks_add_pscaled(hd_context *c, uint64_t *u, const uint64_t *ct, size_t ct_stride, uint32_t B, int ell) {
  add_pscaled_kernel<<<grid_pairs(c->n, B * 2 * ell), TPB, 0, c->stream>>>(
      u, (size_t)2 * (ell + c->K) * c->n, ct, ct_stride, ell, ell + c->K, c->n, c->mt, kip_acc(c, ell, nullptr, 0));
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status ks_moddown(hd_context *c, uint64_t *u, uint32_t X, uint32_t K, int ell, const uint32_t *gal_dev,
                     const uint64_t *c0, size_t c0_stride, uint64_t *dst, size_t dst_stride, bool accumulate,
                     uint64_t *tmp) {
  const int n = c->n, L = c->L;
  if (ks_general(c)) {
    const int Ksp = c->K, ext = ell + Ksp;
    // 1. INTT of the K special limbs of both polys, in place: rows (x*2 + p, k) at u + (r ext + ell + k) n
    RowMap rp{};
    rp.gsize = Ksp;
    rp.gstride = (uint64_t)ext * n;
    rp.mdiv = 1;
    rp.mlen = Ksp;
    for (int k = 0; k < Ksp; k++) rp.midx[k] = (uint8_t)(L + k);
    hd_status s = ntt_run(c, u + (size_t)ell * n, 2 * X * Ksp, rp, true, nullptr, nullptr);
    if (s) return s;
    // 2. fast basis conversion (centred digits) from P = prod p_k into q_0 .. q_{ell-1}: tmp [x][p][l]
    std::vector<int> sm(Ksp), tg(ell);
    for (int k = 0; k < Ksp; k++) sm[k] = L + k;
    for (int l = 0; l < ell; l++) tg[l] = l;
    if ((s = conv_run(c, u + (size_t)ell * n, (size_t)ext * n, 2 * X, tmp, (size_t)ell * n, conv_table(c, sm, tg))))
      return s;
    // 3. NTT_l of the converted rows, final store dst_x[p][l] (+)= (u[x][p][l] - .) P^{-1} (+ pi_g(c0_b)[l])
    RowMap rq = mods_seq(RowMap{}, 1, ell);
    NttEpi epi;
    epi.mode = c0 ? 2 : 1;
    epi.acc = accumulate;
    epi.ell = ell;
    epi.K = K;
    epi.A = u;
    epi.amap.gsize = ell;
    epi.amap.gstride = (uint64_t)ext * n;
    epi.out = dst;
    epi.omap.gsize = 2 * ell;
    epi.omap.gstride = dst_stride;
    epi.c0 = c0;
    epi.c0_stride = c0_stride;
    epi.gal = gal_dev;
    for (int l = 0; l < ell; l++) {
      epi.w[l] = host_powmod(ks_P_mod(c, c->mod[l]), c->mod[l] - 2, c->mod[l]);
      epi.ws[l] = host_shoup(epi.w[l], c->mod[l]);
    }
    return ntt_run(c, tmp, 2 * X * ell, rq, false, nullptr, &epi);
  }
  // 1. INTT of the P limb of both polys, in place: rows r = x*2 + p at u + (r (ell+1) + ell) n
  RowMap rp = rowmap_simple(1, {L}, 1, (uint64_t)(ell + 1) * n);
  hd_status s = ntt_run(c, u + (size_t)ell * n, 2 * X, rp, true, nullptr, nullptr);
  if (s) return s;
  // 2. rows r = (x*2 + p) ell + l: NTT_l of the centred lift of u[x][p][ell] (into tmp),
  //    final store: dst_x[p][l] (+)= (u[x][p][l] - .) P^{-1} (+ pi_g(c0_b)[l] for p == 0)
  RowMap rq = mods_seq(RowMap{}, 1, ell);
  NttSrc lift;
  lift.base = u + (size_t)ell * n;
  lift.lift = true;
  lift.map.gsize = ell;
  lift.map.gstride = (uint64_t)(ell + 1) * n;
  lift.map.g2 = 1;
  lift.map = mods_seq(lift.map, 1, 1, L);
  NttEpi epi;
  epi.mode = c0 ? 2 : 1;
  epi.acc = accumulate;
  epi.ell = ell;
  epi.K = K;
  epi.A = u;
  epi.amap.gsize = ell;
  epi.amap.gstride = (uint64_t)(ell + 1) * n;
  epi.out = dst;
  epi.omap.gsize = 2 * ell;
  epi.omap.gstride = dst_stride;
  epi.c0 = c0;
  epi.c0_stride = c0_stride;
  epi.gal = gal_dev;
  for (int l = 0; l < ell; l++) {
    epi.w[l] = host_powmod(c->mod[L] % c->mod[l], c->mod[l] - 2, c->mod[l]);
    epi.ws[l] = host_shoup(epi.w[l], c->mod[l]);
  }
  return ntt_run(c, tmp, 2 * X * ell, rq, false, &lift, &epi);
}

hd_status ks_rescale(hd_context *c, const uint64_t *S, size_t s_stride, uint32_t B, int ell, uint64_t *out,
                     size_t out_stride, uint64_t *tmp1, uint64_t *tmp2) {
  (void)tmp2;
  const int n = c->n, last = ell - 1, lo = ell - 1;
  // 1. INTT of the last limb of both polys, out of place into tmp1[b*2 + p]
  NttSrc src;
  src.base = S + (size_t)last * n;
  src.map.gsize = 2;
  src.map.gstride = s_stride;
  src.map.s3 = (uint64_t)ell * n;
  RowMap rt = rowmap_simple(1, {last});
  hd_status s = ntt_run(c, tmp1, 2 * B, rt, true, &src, nullptr);
  if (s) return s;
  // 2. rows r = (b*2 + p) lo + l of out: NTT_l of the centred lift of tmp1[b*2 + p],
  //    final store out[b][p][l] = (S[b][p][l] - .) q_last^{-1}
  RowMap ro;
  ro.gsize = 2 * lo;
  ro.gstride = out_stride;
  ro = mods_seq(ro, 1, lo);
  NttSrc lift;
  lift.base = tmp1;
  lift.lift = true;
  lift.map.gsize = lo;
  lift.map.gstride = n;
  lift.map.g2 = 1;
  lift.map = mods_seq(lift.map, 1, 1, last);
  NttEpi epi;
  epi.mode = 1;
  epi.ell = lo;
  epi.A = S;
  epi.amap.gsize = 2 * lo;
  epi.amap.gstride = s_stride;
  epi.amap.g2 = lo;
  epi.amap.s2 = (uint64_t)ell * n;
  epi.out = out;
  epi.omap = ro;
  for (int l = 0; l < lo; l++) {
    epi.w[l] = host_powmod(c->mod[last] % c->mod[l], c->mod[l] - 2, c->mod[l]);
    epi.ws[l] = host_shoup(epi.w[l], c->mod[l]);
  }
  return ntt_run(c, out, 2 * B * lo, ro, false, &lift, &epi);
}

hd_status ks_relin_rescale(hd_context *c, uint64_t *S3, uint32_t B, int ell, const uint64_t *const *rlk_dev,
                           const uint32_t *gal_dev, uint64_t *out, uint64_t *dig, uint64_t *u, uint64_t *tmp,
                           uint64_t *V) {
  if (ks_general(c))  // the two-modulus CRT rounding needs one special prime (R29)
    return hd_fail(HD_E_PARAMS, "relinearisation is implemented for num_special = digit_limbs = 1 only");
  const int n = c->n, L = c->L, lo = ell - 1;
  const size_t s3 = (size_t)3 * ell * n;
  uint64_t *d2 = S3 + (size_t)2 * ell * n;
  hd_status s;
  // 1. X = P (d0, d1) + KIP(ModUp(d2)) over Q_ell u {P}: u [B][2][ell+1][n]
  if ((s = ks_modup(c, d2, s3, B, ell, dig, tmp))) return s;
  if ((s = ks_kip(c, dig, d2, s3, B, 1, ell, rlk_dev, gal_dev, u))) return s;
  if ((s = ks_add_pscaled(c, u, S3, s3, B, ell))) return s;
  // 2. coefficient form of the q_{ell-1} and P rows of X, in place
  RowMap rt = rowmap_simple(1, {lo, L}, 2, (uint64_t)(ell + 1) * n);
  if ((s = ntt_run(c, u + (size_t)lo * n, 4 * B, rt, true, nullptr, nullptr))) return s;
  // 3. centred CRT remainder v = [X mod P q_{ell-1}] into q_0..q_{ell-2}
  const uint64_t P = c->mod[L], qt = c->mod[lo];
  const uint64_t qinvP = host_powmod(qt % P, P - 2, P);
  const unsigned __int128 pq = (unsigned __int128)P * qt;
  const uint32_t total = 2u * B * n;
  crt2_kernel<<<(total + TPB - 1) / TPB, TPB, 0, c->stream>>>(u, ell, c->logn, total, V, c->mt, L, qt, qinvP,
                                                              host_shoup(qinvP, P), (uint64_t)(pq >> 64),
                                                              (uint64_t)pq);
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  // 4. out[b][p][l] = (X[b][p][l] - NTT_l(v)) (P q_{ell-1})^{-1}
  RowMap ro;
  ro.gsize = 2 * lo;
  ro.gstride = (uint64_t)2 * lo * n;
  ro = mods_seq(ro, 1, lo);
  NttSrc src;
  src.base = V;
  NttEpi epi;
  epi.mode = 1;
  epi.ell = lo;
  epi.A = u;
  epi.amap.gsize = 2 * lo;
  epi.amap.gstride = (uint64_t)2 * (ell + 1) * n;
  epi.amap.g2 = lo;
  epi.amap.s2 = (uint64_t)(ell + 1) * n;
  epi.out = out;
  epi.omap = ro;
  for (int l = 0; l < lo; l++) {
    const uint64_t q = c->mod[l];
    epi.w[l] = host_powmod((uint64_t)(pq % q), q - 2, q);
    epi.ws[l] = host_shoup(epi.w[l], q);
  }
  return ntt_run(c, out, 2 * B * lo, ro, false, &src, &epi);
}
