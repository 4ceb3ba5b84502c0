// ks.cu -- hybrid RNS key switching (alpha = 1, one special prime P) and rescale.
//
// Rotation by r (R11): ModUp of c1 (digit d = centred
// INTT of limb d lifted into every other modulus of Q_ell u {P}, then NTT);
// key inner product with the NTT-domain Galois permutation pi_g fused into the
// digit loads; ModDown (centred INTT of the P limb, lift, NTT, (u - .) P^{-1});
// + pi_g(c0).  Rescale drops q_{ell-1} the same way (R12).
#include "common.cuh"
#include "ks.cuh"

namespace {
constexpr int TPB = 256;

// tmp[b][d][t] (coefficient form, mod q_d) -> dig[b][d][s][t], s < ell, in ext
// modulus e = s < d ? s : s + 1 (e == ell is P); dig[b][d][ell] = c1[b][d] (own limb).
__global__ void modup_lift_kernel(const uint64_t *__restrict__ x, const uint64_t *__restrict__ c1,
                                  size_t c1_stride, uint64_t *__restrict__ dig, int ell, int L, int n,
                                  ModTab mt) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t bd = blockIdx.y;  // b * ell + d
  const uint32_t b = bd / ell, d = bd % ell;
  if (t >= (uint32_t)n) return;
  const uint64_t qd = mt.q[d];
  const uint64_t v = x[(size_t)bd * n + t];
  uint64_t *out = dig + (size_t)bd * (ell + 1) * n;
  for (int s = 0; s < ell; s++) {
    int e = s < (int)d ? s : s + 1;
    int gm = e < ell ? e : L;
    out[(size_t)s * n + t] = lift_centred(v, qd, mt.q[gm], mt.bar[gm]);
  }
  out[(size_t)ell * n + t] = c1[(size_t)b * c1_stride + (size_t)d * n + t];
}

// Key inner product; x = b * K + k.  Output u[x][p][e][t], e <= ell (e == ell: P).
__global__ void kip_kernel(const uint64_t *__restrict__ dig, uint64_t *__restrict__ u, int ell, int K, int L,
                           int logn, const uint64_t *const *__restrict__ kptr, const uint32_t *__restrict__ gal,
                           ModTab mt) {
  const int n = 1 << logn;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t xe = blockIdx.y;
  const uint32_t x = xe / (ell + 1), e = xe % (ell + 1);
  const uint32_t b = x / K, k = x % K;
  if (t >= (uint32_t)n) return;
  const int gm = (int)e < ell ? (int)e : L;
  const uint32_t src = galois_src(t, gal[k], logn);
  const uint64_t *key = kptr[k];
  const uint64_t *dg = dig + (size_t)b * ell * (ell + 1) * n;
  uint64_t a0l = 0, a0h = 0, a1l = 0, a1h = 0;
  for (int d = 0; d < ell; d++) {
    int slot = ((int)e == d) ? ell : ((int)e < d ? (int)e : (int)e - 1);
    uint64_t v = dg[((size_t)d * (ell + 1) + slot) * n + src];
    uint64_t k0 = key[((size_t)(d * 2 + 0) * (L + 1) + gm) * n + t];
    uint64_t k1 = key[((size_t)(d * 2 + 1) * (L + 1) + gm) * n + t];
    mac128(a0l, a0h, v, k0);
    mac128(a1l, a1h, v, k1);
  }
  const uint64_t q = mt.q[gm];
  u[((size_t)(x * 2 + 0) * (ell + 1) + e) * n + t] = reduce128(a0h, a0l, q, mt.bar[gm], mt.r64[gm], mt.r64s[gm]);
  u[((size_t)(x * 2 + 1) * (ell + 1) + e) * n + t] = reduce128(a1h, a1l, q, mt.bar[gm], mt.r64[gm], mt.r64s[gm]);
}

// Lift a coefficient-form row over modulus `src_m` into `nt` target limbs:
// out[r][l][t] = [in[r][t]]_centred mod q_l, l < nt.  in row r at in + r*in_stride.
__global__ void lift_rows_kernel(const uint64_t *__restrict__ in, size_t in_stride, uint64_t *__restrict__ out,
                                 int nt, int src_m, int n, ModTab mt) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t r = blockIdx.y;
  if (t >= (uint32_t)n) return;
  const uint64_t v = in[(size_t)r * in_stride + t];
  const uint64_t qs = mt.q[src_m];
  for (int l = 0; l < nt; l++) out[((size_t)r * nt + l) * n + t] = lift_centred(v, qs, mt.q[l], mt.bar[l]);
}

struct InvTab {
  uint64_t w[HD_MAXMOD], ws[HD_MAXMOD];
};

// ModDown combine: for x, p, l < ell:
//   v = (u[x][p][l] - lifted[x][p][l]) * P^{-1} mod q_l  (+ c0_x[l][pi(t)] when p == 0)
//   dst_x[p][l] = v  (ACC: dst += v)
template <bool ACC>
__global__ void moddown_combine_kernel(const uint64_t *__restrict__ u, const uint64_t *__restrict__ lifted,
                                       uint64_t *__restrict__ dst, size_t dst_stride, const uint64_t *__restrict__ c0,
                                       size_t c0_stride, int K, int ell, int logn, const uint32_t *__restrict__ gal,
                                       ModTab mt, InvTab pinv) {
  const int n = 1 << logn;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t xpl = blockIdx.y;
  const uint32_t l = xpl % ell, xp = xpl / ell, p = xp % 2, x = xp / 2;
  const uint32_t b = x / K, k = x % K;
  if (t >= (uint32_t)n) return;
  const uint64_t q = mt.q[l];
  uint64_t a = u[((size_t)xp * (ell + 1) + l) * n + t];
  uint64_t c = lifted[((size_t)xp * ell + l) * n + t];
  uint64_t v = shoup(submod(a, c, q), pinv.w[l], pinv.ws[l], q);
  if (p == 0 && c0) {
    uint32_t src = galois_src(t, gal[k], logn);
    v = addmod(v, c0[(size_t)b * c0_stride + (size_t)l * n + src], q);
  }
  uint64_t *o = dst + (size_t)x * dst_stride + ((size_t)p * ell + l) * n + t;
  *o = ACC ? addmod(*o, v, q) : v;
}

// Rescale combine: out[b][p][l] = (S[b][p][l] - lifted[b][p][l]) * q_last^{-1} mod q_l.
__global__ void rescale_combine_kernel(const uint64_t *__restrict__ S, size_t s_stride,
                                       const uint64_t *__restrict__ lifted, uint64_t *__restrict__ out,
                                       size_t out_stride, int ell, int n, ModTab mt, InvTab qinv) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t bpl = blockIdx.y;
  const int lo = ell - 1;
  const uint32_t l = bpl % lo, bp = bpl / lo, p = bp % 2, b = bp / 2;
  if (t >= (uint32_t)n) return;
  const uint64_t q = mt.q[l];
  uint64_t a = S[(size_t)b * s_stride + ((size_t)p * ell + l) * n + t];
  uint64_t c = lifted[((size_t)bp * lo + l) * n + t];
  out[(size_t)b * out_stride + ((size_t)p * lo + l) * n + t] = shoup(submod(a, c, q), qinv.w[l], qinv.ws[l], q);
}

// gather rows: out[r] = in[(r / per) * gstride + (r % per) * rstride + off] (n elements)
__global__ void gather_rows_kernel(const uint64_t *__restrict__ in, uint64_t *__restrict__ out, uint32_t per,
                                   size_t gstride, size_t rstride, int n) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t r = blockIdx.y;
  if (t >= (uint32_t)n) return;
  out[(size_t)r * n + t] = in[(size_t)(r / per) * gstride + (size_t)(r % per) * rstride + t];
}

__global__ void add_ct_kernel(uint64_t *__restrict__ dst, size_t dst_stride, const uint64_t *__restrict__ src,
                              size_t src_stride, int ell, int n, ModTab mt) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t bpl = blockIdx.y;
  const uint32_t l = bpl % ell, bp = bpl / ell, b = bp / 2, p = bp % 2;
  if (t >= (uint32_t)n) return;
  size_t off = ((size_t)p * ell + l) * n + t;
  uint64_t *o = dst + (size_t)b * dst_stride + off;
  *o = addmod(*o, src[(size_t)b * src_stride + off], mt.q[l]);
}

inline dim3 grid_rows(int n, uint32_t rows) { return dim3((n + TPB - 1) / TPB, rows); }
}  // namespace

hd_status ks_modup(hd_context *c, const uint64_t *c1, size_t c1_stride, uint32_t B, int ell, uint64_t *dig,
                   uint64_t *tmp) {
  const int n = c->n;
  // 1. gather the c1 limbs [B][ell] and INTT them
  gather_rows_kernel<<<grid_rows(n, B * ell), TPB, 0, c->stream>>>(c1, tmp, ell, c1_stride, n, n); ++c->launches;
  RowMap rm{};
  rm.gsize = 1u << 30;
  rm.mdiv = 1;
  rm.mlen = ell;
  for (int i = 0; i < ell; i++) rm.midx[i] = i;
  hd_status s = ntt_rows(c, tmp, B * ell, rm, true);
  if (s) return s;
  // 2. lift into the other moduli; own limb copied
  modup_lift_kernel<<<grid_rows(n, B * ell), TPB, 0, c->stream>>>(tmp, c1, c1_stride, dig, ell, c->L, n, c->mt); ++c->launches;
  // 3. NTT the lifted rows: rows (b, d, s<ell) at dig + ((b ell + d)(ell+1) + s) n
  RowMap rn{};
  rn.gsize = ell;
  rn.gstride = (uint64_t)(ell + 1) * n;
  rn.mdiv = 1;
  rn.mlen = ell * ell;
  for (int d = 0; d < ell; d++)
    for (int s2 = 0; s2 < ell; s2++) {
      int e = s2 < d ? s2 : s2 + 1;
      rn.midx[d * ell + s2] = (uint8_t)(e < ell ? e : c->L);
    }
  return ntt_rows(c, dig, B * ell * ell, rn, false);
}

hd_status ks_kip(hd_context *c, const uint64_t *dig, uint32_t B, uint32_t K, int ell,
                 const uint64_t *const *kptr_dev, const uint32_t *gal_dev, uint64_t *u) {
  kip_kernel<<<grid_rows(c->n, B * K * (ell + 1)), TPB, 0, c->stream>>>(dig, u, ell, K, c->L, c->logn, kptr_dev,
                                                                       gal_dev, c->mt); ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status ks_moddown(hd_context *c, uint64_t *u, uint32_t X, uint32_t K, int ell, const uint32_t *gal_dev,
                     const uint64_t *c0, size_t c0_stride, uint64_t *dst, size_t dst_stride, bool accumulate,
                     uint64_t *tmp) {
  const int n = c->n, L = c->L;
  // 1. INTT of the P limb of both polys: rows r = x*2 + p at u + (r (ell+1) + ell) n
  RowMap rp = rowmap_simple(1, {L}, 1, (uint64_t)(ell + 1) * n);
  hd_status s = ntt_rows(c, u + (size_t)ell * n, 2 * X, rp, true);
  if (s) return s;
  // 2. lift to q_0..q_{ell-1}
  lift_rows_kernel<<<grid_rows(n, 2 * X), TPB, 0, c->stream>>>(u + (size_t)ell * n, (size_t)(ell + 1) * n, tmp,
                                                               ell, L, n, c->mt); ++c->launches;
  // 3. NTT
  RowMap rq{};
  rq.gsize = 1u << 30;
  rq.mdiv = 1;
  rq.mlen = ell;
  for (int i = 0; i < ell; i++) rq.midx[i] = i;
  if ((s = ntt_rows(c, tmp, 2 * X * ell, rq, false))) return s;
  // 4. combine
  InvTab pinv{};
  for (int l = 0; l < ell; l++) {
    pinv.w[l] = host_powmod(c->mod[L] % c->mod[l], c->mod[l] - 2, c->mod[l]);
    pinv.ws[l] = host_shoup(pinv.w[l], c->mod[l]);
  }
  dim3 g = grid_rows(n, 2 * X * ell);
  if (accumulate)
    moddown_combine_kernel<true><<<g, TPB, 0, c->stream>>>(u, tmp, dst, dst_stride, c0, c0_stride, K, ell, c->logn,
                                                           gal_dev, c->mt, pinv);
  else
    moddown_combine_kernel<false><<<g, TPB, 0, c->stream>>>(u, tmp, dst, dst_stride, c0, c0_stride, K, ell, c->logn,
                                                            gal_dev, c->mt, pinv);
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status ks_rescale(hd_context *c, const uint64_t *S, size_t s_stride, uint32_t B, int ell, uint64_t *out,
                     size_t out_stride, uint64_t *tmp1, uint64_t *tmp2) {
  const int n = c->n, last = ell - 1;
  // 1. gather the last limb of both polys: row r = b*2 + p at S + b*s_stride + (p ell + last) n
  gather_rows_kernel<<<grid_rows(n, 2 * B), TPB, 0, c->stream>>>(S + (size_t)last * n, tmp1, 2, s_stride,
                                                                 (size_t)ell * n, n); ++c->launches;
  hd_status s = ntt_rows(c, tmp1, 2 * B, rowmap_simple(1, {last}), true);
  if (s) return s;
  lift_rows_kernel<<<grid_rows(n, 2 * B), TPB, 0, c->stream>>>(tmp1, (size_t)n, tmp2, last, last, n, c->mt); ++c->launches;
  RowMap rq{};
  rq.gsize = 1u << 30;
  rq.mdiv = 1;
  rq.mlen = last;
  for (int i = 0; i < last; i++) rq.midx[i] = i;
  if ((s = ntt_rows(c, tmp2, 2 * B * last, rq, false))) return s;
  InvTab qi{};
  for (int l = 0; l < last; l++) {
    qi.w[l] = host_powmod(c->mod[last] % c->mod[l], c->mod[l] - 2, c->mod[l]);
    qi.ws[l] = host_shoup(qi.w[l], c->mod[l]);
  }
  rescale_combine_kernel<<<grid_rows(n, 2 * B * last), TPB, 0, c->stream>>>(S, s_stride, tmp2, out, out_stride, ell,
                                                                            n, c->mt, qi); ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status ct_add(hd_context *c, uint64_t *dst, size_t dst_stride, const uint64_t *src, size_t src_stride,
                 uint32_t B, int ell) {
  add_ct_kernel<<<grid_rows(c->n, B * 2 * ell), TPB, 0, c->stream>>>(dst, dst_stride, src, src_stride, ell, c->n,
                                                                     c->mt); ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}
