// ntt.cu -- batched 64-bit negacyclic NTT / INTT for sm_100a (K9 of SURVEY 2.2).
//
// Forward: Cooley-Tukey, natural order in, bit-reversed evaluation order out
// (R13); inverse: Gentleman-Sande, then x n^{-1}.  Twiddles are
// psi^{br(k)} with Shoup companions, per modulus.
//
// log n = s1 + s2.  The s1 "high" stages act on columns {hi 2^s2 + lo : hi} (one
// CTA holds CH columns of 2^s1 elements, loaded with coalesced row segments);
// the s2 "low" stages act on contiguous chunks of 2^s2 elements.  Each phase is
// one kernel with the data staged in shared memory; every butterfly keeps its
// operands fully reduced in [0, q).
#include "common.cuh"

namespace {

constexpr int NTT_THREADS = 256;
constexpr int LO_BITS_MAX = 11;  // 2^11 u64 = 16 KiB per chunk

__device__ __forceinline__ void ct_bfly(uint64_t &a, uint64_t &b, uint64_t w, uint64_t ws, uint64_t q) {
  uint64_t V = shoup(b, w, ws, q);
  uint64_t U = a;
  a = addmod(U, V, q);
  b = submod(U, V, q);
}
__device__ __forceinline__ void gs_bfly(uint64_t &a, uint64_t &b, uint64_t w, uint64_t ws, uint64_t q) {
  uint64_t U = a, V = b;
  a = addmod(U, V, q);
  b = shoup(submod(U, V, q), w, ws, q);
}

// High stages (mm = 1 .. 2^(s1-1)) forward / (2^(s1-1) .. 1) inverse.
template <bool INV>
__global__ void __launch_bounds__(NTT_THREADS) ntt_hi_kernel(uint64_t *base, RowMap rm, ModTab mt,
                                                             const uint64_t *__restrict__ tw,
                                                             const uint64_t *__restrict__ tws, int logn,
                                                             int s1, int ch, const uint64_t *ninv,
                                                             const uint64_t *ninvs, uint32_t r0) {
  extern __shared__ uint64_t sm[];
  const uint32_t n = 1u << logn, s2 = logn - s1;
  const uint32_t row = blockIdx.y + r0;
  const int m = row_mod(rm, row);
  const uint64_t q = mt.q[m];
  uint64_t *a = row_ptr(base, rm, row, n);
  const uint64_t *T = tw + (size_t)m * n, *TS = tws + (size_t)m * n;
  const uint32_t col0 = blockIdx.x * ch;
  const uint32_t H = 1u << s1, tot = H * ch;
  for (uint32_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    uint32_t hi = idx / ch, c = idx % ch;
    sm[idx] = a[((size_t)hi << s2) + col0 + c];
  }
  __syncthreads();
  const uint32_t nb = (H / 2) * ch;
  for (int k = 0; k < s1; k++) {
    int st = INV ? (s1 - 1 - k) : k;
    uint32_t mm = 1u << st, th = 1u << (s1 - 1 - st);
    for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
      uint32_t c = b % ch, bi = b / ch;
      uint32_t grp = bi >> (s1 - 1 - st);
      uint32_t h0 = grp * 2 * th + (bi & (th - 1));
      uint64_t &x0 = sm[h0 * ch + c], &x1 = sm[(h0 + th) * ch + c];
      uint64_t w = T[mm + grp], ws = TS[mm + grp];
      uint64_t u = x0, v = x1;
      if (INV) gs_bfly(u, v, w, ws, q);
      else ct_bfly(u, v, w, ws, q);
      x0 = u;
      x1 = v;
    }
    __syncthreads();
  }
  for (uint32_t idx = threadIdx.x; idx < tot; idx += blockDim.x) {
    uint32_t hi = idx / ch, c = idx % ch;
    uint64_t v = sm[idx];
    if (INV) v = shoup(v, ninv[m], ninvs[m], q);
    a[((size_t)hi << s2) + col0 + c] = v;
  }
}

// Low stages on contiguous chunks of 2^s2 elements.
template <bool INV>
__global__ void __launch_bounds__(NTT_THREADS) ntt_lo_kernel(uint64_t *base, RowMap rm, ModTab mt,
                                                             const uint64_t *__restrict__ tw,
                                                             const uint64_t *__restrict__ tws, int logn,
                                                             int s1, const uint64_t *ninv,
                                                             const uint64_t *ninvs, uint32_t r0) {
  extern __shared__ uint64_t sm[];
  const uint32_t n = 1u << logn, s2 = logn - s1, C = 1u << s2;
  const uint32_t row = blockIdx.y + r0, hi = blockIdx.x;
  const int m = row_mod(rm, row);
  const uint64_t q = mt.q[m];
  uint64_t *a = row_ptr(base, rm, row, n) + ((size_t)hi << s2);
  const uint64_t *T = tw + (size_t)m * n, *TS = tws + (size_t)m * n;
  for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) sm[i] = a[i];
  __syncthreads();
  for (int k = 0; k < (int)s2; k++) {
    int st = INV ? ((int)s2 - 1 - k) : k;  // stage within the low part
    uint32_t mm = 1u << (s1 + st);
    uint32_t t = 1u << (s2 - 1 - st);
    for (uint32_t b = threadIdx.x; b < C / 2; b += blockDim.x) {
      uint32_t grp_l = b / t, off = b % t;  // group inside the chunk
      uint32_t j0 = grp_l * 2 * t + off;
      uint32_t grp = (hi << st) + grp_l;
      uint64_t w = T[mm + grp], ws = TS[mm + grp];
      uint64_t u = sm[j0], v = sm[j0 + t];
      if (INV) gs_bfly(u, v, w, ws, q);
      else ct_bfly(u, v, w, ws, q);
      sm[j0] = u;
      sm[j0 + t] = v;
    }
    __syncthreads();
  }
  const bool scale = INV && s1 == 0;
  for (uint32_t i = threadIdx.x; i < C; i += blockDim.x) {
    uint64_t v = sm[i];
    if (scale) v = shoup(v, ninv[m], ninvs[m], q);
    a[i] = v;
  }
}

}  // namespace

RowMap rowmap_simple(uint32_t mdiv, std::initializer_list<int> mods, uint32_t gsize, uint64_t gstride) {
  RowMap rm{};
  rm.gsize = gsize;
  rm.gstride = gstride;
  rm.mdiv = mdiv;
  rm.mlen = (uint32_t)mods.size();
  int i = 0;
  for (int v : mods) rm.midx[i++] = (uint8_t)v;
  return rm;
}

// Constants n^{-1} per modulus live in a small device array inside the context's
// twiddle allocation (see context.cu): ninv_dev = itw + (L+1) n, shoup after it.
hd_status ntt_rows(hd_context *c, uint64_t *base, uint32_t rows, const RowMap &rm, bool inverse) {
  if (rows == 0) return HD_OK;
  const int logn = c->logn;
  const int s2 = logn <= 12 ? logn : LO_BITS_MAX;
  const int s1 = logn - s2;
  const uint64_t *ninv = c->itw + (size_t)(c->L + 1) * c->n;
  const uint64_t *ninvs = ninv + HD_MAXMOD;
  const size_t lo_smem = sizeof(uint64_t) << s2;
  int ch = s1 ? (2048 >> s1) : 0;
  if (ch < 16) ch = 16;
  const size_t hi_smem = sizeof(uint64_t) * ((size_t)ch << s1);
  dim3 glo(1u << s1, rows), ghi((1u << s2) / ch, rows);
  for (uint32_t r0 = 0; r0 < rows; r0 += 65535) {
    uint32_t rr = rows - r0 < 65535 ? rows - r0 : 65535;
    glo.y = rr;
    ghi.y = rr;
    if (!inverse) {
      if (s1) { ntt_hi_kernel<false><<<ghi, NTT_THREADS, hi_smem, c->stream>>>(base, rm, c->mt, c->tw, c->tws, logn, s1, ch, ninv, ninvs, r0); ++c->launches; }
      ntt_lo_kernel<false><<<glo, NTT_THREADS, lo_smem, c->stream>>>(base, rm, c->mt, c->tw, c->tws, logn, s1, ninv, ninvs, r0); ++c->launches;
    } else {
      ntt_lo_kernel<true><<<glo, NTT_THREADS, lo_smem, c->stream>>>(base, rm, c->mt, c->itw, c->itws, logn, s1, ninv, ninvs, r0); ++c->launches;
      if (s1) { ntt_hi_kernel<true><<<ghi, NTT_THREADS, hi_smem, c->stream>>>(base, rm, c->mt, c->itw, c->itws, logn, s1, ch, ninv, ninvs, r0); ++c->launches; }
    }
  }
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}
