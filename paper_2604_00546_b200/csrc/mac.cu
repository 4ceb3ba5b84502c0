// mac.cu -- fused diagonal x ciphertext multiply-accumulate (K14; a5 of SURVEY 8(a)).
//
// For every local aggregate a, limb m, coefficient t and giant step j
// (Alg. sender-bsgs Step 2b):
//   S[a][j][p][m][t] = sum_{i = i_lo(j)}^{i_hi(j)} r[i][p][m][t] * D[a][k(j,i)][m][t]  mod q_m
// with k(j,i) = (j n1 + i) mod N.  Products (< q^2 < 2^120) are accumulated
// exactly in 128 bits and reduced once per (a, j) -- lazy reduction; the sum is
// folded every 255 terms so any n1 is safe.
//
// The D stream (A_loc N L n u64, read exactly once per query) is the dominant
// HBM traffic of the whole path: each CTA owns 128 consecutive coefficients of
// one limb of one aggregate; a warp reads 256 contiguous bytes per diagonal.
#include "common.cuh"
#include "ks.cuh"

namespace {
constexpr int MAC_TPB = 128;

__global__ void __launch_bounds__(MAC_TPB) mac_kernel(const uint64_t *__restrict__ D,
                                                      const uint64_t *__restrict__ r, uint64_t *__restrict__ S,
                                                      int n1, int N, int L, int logn, int jmin, int nj, ModTab mt) {
  const int n = 1 << logn;
  const uint32_t t = blockIdx.x * MAC_TPB + threadIdx.x;
  const int m = blockIdx.y;
  const uint32_t a = blockIdx.z;
  if (t >= (uint32_t)n) return;
  const size_t limb_stride = (size_t)L * n;  // between diagonals / between (i,p) of r
  const uint64_t *Da = D + (size_t)a * N * limb_stride + (size_t)m * n + t;
  const uint64_t *rr = r + (size_t)m * n + t;
  uint64_t *Sa = S + (size_t)a * nj * 2 * limb_stride + (size_t)m * n + t;
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  for (int jj = 0; jj < nj; jj++) {
    const int j = jmin + jj;
    int i_lo = -j * n1 - N / 2;
    if (i_lo < 0) i_lo = 0;
    int i_hi = N / 2 - 1 - j * n1;
    if (i_hi > n1 - 1) i_hi = n1 - 1;
    uint64_t a0l = 0, a0h = 0, a1l = 0, a1h = 0;
    int cnt = 0;
    for (int i = i_lo; i <= i_hi; i++) {
      const int k = (j * n1 + i) & (N - 1);
      const uint64_t d = __ldcs(Da + (size_t)k * limb_stride);  // streamed once: evict-first
      const uint64_t r0 = __ldg(rr + (size_t)(2 * i) * limb_stride);
      const uint64_t r1 = __ldg(rr + (size_t)(2 * i + 1) * limb_stride);
      mac128(a0l, a0h, r0, d);
      mac128(a1l, a1h, r1, d);
      if (++cnt == 255) {
        a0l = reduce128(a0h, a0l, q, bar, r64, r64s);
        a1l = reduce128(a1h, a1l, q, bar, r64, r64s);
        a0h = a1h = 0;
        cnt = 0;
      }
    }
    uint64_t s0 = reduce128(a0h, a0l, q, bar, r64, r64s);
    uint64_t s1 = reduce128(a1h, a1l, q, bar, r64, r64s);
    Sa[(size_t)(jj * 2 + 0) * limb_stride] = s0;
    Sa[(size_t)(jj * 2 + 1) * limb_stride] = s1;
  }
}
}  // namespace

hd_status mac_run(hd_context *c, const uint64_t *D, const uint64_t *r, uint64_t *S, uint32_t A_loc, int n1, int N,
                  const std::vector<int32_t> &js) {
  if (js.empty() || A_loc == 0) return HD_OK;
  const int jmin = js.front(), nj = (int)js.size();
  dim3 grid((c->n + MAC_TPB - 1) / MAC_TPB, c->L, A_loc);
  mac_kernel<<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt); ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}
