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

#include <cstdlib>

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
// Full-range variant (n1 | N/2, so every giant step uses all n1 baby steps): baby
// step i outer, JT giant steps inner with their 128-bit accumulators in registers.
// Each i issues JT independent coalesced D loads (memory-level parallelism) and
// reuses the two r[i] words JT times.  blockIdx.x = aggregate (fastest), so the
// CTAs resident at any time share few (limb, tile) r tiles -> r stays in L2 and
// the D stream is the only HBM traffic.
template <int JT>
__global__ void __launch_bounds__(MAC_TPB) mac_full_kernel(const uint64_t *__restrict__ D,
                                                           const uint64_t *__restrict__ r, uint64_t *__restrict__ S,
                                                           int n1, int N, int L, int logn, int jmin, int nj,
                                                           ModTab mt) {
  const int n = 1 << logn;
  const uint32_t a = blockIdx.x;
  const uint32_t t = blockIdx.y * MAC_TPB + threadIdx.x;
  const int ngrp = nj / JT;
  const int m = blockIdx.z / ngrp, jg = blockIdx.z % ngrp;
  const size_t ls = (size_t)L * n;
  const uint64_t *Da = D + (size_t)a * N * ls + (size_t)m * n + t;
  const uint64_t *rr = r + (size_t)m * n + t;
  int kb[JT];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) kb[jj] = (jmin + jg * JT + jj) * n1;
  uint64_t acc[JT][4];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) acc[jj][0] = acc[jj][1] = acc[jj][2] = acc[jj][3] = 0;
  for (int i = 0; i < n1; i++) {
    const uint64_t r0 = __ldg(rr + (size_t)(2 * i) * ls);
    const uint64_t r1 = __ldg(rr + (size_t)(2 * i + 1) * ls);
    uint64_t d[JT];
#pragma unroll
    for (int jj = 0; jj < JT; jj++) d[jj] = __ldcs(Da + (size_t)((kb[jj] + i) & (N - 1)) * ls);
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      mac128(acc[jj][0], acc[jj][1], r0, d[jj]);
      mac128(acc[jj][2], acc[jj][3], r1, d[jj]);
    }
  }
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  uint64_t *Sa = S + (size_t)a * nj * 2 * ls + (size_t)m * n + t;
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    const size_t jx = (size_t)(jg * JT + jj);
    Sa[(jx * 2 + 0) * ls] = reduce128(acc[jj][1], acc[jj][0], q, bar, r64, r64s);
    Sa[(jx * 2 + 1) * ls] = reduce128(acc[jj][3], acc[jj][2], q, bar, r64, r64s);
  }
}
// ---- carry-save variant (q < 2^60, n1 <= 128) ----------------------------------------
// a = a1 2^32 + a0, b = b1 2^32 + b0 (a1, b1 < 2^28).  Per product:
//   lo  += a0 b0          (64-bit add, carry counted in cnt)
//   mid += a0 b1 + a1 b0  (mad.wide into 64 bits: each term < 2^60, folded every 8 i)
//   hi  += a1 b1          (< 2^56 per term)
// i.e. 4 IMAD.WIDE + 3 IADD per product instead of a full 64x64->128 multiply and a
// 128-bit add.  value = lo + mid 2^32 + (hi + cnt) 2^64, reduced once per (a, j).
struct CsAcc {
  uint64_t lo, mid, hi;
  uint32_t cnt;
};
__device__ __forceinline__ void cs_mac(CsAcc &A, uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
  asm("{\n\t.reg .u64 t;\n\t"
      "mul.wide.u32 t, %4, %6;\n\t"
      "add.cc.u64 %0, %0, t;\n\t"
      "addc.u32 %3, %3, 0;\n\t"
      "mad.wide.u32 %1, %4, %7, %1;\n\t"
      "mad.wide.u32 %1, %5, %6, %1;\n\t"
      "mad.wide.u32 %2, %5, %7, %2;\n\t"
      "}"
      : "+l"(A.lo), "+l"(A.mid), "+l"(A.hi), "+r"(A.cnt)
      : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void cs_fold(CsAcc &A) {
  const uint64_t ml = A.mid << 32, mh = A.mid >> 32;
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+l"(A.lo), "+r"(A.cnt) : "l"(ml));
  A.hi += mh;
  A.mid = 0;
}
__device__ __forceinline__ uint64_t ld_stream(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.global.cs.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

template <int JT>
__global__ void __launch_bounds__(MAC_TPB) mac_cs_kernel(const uint64_t *__restrict__ D,
                                                         const uint64_t *__restrict__ r, uint64_t *__restrict__ S,
                                                         int n1, int N, int L, int logn, int jmin, int nj, ModTab mt) {
  const int n = 1 << logn;
  const uint32_t a = blockIdx.x;
  const uint32_t t = blockIdx.y * MAC_TPB + threadIdx.x;
  const int ngrp = nj / JT;
  const int m = blockIdx.z / ngrp, jg = blockIdx.z % ngrp;
  const size_t ls = (size_t)L * n;
  const uint64_t *Da = D + (size_t)a * N * ls + (size_t)m * n + t;
  const uint64_t *rr = r + (size_t)m * n + t;
  const uint64_t *p[JT];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) p[jj] = Da + (size_t)(((jmin + jg * JT + jj) * n1) & (N - 1)) * ls;
  CsAcc acc[JT][2];
#pragma unroll
  for (int jj = 0; jj < JT; jj++)
#pragma unroll
    for (int q2 = 0; q2 < 2; q2++) acc[jj][q2] = CsAcc{0, 0, 0, 0};
  for (int i0 = 0; i0 < n1; i0 += 8) {
#pragma unroll 2
    for (int i = i0; i < i0 + 8 && i < n1; i++) {
      uint64_t d[JT];
#pragma unroll
      for (int jj = 0; jj < JT; jj++) d[jj] = ld_stream(p[jj] + (size_t)i * ls);
      const uint64_t r0 = __ldg(rr + (size_t)(2 * i) * ls);
      const uint64_t r1 = __ldg(rr + (size_t)(2 * i + 1) * ls);
      const uint32_t r00 = (uint32_t)r0, r01 = (uint32_t)(r0 >> 32), r10 = (uint32_t)r1, r11 = (uint32_t)(r1 >> 32);
#pragma unroll
      for (int jj = 0; jj < JT; jj++) {
        const uint32_t b0 = (uint32_t)d[jj], b1 = (uint32_t)(d[jj] >> 32);
        cs_mac(acc[jj][0], r00, r01, b0, b1);
        cs_mac(acc[jj][1], r10, r11, b0, b1);
      }
    }
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      cs_fold(acc[jj][0]);
      cs_fold(acc[jj][1]);
    }
  }
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  uint64_t *Sa = S + (size_t)a * nj * 2 * ls + (size_t)m * n + t;
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    const size_t jx = (size_t)(jg * JT + jj);
#pragma unroll
    for (int q2 = 0; q2 < 2; q2++) {
      const CsAcc &A = acc[jj][q2];
      Sa[(jx * 2 + q2) * ls] = reduce128(A.hi + A.cnt, A.lo, q, bar, r64, r64s);
    }
  }
}
// ---- carry-save, software-pipelined loads: the JT loads of baby step i+1 are issued
// before the arithmetic of step i (2 JT loads in flight per thread), running pointers. --
template <int JT, bool FLUSH = false>
__global__ void __launch_bounds__(MAC_TPB) mac_cs2_kernel(const uint64_t *__restrict__ D,
                                                          const uint64_t *__restrict__ r, uint64_t *__restrict__ S,
                                                          int n1, int N, int L, int logn, int jmin, int nj,
                                                          ModTab mt) {
  const int n = 1 << logn;
  const uint32_t a = blockIdx.x;
  const uint32_t t = blockIdx.y * MAC_TPB + threadIdx.x;
  const int ngrp = nj / JT;
  const int m = blockIdx.z / ngrp, jg = blockIdx.z % ngrp;
  const size_t ls = (size_t)L * n;
  const uint64_t *Da = D + (size_t)a * N * ls + (size_t)m * n + t;
  const uint64_t *rr = r + (size_t)m * n + t;
  const uint64_t *p[JT];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) p[jj] = Da + (size_t)(((jmin + jg * JT + jj) * n1) & (N - 1)) * ls;
  CsAcc acc[JT][2];
  uint64_t part[JT][2];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    acc[jj][0] = acc[jj][1] = CsAcc{0, 0, 0, 0};
    part[jj][0] = part[jj][1] = 0;
  }
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  uint64_t d[JT], dn[JT];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    d[jj] = ld_stream(p[jj]);
    p[jj] += ls;
  }
  uint64_t r0 = __ldg(rr), r1 = __ldg(rr + ls);
  for (int i = 0; i < n1; i++) {
    const bool more = i + 1 < n1;
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      dn[jj] = more ? ld_stream(p[jj]) : 0;
      p[jj] += ls;
    }
    const uint64_t rn0 = more ? __ldg(rr + (size_t)(2 * i + 2) * ls) : 0;
    const uint64_t rn1 = more ? __ldg(rr + (size_t)(2 * i + 3) * ls) : 0;
    const uint32_t r00 = (uint32_t)r0, r01 = (uint32_t)(r0 >> 32), r10 = (uint32_t)r1, r11 = (uint32_t)(r1 >> 32);
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      const uint32_t b0 = (uint32_t)d[jj], b1 = (uint32_t)(d[jj] >> 32);
      cs_mac(acc[jj][0], r00, r01, b0, b1);
      cs_mac(acc[jj][1], r10, r11, b0, b1);
      d[jj] = dn[jj];
    }
    r0 = rn0;
    r1 = rn1;
    if ((i & 7) == 7) {
#pragma unroll
      for (int jj = 0; jj < JT; jj++) {
        cs_fold(acc[jj][0]);
        cs_fold(acc[jj][1]);
      }
    }
    if (FLUSH && (i & 127) == 127 && more) {  // n1 > 128: bank the carry-save sums every 128 terms
#pragma unroll
      for (int jj = 0; jj < JT; jj++)
#pragma unroll
        for (int q2 = 0; q2 < 2; q2++) {
          CsAcc &A = acc[jj][q2];
          part[jj][q2] = addmod(part[jj][q2], reduce128(A.hi + A.cnt, A.lo, q, bar, r64, r64s), q);
          A = CsAcc{0, 0, 0, 0};
        }
    }
  }
  uint64_t *Sa = S + (size_t)a * nj * 2 * ls + (size_t)m * n + t;
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    const size_t jx = (size_t)(jg * JT + jj);
#pragma unroll
    for (int q2 = 0; q2 < 2; q2++) {
      CsAcc &A = acc[jj][q2];
      cs_fold(A);
      Sa[(jx * 2 + q2) * ls] = addmod(part[jj][q2], reduce128(A.hi + A.cnt, A.lo, q, bar, r64, r64s), q);
    }
  }
}

// ---- carry-save with a PD-deep register prefetch ring: the loads of baby steps
// i+1 .. i+PD are in flight while step i is accumulated (JT PD loads per thread). --------
template <int JT, int PD>
__global__ void __launch_bounds__(MAC_TPB) mac_cs5_kernel(const uint64_t *__restrict__ D,
                                                          const uint64_t *__restrict__ r, uint64_t *__restrict__ S,
                                                          int n1, int N, int L, int logn, int jmin, int nj,
                                                          ModTab mt) {
  const int n = 1 << logn;
  const uint32_t a = blockIdx.x;
  const uint32_t t = blockIdx.y * MAC_TPB + threadIdx.x;
  const int ngrp = nj / JT;
  const int m = blockIdx.z / ngrp, jg = blockIdx.z % ngrp;
  const size_t ls = (size_t)L * n;
  const uint64_t *Da = D + (size_t)a * N * ls + (size_t)m * n + t;
  const uint64_t *rr = r + (size_t)m * n + t;
  const uint64_t *p[JT];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) p[jj] = Da + (size_t)(((jmin + jg * JT + jj) * n1) & (N - 1)) * ls;
  CsAcc acc[JT][2];
  uint64_t part[JT][2];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    acc[jj][0] = acc[jj][1] = CsAcc{0, 0, 0, 0};
    part[jj][0] = part[jj][1] = 0;
  }
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  uint64_t d[PD][JT], rv[PD][2];
#pragma unroll
  for (int s = 0; s < PD; s++) {
#pragma unroll
    for (int jj = 0; jj < JT; jj++) d[s][jj] = s < n1 ? ld_stream(p[jj] + (size_t)s * ls) : 0;
    rv[s][0] = s < n1 ? __ldg(rr + (size_t)(2 * s) * ls) : 0;
    rv[s][1] = s < n1 ? __ldg(rr + (size_t)(2 * s + 1) * ls) : 0;
  }
  for (int i0 = 0; i0 < n1; i0 += PD) {
#pragma unroll
    for (int s = 0; s < PD; s++) {
      const int i = i0 + s;
      if (i < n1) {
        const uint64_t r0 = rv[s][0], r1 = rv[s][1];
        uint64_t dc[JT];
#pragma unroll
        for (int jj = 0; jj < JT; jj++) dc[jj] = d[s][jj];
        const int nx = i + PD;  // refill this slot with baby step i + PD
        if (nx < n1) {
#pragma unroll
          for (int jj = 0; jj < JT; jj++) d[s][jj] = ld_stream(p[jj] + (size_t)nx * ls);
          rv[s][0] = __ldg(rr + (size_t)(2 * nx) * ls);
          rv[s][1] = __ldg(rr + (size_t)(2 * nx + 1) * ls);
        }
        const uint32_t r00 = (uint32_t)r0, r01 = (uint32_t)(r0 >> 32), r10 = (uint32_t)r1, r11 = (uint32_t)(r1 >> 32);
#pragma unroll
        for (int jj = 0; jj < JT; jj++) {
          const uint32_t b0 = (uint32_t)dc[jj], b1 = (uint32_t)(dc[jj] >> 32);
          cs_mac(acc[jj][0], r00, r01, b0, b1);
          cs_mac(acc[jj][1], r10, r11, b0, b1);
        }
        if ((i & 7) == 7) {
#pragma unroll
          for (int jj = 0; jj < JT; jj++) {
            cs_fold(acc[jj][0]);
            cs_fold(acc[jj][1]);
          }
        }
        if ((i & 127) == 127 && i + 1 < n1) {  // n1 > 128: bank the carry-save sums every 128 terms
#pragma unroll
          for (int jj = 0; jj < JT; jj++)
#pragma unroll
            for (int q2 = 0; q2 < 2; q2++) {
              CsAcc &A = acc[jj][q2];
              part[jj][q2] = addmod(part[jj][q2], reduce128(A.hi + A.cnt, A.lo, q, bar, r64, r64s), q);
              A = CsAcc{0, 0, 0, 0};
            }
        }
      }
    }
  }
  uint64_t *Sa = S + (size_t)a * nj * 2 * ls + (size_t)m * n + t;
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    const size_t jx = (size_t)(jg * JT + jj);
#pragma unroll
    for (int q2 = 0; q2 < 2; q2++) {
      CsAcc &A = acc[jj][q2];
      cs_fold(A);
      Sa[(jx * 2 + q2) * ls] = addmod(part[jj][q2], reduce128(A.hi + A.cnt, A.lo, q, bar, r64, r64s), q);
    }
  }
}

// ---- two coefficients per thread (128-bit loads), 6-instruction carry-save product ------
// lo is kept as two 32-bit words so a0*b0 is added with mad.lo.cc / madc.hi.cc (carry
// into cnt): 2 IMAD + 1 IADD + 3 IMAD.WIDE per product.
struct CsAcc2 {
  uint32_t lo0, lo1;
  uint64_t mid, hi;
  uint32_t cnt;
};
__device__ __forceinline__ void cs2_mac(CsAcc2 &A, uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
  asm("mad.lo.cc.u32 %0, %5, %7, %0;\n\t"
      "madc.hi.cc.u32 %1, %5, %7, %1;\n\t"
      "addc.u32 %4, %4, 0;\n\t"
      "mad.wide.u32 %2, %5, %8, %2;\n\t"
      "mad.wide.u32 %2, %6, %7, %2;\n\t"
      "mad.wide.u32 %3, %6, %8, %3;"
      : "+r"(A.lo0), "+r"(A.lo1), "+l"(A.mid), "+l"(A.hi), "+r"(A.cnt)
      : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void cs2_fold(CsAcc2 &A) {
  asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+r"(A.lo1), "+r"(A.cnt) : "r"((uint32_t)A.mid));
  A.hi += A.mid >> 32;
  A.mid = 0;
}
__device__ __forceinline__ ulonglong2 ld_stream2(const uint64_t *p) {
  ulonglong2 v;
  asm volatile("ld.global.cs.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}

template <int JT>
__global__ void __launch_bounds__(MAC_TPB) mac_cs4_kernel(const uint64_t *__restrict__ D,
                                                          const uint64_t *__restrict__ r, uint64_t *__restrict__ S,
                                                          int n1, int N, int L, int logn, int jmin, int nj,
                                                          ModTab mt) {
  const int n = 1 << logn;
  const uint32_t a = blockIdx.x;
  const uint32_t t = 2 * (blockIdx.y * MAC_TPB + threadIdx.x);
  const int ngrp = nj / JT;
  const int m = blockIdx.z / ngrp, jg = blockIdx.z % ngrp;
  const size_t ls = (size_t)L * n;
  const uint64_t *Da = D + (size_t)a * N * ls + (size_t)m * n + t;
  const uint64_t *rr = r + (size_t)m * n + t;
  const uint64_t *p[JT];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) p[jj] = Da + (size_t)(((jmin + jg * JT + jj) * n1) & (N - 1)) * ls;
  CsAcc2 acc[JT][2][2];  // [jj][poly][coefficient]
#pragma unroll
  for (int jj = 0; jj < JT; jj++)
#pragma unroll
    for (int x = 0; x < 4; x++) acc[jj][x / 2][x % 2] = CsAcc2{0, 0, 0, 0, 0};
  ulonglong2 d[JT], dn[JT];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    d[jj] = ld_stream2(p[jj]);
    p[jj] += ls;
  }
  ulonglong2 r0 = *reinterpret_cast<const ulonglong2 *>(rr), r1 = *reinterpret_cast<const ulonglong2 *>(rr + ls);
  for (int i = 0; i < n1; i++) {
    const bool more = i + 1 < n1;
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      dn[jj] = more ? ld_stream2(p[jj]) : make_ulonglong2(0, 0);
      p[jj] += ls;
    }
    ulonglong2 rn0 = make_ulonglong2(0, 0), rn1 = make_ulonglong2(0, 0);
    if (more) {
      rn0 = __ldg(reinterpret_cast<const ulonglong2 *>(rr + (size_t)(2 * i + 2) * ls));
      rn1 = __ldg(reinterpret_cast<const ulonglong2 *>(rr + (size_t)(2 * i + 3) * ls));
    }
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      cs2_mac(acc[jj][0][0], (uint32_t)r0.x, (uint32_t)(r0.x >> 32), (uint32_t)d[jj].x, (uint32_t)(d[jj].x >> 32));
      cs2_mac(acc[jj][1][0], (uint32_t)r1.x, (uint32_t)(r1.x >> 32), (uint32_t)d[jj].x, (uint32_t)(d[jj].x >> 32));
      cs2_mac(acc[jj][0][1], (uint32_t)r0.y, (uint32_t)(r0.y >> 32), (uint32_t)d[jj].y, (uint32_t)(d[jj].y >> 32));
      cs2_mac(acc[jj][1][1], (uint32_t)r1.y, (uint32_t)(r1.y >> 32), (uint32_t)d[jj].y, (uint32_t)(d[jj].y >> 32));
      d[jj] = dn[jj];
    }
    r0 = rn0;
    r1 = rn1;
    if ((i & 7) == 7) {
#pragma unroll
      for (int jj = 0; jj < JT; jj++)
#pragma unroll
        for (int x = 0; x < 4; x++) cs2_fold(acc[jj][x / 2][x % 2]);
    }
  }
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  uint64_t *Sa = S + (size_t)a * nj * 2 * ls + (size_t)m * n + t;
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    const size_t jx = (size_t)(jg * JT + jj);
#pragma unroll
    for (int p2 = 0; p2 < 2; p2++) {
      uint64_t o[2];
#pragma unroll
      for (int cc = 0; cc < 2; cc++) {
        CsAcc2 &A = acc[jj][p2][cc];
        cs2_fold(A);
        const uint64_t lo = (uint64_t)A.lo0 | ((uint64_t)A.lo1 << 32);
        o[cc] = reduce128(A.hi + A.cnt, lo, q, bar, r64, r64s);
      }
      *reinterpret_cast<ulonglong2 *>(Sa + (jx * 2 + p2) * ls) = make_ulonglong2(o[0], o[1]);
    }
  }
}

// ---- bulk-copy pipelined variant: TMA (cp.async.bulk) ring + carry-save MAC -----------
// The CTA owns (aggregate a, tile of MT = 128 coefficients of limb m, JT giant steps).
// Stage i of the ring holds the JT diagonal rows D[a][k(j,i)][m][tile] (JT x 1 KiB,
// contiguous in HBM) and the two baby-step rows r[i][0/1][m][tile]; one elected thread
// issues the bulk copies, completion is tracked by one mbarrier per slot (expect_tx),
// and NS stages (NS (JT+2) KiB per CTA) are in flight: HBM latency is hidden by
// bytes in flight, not by warps.
constexpr int MT = MAC_TPB;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int JT, int NS>
__global__ void __launch_bounds__(MT) mac_tma_kernel(const uint64_t *__restrict__ D, const uint64_t *__restrict__ r,
                                                     uint64_t *__restrict__ S, int n1, int N, int L, int logn, int jmin,
                                                     int nj, ModTab mt) {
  extern __shared__ __align__(128) uint64_t ring[];  // [NS][JT + 2][MT]
  __shared__ __align__(8) uint64_t full_bar[NS];
  constexpr int ROWS = JT + 2;
  constexpr uint32_t STAGE_BYTES = ROWS * MT * 8;
  const int n = 1 << logn;
  const uint32_t a = blockIdx.x;
  const uint32_t t0 = blockIdx.y * MT;
  const int ngrp = nj / JT;
  const int m = blockIdx.z / ngrp, jg = blockIdx.z % ngrp;
  const size_t ls = (size_t)L * n;
  const uint64_t *Dt = D + (size_t)a * N * ls + (size_t)m * n + t0;
  const uint64_t *rt = r + (size_t)m * n + t0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; s++) mbar_init(&full_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int i, int slot) {
    uint64_t *dst = ring + (size_t)slot * ROWS * MT;
    mbar_expect_tx(&full_bar[slot], STAGE_BYTES);
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      const int k = (((jmin + jg * JT + jj) * n1) & (N - 1)) + i;  // no wrap: n1 | N/2
      bulk_g2s(dst + jj * MT, Dt + (size_t)k * ls, MT * 8, &full_bar[slot]);
    }
    bulk_g2s(dst + JT * MT, rt + (size_t)(2 * i) * ls, MT * 8, &full_bar[slot]);
    bulk_g2s(dst + (JT + 1) * MT, rt + (size_t)(2 * i + 1) * ls, MT * 8, &full_bar[slot]);
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < NS && s < n1; s++) issue(s, s);
  CsAcc acc[JT][2];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) acc[jj][0] = acc[jj][1] = CsAcc{0, 0, 0, 0};
  for (int i = 0; i < n1; i++) {
    const int slot = i % NS;
    mbar_wait(&full_bar[slot], (uint32_t)((i / NS) & 1));
    const uint64_t *st = ring + (size_t)slot * ROWS * MT + threadIdx.x;
    uint64_t d[JT];
#pragma unroll
    for (int jj = 0; jj < JT; jj++) d[jj] = st[jj * MT];
    const uint64_t r0 = st[JT * MT], r1 = st[(JT + 1) * MT];
    __syncthreads();  // every thread has its words of this slot: refill it
    if (threadIdx.x == 0 && i + NS < n1) issue(i + NS, slot);
    const uint32_t r00 = (uint32_t)r0, r01 = (uint32_t)(r0 >> 32), r10 = (uint32_t)r1, r11 = (uint32_t)(r1 >> 32);
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      const uint32_t b0 = (uint32_t)d[jj], b1 = (uint32_t)(d[jj] >> 32);
      cs_mac(acc[jj][0], r00, r01, b0, b1);
      cs_mac(acc[jj][1], r10, r11, b0, b1);
    }
    if ((i & 7) == 7) {
#pragma unroll
      for (int jj = 0; jj < JT; jj++) {
        cs_fold(acc[jj][0]);
        cs_fold(acc[jj][1]);
      }
    }
  }
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  uint64_t *Sa = S + (size_t)a * nj * 2 * ls + (size_t)m * n + t0 + threadIdx.x;
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    const size_t jx = (size_t)(jg * JT + jj);
#pragma unroll
    for (int q2 = 0; q2 < 2; q2++) {
      CsAcc &A = acc[jj][q2];
      cs_fold(A);
      Sa[(jx * 2 + q2) * ls] = reduce128(A.hi + A.cnt, A.lo, q, bar, r64, r64s);
    }
  }
}
// ---- warp-specialised variant: 4 compute warps + 1 producer warp ---------------------
// Same stage contents as mac_tma_kernel, but the producer warp refills a slot as soon as
// the four compute warps have released it (per-slot "empty" mbarrier, one arrival per
// warp), so compute warps never meet at a CTA-wide barrier inside the i loop.
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int JT, int NS>
__global__ void __launch_bounds__(MT + 32) mac_ws_kernel(const uint64_t *__restrict__ D,
                                                         const uint64_t *__restrict__ r, uint64_t *__restrict__ S,
                                                         int n1, int N, int L, int logn, int jmin, int nj, ModTab mt) {
  extern __shared__ __align__(128) uint64_t ring[];  // [NS][JT + 2][MT]
  __shared__ __align__(8) uint64_t full_bar[NS], empty_bar[NS];
  constexpr int ROWS = JT + 2;
  constexpr uint32_t STAGE_BYTES = ROWS * MT * 8;
  constexpr int NCW = MT / 32;  // compute warps
  const int n = 1 << logn;
  const uint32_t a = blockIdx.x;
  const uint32_t t0 = blockIdx.y * MT;
  const int ngrp = nj / JT;
  const int m = blockIdx.z / ngrp, jg = blockIdx.z % ngrp;
  const size_t ls = (size_t)L * n;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; s++) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NCW) {  // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t *Dt = D + (size_t)a * N * ls + (size_t)m * n + t0;
      const uint64_t *rt = r + (size_t)m * n + t0;
      int kb[JT];
#pragma unroll
      for (int jj = 0; jj < JT; jj++) kb[jj] = ((jmin + jg * JT + jj) * n1) & (N - 1);  // no wrap: n1 | N/2
      for (int i = 0; i < n1; i++) {
        const int slot = i % NS;
        if (i >= NS) mbar_wait(&empty_bar[slot], (uint32_t)(((i / NS) - 1) & 1));
        uint64_t *dst = ring + (size_t)slot * ROWS * MT;
        mbar_expect_tx(&full_bar[slot], STAGE_BYTES);
#pragma unroll
        for (int jj = 0; jj < JT; jj++) bulk_g2s(dst + jj * MT, Dt + (size_t)(kb[jj] + i) * ls, MT * 8, &full_bar[slot]);
        bulk_g2s(dst + JT * MT, rt + (size_t)(2 * i) * ls, MT * 8, &full_bar[slot]);
        bulk_g2s(dst + (JT + 1) * MT, rt + (size_t)(2 * i + 1) * ls, MT * 8, &full_bar[slot]);
      }
    }
    return;
  }
  // ---------------- compute warps ----------------
  CsAcc acc[JT][2];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) acc[jj][0] = acc[jj][1] = CsAcc{0, 0, 0, 0};
  for (int i = 0; i < n1; i++) {
    const int slot = i % NS;
    mbar_wait(&full_bar[slot], (uint32_t)((i / NS) & 1));
    const uint64_t *st = ring + (size_t)slot * ROWS * MT + threadIdx.x;
    uint64_t d[JT];
#pragma unroll
    for (int jj = 0; jj < JT; jj++) d[jj] = st[jj * MT];
    const uint64_t r0 = st[JT * MT], r1 = st[(JT + 1) * MT];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[slot]);
    const uint32_t r00 = (uint32_t)r0, r01 = (uint32_t)(r0 >> 32), r10 = (uint32_t)r1, r11 = (uint32_t)(r1 >> 32);
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      const uint32_t b0 = (uint32_t)d[jj], b1 = (uint32_t)(d[jj] >> 32);
      cs_mac(acc[jj][0], r00, r01, b0, b1);
      cs_mac(acc[jj][1], r10, r11, b0, b1);
    }
    if ((i & 7) == 7) {
#pragma unroll
      for (int jj = 0; jj < JT; jj++) {
        cs_fold(acc[jj][0]);
        cs_fold(acc[jj][1]);
      }
    }
  }
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  uint64_t *Sa = S + (size_t)a * nj * 2 * ls + (size_t)m * n + t0 + threadIdx.x;
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    const size_t jx = (size_t)(jg * JT + jj);
#pragma unroll
    for (int q2 = 0; q2 < 2; q2++) {
      CsAcc &A = acc[jj][q2];
      cs_fold(A);
      Sa[(jx * 2 + q2) * ls] = reduce128(A.hi + A.cnt, A.lo, q, bar, r64, r64s);
    }
  }
}
// ---- persistent warp-specialised variant ------------------------------------------------
// gridDim.x CTAs (a few per SM) walk the flattened work list w = (a, tile, m, jg) with
// the aggregate fastest (consecutive CTAs share the same r tile -> r stays in L2).  The
// producer warp streams stage after stage across work items, so the ring never drains
// between tiles and the per-CTA prologue is paid once.
template <int JT, int NS>
__global__ void __launch_bounds__(MT + 32) mac_pers_kernel(const uint64_t *__restrict__ D,
                                                           const uint64_t *__restrict__ r, uint64_t *__restrict__ S,
                                                           int n1, int N, int L, int logn, int jmin, int nj,
                                                           uint32_t A_loc, ModTab mt) {
  extern __shared__ __align__(128) uint64_t ring[];  // [NS][JT + 2][MT]
  __shared__ __align__(8) uint64_t full_bar[NS], empty_bar[NS];
  constexpr int ROWS = JT + 2;
  constexpr uint32_t STAGE_BYTES = ROWS * MT * 8;
  constexpr int NCW = MT / 32;
  const int n = 1 << logn;
  const size_t ls = (size_t)L * n;
  const int ngrp = nj / JT;
  const uint32_t tiles = n / MT;
  const uint32_t nwork = A_loc * tiles * L * ngrp;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; s++) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto decode = [&](uint32_t w, uint32_t &a, uint32_t &t0, int &m, int &jg) {
    a = w % A_loc;
    uint32_t rest = w / A_loc;
    t0 = (rest % tiles) * MT;
    rest /= tiles;
    m = (int)(rest % L);
    jg = (int)(rest / L);
  };
  if (warp == NCW) {  // ---------------- producer ----------------
    if (lane == 0) {
      uint32_t it = 0;  // global stage counter
      for (uint32_t w = blockIdx.x; w < nwork; w += gridDim.x) {
        uint32_t a, t0;
        int m, jg;
        decode(w, a, t0, m, jg);
        const uint64_t *Dt = D + (size_t)a * N * ls + (size_t)m * n + t0;
        const uint64_t *rt = r + (size_t)m * n + t0;
        for (int i = 0; i < n1; i++, it++) {
          const uint32_t slot = it % NS;
          if (it >= NS) mbar_wait(&empty_bar[slot], ((it / NS) - 1) & 1);
          uint64_t *dst = ring + (size_t)slot * ROWS * MT;
          mbar_expect_tx(&full_bar[slot], STAGE_BYTES);
#pragma unroll
          for (int jj = 0; jj < JT; jj++) {
            const int k = (((jmin + jg * JT + jj) * n1) & (N - 1)) + i;  // no wrap: n1 | N/2
            bulk_g2s(dst + jj * MT, Dt + (size_t)k * ls, MT * 8, &full_bar[slot]);
          }
          bulk_g2s(dst + JT * MT, rt + (size_t)(2 * i) * ls, MT * 8, &full_bar[slot]);
          bulk_g2s(dst + (JT + 1) * MT, rt + (size_t)(2 * i + 1) * ls, MT * 8, &full_bar[slot]);
        }
      }
    }
    return;
  }
  // ---------------- compute warps ----------------
  uint32_t it = 0;
  for (uint32_t w = blockIdx.x; w < nwork; w += gridDim.x) {
    uint32_t a, t0;
    int m, jg;
    decode(w, a, t0, m, jg);
    CsAcc acc[JT][2];
#pragma unroll
    for (int jj = 0; jj < JT; jj++) acc[jj][0] = acc[jj][1] = CsAcc{0, 0, 0, 0};
    for (int i = 0; i < n1; i++, it++) {
      const uint32_t slot = it % NS;
      mbar_wait(&full_bar[slot], (it / NS) & 1);
      const uint64_t *st = ring + (size_t)slot * ROWS * MT + threadIdx.x;
      uint64_t d[JT];
#pragma unroll
      for (int jj = 0; jj < JT; jj++) d[jj] = st[jj * MT];
      const uint64_t r0 = st[JT * MT], r1 = st[(JT + 1) * MT];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_bar[slot]);
      const uint32_t r00 = (uint32_t)r0, r01 = (uint32_t)(r0 >> 32), r10 = (uint32_t)r1, r11 = (uint32_t)(r1 >> 32);
#pragma unroll
      for (int jj = 0; jj < JT; jj++) {
        const uint32_t b0 = (uint32_t)d[jj], b1 = (uint32_t)(d[jj] >> 32);
        cs_mac(acc[jj][0], r00, r01, b0, b1);
        cs_mac(acc[jj][1], r10, r11, b0, b1);
      }
      if ((i & 7) == 7) {
#pragma unroll
        for (int jj = 0; jj < JT; jj++) {
          cs_fold(acc[jj][0]);
          cs_fold(acc[jj][1]);
        }
      }
    }
    const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
    uint64_t *Sa = S + (size_t)a * nj * 2 * ls + (size_t)m * n + t0 + threadIdx.x;
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      const size_t jx = (size_t)(jg * JT + jj);
#pragma unroll
      for (int q2 = 0; q2 < 2; q2++) {
        CsAcc &Ac = acc[jj][q2];
        cs_fold(Ac);
        Sa[(jx * 2 + q2) * ls] = reduce128(Ac.hi + Ac.cnt, Ac.lo, q, bar, r64, r64s);
      }
    }
  }
}
}  // namespace

namespace {
// ---- MAC over the tiled diagonal layout (default): each CTA streams one contiguous
// block D_tiled[a][m][T][jg][i][jj][0..127] (n1 JT KiB), JT giant steps x 128 coefficients,
// carry-save accumulation, PD-deep register prefetch, banked every 128 baby steps. ------
constexpr int TILE = 128;

template <int JT, int PD>
__global__ void __launch_bounds__(TILE) mac_tiled_kernel(const uint64_t *__restrict__ D,
                                                         const uint64_t *__restrict__ r, uint64_t *__restrict__ S,
                                                         int n1, int N, int L, int logn, int nj, ModTab mt) {
  const int n = 1 << logn;
  const uint32_t a = blockIdx.x, T = blockIdx.y;
  const int ngrp = nj / JT;
  const int m = blockIdx.z / ngrp, jg = blockIdx.z % ngrp;
  const size_t ls = (size_t)L * n;
  const uint32_t NT = n / TILE;
  const uint32_t c = threadIdx.x, t = T * TILE + c;
  const uint64_t *Dt = D + (size_t)a * N * ls + ((((size_t)m * NT + T) * ngrp + jg) * n1) * JT * TILE + c;
  const uint64_t *rr = r + (size_t)m * n + t;
  CsAcc acc[JT][2];
  uint64_t part[JT][2];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    acc[jj][0] = acc[jj][1] = CsAcc{0, 0, 0, 0};
    part[jj][0] = part[jj][1] = 0;
  }
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  uint64_t d[PD][JT], rv[PD][2];
#pragma unroll
  for (int s = 0; s < PD; s++) {
#pragma unroll
    for (int jj = 0; jj < JT; jj++) d[s][jj] = s < n1 ? ld_stream(Dt + (size_t)(s * JT + jj) * TILE) : 0;
    rv[s][0] = s < n1 ? __ldg(rr + (size_t)(2 * s) * ls) : 0;
    rv[s][1] = s < n1 ? __ldg(rr + (size_t)(2 * s + 1) * ls) : 0;
  }
  for (int i0 = 0; i0 < n1; i0 += PD) {
#pragma unroll
    for (int s = 0; s < PD; s++) {
      const int i = i0 + s;
      if (i < n1) {
        const uint64_t r0 = rv[s][0], r1 = rv[s][1];
        uint64_t dc[JT];
#pragma unroll
        for (int jj = 0; jj < JT; jj++) dc[jj] = d[s][jj];
        const int nx = i + PD;
        if (nx < n1) {
#pragma unroll
          for (int jj = 0; jj < JT; jj++) d[s][jj] = ld_stream(Dt + (size_t)(nx * JT + jj) * TILE);
          rv[s][0] = __ldg(rr + (size_t)(2 * nx) * ls);
          rv[s][1] = __ldg(rr + (size_t)(2 * nx + 1) * ls);
        }
        const uint32_t r00 = (uint32_t)r0, r01 = (uint32_t)(r0 >> 32), r10 = (uint32_t)r1, r11 = (uint32_t)(r1 >> 32);
#pragma unroll
        for (int jj = 0; jj < JT; jj++) {
          const uint32_t b0 = (uint32_t)dc[jj], b1 = (uint32_t)(dc[jj] >> 32);
          cs_mac(acc[jj][0], r00, r01, b0, b1);
          cs_mac(acc[jj][1], r10, r11, b0, b1);
        }
        if ((i & 7) == 7) {
#pragma unroll
          for (int jj = 0; jj < JT; jj++) {
            cs_fold(acc[jj][0]);
            cs_fold(acc[jj][1]);
          }
        }
        if ((i & 127) == 127 && i + 1 < n1) {
#pragma unroll
          for (int jj = 0; jj < JT; jj++)
#pragma unroll
            for (int q2 = 0; q2 < 2; q2++) {
              CsAcc &A = acc[jj][q2];
              part[jj][q2] = addmod(part[jj][q2], reduce128(A.hi + A.cnt, A.lo, q, bar, r64, r64s), q);
              A = CsAcc{0, 0, 0, 0};
            }
        }
      }
    }
  }
  uint64_t *Sa = S + (size_t)a * nj * 2 * ls + (size_t)m * n + t;
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    const size_t jx = (size_t)(jg * JT + jj);
#pragma unroll
    for (int q2 = 0; q2 < 2; q2++) {
      CsAcc &A = acc[jj][q2];
      cs_fold(A);
      Sa[(jx * 2 + q2) * ls] = addmod(part[jj][q2], reduce128(A.hi + A.cnt, A.lo, q, bar, r64, r64s), q);
    }
  }
}

// Ping-pong variant of the tiled MAC: baby steps in pairs (registers dA / dB), the loads of
// the next pair issued before the arithmetic of the current one, no register rotation.
template <int JT>
__device__ __forceinline__ void mac_step(CsAcc (&acc)[JT][2], const uint64_t (&d)[JT], uint64_t r0, uint64_t r1) {
  const uint32_t r00 = (uint32_t)r0, r01 = (uint32_t)(r0 >> 32), r10 = (uint32_t)r1, r11 = (uint32_t)(r1 >> 32);
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    const uint32_t b0 = (uint32_t)d[jj], b1 = (uint32_t)(d[jj] >> 32);
    cs_mac(acc[jj][0], r00, r01, b0, b1);
    cs_mac(acc[jj][1], r10, r11, b0, b1);
  }
}

template <int JT, bool FLUSH = false>
__global__ void __launch_bounds__(TILE) mac_tiled2_kernel(const uint64_t *__restrict__ D,
                                                          const uint64_t *__restrict__ r, uint64_t *__restrict__ S,
                                                          int n1, int N, int L, int logn, int nj, ModTab mt) {
  const int n = 1 << logn;
  const uint32_t a = blockIdx.x, T = blockIdx.y;
  const int ngrp = nj / JT;
  const int m = blockIdx.z / ngrp, jg = blockIdx.z % ngrp;
  const size_t ls = (size_t)L * n;
  const uint32_t NT = n / TILE;
  const uint32_t c = threadIdx.x, t = T * TILE + c;
  const uint64_t *Dt = D + (size_t)a * N * ls + ((((size_t)m * NT + T) * ngrp + jg) * n1) * JT * TILE + c;
  const uint64_t *rr = r + (size_t)m * n + t;
  CsAcc acc[JT][2];
  uint64_t part[JT][2];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    acc[jj][0] = acc[jj][1] = CsAcc{0, 0, 0, 0};
    part[jj][0] = part[jj][1] = 0;
  }
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  uint64_t dA[JT], dB[JT], rA0, rA1, rB0, rB1;
#pragma unroll
  for (int jj = 0; jj < JT; jj++) dA[jj] = ld_stream(Dt + jj * TILE);
  rA0 = __ldg(rr);
  rA1 = __ldg(rr + ls);
  for (int i = 0; i < n1; i += 2) {  // n1 is even here (n1 | N/2, N >= 4)
    const uint64_t *nxt = Dt + (size_t)(i + 1) * JT * TILE;
#pragma unroll
    for (int jj = 0; jj < JT; jj++) dB[jj] = ld_stream(nxt + jj * TILE);
    rB0 = __ldg(rr + (size_t)(2 * i + 2) * ls);
    rB1 = __ldg(rr + (size_t)(2 * i + 3) * ls);
    mac_step<JT>(acc, dA, rA0, rA1);
    if (i + 2 < n1) {
      const uint64_t *nn = Dt + (size_t)(i + 2) * JT * TILE;
#pragma unroll
      for (int jj = 0; jj < JT; jj++) dA[jj] = ld_stream(nn + jj * TILE);
      rA0 = __ldg(rr + (size_t)(2 * i + 4) * ls);
      rA1 = __ldg(rr + (size_t)(2 * i + 5) * ls);
    }
    mac_step<JT>(acc, dB, rB0, rB1);
    if ((i & 7) == 6) {
#pragma unroll
      for (int jj = 0; jj < JT; jj++) {
        cs_fold(acc[jj][0]);
        cs_fold(acc[jj][1]);
      }
    }
    if (FLUSH && (i & 127) == 126 && i + 2 < n1) {
#pragma unroll
      for (int jj = 0; jj < JT; jj++)
#pragma unroll
        for (int q2 = 0; q2 < 2; q2++) {
          CsAcc &A = acc[jj][q2];
          part[jj][q2] = addmod(part[jj][q2], reduce128(A.hi + A.cnt, A.lo, q, bar, r64, r64s), q);
          A = CsAcc{0, 0, 0, 0};
        }
    }
  }
  uint64_t *Sa = S + (size_t)a * nj * 2 * ls + (size_t)m * n + t;
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    const size_t jx = (size_t)(jg * JT + jj);
#pragma unroll
    for (int q2 = 0; q2 < 2; q2++) {
      CsAcc &A = acc[jj][q2];
      cs_fold(A);
      Sa[(jx * 2 + q2) * ls] = addmod(part[jj][q2], reduce128(A.hi + A.cnt, A.lo, q, bar, r64, r64s), q);
    }
  }
}

// dst (tiled) <- src [k][m][coef]; one thread per destination element
__global__ void tile_kernel(const uint64_t *__restrict__ src, uint64_t *__restrict__ dst, int N, int L, int logn,
                            int n1, int jmin, int nj, int JT) {
  const size_t total = (size_t)N * L << logn;
  const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int n = 1 << logn, NT = n / TILE, ngrp = nj / JT;
  size_t x = idx;
  const int cc = (int)(x % TILE);
  x /= TILE;
  const int jj = (int)(x % JT);
  x /= JT;
  const int i = (int)(x % n1);
  x /= n1;
  const int jg = (int)(x % ngrp);
  x /= ngrp;
  const int T = (int)(x % NT);
  const int m = (int)(x / NT);
  const int j = jmin + jg * JT + jj;
  const int k = (j * n1 + i) & (N - 1);
  dst[idx] = src[((size_t)k * L + m) * n + (size_t)T * TILE + cc];
}

__global__ void untile_kernel(const uint64_t *__restrict__ src, uint64_t *__restrict__ dst, int N, int L, int logn,
                              int n1, int jmin, int nj, int JT, int k) {
  const int n = 1 << logn, NT = n / TILE, ngrp = nj / JT;
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // [m][coef]
  if (e >= (size_t)L * n) return;
  const int m = (int)(e / n), coef = (int)(e % n), T = coef / TILE, cc = coef % TILE;
  // find (j, i) with (j n1 + i) mod N == k
  const int ks = k < N / 2 ? k : k - N;
  const int j = ks >= 0 ? ks / n1 : -((-ks + n1 - 1) / n1);
  const int i = ks - j * n1;
  const int jg = (j - jmin) / JT, jj = (j - jmin) % JT;
  dst[e] = src[(((((size_t)m * NT + T) * ngrp + jg) * n1 + i) * JT + jj) * TILE + cc];
}
}  // namespace

hd_status mac_tile_aggregate(hd_context *c, const uint64_t *src, uint64_t *dst, int N, int n1, int jmin, int nj,
                             int JT) {
  const size_t total = (size_t)N * c->L * c->n;
  tile_kernel<<<(unsigned)((total + 255) / 256), 256, 0, c->stream>>>(src, dst, N, c->L, c->logn, n1, jmin, nj, JT);
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status mac_untile_diagonal(hd_context *c, const uint64_t *src, uint64_t *dst, int N, int n1, int jmin, int nj,
                              int JT, int k) {
  const size_t total = (size_t)c->L * c->n;
  untile_kernel<<<(unsigned)((total + 255) / 256), 256, 0, c->stream>>>(src, dst, N, c->L, c->logn, n1, jmin, nj, JT,
                                                                         k);
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status mac_run(hd_context *c, const uint64_t *D, const uint64_t *r, uint64_t *S, uint32_t A_loc, int n1, int N,
                  const std::vector<int32_t> &js, bool tiled, int tile_jt) {
  if (js.empty() || A_loc == 0) return HD_OK;
  const int jmin = js.front(), nj = (int)js.size();
  if (tiled) {
    const char *pd = getenv("HD_MAC_PD");
    const int PD = pd ? atoi(pd) : 0;
    dim3 grid(A_loc, c->n / TILE, c->L * (nj / tile_jt));
    if (n1 % 2 == 0 && PD == 0) {  // default: ping-pong pairs
      const bool fl = n1 > 128;
      if (tile_jt == 2 && !fl)
        mac_tiled2_kernel<2, false><<<grid, TILE, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, nj, c->mt);
      else if (tile_jt == 2)
        mac_tiled2_kernel<2, true><<<grid, TILE, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, nj, c->mt);
      else if (!fl)
        mac_tiled2_kernel<1, false><<<grid, TILE, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, nj, c->mt);
      else
        mac_tiled2_kernel<1, true><<<grid, TILE, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, nj, c->mt);
    } else if (tile_jt == 2) {
      if (PD >= 4) mac_tiled_kernel<2, 4><<<grid, TILE, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, nj, c->mt);
      else if (PD >= 2) mac_tiled_kernel<2, 2><<<grid, TILE, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, nj, c->mt);
      else mac_tiled_kernel<2, 1><<<grid, TILE, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, nj, c->mt);
    } else {
      mac_tiled_kernel<1, 2><<<grid, TILE, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, nj, c->mt);
    }
    ++c->launches;
    HD_CUDA(cudaGetLastError());
    return HD_OK;
  }
  const bool full = (N / 2) % n1 == 0 && n1 <= 256 && c->n % MAC_TPB == 0;
  bool small_q = true;
  for (int l = 0; l < c->L; l++) small_q = small_q && c->mod[l] < (1ull << 60);
  const char *force = getenv("HD_MAC_VARIANT");
  const bool use_cs = full && small_q && n1 <= 128 && nj % 4 == 0 && !(force && force[0] == 'f');
  // variants: 3 (default) carry-save, JT = 2, software-pipelined loads; 2 same with JT = 4;
  // c carry-save JT = 4; w / p / q / t bulk-copy (TMA) rings; f 128-bit accumulators
  const char v = force ? force[0] : '3';
  const bool use_tma = use_cs && (v == 't' || v == 'w');
  const bool use_ws = use_cs && v == 'w';
  const bool use_pers = use_cs && (v == 'p' || v == 'q');
  if (use_cs && (v == '6' || v == '7' || v == '8') && nj % 2 == 0) {
    dim3 grid(A_loc, c->n / MAC_TPB, c->L * (nj / 2));
    if (v == '6') mac_cs5_kernel<2, 2><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
    else if (v == '7') mac_cs5_kernel<2, 4><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
    else mac_cs5_kernel<2, 8><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
  } else if (use_cs && (v == '4' || v == '5') && c->n % (2 * MAC_TPB) == 0) {
    const int JT = v == '4' ? 2 : 1;
    dim3 grid(A_loc, c->n / (2 * MAC_TPB), c->L * (nj / JT));
    if (JT == 2) mac_cs4_kernel<2><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
    else mac_cs4_kernel<1><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
  } else if (full && small_q && v == '3' && nj % 2 == 0) {  // default (any n1: banked every 128 terms)
    dim3 g2(A_loc, c->n / MAC_TPB, c->L * (nj / 2));
    if (n1 > 128)
      mac_cs2_kernel<2, true><<<g2, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
    else
      mac_cs2_kernel<2, false><<<g2, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
  } else if (use_cs && (v == '2' || v == '3')) {
    dim3 grid(A_loc, c->n / MAC_TPB, c->L * (nj / 4));
    if (v == '2') mac_cs2_kernel<4><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
    else {
      dim3 g2(A_loc, c->n / MAC_TPB, c->L * (nj / 2));
      if (nj % 2) return hd_fail(HD_E_PARAMS, "variant 3 needs an even giant-step count");
      mac_cs2_kernel<2><<<g2, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
    }
  } else if (use_pers) {
    constexpr int JT = 4, NS = 12;
    const size_t smem = (size_t)NS * (JT + 2) * MT * 8;
    static bool attr_p = false;
    if (!attr_p) {
      cudaFuncSetAttribute(mac_pers_kernel<JT, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr_p = true;
    }
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c->device);
    const int per_sm = v == 'q' ? 2 : 3;
    mac_pers_kernel<JT, NS><<<dev_sms * per_sm, MAC_TPB + 32, smem, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin,
                                                                                  nj, A_loc, c->mt);
  } else if (use_ws) {
    constexpr int JT = 4, NS = 12;
    const size_t smem = (size_t)NS * (JT + 2) * MT * 8;
    static bool attr_ws = false;
    if (!attr_ws) {
      cudaFuncSetAttribute(mac_ws_kernel<JT, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr_ws = true;
    }
    dim3 grid(A_loc, c->n / MAC_TPB, c->L * (nj / JT));
    mac_ws_kernel<JT, NS><<<grid, MAC_TPB + 32, smem, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
  } else if (use_tma) {
    constexpr int JT = 4, NS = 8;
    const size_t smem = (size_t)NS * (JT + 2) * MT * 8;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(mac_tma_kernel<JT, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    dim3 grid(A_loc, c->n / MAC_TPB, c->L * (nj / JT));
    mac_tma_kernel<JT, NS><<<grid, MAC_TPB, smem, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
  } else if (use_cs) {
    dim3 grid(A_loc, c->n / MAC_TPB, c->L * (nj / 4));
    mac_cs_kernel<4><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
  } else if (full && nj % 8 == 0) {
    dim3 grid(A_loc, c->n / MAC_TPB, c->L * (nj / 8));
    mac_full_kernel<8><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
  } else if (full && nj % 4 == 0) {
    dim3 grid(A_loc, c->n / MAC_TPB, c->L * (nj / 4));
    mac_full_kernel<4><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
  } else {
    dim3 grid((c->n + MAC_TPB - 1) / MAC_TPB, c->L, A_loc);
    mac_kernel<<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
  }
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}
