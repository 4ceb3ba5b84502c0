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
                                                      int n1, int N, int L, int logn, int jmin, int nj, ModTab mt,
                                                      int flat) {
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
    // replicated: P:L206-207; flat (R27): diagonals j n1 + i < N
    int i_lo = flat ? 0 : -j * n1 - N / 2;
    if (i_lo < 0) i_lo = 0;
    int i_hi = flat ? N - 1 - j * n1 : N / 2 - 1 - j * n1;
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

// ---- streaming kernel (the default whenever every giant step uses all n1 baby steps) --
// Baby step i outer, JT giant steps inner: each i issues JT coalesced D loads and
// reuses the two r[i] words JT times; the loads of step i+1 are issued before the
// arithmetic of step i (software pipelining).  blockIdx.x = aggregate (fastest), so the
// CTAs resident at any time share few (limb, tile) r tiles: r stays in L2 and the D
// stream is the only HBM traffic.  FLUSH (n1 > 128) banks the carry-save sums every
// 128 terms so value < 2^128 holds for n1 up to 256.
// Measured alternatives that lost on B200 at 2^20 x 512 (tools/mac_sweep.py, DESIGN.md
// section 5): 128-bit accumulators; JT = 4 or 8 (register pressure); deeper register
// prefetch; cp.async / TMA shared-memory rings (with and without warp specialisation);
// a tile-contiguous D layout; split 30-bit operands.
template <int JT, bool FLUSH = false>
__global__ void __launch_bounds__(MAC_TPB) mac_cs_kernel(const uint64_t *__restrict__ D,
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

// ---- encrypted diagonals (NEXT-1, R26): degree-2 MAC ---------------------------------
// S_{a,j} = sum_i r[i] (x) Dct[a][k(j,i)], the tensor of (r0, r1) and
// (D0, D1): d0 += r0 D0, d1 += r0 D1 + r1 D0, d2 += r1 D1, each in a carry-save
// accumulator (folded every 4 steps: d1 takes 4 mid terms per step), banked into a
// reduced partial sum every 64 steps so any n1 and partial giant-step ranges are safe.
// One (a, j, limb, 128-coefficient tile) per CTA; S: [a][j][3][L][n].
__global__ void __launch_bounds__(MAC_TPB) mac_ct_kernel(const uint64_t *__restrict__ D,
                                                          const uint64_t *__restrict__ r, uint64_t *__restrict__ S,
                                                          int n1, int N, int L, int logn, int jmin, int nj,
                                                          ModTab mt, int flat, int njs) {
  const int n = 1 << logn;
  const uint32_t a = blockIdx.x;
  const uint32_t t = blockIdx.y * MAC_TPB + threadIdx.x;
  const int m = blockIdx.z / nj, jj = blockIdx.z % nj;
  const int j = jmin + jj;
  const size_t ls = (size_t)L * n, ds = 2 * ls;
  const uint64_t *Da = D + (size_t)a * N * ds + (size_t)m * n + t;
  const uint64_t *rr = r + (size_t)m * n + t;
  const int i_lo = flat ? 0 : max(0, -j * n1 - N / 2);
  const int i_hi = flat ? min(n1 - 1, N - 1 - j * n1) : min(n1 - 1, N / 2 - 1 - j * n1);
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  CsAcc acc[3] = {CsAcc{0, 0, 0, 0}, CsAcc{0, 0, 0, 0}, CsAcc{0, 0, 0, 0}};
  uint64_t part[3] = {0, 0, 0};
  auto bank = [&]() {
#pragma unroll
    for (int e = 0; e < 3; e++) {
      cs_fold(acc[e]);
      part[e] = addmod(part[e], reduce128(acc[e].hi + acc[e].cnt, acc[e].lo, q, bar, r64, r64s), q);
      acc[e] = CsAcc{0, 0, 0, 0};
    }
  };
  for (int i = i_lo, c = 0; i <= i_hi; i++, c++) {
    const int k = (j * n1 + i) & (N - 1);
    const uint64_t *dk = Da + (size_t)k * ds;
    const uint64_t d0 = ld_stream(dk), d1 = ld_stream(dk + ls);
    const uint64_t r0 = __ldg(rr + (size_t)(2 * i) * ls), r1 = __ldg(rr + (size_t)(2 * i + 1) * ls);
    const uint32_t r00 = (uint32_t)r0, r01 = (uint32_t)(r0 >> 32), r10 = (uint32_t)r1, r11 = (uint32_t)(r1 >> 32);
    const uint32_t a00 = (uint32_t)d0, a01 = (uint32_t)(d0 >> 32), a10 = (uint32_t)d1, a11 = (uint32_t)(d1 >> 32);
    cs_mac(acc[0], r00, r01, a00, a01);
    cs_mac(acc[1], r00, r01, a10, a11);
    cs_mac(acc[1], r10, r11, a00, a01);
    cs_mac(acc[2], r10, r11, a10, a11);
    if ((c & 3) == 3) {
      cs_fold(acc[0]);
      cs_fold(acc[1]);
      cs_fold(acc[2]);
    }
    if ((c & 63) == 63) bank();
  }
  bank();
  uint64_t *Sa = S + ((size_t)a * njs + jj) * 3 * ls + (size_t)m * n + t;  // njs: giant steps in S's layout
#pragma unroll
  for (int e = 0; e < 3; e++) Sa[(size_t)e * ls] = part[e];
}

// Streaming variant for the full-range case (every giant step uses all n1 baby steps,
// n1 | N/2): running pointers and the loads of step i+1 issued before the arithmetic of
// step i, as in mac_cs_kernel.  Grid (A_loc, n / 128, L nj).
template <int JT>
__global__ void __launch_bounds__(MAC_TPB) mac_ct_stream_kernel(const uint64_t *__restrict__ D,
                                                                 const uint64_t *__restrict__ r,
                                                                 uint64_t *__restrict__ S, int n1, int N, int L,
                                                                 int logn, int jmin, int nj, ModTab mt, int njs) {
  const int n = 1 << logn;
  const uint32_t a = blockIdx.x;
  const uint32_t t = blockIdx.y * MAC_TPB + threadIdx.x;
  const int ngrp = nj / JT;
  const int m = blockIdx.z / ngrp, jg = blockIdx.z % ngrp;
  const size_t ls = (size_t)L * n, ds = 2 * ls;
  const uint64_t *Da = D + (size_t)a * N * ds + (size_t)m * n + t;
  const uint64_t *p[JT];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) p[jj] = Da + (size_t)(((jmin + jg * JT + jj) * n1) & (N - 1)) * ds;
  const uint64_t *rr = r + (size_t)m * n + t;
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  CsAcc acc[JT][3];
  uint64_t part[JT][3];
#pragma unroll
  for (int jj = 0; jj < JT; jj++)
#pragma unroll
    for (int e = 0; e < 3; e++) {
      acc[jj][e] = CsAcc{0, 0, 0, 0};
      part[jj][e] = 0;
    }
  uint64_t d0[JT], d1[JT];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    d0[jj] = ld_stream(p[jj]);
    d1[jj] = ld_stream(p[jj] + ls);
    p[jj] += ds;
  }
  uint64_t r0 = __ldg(rr), r1 = __ldg(rr + ls);
  for (int i = 0; i < n1; i++) {
    const bool more = i + 1 < n1;
    uint64_t dn0[JT], dn1[JT];
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      dn0[jj] = more ? ld_stream(p[jj]) : 0;
      dn1[jj] = more ? ld_stream(p[jj] + ls) : 0;
      p[jj] += ds;
    }
    const uint64_t rn0 = more ? __ldg(rr + (size_t)(2 * i + 2) * ls) : 0;
    const uint64_t rn1 = more ? __ldg(rr + (size_t)(2 * i + 3) * ls) : 0;
    const uint32_t r00 = (uint32_t)r0, r01 = (uint32_t)(r0 >> 32), r10 = (uint32_t)r1, r11 = (uint32_t)(r1 >> 32);
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      const uint32_t a00 = (uint32_t)d0[jj], a01 = (uint32_t)(d0[jj] >> 32);
      const uint32_t a10 = (uint32_t)d1[jj], a11 = (uint32_t)(d1[jj] >> 32);
      cs_mac(acc[jj][0], r00, r01, a00, a01);
      cs_mac(acc[jj][1], r00, r01, a10, a11);
      cs_mac(acc[jj][1], r10, r11, a00, a01);
      cs_mac(acc[jj][2], r10, r11, a10, a11);
      d0[jj] = dn0[jj];
      d1[jj] = dn1[jj];
    }
    r0 = rn0;
    r1 = rn1;
    if ((i & 3) == 3) {
#pragma unroll
      for (int jj = 0; jj < JT; jj++)
#pragma unroll
        for (int e = 0; e < 3; e++) cs_fold(acc[jj][e]);
    }
    if ((i & 63) == 63) {
#pragma unroll
      for (int jj = 0; jj < JT; jj++)
#pragma unroll
        for (int e = 0; e < 3; e++) {
          cs_fold(acc[jj][e]);
          part[jj][e] = addmod(part[jj][e], reduce128(acc[jj][e].hi + acc[jj][e].cnt, acc[jj][e].lo, q, bar, r64,
                                                      r64s), q);
          acc[jj][e] = CsAcc{0, 0, 0, 0};
        }
    }
  }
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    uint64_t *Sa = S + ((size_t)a * njs + jg * JT + jj) * 3 * ls + (size_t)m * n + t;
#pragma unroll
    for (int e = 0; e < 3; e++) {
      cs_fold(acc[jj][e]);
      Sa[(size_t)e * ls] = addmod(part[jj][e], reduce128(acc[jj][e].hi + acc[jj][e].cnt, acc[jj][e].lo, q, bar, r64,
                                                         r64s), q);
    }
  }
}
// ---- query batching (NEXT-4): one D stream serves QB queries ---------------------------
// As mac_cs_kernel with one giant step per thread, but every diagonal word loaded from HBM
// is multiplied into the baby steps of QB queries (r: [QB][n1][2][L][n], S: [QB][A][nj][2][L][n]):
// the D bytes per query drop QB-fold and the kernel turns from HBM- to issue-bound.
template <int QB, int JT, bool FLUSH>
__global__ void __launch_bounds__(MAC_TPB) mac_cs_batch_kernel(const uint64_t *__restrict__ D,
                                                               const uint64_t *__restrict__ r,
                                                               uint64_t *__restrict__ S, int n1, int N, int L,
                                                               int logn, int jmin, int nj, uint32_t A, ModTab mt) {
  const int n = 1 << logn;
  const uint32_t a = blockIdx.x;
  const uint32_t t = blockIdx.y * MAC_TPB + threadIdx.x;
  const int ngrp = nj / JT;
  const int m = blockIdx.z / ngrp, jg = blockIdx.z % ngrp;
  const size_t ls = (size_t)L * n, rq = (size_t)n1 * 2 * ls;  // r stride between queries
  const uint64_t *Da = D + (size_t)a * N * ls + (size_t)m * n + t;
  const uint64_t *p[JT];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) p[jj] = Da + (size_t)(((jmin + jg * JT + jj) * n1) & (N - 1)) * ls;
  const uint64_t *rr = r + (size_t)m * n + t;
  CsAcc acc[JT][QB][2];
  uint64_t part[JT][QB][2];
#pragma unroll
  for (int jj = 0; jj < JT; jj++)
#pragma unroll
    for (int b = 0; b < QB; b++) {
      acc[jj][b][0] = acc[jj][b][1] = CsAcc{0, 0, 0, 0};
      part[jj][b][0] = part[jj][b][1] = 0;
    }
  const uint64_t q = mt.q[m], bar = mt.bar[m], r64 = mt.r64[m], r64s = mt.r64s[m];
  // software pipeline: the D words and the QB r pairs of step i+1 are in flight while step i
  // is multiplied (the r loads are L2 hits; without the prefetch the kernel is latency-bound)
  uint64_t d[JT];
#pragma unroll
  for (int jj = 0; jj < JT; jj++) {
    d[jj] = ld_stream(p[jj]);
    p[jj] += ls;
  }
  uint64_t rc[QB][2];
#pragma unroll
  for (int b = 0; b < QB; b++) {
    rc[b][0] = __ldg(rr + b * rq);
    rc[b][1] = __ldg(rr + b * rq + ls);
  }
  for (int i = 0; i < n1; i++) {
    const bool more = i + 1 < n1;
    uint64_t dn[JT];
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      dn[jj] = more ? ld_stream(p[jj]) : 0;
      p[jj] += ls;
    }
    uint64_t rn[QB][2];
#pragma unroll
    for (int b = 0; b < QB; b++) {
      const uint64_t *rb = rr + b * rq + (size_t)(2 * i + 2) * ls;
      rn[b][0] = more ? __ldg(rb) : 0;
      rn[b][1] = more ? __ldg(rb + ls) : 0;
    }
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      const uint32_t b0 = (uint32_t)d[jj], b1 = (uint32_t)(d[jj] >> 32);
#pragma unroll
      for (int b = 0; b < QB; b++) {
        cs_mac(acc[jj][b][0], (uint32_t)rc[b][0], (uint32_t)(rc[b][0] >> 32), b0, b1);
        cs_mac(acc[jj][b][1], (uint32_t)rc[b][1], (uint32_t)(rc[b][1] >> 32), b0, b1);
      }
      d[jj] = dn[jj];
    }
#pragma unroll
    for (int b = 0; b < QB; b++) {
      rc[b][0] = rn[b][0];
      rc[b][1] = rn[b][1];
    }
    if ((i & 7) == 7) {
#pragma unroll
      for (int jj = 0; jj < JT; jj++)
#pragma unroll
        for (int b = 0; b < QB; b++) {
          cs_fold(acc[jj][b][0]);
          cs_fold(acc[jj][b][1]);
        }
    }
    if (FLUSH && (i & 127) == 127 && more) {
#pragma unroll
      for (int jj = 0; jj < JT; jj++)
#pragma unroll
        for (int b = 0; b < QB; b++)
#pragma unroll
          for (int q2 = 0; q2 < 2; q2++) {
            CsAcc &X = acc[jj][b][q2];
            part[jj][b][q2] = addmod(part[jj][b][q2], reduce128(X.hi + X.cnt, X.lo, q, bar, r64, r64s), q);
            X = CsAcc{0, 0, 0, 0};
          }
    }
  }
#pragma unroll
  for (int jj = 0; jj < JT; jj++)
#pragma unroll
    for (int b = 0; b < QB; b++) {
      uint64_t *Sb = S + (((size_t)b * A + a) * nj + jg * JT + jj) * 2 * ls + (size_t)m * n + t;
#pragma unroll
      for (int q2 = 0; q2 < 2; q2++) {
        CsAcc &X = acc[jj][b][q2];
        cs_fold(X);
        Sb[(size_t)q2 * ls] = addmod(part[jj][b][q2], reduce128(X.hi + X.cnt, X.lo, q, bar, r64, r64s), q);
      }
    }
}

template <int QB, int JT>
void launch_batch(hd_context *c, const uint64_t *D, const uint64_t *r, uint64_t *S, uint32_t A, int n1, int N,
                  int jmin, int nj) {
  const dim3 grid(A, c->n / MAC_TPB, c->L * (nj / JT));
  if (n1 > 128)
    mac_cs_batch_kernel<QB, JT, true><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, A,
                                                                       c->mt);
  else
    mac_cs_batch_kernel<QB, JT, false><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, A,
                                                                        c->mt);
}
}  // namespace

hd_status mac_ct_run(hd_context *c, const uint64_t *Dct, const uint64_t *r, uint64_t *S3, uint32_t A_loc, int n1,
                     int N, const std::vector<int32_t> &js, bool flat, const DPack &dp) {
  if (js.empty() || A_loc == 0) return HD_OK;
  if (c->n % MAC_TPB) return hd_fail(HD_E_PARAMS, "ring too small for the encrypted MAC");
  if (mac_tma_ct_supported(c, n1, N, flat)) return mac_tma_ct_run(c, Dct, r, S3, A_loc, n1, N, js, flat, dp);
  if (dp.on) return hd_fail(HD_E_STATE, "packed diagonals (R34) need the TMA MAC (HD_MAC_VARIANT set after enrollment?)");
  const int jmin = js.front(), nj = (int)js.size();
  const char *force = getenv("HD_MAC_VARIANT");  // 'g': the generic kernel (tests)
  const bool generic = force && force[0] == 'g';
  // one giant step per thread (64 registers): two per thread (110 registers) measured
  // 34.5 ms vs 28.0 ms at 2^20 x 512
  if ((flat ? N % n1 : (N / 2) % n1) == 0 && !generic) {
    const dim3 grid(A_loc, c->n / MAC_TPB, c->L * nj);
    mac_ct_stream_kernel<1><<<grid, MAC_TPB, 0, c->stream>>>(Dct, r, S3, n1, N, c->L, c->logn, jmin, nj, c->mt, nj);
  } else if (flat && nj > 1 && !generic) {
    // flat packing with n1 not dividing N (e.g. the paper's n1 = 23): giant steps 0 .. nj-2
    // use all n1 baby steps (streaming kernel), only the last one is partial (general kernel)
    const dim3 g_full(A_loc, c->n / MAC_TPB, c->L * (nj - 1)), g_tail(A_loc, c->n / MAC_TPB, c->L);
    mac_ct_stream_kernel<1><<<g_full, MAC_TPB, 0, c->stream>>>(Dct, r, S3, n1, N, c->L, c->logn, jmin, nj - 1,
                                                                c->mt, nj);
    ++c->launches;
    HD_CUDA(cudaGetLastError());
    const size_t ls = (size_t)c->L * c->n;
    mac_ct_kernel<<<g_tail, MAC_TPB, 0, c->stream>>>(Dct, r, S3 + (size_t)(nj - 1) * 3 * ls, n1, N, c->L, c->logn,
                                                     jmin + nj - 1, 1, c->mt, 1, nj);
  } else {
    const dim3 grid(A_loc, c->n / MAC_TPB, c->L * nj);
    mac_ct_kernel<<<grid, MAC_TPB, 0, c->stream>>>(Dct, r, S3, n1, N, c->L, c->logn, jmin, nj, c->mt, flat ? 1 : 0,
                                                   nj);
  }
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status mac_run(hd_context *c, const uint64_t *D, const uint64_t *r, uint64_t *S, uint32_t A_loc, int n1, int N,
                  const std::vector<int32_t> &js, bool flat, const DPack &dp) {
  if (js.empty() || A_loc == 0) return HD_OK;
  if (mac_tma_supported(c, n1, N, flat, 1)) return mac_tma_run(c, D, r, S, A_loc, n1, N, js, 1, flat, dp);
  if (dp.on) return hd_fail(HD_E_STATE, "packed diagonals (R34) need the TMA MAC (HD_MAC_VARIANT set after enrollment?)");
  const int jmin = js.front(), nj = (int)js.size();
  // every giant step uses all n1 baby steps (replicated: n1 | N/2; flat: n1 | N)
  const bool full = (flat ? N % n1 : (N / 2) % n1) == 0 && n1 <= 256 && c->n % MAC_TPB == 0;
  bool small_q = true;
  for (int l = 0; l < c->L; l++) small_q = small_q && c->mod[l] < (1ull << 60);
  const char *force = getenv("HD_MAC_VARIANT");  // 'g': force the generic kernel (tests)
  if (full && small_q && !(force && force[0] == 'g')) {
    const int JT = nj % 2 == 0 ? 2 : 1;
    const dim3 grid(A_loc, c->n / MAC_TPB, c->L * (nj / JT));
    const bool fl = n1 > 128;
    if (JT == 2 && !fl)
      mac_cs_kernel<2, false><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
    else if (JT == 2)
      mac_cs_kernel<2, true><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
    else if (!fl)
      mac_cs_kernel<1, false><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
    else
      mac_cs_kernel<1, true><<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt);
  } else {
    const dim3 grid((c->n + MAC_TPB - 1) / MAC_TPB, c->L, A_loc);
    mac_kernel<<<grid, MAC_TPB, 0, c->stream>>>(D, r, S, n1, N, c->L, c->logn, jmin, nj, c->mt, flat ? 1 : 0);
  }
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status mac_batch_run(hd_context *c, const uint64_t *D, const uint64_t *r, uint64_t *S, uint32_t A_loc, int n1,
                        int N, const std::vector<int32_t> &js, bool flat, uint32_t Q, const DPack &dp) {
  if (js.empty() || A_loc == 0 || Q == 0) return HD_OK;
  const int jmin = js.front(), nj = (int)js.size();
  const size_t ls = (size_t)c->L * c->n, rq = (size_t)n1 * 2 * ls, sq = (size_t)A_loc * nj * 2 * ls;
  if (mac_tma_supported(c, n1, N, flat, 1)) {  // groups of up to 2 (HD_MAC_BATCH: 1..4) queries per pass
    // measured at 2^20 x 512 with the Karatsuba MAC: pairs (QB 2, JT 2) 80.7 q/s, groups of 4
    // (QB 4, JT 1: each r word serves one diagonal word) 77.3, single queries 73.2
    const char *g_env = getenv("HD_MAC_BATCH");
    const uint32_t gmax = g_env ? std::max(1, std::min(4, atoi(g_env))) : 2;
    for (uint32_t b0 = 0; b0 < Q;) {
      const uint32_t g = std::min(gmax, Q - b0);
      hd_status s = mac_tma_run(c, D, r + b0 * rq, S + b0 * sq, A_loc, n1, N, js, g, flat, dp);
      if (s) return s;
      b0 += g;
    }
    return HD_OK;
  }
  if (dp.on) return hd_fail(HD_E_STATE, "packed diagonals (R34) need the TMA MAC");
  const bool full = (flat ? N % n1 : (N / 2) % n1) == 0 && n1 <= 256 && c->n % MAC_TPB == 0;
  bool small_q = true;
  for (int l = 0; l < c->L; l++) small_q = small_q && c->mod[l] < (1ull << 60);
  // Measured at 2^20 x 512 (n1 = 128, one B200): the shared-D kernel costs 12.5 ms per query
  // in groups of 2 and 19 ms in groups of 4, against 11.1 ms for the single-query kernel: its
  // 2 QB baby-step words per diagonal word come from L2 and L2 bandwidth / latency, not HBM,
  // bounds it.  So the default runs the tuned single-query kernel per query; HD_MAC_BATCH=2|4
  // selects the shared-D grouping.
  const char *g_env = getenv("HD_MAC_BATCH");
  if (!(full && small_q) || !g_env) {  // per-query kernels
    for (uint32_t b = 0; b < Q; b++) {
      hd_status s = mac_run(c, D, r + b * rq, S + b * sq, A_loc, n1, N, js, flat, dp);
      if (s) return s;
    }
    return HD_OK;
  }
  // groups of up to G queries per D pass (HD_MAC_BATCH = max group 1, 2 or 4; default 4);
  // two giant steps per thread (JT = 2) for groups of 1 and 2 (HD_MAC_BATCH_JT=1 disables)
  const char *jt_env = getenv("HD_MAC_BATCH_JT");
  const uint32_t gmax = (uint32_t)atoi(g_env);
  for (uint32_t b0 = 0; b0 < Q;) {
    const uint32_t left = Q - b0;
    const uint32_t g = (left >= 4 && gmax >= 4) ? 4 : ((left >= 2 && gmax >= 2) ? 2 : 1);
    const uint64_t *rb = r + b0 * rq;
    uint64_t *Sb = S + b0 * sq;
    const bool jt2 = nj % 2 == 0 && !(jt_env && jt_env[0] == '1');
    if (g == 4) launch_batch<4, 1>(c, D, rb, Sb, A_loc, n1, N, jmin, nj);
    else if (g == 2 && jt2) launch_batch<2, 2>(c, D, rb, Sb, A_loc, n1, N, jmin, nj);
    else if (g == 2) launch_batch<2, 1>(c, D, rb, Sb, A_loc, n1, N, jmin, nj);
    else if (jt2) launch_batch<1, 2>(c, D, rb, Sb, A_loc, n1, N, jmin, nj);
    else launch_batch<1, 1>(c, D, rb, Sb, A_loc, n1, N, jmin, nj);
    ++c->launches;
    HD_CUDA(cudaGetLastError());
    b0 += g;
  }
  return HD_OK;
}
