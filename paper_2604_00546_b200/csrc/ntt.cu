// ntt.cu -- batched 64-bit negacyclic NTT / INTT for sm_100a (K9 of SURVEY 2.2).
//
// Forward: Cooley-Tukey, natural order in, bit-reversed evaluation order out
// (R13); inverse: Gentleman-Sande, then x n^{-1}.  Twiddles psi^{br(k)}
// are stored interleaved with their Shoup companions ({w, floor(w 2^64 / q)}: one
// 128-bit load per butterfly group).
//
// Decomposition: log n = s1 + s2.  Kernel "cols" runs the s1 high stages on
// columns {x 2^s2 + c : x < 2^s1} (a CTA owns TPC consecutive columns; global
// loads/stores are coalesced across columns); kernel "chunks" runs the s2 low
// stages on contiguous chunks of 2^s2 elements (staged through shared memory
// with flat 128-bit coalesced copies).  Inside a kernel every thread holds 16
// elements and performs up to 4 butterfly stages in registers per pass
// (radix-16); passes exchange through padded shared memory.  Every index is a
// compile-time function of (S, pass, slot) plus the thread id.  Harvey lazy
// reduction: forward values live in [0, 4q), inverse values in [0, 2q); the last
// kernel reduces to [0, q).  Moduli are < 2^60, so 4q < 2^62.
//
// Fusion (ntt_run): the first kernel may load its rows from another row map (out
// of place) and lift centred residues from the source modulus (ModUp / ModDown /
// rescale lifts, R12); the final forward store may apply the ModDown / rescale
// combine (A - v) w (+ pi_g(c0)), written or accumulated into a third row map.
//
// Rows whose modulus is below 2^45 (the 45-bit scaling limbs) run the same passes with FP64
// butterflies instead (R33, below): the integer Shoup product is bound by the IMAD pipe, the
// FP64 one runs on the FP64 pipe at ~2.2x the butterfly rate (tools/micro/bfly_bench.cu).
#include "common.cuh"

#include <cstdlib>

// 1: the chunk kernel stages its chunks' twiddles in shared memory at start (2 CTAs per SM
// instead of 3); 0: read from L1/L2 during the passes (A/B)
#ifndef HD_NTT_TW_SMEM
#define HD_NTT_TW_SMEM 0
#endif

namespace {

constexpr int E = 16;  // elements per thread

__device__ __forceinline__ uint32_t pad_idx(uint32_t x) { return x + (x >> 4); }

// The rows one launch transforms: row = r0 + (y / count) period + pos[y % count] for grid row y
// (the rows of one kind -- FP64 or integer butterflies -- of a row map whose modulus pattern
// repeats every `period` rows); rows at or past `end` exit.
struct RowSel {
  uint32_t period = 1, count = 1, end = 0;
  FDiv fc;
  uint8_t pos[64] = {0};
};
__device__ __forceinline__ uint32_t sel_row(const RowSel &s, uint32_t r0, uint32_t y) {
  const uint32_t k = fdiv_q(y, s.fc);
  return r0 + k * s.period + s.pos[y - k * s.count];
}

template <bool INV, int S, int P>
struct Pass {
  static constexpr int NP = (S + 3) / 4;
  static constexpr int LAST = S - 4 * (NP - 1);
  static constexpr int KP = INV ? (P == 0 ? LAST : 4) : (P == NP - 1 ? LAST : 4);
  static constexpr int REM = INV ? (LAST + 4 * P) : (S - 4 * P);
};

// Thread element of slot = g 2^KP + e:  x = (y >> DL) 2^REM + e 2^DL + (y & (2^DL - 1)),
// y = g 2^(S-4) + tid, DL = REM - KP.
template <int KP, int REM, int S>
__device__ __forceinline__ uint32_t elem_of(int slot, uint32_t tid) {
  constexpr int DL = REM - KP;
  const int g = slot >> KP, e = slot & ((1 << KP) - 1);
  const uint32_t y = ((uint32_t)g << (S - 4)) + tid;
  return ((y >> DL) << REM) + ((uint32_t)e << DL) + (y & ((1u << DL) - 1));
}

// Twiddles of a kernel, staged in shared memory at kernel start: for every level k
// (2^k butterfly groups per transform) the tpc transforms of the CTA use the contiguous
// table range T[(b0 + tr) 2^k + local], b0 = first transform's block index; level k is
// stored at tpc (2^k - 1) + tr 2^k + local.
struct TwShared {
  const ulonglong2 *sm;
  uint32_t tr, tpc;
  __device__ __forceinline__ ulonglong2 get(int k, uint32_t local) const {
    return sm[tpc * ((1u << k) - 1) + (tr << k) + local];
  }
};
// Twiddles read straight from the global table (L1/L2): T[(b0 + tr) 2^k + local].
struct TwGlobal {
  const ulonglong2 *T;
  uint32_t blk;  // b0 + tr
  __device__ __forceinline__ ulonglong2 get(int k, uint32_t local) const {
    return __ldg(&T[((size_t)blk << k) + local]);
  }
};
// Column twiddles (b0 = 1, one transform per table): level k lives at (2^k - 1) + local
// and comes from T[2^k + local], i.e. the staged table is T[1 .. 2^S - 1] copied flat
// (all loads issued before any store: one global latency, not S).
template <int S>
__device__ __forceinline__ void stage_twiddles(ulonglong2 *dst, const ulonglong2 *__restrict__ T) {
  constexpr uint32_t CNT = (1u << S) - 1;
  constexpr int PER = (CNT + 127) / 128;  // blockDim.x >= 128 for S <= 8
  ulonglong2 t[PER];
#pragma unroll
  for (int k = 0; k < PER; k++) {
    const uint32_t i = threadIdx.x + k * blockDim.x;
    if (i < CNT) t[k] = __ldg(T + 1 + i);
  }
#pragma unroll
  for (int k = 0; k < PER; k++) {
    const uint32_t i = threadIdx.x + k * blockDim.x;
    if (i < CNT) dst[i] = t[k];
  }
}

// a w mod q in [0, 2q) (Shoup), written as 32-bit multiply / carry chains: the quotient
// umulhi(a, ws) from mul.hi / mad.lo.cc / madc.hi and both low products from mul.lo / mad.lo.
// 2.6 % (forward) and 7.4 % (inverse) more butterflies/s than __umul64hi on B200
// (tools/micro/bfly_bench.cu, V4): fewer IMAD.WIDE on the integer-multiply pipe that bounds it.
__device__ __forceinline__ uint64_t shoup_lazy32(uint64_t a, uint64_t w, uint64_t ws, uint64_t q) {
  uint32_t r0, r1;
  asm("{\n\t.reg .u32 a0, a1, s0, s1, w0, w1, q0, q1, t, m0, m1, m2, h0, h1, p0, p1, x0, x1;\n\t"
      "mov.b64 {a0, a1}, %2;\n\t"
      "mov.b64 {s0, s1}, %4;\n\t"
      "mov.b64 {w0, w1}, %3;\n\t"
      "mov.b64 {q0, q1}, %5;\n\t"
      "mul.hi.u32 t, a0, s0;\n\t"
      "mad.lo.cc.u32 m0, a0, s1, t;\n\t"
      "madc.hi.u32 m1, a0, s1, 0;\n\t"
      "mad.lo.cc.u32 m0, a1, s0, m0;\n\t"
      "madc.hi.cc.u32 m1, a1, s0, m1;\n\t"
      "addc.u32 m2, 0, 0;\n\t"
      "mad.lo.cc.u32 h0, a1, s1, m1;\n\t"
      "madc.hi.u32 h1, a1, s1, m2;\n\t"
      "mul.lo.u32 p0, a0, w0;\n\t"
      "mul.hi.u32 p1, a0, w0;\n\t"
      "mad.lo.u32 p1, a0, w1, p1;\n\t"
      "mad.lo.u32 p1, a1, w0, p1;\n\t"
      "mul.lo.u32 x0, h0, q0;\n\t"
      "mul.hi.u32 x1, h0, q0;\n\t"
      "mad.lo.u32 x1, h0, q1, x1;\n\t"
      "mad.lo.u32 x1, h1, q0, x1;\n\t"
      "sub.cc.u32 %0, p0, x0;\n\t"
      "subc.u32 %1, p1, x1;\n\t"
      "}"
      : "=r"(r0), "=r"(r1)
      : "l"(a), "l"(w), "l"(ws), "l"(q));
  return ((uint64_t)r1 << 32) | r0;
}

// KP <= 4 butterfly stages in registers.  The butterfly at distance d = 2^(u + DL)
// uses the twiddle of level k = S-1-u-DL, local index (y >> DL) 2^(KP-u-1) + (e >> (u+1)).
template <bool INV, int KP, int REM, int S, class TW>
__device__ __forceinline__ void radix_pass(uint64_t (&v)[E], uint32_t tid, const TW &tw, uint64_t q) {
  constexpr int NG = 1 << (4 - KP);
  constexpr int DL = REM - KP;
  const uint64_t two_q = 2 * q;
#pragma unroll
  for (int uu = 0; uu < KP; uu++) {
    const int u = INV ? uu : (KP - 1 - uu);
#pragma unroll
    for (int g = 0; g < NG; g++) {
      const uint32_t y = ((uint32_t)g << (S - 4)) + tid;
      const uint32_t tloc = (y >> DL) << (KP - u - 1);
#pragma unroll
      for (int e = 0; e < (1 << KP); e++) {
        if (!(e & (1 << u))) {
          const int i0 = g * (1 << KP) + e, i1 = i0 + (1 << u);
          const ulonglong2 w = tw.get(S - 1 - u - DL, tloc + (e >> (u + 1)));
          const uint64_t X = v[i0], Y = v[i1];
          if (!INV) {
            const uint64_t Xr = X >= two_q ? X - two_q : X;
            const uint64_t t = shoup_lazy32(Y, w.x, w.y, q);
            v[i0] = Xr + t;
            v[i1] = Xr - t + two_q;
          } else {
            const uint64_t a = X + Y;
            v[i0] = a >= two_q ? a - two_q : a;
            v[i1] = shoup_lazy32(X - Y + two_q, w.x, w.y, q);
          }
        }
      }
    }
  }
}

__device__ __forceinline__ uint64_t final_reduce(uint64_t x, uint64_t q) {  // [0, 4q) -> [0, q)
  if (x >= 2 * q) x -= 2 * q;
  if (x >= q) x -= q;
  return x;
}

// ---- FP64 butterflies for moduli q < 2^45 (R33) ----
// The 64-bit Shoup product above costs ~15 IMAD-class instructions on the integer multiply
// (fmaheavy) pipe, which bounds the integer NTT.  Below 2^45 a residue is an exact double, and
// y w mod q follows from an error-free product ph + pl = y w (DMUL + DFMA), a rounded quotient
// Q = rint(ph / q) and t = (ph - Q q) + pl, both steps exact (|ph - Q q| < 2^53): 7 FP64
// operations on the FP64 pipe, |t| <= 1.25 q for |y| < 2^51.  Values stay signed and unreduced:
// forward, |X| <= q + 1.25 q per stage (<= 21 q after 16 stages); inverse, every radix-16 pass
// starts by reducing its 16 values to |x| <= q/2 (X + Y doubles per stage: <= 10 q after a
// pass).  Every bound stays below 2^51, where the 1.5 * 2^52 rounding constant is exact, for
// inputs up to 4q (Harvey-lazy rows from any caller): the bound 2^45 leaves that margin.
// Between the two kernels of one transform a row holds these doubles (bit patterns) in place.
constexpr double kRnd = 6755399441055744.0;  // 1.5 * 2^52: x + kRnd - kRnd = rint(x), |x| < 2^51
__device__ __forceinline__ double f_mulmod(double y, double w, double q, double qinv) {
  const double ph = __dmul_rn(y, w);
  const double pl = __fma_rn(y, w, -ph);
  const double Q = __dsub_rn(__dadd_rn(__dmul_rn(ph, qinv), kRnd), kRnd);
  return __dadd_rn(__fma_rn(-Q, q, ph), pl);
}
__device__ __forceinline__ double f_red(double x, double q, double qinv) {  // |result| <= q/2 (+ tiny)
  const double Q = __dsub_rn(__dadd_rn(__dmul_rn(x, qinv), kRnd), kRnd);
  return __fma_rn(-Q, q, x);
}
__device__ __forceinline__ double u2d(uint64_t x) {  // exact for x < 2^52
  return __dsub_rn(__longlong_as_double((long long)(x | 0x4330000000000000ull)), 4503599627370496.0);
}
__device__ __forceinline__ uint64_t d2u_canon(double x, double q, double qinv) {  // |x| < 2^51 -> [0, q)
  double r = f_red(x, q, qinv);
  if (r < 0) r = __dadd_rn(r, q);
  return (uint64_t)__double_as_longlong(__dadd_rn(r, 4503599627370496.0)) & 0xFFFFFFFFFFFFFull;
}
__device__ __forceinline__ double bits_d(uint64_t w) { return __longlong_as_double((long long)w); }
__device__ __forceinline__ uint64_t d_bits(double d) { return (uint64_t)__double_as_longlong(d); }

struct FMod {
  double q, qinv;
};
__device__ __forceinline__ FMod fmod_of(uint64_t q) {
  FMod f;
  f.q = u2d(q);
  f.qinv = 1.0 / f.q;
  return f;
}

struct TwSharedD {
  const double *sm;
  __device__ __forceinline__ double get(int k, uint32_t local) const { return sm[((1u << k) - 1) + local]; }
};
struct TwGlobalD {
  const double *T;
  uint32_t blk;
  __device__ __forceinline__ double get(int k, uint32_t local) const {
    return __ldg(&T[((size_t)blk << k) + local]);
  }
};

template <bool INV, int KP, int REM, int S, class TW>
__device__ __forceinline__ void radix_pass_f(double (&v)[E], uint32_t tid, const TW &tw, const FMod &F) {
  constexpr int NG = 1 << (4 - KP);
  constexpr int DL = REM - KP;
#pragma unroll
  for (int uu = 0; uu < KP; uu++) {
    const int u = INV ? uu : (KP - 1 - uu);
#pragma unroll
    for (int g = 0; g < NG; g++) {
      const uint32_t y = ((uint32_t)g << (S - 4)) + tid;
      const uint32_t tloc = (y >> DL) << (KP - u - 1);
#pragma unroll
      for (int e = 0; e < (1 << KP); e++) {
        if (!(e & (1 << u))) {
          const int i0 = g * (1 << KP) + e, i1 = i0 + (1 << u);
          const double w = tw.get(S - 1 - u - DL, tloc + (e >> (u + 1)));
          const double X = v[i0], Y = v[i1];
          if (!INV) {
            const double t = f_mulmod(Y, w, F.q, F.qinv);
            v[i0] = __dadd_rn(X, t);
            v[i1] = __dsub_rn(X, t);
          } else {
            v[i0] = __dadd_rn(X, Y);
            v[i1] = f_mulmod(__dsub_rn(X, Y), w, F.q, F.qinv);
          }
        }
      }
    }
  }
}

// input element of the first kernel: in-place row, or source row (+ centred lift)
struct InRow {
  const uint64_t *p;
  bool lift;
  uint64_t qs, q, bar;
  __device__ __forceinline__ uint64_t ld(size_t i) const {
    const uint64_t v = p[i];
    return lift ? lift_centred(v, qs, q, bar) : v;
  }
};

__device__ __forceinline__ InRow in_row(uint64_t *data, const RowMap &map, const NttSrc &src, uint32_t row, uint32_t n,
                                        int m, const ModTab &mt) {
  InRow I;
  if (src.base) {
    I.p = src.base + row_off(src.map, row, n);
    I.lift = src.lift;
    I.qs = mt.q[row_mod(src.map, row)];
  } else {
    I.p = data + row_off(map, row, n);
    I.lift = false;
    I.qs = 0;
  }
  I.q = mt.q[m];
  I.bar = mt.bar[m];
  return I;
}

struct ColArgs {
  uint32_t s2, tid, c;
  uint64_t *a, *smt;
  InRow in;
  TwShared tw;
  uint64_t q;
  const uint64_t *ninv;
  int m;
  bool final_out;
};

template <bool INV, int S, int P>
__device__ __forceinline__ void cols_rec(uint64_t (&v)[E], const ColArgs &A) {
  using PP = Pass<INV, S, P>;
#pragma unroll
  for (int i = 0; i < E; i++) {
    const uint32_t x = elem_of<PP::KP, PP::REM, S>(i, A.tid);
    v[i] = P == 0 ? A.in.ld(((size_t)x << A.s2) + A.c) : A.smt[pad_idx(x)];
  }
  radix_pass<INV, PP::KP, PP::REM, S>(v, A.tid, A.tw, A.q);
  if constexpr (P == PP::NP - 1) {
#pragma unroll
    for (int i = 0; i < E; i++) {
      uint64_t o = v[i];
      if (INV) o = shoup(o, A.ninv[A.m], A.ninv[HD_MAXMOD + A.m], A.q);
      else if (A.final_out) o = final_reduce(o, A.q);
      A.a[((size_t)elem_of<PP::KP, PP::REM, S>(i, A.tid) << A.s2) + A.c] = o;
    }
  } else {
    if (P > 0) __syncthreads();
#pragma unroll
    for (int i = 0; i < E; i++) A.smt[pad_idx(elem_of<PP::KP, PP::REM, S>(i, A.tid))] = v[i];
    __syncthreads();
    cols_rec<INV, S, P + 1>(v, A);
  }
}

// FP64 columns pass chain: forward (first kernel) reads residues and writes the raw doubles of
// the intermediate; inverse (second kernel) reads the raw doubles and writes x n^{-1} in [0, q).
struct ColArgsF {
  uint32_t s2, tid, c;
  uint64_t *a;
  double *smt;
  InRow in;
  TwSharedD tw;
  FMod F;
  double ninv;
};
template <bool INV, int S, int P>
__device__ __forceinline__ void cols_rec_f(double (&v)[E], const ColArgsF &A) {
  using PP = Pass<INV, S, P>;
#pragma unroll
  for (int i = 0; i < E; i++) {
    const uint32_t x = elem_of<PP::KP, PP::REM, S>(i, A.tid);
    if (P == 0) {
      const size_t gi = ((size_t)x << A.s2) + A.c;
      v[i] = INV ? bits_d(A.in.p[gi]) : u2d(A.in.ld(gi));
    } else {
      v[i] = A.smt[pad_idx(x)];
    }
    if (INV) v[i] = f_red(v[i], A.F.q, A.F.qinv);  // every inverse pass starts reduced
  }
  radix_pass_f<INV, PP::KP, PP::REM, S>(v, A.tid, A.tw, A.F);
  if constexpr (P == PP::NP - 1) {
#pragma unroll
    for (int i = 0; i < E; i++) {
      const uint64_t o = INV ? d2u_canon(f_mulmod(v[i], A.ninv, A.F.q, A.F.qinv), A.F.q, A.F.qinv) : d_bits(v[i]);
      A.a[((size_t)elem_of<PP::KP, PP::REM, S>(i, A.tid) << A.s2) + A.c] = o;
    }
  } else {
    if (P > 0) __syncthreads();
#pragma unroll
    for (int i = 0; i < E; i++) A.smt[pad_idx(elem_of<PP::KP, PP::REM, S>(i, A.tid))] = v[i];
    __syncthreads();
    cols_rec_f<INV, S, P + 1>(v, A);
  }
}

template <int S>
__device__ __forceinline__ void stage_twiddles_d(double *dst, const double *__restrict__ T) {
  constexpr uint32_t CNT = (1u << S) - 1;
  constexpr int PER = (CNT + 127) / 128;
  double t[PER];
#pragma unroll
  for (int k = 0; k < PER; k++) {
    const uint32_t i = threadIdx.x + k * blockDim.x;
    if (i < CNT) t[k] = __ldg(T + 1 + i);
  }
#pragma unroll
  for (int k = 0; k < PER; k++) {
    const uint32_t i = threadIdx.x + k * blockDim.x;
    if (i < CNT) dst[i] = t[k];
  }
}

// ---- columns kernel: the S high stages; tpc columns per CTA, 2^(S-4) threads per column ----
template <bool INV, int S, bool FP>
__global__ void __launch_bounds__(256, 3) ntt_cols_kernel(uint64_t *base, RowMap rm, ModTab mt,
                                                       const ulonglong2 *__restrict__ tw, int logn, int tpc,
                                                       const uint64_t *__restrict__ ninv, uint32_t r0, bool final_out,
                                                       NttSrc src, const double *__restrict__ twd, RowSel sel) {
  extern __shared__ uint64_t sm[];
  const uint32_t n = 1u << logn;
  const uint32_t row = sel_row(sel, r0, blockIdx.y);
  if (row >= sel.end) return;
  const int m = row_mod(rm, row);
  if constexpr (FP) {  // FP64 butterflies: every row of this launch has a modulus below 2^45
    (void)tw;
    ColArgsF A;
    A.s2 = logn - S;
    A.F = fmod_of(mt.q[m]);
    A.ninv = u2d(ninv[m]);
    A.a = row_ptr(base, rm, row, n);
    A.in = in_row(base, rm, src, row, n, m, mt);
    const uint32_t tr = threadIdx.x & (tpc - 1);
    A.tid = threadIdx.x >> (__ffs(tpc) - 1);
    A.c = blockIdx.x * tpc + tr;
    const uint32_t col_stride = pad_idx(1u << S) + 1;
    A.smt = reinterpret_cast<double *>(sm) + tr * col_stride;
    double *tws = reinterpret_cast<double *>(sm) + ((tpc * col_stride + 1) & ~1u);
    stage_twiddles_d<S>(tws, twd + (size_t)m * n);
    A.tw.sm = tws;
    __syncthreads();
    double v[E];
    cols_rec_f<INV, S, 0>(v, A);
  } else {
  ColArgs A;
  A.s2 = logn - S;
  A.q = mt.q[m];
  A.a = row_ptr(base, rm, row, n);
  A.in = in_row(base, rm, src, row, n, m, mt);
  const uint32_t tr = threadIdx.x & (tpc - 1);  // tpc is a power of two (ntt_run)
  A.tid = threadIdx.x >> (__ffs(tpc) - 1);
  A.c = blockIdx.x * tpc + tr;
  const uint32_t col_stride = pad_idx(1u << S) + 1;  // odd column stride: conflict-free across columns
  A.smt = sm + tr * col_stride;
  // every column of the row uses the same twiddles T[1 .. 2^S - 1]
  ulonglong2 *tws = reinterpret_cast<ulonglong2 *>(sm + ((tpc * col_stride + 1) & ~1u));
  stage_twiddles<S>(tws, tw + (size_t)m * n);
  A.tw.sm = tws;
  A.tw.tr = 0;
  A.tw.tpc = 1;
  A.ninv = ninv;
  A.m = m;
  A.final_out = final_out;
  __syncthreads();
  uint64_t v[E];
  cols_rec<INV, S, 0>(v, A);
  }
}

template <bool INV, int S, int P, class TW>
__device__ __forceinline__ void chunks_rec(uint64_t (&v)[E], uint32_t tid, uint64_t *smt, const TW &tw,
                                           uint64_t q) {
  using PP = Pass<INV, S, P>;
#pragma unroll
  for (int i = 0; i < E; i++) v[i] = smt[pad_idx(elem_of<PP::KP, PP::REM, S>(i, tid))];
  radix_pass<INV, PP::KP, PP::REM, S>(v, tid, tw, q);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < E; i++) smt[pad_idx(elem_of<PP::KP, PP::REM, S>(i, tid))] = v[i];
  __syncthreads();
  if constexpr (P < PP::NP - 1) chunks_rec<INV, S, P + 1, TW>(v, tid, smt, tw, q);
}

template <bool INV, int S, int P>
__device__ __forceinline__ void chunks_rec_f(double (&v)[E], uint32_t tid, double *smt, const TwGlobalD &tw,
                                             const FMod &F) {
  using PP = Pass<INV, S, P>;
#pragma unroll
  for (int i = 0; i < E; i++) {
    v[i] = smt[pad_idx(elem_of<PP::KP, PP::REM, S>(i, tid))];
    // the inverse reduces at every pass but the first (its inputs are residues below 4 q)
    if (INV && P > 0) v[i] = f_red(v[i], F.q, F.qinv);
  }
  radix_pass_f<INV, PP::KP, PP::REM, S>(v, tid, tw, F);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < E; i++) smt[pad_idx(elem_of<PP::KP, PP::REM, S>(i, tid))] = v[i];
  __syncthreads();
  if constexpr (P < PP::NP - 1) chunks_rec_f<INV, S, P + 1>(v, tid, smt, tw, F);
}

// ---- chunks kernel: the S low stages on contiguous chunks of 2^S; tpc chunks per CTA ----
// One body per row kind (FP: FP64 butterflies, R33); ntt_run launches the rows of each kind
// separately (a CTA running one body beside a CTA running the other thrashes the instruction
// cache: no_instruction stalls 6.4 per issue).  The kind is a compile-time constant (a runtime
// flag mixed into the store-path predicates was also miscompiled: the scaling predicate came
// out as fp && s1 != 0 instead of !fp && s1 == 0).
template <bool INV, int S, bool FP>
__device__ __forceinline__ void chunks_body(uint64_t *base, const RowMap &rm, const ModTab &mt,
                                            const ulonglong2 *__restrict__ tw, int logn, int tpc,
                                            const uint64_t *__restrict__ ninv, uint32_t row, bool final_out,
                                            const NttSrc &src, const NttEpi &epi, const double *__restrict__ twd) {
  extern __shared__ uint64_t sm[];
  constexpr uint32_t SZ = 1u << S, TPT = SZ / E, PS = SZ + (SZ >> 4);
  const uint32_t n = 1u << logn, s1 = logn - S;
  const int m = row_mod(rm, row);
  const uint64_t q = mt.q[m];
  // FP64 rows (R33): the forward chunks kernel after a columns kernel reads the raw doubles
  // of the intermediate; the inverse chunks kernel before one writes them
  const bool raw_in = FP && !INV && s1 > 0, raw_out = FP && INV && s1 > 0;
  const uint32_t chunk0 = blockIdx.x * tpc;
  const size_t off0 = (size_t)chunk0 * SZ;
  uint64_t *a = row_ptr(base, rm, row, n) + off0;
  const InRow in = in_row(base, rm, src, row, n, m, mt);
  const uint32_t tr = threadIdx.x / TPT, tid = threadIdx.x % TPT;
  // twiddles of this chunk: transform block index 2^s1 + chunk0 + tr at every level
  // (each chunk uses its own 2^S - 1 entries: read from L1/L2, not staged)
  TwGlobal twv;
  twv.T = tw + (size_t)m * n;
  twv.blk = (1u << s1) + chunk0 + tr;
  // blockDim.x * E == total: every thread moves exactly E elements (E/2 128-bit words);
  // all loads are issued before the first shared-memory store.
  uint64_t v[E];
  {
    ulonglong2 w[E / 2];
#pragma unroll
    for (int k = 0; k < E / 2; k++)
      w[k] = *reinterpret_cast<const ulonglong2 *>(in.p + off0 + 2 * (threadIdx.x + k * blockDim.x));
#pragma unroll
    for (int k = 0; k < E / 2; k++) {
      const uint32_t i = 2 * (threadIdx.x + k * blockDim.x);
      uint64_t w0 = w[k].x, w1 = w[k].y;
      if (in.lift) {
        w0 = lift_centred(w0, in.qs, in.q, in.bar);
        w1 = lift_centred(w1, in.qs, in.q, in.bar);
      }
      if (FP && !raw_in) {
        w0 = d_bits(u2d(w0));
        w1 = d_bits(u2d(w1));
      }
      const uint32_t t0 = i >> S, x0 = i & (SZ - 1);
      sm[t0 * PS + pad_idx(x0)] = w0;
      sm[t0 * PS + pad_idx(x0 + 1)] = w1;
    }
  }
  FMod F{};
  double ninv_f = 0;
  if constexpr (FP) {
    F = fmod_of(q);
    __syncthreads();
    TwGlobalD twf;
    twf.T = twd + (size_t)m * n;
    twf.blk = (1u << s1) + chunk0 + tr;
    double vf[E];
    chunks_rec_f<INV, S, 0>(vf, tid, reinterpret_cast<double *>(sm) + tr * PS, twf, F);
    ninv_f = u2d(ninv[m]);
  } else {
#if HD_NTT_TW_SMEM
  ulonglong2 *tws = reinterpret_cast<ulonglong2 *>(sm + tpc * PS);
  for (int k = 0; k < S; k++) {
    const uint32_t cnt = (uint32_t)tpc << k;
    const ulonglong2 *srcw = twv.T + ((size_t)((1u << s1) + chunk0) << k);
    ulonglong2 *dstw = tws + (size_t)tpc * ((1u << k) - 1);
    for (uint32_t i = threadIdx.x; i < cnt; i += blockDim.x) dstw[i] = __ldg(srcw + i);
  }
  __syncthreads();
  TwShared twsm;
  twsm.sm = tws;
  twsm.tr = tr;
  twsm.tpc = tpc;
  chunks_rec<INV, S, 0, TwShared>(v, tid, sm + tr * PS, twsm, q);
#else
  __syncthreads();
  chunks_rec<INV, S, 0, TwGlobal>(v, tid, sm + tr * PS, twv, q);
#endif
  }
  // a finished word of the transform: FP64 rows convert their doubles to [0, q) (x n^{-1} when
  // this kernel ends an inverse transform) unless the intermediate stays raw for the next kernel
  auto outw = [&](uint32_t idx) -> uint64_t {
    const uint64_t w = sm[idx];
    if (!FP || raw_out) return w;
    double d = bits_d(w);
    if (INV) d = f_mulmod(d, ninv_f, F.q, F.qinv);  // s1 == 0 (raw_out otherwise)
    return d2u_canon(d, F.q, F.qinv);
  };
  const bool scale = !FP && INV && s1 == 0;
  const bool fin = !INV && final_out;
  // epilogue rows: r = (x 2 + p) ell + l
  const uint32_t rq = fdiv_q(row, epi.fell), l = row - rq * epi.ell, p = rq & 1, x = fdiv_q(row, epi.f2ell);
  uint64_t *dst = a;
  const uint64_t *Arow = nullptr, *c0row = nullptr;
  uint32_t g = 1;
  if (fin && epi.mode) {
    dst = row_ptr(epi.out, epi.omap, row, n) + off0;
    Arow = epi.A + row_off(epi.amap, row, n) + off0;
    if (epi.mode == 2 && p == 0) {
      const uint32_t xk = fdiv_q(x, epi.fK);
      c0row = epi.c0 + (size_t)xk * epi.c0_stride + (size_t)l * n;
      g = epi.gal[x - xk * epi.K];
    }
  }
  if (fin && epi.mode) {
    // combine epilogue, in batches of H 128-bit words: the batch's global operands
    // (A, the Galois-gathered c0, the accumulator) are all loaded before use.
    constexpr int H = E / 4;
    const uint64_t w = epi.w[m], ws = epi.ws[m];
#pragma unroll
    for (int b = 0; b < E / 2; b += H) {
      ulonglong2 av[H], cv[H], dv[H];
#pragma unroll
      for (int k = 0; k < H; k++) {
        const uint32_t i = 2 * (threadIdx.x + (b + k) * blockDim.x);
        av[k] = *reinterpret_cast<const ulonglong2 *>(Arow + i);
        if (c0row) {
          const uint32_t gi = (uint32_t)(off0 + i);
          cv[k].x = c0row[galois_src(gi, g, logn)];
          cv[k].y = c0row[galois_src(gi + 1, g, logn)];
        }
        if (epi.acc) dv[k] = *reinterpret_cast<const ulonglong2 *>(dst + i);
      }
#pragma unroll
      for (int k = 0; k < H; k++) {
        const uint32_t i = 2 * (threadIdx.x + (b + k) * blockDim.x);
        const uint32_t t0 = i >> S, x0 = i & (SZ - 1);
        uint64_t o0 = final_reduce(outw(t0 * PS + pad_idx(x0)), q);
        uint64_t o1 = final_reduce(outw(t0 * PS + pad_idx(x0 + 1)), q);
        o0 = shoup(submod(av[k].x, o0, q), w, ws, q);
        o1 = shoup(submod(av[k].y, o1, q), w, ws, q);
        if (c0row) {
          o0 = addmod(o0, cv[k].x, q);
          o1 = addmod(o1, cv[k].y, q);
        }
        if (epi.acc) {
          o0 = addmod(o0, dv[k].x, q);
          o1 = addmod(o1, dv[k].y, q);
        }
        *reinterpret_cast<ulonglong2 *>(dst + i) = make_ulonglong2(o0, o1);
      }
    }
    return;
  }
#pragma unroll
  for (int k = 0; k < E / 2; k++) {
    const uint32_t i = 2 * (threadIdx.x + k * blockDim.x);
    const uint32_t t0 = i >> S, x0 = i & (SZ - 1);
    uint64_t o0 = outw(t0 * PS + pad_idx(x0)), o1 = outw(t0 * PS + pad_idx(x0 + 1));
    if (scale) {
      o0 = shoup(o0, ninv[m], ninv[HD_MAXMOD + m], q);
      o1 = shoup(o1, ninv[m], ninv[HD_MAXMOD + m], q);
    } else if (fin) {
      o0 = final_reduce(o0, q);
      o1 = final_reduce(o1, q);
    }
    *reinterpret_cast<ulonglong2 *>(dst + i) = make_ulonglong2(o0, o1);
  }
}

template <bool INV, int S, bool FP>
__global__ void __launch_bounds__(256, 3) ntt_chunks_kernel(uint64_t *base, RowMap rm, ModTab mt,
                                                         const ulonglong2 *__restrict__ tw, int logn, int tpc,
                                                         const uint64_t *__restrict__ ninv, uint32_t r0, bool final_out,
                                                         NttSrc src, NttEpi epi, const double *__restrict__ twd,
                                                         RowSel sel) {
  const uint32_t row = sel_row(sel, r0, blockIdx.y);
  if (row >= sel.end) return;
  chunks_body<INV, S, FP>(base, rm, mt, tw, logn, tpc, ninv, row, final_out, src, epi, twd);
}

typedef void (*cols_kernel_t)(uint64_t *, RowMap, ModTab, const ulonglong2 *, int, int, const uint64_t *, uint32_t,
                              bool, NttSrc, const double *, RowSel);
typedef void (*chunks_kernel_t)(uint64_t *, RowMap, ModTab, const ulonglong2 *, int, int, const uint64_t *, uint32_t,
                                bool, NttSrc, NttEpi, const double *, RowSel);

template <bool INV, bool FP>
cols_kernel_t cols_for(int s) {
  switch (s) {
    case 5: return ntt_cols_kernel<INV, 5, FP>;
    case 6: return ntt_cols_kernel<INV, 6, FP>;
    case 7: return ntt_cols_kernel<INV, 7, FP>;
    case 8: return ntt_cols_kernel<INV, 8, FP>;
  }
  return nullptr;
}
template <bool INV, bool FP>
chunks_kernel_t chunks_for(int s) {
  switch (s) {
    case 4: return ntt_chunks_kernel<INV, 4, FP>;
    case 5: return ntt_chunks_kernel<INV, 5, FP>;
    case 6: return ntt_chunks_kernel<INV, 6, FP>;
    case 7: return ntt_chunks_kernel<INV, 7, FP>;
    case 8: return ntt_chunks_kernel<INV, 8, FP>;
    case 9: return ntt_chunks_kernel<INV, 9, FP>;
    case 10: return ntt_chunks_kernel<INV, 10, FP>;
    case 11: return ntt_chunks_kernel<INV, 11, FP>;
    case 12: return ntt_chunks_kernel<INV, 12, FP>;
  }
  return nullptr;
}
cols_kernel_t cols_pick(bool inv, bool fp, int s) {
  return inv ? (fp ? cols_for<true, true>(s) : cols_for<true, false>(s))
             : (fp ? cols_for<false, true>(s) : cols_for<false, false>(s));
}
chunks_kernel_t chunks_pick(bool inv, bool fp, int s) {
  return inv ? (fp ? chunks_for<true, true>(s) : chunks_for<true, false>(s))
             : (fp ? chunks_for<false, true>(s) : chunks_for<false, false>(s));
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

hd_status ntt_run(hd_context *c, uint64_t *data, uint32_t rows, const RowMap &map_in, bool inverse,
                  const NttSrc *srcp, const NttEpi *epip) {
  if (rows == 0) return HD_OK;
  const int logn = c->logn;
  const int s2 = logn <= 12 ? logn : 8;  // chunk stages
  const int s1 = logn - s2;              // column stages (0, or 5..8)
  const ulonglong2 *tw = reinterpret_cast<const ulonglong2 *>(inverse ? c->itw2 : c->tw2);
  const uint64_t *ninv = c->ninv_dev;
  // FP64 butterflies for the moduli below 2^45 (R33); HD_NTT_FP64=0 keeps every row on the
  // integer path (A/B knob)
  static const bool fp64_off = [] {
    const char *e = getenv("HD_NTT_FP64");
    return e && e[0] == '0';
  }();
  const double *twd = fp64_off ? nullptr : (inverse ? c->itwd : c->twd);
  NttSrc none_src{};
  NttEpi none_epi{};
  NttSrc src = srcp ? *srcp : none_src;
  NttEpi epi = epip ? *epip : none_epi;
  RowMap map = map_in;  // fast row divisions for the device
  rowmap_finalize(map);
  rowmap_finalize(src.map);
  rowmap_finalize(none_src.map);
  rowmap_finalize(epi.amap);
  rowmap_finalize(epi.omap);
  epi.fell = fdiv_make((uint32_t)epi.ell);
  epi.f2ell = fdiv_make(2u * (uint32_t)epi.ell);
  epi.fK = fdiv_make((uint32_t)epi.K);
  none_epi.fell = none_epi.f2ell = none_epi.fK = fdiv_make(1);
  if (inverse && epi.mode) return hd_fail(HD_E_INVALID_ARG, "epilogue only on forward transforms");
  const int tpt_b = 1 << (s2 - 4);
  const int tpc_b = std::max(1, std::min(256 / tpt_b, 1 << s1));
  const size_t smem_b = sizeof(uint64_t) * tpc_b * (size_t)((1 << s2) + ((1 << s2) >> 4)) +
                        (HD_NTT_TW_SMEM ? 16 * (size_t)tpc_b * ((1 << s2) - 1) : 0);
  const int tpt_a = s1 >= 4 ? 1 << (s1 - 4) : 1;
  const int tpc_a = std::max(1, std::min(256 / tpt_a, 1 << s2));
  const size_t smem_a = sizeof(uint64_t) * (tpc_a * (size_t)((1 << s1) + ((1 << s1) >> 4) + 1) + 2) +
                        16 * (size_t)((1 << s1) - 1);
  if (!chunks_pick(inverse, false, s2) || (s1 && !cols_pick(inverse, false, s1)))
    return hd_fail(HD_E_PARAMS, "unsupported NTT size");
  if (!c->ntt_attr_set) {
    for (int k = 0; k < 4; k++) {
      for (int s = 4; s <= 12; s++)
        cudaFuncSetAttribute(chunks_pick(k & 1, k & 2, s), cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      for (int s = 5; s <= 8; s++)
        cudaFuncSetAttribute(cols_pick(k & 1, k & 2, s), cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    }
    c->ntt_attr_set = true;
  }
  // Rows by kind (R33): the map's modulus pattern repeats every mdiv * mlen rows; the positions
  // of FP64 rows (modulus < 2^45) and of integer rows within one period go to separate launches.
  // A map with a longer period runs every row on the integer kernels, and so does a small
  // batch (below HD_NTT_SPLIT_MIN rows, default 96): there the second launch pair costs more
  // than the FP64 butterflies save (launch-bound; C2's query 1.04 -> 1.29 ms when split).
  RowSel sel[2];
  const uint32_t period = map.mdiv * map.mlen;
  bool any[2] = {false, false};
  static const uint32_t split_min = [] {
    const char *e = getenv("HD_NTT_SPLIT_MIN");
    return e ? (uint32_t)atol(e) : 96u;
  }();
  bool one_kind_fp = false;  // every row of the map has a modulus below 2^45
  if (twd && period <= 64) {
    one_kind_fp = true;
    for (uint32_t p = 0; p < period; p++) one_kind_fp &= c->mod[map.midx[(p / map.mdiv) % map.mlen]] < kNttFp64Bound;
  }
  if (twd && period <= 64 && (rows >= split_min || one_kind_fp)) {
    for (int k = 0; k < 2; k++) {
      sel[k].period = period;
      sel[k].count = 0;
    }
    for (uint32_t p = 0; p < period; p++) {
      const int m = map.midx[(p / map.mdiv) % map.mlen];
      const int k = c->mod[m] < kNttFp64Bound ? 1 : 0;
      sel[k].pos[sel[k].count++] = (uint8_t)p;
    }
    for (int k = 0; k < 2; k++) any[k] = sel[k].count > 0;
    for (int k = 0; k < 2; k++)
      if (any[k] && !any[1 - k]) {  // one kind only: every row, no gaps
        sel[k].period = sel[k].count = 1;
        sel[k].pos[0] = 0;
      }
  } else {
    any[0] = true;  // sel[0]: identity
  }
  for (int k = 0; k < 2; k++) sel[k].fc = fdiv_make(std::max(1u, sel[k].count));
  // HD_NTT_CHUNK (A/B knob): rows per launch pair, so the intermediate of the two kernels stays
  // L2-resident.  Measured slower at 2^20 x 512 (96 rows: 61.4 vs 62.4 q/s; 24 rows: 55.4):
  // the kernels are issue-bound and the extra fill / drain costs more; default one batch.
  uint32_t chunk = 65535;
  if (const char *ce = getenv("HD_NTT_CHUNK"))
    if (atol(ce) > 0) chunk = (uint32_t)std::min(65535L, atol(ce));
  const uint32_t per = std::max(sel[0].period, sel[1].period);
  chunk = std::max(per, chunk - chunk % per);  // chunks start on a period boundary
  for (uint32_t r0 = 0; r0 < rows; r0 += chunk) {
    const uint32_t rr = rows - r0 < chunk ? rows - r0 : chunk;
    for (int k = 0; k < 2; k++) {
      if (!any[k]) continue;
      RowSel sk = sel[k];
      sk.end = r0 + rr;
      const uint32_t gy = (rr + sk.period - 1) / sk.period * sk.count;
      const double *tk = k ? twd : nullptr;
      chunks_kernel_t kb = chunks_pick(inverse, k, s2);
      cols_kernel_t ka = s1 ? cols_pick(inverse, k, s1) : nullptr;
      const dim3 ga(s1 ? (1u << s2) / tpc_a : 1, gy), gb((1u << s1) / tpc_b, gy);
      if (!inverse) {
        if (s1) {
          ka<<<ga, tpc_a * tpt_a, smem_a, c->stream>>>(data, map, c->mt, tw, logn, tpc_a, ninv, r0, false, src, tk, sk);
          ++c->launches;
        }
        kb<<<gb, tpc_b * tpt_b, smem_b, c->stream>>>(data, map, c->mt, tw, logn, tpc_b, ninv, r0, true,
                                                     s1 ? none_src : src, epi, tk, sk);
        ++c->launches;
      } else {
        kb<<<gb, tpc_b * tpt_b, smem_b, c->stream>>>(data, map, c->mt, tw, logn, tpc_b, ninv, r0, false, src,
                                                     none_epi, tk, sk);
        ++c->launches;
        if (s1) {
          ka<<<ga, tpc_a * tpt_a, smem_a, c->stream>>>(data, map, c->mt, tw, logn, tpc_a, ninv, r0, true, none_src,
                                                       tk, sk);
          ++c->launches;
        }
      }
    }
  }
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status ntt_rows(hd_context *c, uint64_t *base, uint32_t rows, const RowMap &rm, bool inverse) {
  return ntt_run(c, base, rows, rm, inverse, nullptr, nullptr);
}
