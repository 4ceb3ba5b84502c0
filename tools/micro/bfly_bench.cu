// Micro-benchmark of 64-bit Shoup butterfly variants (profiling aid, not part of libhd).
//   V0: __umul64hi quotient (exact), as ntt.cu
//   V1: truncated quotient a1 s1 + hi(a0 s1) + hi(a1 s0) (1 IMAD.WIDE + 2 IMAD.HI; error <= 2,
//       so t in [0, 4q)), one conditional subtraction brings t back to [0, 2q)
//   V2: exact quotient from 32-bit mad.lo/madc.hi carry chains (no IMAD.WIDE)
// Every variant runs the same butterfly network; outputs reduced to [0, q) must agree bit for bit.
#include <cstdint>
#include <cstdio>
#include <vector>
#include <random>

__device__ __forceinline__ uint64_t q_exact(uint64_t a, uint64_t s) { return __umul64hi(a, s); }
__device__ __forceinline__ uint64_t q_trunc(uint64_t a, uint64_t s) {
  uint64_t r;
  asm("{\n\t.reg .u32 a0, a1, s0, s1, x, y, z, c;\n\t"
      "mov.b64 {a0, a1}, %1;\n\t"
      "mov.b64 {s0, s1}, %2;\n\t"
      "mul.hi.u32 x, a0, s1;\n\t"
      "mul.hi.u32 y, a1, s0;\n\t"
      "add.cc.u32 z, x, y;\n\t"
      "addc.u32 c, 0, 0;\n\t"
      "mov.b64 %0, {z, c};\n\t"
      "mad.wide.u32 %0, a1, s1, %0;\n\t"
      "}"
      : "=l"(r) : "l"(a), "l"(s));
  return r;
}
__device__ __forceinline__ uint64_t q_chain(uint64_t a, uint64_t s) {
  uint32_t h0, h1;
  asm("{\n\t.reg .u32 a0, a1, s0, s1, t, m0, m1, m2;\n\t"
      "mov.b64 {a0, a1}, %2;\n\t"
      "mov.b64 {s0, s1}, %3;\n\t"
      "mul.hi.u32 t, a0, s0;\n\t"
      "mad.lo.cc.u32 m0, a0, s1, t;\n\t"
      "madc.hi.u32 m1, a0, s1, 0;\n\t"
      "mad.lo.cc.u32 m0, a1, s0, m0;\n\t"
      "madc.hi.cc.u32 m1, a1, s0, m1;\n\t"
      "addc.u32 m2, 0, 0;\n\t"
      "mad.lo.cc.u32 %0, a1, s1, m1;\n\t"
      "madc.hi.u32 %1, a1, s1, m2;\n\t"
      "}"
      : "=r"(h0), "=r"(h1) : "l"(a), "l"(s));
  return ((uint64_t)h1 << 32) | h0;
}


// V4: the whole lazy Shoup product in 32-bit PTX (exact quotient, carries on add.cc/addc)
__device__ __forceinline__ uint64_t mul_v4(uint64_t a, uint64_t w, uint64_t ws, uint64_t q) {
  uint32_t r0, r1;
  asm("{\n\t.reg .u32 a0, a1, s0, s1, w0, w1, q0, q1, t, m0, m1, m2, h0, h1, p0, p1, x0, x1;\n\t"
      "mov.b64 {a0, a1}, %2;\n\t"
      "mov.b64 {s0, s1}, %4;\n\t"
      "mov.b64 {w0, w1}, %3;\n\t"
      "mov.b64 {q0, q1}, %5;\n\t"
      // h = umulhi(a, ws)
      "mul.hi.u32 t, a0, s0;\n\t"
      "mad.lo.cc.u32 m0, a0, s1, t;\n\t"
      "madc.hi.u32 m1, a0, s1, 0;\n\t"
      "mad.lo.cc.u32 m0, a1, s0, m0;\n\t"
      "madc.hi.cc.u32 m1, a1, s0, m1;\n\t"
      "addc.u32 m2, 0, 0;\n\t"
      "mad.lo.cc.u32 h0, a1, s1, m1;\n\t"
      "madc.hi.u32 h1, a1, s1, m2;\n\t"
      // p = a * w mod 2^64
      "mul.lo.u32 p0, a0, w0;\n\t"
      "mul.hi.u32 p1, a0, w0;\n\t"
      "mad.lo.u32 p1, a0, w1, p1;\n\t"
      "mad.lo.u32 p1, a1, w0, p1;\n\t"
      // x = h * q mod 2^64
      "mul.lo.u32 x0, h0, q0;\n\t"
      "mul.hi.u32 x1, h0, q0;\n\t"
      "mad.lo.u32 x1, h0, q1, x1;\n\t"
      "mad.lo.u32 x1, h1, q0, x1;\n\t"
      "sub.cc.u32 %0, p0, x0;\n\t"
      "subc.u32 %1, p1, x1;\n\t"
      "}"
      : "=r"(r0), "=r"(r1) : "l"(a), "l"(w), "l"(ws), "l"(q));
  return ((uint64_t)r1 << 32) | r0;
}

template <int V>
__device__ __forceinline__ uint64_t mulw(uint64_t a, uint64_t w, uint64_t ws, uint64_t q, uint64_t two_q) {
  if (V == 0) return a * w - q_exact(a, ws) * q;
  if (V == 2) return a * w - q_chain(a, ws) * q;
  if (V == 4) return mul_v4(a, w, ws, q);
  uint64_t t = a * w - q_trunc(a, ws) * q;  // [0, 4q)
  return t >= two_q ? t - two_q : t;
}

template <int V, bool INV>
__global__ void __launch_bounds__(256, 3) k(uint64_t *v, const ulonglong2 *tw, uint64_t q, int n) {
  uint64_t x[16];
  const size_t base = (size_t)blockIdx.x * 256 * 16 + threadIdx.x;
  for (int i = 0; i < 16; i++) x[i] = v[base + i * 256];
  const uint64_t two_q = 2 * q;
#pragma unroll 1
  for (int it = 0; it < n; it++) {
#pragma unroll
    for (int u = 0; u < 4; u++) {
#pragma unroll
      for (int i = 0; i < 16; i++) {
        if (i & (1 << u)) continue;
        const int j = i + (1 << u);
        const ulonglong2 w = __ldg(&tw[(it * 4 + u) * 16 + i]);
        const uint64_t X = x[i], Y = x[j];
        if (!INV) {
          const uint64_t Xr = X >= two_q ? X - two_q : X;
          const uint64_t t = mulw<V>(Y, w.x, w.y, q, two_q);
          x[i] = Xr + t;
          x[j] = Xr - t + two_q;
        } else {
          const uint64_t a = X + Y;
          x[i] = a >= two_q ? a - two_q : a;
          x[j] = mulw<V>(X - Y + two_q, w.x, w.y, q, two_q);
        }
      }
    }
  }
  for (int i = 0; i < 16; i++) {
    uint64_t o = x[i];
    if (o >= two_q) o -= two_q;
    if (o >= q) o -= q;
    v[base + i * 256] = o;
  }
}


// V3: FP64 butterflies for moduli q < 2^46: values are doubles holding integers in a centred,
// unreduced representation; t = Y w mod q by an exact two-product (ph + pl = Y w) and a
// round-to-nearest quotient: t in about (-q, q).
__device__ __forceinline__ double mulmod_f(double y, double w, double q, double qinv) {
  const double M = 6755399441055744.0;  // 1.5 * 2^52: round to nearest integer
  const double ph = __dmul_rn(y, w);
  const double pl = __fma_rn(y, w, -ph);
  const double Q = __dsub_rn(__dadd_rn(__dmul_rn(ph, qinv), M), M);
  return __dadd_rn(__fma_rn(-Q, q, ph), pl);
}
__device__ __forceinline__ double red_f(double x, double q, double qinv) {
  const double M = 6755399441055744.0;
  const double Q = __dsub_rn(__dadd_rn(__dmul_rn(x, qinv), M), M);
  return __fma_rn(-Q, q, x);
}
template <bool INV>
__global__ void __launch_bounds__(256, 3) kf(uint64_t *v, const double2 *tw, uint64_t qi, int n) {
  double x[16];
  const double q = (double)qi, qinv = 1.0 / q;
  const size_t base = (size_t)blockIdx.x * 256 * 16 + threadIdx.x;
  for (int i = 0; i < 16; i++) x[i] = (double)v[base + i * 256];
#pragma unroll 1
  for (int it = 0; it < n; it++) {
    if (INV) {
#pragma unroll
      for (int i = 0; i < 16; i++) x[i] = red_f(x[i], q, qinv);
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
#pragma unroll
      for (int i = 0; i < 16; i++) {
        if (i & (1 << u)) continue;
        const int j = i + (1 << u);
        const double w = __ldg(&tw[(it * 4 + u) * 16 + i]).x;
        const double X = x[i], Y = x[j];
        if (!INV) {
          const double t = mulmod_f(Y, w, q, qinv);
          x[i] = __dadd_rn(X, t);
          x[j] = __dsub_rn(X, t);
        } else {
          x[i] = __dadd_rn(X, Y);
          x[j] = mulmod_f(__dsub_rn(X, Y), w, q, qinv);
        }
      }
    }
    if (!INV) {  // forward growth bound: reduce X every 4 passes in this synthetic loop
      if ((it & 3) == 3) {
#pragma unroll
        for (int i = 0; i < 16; i++) x[i] = red_f(x[i], q, qinv);
      }
    }
  }
  for (int i = 0; i < 16; i++) {
    double r = red_f(x[i], q, qinv);
    if (r < 0) r = __dadd_rn(r, q);
    v[base + i * 256] = (uint64_t)r;
  }
}

static uint64_t mulmod_h(uint64_t a, uint64_t b, uint64_t m) { return (unsigned __int128)a * b % m; }

int main() {
  const uint64_t qs[2] = {1152921504606584833ull /* < 2^60 */, 35184372088833ull /* 2^45 + 1? any odd */};
  const int blocks = 148 * 3 * 8, n = 64;
  const size_t N = (size_t)blocks * 256 * 16;
  uint64_t *d;
  ulonglong2 *tw;
  cudaMalloc(&d, N * 8);
  cudaMalloc(&tw, 4 * n * 16 * 16);
  for (int qi = 0; qi < 2; qi++) {
    const uint64_t q = qs[qi];
    std::mt19937_64 g(1);
    std::vector<ulonglong2> T(4 * n * 16);
    for (auto &t : T) {
      t.x = g() % q;
      t.y = (uint64_t)(((unsigned __int128)t.x << 64) / q);
    }
    cudaMemcpy(tw, T.data(), T.size() * 16, cudaMemcpyHostToDevice);
    std::vector<uint64_t> H(N), R[5];
    for (auto &h : H) h = g() % q;
    for (int inv = 0; inv < 2; inv++) {
      for (int V = 0; V < 5; V++) {
        if (V == 3) continue;
        cudaMemcpy(d, H.data(), N * 8, cudaMemcpyHostToDevice);
        auto kern = inv ? (V == 0 ? k<0, true> : V == 1 ? k<1, true> : V == 2 ? k<2, true> : k<4, true>)
                        : (V == 0 ? k<0, false> : V == 1 ? k<1, false> : V == 2 ? k<2, false> : k<4, false>);
        kern<<<blocks, 256>>>(d, tw, q, 1);  // warm
        cudaMemcpy(d, H.data(), N * 8, cudaMemcpyHostToDevice);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        kern<<<blocks, 256>>>(d, tw, q, n);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        R[V].resize(N);
        cudaMemcpy(R[V].data(), d, N * 8, cudaMemcpyDeviceToHost);
        const double bfly = (double)blocks * 256 * n * 4 * 8;
        printf("q%d %s V%d: %.3f ms  %.1f Gbfly/s  %s\n", qi, inv ? "inv" : "fwd", V, ms, bfly / ms / 1e6,
               V && R[V] != R[0] ? "MISMATCH" : "ok");
      }
    }
  }

  {  // FP64 variant at a 45-bit modulus vs V0
    const uint64_t q = 35184372088833ull - 2;  // < 2^45
    std::mt19937_64 g(7);
    std::vector<ulonglong2> T(4 * n * 16);
    std::vector<double2> TD(4 * n * 16);
    for (size_t i = 0; i < T.size(); i++) {
      T[i].x = g() % q;
      T[i].y = (uint64_t)(((unsigned __int128)T[i].x << 64) / q);
      TD[i].x = (double)T[i].x;
      TD[i].y = 0;
    }
    double2 *twd;
    cudaMalloc(&twd, TD.size() * 16);
    cudaMemcpy(twd, TD.data(), TD.size() * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(tw, T.data(), T.size() * 16, cudaMemcpyHostToDevice);
    std::vector<uint64_t> H(N), R0(N), R3(N);
    for (auto &h : H) h = g() % q;
    for (int inv = 0; inv < 2; inv++) {
      for (int V = 0; V < 2; V++) {
        auto kern0 = inv ? k<0, true> : k<0, false>;
        auto kern3 = inv ? kf<true> : kf<false>;
        cudaMemcpy(d, H.data(), N * 8, cudaMemcpyHostToDevice);
        if (V == 0) kern0<<<blocks, 256>>>(d, tw, q, 1); else kern3<<<blocks, 256>>>(d, twd, q, 1);
        cudaMemcpy(d, H.data(), N * 8, cudaMemcpyHostToDevice);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        if (V == 0) kern0<<<blocks, 256>>>(d, tw, q, n); else kern3<<<blocks, 256>>>(d, twd, q, n);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        cudaMemcpy((V ? R3 : R0).data(), d, N * 8, cudaMemcpyDeviceToHost);
        const double bfly = (double)blocks * 256 * n * 4 * 8;
        printf("q45 %s %s: %.3f ms  %.1f Gbfly/s  %s\n", inv ? "inv" : "fwd", V ? "FP64" : "V0", ms, bfly / ms / 1e6,
               V && R3 != R0 ? "MISMATCH" : "ok");
      }
    }
  }
  (void)mulmod_h;
  return 0;
}
