// common.cuh -- shared device arithmetic and host plumbing of libhd (sm_100a).
//
// Moduli are < 2^61 (q0, P ~ 2^60; q1, q2 ~ 2^45; R5), so lazy sums of
// up to 4 reduced values fit in 64 bits.  Multiplication by a fixed operand uses
// Shoup's precomputed quotient; products of two variable operands are
// accumulated exactly in 128 bits and reduced once (reduce128).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hd.h"

#define HD_MAXMOD 20  // q_0..q_{L-1} and the K special primes (paper-depth profile: 12 + 4)

// ---------------------------------------------------------------------------
// Per-modulus constants, passed to kernels by value.
// ---------------------------------------------------------------------------
// Moduli below this bound run the FP64 NTT butterflies of ntt.cu (R33).
constexpr uint64_t kNttFp64Bound = 1ull << 45;

struct ModTab {
  uint64_t q[HD_MAXMOD];
  uint64_t bar[HD_MAXMOD];   // floor(2^64 / q)
  uint64_t r64[HD_MAXMOD];   // 2^64 mod q
  uint64_t r64s[HD_MAXMOD];  // Shoup companion of r64
};

struct InvTab2 {
  uint64_t w[HD_MAXMOD];
};

// Division by a runtime divisor d without the ~25-instruction integer division: a shift
// when d is a power of two, else floor(r / d) = floor(r m / 2^48) with m = floor(2^48/d)+1,
// exact for r < 2^31 and d < 2^17 (error < r / 2^48 < 1/d); other d divide plainly.
struct FDiv {
  uint64_t m = 0;
  uint32_t d = 1;
  int32_t sh = 0;  // >= 0: shift; -1: multiply-high; -2: plain division
};
inline FDiv fdiv_make(uint32_t d) {
  FDiv f;
  f.d = d ? d : 1;
  if ((f.d & (f.d - 1)) == 0) {
    f.sh = 0;
    while ((1u << f.sh) < f.d) f.sh++;
  } else if (f.d < (1u << 17)) {
    f.sh = -1;
    f.m = (uint64_t)((((unsigned __int128)1) << 48) / f.d) + 1;
  } else {
    f.sh = -2;
  }
  return f;
}
__host__ __device__ __forceinline__ uint32_t fdiv_q(uint32_t r, const FDiv &f) {
#ifdef __CUDA_ARCH__
  if (f.sh >= 0) return r >> f.sh;
  if (f.sh == -1) return (uint32_t)__umul64hi((uint64_t)r << 16, f.m);
#endif
  return r / f.d;
}

// Row addressing for batched kernels: row r lives at
//   base + (r / gsize) * gstride + ((r % gsize) / g2) * s2 + (r % g2) * s3   (s3 == 0 means n)
// and is reduced modulo q[midx[(r / mdiv) % mlen]].  Defaults (g2 = gsize, s3 = 0)
// give base + (r / gsize) * gstride + (r % gsize) * n.
struct RowMap {
  uint32_t gsize = 1u << 30;
  uint32_t mdiv = 1, mlen = 1;
  uint32_t g2 = 1u << 30;
  uint64_t gstride = 0, s2 = 0, s3 = 0;
  uint8_t midx[64] = {0};  // ell*ell ModUp rows up to ell = 7 (L = 7, HD_MAXMOD 8)
  // fast divisors for gsize, min(g2, gsize), mdiv, mlen (rowmap_finalize; device use only)
  bool fast = false;
  FDiv fg, fg2, fmd, fml;
};
inline void rowmap_finalize(RowMap &rm) {
  rm.fg = fdiv_make(rm.gsize);
  rm.fg2 = fdiv_make(rm.g2 < rm.gsize ? rm.g2 : rm.gsize);
  rm.fmd = fdiv_make(rm.mdiv);
  rm.fml = fdiv_make(rm.mlen);
  rm.fast = true;
}

// ---------------------------------------------------------------------------
// Device arithmetic
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mulhi64(uint64_t a, uint64_t b) { return __umul64hi(a, b); }

// a * w mod q with Shoup companion ws = floor(w 2^64 / q); result in [0, 2q).
__device__ __forceinline__ uint64_t shoup_lazy(uint64_t a, uint64_t w, uint64_t ws, uint64_t q) {
  uint64_t qh = __umul64hi(a, ws);
  return a * w - qh * q;
}
__device__ __forceinline__ uint64_t shoup(uint64_t a, uint64_t w, uint64_t ws, uint64_t q) {
  uint64_t r = shoup_lazy(a, w, ws, q);
  return r >= q ? r - q : r;
}
// x mod q for any 64-bit x; bar = floor(2^64/q).
__device__ __forceinline__ uint64_t reduce64(uint64_t x, uint64_t q, uint64_t bar) {
  uint64_t r = x - __umul64hi(x, bar) * q;  // [0, 2q)
  return r >= q ? r - q : r;
}
// (hi 2^64 + lo) mod q.
__device__ __forceinline__ uint64_t reduce128(uint64_t hi, uint64_t lo, uint64_t q, uint64_t bar,
                                              uint64_t r64, uint64_t r64s) {
  uint64_t t = shoup_lazy(hi, r64, r64s, q);     // [0, 2q)
  uint64_t u = lo - __umul64hi(lo, bar) * q;     // [0, 2q)
  uint64_t s = t + u;                            // < 4q < 2^63
  if (s >= 2 * q) s -= 2 * q;
  if (s >= q) s -= q;
  return s;
}
__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b, const ModTab &M, int m) {
  return reduce128(__umul64hi(a, b), a * b, M.q[m], M.bar[m], M.r64[m], M.r64s[m]);
}
__device__ __forceinline__ uint64_t addmod(uint64_t a, uint64_t b, uint64_t q) {
  uint64_t s = a + b;
  return s >= q ? s - q : s;
}
__device__ __forceinline__ uint64_t submod(uint64_t a, uint64_t b, uint64_t q) {
  return a >= b ? a - b : a + q - b;
}
// 128-bit accumulate acc += a*b (exact).
__device__ __forceinline__ void mac128(uint64_t &lo, uint64_t &hi, uint64_t a, uint64_t b) {
  uint64_t plo = a * b, phi = __umul64hi(a, b);
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(plo), "l"(phi));
}
// Karatsuba accumulation (R35).  With r = rl + rh 2^31 and d = dl + dh 2^31 (rl, dl < 2^31;
// rh < 2^29 for residues below 2^60, dh < 2^16 for a packed narrow limb),
//   r d = rl dl + ((rl + rh)(dl + dh) - rl dl - rh dh) 2^31 + rh dh 2^62,
// and (rl + rh), (dl + dh) < 2^32.  The three products are summed over the baby steps
// separately (the identity is linear) and combined once per unit: 2 IMAD.WIDE + 1 IMAD per
// product for a narrow limb (rh dh < 2^32), 3 IMAD.WIDE for a wide one, against the 4
// IMAD.WIDE of the schoolbook 32-bit split -- the MAC's compute is bound by that pipe.
// Sums: s0 = sum rl dl and sm = sum (rl+rh)(dl+dh) as 64-bit words plus 32-bit carry counts
// (< 2^71 for 128 terms), s2 = sum rh dh likewise (narrow: < 2^32 per term).
struct KAcc {
  uint64_t s0, sm, s2;
  uint32_t c0, cm, c2;
};
template <bool NARROW>
__device__ __forceinline__ void kmac(KAcc &A, uint32_t rl, uint32_t rh, uint32_t rs, uint32_t dl, uint32_t dh,
                                     uint32_t ds) {
  asm("{\n\t.reg .u64 t;\n\t"
      "mul.wide.u32 t, %4, %6;\n\t"
      "add.cc.u64 %0, %0, t;\n\t"
      "addc.u32 %2, %2, 0;\n\t"
      "mul.wide.u32 t, %5, %7;\n\t"
      "add.cc.u64 %1, %1, t;\n\t"
      "addc.u32 %3, %3, 0;\n\t"
      "}"
      : "+l"(A.s0), "+l"(A.sm), "+r"(A.c0), "+r"(A.cm)
      : "r"(rl), "r"(rs), "r"(dl), "r"(ds));
  if (NARROW) {
    asm("{\n\t.reg .u32 l, h;\n\t"
        "mov.b64 {l, h}, %0;\n\t"
        "mad.lo.cc.u32 l, %1, %2, l;\n\t"
        "addc.u32 h, h, 0;\n\t"
        "mov.b64 %0, {l, h};\n\t"
        "}"
        : "+l"(A.s2)
        : "r"(rh), "r"(dh));
  } else {
    asm("{\n\t.reg .u64 t;\n\t"
        "mul.wide.u32 t, %2, %3;\n\t"
        "add.cc.u64 %0, %0, t;\n\t"
        "addc.u32 %1, %1, 0;\n\t"
        "}"
        : "+l"(A.s2), "+r"(A.c2)
        : "r"(rh), "r"(dh));
  }
}
// sum r d = s0 + (sm - s0 - s2) 2^31 + s2 2^62 (< 2^127 for 128 terms below 2^60) mod q
__device__ __forceinline__ uint64_t kacc_reduce(const KAcc &A, uint64_t q, uint64_t bar, uint64_t r64,
                                                uint64_t r64s) {
  const unsigned __int128 x0 = ((unsigned __int128)A.c0 << 64) | A.s0;
  const unsigned __int128 xm = ((unsigned __int128)A.cm << 64) | A.sm;
  const unsigned __int128 x2 = ((unsigned __int128)A.c2 << 64) | A.s2;
  const unsigned __int128 x = x0 + ((xm - x0 - x2) << 31) + (x2 << 62);
  return reduce128((uint64_t)(x >> 64), (uint64_t)x, q, bar, r64, r64s);
}

// r d (r, d < 2^60; narrow: both < 2^47) into a Karatsuba sum, splitting both at bit 31
template <bool NARROW>
__device__ __forceinline__ void kmac64(KAcc &A, uint64_t r, uint64_t d) {
  const uint32_t rl = (uint32_t)r & 0x7fffffffu, rh = (uint32_t)(r >> 31);
  const uint32_t dl = (uint32_t)d & 0x7fffffffu, dh = (uint32_t)(d >> 31);
  kmac<NARROW>(A, rl, rh, rl + rh, dl, dh, dl + dh);
}

// centred lift (R12) of x in [0, qs) into modulus m (bar_m = floor(2^64/m)).
__device__ __forceinline__ uint64_t lift_centred(uint64_t x, uint64_t qs, uint64_t m, uint64_t bar_m) {
  // branch-free (no divergence): reduce |centred x|, negate when x > qs/2
  const bool neg = x > (qs >> 1);
  const uint64_t r = reduce64(neg ? qs - x : x, m, bar_m);
  return neg ? (r ? m - r : 0) : r;
}
// Galois index map in the NTT domain (R11): out[t] = in[pi_g(t)],
// pi_g(t) = br(((g (2 br(t) + 1)) mod 2n - 1) / 2).
__device__ __forceinline__ uint32_t galois_src(uint32_t t, uint32_t g, int logn) {
  uint32_t bt = __brev(t) >> (32 - logn);
  uint32_t mask = (2u << logn) - 1u;  // mod 2n
  uint32_t e = (uint32_t)(((uint64_t)g * (2u * bt + 1u)) & mask);
  return __brev((e - 1u) >> 1) >> (32 - logn);
}

__host__ __device__ __forceinline__ uint64_t row_off(const RowMap &rm, uint32_t r, uint32_t n) {
  const uint32_t g2 = rm.g2 < rm.gsize ? rm.g2 : rm.gsize;
  if (rm.fast) {
    const uint32_t gq = fdiv_q(r, rm.fg), in = r - gq * rm.gsize;
    const uint32_t q2 = fdiv_q(in, rm.fg2), i2 = in - q2 * g2;
    return (uint64_t)gq * rm.gstride + (uint64_t)q2 * rm.s2 + (uint64_t)i2 * (rm.s3 ? rm.s3 : n);
  }
  const uint32_t in = r % rm.gsize;
  return (uint64_t)(r / rm.gsize) * rm.gstride + (uint64_t)(in / g2) * rm.s2 + (uint64_t)(in % g2) * (rm.s3 ? rm.s3 : n);
}
__device__ __forceinline__ uint64_t *row_ptr(uint64_t *base, const RowMap &rm, uint32_t r, uint32_t n) {
  return base + row_off(rm, r, n);
}
__device__ __forceinline__ int row_mod(const RowMap &rm, uint32_t r) {
  if (rm.fast) {
    const uint32_t a = fdiv_q(r, rm.fmd);
    return rm.midx[a - fdiv_q(a, rm.fml) * rm.mlen];
  }
  return rm.midx[(r / rm.mdiv) % rm.mlen];
}

// ---------------------------------------------------------------------------
// Host-side context (C++ only).
// ---------------------------------------------------------------------------
struct hd_context {
  hd_params params;
  int device = 0;
  cudaStream_t stream = nullptr;
  int logn = 0, n = 0, ns = 0, L = 0;
  int K = 1, alpha = 1;  // special primes, limbs per key-switching digit (R11; general: R31)
  uint64_t mod[HD_MAXMOD] = {0};  // q_0..q_{L-1}, P at index L
  uint64_t psi[HD_MAXMOD] = {0};
  ModTab mt;
  // device tables
  uint64_t *tw2 = nullptr, *itw2 = nullptr;  // [L+1][n] x {w, shoup(w)}: psi^{br(k)}, psi^{-br(k)}
  uint64_t *ninv_dev = nullptr;              // [2 HD_MAXMOD]: n^{-1} mod q_l, then Shoup companions
  // the same twiddles as doubles (exact: moduli below 2^45 only, else 0) for the FP64
  // butterflies of ntt.cu (R33)
  double *twd = nullptr, *itwd = nullptr;  // [L+K][n]
  bool ntt_attr_set = false;
  uint64_t ninv[HD_MAXMOD], ninvs[HD_MAXMOD];
  double *xi_re = nullptr, *xi_im = nullptr;  // [2n]: xi^t, R15
  uint32_t *rotg = nullptr;                   // [ns]: 5^j mod 2n
  // scratch (grown on demand at setup time only)
  void *scratch = nullptr;
  size_t scratch_bytes = 0;
  int *d_flag = nullptr;  // device error flag
constexpr static int kPhaseEvents = 9;
  cudaEvent_t ev[64][kPhaseEvents] = {};  // per-query phase events (ring of 64 queries)
  int ev_next = 0, ev_pending = 0;
  double last_phase_ms[6] = {0, 0, 0, 0, 0, 0};
  uint64_t launches = 0;  // kernels launched on this context (hd_launch_count)
  cudaStream_t sA = nullptr, sB = nullptr;  // internal streams of the query pipeline
  cudaStream_t sIO = nullptr;               // device->host result downloads (export_async)
  cudaStream_t sUp = nullptr;               // host->device uploads (import_into from host)
  // Device memory: the caller's allocator (the torch caching allocator in the
  // Python binding) or, without one, the device's stream-ordered pool (cudaMallocAsync).
  hd_allocator alloc{};
  bool has_alloc = false;
  // Stream-ordered workspace cache for per-call temporaries (hd_compare): blocks freed by a
  // call are reused by the next one on the same stream without touching the allocator.
  struct WsBlock {
    void *p;
    size_t bytes;
    cudaStream_t stream;
  };
  std::vector<WsBlock> ws_free;
  // lifetime: 1 for the caller's handle + 1 per live object made by this context (keys,
  // ciphertexts, databases); hd_context_destroy drops the caller's reference and the tables
  // go when the last object goes, so objects may be destroyed in any order (e.g. by a GC)
  int refs = 1;
};
void ctx_retain(hd_context *c);
void ctx_release(hd_context *c);

// Key-switching geometry (R11, R31).  Extended basis of a ciphertext at ell limbs: ext index
// e < ell is q_e, e >= ell the special prime p_{e-ell} (modulus index L + e - ell); a key
// holds beta(L) digits over the M = L + K moduli.  The alpha = K = 1 profile (the north-star
// scan) keeps its fused single-limb lifts; any other profile runs the general conversions.
inline bool ks_general(const hd_context *c) { return c->K != 1 || c->alpha != 1; }
inline int ks_M(const hd_context *c) { return c->L + c->K; }
inline int ks_beta(const hd_context *c, int ell) { return (ell + c->alpha - 1) / c->alpha; }
inline int ks_ext_mod(const hd_context *c, int ell, int e) { return e < ell ? e : c->L + (e - ell); }
// ModUp digit rows per ciphertext: alpha = K = 1 keeps ell slots per digit (the own limb is
// read from c1), the general layout every one of the ell + K moduli per digit
inline size_t ks_dig_elems(const hd_context *c, int ell) {
  return ks_general(c) ? (size_t)ks_beta(c, ell) * (ell + c->K) * c->n : (size_t)ell * ell * c->n;
}
inline size_t ks_key_elems(const hd_context *c) { return (size_t)ks_beta(c, c->L) * 2 * ks_M(c) * c->n; }
uint64_t ks_P_mod(const hd_context *c, uint64_t q);  // prod_k p_k mod q (host)

// Every device allocation of the library goes through these (no other cudaMalloc).
// dev_alloc / dev_free: long-lived objects; dev_free first waits for the context's streams
// (the memory may still be read by the query pipeline).  ws_alloc / ws_free: stream-ordered
// temporaries of one call on c->stream, cached per context (never returned mid-run).
cudaError_t dev_alloc(hd_context *c, void **p, size_t bytes);
void dev_free(hd_context *c, void *p);
void *ws_alloc(hd_context *c, size_t bytes);
void ws_free(hd_context *c, void *p, size_t bytes);
template <class T>
static inline cudaError_t dev_alloc(hd_context *c, T **p, size_t bytes) {
  return dev_alloc(c, reinterpret_cast<void **>(p), bytes);
}

struct hd_secret_key {
  hd_context *ctx;
  uint64_t *s_ntt;  // [(L+1)][n]
};

// process-unique generation ids: a key set gets a fresh one whenever its storage is
// (re)allocated, so caches keyed on it never outlive the storage (no address ABA)
uint64_t hd_next_generation();

struct hd_eval_keys {
  hd_context *ctx;
  std::vector<int32_t> steps;
  uint64_t *keys = nullptr;  // [count][L][2][L+1][n]
  size_t key_elems = 0;      // per key
  uint64_t gen = hd_next_generation();
  const uint64_t *find(int32_t step) const {
    for (size_t i = 0; i < steps.size(); i++)
      if (steps[i] == step) return keys + key_elems * i;
    return nullptr;
  }
};

// Public key (encrypted-database mode, R26): pk = (b, a) over the L ciphertext moduli.
struct hd_public_key {
  hd_context *ctx;
  uint64_t *pk;  // [2][L][n], NTT form
};

// Relinearisation key (s^2 -> s) stored in hd_eval_keys under this reserved step.
constexpr int32_t HD_RELIN_STEP = 0;

struct hd_ciphertext {
  hd_context *ctx;
  uint32_t limbs;
  uint64_t *data;                 // [2][limbs][n]
  double scale = 0.0;             // CKKS scale of the message (2^scale_bits unless an
                                  // evaluation changed it, R29)
  cudaEvent_t ready = nullptr;    // recorded by the last writer (any stream); readers wait on it
  cudaEvent_t used = nullptr;     // recorded by the last asynchronous reader (export_async);
                                  // writers wait on it before overwriting data
};

// Packed plaintext diagonals (R34).  A residue of a limb whose modulus is below 2^47
// ("narrow": the 45-bit scaling limbs) is stored in 6 bytes, not 8: bits 0..30 in a u32 low
// plane, bits 31..46 in a u16 high plane (the 31-bit split is the one the MAC's Karatsuba
// products use); other limbs ("wide") stay u64 words.  One diagonal is
//   [wide limbs: W x n u64][narrow low planes: R x n u32][narrow high planes: R x n u16]
// = (8 W + 6 R) n bytes (20 n instead of 24 n at L = 3).  Unpacked: W = L, R = 0.
constexpr uint64_t kNarrowBound = 1ull << 47;
struct DPack {
  bool on = false;
  int W = 0, R = 0;
  int polys = 1;                 // 2: encrypted diagonals, one packed block per polynomial
  uint8_t cls[HD_MAXMOD] = {0};  // 0 wide, 1 narrow
  uint8_t idx[HD_MAXMOD] = {0};  // position within its class
  size_t pp_bytes = 0;           // one polynomial: (8 W + 6 R) n
  size_t diag_bytes = 0;         // one diagonal: polys x pp_bytes
};
DPack dpack_make(const hd_context *c, bool on, int polys = 1);
__host__ __device__ __forceinline__ uint64_t dp_get(const uint8_t *diag, const DPack &P, int limb, size_t t, size_t n) {
  if (!P.cls[limb]) return reinterpret_cast<const uint64_t *>(diag)[(size_t)P.idx[limb] * n + t];
  const uint32_t lo = reinterpret_cast<const uint32_t *>(diag + 8 * (size_t)P.W * n)[(size_t)P.idx[limb] * n + t];
  const uint16_t hi =
      reinterpret_cast<const uint16_t *>(diag + (8 * (size_t)P.W + 4 * (size_t)P.R) * n)[(size_t)P.idx[limb] * n + t];
  return lo | ((uint64_t)hi << 31);
}
__host__ __device__ __forceinline__ void dp_put(uint8_t *diag, const DPack &P, int limb, size_t t, size_t n,
                                                uint64_t v) {
  if (!P.cls[limb]) {
    reinterpret_cast<uint64_t *>(diag)[(size_t)P.idx[limb] * n + t] = v;
    return;
  }
  reinterpret_cast<uint32_t *>(diag + 8 * (size_t)P.W * n)[(size_t)P.idx[limb] * n + t] = (uint32_t)(v & 0x7fffffffu);
  reinterpret_cast<uint16_t *>(diag + (8 * (size_t)P.W + 4 * (size_t)P.R) * n)[(size_t)P.idx[limb] * n + t] =
      (uint16_t)(v >> 31);
}

struct hd_database {
  hd_context *ctx;
  hd_layout lay;
  uint32_t N, M, n1, A_loc;
  std::vector<int32_t> js;       // giant steps j (contiguous, non-empty ranges)
  std::vector<int32_t> pre;      // preRot(j) per j
  uint64_t *D = nullptr;         // [A_loc][N][L][n] diagonal plaintexts (packed: [A_loc][N] x
                                 // dp.diag_bytes, R34), or [A_loc][N][2][L][n] diagonal
                                 // ciphertexts (encrypted; never packed)
  DPack dp;                      // packing of the plaintext diagonals
  bool encrypted = false;        // encrypted-database mode (NEXT-1, R26)
  bool flat = false;             // flat pre-rotated packing (NEXT-2, R27): no fold
  bool needs_prerotation = false;  // FLAT_TBS before hd_database_prerotate
  uint32_t spoly = 2;            // polynomials per giant-step sum: 2, or 3 (degree 2) encrypted
  // query workspaces (allocated at enrollment; reused by every hd_query)
  uint64_t *r = nullptr;         // [n1][2][L][n] baby steps
  uint64_t *S = nullptr;         // [A_loc][nj][spoly][L][n] giant-step sums
  uint64_t *Sp = nullptr;        // [A_loc][nj][2][L-1][n] rescaled
  uint64_t *y = nullptr;         // [A_loc][2][L-1][n]
  uint64_t *outbuf = nullptr;    // [A_loc][2][L-1][n] folded outputs
  uint64_t *dig = nullptr;       // ModUp digits
  uint64_t *u = nullptr;         // KIP output
  uint64_t *tmp = nullptr;       // INTT / lift scratch
  uint64_t *tmp2 = nullptr;      // rescale scratch
  uint32_t rescale_chunk = 1;
  // two-stream pipeline (query.cu): baby steps + MAC of query q+1 on stream A overlap the
  // rescale / giant / fold of query q on stream B; S is double-buffered.
  uint64_t *S2 = nullptr;                                  // second giant-sum buffer
  uint64_t *dig_b = nullptr, *u_b = nullptr, *tmp_b = nullptr;  // baby-step scratch (stream A)
  uint64_t qcount = 0;
  // query batching (NEXT-4, hd_query_batch): baby steps of Q queries and their giant-step
  // sums (double-buffered), allocated on the first batch of a given size
  uint64_t *rB = nullptr, *SB[2] = {nullptr, nullptr};
  uint32_t qb_cap = 0;
  cudaEvent_t ev_in = nullptr, ev_mac = nullptr, ev_done = nullptr, ev_sfree[2] = {nullptr, nullptr};
  // last hd_baby_steps on the caller's stream: the next scan's stream A waits on it before
  // reusing the baby-step workspaces (dig_b, u_b, tmp_b)
  cudaEvent_t ev_bs = nullptr;
  bool bs_pending = false;
  // rotation-key tables for the (db, evk) pair last used: [0, n1-1) baby i = 1..n1-1,
  // [n1-1, n1-1+nj) giant j (NULL key when preRot = 0), [n1-1+nj] fold
  // [n1+nj] relinearisation key (encrypted mode), gal 1 (identity permutation)
  const hd_eval_keys *keyed_for = nullptr;
  uint64_t keyed_gen = 0;        // hd_eval_keys::gen of the bound key storage
  const uint64_t **kptr = nullptr;
  uint32_t *gal = nullptr;
  uint32_t relin_chunk = 1;      // giant-step sums relinearised per batch (encrypted mode)
  size_t bytes = 0;
  bool has_run = false;
};

// error plumbing
hd_status hd_fail(hd_status s, const std::string &msg);
#define HD_CUDA(call)                                                                     \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) return hd_fail(HD_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// kernels / host drivers (defined in the .cu files)
hd_status ntt_rows(hd_context *c, uint64_t *base, uint32_t rows, const RowMap &rm, bool inverse);

// Fused NTT jobs (ntt.cu).  The first kernel of the transform may read its input from
// another row map (out-of-place), optionally lifting the centred representative of a
// coefficient-form residue mod q[row_mod(src.map, r)] into the row's modulus (R12); the
// final forward store may combine: out[r] (=|+=) (A[r] - v) * w[l] (+ c0 permuted by the
// Galois map, for p == 0), rows r = (x 2 + p) ell + l.
struct NttSrc {
  const uint64_t *base = nullptr;
  RowMap map;
  bool lift = false;
};
struct NttEpi {
  int mode = 0;  // 0: none, 1: (A - v) w, 2: (A - v) w + pi_g(c0) on p == 0
  bool acc = false;
  int ell = 1, K = 1;
  const uint64_t *A = nullptr;
  RowMap amap;
  uint64_t *out = nullptr;
  RowMap omap;
  const uint64_t *c0 = nullptr;
  uint64_t c0_stride = 0;
  const uint32_t *gal = nullptr;
  uint64_t w[HD_MAXMOD] = {0}, ws[HD_MAXMOD] = {0};
  FDiv fell, f2ell, fK;  // ell, 2 ell, K (set by ntt_run)
};
hd_status ntt_run(hd_context *c, uint64_t *data, uint32_t rows, const RowMap &map, bool inverse, const NttSrc *src,
                  const NttEpi *epi);
RowMap rowmap_simple(uint32_t mdiv, std::initializer_list<int> mods, uint32_t gsize = 1u << 30,
                     uint64_t gstride = 0);
uint64_t host_mulmod(uint64_t a, uint64_t b, uint64_t m);
uint64_t host_powmod(uint64_t b, uint64_t e, uint64_t m);
uint64_t host_shoup(uint64_t w, uint64_t q);
