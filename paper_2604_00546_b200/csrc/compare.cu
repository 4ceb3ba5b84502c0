// compare.cu -- encrypted comparison and the scenario tails (NEXT-3, R29).
//
// ChebyshevCompare (Alg. gpu-chebyshev): f(x) = 1/2 (sign(x - delta) + 1)
// approximated by a degree-n Chebyshev series evaluated with Paterson-Stockmeyer in the
// Chebyshev basis; identification = compare every score ciphertext (Alg. index,
// P:L1541-1560); membership = sum of the comparisons + RotateAndSum (Alg. membership,
// P:L1513-1537).
//
// B200 design: every homomorphic operation of the evaluation runs ONCE over a batch of
// ciphertexts (all aggregates of a query follow the same schedule), so each step is one
// launch over B x 2 x ell x n residues: the tensor / linear-combination kernels are
// elementwise HBM streams, relinearisation and rescale reuse the batched key-switching
// NTT pipeline of ks.cu (the relinearisation key is read once per product for the whole
// batch).  MatchLevel is free: every kernel reads its operands with their own limb count
// as the layout stride and the target count as the extent.
#include <cmath>
#include <memory>

#include "ks.cuh"

namespace {

constexpr int CTPB = 256;

// out[b][p][l][t] = ka_l a + kb_l b (+ kc_l on p == 0), a/b read with layout limbs la/lb.
struct Lin {
  uint64_t ka[HD_MAXMOD], kb[HD_MAXMOD], kc[HD_MAXMOD];
};

// Grid (n / CTPB, ell, 2 B): no runtime divisions; a unit multiplier skips its product.
__global__ void __launch_bounds__(CTPB) lincomb_kernel(const uint64_t *__restrict__ a, int la,
                                                       const uint64_t *__restrict__ b, int lb,
                                                       uint64_t *__restrict__ out, int ell, int logn, Lin k,
                                                       ModTab mt) {
  const uint32_t n = 1u << logn, t = blockIdx.x * CTPB + threadIdx.x, l = blockIdx.y, bp = blockIdx.z;
  if (t >= n) return;
  const uint32_t p = bp & 1;
  const uint64_t q = mt.q[l], ka = k.ka[l], kb = k.kb[l];
  const uint64_t av = a[((size_t)bp * la + l) * n + t];
  uint64_t v = ka == 1 ? av : mulmod(av, ka, mt, l);
  if (b) {
    const uint64_t bv = b[((size_t)bp * lb + l) * n + t];
    v = addmod(v, kb == 1 ? bv : (kb == q - 1 ? (bv ? q - bv : 0) : mulmod(bv, kb, mt, l)), q);
  }
  if (p == 0) v = addmod(v, k.kc[l], q);
  out[((size_t)bp * ell + l) * n + t] = v;
}

// Tensor product of B ciphertext pairs at ell limbs: out [B][3][ell][n] =
// (a0 b0, a0 b1 + a1 b0, a1 b1), operands read with layout limbs la / lb (MatchLevel).
// Grid (n / CTPB, ell, B).
__global__ void __launch_bounds__(CTPB) tensor_kernel(const uint64_t *__restrict__ a, int la,
                                                      const uint64_t *__restrict__ b, int lb,
                                                      uint64_t *__restrict__ out, int ell, int logn, ModTab mt) {
  const uint32_t n = 1u << logn, t = blockIdx.x * CTPB + threadIdx.x, l = blockIdx.y, bb = blockIdx.z;
  if (t >= n) return;
  const uint64_t q = mt.q[l], bar = mt.bar[l];
  const uint64_t a0 = a[((size_t)bb * 2 * la + l) * n + t], a1 = a[((size_t)bb * 2 * la + la + l) * n + t];
  const uint64_t b0 = b[((size_t)bb * 2 * lb + l) * n + t], b1 = b[((size_t)bb * 2 * lb + lb + l) * n + t];
  uint64_t lo, hi;
  uint64_t *o = out + ((size_t)bb * 3 * ell + l) * n + t;
  o[0] = mulmod(a0, b0, mt, l);
  lo = a0 * b1;
  hi = __umul64hi(a0, b1);
  mac128(lo, hi, a1, b0);
  o[(size_t)ell * n] = reduce128(hi, lo, q, bar, mt.r64[l], mt.r64s[l]);
  o[(size_t)2 * ell * n] = mulmod(a1, b1, mt, l);
}

// A batch of B ciphertexts [B][2][lay][n] with a common scale, of which the first ell limbs
// are used (ell < lay: a MatchLevel view, no copy).
struct Batch {
  std::shared_ptr<uint64_t> d;
  int ell = 0, lay = 0;
  double scale = 0.0;
  uint64_t *ptr() const { return d.get(); }
};
Batch at_level(const Batch &a, int ell) {  // MatchLevel ahead of use (R29)
  Batch v = a;
  v.ell = std::min(a.ell, ell);
  return v;
}

// A value of the evaluation: a ciphertext batch, or a plain constant (R29).
struct Val {
  bool is_ct = false;
  Batch ct;
  double k = 0.0;
};

uint64_t res_of(int64_t v, uint64_t q) {  // signed integer -> residue in [0, q)
  if (v >= 0) return (uint64_t)v % q;
  const uint64_t r = (uint64_t)(-(v + 1)) % q;
  return (q - 1 - r) % q;
}

struct Eval {
  hd_context *c;
  uint32_t B;
  const uint64_t *const *rlk_ptr = nullptr;  // device: {relinearisation key}
  const uint32_t *rlk_gal = nullptr;         // device: {1}
  hd_status err = HD_OK;

  Batch alloc(int ell, double scale) {
    Batch r;
    r.ell = r.lay = ell;
    r.scale = scale;
    if (err) return r;
    const size_t bytes = (size_t)B * 2 * ell * c->n * 8;
    uint64_t *p = static_cast<uint64_t *>(ws_alloc(c, bytes));
    if (!p) {
      err = hd_fail(HD_E_CAPACITY, "comparison workspace");
      return r;
    }
    hd_context *cc = c;
    r.d = std::shared_ptr<uint64_t>(p, [cc, bytes](uint64_t *q) { ws_free(cc, q, bytes); });
    return r;
  }
  uint64_t *scratch(size_t elems, std::shared_ptr<uint64_t> &keep) {
    if (err) return nullptr;
    const size_t bytes = elems * 8;
    uint64_t *p = static_cast<uint64_t *>(ws_alloc(c, bytes));
    if (!p) {
      err = hd_fail(HD_E_CAPACITY, "comparison workspace");
      return nullptr;
    }
    hd_context *cc = c;
    keep = std::shared_ptr<uint64_t>(p, [cc, bytes](uint64_t *q) { ws_free(cc, q, bytes); });
    return p;
  }
  void launch_check() {
    ++c->launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess && !err) err = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
  }

  // out = ka a + kb b + kc (per-limb integer residues), at min(a.ell, b.ell) limbs.
  Batch lincomb(const Batch &a, const Batch *b, const Lin &k, double scale) {
    const int ell = b ? std::min(a.ell, b->ell) : a.ell;
    Batch r = alloc(ell, scale);
    if (err) return r;
    const dim3 grid((c->n + CTPB - 1) / CTPB, ell, 2 * B);
    lincomb_kernel<<<grid, CTPB, 0, c->stream>>>(a.ptr(), a.lay, b ? b->ptr() : nullptr, b ? b->lay : 0, r.ptr(), ell,
                                                 c->logn, k, c->mt);
    launch_check();
    return r;
  }
  // a + sgn b (MatchLevel; a's scale, R29)
  Batch add(const Batch &a, const Batch &b, int sgn) {
    Lin k{};
    for (int l = 0; l < c->L; l++) {
      k.ka[l] = 1;
      k.kb[l] = sgn > 0 ? 1 : c->mod[l] - 1;
    }
    return lincomb(a, &b, k, a.scale);
  }
  // a + cst: round(cst * scale) (half-even) on c0 in every NTT slot
  Batch add_const(const Batch &a, double cst) {
    Lin k{};
    const int64_t v = llrint(cst * a.scale);
    for (int l = 0; l < c->L; l++) {
      k.ka[l] = 1;
      k.kc[l] = res_of(v, c->mod[l]);
    }
    return lincomb(a, nullptr, k, a.scale);
  }
  // Rescale of a batch [B][stride] at ell limbs -> ell - 1 limbs
  Batch rescale(const uint64_t *src, size_t stride, int ell, double scale) {
    Batch r = alloc(ell - 1, scale);
    std::shared_ptr<uint64_t> k1;
    uint64_t *t1 = scratch((size_t)2 * B * c->n, k1);
    if (err) return r;
    hd_status s = ks_rescale(c, src, stride, B, ell, r.ptr(), (size_t)2 * (ell - 1) * c->n, t1, nullptr);
    if (s && !err) err = s;
    return r;
  }
  // cst * a for a real cst: times round(cst * q_{ell-1}), then Rescale (scale kept, R29)
  Batch mul_const(const Batch &a, double cst) {
    if (a.ell < 2) {
      if (!err) err = hd_fail(HD_E_LEVEL, "comparison needs more limbs (scalar product at one limb)");
      return Batch{};
    }
    Lin k{};
    const int64_t C = llrint(cst * (double)c->mod[a.ell - 1]);
    for (int l = 0; l < c->L; l++) k.ka[l] = res_of(C, c->mod[l]);
    Batch x = lincomb(a, nullptr, k, a.scale);
    if (err) return Batch{};
    return rescale(x.ptr(), (size_t)2 * a.ell * c->n, a.ell, a.scale);
  }
  // a * b: MatchLevel, tensor, Relinearize, Rescale; scale s_a s_b / q_{ell-1}
  Batch mul(const Batch &a, const Batch &b) {
    const int ell = std::min(a.ell, b.ell), n = c->n;
    if (ell < 2) {
      if (!err) err = hd_fail(HD_E_LEVEL, "comparison needs more limbs (product at one limb)");
      return Batch{};
    }
    const size_t s3 = (size_t)3 * ell * n;
    std::shared_ptr<uint64_t> kS, kd, ku, kt;
    uint64_t *S3 = scratch((size_t)B * s3, kS);
    uint64_t *dig = scratch((size_t)B * ell * ell * n, kd);
    uint64_t *u = scratch((size_t)B * 2 * (ell + 1) * n, ku);
    uint64_t *tmp = scratch((size_t)2 * B * ell * n, kt);
    if (err) return Batch{};
    const dim3 grid((n + CTPB - 1) / CTPB, ell, B);
    tensor_kernel<<<grid, CTPB, 0, c->stream>>>(a.ptr(), a.lay, b.ptr(), b.lay, S3, ell, c->logn, c->mt);
    launch_check();
    // Relinearize and Rescale in one rounding by P q_{ell-1}: bit-identical to the
    // two-stage schedule (mixed-radix identity, R29), 2 ell NTT rows fewer per product
    Batch r = alloc(ell - 1, a.scale * b.scale / (double)c->mod[ell - 1]);
    std::shared_ptr<uint64_t> kV;
    uint64_t *V = scratch((size_t)B * 2 * (ell - 1) * n, kV);
    if (err) return Batch{};
    hd_status s = ks_relin_rescale(c, S3, B, ell, rlk_ptr, rlk_gal, r.ptr(), dig, u, tmp, V);
    if (s) {
      if (!err) err = s;
      return Batch{};
    }
    return r;
  }
  // 2 a b - (c_ct or c_const)
  Batch two_ab_minus(const Batch &a, const Batch &b, const Batch *c_ct, double c_const) {
    Batch ab = mul(a, b);
    if (err) return Batch{};
    Lin k{};
    if (c_ct) {  // MatchLevel inside lincomb
      for (int l = 0; l < c->L; l++) {
        k.ka[l] = 2 % c->mod[l];
        k.kb[l] = c->mod[l] - 1;
      }
      return lincomb(ab, c_ct, k, ab.scale);
    }
    const int64_t v = llrint(-c_const * ab.scale);
    for (int l = 0; l < c->L; l++) {
      k.ka[l] = 2 % c->mod[l];
      k.kc[l] = res_of(v, c->mod[l]);
    }
    return lincomb(ab, nullptr, k, ab.scale);
  }
};

// Paterson-Stockmeyer in the Chebyshev basis (R29), host-side schedule over batches.
struct Ps {
  Eval &E;
  int d1 = 0, d2 = 0;
  std::vector<Batch> T;  // T[1..d1]
  std::vector<Batch> G;  // G[j] = T_{d1 2^j}

  // chunk at `need` limbs: each T[i] dropped to need + 1 before its scalar product (R29)
  Val chunk(const std::vector<double> &cf, int m, int need) {
    Val acc;
    for (int i = 1; i <= m; i++) {
      if (cf[i] == 0.0) continue;
      Batch t = E.mul_const(at_level(T[i], need + 1), cf[i]);
      if (E.err) return acc;
      if (!acc.is_ct) {
        acc.is_ct = true;
        acc.ct = t;
      } else {
        acc.ct = E.add(acc.ct, t, 1);
      }
    }
    if (!acc.is_ct) {
      acc.k = cf[0];
      return acc;
    }
    if (cf[0] != 0.0) acc.ct = E.add_const(acc.ct, cf[0]);
    return acc;
  }
  // result wanted at `need` limbs: q T_k taken at need + 1, r evaluated for need (R29)
  Val eval(const std::vector<double> &cf0, int m, int need) {
    while (m > 0 && cf0[m] == 0.0) m--;
    if (m < d1) return chunk(cf0, m, need);
    int j = 0;
    while (j + 1 < (int)G.size() && (d1 << (j + 1)) <= m) j++;
    const int k = d1 << j;
    std::vector<double> q(m - k + 1), r(k);
    q[0] = cf0[k];
    for (int i = 1; i <= m - k; i++) q[i] = 2.0 * cf0[k + i];
    for (int i = 0; i < k; i++) r[i] = cf0[i];
    for (int i = 1; i <= m - k; i++) r[k - i] = r[k - i] - cf0[k + i];
    Val Q = eval(q, m - k, need + 1);
    if (E.err) return Val{};
    Val R = eval(r, k - 1, need);
    if (E.err) return Val{};
    Val P;
    const Batch Gj = at_level(G[j], need + 1);
    if (Q.is_ct) {
      P.is_ct = true;
      P.ct = E.mul(Q.ct, Gj);
    } else if (Q.k != 0.0) {
      P.is_ct = true;
      P.ct = E.mul_const(Gj, Q.k);
    }
    if (E.err) return Val{};
    if (!P.is_ct) return R;
    if (R.is_ct) P.ct = E.add(P.ct, R.ct, 1);
    else if (R.k != 0.0) P.ct = E.add_const(P.ct, R.k);
    return P;
  }
};

void ps_split(int n, int &d1, int &d2) {  // P:L725-727, ties to the smaller d2 (R29)
  int best = 1 << 30;
  d1 = d2 = 0;
  for (int g = 1; g <= 31; g++)
    for (int b = 1; b <= n; b++) {
      if (((long long)b << (g - 1)) < n) continue;
      if (b + g < best) {
        best = b + g;
        d1 = b;
        d2 = g;
      }
      break;
    }
}

hd_status check_inputs(hd_context *c, const hd_ciphertext *const *in, size_t count, uint32_t &ell, double &scale) {
  if (!c || !in || count == 0) return hd_fail(HD_E_INVALID_ARG, "null argument or empty input");
  for (size_t i = 0; i < count; i++) {
    if (!in[i]) return hd_fail(HD_E_INVALID_ARG, "null ciphertext");
    if (in[i]->ctx != c) return hd_fail(HD_E_STATE, "ciphertext from another context");
    if (i == 0) {
      ell = in[i]->limbs;
      scale = in[i]->scale;
    } else if (in[i]->limbs != ell || in[i]->scale != scale) {
      return hd_fail(HD_E_LEVEL, "inputs at different levels or scales");
    }
  }
  return HD_OK;
}

// Gathers the inputs [i0, i0 + B) into one batch on the context stream (after their writers).
hd_status gather(Eval &E, const hd_ciphertext *const *in, size_t i0, uint32_t B, uint32_t ell, double scale,
                 Batch &out) {
  hd_context *c = E.c;
  out = E.alloc((int)ell, scale);
  if (E.err) return E.err;
  const size_t ct = (size_t)2 * ell * c->n;
  for (uint32_t b = 0; b < B; b++) {
    HD_CUDA(cudaStreamWaitEvent(c->stream, in[i0 + b]->ready, 0));
    HD_CUDA(cudaMemcpyAsync(out.ptr() + b * ct, in[i0 + b]->data, ct * 8, cudaMemcpyDeviceToDevice, c->stream));
  }
  return HD_OK;
}

hd_status mark_read(hd_context *c, const hd_ciphertext *ct) {
  hd_ciphertext *m = const_cast<hd_ciphertext *>(ct);  // reader bookkeeping only
  if (!m->used) HD_CUDA(cudaEventCreateWithFlags(&m->used, cudaEventDisableTiming));
  HD_CUDA(cudaEventRecord(m->used, c->stream));
  return HD_OK;
}

hd_status scatter(hd_context *c, const Batch &res, size_t i0, uint32_t B, hd_ciphertext **out) {
  const size_t ct = (size_t)2 * res.ell * c->n;
  for (uint32_t b = 0; b < B; b++) {
    hd_ciphertext *&o = out[i0 + b];
    if (o && (o->ctx != c || o->limbs != (uint32_t)res.ell)) return hd_fail(HD_E_LEVEL, "output shape mismatch");
    if (!o) {
      hd_status s = alloc_ct(c, (uint32_t)res.ell, &o);
      if (s) return s;
    }
    if (o->used) HD_CUDA(cudaStreamWaitEvent(c->stream, o->used, 0));
    HD_CUDA(cudaMemcpyAsync(o->data, res.ptr() + b * ct, ct * 8, cudaMemcpyDeviceToDevice, c->stream));
    o->scale = res.scale;
    HD_CUDA(cudaEventRecord(o->ready, c->stream));
  }
  return HD_OK;
}

struct DevKeys {  // device arrays {key pointers}, {Galois elements}
  std::shared_ptr<void> mem;
  const uint64_t *const *kp = nullptr;
  const uint32_t *gal = nullptr;
};
hd_status upload_keys(hd_context *c, const std::vector<const uint64_t *> &kp, const std::vector<uint32_t> &gl,
                      DevKeys &dk) {
  // stream-ordered: no device-wide synchronisation (the pageable source is staged by the
  // runtime before cudaMemcpyAsync returns)
  const size_t cnt = kp.size(), bytes = cnt * sizeof(uint64_t *) + cnt * sizeof(uint32_t);
  std::vector<char> host(bytes);
  memcpy(host.data(), kp.data(), cnt * sizeof(uint64_t *));
  memcpy(host.data() + cnt * sizeof(uint64_t *), gl.data(), cnt * sizeof(uint32_t));
  void *p = ws_alloc(c, bytes);
  if (!p) return hd_fail(HD_E_CAPACITY, "comparison key table");
  dk.mem = std::shared_ptr<void>(p, [c, bytes](void *q) { ws_free(c, q, bytes); });
  HD_CUDA(cudaMemcpyAsync(p, host.data(), bytes, cudaMemcpyHostToDevice, c->stream));
  dk.kp = (const uint64_t *const *)p;
  dk.gal = (const uint32_t *)((char *)p + cnt * sizeof(uint64_t *));
  return HD_OK;
}

constexpr uint32_t kCompareChunk = 64;  // ciphertexts evaluated together (workspace ~2 GB at 2^16, L = 6)

}  // namespace

extern "C" hd_status hd_chebyshev_degree(uint32_t kappa, uint32_t *degree) {
  if (!degree) return hd_fail(HD_E_INVALID_ARG, "null argument");
  static const uint32_t tab[4] = {5, 13, 27, 59};
  if (kappa < 7 || kappa > 10) return hd_fail(HD_E_INVALID_ARG, "kappa outside the paper's table (7..10)");
  *degree = tab[kappa - 7];
  return HD_OK;
}

extern "C" hd_status hd_chebyshev_coefficients(double delta, uint32_t degree, double *coeffs, size_t cap) {
  if (!coeffs || degree < 1) return hd_fail(HD_E_INVALID_ARG, "null argument or degree 0");
  if (cap < (size_t)degree + 1) return hd_fail(HD_E_INVALID_ARG, "coefficient capacity too small");
  const double pi = 3.14159265358979323846;
  const int n = (int)degree;
  for (int i = 0; i <= n; i++) {  // DCT-II at the first-kind Chebyshev nodes (R29)
    double s = 0.0;
    for (int k = 0; k <= n; k++) {
      const double xk = std::cos(pi * ((double)k + 0.5) / (double)(n + 1));
      const double fk = xk >= delta ? 1.0 : 0.0;
      s = s + fk * std::cos(pi * (double)i * ((double)k + 0.5) / (double)(n + 1));
    }
    coeffs[i] = 2.0 * s / (double)(n + 1);
  }
  coeffs[0] = coeffs[0] / 2.0;
  return HD_OK;
}

extern "C" hd_status hd_compare_ex(hd_context *c, const hd_eval_keys *evk, const hd_ciphertext *const *in,
                                   size_t count, const double *coeffs, uint32_t degree, uint32_t out_limbs,
                                   hd_ciphertext **out);

extern "C" hd_status hd_compare(hd_context *c, const hd_eval_keys *evk, const hd_ciphertext *const *in, size_t count,
                                const double *coeffs, uint32_t degree, hd_ciphertext **out) {
  return hd_compare_ex(c, evk, in, count, coeffs, degree, 1, out);
}

extern "C" hd_status hd_compare_ex(hd_context *c, const hd_eval_keys *evk, const hd_ciphertext *const *in,
                                   size_t count, const double *coeffs, uint32_t degree, uint32_t out_limbs,
                                   hd_ciphertext **out) {
  uint32_t ell = 0;
  double scale = 0.0;
  hd_status s = check_inputs(c, in, count, ell, scale);
  if (s) return s;
  if (ks_general(c))  // relinearise-rescale in one rounding needs one special prime (R29)
    return hd_fail(HD_E_PARAMS, "the comparison is implemented for num_special = digit_limbs = 1 only");
  if (!evk || !coeffs || !out || degree < 1) return hd_fail(HD_E_INVALID_ARG, "null argument");
  if (out_limbs < 1 || out_limbs >= ell) return hd_fail(HD_E_LEVEL, "out_limbs must be in [1, input limbs)");
  if (evk->ctx != c) return hd_fail(HD_E_STATE, "keys from another context");
  const uint64_t *rk = evk->find(HD_RELIN_STEP);
  if (!rk) return hd_fail(HD_E_MISSING_KEY, "missing relinearisation key (hd_relin_keygen)");
  std::vector<double> cf(coeffs, coeffs + degree + 1);
  bool any = false;
  for (uint32_t i = 1; i <= degree; i++) any = any || cf[i] != 0.0;
  if (!any) return hd_fail(HD_E_INVALID_ARG, "constant series: nothing to evaluate");
  DevKeys dk;
  if ((s = upload_keys(c, {rk}, {1u}, dk))) return s;
  int d1, d2;
  ps_split((int)degree, d1, d2);
  if (d1 > 63) return hd_fail(HD_E_INVALID_ARG, "degree too large");
  for (size_t i0 = 0; i0 < count; i0 += kCompareChunk) {
    const uint32_t B = (uint32_t)std::min<size_t>(kCompareChunk, count - i0);
    Eval E{c, B, dk.kp, dk.gal};
    Ps P{E, d1, d2};
    P.T.resize(d1 + 1);
    if ((s = gather(E, in, i0, B, ell, scale, P.T[1]))) return s;
    for (size_t b = 0; b < B; b++)
      if ((s = mark_read(c, in[i0 + b]))) return s;
    // Step 1: baby powers
    for (int i = 2; i <= d1 && !E.err; i++) {
      if ((i & (i - 1)) == 0) P.T[i] = E.two_ab_minus(P.T[i / 2], P.T[i / 2], nullptr, 1.0);
      else P.T[i] = E.two_ab_minus(P.T[i / 2], P.T[(i + 1) / 2], &P.T[1], 0.0);
    }
    // Step 2: giant powers by doubling, while d1 2^j <= degree (R29)
    if (!E.err) P.G.push_back(P.T[d1]);
    while (!E.err && (d1 << P.G.size()) <= (int)degree) P.G.push_back(E.two_ab_minus(P.G.back(), P.G.back(), nullptr, 1.0));
    // Step 3: chunks and the Chebyshev-basis combination (R29)
    Val V;
    if (!E.err) V = P.eval(cf, (int)degree, (int)out_limbs);  // the result at out_limbs limbs (R29)
    if (E.err) return E.err;
    if (!V.is_ct) return hd_fail(HD_E_INVALID_ARG, "constant series: nothing to evaluate");
    if (V.ct.ell < (int)out_limbs) return hd_fail(HD_E_LEVEL, "not enough limbs for the requested output level");
    if (V.ct.lay != V.ct.ell) {  // a MatchLevel view: materialise before the copy-out
      Lin id{};
      for (int l = 0; l < c->L; l++) id.ka[l] = 1;
      V.ct = E.lincomb(V.ct, nullptr, id, V.ct.scale);
      if (E.err) return E.err;
    }
    if ((s = scatter(c, V.ct, i0, B, out))) return s;
  }
  return HD_OK;
}

extern "C" hd_status hd_membership_steps(const hd_context *c, int32_t *steps, size_t cap, size_t *count) {
  if (!c || !count) return hd_fail(HD_E_INVALID_ARG, "null argument");
  size_t k = 0;
  for (int s = 1; s < c->ns; s <<= 1) {
    if (steps && k < cap) steps[k] = s;
    k++;
  }
  *count = k;
  if (steps && cap < k) return hd_fail(HD_E_INVALID_ARG, "steps capacity too small");
  return HD_OK;
}

extern "C" hd_status hd_membership(hd_context *c, const hd_eval_keys *evk, const hd_ciphertext *const *in,
                                   size_t count, hd_ciphertext **out) {
  uint32_t ell = 0;
  double scale = 0.0;
  hd_status s = check_inputs(c, in, count, ell, scale);
  if (s) return s;
  if (!evk || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  if (evk->ctx != c) return hd_fail(HD_E_STATE, "keys from another context");
  std::vector<const uint64_t *> kp;
  std::vector<uint32_t> gl;
  for (int k = 1; k < c->ns; k <<= 1) {
    const uint64_t *key = evk->find(k);
    if (!key) return hd_fail(HD_E_MISSING_KEY, "missing rotation key for step " + std::to_string(k));
    kp.push_back(key);
    gl.push_back((uint32_t)host_powmod(5, (uint64_t)k, 2ull * c->n));
  }
  DevKeys dk;
  if ((s = upload_keys(c, kp, gl, dk))) return s;
  const int n = c->n, e = (int)ell;
  // EvalAddMany: acc = sum_i in_i, one batch of 1
  Eval E{c, 1, nullptr, nullptr};
  Batch acc;
  if ((s = gather(E, in, 0, 1, ell, scale, acc))) return s;
  if ((s = mark_read(c, in[0]))) return s;
  for (size_t i = 1; i < count; i++) {
    Batch x;
    if ((s = gather(E, in, i, 1, ell, scale, x))) return s;
    if ((s = mark_read(c, in[i]))) return s;
    acc = E.add(acc, x, 1);
    if (E.err) return E.err;
  }
  // RotateAndSum over numSlots: acc += Rot_k(acc), k = 1, 2, ..., numSlots / 2
  std::shared_ptr<uint64_t> kd, ku, kt;
  uint64_t *dig = E.scratch((size_t)e * e * n, kd);
  uint64_t *u = E.scratch((size_t)2 * (e + 1) * n, ku);
  uint64_t *tmp = E.scratch((size_t)2 * e * n, kt);
  if (E.err) return E.err;
  for (size_t r = 0; r < kp.size(); r++) {
    Batch rot = E.alloc(e, scale);
    if (E.err) return E.err;
    const uint64_t *c1 = acc.ptr() + (size_t)e * n;
    if ((s = ks_modup(c, c1, 0, 1, e, dig, tmp)) || (s = ks_kip(c, dig, c1, 0, 1, 1, e, dk.kp + r, dk.gal + r, u)) ||
        (s = ks_moddown(c, u, 1, 1, e, dk.gal + r, acc.ptr(), 0, rot.ptr(), (size_t)2 * e * n, false, tmp)))
      return s;
    acc = E.add(acc, rot, 1);
    if (E.err) return E.err;
  }
  return scatter(c, acc, 0, 1, out);
}

extern "C" hd_status hd_eval_add_many(hd_context *c, const hd_ciphertext *const *in, size_t count,
                                      hd_ciphertext **out) {
  uint32_t ell = 0;
  double scale = 0.0;
  hd_status s = check_inputs(c, in, count, ell, scale);
  if (s) return s;
  if (!out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  Eval E{c, 1, nullptr, nullptr};
  Batch acc;
  if ((s = gather(E, in, 0, 1, ell, scale, acc))) return s;
  if ((s = mark_read(c, in[0]))) return s;
  for (size_t i = 1; i < count; i++) {
    Batch x;
    if ((s = gather(E, in, i, 1, ell, scale, x))) return s;
    if ((s = mark_read(c, in[i]))) return s;
    acc = E.add(acc, x, 1);
    if (E.err) return E.err;
  }
  return scatter(c, acc, 0, 1, out);
}

extern "C" hd_status hd_ciphertext_scale(const hd_ciphertext *ct, double *scale) {
  if (!ct || !scale) return hd_fail(HD_E_INVALID_ARG, "null argument");
  *scale = ct->scale;
  return HD_OK;
}
