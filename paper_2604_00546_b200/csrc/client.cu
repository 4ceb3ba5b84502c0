// client.cu -- secret key, rotation keys, query encryption, decryption and decoding
// (P:L302-310), all on the device.
//
// Randomness (R14): Philox4x32-10 keyed by (seed_lo, seed_hi) with
// counter (coef j, modulus index l, object, tag<<16 | sub).
#include <cmath>

#include "common.cuh"
#include "ks.cuh"
#include "rng.cuh"

hd_status normalize_on_device(hd_context *c, const float *dv, int rows, int dim, double *U);
hd_status check_flag(hd_context *c);

namespace {
constexpr int TPB = 256;

// s (ternary) into every modulus row [(L+1)][n] (coefficient form).
__global__ void secret_kernel(uint64_t seed, int n, int nm, uint64_t *__restrict__ s, ModTab mt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  uint64_t w0, w1;
  draw(seed, j, 0, 0, TAG_SECRET, 0, w0, w1);
  const int64_t v = (int64_t)(w0 % 3) - 1;
  for (int l = 0; l < nm; l++) s[(size_t)l * n + j] = smod_dev(v, mt.q[l], mt.bar[l]);
}

// error rows of a key: key[d][0][l][j] = CBD draw of (j, obj, d) mod q_l (coefficient form),
// l over the M = L + K moduli.
__global__ void key_error_kernel(uint64_t seed, uint32_t step, uint32_t tag, int n, int M, uint64_t *__restrict__ key,
                                 ModTab mt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int d = blockIdx.y;
  if (j >= n) return;
  uint64_t w0, w1;
  draw(seed, j, 0, step, tag, d, w0, w1);
  const int64_t e = cbd21(w0);
  for (int l = 0; l < M; l++) key[((size_t)(d * 2) * M + l) * n + j] = smod_dev(e, mt.q[l], mt.bar[l]);
}

// b_d = e_d - a_d s + [l in I_d] (P mod q_l) s';  a_d uniform in NTT form (R11, R14, R31):
// digit d = limbs [d alpha, (d+1) alpha) (alpha = K = 1: [l == d] (P mod q_d) s').
// s' = sigma_g(s) (rotation key, g = Galois element) or s^2 (g = 0: relinearisation key, R26).
__global__ void key_combine_kernel(uint64_t seed, uint32_t step, uint32_t tag_a, uint32_t g, int logn, int L, int M,
                                   int alpha, const uint64_t *__restrict__ s_ntt, uint64_t *__restrict__ key,
                                   ModTab mt, InvTab2 pmod) {
  const int n = 1 << logn;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int dl = blockIdx.y;
  const int d = dl / M, l = dl % M;
  if (j >= n) return;
  const uint64_t q = mt.q[l];
  uint64_t w0, w1;
  draw(seed, j, l, step, tag_a, d, w0, w1);
  const uint64_t a = reduce128(w0, w1, q, mt.bar[l], mt.r64[l], mt.r64s[l]);
  uint64_t *kb = key + ((size_t)(d * 2 + 0) * M + l) * n;
  uint64_t *ka = key + ((size_t)(d * 2 + 1) * M + l) * n;
  uint64_t b = submod(kb[j], mulmod(a, s_ntt[(size_t)l * n + j], mt, l), q);
  if (l < L && l / alpha == d) {
    const uint64_t sj = s_ntt[(size_t)l * n + j];
    const uint64_t sp = g ? s_ntt[(size_t)l * n + galois_src(j, g, logn)]  // sigma_g(s) in the NTT domain
                          : mulmod(sj, sj, mt, l);                          // s^2
    b = addmod(b, mulmod(pmod.w[l], sp, mt, l), q);
  }
  kb[j] = b;
  ka[j] = a;
}

// encryption: ct c0 holds pt, c1 holds e (NTT form): c0 = e - a s + pt, c1 = a.
__global__ void enc_error_kernel(uint64_t seed, int n, int nl, uint64_t *__restrict__ c1, ModTab mt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  uint64_t w0, w1;
  draw(seed, j, 0, 0, TAG_ENC_E, 0, w0, w1);
  const int64_t e = cbd21(w0);
  for (int l = 0; l < nl; l++) c1[(size_t)l * n + j] = smod_dev(e, mt.q[l], mt.bar[l]);
}
__global__ void enc_combine_kernel(uint64_t seed, int n, int nl, const uint64_t *__restrict__ s_ntt,
                                   uint64_t *__restrict__ ct, ModTab mt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (j >= n) return;
  const uint64_t q = mt.q[l];
  uint64_t w0, w1;
  draw(seed, j, l, 0, TAG_ENC_A, 0, w0, w1);
  const uint64_t a = reduce128(w0, w1, q, mt.bar[l], mt.r64[l], mt.r64s[l]);
  uint64_t *c0 = ct + (size_t)l * n, *c1 = ct + ((size_t)nl + l) * n;
  uint64_t v = submod(c1[j], mulmod(a, s_ntt[(size_t)l * n + j], mt, l), q);
  c0[j] = addmod(v, c0[j], q);
  c1[j] = a;
}

// query slots: z_s = u_{s mod N} (R8)
__global__ void query_slots_kernel(const double *__restrict__ u, int N, int ns, double *__restrict__ re,
                                   double *__restrict__ im, double msg_scale) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= ns) return;
  re[s] = msg_scale == 1.0 ? u[s % N] : __dmul_rn(u[s % N], msg_scale);
  im[s] = 0.0;
}

// m = c0 + c1 s (NTT form)
__global__ void decrypt_kernel(const uint64_t *__restrict__ ct, const uint64_t *__restrict__ s_ntt, int n, int nl,
                               uint64_t *__restrict__ m, ModTab mt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (j >= n) return;
  const uint64_t q = mt.q[l];
  m[(size_t)l * n + j] = addmod(ct[(size_t)l * n + j], mulmod(ct[((size_t)nl + l) * n + j], s_ntt[(size_t)l * n + j], mt, l), q);
}

struct CrtTab {
  uint64_t inv[HD_MAXMOD][HD_MAXMOD];  // inv[i][k] = q_k^{-1} mod q_i
  uint64_t Q[HD_MAXMOD + 1];           // prod_{k<nl} q_k, little-endian words
  uint64_t W[HD_MAXMOD][HD_MAXMOD + 1]; // W[i] = prod_{k<i} q_k
};

// centred CRT (Garner) of coefficient-form limbs -> double / delta; complex slots
// w_k = (m_k, m_{k+ns}) / delta written bit-reversed (input of the forward special FFT).
__global__ void crt_decode_kernel(const uint64_t *__restrict__ m, int n, int nl, double delta, int logns,
                                  double *__restrict__ re, double *__restrict__ im, ModTab mt, CrtTab ct) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int ns = n / 2;
  uint64_t v[HD_MAXMOD];
  for (int i = 0; i < nl; i++) {
    const uint64_t qi = mt.q[i];
    uint64_t t = m[(size_t)i * n + c];
    for (int k = 0; k < i; k++) t = mulmod(submod(t, reduce64(v[k], qi, mt.bar[i]), qi), ct.inv[i][k], mt, i);
    v[i] = t;
  }
  // X = sum_i v_i W_i
  uint64_t X[HD_MAXMOD + 1];
  for (int w = 0; w <= nl; w++) X[w] = 0;
  for (int i = 0; i < nl; i++) {
    unsigned __int128 carry = 0;
    for (int w = 0; w <= nl; w++) {
      unsigned __int128 s = (unsigned __int128)v[i] * ct.W[i][w] + X[w] + carry;
      X[w] = (uint64_t)s;
      carry = s >> 64;
    }
  }
  // negative iff 2X > Q
  bool gt = false;
  {
    uint64_t c2 = 0;
    uint64_t X2[HD_MAXMOD + 1];
    for (int w = 0; w <= nl; w++) {
      X2[w] = (X[w] << 1) | c2;
      c2 = X[w] >> 63;
    }
    for (int w = nl; w >= 0; w--)
      if (X2[w] != ct.Q[w]) {
        gt = X2[w] > ct.Q[w];
        break;
      }
  }
  if (gt) {
    unsigned __int128 borrow = 0;
    for (int w = 0; w <= nl; w++) {
      unsigned __int128 d = (unsigned __int128)ct.Q[w] - X[w] - borrow;
      X[w] = (uint64_t)d;
      borrow = (d >> 64) ? 1 : 0;
    }
  }
  double r = 0.0;
  for (int w = nl; w >= 0; w--) r = r * 18446744073709551616.0 + (double)X[w];
  if (gt) r = -r;
  r = r / delta;
  const int k = c < ns ? c : c - ns;
  const int pos = __brev((uint32_t)k) >> (32 - logns);
  if (c < ns) re[pos] = r;
  else im[pos] = r;
}

__global__ void fft_fwd_stage_kernel(double *__restrict__ re, double *__restrict__ im, int ns, int len,
                                     const uint32_t *__restrict__ rotg, const double *__restrict__ xr,
                                     const double *__restrict__ xim, uint32_t two_n) {
  const int bf = blockIdx.x * blockDim.x + threadIdx.x;
  if (bf >= ns / 2) return;
  const int lenh = len >> 1;
  const uint32_t lenq = (uint32_t)len << 2;
  const int blk = bf / lenh, j = bf % lenh;
  const int i0 = blk * len + j, i1 = i0 + lenh;
  const uint32_t idx = (rotg[j] % lenq) * (two_n / lenq);
  const double wr = xr[idx], wi = xim[idx];
  const double xr1 = re[i1], xi1 = im[i1];
  const double vr = __dsub_rn(__dmul_rn(xr1, wr), __dmul_rn(xi1, wi));
  const double vi = __dadd_rn(__dmul_rn(xr1, wi), __dmul_rn(xi1, wr));
  const double ur = re[i0], ui = im[i0];
  re[i0] = __dadd_rn(ur, vr);
  im[i0] = __dadd_rn(ui, vi);
  re[i1] = __dsub_rn(ur, vr);
  im[i1] = __dsub_rn(ui, vi);
}

// scores of aggregate agg: v = (agg G + b) N + t -> slot b stride + t, G groups per ciphertext
// (replicated, R4: G = M/2, stride 2N; flat, R27: G = M, stride N)
__global__ void scores_kernel(const double *__restrict__ z, int N, int G, int stride, long long agg,
                              long long v_first, long long v_end, double *__restrict__ scores) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G * N) return;
  const int b = i / N, t = i % N;
  const long long v = (agg * G + b) * N + t;
  if (v >= v_first && v < v_end) scores[v - v_first] = z[(size_t)b * stride + t];
}
// ---- encrypted-database mode (NEXT-1, R26) -------------------------------------------
// public key: b rows hold e (coefficient form) before the NTT; then b = e - a s, a uniform.
__global__ void pk_error_kernel(uint64_t seed, int n, int L, uint64_t *__restrict__ b, ModTab mt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  uint64_t w0, w1;
  draw(seed, j, 0, 0, TAG_PK_E, 0, w0, w1);
  const int64_t e = cbd21(w0);
  for (int l = 0; l < L; l++) b[(size_t)l * n + j] = smod_dev(e, mt.q[l], mt.bar[l]);
}
__global__ void pk_combine_kernel(uint64_t seed, int n, int L, const uint64_t *__restrict__ s_ntt,
                                  uint64_t *__restrict__ pk, ModTab mt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int l = blockIdx.y;
  if (j >= n) return;
  const uint64_t q = mt.q[l];
  uint64_t w0, w1;
  draw(seed, j, l, 0, TAG_PK_A, 0, w0, w1);
  const uint64_t a = reduce128(w0, w1, q, mt.bar[l], mt.r64[l], mt.r64s[l]);
  uint64_t *b = pk + (size_t)l * n;
  b[j] = submod(b[j], mulmod(a, s_ntt[(size_t)l * n + j], mt, l), q);
  pk[((size_t)L + l) * n + j] = a;
}
// public-key encryption of B ciphertexts (ct_x at ct + x*ct_stride, c0 holding the plaintext):
// v (ternary) and e0 into scratch rows [x][l], e1 into the c1 rows, coefficient form.
__global__ void pke_draw_kernel(uint64_t seed, uint32_t obj0, int n, int L, uint64_t *__restrict__ ct,
                                size_t ct_stride, uint64_t *__restrict__ V, uint64_t *__restrict__ E0, ModTab mt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t x = blockIdx.y;
  if (j >= n) return;
  const uint32_t obj = obj0 + x;
  uint64_t w0, w1;
  draw(seed, j, 0, obj, TAG_PKE_V, 0, w0, w1);
  const int64_t v = (int64_t)(w0 % 3) - 1;
  draw(seed, j, 0, obj, TAG_PKE_E, 0, w0, w1);
  const int64_t e0 = cbd21(w0);
  draw(seed, j, 0, obj, TAG_PKE_E, 1, w0, w1);
  const int64_t e1 = cbd21(w0);
  uint64_t *c1 = ct + (size_t)x * ct_stride + (size_t)L * n;
  for (int l = 0; l < L; l++) {
    const size_t o = ((size_t)x * L + l) * n + j;
    V[o] = smod_dev(v, mt.q[l], mt.bar[l]);
    E0[o] = smod_dev(e0, mt.q[l], mt.bar[l]);
    c1[(size_t)l * n + j] = smod_dev(e1, mt.q[l], mt.bar[l]);
  }
}
// c0 = v b + e0 + pt, c1 = v a + e1 (all NTT form)
__global__ void pke_combine_kernel(int n, int L, const uint64_t *__restrict__ pk, uint64_t *__restrict__ ct,
                                   size_t ct_stride, const uint64_t *__restrict__ V, const uint64_t *__restrict__ E0,
                                   ModTab mt) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t xl = blockIdx.y, x = xl / L, l = xl % L;
  if (j >= n) return;
  const uint64_t q = mt.q[l];
  const size_t o = ((size_t)x * L + l) * n + j;
  const uint64_t v = V[o];
  uint64_t *c0 = ct + (size_t)x * ct_stride + (size_t)l * n, *c1 = c0 + (size_t)L * n;
  c0[j] = addmod(addmod(mulmod(v, pk[(size_t)l * n + j], mt, l), E0[o], q), c0[j], q);
  c1[j] = addmod(mulmod(v, pk[((size_t)L + l) * n + j], mt, l), c1[j], q);
}
}  // namespace

static uint64_t inv_host(uint64_t a, uint64_t q) { return host_powmod(a % q, q - 2, q); }

extern "C" hd_status hd_keygen(hd_context *c, const int32_t *steps, size_t count, hd_secret_key **sk_out,
                               hd_eval_keys **evk_out) {
  if (!c || !sk_out || !evk_out || (count && !steps)) return hd_fail(HD_E_INVALID_ARG, "null argument");
  *sk_out = nullptr;
  *evk_out = nullptr;
  for (size_t i = 0; i < count; i++)
    if (steps[i] <= 0 || steps[i] >= c->ns) return hd_fail(HD_E_INVALID_ARG, "rotation step outside (0, numSlots)");
  HD_CUDA(cudaSetDevice(c->device));
  const int n = c->n, L = c->L, M = ks_M(c), beta = ks_beta(c, L);
  hd_secret_key *sk = new hd_secret_key{c, nullptr};
  hd_eval_keys *evk = new hd_eval_keys();
  evk->ctx = c;
  ctx_retain(c);
  ctx_retain(c);
  evk->steps.assign(steps, steps + count);
  evk->key_elems = ks_key_elems(c);
  auto fail = [&](hd_status s) {
    hd_secret_key_destroy(sk);
    hd_eval_keys_destroy(evk);
    return s;
  };
  cudaError_t e = dev_alloc(c, &sk->s_ntt, (size_t)M * n * 8);
  if (!e && count) e = dev_alloc(c, &evk->keys, evk->key_elems * count * 8);
  if (e) return fail(hd_fail(HD_E_CAPACITY, cudaGetErrorString(e)));
  const uint64_t seed = c->params.seed;
  secret_kernel<<<(n + TPB - 1) / TPB, TPB, 0, c->stream>>>(seed, n, M, sk->s_ntt, c->mt); ++c->launches;
  RowMap rm{};
  rm.gsize = 1u << 30;
  rm.mdiv = 1;
  rm.mlen = M;
  for (int l = 0; l < M; l++) rm.midx[l] = l;
  hd_status s = ntt_rows(c, sk->s_ntt, M, rm, false);
  if (s) return fail(s);
  InvTab2 pmod{};
  for (int l = 0; l < L; l++) pmod.w[l] = ks_P_mod(c, c->mod[l]);
  for (size_t i = 0; i < count; i++) {
    uint64_t *key = evk->keys + evk->key_elems * i;
    const uint32_t step = (uint32_t)steps[i];
    const uint32_t g = (uint32_t)host_powmod(5, step, 2ull * n);
    key_error_kernel<<<dim3((n + TPB - 1) / TPB, beta), TPB, 0, c->stream>>>(seed, step, TAG_KEY_E, n, M, key, c->mt); ++c->launches;
    RowMap rk{};  // rows (d, l) at key + (d 2 M + l) n
    rk.gsize = M;
    rk.gstride = (uint64_t)2 * M * n;
    rk.mdiv = 1;
    rk.mlen = M;
    for (int l = 0; l < M; l++) rk.midx[l] = l;
    if ((s = ntt_rows(c, key, beta * M, rk, false))) return fail(s);
    key_combine_kernel<<<dim3((n + TPB - 1) / TPB, beta * M), TPB, 0, c->stream>>>(
        seed, step, TAG_KEY_A, g, c->logn, L, M, c->alpha, sk->s_ntt, key, c->mt, pmod); ++c->launches;
  }
  e = cudaStreamSynchronize(c->stream);
  if (e) return fail(hd_fail(HD_E_CUDA, cudaGetErrorString(e)));
  *sk_out = sk;
  *evk_out = evk;
  return HD_OK;
}

extern "C" hd_status hd_encrypt_query(hd_context *c, const hd_secret_key *sk, const float *q, uint32_t vector_dim,
                                      uint64_t enc_seed, hd_ciphertext **out) {
  return hd_encrypt_query_ex(c, sk, q, vector_dim, enc_seed, 1.0, out);
}

extern "C" hd_status hd_encrypt_query_ex(hd_context *c, const hd_secret_key *sk, const float *q, uint32_t vector_dim,
                                         uint64_t enc_seed, double msg_scale, hd_ciphertext **out) {
  if (!c || !sk || !q || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  if (!(msg_scale > 0.0) || msg_scale > 1.0) return hd_fail(HD_E_INVALID_ARG, "msg_scale must be in (0, 1]");
  *out = nullptr;
  if (vector_dim < 2 || (vector_dim & (vector_dim - 1)) || (uint32_t)c->ns % (2 * vector_dim))
    return hd_fail(HD_E_LAYOUT, "vector_dim must be a power of two with numSlots % (2 vector_dim) == 0");
  HD_CUDA(cudaSetDevice(c->device));
  const int n = c->n, ns = c->ns, L = c->L, N = (int)vector_dim;
  float *dq = nullptr;
  double *U = nullptr, *re = nullptr, *im = nullptr;
  hd_ciphertext *ct = nullptr;
  hd_status s = alloc_ct(c, L, &ct);
  if (s) return s;
  cudaError_t e = dev_alloc(c, &dq, N * 4);
  if (!e) e = dev_alloc(c, &U, N * 8);
  if (!e) e = dev_alloc(c, &re, (size_t)ns * 8);
  if (!e) e = dev_alloc(c, &im, (size_t)ns * 8);
  if (!e) e = cudaMemcpyAsync(dq, q, N * 4, cudaMemcpyHostToDevice, c->stream);
  if (e) s = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
  if (!s) s = normalize_on_device(c, dq, 1, N, U);
  if (!s) s = check_flag(c);
  if (!s) {
    query_slots_kernel<<<(ns + TPB - 1) / TPB, TPB, 0, c->stream>>>(U, N, ns, re, im, msg_scale); ++c->launches;
    s = encode_batch(c, re, im, 1, std::ldexp(1.0, (int)c->params.scale_bits), L, ct->data, (size_t)2 * L * n);
  }
  if (!s) {
    enc_error_kernel<<<(n + TPB - 1) / TPB, TPB, 0, c->stream>>>(enc_seed, n, L, ct->data + (size_t)L * n, c->mt); ++c->launches;
    RowMap rm{};
    rm.gsize = 1u << 30;
    rm.mdiv = 1;
    rm.mlen = L;
    for (int l = 0; l < L; l++) rm.midx[l] = l;
    s = ntt_rows(c, ct->data + (size_t)L * n, L, rm, false);
  }
  if (!s) {
    enc_combine_kernel<<<dim3((n + TPB - 1) / TPB, L), TPB, 0, c->stream>>>(enc_seed, n, L, sk->s_ntt, ct->data, c->mt); ++c->launches;
    s = check_flag(c);
  }
  dev_free(c, dq);
  dev_free(c, U);
  dev_free(c, re);
  dev_free(c, im);
  if (s) {
    hd_ciphertext_destroy(ct);
    return s;
  }
  HD_CUDA(cudaEventRecord(ct->ready, c->stream));
  *out = ct;
  return HD_OK;
}

static hd_status decrypt_to(hd_context *c, const hd_secret_key *sk, const hd_ciphertext *ct, uint64_t *m) {
  const int n = c->n;
  HD_CUDA(cudaStreamWaitEvent(c->stream, ct->ready, 0));
  decrypt_kernel<<<dim3((n + TPB - 1) / TPB, ct->limbs), TPB, 0, c->stream>>>(ct->data, sk->s_ntt, n, ct->limbs, m,
                                                                             c->mt); ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

extern "C" hd_status hd_decrypt(hd_context *c, const hd_secret_key *sk, const hd_ciphertext *ct, uint64_t *pt_host,
                                size_t cap) {
  if (!c || !sk || !ct || !pt_host) return hd_fail(HD_E_INVALID_ARG, "null argument");
  const size_t need = (size_t)ct->limbs * c->n;
  if (cap < need) return hd_fail(HD_E_INVALID_ARG, "capacity too small");
  uint64_t *m;
  HD_CUDA(dev_alloc(c, &m, need * 8));
  hd_status s = decrypt_to(c, sk, ct, m);
  cudaError_t e = cudaMemcpyAsync(pt_host, m, need * 8, cudaMemcpyDeviceToHost, c->stream);
  if (!e) e = cudaStreamSynchronize(c->stream);
  dev_free(c, m);
  if (!s && e) s = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
  return s;
}

static CrtTab crt_table(const hd_context *c, uint32_t nl) {
  CrtTab ctab{};
  for (uint32_t i = 0; i < nl; i++)
    for (uint32_t k = 0; k < i; k++) ctab.inv[i][k] = inv_host(c->mod[k], c->mod[i]);
  {
    std::vector<uint64_t> W(nl + 1, 0);
    W[0] = 1;
    for (uint32_t i = 0; i < nl; i++) {
      for (uint32_t w = 0; w <= nl; w++) ctab.W[i][w] = W[w];
      unsigned __int128 carry = 0;
      for (uint32_t w = 0; w <= nl; w++) {
        unsigned __int128 s2 = (unsigned __int128)W[w] * c->mod[i] + carry;
        W[w] = (uint64_t)s2;
        carry = s2 >> 64;
      }
    }
    for (uint32_t w = 0; w <= nl; w++) ctab.Q[w] = W[w];
  }
  return ctab;
}

extern "C" hd_status hd_decrypt_scores(hd_context *c, const hd_secret_key *sk, const hd_layout *lay,
                                       const hd_ciphertext *const *cts, size_t n_ct, double *scores, size_t capacity,
                                       size_t *written) {
  if (!c || !sk || !lay || !cts || !scores) return hd_fail(HD_E_INVALID_ARG, "null argument");
  const int n = c->n, ns = c->ns, N = (int)lay->block_n, M = (int)lay->blocks_m;
  const int G = (int)lay->groups_per_ct, stride = lay->packing == HD_PACKING_REPLICATED ? 2 * N : N;
  const long long per = (long long)G * N;
  const long long v_first = (long long)lay->agg_begin * per;
  const long long v_end = std::min<long long>((long long)lay->num_vectors, (long long)(lay->agg_begin + n_ct) * per);
  if (v_end <= v_first) return hd_fail(HD_E_INVALID_ARG, "no vectors in the given aggregates");
  if (capacity < (size_t)(v_end - v_first)) return hd_fail(HD_E_INVALID_ARG, "scores capacity too small");
  uint32_t nl = 0;
  for (size_t i = 0; i < n_ct; i++) {
    if (!cts[i]) return hd_fail(HD_E_INVALID_ARG, "null ciphertext");
    if (i == 0) nl = cts[i]->limbs;
    if (cts[i]->limbs != nl) return hd_fail(HD_E_LEVEL, "mixed ciphertext levels");
  }
  const CrtTab ctab = crt_table(c, nl);
  uint64_t *m = nullptr;
  double *re = nullptr, *im = nullptr, *dsc = nullptr;
  const size_t nsc = (size_t)(v_end - v_first);
  cudaError_t e = dev_alloc(c, &m, (size_t)nl * n * 8);
  if (!e) e = dev_alloc(c, &re, (size_t)ns * 8);
  if (!e) e = dev_alloc(c, &im, (size_t)ns * 8);
  if (!e) e = dev_alloc(c, &dsc, nsc * 8);
  hd_status s = e ? hd_fail(HD_E_CUDA, cudaGetErrorString(e)) : HD_OK;
  const double delta = std::ldexp(1.0, (int)c->params.scale_bits);
  RowMap rm{};
  rm.gsize = 1u << 30;
  rm.mdiv = 1;
  rm.mlen = nl;
  for (uint32_t l = 0; l < nl; l++) rm.midx[l] = l;
  for (size_t i = 0; i < n_ct && !s; i++) {
    if ((s = decrypt_to(c, sk, cts[i], m))) break;
    if ((s = ntt_rows(c, m, nl, rm, true))) break;
    crt_decode_kernel<<<(n + TPB - 1) / TPB, TPB, 0, c->stream>>>(m, n, nl, delta, c->logn - 1, re, im, c->mt, ctab); ++c->launches;
    for (int len = 2; len <= ns; len <<= 1)
      fft_fwd_stage_kernel<<<(ns / 2 + TPB - 1) / TPB, TPB, 0, c->stream>>>(re, im, ns, len, c->rotg, c->xi_re,
                                                                            c->xi_im, 2u * n);
    c->launches += c->logn - 1;
    scores_kernel<<<(G * N + TPB - 1) / TPB, TPB, 0, c->stream>>>(re, N, G, stride, (long long)(lay->agg_begin + i),
                                                                 v_first, v_end, dsc); ++c->launches;
  }
  if (!s) {
    e = cudaMemcpyAsync(scores, dsc, nsc * 8, cudaMemcpyDeviceToHost, c->stream);
    if (!e) e = cudaStreamSynchronize(c->stream);
    if (e) s = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
  }
  dev_free(c, m);
  dev_free(c, re);
  dev_free(c, im);
  dev_free(c, dsc);
  if (!s && written) *written = nsc;
  return s;
}

// Decrypt + decode one ciphertext at its own scale (R29): the real parts of all numSlots slots.
extern "C" hd_status hd_decrypt_slots(hd_context *c, const hd_secret_key *sk, const hd_ciphertext *ct, double *slots,
                                      size_t cap) {
  if (!c || !sk || !ct || !slots) return hd_fail(HD_E_INVALID_ARG, "null argument");
  if (cap < (size_t)c->ns) return hd_fail(HD_E_INVALID_ARG, "slots capacity too small");
  const int n = c->n, ns = c->ns;
  const uint32_t nl = ct->limbs;
  const CrtTab ctab = crt_table(c, nl);
  uint64_t *m = nullptr;
  double *re = nullptr, *im = nullptr;
  cudaError_t e = dev_alloc(c, &m, (size_t)nl * n * 8);
  if (!e) e = dev_alloc(c, &re, (size_t)ns * 8);
  if (!e) e = dev_alloc(c, &im, (size_t)ns * 8);
  hd_status s = e ? hd_fail(HD_E_CUDA, cudaGetErrorString(e)) : HD_OK;
  RowMap rm{};
  rm.gsize = 1u << 30;
  rm.mdiv = 1;
  rm.mlen = nl;
  for (uint32_t l = 0; l < nl; l++) rm.midx[l] = l;
  if (!s) s = decrypt_to(c, sk, ct, m);
  if (!s) s = ntt_rows(c, m, nl, rm, true);
  if (!s) {
    crt_decode_kernel<<<(n + TPB - 1) / TPB, TPB, 0, c->stream>>>(m, n, nl, ct->scale, c->logn - 1, re, im, c->mt, ctab);
    ++c->launches;
    for (int len = 2; len <= ns; len <<= 1)
      fft_fwd_stage_kernel<<<(ns / 2 + TPB - 1) / TPB, TPB, 0, c->stream>>>(re, im, ns, len, c->rotg, c->xi_re,
                                                                            c->xi_im, 2u * n);
    c->launches += c->logn - 1;
    e = cudaMemcpyAsync(slots, re, (size_t)ns * 8, cudaMemcpyDeviceToHost, c->stream);
    if (!e) e = cudaStreamSynchronize(c->stream);
    if (e) s = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
  }
  dev_free(c, m);
  dev_free(c, re);
  dev_free(c, im);
  return s;
}

// ---------------------------------------------------------------------------
// Encrypted-database mode (NEXT-1, R26): public key, relinearisation key, public-key
// encryption of batches of plaintext rows (the enroller's diagonals).
// ---------------------------------------------------------------------------
static RowMap limb_rows(int L, uint32_t gsize, uint64_t gstride) {
  RowMap rm{};
  rm.gsize = gsize;
  rm.gstride = gstride;
  rm.mdiv = 1;
  rm.mlen = L;
  for (int l = 0; l < L; l++) rm.midx[l] = (uint8_t)l;
  return rm;
}

extern "C" hd_status hd_public_keygen(hd_context *c, const hd_secret_key *sk, hd_public_key **out) {
  if (!c || !sk || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  *out = nullptr;
  HD_CUDA(cudaSetDevice(c->device));
  const int n = c->n, L = c->L;
  hd_public_key *pk = new hd_public_key{c, nullptr};
  ctx_retain(c);
  if (dev_alloc(c, &pk->pk, (size_t)2 * L * n * 8) != cudaSuccess) {
    hd_public_key_destroy(pk);
    return hd_fail(HD_E_CAPACITY, "public key alloc");
  }
  const uint64_t seed = c->params.seed;
  pk_error_kernel<<<(n + TPB - 1) / TPB, TPB, 0, c->stream>>>(seed, n, L, pk->pk, c->mt); ++c->launches;
  hd_status s = ntt_rows(c, pk->pk, L, limb_rows(L, 1u << 30, 0), false);
  if (!s) {
    pk_combine_kernel<<<dim3((n + TPB - 1) / TPB, L), TPB, 0, c->stream>>>(seed, n, L, sk->s_ntt, pk->pk, c->mt); ++c->launches;
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) s = hd_fail(HD_E_CUDA, "public keygen");
  }
  if (s) {
    hd_public_key_destroy(pk);
    return s;
  }
  *out = pk;
  return HD_OK;
}

extern "C" void hd_public_key_destroy(hd_public_key *pk) {
  if (!pk) return;
  hd_context *c = pk->ctx;
  dev_free(c, pk->pk);
  delete pk;
  ctx_release(c);
}

extern "C" hd_status hd_public_key_export(const hd_public_key *pk, uint64_t *dst, size_t cap) {
  if (!pk || !dst) return hd_fail(HD_E_INVALID_ARG, "null argument");
  const size_t need = (size_t)2 * pk->ctx->L * pk->ctx->n;
  if (cap < need) return hd_fail(HD_E_INVALID_ARG, "capacity too small");
  HD_CUDA(cudaMemcpy(dst, pk->pk, need * 8, cudaMemcpyDeviceToHost));
  return HD_OK;
}

extern "C" hd_status hd_public_key_import(hd_context *c, const uint64_t *src, size_t count, hd_public_key **out) {
  if (!c || !src || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  *out = nullptr;
  const size_t need = (size_t)2 * c->L * c->n;
  if (count != need) return hd_fail(HD_E_FORMAT, "public key must hold 2 L n residues");
  for (size_t i = 0; i < need; i++)
    if (src[i] >= c->mod[(i / c->n) % c->L]) return hd_fail(HD_E_FORMAT, "public key residue out of range");
  hd_public_key *pk = new hd_public_key{c, nullptr};
  ctx_retain(c);
  if (dev_alloc(c, &pk->pk, need * 8) != cudaSuccess) {
    hd_public_key_destroy(pk);
    return hd_fail(HD_E_CAPACITY, "public key alloc");
  }
  if (cudaMemcpy(pk->pk, src, need * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
    hd_public_key_destroy(pk);
    return hd_fail(HD_E_CUDA, "public key copy");
  }
  *out = pk;
  return HD_OK;
}

extern "C" hd_status hd_relin_keygen(hd_context *c, const hd_secret_key *sk, hd_eval_keys *evk) {
  if (!c || !sk || !evk) return hd_fail(HD_E_INVALID_ARG, "null argument");
  if (evk->ctx != c || sk->ctx != c) return hd_fail(HD_E_STATE, "objects from another context");
  if (evk->find(HD_RELIN_STEP)) return HD_OK;  // already present
  HD_CUDA(cudaSetDevice(c->device));
  const int n = c->n, L = c->L, M = ks_M(c), beta = ks_beta(c, L);
  const size_t cnt = evk->steps.size(), ke = ks_key_elems(c);
  uint64_t *keys = nullptr;
  if (dev_alloc(c, &keys, ke * (cnt + 1) * 8) != cudaSuccess) return hd_fail(HD_E_CAPACITY, "relinearisation key alloc");
  if (cnt) HD_CUDA(cudaMemcpyAsync(keys, evk->keys, ke * cnt * 8, cudaMemcpyDeviceToDevice, c->stream));
  uint64_t *key = keys + ke * cnt;
  const uint64_t seed = c->params.seed;
  key_error_kernel<<<dim3((n + TPB - 1) / TPB, beta), TPB, 0, c->stream>>>(seed, 0, TAG_RLK_E, n, M, key, c->mt); ++c->launches;
  RowMap rk = limb_rows(M, M, (uint64_t)2 * M * n);  // rows (d, l) of the b halves
  hd_status s = ntt_rows(c, key, beta * M, rk, false);
  if (s) {
    dev_free(c, keys);
    return s;
  }
  InvTab2 pmod{};
  for (int l = 0; l < L; l++) pmod.w[l] = ks_P_mod(c, c->mod[l]);
  key_combine_kernel<<<dim3((n + TPB - 1) / TPB, beta * M), TPB, 0, c->stream>>>(
      seed, 0, TAG_RLK_A, 0, c->logn, L, M, c->alpha, sk->s_ntt, key, c->mt, pmod); ++c->launches;
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) {
    dev_free(c, keys);
    return hd_fail(HD_E_CUDA, "relinearisation keygen");
  }
  dev_free(c, evk->keys);
  evk->keys = keys;
  evk->key_elems = ke;
  evk->gen = hd_next_generation();  // invalidates every database's cached key pointers
  evk->steps.push_back(HD_RELIN_STEP);
  return HD_OK;
}

hd_status pk_encrypt_rows(hd_context *c, const hd_public_key *pk, uint64_t *ct, size_t ct_stride, uint32_t count,
                          uint64_t enc_seed, uint32_t obj0, uint64_t *V, uint64_t *E0) {
  if (count == 0) return HD_OK;
  const int n = c->n, L = c->L;
  pke_draw_kernel<<<dim3((n + TPB - 1) / TPB, count), TPB, 0, c->stream>>>(enc_seed, obj0, n, L, ct, ct_stride, V, E0,
                                                                           c->mt); ++c->launches;
  hd_status s = ntt_rows(c, V, count * L, limb_rows(L, 1u << 30, 0), false);
  if (!s) s = ntt_rows(c, E0, count * L, limb_rows(L, 1u << 30, 0), false);
  if (!s) s = ntt_rows(c, ct + (size_t)L * n, count * L, limb_rows(L, L, ct_stride), false);
  if (s) return s;
  pke_combine_kernel<<<dim3((n + TPB - 1) / TPB, count * L), TPB, 0, c->stream>>>(n, L, pk->pk, ct, ct_stride, V, E0,
                                                                                 c->mt); ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}
