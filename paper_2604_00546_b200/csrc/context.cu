// context.cu -- parameters, tables, object lifetimes and serialisation of libhd.
//
// Moduli (R5): q0 = largest prime < 2^q0_bits, P = largest below q0,
// q1 > q2 > ... = largest primes < 2^scale_bits, all = 1 (mod 2n).
// psi (R13) = the smallest primitive 2n-th root of unity mod each modulus.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>

#include "common.cuh"

typedef unsigned __int128 u128;

static thread_local std::string g_last_error;

hd_status hd_fail(hd_status s, const std::string &msg) {
  g_last_error = msg;
  return s;
}

uint64_t hd_next_generation() {
  static std::atomic<uint64_t> g{1};
  return g.fetch_add(1);
}

extern "C" const char *hd_last_error(void) { return g_last_error.c_str(); }

extern "C" const char *hd_status_string(hd_status s) {
  switch (s) {
    case HD_OK: return "ok";
    case HD_E_INVALID_ARG: return "invalid argument";
    case HD_E_PARAMS: return "unsupported parameters";
    case HD_E_LAYOUT: return "layout error (vector_dim must be a power of two with numSlots % 2N == 0)";
    case HD_E_ZERO_VECTOR: return "zero vector cannot be L2-normalised";
    case HD_E_MISSING_KEY: return "missing rotation key";
    case HD_E_LEVEL: return "ciphertext level mismatch";
    case HD_E_CAPACITY: return "device capacity exceeded";
    case HD_E_CUDA: return "CUDA error";
    case HD_E_STATE: return "object state / context mismatch";
    case HD_E_FORMAT: return "bad serialised format";
  }
  return "unknown status";
}

// ---------------------------------------------------------------------------
// host number theory (independent of oracle/)
// ---------------------------------------------------------------------------
uint64_t host_mulmod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((u128)a * b % m); }
uint64_t host_powmod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1;
  b %= m;
  for (; e; e >>= 1, b = host_mulmod(b, b, m))
    if (e & 1) r = host_mulmod(r, b, m);
  return r;
}
uint64_t host_shoup(uint64_t w, uint64_t q) { return (uint64_t)(((u128)w << 64) / q); }

static bool miller_rabin(uint64_t n) {
  if (n < 4) return n == 2 || n == 3;
  if (n % 2 == 0) return false;
  uint64_t d = n - 1;
  int r = 0;
  while (!(d & 1)) d >>= 1, ++r;
  const uint64_t witnesses[] = {2, 325, 9375, 28178, 450775, 9780504, 1795265022};  // deterministic < 2^64
  for (uint64_t a : witnesses) {
    a %= n;
    if (a == 0) continue;
    uint64_t x = host_powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool ok = false;
    for (int i = 1; i < r && !ok; i++) {
      x = host_mulmod(x, x, n);
      ok = (x == n - 1);
    }
    if (!ok) return false;
  }
  return true;
}

// largest prime p < bound with p = 1 mod 2n
static uint64_t ntt_prime_below(uint64_t bound, uint64_t two_n) {
  uint64_t c = ((bound - 1) / two_n) * two_n + 1;
  if (c >= bound) c -= two_n;
  for (; c > two_n; c -= two_n)
    if (miller_rabin(c)) return c;
  return 0;
}

static uint64_t smallest_primitive_root(uint64_t q, uint64_t n) {
  const uint64_t two_n = 2 * n;
  uint64_t y = 0;
  for (uint64_t x = 2;; x++) {
    y = host_powmod(x, (q - 1) / two_n, q);
    if (host_powmod(y, n, q) == q - 1) break;
  }
  uint64_t best = y, cur = y, y2 = host_mulmod(y, y, q);
  for (uint64_t k = 1; k < n; k++) {
    cur = host_mulmod(cur, y2, q);
    if (cur < best) best = cur;
  }
  return best;
}

static uint32_t bitrev_host(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int i = 0; i < bits; i++) r = (r << 1) | ((x >> i) & 1);
  return r;
}

// ---------------------------------------------------------------------------
// device memory: the caller's allocator or the device's stream-ordered pool
// ---------------------------------------------------------------------------
cudaError_t dev_alloc(hd_context *c, void **p, size_t bytes) {
  *p = nullptr;
  if (bytes == 0) bytes = 8;
  if (c->has_alloc) {
    *p = c->alloc.alloc(bytes, (void *)c->stream, c->alloc.user);
    return *p ? cudaSuccess : cudaErrorMemoryAllocation;
  }
  cudaError_t e = cudaMallocAsync(p, bytes, c->stream);
  // the allocation is ordered on the caller's stream; the pipeline streams may use it next
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  return e;
}

static void quiesce(hd_context *c) {
  for (cudaStream_t s : {c->stream, c->sA, c->sB, c->sIO, c->sUp})
    if (s || s == c->stream) cudaStreamSynchronize(s);
}

void dev_free(hd_context *c, void *p) {
  if (!p) return;
  quiesce(c);  // no stream of the context may still touch the memory
  if (c->has_alloc)
    c->alloc.free(p, (void *)c->stream, c->alloc.user);
  else
    cudaFreeAsync(p, c->stream);
}

void *ws_alloc(hd_context *c, size_t bytes) {
  // smallest cached block that fits and is not more than twice as large
  size_t best = SIZE_MAX;
  for (size_t i = 0; i < c->ws_free.size(); i++) {
    const auto &b = c->ws_free[i];
    if (b.bytes >= bytes && b.bytes <= 2 * bytes + (1u << 20) && (best == SIZE_MAX || b.bytes < c->ws_free[best].bytes))
      best = i;
  }
  if (best != SIZE_MAX) {
    auto b = c->ws_free[best];
    c->ws_free.erase(c->ws_free.begin() + best);
    if (b.stream != c->stream) cudaStreamSynchronize(b.stream);  // freed in another stream's order
    return b.p;
  }
  void *p = nullptr;
  if (c->has_alloc) return c->alloc.alloc(bytes, (void *)c->stream, c->alloc.user);
  return cudaMallocAsync(&p, bytes, c->stream) == cudaSuccess ? p : nullptr;
}

void ws_free(hd_context *c, void *p, size_t bytes) {
  if (p) c->ws_free.push_back({p, bytes, c->stream});  // reusable in c->stream's order
}

extern "C" hd_status hd_context_create(const hd_params *params, int cuda_device, void *cuda_stream,
                                       const hd_allocator *allocator, hd_context **out) {
  if (!params || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  *out = nullptr;
  hd_params p = *params;
  if (!p.num_limbs) p.num_limbs = 3;
  if (!p.q0_bits) p.q0_bits = 60;
  if (!p.scale_bits) p.scale_bits = 45;
  if (!p.special_bits) p.special_bits = 60;
  if (!p.num_special) p.num_special = 1;
  if (!p.digit_limbs) p.digit_limbs = 1;
  if (p.log_n < 4 || p.log_n > 16 || p.num_limbs < 2 || p.num_limbs + p.num_special > HD_MAXMOD ||
      p.digit_limbs > p.num_limbs || p.q0_bits > 60 || p.special_bits != p.q0_bits || p.scale_bits > 60 ||
      p.scale_bits < 20)
    return hd_fail(HD_E_PARAMS, "supported: log_n in [4,16], num_limbs + num_special <= 20, digit_limbs <= num_limbs, "
                                "moduli <= 60 bits");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return hd_fail(HD_E_CUDA, "no CUDA device (libhd has no CPU fallback)");
  if (cuda_device < 0 || cuda_device >= ndev) return hd_fail(HD_E_INVALID_ARG, "bad device index");
  HD_CUDA(cudaSetDevice(cuda_device));
  if (allocator && (!allocator->alloc || !allocator->free))
    return hd_fail(HD_E_INVALID_ARG, "allocator needs both alloc and free");
  if (!allocator) {  // the default pool keeps freed memory mapped for reuse between calls
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, cuda_device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  hd_context *c = new hd_context();
  if (allocator) {
    c->alloc = *allocator;
    c->has_alloc = true;
  }
  c->params = p;
  c->device = cuda_device;
  c->stream = (cudaStream_t)cuda_stream;
  c->logn = (int)p.log_n;
  c->n = 1 << c->logn;
  c->ns = c->n / 2;
  c->L = (int)p.num_limbs;
  c->K = (int)p.num_special;
  c->alpha = (int)p.digit_limbs;
  const uint64_t two_n = 2 * (uint64_t)c->n;
  c->mod[0] = ntt_prime_below(1ull << p.q0_bits, two_n);
  // special primes: the next NTT primes below q0, descending (K = 1: P, R5; R31)
  for (int k = 0; k < c->K; k++) c->mod[c->L + k] = ntt_prime_below(k ? c->mod[c->L + k - 1] : c->mod[0], two_n);
  uint64_t bound = 1ull << p.scale_bits;
  for (int i = 1; i < c->L; i++) bound = c->mod[i] = ntt_prime_below(bound, two_n);
  for (int i = 0; i < c->L + c->K; i++) {
    if (!c->mod[i]) { delete c; return hd_fail(HD_E_PARAMS, "no NTT prime"); }
    c->psi[i] = smallest_primitive_root(c->mod[i], c->n);
    uint64_t q = c->mod[i];
    c->mt.q[i] = q;
    c->mt.bar[i] = (uint64_t)(((u128)1 << 64) / q);
    c->mt.r64[i] = (uint64_t)(((u128)1 << 64) % q);
    c->mt.r64s[i] = host_shoup(c->mt.r64[i], q);
  }
  // NTT twiddles psi^{br(k)} and inverse, Shoup companions, n^{-1}
  const int n = c->n, M = c->L + c->K;
  // interleaved {w, shoup(w)} per index (one 128-bit load per butterfly group)
  std::vector<uint64_t> tw((size_t)2 * M * n), itw((size_t)2 * M * n), nv(2 * HD_MAXMOD, 0);
  std::vector<double> twd((size_t)M * n, 0.0), itwd((size_t)M * n, 0.0);
  for (int l = 0; l < M; l++) {
    uint64_t q = c->mod[l], g = c->psi[l], gi = host_powmod(g, q - 2, q);
    std::vector<uint64_t> pw(n), ipw(n);
    pw[0] = ipw[0] = 1;
    for (int k = 1; k < n; k++) {
      pw[k] = host_mulmod(pw[k - 1], g, q);
      ipw[k] = host_mulmod(ipw[k - 1], gi, q);
    }
    for (int k = 0; k < n; k++) {
      uint32_t b = bitrev_host(k, c->logn);
      tw[2 * ((size_t)l * n + k)] = pw[b];
      tw[2 * ((size_t)l * n + k) + 1] = host_shoup(pw[b], q);
      itw[2 * ((size_t)l * n + k)] = ipw[b];
      itw[2 * ((size_t)l * n + k) + 1] = host_shoup(ipw[b], q);
      if (q < kNttFp64Bound) {  // exact as doubles (< 2^45)
        twd[(size_t)l * n + k] = (double)pw[b];
        itwd[(size_t)l * n + k] = (double)ipw[b];
      }
    }
    c->ninv[l] = host_powmod((uint64_t)n, q - 2, q);
    c->ninvs[l] = host_shoup(c->ninv[l], q);
    nv[l] = c->ninv[l];
    nv[HD_MAXMOD + l] = c->ninvs[l];
  }
  // FFT tables for the special (I)FFT (R15): xi^t = exp(2 pi i t / 2n)
  std::vector<double> xr(two_n), xim(two_n);
  for (uint64_t t = 0; t < two_n; t++) {
    double ang = (2.0 * 3.141592653589793 * (double)t) / (double)two_n;
    xr[t] = std::cos(ang);
    xim[t] = std::sin(ang);
  }
  std::vector<uint32_t> rg(c->ns);
  uint64_t r = 1;
  for (int j = 0; j < c->ns; j++) {
    rg[j] = (uint32_t)r;
    r = r * 5 % two_n;
  }
  auto fail = [&](cudaError_t e) {
    hd_context_destroy(c);
    return hd_fail(HD_E_CUDA, std::string("context tables: ") + cudaGetErrorString(e));
  };
  cudaError_t e;
  if ((e = dev_alloc(c, &c->tw2, tw.size() * 8)) || (e = dev_alloc(c, &c->itw2, itw.size() * 8)) ||
      (e = dev_alloc(c, &c->twd, twd.size() * 8)) || (e = dev_alloc(c, &c->itwd, itwd.size() * 8)) ||
      (e = dev_alloc(c, &c->ninv_dev, nv.size() * 8)) ||
      (e = dev_alloc(c, &c->xi_re, two_n * 8)) || (e = dev_alloc(c, &c->xi_im, two_n * 8)) ||
      (e = dev_alloc(c, &c->rotg, c->ns * 4)) || (e = dev_alloc(c, &c->d_flag, 64)))
    return fail(e);
  if ((e = cudaMemcpy(c->tw2, tw.data(), tw.size() * 8, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(c->itw2, itw.data(), itw.size() * 8, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(c->twd, twd.data(), twd.size() * 8, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(c->itwd, itwd.data(), itwd.size() * 8, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(c->ninv_dev, nv.data(), nv.size() * 8, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(c->xi_re, xr.data(), two_n * 8, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(c->xi_im, xim.data(), two_n * 8, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(c->rotg, rg.data(), c->ns * 4, cudaMemcpyHostToDevice)) ||
      (e = cudaMemset(c->d_flag, 0, 64)))
    return fail(e);
  for (int i = 0; i < hd_context::kPhaseEvents; i++)
    for (int k = 0; k < 64; k++)
      if ((e = cudaEventCreate(&c->ev[k][i]))) return fail(e);
  *out = c;
  return HD_OK;
}

static std::mutex g_ctx_mu;
void ctx_retain(hd_context *c) {
  std::lock_guard<std::mutex> g(g_ctx_mu);
  ++c->refs;
}
static void context_teardown(hd_context *c);
void ctx_release(hd_context *c) {
  bool last;
  {
    std::lock_guard<std::mutex> g(g_ctx_mu);
    last = --c->refs == 0;
  }
  if (last) context_teardown(c);
}

extern "C" void hd_context_destroy(hd_context *c) {
  if (c) ctx_release(c);
}

static void context_teardown(hd_context *c) {
  cudaSetDevice(c->device);
  quiesce(c);
  for (void *p : {(void *)c->tw2, (void *)c->itw2, (void *)c->twd, (void *)c->itwd, (void *)c->ninv_dev, (void *)c->xi_re, (void *)c->xi_im,
                  (void *)c->rotg, (void *)c->d_flag, c->scratch})
    dev_free(c, p);
  for (auto &b : c->ws_free) dev_free(c, b.p);
  c->ws_free.clear();
  if (c->sA) cudaStreamDestroy(c->sA);
  if (c->sB) cudaStreamDestroy(c->sB);
  if (c->sIO) cudaStreamDestroy(c->sIO);
  if (c->sUp) cudaStreamDestroy(c->sUp);
  for (int i = 0; i < hd_context::kPhaseEvents; i++)
    for (int k = 0; k < 64; k++)
      if (c->ev[k][i]) cudaEventDestroy(c->ev[k][i]);
  delete c;
}

extern "C" hd_status hd_launch_count(const hd_context *c, uint64_t *count) {
  if (!c || !count) return hd_fail(HD_E_INVALID_ARG, "null argument");
  *count = c->launches;
  return HD_OK;
}

extern "C" hd_status hd_context_set_stream(hd_context *c, void *s) {
  if (!c) return hd_fail(HD_E_INVALID_ARG, "null context");
  c->stream = (cudaStream_t)s;
  return HD_OK;
}

uint64_t ks_P_mod(const hd_context *c, uint64_t q) {
  uint64_t r = 1 % q;
  for (int k = 0; k < c->K; k++) r = host_mulmod(r, c->mod[c->L + k] % q, q);
  return r;
}

extern "C" hd_status hd_context_moduli(const hd_context *c, uint64_t *moduli, uint64_t *psi, size_t cap) {
  if (!c || cap < (size_t)(c->L + c->K)) return hd_fail(HD_E_INVALID_ARG, "capacity < L + K");
  for (int i = 0; i < c->L + c->K; i++) {
    if (moduli) moduli[i] = c->mod[i];
    if (psi) psi[i] = c->psi[i];
  }
  return HD_OK;
}

// ---------------------------------------------------------------------------
// serialisation: 64-byte header + payload
// ---------------------------------------------------------------------------
namespace {
struct Header {
  char magic[8];     // "HDBSGS01"
  uint32_t kind;     // 1 ciphertext, 2 eval keys
  uint32_t log_n;
  uint32_t limbs;    // ciphertext limbs / L for keys
  uint32_t count;    // number of keys
  uint64_t mod_fp;   // fingerprint of the modulus chain
  uint64_t payload;  // bytes after the header
  double scale;      // ciphertext scale (0 in files of older writers: 2^scale_bits)
  uint8_t pad[16];
};
static_assert(sizeof(Header) == 64, "header");

uint64_t mod_fingerprint(const hd_context *c) {
  uint64_t h = 1469598103934665603ull;
  for (int i = 0; i < c->L + c->K; i++) h = (h ^ c->mod[i]) * 1099511628211ull;
  return h;
}
cudaMemcpyKind kind_of(int dst_dev, int src_dev) {
  if (dst_dev && src_dev) return cudaMemcpyDeviceToDevice;
  if (dst_dev) return cudaMemcpyHostToDevice;
  if (src_dev) return cudaMemcpyDeviceToHost;
  return cudaMemcpyHostToHost;
}
}  // namespace

hd_status alloc_ct(hd_context *c, uint32_t limbs, hd_ciphertext **out) {
  hd_ciphertext *ct = new hd_ciphertext{c, limbs, nullptr};
  ctx_retain(c);
  ct->scale = std::ldexp(1.0, (int)c->params.scale_bits);
  cudaError_t e = dev_alloc(c, &ct->data, sizeof(uint64_t) * 2 * limbs * c->n);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ct->ready, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    dev_free(c, ct->data);
    delete ct;
    ctx_release(c);
    return hd_fail(e == cudaErrorMemoryAllocation ? HD_E_CAPACITY : HD_E_CUDA, "ciphertext alloc");
  }
  *out = ct;
  return HD_OK;
}

extern "C" hd_status hd_ciphertext_limbs(const hd_ciphertext *ct, uint32_t *limbs) {
  if (!ct || !limbs) return hd_fail(HD_E_INVALID_ARG, "null argument");
  *limbs = ct->limbs;
  return HD_OK;
}

extern "C" hd_status hd_ciphertext_export_level(const hd_ciphertext *ct, uint32_t nlimbs, void *dst, size_t cap,
                                                int dst_on_device, size_t *written) {
  if (!ct) return hd_fail(HD_E_INVALID_ARG, "null ciphertext");
  const hd_context *c = ct->ctx;
  if (nlimbs == 0) nlimbs = ct->limbs;
  if (nlimbs > ct->limbs) return hd_fail(HD_E_LEVEL, "cannot export more limbs than the ciphertext has");
  const size_t limb_bytes = sizeof(uint64_t) * c->n;
  size_t payload = 2 * nlimbs * limb_bytes, total = sizeof(Header) + payload;
  if (written) *written = total;
  if (!dst) return HD_OK;
  if (cap < total) return hd_fail(HD_E_INVALID_ARG, "export capacity too small");
  Header h{};
  memcpy(h.magic, "HDBSGS01", 8);
  h.kind = 1;
  h.log_n = c->logn;
  h.limbs = nlimbs;
  h.mod_fp = mod_fingerprint(c);
  h.payload = payload;
  h.scale = ct->scale;
  HD_CUDA(cudaStreamWaitEvent(c->stream, ct->ready, 0));  // last writer (e.g. hd_query's stream B)
  HD_CUDA(cudaMemcpyAsync(dst, &h, sizeof(h), kind_of(dst_on_device, 0), c->stream));
  char *p = (char *)dst + sizeof(h);
  const cudaMemcpyKind kind = kind_of(dst_on_device, 1);
  if (nlimbs == ct->limbs) {
    HD_CUDA(cudaMemcpyAsync(p, ct->data, payload, kind, c->stream));
  } else {  // c0 limbs 0..nlimbs-1, then c1 limbs 0..nlimbs-1 (dropping the top limbs: R24)
    HD_CUDA(cudaMemcpyAsync(p, ct->data, nlimbs * limb_bytes, kind, c->stream));
    HD_CUDA(cudaMemcpyAsync(p + nlimbs * limb_bytes, ct->data + (size_t)ct->limbs * c->n, nlimbs * limb_bytes, kind,
                            c->stream));
  }
  if (!dst_on_device) HD_CUDA(cudaStreamSynchronize(c->stream));  // host copy complete on return
  return HD_OK;
}

extern "C" hd_status hd_ciphertext_export(const hd_ciphertext *ct, void *dst, size_t cap, int dst_on_device,
                                          size_t *written) {
  return hd_ciphertext_export_level(ct, 0, dst, cap, dst_on_device, written);
}

// Every residue row r (n words) must lie in [0, q_m) with m = chain[r % period]; rows of a
// ciphertext [2][limbs][n] use chain = identity, period = limbs; rows of a key set
// [count][L][2][L+1][n] use period L+1 (index L is the special prime P).  One pass on
// the context's stream; the caller's import syncs on it anyway.
__global__ void range_check_kernel(const uint64_t *__restrict__ d, size_t rows, int period, int logn, ModTab mt,
                                   int *flag) {
  const size_t total = rows << logn;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int m = (int)((i >> logn) % (size_t)period);
    if (d[i] >= mt.q[m]) {
      atomicOr(flag, 1);
      return;
    }
  }
}

hd_status check_residues(hd_context *c, const uint64_t *d, size_t rows, int period) {
  int f = 0;
  HD_CUDA(cudaMemsetAsync(c->d_flag, 0, sizeof(int), c->stream));
  range_check_kernel<<<4 * 148, 256, 0, c->stream>>>(d, rows, period, c->logn, c->mt, c->d_flag); ++c->launches;
  HD_CUDA(cudaMemcpyAsync(&f, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  HD_CUDA(cudaStreamSynchronize(c->stream));
  if (f) return hd_fail(HD_E_FORMAT, "serialised residue out of range [0, q)");
  return HD_OK;
}

static hd_status read_header(hd_context *c, const void *src, size_t bytes, int src_dev, Header &h) {
  if (!src || bytes < sizeof(Header)) return hd_fail(HD_E_FORMAT, "short buffer");
  if (src_dev) {
    HD_CUDA(cudaMemcpyAsync(&h, src, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    HD_CUDA(cudaStreamSynchronize(c->stream));
  } else {
    memcpy(&h, src, sizeof(h));
  }
  if (memcmp(h.magic, "HDBSGS01", 8) != 0) return hd_fail(HD_E_FORMAT, "bad magic");
  if (h.log_n != (uint32_t)c->logn || h.mod_fp != mod_fingerprint(c))
    return hd_fail(HD_E_FORMAT, "serialised object belongs to other parameters");
  if (bytes < sizeof(Header) + h.payload) return hd_fail(HD_E_FORMAT, "truncated payload");
  return HD_OK;
}

extern "C" hd_status hd_ciphertext_import(hd_context *c, const void *src, size_t bytes, int src_on_device,
                                          hd_ciphertext **out) {
  if (!c || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  *out = nullptr;
  Header h;
  hd_status s = read_header(c, src, bytes, src_on_device, h);
  if (s) return s;
  if (h.kind != 1 || h.limbs < 1 || h.limbs > (uint32_t)c->L) return hd_fail(HD_E_FORMAT, "not a ciphertext");
  if (h.payload != sizeof(uint64_t) * 2 * h.limbs * c->n)
    return hd_fail(HD_E_FORMAT, "ciphertext payload size does not match its header");
  if (!(h.scale >= 0.0) || std::isinf(h.scale)) return hd_fail(HD_E_FORMAT, "bad ciphertext scale");
  hd_ciphertext *ct;
  if ((s = alloc_ct(c, h.limbs, &ct))) return s;
  if (h.scale > 0.0) ct->scale = h.scale;
  cudaError_t e = cudaMemcpyAsync(ct->data, (const char *)src + sizeof(Header), h.payload,
                                  kind_of(1, src_on_device), c->stream);
  if (e == cudaSuccess) e = cudaEventRecord(ct->ready, c->stream);
  if (e != cudaSuccess) {
    hd_ciphertext_destroy(ct);
    return hd_fail(HD_E_CUDA, cudaGetErrorString(e));
  }
  if ((s = check_residues(c, ct->data, (size_t)2 * h.limbs, h.limbs))) {
    hd_ciphertext_destroy(ct);
    return s;
  }
  *out = ct;
  return HD_OK;
}

extern "C" hd_status hd_ciphertext_import_into(hd_ciphertext *ct, const void *src, size_t bytes,
                                               int src_on_device) {
  if (!ct) return hd_fail(HD_E_INVALID_ARG, "null ciphertext");
  hd_context *c = ct->ctx;
  size_t payload = sizeof(uint64_t) * 2 * ct->limbs * c->n;
  if (!src || bytes < sizeof(Header) + payload) return hd_fail(HD_E_FORMAT, "short buffer");
  if (!src_on_device) {  // header check only for host sources (device: no sync in the hot path)
    Header h;
    hd_status s = read_header(c, src, bytes, 0, h);
    if (s) return s;
    if (h.kind != 1 || h.limbs != ct->limbs || h.payload != payload) return hd_fail(HD_E_LEVEL, "shape mismatch");
    ct->scale = h.scale > 0.0 ? h.scale : std::ldexp(1.0, (int)c->params.scale_bits);
  }
  // Host sources are uploaded on the context's upload stream, ordered only after the
  // ciphertext's last reader (e.g. the baby steps of the previous hd_query on it) and last
  // writer, so the upload of the next query overlaps the current scan.  Device sources
  // (e.g. an NCCL broadcast buffer) are ordered on the caller's stream that produced them.
  cudaStream_t s = c->stream;
  if (!src_on_device) {
    if (!c->sUp) HD_CUDA(cudaStreamCreateWithFlags(&c->sUp, cudaStreamNonBlocking));
    s = c->sUp;  // not behind the result downloads on sIO
    HD_CUDA(cudaStreamWaitEvent(s, ct->ready, 0));
  }
  if (ct->used) HD_CUDA(cudaStreamWaitEvent(s, ct->used, 0));  // pending readers
  HD_CUDA(cudaMemcpyAsync(ct->data, (const char *)src + sizeof(Header), payload, kind_of(1, src_on_device), s));
  HD_CUDA(cudaEventRecord(ct->ready, s));
  return HD_OK;
}

extern "C" hd_status hd_ciphertext_export_async(hd_ciphertext *ct, uint32_t nlimbs, void *dst, size_t cap,
                                                int dst_on_device, size_t *written) {
  if (!ct) return hd_fail(HD_E_INVALID_ARG, "null ciphertext");
  hd_context *c = ct->ctx;
  if (nlimbs == 0) nlimbs = ct->limbs;
  if (nlimbs > ct->limbs) return hd_fail(HD_E_LEVEL, "cannot export more limbs than the ciphertext has");
  const size_t limb_bytes = sizeof(uint64_t) * c->n;
  const size_t payload = 2 * nlimbs * limb_bytes, total = sizeof(Header) + payload;
  if (written) *written = total;
  if (!dst) return HD_OK;
  if (cap < total) return hd_fail(HD_E_INVALID_ARG, "export capacity too small");
  if (!c->sIO) HD_CUDA(cudaStreamCreateWithFlags(&c->sIO, cudaStreamNonBlocking));
  if (!ct->used) {
    HD_CUDA(cudaEventCreateWithFlags(&ct->used, cudaEventDisableTiming));
    HD_CUDA(cudaEventRecord(ct->used, c->sIO));
  }
  Header h{};
  memcpy(h.magic, "HDBSGS01", 8);
  h.kind = 1;
  h.log_n = c->logn;
  h.limbs = nlimbs;
  h.mod_fp = mod_fingerprint(c);
  h.payload = payload;
  h.scale = ct->scale;
  if (dst_on_device)  // pageable source: staged by the runtime before this call returns
    HD_CUDA(cudaMemcpyAsync(dst, &h, sizeof(h), cudaMemcpyHostToDevice, c->sIO));
  else
    memcpy(dst, &h, sizeof(h));
  HD_CUDA(cudaStreamWaitEvent(c->sIO, ct->ready, 0));
  HD_CUDA(cudaStreamWaitEvent(c->sIO, ct->used, 0));  // the new `used` covers earlier readers too
  char *p = (char *)dst + sizeof(h);
  const cudaMemcpyKind kind = kind_of(dst_on_device, 1);
  // c0 limbs 0..nlimbs-1, then c1 limbs 0..nlimbs-1 (dropping the top limbs: R24)
  HD_CUDA(cudaMemcpyAsync(p, ct->data, nlimbs * limb_bytes, kind, c->sIO));
  HD_CUDA(cudaMemcpyAsync(p + nlimbs * limb_bytes, ct->data + (size_t)ct->limbs * c->n, nlimbs * limb_bytes, kind,
                          c->sIO));
  HD_CUDA(cudaEventRecord(ct->used, c->sIO));
  return HD_OK;
}

extern "C" hd_status hd_context_synchronize(hd_context *c) {
  if (!c) return hd_fail(HD_E_INVALID_ARG, "null context");
  for (cudaStream_t s : {c->stream, c->sA, c->sB, c->sIO, c->sUp})
    if (s || s == c->stream) HD_CUDA(cudaStreamSynchronize(s));
  return HD_OK;
}

extern "C" void hd_ciphertext_destroy(hd_ciphertext *ct) {
  if (!ct) return;
  if (ct->ready) {
    cudaEventSynchronize(ct->ready);
    cudaEventDestroy(ct->ready);
  }
  if (ct->used) {
    cudaEventSynchronize(ct->used);
    cudaEventDestroy(ct->used);
  }
  hd_context *c = ct->ctx;
  dev_free(c, ct->data);
  delete ct;
  ctx_release(c);
}

extern "C" hd_status hd_eval_keys_export(const hd_eval_keys *k, void *dst, size_t cap, int dst_on_device,
                                         size_t *written) {
  if (!k) return hd_fail(HD_E_INVALID_ARG, "null keys");
  const hd_context *c = k->ctx;
  size_t nk = k->steps.size();
  size_t steps_bytes = ((nk * 4 + 63) / 64) * 64;
  size_t payload = steps_bytes + sizeof(uint64_t) * k->key_elems * nk, total = sizeof(Header) + payload;
  if (written) *written = total;
  if (!dst) return HD_OK;
  if (cap < total) return hd_fail(HD_E_INVALID_ARG, "export capacity too small");
  Header h{};
  memcpy(h.magic, "HDBSGS01", 8);
  h.kind = 2;
  h.log_n = c->logn;
  h.limbs = c->L;
  h.count = (uint32_t)nk;
  h.mod_fp = mod_fingerprint(c);
  h.payload = payload;
  std::vector<char> head(sizeof(h) + steps_bytes, 0);
  memcpy(head.data(), &h, sizeof(h));
  memcpy(head.data() + sizeof(h), k->steps.data(), nk * 4);
  HD_CUDA(cudaMemcpyAsync(dst, head.data(), head.size(), kind_of(dst_on_device, 0), c->stream));
  HD_CUDA(cudaMemcpyAsync((char *)dst + head.size(), k->keys, sizeof(uint64_t) * k->key_elems * nk,
                          kind_of(dst_on_device, 1), c->stream));
  HD_CUDA(cudaStreamSynchronize(c->stream));
  return HD_OK;
}

extern "C" hd_status hd_eval_keys_import(hd_context *c, const void *src, size_t bytes, int src_on_device,
                                         hd_eval_keys **out) {
  if (!c || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  *out = nullptr;
  Header h;
  hd_status s = read_header(c, src, bytes, src_on_device, h);
  if (s) return s;
  if (h.kind != 2 || h.limbs != (uint32_t)c->L) return hd_fail(HD_E_FORMAT, "not an eval-key set");
  size_t nk = h.count, steps_bytes = ((nk * 4 + 63) / 64) * 64;
  const size_t key_elems = ks_key_elems(c);
  if (nk == 0 || nk > (size_t)c->ns + 1 || h.payload != steps_bytes + sizeof(uint64_t) * key_elems * nk)
    return hd_fail(HD_E_FORMAT, "eval-key payload size does not match its header");
  hd_eval_keys *k = new hd_eval_keys();
  k->ctx = c;
  ctx_retain(c);
  k->steps.resize(nk);
  k->key_elems = key_elems;
  const char *p = (const char *)src + sizeof(Header);
  cudaError_t e = cudaMemcpyAsync(k->steps.data(), p, nk * 4, kind_of(0, src_on_device), c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess) {  // steps: each in [0, numSlots) (0 = relinearisation key), no duplicates
    std::vector<int32_t> st(k->steps);
    std::sort(st.begin(), st.end());
    for (size_t i = 0; i < nk; i++)
      if (st[i] < 0 || st[i] >= c->ns || (i && st[i] == st[i - 1])) {
        hd_eval_keys_destroy(k);
        return hd_fail(HD_E_FORMAT, "eval-key set has an out-of-range or duplicate rotation step");
      }
  }
  if (e == cudaSuccess) e = dev_alloc(c, &k->keys, sizeof(uint64_t) * k->key_elems * nk);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(k->keys, p + steps_bytes, sizeof(uint64_t) * k->key_elems * nk, kind_of(1, src_on_device),
                        c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    hd_eval_keys_destroy(k);
    return hd_fail(e == cudaErrorMemoryAllocation ? HD_E_CAPACITY : HD_E_CUDA, cudaGetErrorString(e));
  }
  if ((s = check_residues(c, k->keys, nk * ks_beta(c, c->L) * 2 * ks_M(c), ks_M(c)))) {
    hd_eval_keys_destroy(k);
    return s;
  }
  *out = k;
  return HD_OK;
}

extern "C" void hd_eval_keys_destroy(hd_eval_keys *k) {
  if (!k) return;
  hd_context *c = k->ctx;
  dev_free(c, k->keys);
  delete k;
  ctx_release(c);
}

extern "C" hd_status hd_secret_key_export(const hd_secret_key *sk, uint64_t *dst, size_t cap) {
  if (!sk || !dst) return hd_fail(HD_E_INVALID_ARG, "null argument");
  const hd_context *c = sk->ctx;
  size_t need = (size_t)ks_M(c) * c->n;
  if (cap < need) return hd_fail(HD_E_INVALID_ARG, "capacity too small");
  HD_CUDA(cudaMemcpy(dst, sk->s_ntt, need * 8, cudaMemcpyDeviceToHost));
  return HD_OK;
}

extern "C" void hd_secret_key_destroy(hd_secret_key *sk) {
  if (!sk) return;
  hd_context *c = sk->ctx;
  dev_free(c, sk->s_ntt);
  delete sk;
  ctx_release(c);
}

extern "C" hd_status hd_test_ntt(hd_context *c, uint64_t *data, uint32_t n_rows, const uint32_t *modulus_idx,
                                 int inverse) {
  if (!c || !data || !modulus_idx) return hd_fail(HD_E_INVALID_ARG, "null argument");
  for (uint32_t r = 0; r < n_rows; r++)
    if (modulus_idx[r] >= (uint32_t)(c->L + c->K)) return hd_fail(HD_E_INVALID_ARG, "modulus index >= L + K");
  uint64_t *d;
  size_t bytes = (size_t)n_rows * c->n * 8;
  HD_CUDA(dev_alloc(c, &d, bytes));
  HD_CUDA(cudaMemcpy(d, data, bytes, cudaMemcpyHostToDevice));
  // rows may have arbitrary moduli: launch one row-group per run of equal index
  hd_status s = HD_OK;
  for (uint32_t r = 0; r < n_rows && !s;) {
    uint32_t e = r;
    while (e < n_rows && modulus_idx[e] == modulus_idx[r]) e++;
    RowMap rm = rowmap_simple(1, {(int)modulus_idx[r]});
    s = ntt_rows(c, d + (size_t)r * c->n, e - r, rm, inverse != 0);
    r = e;
  }
  if (!s) {
    cudaError_t e = cudaStreamSynchronize(c->stream);
    if (e == cudaSuccess) e = cudaMemcpy(data, d, bytes, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) s = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
  }
  dev_free(c, d);
  return s;
}
