// enroll.cu -- enrollment (Alg. enroller_bsgs) and CKKS encoding on the GPU.
//
// Pipeline per aggregate (K16 of SURVEY 2.2): upload the aggregate's rows ->
// normalise (Step 1, R16: sequential double sum, IEEE-rounded ops, no FMA) ->
// pack the slot vectors of a batch of diagonals (Steps 2-5: diagonal, giant-step
// right pre-shift shiftN, stride-2N placement) -> special inverse FFT (R15,
// HEAAN order, __dmul_rn/__dadd_rn so nothing is contracted) -> bit-reverse,
// / numSlots, x Delta, round-half-even -> residues mod q_l -> NTT, written
// straight into the device-resident diagonal array D[a][k][l][t].
#include <cmath>

#include "common.cuh"
#include "ks.cuh"

namespace {
constexpr int TPB = 256;

__global__ void normalize_rows_kernel(const float *__restrict__ v, int rows, int dim, double *__restrict__ U,
                                      int *flag) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const float *x = v + (size_t)r * dim;
  double s = 0.0;
  for (int i = 0; i < dim; i++) {
    double xi = (double)x[i];
    s = __dadd_rn(s, __dmul_rn(xi, xi));
  }
  if (s == 0.0) {
    atomicExch(flag, 1);
    return;
  }
  double nrm = __dsqrt_rn(s);
  double *u = U + (size_t)r * dim;
  for (int i = 0; i < dim; i++) u[i] = __ddiv_rn((double)x[i], nrm);
}

// Slot vectors of diagonals k0..k0+B-1 of aggregate `agg` (R4):
// slot b*2N + t (t < N) = diagonal_g[k][(t - shiftN) mod N], g = agg*M/2 + b,
// diagonal_g[k][s] = U[g N + s][(s + k) mod N] (0 beyond the database); gaps 0.
__global__ void pack_kernel(const double *__restrict__ U, long long v_first, long long num_vectors, int N, int M,
                            int n1, long long agg, int k0, int ns, double *__restrict__ re, double *__restrict__ im) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int kk = blockIdx.y;
  if (s >= ns) return;
  const int k = k0 + kk;
  const int b = s / (2 * N), t = s % (2 * N);
  double val = 0.0;
  if (t < N) {
    const int ks = k < N / 2 ? k : k - N;
    const int j = ks >= 0 ? ks / n1 : -((-ks + n1 - 1) / n1);  // floor (R3)
    const int shift = ((n1 * j) % N + N) % N;
    const int src = (t - shift + N) % N;
    const long long g = agg * (M / 2) + b;
    const long long v = g * N + src;
    if (v < num_vectors) val = U[(size_t)(v - v_first) * N + ((src + k) % N)];
  }
  re[(size_t)kk * ns + s] = val;
  im[(size_t)kk * ns + s] = 0.0;
}

// Flat pre-rotated packing (NEXT-2, R27): slot s of diagonal k of aggregate agg is
// diag_k[(s - j n1) mod ns], j = floor(k / n1), with diag_k[b N + t] =
// U[(agg M + b) N + t][(t + k) mod N] (0 beyond the database), M = ns / N, no gaps.
__global__ void pack_flat_kernel(const double *__restrict__ U, long long v_first, long long num_vectors, int N,
                                 int M, int n1, long long agg, int k0, int ns, int prerotate, double *__restrict__ re,
                                 double *__restrict__ im) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  const int kk = blockIdx.y;
  if (s >= ns) return;
  const int k = k0 + kk;
  const int src = prerotate ? ((s - (k / n1) * n1) % ns + ns) % ns : s;  // Rot_{-j n1} (TBE) or none (TBS)
  const int b = src / N, t = src % N;
  const long long v = (agg * M + b) * N + t;
  double val = 0.0;
  if (v < num_vectors) val = U[(size_t)(v - v_first) * N + ((t + k) % N)];
  re[(size_t)kk * ns + s] = val;
  im[(size_t)kk * ns + s] = 0.0;
}

// One stage (len) of the special inverse FFT over B vectors of ns complex slots.
__global__ void fft_inv_stage_kernel(double *__restrict__ re, double *__restrict__ im, int ns, int len,
                                     const uint32_t *__restrict__ rotg, const double *__restrict__ xr,
                                     const double *__restrict__ xim, uint32_t two_n) {
  const int bf = blockIdx.x * blockDim.x + threadIdx.x;
  if (bf >= ns / 2) return;
  const size_t base = (size_t)blockIdx.y * ns;
  const int lenh = len >> 1;
  const uint32_t lenq = (uint32_t)len << 2;
  const int blk = bf / lenh, j = bf % lenh;
  const int i0 = blk * len + j, i1 = i0 + lenh;
  const uint32_t idx = (lenq - (rotg[j] % lenq)) * (two_n / lenq);
  const double wr = xr[idx], wi = xim[idx];
  const double ar = re[base + i0], ai = im[base + i0], br = re[base + i1], bi = im[base + i1];
  const double ur = __dadd_rn(ar, br), ui = __dadd_rn(ai, bi);
  const double vr = __dsub_rn(ar, br), vi = __dsub_rn(ai, bi);
  re[base + i0] = ur;
  im[base + i0] = ui;
  re[base + i1] = __dsub_rn(__dmul_rn(vr, wr), __dmul_rn(vi, wi));
  im[base + i1] = __dadd_rn(__dmul_rn(vr, wi), __dmul_rn(vi, wr));
}

// bit-reverse, / ns, x delta, llrint, residues: out[b][l][c] for c < n.
__global__ void round_kernel(const double *__restrict__ re, const double *__restrict__ im, int ns, int logns,
                             double delta, int nlimbs, uint64_t *__restrict__ out, size_t out_stride, ModTab mt,
                             int *flag) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = 2 * ns;
  if (c >= n) return;
  const size_t b = blockIdx.y;
  const int k = c < ns ? c : c - ns;
  const uint32_t src = __brev((uint32_t)k) >> (32 - logns);
  const double v = (c < ns ? re : im)[b * ns + src];
  const double x = __dmul_rn(__ddiv_rn(v, (double)ns), delta);
  if (!(fabs(x) < 4611686018427387904.0)) atomicExch(flag, 2);
  const long long coef = __double2ll_rn(x);
  uint64_t *o = out + b * out_stride + c;
  for (int l = 0; l < nlimbs; l++) {
    const uint64_t q = mt.q[l];
    uint64_t r;
    if (coef >= 0) {
      r = reduce64((uint64_t)coef, q, mt.bar[l]);
    } else {
      r = reduce64((uint64_t)(-coef), q, mt.bar[l]);
      r = r ? q - r : 0;
    }
    o[(size_t)l * n] = r;
  }
}
}  // namespace

hd_status encode_batch(hd_context *c, double *re, double *im, uint32_t B, double delta, int nlimbs, uint64_t *out,
                       size_t out_stride) {
  const int ns = c->ns;
  int logns = c->logn - 1;
  dim3 g((ns / 2 + TPB - 1) / TPB, B);
  for (int len = ns; len >= 2; len >>= 1)
    fft_inv_stage_kernel<<<g, TPB, 0, c->stream>>>(re, im, ns, len, c->rotg, c->xi_re, c->xi_im, 2u * c->n);
  c->launches += c->logn - 1;
  round_kernel<<<dim3((c->n + TPB - 1) / TPB, B), TPB, 0, c->stream>>>(re, im, ns, logns, delta, nlimbs, out,
                                                                       out_stride, c->mt, c->d_flag); ++c->launches;
  HD_CUDA(cudaGetLastError());
  RowMap rm{};
  rm.gsize = nlimbs;
  rm.gstride = out_stride;
  rm.mdiv = 1;
  rm.mlen = nlimbs;
  for (int l = 0; l < nlimbs; l++) rm.midx[l] = l;
  return ntt_rows(c, out, B * nlimbs, rm, false);
}

hd_status normalize_on_device(hd_context *c, const float *dv, int rows, int dim, double *U) {
  normalize_rows_kernel<<<(rows + TPB - 1) / TPB, TPB, 0, c->stream>>>(dv, rows, dim, U, c->d_flag); ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

hd_status check_flag(hd_context *c) {
  int f = 0;
  HD_CUDA(cudaMemcpyAsync(&f, c->d_flag, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  HD_CUDA(cudaStreamSynchronize(c->stream));
  if (f) {
    HD_CUDA(cudaMemset(c->d_flag, 0, sizeof(int)));
    if (f == 1) return hd_fail(HD_E_ZERO_VECTOR, "an input vector is all zero (cannot L2-normalise)");
    return hd_fail(HD_E_PARAMS, "encoded coefficient exceeds 2^62");
  }
  return HD_OK;
}

// ---------------------------------------------------------------------------
// layout helpers
// ---------------------------------------------------------------------------
static int floordiv_i(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

hd_status layout_make(const hd_context *c, uint64_t K, uint32_t dim, uint32_t n1, uint32_t packing,
                      hd_layout *lay) {
  if (dim < 2 || n1 < 1 || K < 1) return hd_fail(HD_E_INVALID_ARG, "vector_dim >= 2, n1 >= 1, num_vectors >= 1");
  if (packing != HD_PACKING_REPLICATED && packing != HD_PACKING_FLAT && packing != HD_PACKING_FLAT_TBS)
    return hd_fail(HD_E_INVALID_ARG, "packing");
  if ((dim & (dim - 1)) != 0 || (uint32_t)c->ns % (2 * dim) != 0)
    return hd_fail(HD_E_LAYOUT, "vector_dim must be a power of two with numSlots % (2 vector_dim) == 0");
  memset(lay, 0, sizeof(*lay));
  lay->vector_dim = dim;
  lay->n1 = n1;
  lay->num_slots = c->ns;
  lay->block_n = dim;                 // N = min(VECTOR_DIM, numSlots) = VECTOR_DIM
  lay->blocks_m = c->ns / dim;        // M
  lay->groups_per_ct = lay->blocks_m / 2;
  lay->num_vectors = K;
  lay->num_groups = (K + dim - 1) / dim;                                      // G
  lay->num_aggregates = (2 * lay->num_groups + lay->blocks_m - 1) / lay->blocks_m;  // A
  lay->giant_min = floordiv_i(-(int)(dim / 2), (int)n1);                      // R6
  lay->giant_max = floordiv_i((int)(dim / 2) - 1, (int)n1);
  lay->packing = packing;
  if (packing != HD_PACKING_REPLICATED) {  // R27: M groups per ciphertext, j = 0 .. ceil(N/n1) - 1
    lay->groups_per_ct = lay->blocks_m;
    lay->num_aggregates = (lay->num_groups + lay->blocks_m - 1) / lay->blocks_m;
    lay->giant_min = 0;
    lay->giant_max = (int)((dim + n1 - 1) / n1) - 1;
  }
  return HD_OK;
}

extern "C" hd_status hd_rotation_steps_ex(const hd_context *c, uint32_t vector_dim, uint32_t n1, uint32_t packing,
                                          int32_t *steps, size_t cap, size_t *count) {
  if (!c || !count) return hd_fail(HD_E_INVALID_ARG, "null argument");
  hd_layout lay;
  hd_status s = layout_make(c, 1, vector_dim, n1, packing, &lay);
  if (s) return s;
  const int N = (int)vector_dim, ns = c->ns;
  std::vector<char> used(ns, 0);
  for (uint32_t i = 1; i < n1; i++) used[i % ns] = 1;
  if (packing != HD_PACKING_REPLICATED) {  // giant j n1, no fold (R27)
    for (int j = 1; j <= lay.giant_max; j++) used[((int)n1 * j) % ns] = 1;
  } else {
    for (int j = lay.giant_min; j <= lay.giant_max; j++) {
      int pr = (((int)n1 * j) % N + N) % N;
      if (pr) used[pr] = 1;
    }
    used[ns - N] = 1;
  }
  size_t cnt = 0;
  for (int st = 1; st < ns; st++)
    if (used[st]) {
      if (steps && cnt < cap) steps[cnt] = st;
      cnt++;
    }
  *count = cnt;
  if (steps && cnt > cap) return hd_fail(HD_E_INVALID_ARG, "steps capacity too small");
  return HD_OK;
}

extern "C" hd_status hd_rotation_steps(const hd_context *c, uint32_t vector_dim, uint32_t n1, int32_t *steps,
                                       size_t cap, size_t *count) {
  return hd_rotation_steps_ex(c, vector_dim, n1, HD_PACKING_REPLICATED, steps, cap, count);
}

extern "C" hd_status hd_database_layout(const hd_database *db, hd_layout *out) {
  if (!db || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  *out = db->lay;
  return HD_OK;
}

extern "C" hd_status hd_database_diagonal_bytes(const hd_database *db, size_t *bytes, int *packed) {
  if (!db || !bytes) return hd_fail(HD_E_INVALID_ARG, "null argument");
  const hd_context *c = db->ctx;
  *bytes = db->dp.on ? db->dp.diag_bytes : (db->encrypted ? 2 : 1) * (size_t)c->L * c->n * 8;
  if (packed) *packed = db->dp.on ? 1 : 0;
  return HD_OK;
}

extern "C" void hd_database_destroy(hd_database *db) {
  if (!db) return;
  hd_context *c = db->ctx;
  dev_free(c, db->D);
  dev_free(c, db->r);
  dev_free(c, db->S);
  dev_free(c, db->Sp);
  dev_free(c, db->y);
  dev_free(c, db->dig);
  dev_free(c, db->u);
  dev_free(c, db->tmp);
  dev_free(c, db->tmp2);
  dev_free(c, db->outbuf);
  dev_free(c, db->kptr);
  dev_free(c, db->gal);
  dev_free(c, db->S2);
  dev_free(c, db->rB);
  dev_free(c, db->SB[0]);
  dev_free(c, db->SB[1]);
  dev_free(c, db->dig_b);
  dev_free(c, db->u_b);
  dev_free(c, db->tmp_b);
  for (cudaEvent_t e : {db->ev_in, db->ev_mac, db->ev_done, db->ev_sfree[0], db->ev_sfree[1], db->ev_bs})
    if (e) cudaEventDestroy(e);
  delete db;
  ctx_release(c);
}

DPack dpack_make(const hd_context *c, bool on, int polys) {
  DPack P;
  P.on = on;
  P.polys = polys;
  for (int l = 0; l < c->L; l++) {
    const bool narrow = on && c->mod[l] < kNarrowBound;
    P.cls[l] = narrow ? 1 : 0;
    P.idx[l] = (uint8_t)(narrow ? P.R++ : P.W++);
  }
  if (P.R == 0) P.on = false;  // nothing to pack
  P.pp_bytes = (8 * (size_t)P.W + 6 * (size_t)P.R) * c->n;
  P.diag_bytes = (size_t)polys * P.pp_bytes;
  return P;
}

// u64 rows [B][polys][L][n] -> B packed diagonals (R34)
__global__ void pack_d_kernel(const uint64_t *__restrict__ src, uint8_t *__restrict__ dst, DPack P, int L, int logn) {
  const uint32_t n = 1u << logn;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint32_t b = blockIdx.y;
  for (int p = 0; p < P.polys; p++) {
    uint8_t *blk = dst + (size_t)b * P.diag_bytes + (size_t)p * P.pp_bytes;
    for (int l = 0; l < L; l++) dp_put(blk, P, l, t, n, src[(((size_t)b * P.polys + p) * L + l) * n + t]);
  }
}

// Device objects of a database handle: diagonals D (uninitialised), query workspaces, events.
// footprint != NULL: only report the device bytes the handle needs (the paper's pre-upload
// footprint check) and allocate nothing.
static hd_status db_alloc(hd_context *c, const hd_layout &lay, uint32_t packing, bool encrypted, uint32_t n1,
                          hd_database **out, size_t *footprint = nullptr, int pack_override = -1) {
  HD_CUDA(cudaSetDevice(c->device));
  hd_database *db = new hd_database();
  db->ctx = c;
  ctx_retain(c);
  db->lay = lay;
  db->N = lay.vector_dim;
  db->M = lay.blocks_m;
  db->n1 = n1;
  db->A_loc = lay.agg_end - lay.agg_begin;
  db->encrypted = encrypted;
  db->spoly = encrypted ? 3 : 2;
  const int N = (int)db->N, L = c->L, n = c->n, ns = c->ns;
  db->flat = packing != HD_PACKING_REPLICATED;
  db->needs_prerotation = packing == HD_PACKING_FLAT_TBS;
  for (int j = lay.giant_min; j <= lay.giant_max; j++) {
    if (db->flat) {  // R27: diagonals j n1 .. j n1 + n1 - 1 (< N), rotation j n1
      db->js.push_back(j);
      db->pre.push_back((int)((int64_t)n1 * j % ns));
      continue;
    }
    int lo = std::max(0, -j * (int)n1 - N / 2), hi = std::min((int)n1 - 1, N / 2 - 1 - j * (int)n1);
    if (lo > hi) continue;
    db->js.push_back(j);
    db->pre.push_back((((int)n1 * j) % N + N) % N);
  }
  for (size_t i = 1; i < db->js.size(); i++)
    if (db->js[i] != db->js[i - 1] + 1) {
      hd_database_destroy(db);
      return hd_fail(HD_E_LAYOUT, "non-contiguous giant steps");
    }
  const size_t A = db->A_loc, nj = db->js.size(), ctL = (size_t)2 * L * n, ct1 = (size_t)2 * (L - 1) * n;
  const size_t rescale_chunk = std::min<size_t>(A * nj, 256);
  const size_t nb = n1 > 1 ? n1 - 1 : 1;
  // giant / fold / rescale scratch (stream B) and baby-step scratch (stream A)
  // the giant steps' ModUp digits: one slice per rotated giant step (summed by one
  // ks_giant_sum pass, alpha = K = 1), one slice otherwise
  size_t nrot = 0;
  for (int p : db->pre) nrot += p != 0;
  size_t dig_e = A * ks_dig_elems(c, L - 1) * (ks_general(c) ? 1 : std::max<size_t>(1, nrot));
  size_t u_e = A * 2 * (L - 1 + c->K) * n;
  size_t tmp_e = std::max({A * 2 * (L - 1) * n, rescale_chunk * 2 * n, (size_t)L * n});
  const size_t sL = (size_t)db->spoly * L * n;  // one giant-step sum
  if (encrypted) {  // relinearisation of A sums at a time at L limbs (ModUp digits, KIP, ModDown)
    db->relin_chunk = (uint32_t)A;
    dig_e = std::max(dig_e, A * ks_dig_elems(c, L));
    u_e = std::max(u_e, A * 2 * (L + c->K) * n);
    tmp_e = std::max(tmp_e, A * 2 * L * n);
  }
  const size_t dstride = (encrypted ? 2 : 1) * (size_t)L * n;  // one diagonal (pt, or ct)
  // plaintext diagonals are packed (R34) whenever the TMA MAC (the only kernel that reads the
  // packed form) serves this layout; HD_PACK_D=0 keeps u64 words (A/B knob)
  const char *pk_env = getenv("HD_PACK_D");
  const bool tma_ok = encrypted ? mac_tma_ct_supported(c, (int)n1, N, db->flat) && !db->needs_prerotation
                                : mac_tma_supported(c, (int)n1, N, db->flat, 1);
  const bool pack = pack_override >= 0 ? pack_override != 0 : !(pk_env && pk_env[0] == '0') && tma_ok;
  db->dp = dpack_make(c, pack, encrypted ? 2 : 1);
  const size_t d_bytes = db->dp.on ? db->dp.diag_bytes : dstride * 8;
  size_t tmp2_e = encrypted ? A * 2 * (L - 1) * n : 1;  // CRT remainders of the fused relinearise-rescale
  size_t digb_e = ks_dig_elems(c, L), ub_e = nb * 2 * (L + c->K) * n, tmpb_e = std::max(nb * 2 * L * n, (size_t)L * n);
  db->rescale_chunk = (uint32_t)rescale_chunk;
  struct Req {
    void **p;
    size_t bytes;
  } reqs[] = {{(void **)&db->D, A * N * d_bytes},
              {(void **)&db->r, (size_t)n1 * ctL * 8},
              {(void **)&db->S, A * nj * sL * 8},
              {(void **)&db->Sp, A * nj * ct1 * 8},
              {(void **)&db->y, A * ct1 * 8},
              {(void **)&db->outbuf, A * ct1 * 8},
              {(void **)&db->dig, dig_e * 8},
              {(void **)&db->u, u_e * 8},
              {(void **)&db->tmp, tmp_e * 8},
              {(void **)&db->tmp2, tmp2_e * 8},
              {(void **)&db->S2, A * nj * sL * 8},
              {(void **)&db->dig_b, digb_e * 8},
              {(void **)&db->u_b, ub_e * 8},
              {(void **)&db->tmp_b, tmpb_e * 8}};
  size_t total = 0;
  for (auto &q : reqs) total += q.bytes;
  if (footprint) {
    *footprint = total;
    hd_database_destroy(db);
    return HD_OK;
  }
  if (!c->has_alloc) {
    // Default pool: free memory the pool holds but does not use (it keeps freed blocks
    // mapped), then check the footprint before the upload.  With a caller
    // allocator the caller checks hd_enroll_footprint against what it can hand out.
    size_t fr = 0, tot = 0;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, c->device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    HD_CUDA(cudaMemGetInfo(&fr, &tot));
    if (total + (256ull << 20) > fr) {
      hd_database_destroy(db);
      return hd_fail(HD_E_CAPACITY, "database of " + std::to_string(total >> 20) + " MiB exceeds free device memory (" +
                                        std::to_string(fr >> 20) + " MiB); shard the aggregates over more GPUs");
    }
  }
  for (auto &q : reqs) {
    cudaError_t e = dev_alloc(c, q.p, q.bytes);
    if (e != cudaSuccess) {
      hd_database_destroy(db);
      return hd_fail(HD_E_CAPACITY, std::string("device allocation: ") + cudaGetErrorString(e));
    }
  }
  db->bytes = total;
  for (cudaEvent_t *e : {&db->ev_in, &db->ev_mac, &db->ev_done, &db->ev_sfree[0], &db->ev_sfree[1], &db->ev_bs})
    if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) {
      hd_database_destroy(db);
      return hd_fail(HD_E_CUDA, "event creation");
    }
  *out = db;
  return HD_OK;
}

extern "C" hd_status hd_enroll_footprint(hd_context *c, uint64_t num_vectors, uint32_t vector_dim, uint32_t n1,
                                         uint32_t agg_begin, uint32_t agg_end, const hd_enroll_options *opts,
                                         size_t *bytes) {
  if (!c || !bytes) return hd_fail(HD_E_INVALID_ARG, "null argument");
  const uint32_t packing = opts ? opts->packing : HD_PACKING_REPLICATED;
  const bool encrypted = opts && opts->pk;
  hd_layout lay;
  hd_status s = layout_make(c, num_vectors, vector_dim, n1, packing, &lay);
  if (s) return s;
  if (agg_end == 0) agg_end = (uint32_t)lay.num_aggregates;
  if (agg_begin >= agg_end || agg_end > lay.num_aggregates) return hd_fail(HD_E_INVALID_ARG, "bad aggregate range");
  lay.agg_begin = agg_begin;
  lay.agg_end = agg_end;
  return db_alloc(c, lay, packing, encrypted, n1, nullptr, bytes);
}

// pk == NULL: plaintext diagonals (the north-star pt x ct scan); else every diagonal
// plaintext is encrypted under pk (encrypted-database mode, NEXT-1, R26).
static hd_status enroll_impl(hd_context *c, uint32_t packing, const hd_public_key *pk, uint64_t enc_seed,
                             const float *vectors, uint64_t num_vectors, uint32_t vector_dim, uint32_t n1,
                             uint32_t agg_begin, uint32_t agg_end, hd_database **out) {
  if (!c || !vectors || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  if (pk && pk->ctx != c) return hd_fail(HD_E_STATE, "public key from another context");
  if (packing == HD_PACKING_FLAT_TBS && !pk)
    return hd_fail(HD_E_INVALID_ARG, "FLAT_TBS packing needs a public key (encrypted diagonals)");
  *out = nullptr;
  hd_layout lay;
  hd_status s = layout_make(c, num_vectors, vector_dim, n1, packing, &lay);
  if (s) return s;
  if (agg_end == 0) agg_end = (uint32_t)lay.num_aggregates;
  if (agg_begin >= agg_end || agg_end > lay.num_aggregates) return hd_fail(HD_E_INVALID_ARG, "bad aggregate range");
  lay.agg_begin = agg_begin;
  lay.agg_end = agg_end;
  hd_database *db = nullptr;
  if ((s = db_alloc(c, lay, packing, pk != nullptr, n1, &db))) return s;
  const int N = (int)db->N, L = c->L, n = c->n, ns = c->ns;
  const size_t dstride = (pk ? 2 : 1) * (size_t)L * n;  // one diagonal (pt, or ct)
  // enrollment scratch: rows of one aggregate (float + double), FFT buffers for a batch of diagonals
  const size_t rows_per_agg = (size_t)lay.groups_per_ct * N;
  const int KB = std::min(N, std::max(1, (int)((256ull << 20) / ((size_t)ns * 16))));
  float *dv = nullptr;
  double *U = nullptr, *re = nullptr, *im = nullptr;
  cudaError_t e = dev_alloc(c, &dv, rows_per_agg * N * 4);
  if (!e) e = dev_alloc(c, &U, rows_per_agg * N * 8);
  if (!e) e = dev_alloc(c, &re, (size_t)KB * ns * 8);
  if (!e) e = dev_alloc(c, &im, (size_t)KB * ns * 8);
  uint64_t *Pt = nullptr;  // packed diagonals: the u64 rows of a batch before packing (R34)
  if (!e && db->dp.on) e = dev_alloc(c, &Pt, (size_t)KB * dstride * 8);
  uint64_t *V = nullptr, *E0 = nullptr;  // public-key encryption scratch (v, e0 of a batch)
  if (!e && pk) e = dev_alloc(c, &V, (size_t)KB * L * n * 8);
  if (!e && pk) e = dev_alloc(c, &E0, (size_t)KB * L * n * 8);
  auto cleanup = [&]() {
    dev_free(c, dv);
    dev_free(c, U);
    dev_free(c, re);
    dev_free(c, im);
    dev_free(c, V);
    dev_free(c, E0);
    dev_free(c, Pt);
  };
  if (e) {
    cleanup();
    hd_database_destroy(db);
    return hd_fail(HD_E_CAPACITY, "enrollment scratch");
  }
  const double delta = (double)c->mod[L - 1];  // Delta_D = q_{L-1} (R15)
  for (uint32_t a = agg_begin; a < agg_end && !s; a++) {
    const uint64_t v0 = (uint64_t)a * rows_per_agg;
    const uint64_t v1 = std::min<uint64_t>(num_vectors, v0 + rows_per_agg);
    const int rows = (int)(v1 - v0);
    e = cudaMemcpyAsync(dv, vectors + v0 * N, (size_t)rows * N * 4, cudaMemcpyHostToDevice, c->stream);
    if (e) {
      s = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
      break;
    }
    if ((s = normalize_on_device(c, dv, rows, N, U))) break;
    if ((s = check_flag(c))) break;
    uint64_t *Da = db->D + (size_t)(a - agg_begin) * N * dstride;
    for (int k0 = 0; k0 < N && !s; k0 += KB) {
      int kb = std::min(KB, N - k0);
      if (db->flat)
        pack_flat_kernel<<<dim3((ns + TPB - 1) / TPB, kb), TPB, 0, c->stream>>>(
            U, (long long)v0, (long long)num_vectors, N, db->M, n1, a, k0, ns, packing == HD_PACKING_FLAT ? 1 : 0, re,
            im);
      else
        pack_kernel<<<dim3((ns + TPB - 1) / TPB, kb), TPB, 0, c->stream>>>(U, (long long)v0, (long long)num_vectors,
                                                                           N, db->M, n1, a, k0, ns, re, im);
      ++c->launches;
      // plaintext rows (into c0 of each diagonal ciphertext in encrypted mode)
      if (db->dp.on) {  // encode (and encrypt) into u64 rows, then pack (R34)
        s = encode_batch(c, re, im, kb, delta, L, Pt, dstride);
        if (!s && pk)
          s = pk_encrypt_rows(c, pk, Pt, dstride, (uint32_t)kb, enc_seed, (uint32_t)((uint64_t)a * N + k0), V, E0);
        if (!s) {
          uint8_t *Dp = reinterpret_cast<uint8_t *>(db->D) + ((size_t)(a - agg_begin) * N + k0) * db->dp.diag_bytes;
          pack_d_kernel<<<dim3((n + TPB - 1) / TPB, kb), TPB, 0, c->stream>>>(Pt, Dp, db->dp, L, c->logn);
          ++c->launches;
          if (cudaGetLastError() != cudaSuccess) s = hd_fail(HD_E_CUDA, "pack_d_kernel");
        }
        continue;
      }
      s = encode_batch(c, re, im, kb, delta, L, Da + (size_t)k0 * dstride, dstride);
      if (!s && pk)  // Enc_pk with object id a N + k (R26), the oracle's or_enroll_aggregate_encrypted
        s = pk_encrypt_rows(c, pk, Da + (size_t)k0 * dstride, dstride, (uint32_t)kb, enc_seed,
                            (uint32_t)((uint64_t)a * N + k0), V, E0);
    }
    if (!s) s = check_flag(c);
  }
  cleanup();
  if (s) {
    hd_database_destroy(db);
    return s;
  }
  *out = db;
  return HD_OK;
}

// D_out[k][.] = sum_a D[a][k][.] mod q_limb (Alg. online-aggr Step 2).
__global__ void aggregate_kernel(const uint64_t *__restrict__ D, uint64_t *__restrict__ out, uint64_t per_agg,
                                 uint32_t A, int logn, int L, ModTab mt) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= per_agg) return;
  const int l = (int)((e >> logn) % (uint64_t)L);  // [k][poly][limb][coef] or [k][limb][coef]
  const uint64_t q = mt.q[l];
  uint64_t acc = 0;
  for (uint32_t a = 0; a < A; a++) acc = addmod(acc, D[(uint64_t)a * per_agg + e], q);
  out[e] = acc;
}

// the same over packed diagonals (R34): element e = (k, limb, coefficient)
__global__ void aggregate_packed_kernel(const uint8_t *__restrict__ D, uint8_t *__restrict__ out, uint32_t N,
                                        uint32_t A, int logn, int L, ModTab mt, DPack P) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t n = 1ull << logn;
  if (e >= (uint64_t)N * P.polys * L * n) return;
  const uint64_t t = e & (n - 1), kpl = e >> logn;  // (k, poly, limb)
  const int l = (int)(kpl % (uint64_t)L);
  const uint64_t kp = kpl / (uint64_t)L, k = kp / (uint64_t)P.polys, p = kp % (uint64_t)P.polys;
  const uint64_t q = mt.q[l];
  uint64_t acc = 0;
  for (uint32_t a = 0; a < A; a++)
    acc = addmod(acc, dp_get(D + ((uint64_t)a * N + k) * P.diag_bytes + p * P.pp_bytes, P, l, t, n), q);
  dp_put(out + k * P.diag_bytes + p * P.pp_bytes, P, l, t, n, acc);
}

extern "C" hd_status hd_database_aggregate(hd_context *c, const hd_database *src, hd_database **out) {
  if (!c || !src || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  if (src->ctx != c) return hd_fail(HD_E_STATE, "database from another context");
  if (src->needs_prerotation) return hd_fail(HD_E_STATE, "FLAT_TBS database: call hd_database_prerotate first");
  *out = nullptr;
  hd_layout lay = src->lay;
  lay.agg_end = lay.agg_begin + 1;
  hd_database *db = nullptr;
  hd_status s = db_alloc(c, lay, lay.packing, src->encrypted, src->n1, &db, nullptr, src->dp.on ? 1 : 0);
  if (s) return s;
  db->needs_prerotation = false;  // the source's diagonals are already in their final form
  const uint64_t per_agg = (uint64_t)src->N * (src->encrypted ? 2 : 1) * c->L * c->n;
  if (src->dp.on != db->dp.on) {
    hd_database_destroy(db);
    return hd_fail(HD_E_STATE, "aggregate database packing differs from its source");
  }
  if (src->dp.on)  // per_agg = N polys L n elements either way
    aggregate_packed_kernel<<<(unsigned)((per_agg + TPB - 1) / TPB), TPB, 0, c->stream>>>(
        reinterpret_cast<const uint8_t *>(src->D), reinterpret_cast<uint8_t *>(db->D), src->N, src->A_loc, c->logn,
        c->L, c->mt, src->dp);
  else
    aggregate_kernel<<<(unsigned)((per_agg + TPB - 1) / TPB), TPB, 0, c->stream>>>(src->D, db->D, per_agg, src->A_loc,
                                                                                  c->logn, c->L, c->mt);
  ++c->launches;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) {
    hd_database_destroy(db);
    return hd_fail(HD_E_CUDA, cudaGetErrorString(e));
  }
  *out = db;
  return HD_OK;
}

extern "C" hd_status hd_enroll(hd_context *c, const float *vectors, uint64_t num_vectors, uint32_t vector_dim,
                               uint32_t n1, uint32_t agg_begin, uint32_t agg_end, hd_database **out) {
  return enroll_impl(c, HD_PACKING_REPLICATED, nullptr, 0, vectors, num_vectors, vector_dim, n1, agg_begin, agg_end,
                     out);
}

extern "C" hd_status hd_enroll_ex(hd_context *c, const hd_enroll_options *opt, const float *vectors,
                                  uint64_t num_vectors, uint32_t vector_dim, uint32_t n1, uint32_t agg_begin,
                                  uint32_t agg_end, hd_database **out) {
  if (!opt) return hd_enroll(c, vectors, num_vectors, vector_dim, n1, agg_begin, agg_end, out);
  return enroll_impl(c, opt->packing, opt->pk, opt->enc_seed, vectors, num_vectors, vector_dim, n1, agg_begin,
                     agg_end, out);
}

extern "C" hd_status hd_enroll_encrypted(hd_context *c, const hd_public_key *pk, const float *vectors,
                                         uint64_t num_vectors, uint32_t vector_dim, uint32_t n1, uint32_t agg_begin,
                                         uint32_t agg_end, uint64_t enc_seed, hd_database **out) {
  if (!pk) return hd_fail(HD_E_INVALID_ARG, "null public key");
  return enroll_impl(c, HD_PACKING_REPLICATED, pk, enc_seed, vectors, num_vectors, vector_dim, n1, agg_begin,
                     agg_end, out);
}
