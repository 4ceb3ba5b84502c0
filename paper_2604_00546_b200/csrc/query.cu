// query.cu -- the online scan (Alg. sender-bsgs) with the fold
// schedule of DESIGN.md R2, orchestrated on the context stream:
//   a2/a3  hoisted ModUp of q.c1, batched KIP over the n1-1 baby keys, batched ModDown
//   a5     MAC over every local aggregate and giant step (one launch)
//   a6     rescale of every giant-step sum (batched)
//   a7     per giant step j with preRot(j) != 0: ModUp of the c1 of S'_{a,j} for all
//          local aggregates a, KIP with key preRot(j) (read once for all a), ModDown
//          accumulated into y_a; S'_{a,j} with preRot = 0 added directly
//   a8     fold: out_a = y_a + Rot_{numSlots-N}(y_a), batched over a
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "ks.cuh"

#include <nvtx3/nvToolsExt.h>

static hd_status giant_and_fold(hd_database *db, cudaEvent_t *E);
static hd_status scan_tail(hd_database *db, uint64_t *Sbuf, cudaEvent_t *E, bool last, int par, hd_ciphertext **out);

static hd_status bind_keys(hd_database *db, const hd_eval_keys *evk) {
  hd_context *c = db->ctx;
  if (db->keyed_for == evk && db->keyed_gen == evk->gen && db->kptr) return HD_OK;
  const int n1 = (int)db->n1, nj = (int)db->js.size();
  const size_t cnt = (size_t)(n1 - 1) + nj + 1 + (db->encrypted ? 1 : 0);
  std::vector<const uint64_t *> kp(cnt, nullptr);
  std::vector<uint32_t> gl(cnt, 1);
  auto need = [&](int32_t step, size_t slot) -> hd_status {
    const uint64_t *k = evk->find(step);
    if (!k) return hd_fail(HD_E_MISSING_KEY, "missing rotation key for step " + std::to_string(step));
    kp[slot] = k;
    gl[slot] = (uint32_t)host_powmod(5, (uint64_t)step, 2ull * c->n);
    return HD_OK;
  };
  hd_status s;
  for (int i = 1; i < n1; i++)
    if ((s = need(i, i - 1))) return s;
  for (int jj = 0; jj < nj; jj++)
    if (db->pre[jj] && (s = need(db->pre[jj], n1 - 1 + jj))) return s;
  const size_t fold_slot = (size_t)(n1 - 1) + nj;
  if (!db->flat && (s = need(c->ns - (int)db->N, fold_slot))) return s;  // flat packing: no fold (R27)
  if (db->encrypted) {  // relinearisation key: identity permutation (g = 1)
    kp[fold_slot + 1] = evk->find(HD_RELIN_STEP);
    if (!kp[fold_slot + 1])
      return hd_fail(HD_E_MISSING_KEY, "missing relinearisation key (hd_relin_keygen) for an encrypted database");
  }
  if (!db->kptr) {
    HD_CUDA(dev_alloc(c, &db->kptr, cnt * sizeof(uint64_t *)));
    HD_CUDA(dev_alloc(c, &db->gal, cnt * sizeof(uint32_t)));
  }
  HD_CUDA(cudaMemcpyAsync(db->kptr, kp.data(), cnt * sizeof(uint64_t *), cudaMemcpyHostToDevice, c->stream));
  HD_CUDA(cudaMemcpyAsync(db->gal, gl.data(), cnt * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
  HD_CUDA(cudaStreamSynchronize(c->stream));
  db->keyed_for = evk;
  db->keyed_gen = evk->gen;
  return HD_OK;
}

// Stream A: baby steps + MAC of this query (into the S buffer of its parity).
// Stream B: rescale / giant rotations / fold (+ output copies).  A query's B work
// overlaps the next query's A work; S is double-buffered (A waits until B's rescale
// of the query two back has consumed the buffer).  With HD_SERIAL=1 both run on the
// caller's stream.
// NVTX ranges of the query phases (host enqueue side; ncu --nvtx-include "hd_query/mac/" etc.)
struct Nvtx {  // pops whatever is still open when the scope ends (error returns included)
  int depth = 0;
  explicit Nvtx(const char *name) { push(name); }
  void push(const char *name) {
    nvtxRangePushA(name);
    ++depth;
  }
  void pop() {
    if (depth) {
      nvtxRangePop();
      --depth;
    }
  }
  ~Nvtx() {
    while (depth) pop();
  }
};

static hd_status run_scan(hd_database *db, const hd_ciphertext *const *queries, uint32_t Q, cudaStream_t sa,
                          cudaStream_t sb, hd_ciphertext **out, size_t n_out, const uint64_t *r_ext = nullptr) {
  Nvtx range_query("hd_query");
  hd_context *c = db->ctx;
  const int n = c->n, L = c->L, n1 = (int)db->n1, nj = (int)db->js.size();
  const uint32_t A = db->A_loc;
  const size_t ctL = (size_t)2 * L * n, ct1 = (size_t)2 * (L - 1) * n;
  const int par = (int)(db->qcount & 1);
  uint64_t *Sbuf = Q > 1 ? db->SB[par] : (par ? db->S2 : db->S);
  // r_ext: baby steps supplied by the caller (hd_query_baby; written on the caller's stream)
  uint64_t *rbase = r_ext ? const_cast<uint64_t *>(r_ext) : (Q > 1 ? db->rB : db->r);
  const size_t sL = (size_t)db->spoly * L * n;  // one giant-step sum
  const size_t sq = (size_t)A * nj * sL;         // the sums of one query
  cudaStream_t caller = c->stream;
  hd_status s;
  cudaEvent_t *E = c->ev[c->ev_next % 64];
  c->ev_next++;
  c->ev_pending = std::min(c->ev_pending + 1, 64);
  // ---------------- stream A ----------------
  // A depends only on the query's last writer (not on the caller's stream position), so
  // the baby steps + MAC of this query can run while B still finishes the previous one.
  HD_CUDA(cudaEventRecord(db->ev_in, caller));
  if (r_ext) HD_CUDA(cudaStreamWaitEvent(sa, db->ev_in, 0));  // after the caller's baby-step writers
  if (db->bs_pending) {  // an hd_baby_steps on the caller's stream still owns the workspaces
    HD_CUDA(cudaStreamWaitEvent(sa, db->ev_bs, 0));
    db->bs_pending = false;
  }
  for (uint32_t qi = 0; qi < Q && !r_ext; qi++) {
    HD_CUDA(cudaStreamWaitEvent(sa, queries[qi]->ready, 0));
    hd_ciphertext *qmut = const_cast<hd_ciphertext *>(queries[qi]);  // reader bookkeeping only
    if (!qmut->used) {
      HD_CUDA(cudaEventCreateWithFlags(&qmut->used, cudaEventDisableTiming));
    } else {
      HD_CUDA(cudaStreamWaitEvent(sa, qmut->used, 0));  // the new `used` covers earlier readers too
    }
  }
  if (db->qcount >= 2) HD_CUDA(cudaStreamWaitEvent(sa, db->ev_sfree[par], 0));
  c->stream = sa;
  cudaEventRecord(E[0], sa);
  if (n1 <= 1 || r_ext) {  // no baby-step key inner product here: an empty KIP phase
    cudaEventRecord(E[7], sa);
    cudaEventRecord(E[8], sa);
  }
  // ---- baby steps: r[0] = q; r[i] = Rot_i(q), hoisted (per query) ----
  range_query.push("baby_steps");
  for (uint32_t qi = 0; qi < Q && !r_ext; qi++) {
    const hd_ciphertext *query = queries[qi];
    uint64_t *rq = rbase + (size_t)qi * n1 * ctL;
    HD_CUDA(cudaMemcpyAsync(rq, query->data, ctL * 8, cudaMemcpyDeviceToDevice, sa));
    if (n1 > 1) {
      if ((s = ks_modup(c, query->data + (size_t)L * n, 0, 1, L, db->dig_b, db->tmp_b))) return s;
      cudaEventRecord(E[7], sa);
      if ((s = ks_kip(c, db->dig_b, query->data + (size_t)L * n, 0, 1, n1 - 1, L, db->kptr, db->gal, db->u_b)))
        return s;
      cudaEventRecord(E[8], sa);
      if ((s = ks_moddown(c, db->u_b, n1 - 1, n1 - 1, L, db->gal, query->data, 0, rq + ctL, ctL, false,
                          db->tmp_b)))
        return s;
    }
    HD_CUDA(cudaEventRecord(const_cast<hd_ciphertext *>(query)->used, sa));  // not read after the baby steps
  }
  cudaEventRecord(E[1], sa);
  // ---- MAC; a batch streams D once for all its queries (NEXT-4) ----
  range_query.pop();
  range_query.push("mac");
  if (Q > 1) {
    if ((s = mac_batch_run(c, db->D, rbase, Sbuf, A, n1, (int)db->N, db->js, db->flat, Q, db->dp))) return s;
  } else if (db->encrypted) {
    if ((s = mac_ct_run(c, db->D, rbase, Sbuf, A, n1, (int)db->N, db->js, db->flat, db->dp))) return s;
  } else if ((s = mac_run(c, db->D, rbase, Sbuf, A, n1, (int)db->N, db->js, db->flat, db->dp))) {
    return s;
  }
  cudaEventRecord(E[2], sa);
  HD_CUDA(cudaEventRecord(db->ev_mac, sa));
  // ---------------- stream B ----------------
  range_query.pop();
  range_query.push("rescale_giant_fold");
  HD_CUDA(cudaStreamWaitEvent(sb, db->ev_mac, 0));
  c->stream = sb;
  cudaEventRecord(E[3], sb);
  // outputs may still be read by caller-stream work enqueued before this call
  HD_CUDA(cudaStreamWaitEvent(sb, db->ev_in, 0));
  for (uint32_t qi = 0; qi < Q; qi++) {
    if ((s = scan_tail(db, Sbuf + qi * sq, E, qi + 1 == Q, par, out + (size_t)qi * A))) return s;
  }
  HD_CUDA(cudaEventRecord(db->ev_done, sb));
  HD_CUDA(cudaStreamWaitEvent(caller, db->ev_done, 0));
  db->qcount++;
  return HD_OK;
}

// Stream B of one query: relinearisation (encrypted), rescale, giant steps, fold, output copies.
static hd_status scan_tail(hd_database *db, uint64_t *Sbuf, cudaEvent_t *E, bool last, int par, hd_ciphertext **out) {
  hd_context *c = db->ctx;
  const int n = c->n, L = c->L, n1 = (int)db->n1, nj = (int)db->js.size();
  const uint32_t A = db->A_loc;
  const size_t ct1 = (size_t)2 * (L - 1) * n;
  const size_t sL = (size_t)db->spoly * L * n;  // one giant-step sum
  cudaStream_t sb = c->stream;
  hd_status s;
  if (db->encrypted) {
    // ---- Relinearize and Rescale every degree-2 S_{a,j} in one rounding by
    //      P q_{L-1}: bit-identical to KeySwitch_{s^2->s}(d2) added to (d0, d1) then Rescale
    //      (mixed-radix identity, R29), 2 L NTT rows fewer per sum ----
    const uint32_t total = A * nj;
    const size_t rslot = (size_t)(n1 - 1) + nj + 1;
    for (uint32_t b0 = 0; b0 < total; b0 += db->relin_chunk) {
      const uint32_t B = std::min(db->relin_chunk, total - b0);
      if ((s = ks_relin_rescale(c, Sbuf + (size_t)b0 * sL, B, L, db->kptr + rslot, db->gal + rslot,
                                db->Sp + (size_t)b0 * ct1, db->dig, db->u, db->tmp, db->tmp2)))
        return s;
    }
  } else {
    // ---- rescale every S_{a,j} ----
    const uint32_t total = A * nj;
    for (uint32_t b0 = 0; b0 < total; b0 += db->rescale_chunk) {
      uint32_t B = std::min(db->rescale_chunk, total - b0);
      if ((s = ks_rescale(c, Sbuf + (size_t)b0 * sL, sL, B, L, db->Sp + (size_t)b0 * ct1, ct1, db->tmp, db->tmp2)))
        return s;
    }
  }
  if (last) HD_CUDA(cudaEventRecord(db->ev_sfree[par], sb));
  cudaEventRecord(E[4], sb);
  if ((s = giant_and_fold(db, E))) return s;
  for (size_t i = 0; i < A; i++) {
    if (out[i]->used) HD_CUDA(cudaStreamWaitEvent(sb, out[i]->used, 0));  // pending async export
    HD_CUDA(cudaMemcpyAsync(out[i]->data, db->outbuf + i * ct1, ct1 * 8, cudaMemcpyDeviceToDevice, sb));
    out[i]->scale = std::ldexp(1.0, (int)c->params.scale_bits);  // R15: the scan's output scale
    HD_CUDA(cudaEventRecord(out[i]->ready, sb));
  }
  return HD_OK;
}

static hd_status giant_and_fold(hd_database *db, cudaEvent_t *E) {
  hd_context *c = db->ctx;
  const int n = c->n, L = c->L, n1 = (int)db->n1, nj = (int)db->js.size();
  const uint32_t A = db->A_loc;
  const size_t ct1 = (size_t)2 * (L - 1) * n;
  hd_status s;
  // ---- giant rotations and sum (R2), accumulated in Q u {P} with one
  //      ModDown per aggregate (R23) ----
  const int ell = L - 1;
  const size_t ext = (size_t)2 * (ell + c->K) * n;  // u: [A][2][ell+K][n]
  const size_t sp_stride = (size_t)nj * ct1;  // between aggregates for fixed j
  int nrot = 0, nzero = 0;
  for (int jj = 0; jj < nj; jj++) (db->pre[jj] ? nrot : nzero)++;
  if (!ks_general(c) && nrot <= 8 && nzero <= 1) {
    // every rotated step's ModUp into its own digit slice, then the whole sum in one pass
    const size_t dslice = (size_t)A * ks_dig_elems(c, ell);
    std::vector<const uint64_t *> digs, cts;
    std::vector<int> slots;
    const uint64_t *t0 = nullptr;
    for (int jj = 0; jj < nj; jj++) {
      const uint64_t *Sj = db->Sp + (size_t)jj * ct1;
      if (db->pre[jj] == 0) {
        t0 = Sj;
        continue;
      }
      uint64_t *dj = db->dig + digs.size() * dslice;
      if ((s = ks_modup(c, Sj + (size_t)ell * n, sp_stride, A, ell, dj, db->tmp))) return s;
      digs.push_back(dj);
      cts.push_back(Sj);
      slots.push_back(n1 - 1 + jj);
    }
    if ((s = ks_giant_sum(c, A, ell, (int)digs.size(), digs.data(), cts.data(), slots.data(), t0, sp_stride, db->kptr,
                          db->gal, db->u)))
      return s;
  } else {  // general profile: accumulate rotation by rotation
  HD_CUDA(cudaMemsetAsync(db->u, 0, (size_t)A * ext * 8, c->stream));
  for (int jj = 0; jj < nj; jj++) {
    const uint64_t *Sj = db->Sp + (size_t)jj * ct1;
    if (db->pre[jj] == 0) {
      if ((s = ks_add_pscaled(c, db->u, Sj, sp_stride, A, ell))) return s;
      continue;
    }
    const size_t slot = (size_t)(n1 - 1) + jj;
    if ((s = ks_modup(c, Sj + (size_t)ell * n, sp_stride, A, ell, db->dig, db->tmp))) return s;
    if ((s = ks_kip_accumulate(c, db->dig, Sj, sp_stride, A, ell, db->kptr + slot, db->gal + slot, db->u))) return s;
  }
  }
  if ((s = ks_moddown(c, db->u, A, 1, ell, db->gal, nullptr, 0, db->y, ct1, false, db->tmp))) return s;
  cudaEventRecord(E[5], c->stream);
  if (db->flat) {  // flat packing (R27): no gaps, no fold -- out = y
    HD_CUDA(cudaMemcpyAsync(db->outbuf, db->y, (size_t)A * ct1 * 8, cudaMemcpyDeviceToDevice, c->stream));
    cudaEventRecord(E[6], c->stream);
    return HD_OK;
  }
  // ---- fold: out = y + Rot_{numSlots - N}(y) ----
  {
    const size_t slot = (size_t)(n1 - 1) + nj;
    HD_CUDA(cudaMemcpyAsync(db->outbuf, db->y, (size_t)A * ct1 * 8, cudaMemcpyDeviceToDevice, c->stream));
    if ((s = ks_modup(c, db->y + (size_t)(L - 1) * n, ct1, A, L - 1, db->dig, db->tmp))) return s;
    if ((s = ks_kip(c, db->dig, db->y + (size_t)(L - 1) * n, ct1, A, 1, L - 1, db->kptr + slot, db->gal + slot,
                    db->u)))
      return s;
    if ((s = ks_moddown(c, db->u, A, 1, L - 1, db->gal + slot, db->y, ct1, db->outbuf, ct1, true, db->tmp))) return s;
  }
  cudaEventRecord(E[6], c->stream);
  return HD_OK;
}

static hd_status ensure_streams(hd_context *c) {
  // B (key switching, ALU-bound) gets the higher priority: its CTAs are dispatched ahead
  // of the remaining CTAs of the HBM-bound MAC grid running on A.
  int lo = 0, hi = 0;
  HD_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  // HD_PRIO (A/B knob): unset / "B" -> stream B high; "A" -> stream A high; "0" -> equal
  const char *pr = getenv("HD_PRIO");
  const bool a_hi = pr && pr[0] == 'A', b_hi = !(pr && (pr[0] == '0' || pr[0] == 'A'));
  if (!c->sA) HD_CUDA(cudaStreamCreateWithPriority(&c->sA, cudaStreamNonBlocking, a_hi ? hi : lo));
  if (!c->sB) HD_CUDA(cudaStreamCreateWithPriority(&c->sB, cudaStreamNonBlocking, b_hi ? hi : lo));
  return HD_OK;
}

extern "C" hd_status hd_query(hd_context *c, const hd_eval_keys *evk, const hd_database *dbc,
                              const hd_ciphertext *query, hd_ciphertext **out, size_t n_out) {
  if (!c || !evk || !dbc || !query || (!out && n_out)) return hd_fail(HD_E_INVALID_ARG, "null argument");
  hd_database *db = const_cast<hd_database *>(dbc);
  if (db->ctx != c || evk->ctx != c || query->ctx != c) return hd_fail(HD_E_STATE, "objects from another context");
  if (query->limbs != (uint32_t)c->L) return hd_fail(HD_E_LEVEL, "query must be at L limbs");
  if (n_out != db->A_loc) return hd_fail(HD_E_INVALID_ARG, "n_out must equal agg_end - agg_begin");
  if (db->needs_prerotation) return hd_fail(HD_E_STATE, "FLAT_TBS database: call hd_database_prerotate first");
  const int L = c->L, n = c->n;
  const size_t ct1 = (size_t)2 * (L - 1) * n;
  hd_status s = bind_keys(db, evk);
  if (s) return s;
  for (size_t i = 0; i < n_out; i++) {
    if (out[i] && (out[i]->ctx != c || out[i]->limbs != (uint32_t)(L - 1)))
      return hd_fail(HD_E_LEVEL, "reused output ciphertext has the wrong shape");
  }
  (void)ct1;
  std::vector<hd_ciphertext *> fresh;
  std::vector<hd_ciphertext *> outs(out, out + n_out);
  for (size_t i = 0; i < n_out; i++)
    if (!out[i]) {
      hd_ciphertext *ct;
      if ((s = alloc_ct(c, L - 1, &ct))) {
        for (auto *f : fresh) hd_ciphertext_destroy(f);
        return s;
      }
      fresh.push_back(ct);
      outs[i] = ct;
    }
  const char *serial = getenv("HD_SERIAL");
  cudaStream_t sa = c->stream, sb = c->stream;
  if (!(serial && serial[0] == '1')) {
    if ((s = ensure_streams(c))) return s;
    sa = c->sA;
    sb = c->sB;
  }
  cudaStream_t caller = c->stream;
  s = run_scan(db, &query, 1, sa, sb, outs.data(), n_out);
  c->stream = caller;
  if (s) {
    for (auto *f : fresh) hd_ciphertext_destroy(f);
    return s;
  }
  for (size_t i = 0; i < n_out; i++) out[i] = outs[i];
  HD_CUDA(cudaGetLastError());
  db->has_run = true;
  // per-phase times are read lazily by hd_query_stats (no sync here)
  return HD_OK;
}

extern "C" hd_status hd_query_batch(hd_context *c, const hd_eval_keys *evk, const hd_database *dbc,
                                    const hd_ciphertext *const *queries, size_t n_queries, hd_ciphertext **out,
                                    size_t n_out) {
  if (!c || !evk || !dbc || !queries || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  if (n_queries == 0 || n_queries > 64) return hd_fail(HD_E_INVALID_ARG, "n_queries must be in [1, 64]");
  hd_database *db = const_cast<hd_database *>(dbc);
  if (db->ctx != c || evk->ctx != c) return hd_fail(HD_E_STATE, "objects from another context");
  if (db->encrypted) return hd_fail(HD_E_INVALID_ARG, "query batching needs plaintext diagonals (hd_query per query)");
  if (n_out != n_queries * db->A_loc) return hd_fail(HD_E_INVALID_ARG, "n_out must equal n_queries * local aggregates");
  if (db->needs_prerotation) return hd_fail(HD_E_STATE, "FLAT_TBS database: call hd_database_prerotate first");
  const int L = c->L, n = c->n, n1 = (int)db->n1, nj = (int)db->js.size();
  const uint32_t Q = (uint32_t)n_queries;
  for (size_t q = 0; q < n_queries; q++) {
    if (!queries[q]) return hd_fail(HD_E_INVALID_ARG, "null query");
    if (queries[q]->ctx != c) return hd_fail(HD_E_STATE, "query from another context");
    if (queries[q]->limbs != (uint32_t)L) return hd_fail(HD_E_LEVEL, "query must be at L limbs");
  }
  for (size_t i = 0; i < n_out; i++)
    if (out[i] && (out[i]->ctx != c || out[i]->limbs != (uint32_t)(L - 1)))
      return hd_fail(HD_E_LEVEL, "reused output ciphertext has the wrong shape");
  hd_status s = bind_keys(db, evk);
  if (s) return s;
  if (Q > 1 && Q > db->qb_cap) {  // setup-time allocation for this batch size (kept for later batches)
    dev_free(c, db->rB);  // dev_free waits for this context's streams only
    dev_free(c, db->SB[0]);
    dev_free(c, db->SB[1]);
    db->rB = db->SB[0] = db->SB[1] = nullptr;
    db->qb_cap = 0;
    const size_t ctL = (size_t)2 * L * n, sq = (size_t)db->A_loc * nj * 2 * L * n;
    cudaError_t e = dev_alloc(c, &db->rB, (size_t)Q * n1 * ctL * 8);
    if (!e) e = dev_alloc(c, &db->SB[0], (size_t)Q * sq * 8);
    if (!e) e = dev_alloc(c, &db->SB[1], (size_t)Q * sq * 8);
    if (e) return hd_fail(e == cudaErrorMemoryAllocation ? HD_E_CAPACITY : HD_E_CUDA, "query batch workspace");
    db->qb_cap = Q;
  }
  std::vector<hd_ciphertext *> fresh;
  std::vector<hd_ciphertext *> outs(out, out + n_out);
  for (size_t i = 0; i < n_out; i++)
    if (!out[i]) {
      hd_ciphertext *ct;
      if ((s = alloc_ct(c, L - 1, &ct))) {
        for (auto *f : fresh) hd_ciphertext_destroy(f);
        return s;
      }
      fresh.push_back(ct);
      outs[i] = ct;
    }
  const char *serial = getenv("HD_SERIAL");
  cudaStream_t sa = c->stream, sb = c->stream;
  if (!(serial && serial[0] == '1')) {
    if ((s = ensure_streams(c))) return s;
    sa = c->sA;
    sb = c->sB;
  }
  cudaStream_t caller = c->stream;
  s = run_scan(db, queries, Q, sa, sb, outs.data(), n_out);
  c->stream = caller;
  if (s) {
    for (auto *f : fresh) hd_ciphertext_destroy(f);
    return s;
  }
  for (size_t i = 0; i < n_out; i++) out[i] = outs[i];
  HD_CUDA(cudaGetLastError());
  db->has_run = true;
  return HD_OK;
}

// Baby steps r[i], i in [i_begin, i_end), of one query into a caller device buffer laid out
// [n1][2][L][n] (multi-GPU: each rank computes a slice, an all-gather assembles r).
extern "C" hd_status hd_baby_steps(hd_context *c, const hd_eval_keys *evk, const hd_database *dbc,
                                   const hd_ciphertext *query, uint32_t i_begin, uint32_t i_end, void *r_dev) {
  if (!c || !evk || !dbc || !query || !r_dev) return hd_fail(HD_E_INVALID_ARG, "null argument");
  hd_database *db = const_cast<hd_database *>(dbc);
  if (db->ctx != c || evk->ctx != c || query->ctx != c) return hd_fail(HD_E_STATE, "objects from another context");
  if (query->limbs != (uint32_t)c->L) return hd_fail(HD_E_LEVEL, "query must be at L limbs");
  if (i_begin > i_end || i_end > db->n1) return hd_fail(HD_E_INVALID_ARG, "baby-step range outside [0, n1]");
  hd_status s = bind_keys(db, evk);
  if (s) return s;
  const int n = c->n, L = c->L;
  const size_t ctL = (size_t)2 * L * n;
  uint64_t *r = static_cast<uint64_t *>(r_dev);
  HD_CUDA(cudaStreamWaitEvent(c->stream, query->ready, 0));
  if (i_begin == 0 && i_end > 0)
    HD_CUDA(cudaMemcpyAsync(r, query->data, ctL * 8, cudaMemcpyDeviceToDevice, c->stream));
  const uint32_t i0 = i_begin > 1 ? i_begin : 1;
  if (i_end > i0) {
    const uint32_t K = i_end - i0;  // rotations i0 .. i_end - 1 use key slots i0 - 1 ..
    if ((s = ks_modup(c, query->data + (size_t)L * n, 0, 1, L, db->dig_b, db->tmp_b))) return s;
    if ((s = ks_kip(c, db->dig_b, query->data + (size_t)L * n, 0, 1, K, L, db->kptr + (i0 - 1), db->gal + (i0 - 1),
                    db->u_b)))
      return s;
    if ((s = ks_moddown(c, db->u_b, K, K, L, db->gal + (i0 - 1), query->data, 0, r + (size_t)i0 * ctL, ctL, false,
                        db->tmp_b)))
      return s;
  }
  hd_ciphertext *qmut = const_cast<hd_ciphertext *>(query);  // reader bookkeeping only
  if (!qmut->used) HD_CUDA(cudaEventCreateWithFlags(&qmut->used, cudaEventDisableTiming));
  HD_CUDA(cudaEventRecord(qmut->used, c->stream));
  HD_CUDA(cudaEventRecord(db->ev_bs, c->stream));
  db->bs_pending = true;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

// The scan from caller-supplied baby steps (all n1 of them, [n1][2][L][n] on the device).
extern "C" hd_status hd_query_baby(hd_context *c, const hd_eval_keys *evk, const hd_database *dbc, const void *r_dev,
                                   hd_ciphertext **out, size_t n_out) {
  if (!c || !evk || !dbc || !r_dev || (!out && n_out)) return hd_fail(HD_E_INVALID_ARG, "null argument");
  hd_database *db = const_cast<hd_database *>(dbc);
  if (db->ctx != c || evk->ctx != c) return hd_fail(HD_E_STATE, "objects from another context");
  if (n_out != db->A_loc) return hd_fail(HD_E_INVALID_ARG, "n_out must equal agg_end - agg_begin");
  if (db->needs_prerotation) return hd_fail(HD_E_STATE, "FLAT_TBS database: call hd_database_prerotate first");
  const int L = c->L;
  hd_status s = bind_keys(db, evk);
  if (s) return s;
  for (size_t i = 0; i < n_out; i++)
    if (out[i] && (out[i]->ctx != c || out[i]->limbs != (uint32_t)(L - 1)))
      return hd_fail(HD_E_LEVEL, "reused output ciphertext has the wrong shape");
  std::vector<hd_ciphertext *> fresh;
  std::vector<hd_ciphertext *> outs(out, out + n_out);
  for (size_t i = 0; i < n_out; i++)
    if (!out[i]) {
      hd_ciphertext *ct;
      if ((s = alloc_ct(c, L - 1, &ct))) {
        for (auto *f : fresh) hd_ciphertext_destroy(f);
        return s;
      }
      fresh.push_back(ct);
      outs[i] = ct;
    }
  const char *serial = getenv("HD_SERIAL");
  cudaStream_t sa = c->stream, sb = c->stream;
  if (!(serial && serial[0] == '1')) {
    if ((s = ensure_streams(c))) return s;
    sa = c->sA;
    sb = c->sB;
  }
  cudaStream_t caller = c->stream;
  s = run_scan(db, nullptr, 1, sa, sb, outs.data(), n_out, static_cast<const uint64_t *>(r_dev));
  c->stream = caller;
  if (s) {
    for (auto *f : fresh) hd_ciphertext_destroy(f);
    return s;
  }
  for (size_t i = 0; i < n_out; i++) out[i] = outs[i];
  HD_CUDA(cudaGetLastError());
  db->has_run = true;
  return HD_OK;
}

extern "C" hd_status hd_query_stats(const hd_context *cc, double *phase_ms, size_t n_phases) {
  if (!cc || !phase_ms) return hd_fail(HD_E_INVALID_ARG, "null argument");
  hd_context *c = const_cast<hd_context *>(cc);
  // average over the queries issued since the previous call (up to the last 64)
  if (c->ev_pending > 0) {
    // events: 0 A start, 1 baby done, 2 MAC done (A), 3 B start, 4 rescale, 5 giant, 6 fold (B),
    // 7 / 8 around the baby-step key inner product (A; == 0 when n1 == 1)
    static const int from[6] = {0, 1, 3, 4, 5, 7}, to[6] = {1, 2, 4, 5, 6, 8};
    double acc[6] = {0, 0, 0, 0, 0, 0};
    const int last = (c->ev_next - 1) % 64;
    HD_CUDA(cudaEventSynchronize(c->ev[last][6]));
    for (int q = 0; q < c->ev_pending; q++) {
      const int idx = ((c->ev_next - 1 - q) % 64 + 64) % 64;
      for (int i = 0; i < 6; i++) {
        float ms = 0;
        HD_CUDA(cudaEventElapsedTime(&ms, c->ev[idx][from[i]], c->ev[idx][to[i]]));
        acc[i] += ms;
      }
    }
    for (int i = 0; i < 6; i++) c->last_phase_ms[i] = acc[i] / c->ev_pending;
    c->ev_pending = 0;
  }
  for (size_t i = 0; i < n_phases && i < 6; i++) phase_ms[i] = c->last_phase_ms[i];
  return HD_OK;
}

extern "C" hd_status hd_test_stage(const hd_database *db, int which, uint32_t agg, int32_t index, uint64_t *host_dst,
                                   size_t cap) {
  if (!db || !host_dst) return hd_fail(HD_E_INVALID_ARG, "null argument");
  const hd_context *c = db->ctx;
  const int n = c->n, L = c->L, nj = (int)db->js.size();
  const size_t ctL = (size_t)2 * L * n, ct1 = (size_t)2 * (L - 1) * n, ptL = (size_t)L * n;
  if (agg < db->lay.agg_begin || agg >= db->lay.agg_end) return hd_fail(HD_E_INVALID_ARG, "aggregate not in database");
  const size_t a = agg - db->lay.agg_begin;
  const uint64_t *src = nullptr;
  size_t len = 0;
  int jj = index - (db->js.empty() ? 0 : db->js.front());
  switch (which) {
    case 0:
      if (index < 0 || index >= (int)db->n1) return hd_fail(HD_E_INVALID_ARG, "baby index");
      src = db->r + (size_t)index * ctL, len = ctL;
      break;
    case 1:
      if (jj < 0 || jj >= nj) return hd_fail(HD_E_INVALID_ARG, "giant index");
      len = (size_t)db->spoly * L * n;  // encrypted: the degree-2 sum as accumulated
      src = (((db->qcount - 1) & 1) ? db->S2 : db->S) + (a * nj + jj) * len;
      break;
    case 2:
      if (jj < 0 || jj >= nj) return hd_fail(HD_E_INVALID_ARG, "giant index");
      src = db->Sp + (a * nj + jj) * ct1, len = ct1;
      break;
    case 3:
      src = db->y + a * ct1, len = ct1;
      break;
    case 4:
      if (index < 0 || index >= (int)db->N) return hd_fail(HD_E_INVALID_ARG, "diagonal index");
      len = (db->encrypted ? 2 : 1) * ptL;  // plaintext, or the diagonal ciphertext
      if (db->dp.on) {  // packed (R34): copy the diagonal's bytes, unpack on the host
        if (cap < len) return hd_fail(HD_E_INVALID_ARG, "capacity too small");
        std::vector<uint8_t> buf(db->dp.diag_bytes);
        HD_CUDA(cudaStreamSynchronize(c->stream));
        HD_CUDA(cudaMemcpy(buf.data(), reinterpret_cast<const uint8_t *>(db->D) + (a * db->N + index) * db->dp.diag_bytes,
                           buf.size(), cudaMemcpyDeviceToHost));
        for (int p = 0; p < db->dp.polys; p++)
          for (int l = 0; l < L; l++)
            for (int t = 0; t < n; t++)
              host_dst[((size_t)p * L + l) * n + t] = dp_get(buf.data() + p * db->dp.pp_bytes, db->dp, l, t, n);
        return HD_OK;
      }
      src = db->D + (a * db->N + index) * len;
      break;
    default:
      return hd_fail(HD_E_INVALID_ARG, "stage");
  }
  if (which < 4 && !db->has_run) return hd_fail(HD_E_STATE, "no query has run on this database");
  if (cap < len) return hd_fail(HD_E_INVALID_ARG, "capacity too small");
  HD_CUDA(cudaStreamSynchronize(c->stream));
  HD_CUDA(cudaMemcpy(host_dst, src, len * 8, cudaMemcpyDeviceToHost));
  return HD_OK;
}

__global__ void xor_word_kernel(uint64_t *p, uint64_t mask) { *p ^= mask; }
__global__ void xor_u32_kernel(uint32_t *p, uint32_t mask) { *p ^= mask; }
__global__ void xor_u16_kernel(uint16_t *p, uint16_t mask) { *p ^= mask; }

extern "C" hd_status hd_test_inject(hd_database *db, uint32_t agg, int32_t k, uint64_t word, uint64_t mask) {
  if (!db) return hd_fail(HD_E_INVALID_ARG, "null database");
  hd_context *c = db->ctx;
  const size_t dw = (db->encrypted ? 2 : 1) * (size_t)c->L * c->n;  // words of one diagonal
  if (agg < db->lay.agg_begin || agg >= db->lay.agg_end || k < 0 || k >= (int)db->N || word >= dw)
    return hd_fail(HD_E_INVALID_ARG, "fault position outside the database");
  const size_t diag = (size_t)(agg - db->lay.agg_begin) * db->N + k;
  HD_CUDA(cudaStreamSynchronize(c->stream));
  hd_context_synchronize(c);
  if (db->dp.on) {  // packed (R34): the limb's u64 word, or its low (u32) and high (u16) parts
    const int pl = (int)(word / c->n), p = pl / c->L, l = pl % c->L;  // [poly][limb][coef]
    const size_t t = word % c->n;
    uint8_t *dg = reinterpret_cast<uint8_t *>(db->D) + diag * db->dp.diag_bytes + (size_t)p * db->dp.pp_bytes;
    if (!db->dp.cls[l]) {
      xor_word_kernel<<<1, 1, 0, c->stream>>>(reinterpret_cast<uint64_t *>(dg) + (size_t)db->dp.idx[l] * c->n + t, mask);
    } else {
      if (mask >> 47) return hd_fail(HD_E_INVALID_ARG, "mask beyond the 47 bits of a packed residue");
      xor_u32_kernel<<<1, 1, 0, c->stream>>>(
          reinterpret_cast<uint32_t *>(dg + 8 * (size_t)db->dp.W * c->n) + (size_t)db->dp.idx[l] * c->n + t,
          (uint32_t)(mask & 0x7fffffffu));
      xor_u16_kernel<<<1, 1, 0, c->stream>>>(
          reinterpret_cast<uint16_t *>(dg + (8 * (size_t)db->dp.W + 4 * (size_t)db->dp.R) * c->n) +
              (size_t)db->dp.idx[l] * c->n + t,
          (uint16_t)(mask >> 31));
      ++c->launches;
    }
  } else {
    xor_word_kernel<<<1, 1, 0, c->stream>>>(db->D + diag * dw + word, mask);
  }
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  HD_CUDA(cudaStreamSynchronize(c->stream));
  return HD_OK;
}

extern "C" hd_status hd_test_rotate(hd_context *c, const hd_eval_keys *evk, const hd_ciphertext *ct, int32_t step,
                                    hd_ciphertext **out) {
  if (!c || !evk || !ct || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  *out = nullptr;
  const uint64_t *k = evk->find(step);
  if (!k) return hd_fail(HD_E_MISSING_KEY, "missing rotation key for step " + std::to_string(step));
  const int n = c->n, L = c->L, ell = (int)ct->limbs;
  uint64_t *dig, *u, *tmp, **kp;
  uint32_t *g;
  uint32_t gh = (uint32_t)host_powmod(5, (uint64_t)step, 2ull * n);
  HD_CUDA(dev_alloc(c, &dig, ks_dig_elems(c, ell) * 8));
  HD_CUDA(dev_alloc(c, &u, (size_t)2 * (ell + c->K) * n * 8));
  HD_CUDA(dev_alloc(c, &tmp, (size_t)2 * (ell + c->K) * n * 8));
  HD_CUDA(dev_alloc(c, &kp, sizeof(uint64_t *)));
  HD_CUDA(dev_alloc(c, &g, 4));
  HD_CUDA(cudaMemcpy(kp, &k, sizeof(uint64_t *), cudaMemcpyHostToDevice));
  HD_CUDA(cudaMemcpy(g, &gh, 4, cudaMemcpyHostToDevice));
  hd_ciphertext *o;
  hd_status s = alloc_ct(c, ell, &o);
  if (!s) s = ks_modup(c, ct->data + (size_t)ell * n, 0, 1, ell, dig, tmp);
  if (!s) s = ks_kip(c, dig, ct->data + (size_t)ell * n, 0, 1, 1, ell, (const uint64_t *const *)kp, g, u);
  if (!s) s = ks_moddown(c, u, 1, 1, ell, g, ct->data, 0, o->data, 0, false, tmp);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (!s && e) s = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
  dev_free(c, dig);
  dev_free(c, u);
  dev_free(c, tmp);
  dev_free(c, kp);
  dev_free(c, g);
  (void)L;
  if (s) {
    hd_ciphertext_destroy(o);
    return s;
  }
  cudaEventRecord(o->ready, c->stream);
  *out = o;
  return HD_OK;
}

extern "C" hd_status hd_test_rescale(hd_context *c, const hd_ciphertext *ct, hd_ciphertext **out) {
  if (!c || !ct || !out) return hd_fail(HD_E_INVALID_ARG, "null argument");
  *out = nullptr;
  if (ct->limbs < 2) return hd_fail(HD_E_LEVEL, "cannot rescale a 1-limb ciphertext");
  const int n = c->n, ell = (int)ct->limbs;
  uint64_t *t1, *t2;
  HD_CUDA(dev_alloc(c, &t1, (size_t)2 * n * 8));
  HD_CUDA(dev_alloc(c, &t2, (size_t)2 * ell * n * 8));
  hd_ciphertext *o;
  hd_status s = alloc_ct(c, ell - 1, &o);
  if (!s) s = ks_rescale(c, ct->data, 0, 1, ell, o->data, 0, t1, t2);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (!s && e) s = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
  dev_free(c, t1);
  dev_free(c, t2);
  if (s) {
    hd_ciphertext_destroy(o);
    return s;
  }
  cudaEventRecord(o->ready, c->stream);
  *out = o;
  return HD_OK;
}

// ---------------------------------------------------------------------------
// BSGS-RTX-TBS server-side pre-rotation: Dct_k <- Rot_{-j n1}(Dct_k).
// ---------------------------------------------------------------------------
extern "C" hd_status hd_prerotation_steps(const hd_context *c, uint32_t vector_dim, uint32_t n1, int32_t *steps,
                                          size_t cap, size_t *count) {
  if (!c || !count || n1 < 1 || vector_dim < 2) return hd_fail(HD_E_INVALID_ARG, "bad argument");
  std::vector<int32_t> v;
  for (uint32_t j = 1; j * n1 < vector_dim; j++) v.push_back(c->ns - (int32_t)(j * n1 % (uint32_t)c->ns));
  std::sort(v.begin(), v.end());
  *count = v.size();
  if (steps) {
    if (cap < v.size()) return hd_fail(HD_E_INVALID_ARG, "steps capacity too small");
    for (size_t i = 0; i < v.size(); i++) steps[i] = v[i];
  }
  return HD_OK;
}

extern "C" hd_status hd_database_prerotate(hd_context *c, const hd_eval_keys *evk, hd_database *db) {
  if (!c || !evk || !db) return hd_fail(HD_E_INVALID_ARG, "null argument");
  if (db->ctx != c || evk->ctx != c) return hd_fail(HD_E_STATE, "objects from another context");
  if (!db->needs_prerotation) return hd_fail(HD_E_STATE, "not a FLAT_TBS database awaiting pre-rotation");
  HD_CUDA(cudaSetDevice(c->device));
  const int n = c->n, L = c->L, N = (int)db->N, n1 = (int)db->n1;
  const size_t ct = (size_t)2 * L * n;
  const uint32_t Bmax = (uint32_t)std::min(n1, N);
  uint64_t *dig = nullptr, *tmp = nullptr, *u = nullptr, *out = nullptr, **kp = nullptr;
  uint32_t *gal = nullptr;
  cudaError_t e = dev_alloc(c, &dig, (size_t)Bmax * ks_dig_elems(c, L) * 8);
  if (!e) e = dev_alloc(c, &tmp, (size_t)Bmax * 2 * L * n * 8);
  if (!e) e = dev_alloc(c, &u, (size_t)Bmax * 2 * (L + c->K) * n * 8);
  if (!e) e = dev_alloc(c, &out, (size_t)Bmax * ct * 8);
  if (!e) e = dev_alloc(c, &kp, sizeof(uint64_t *));
  if (!e) e = dev_alloc(c, &gal, sizeof(uint32_t));
  hd_status s = e ? hd_fail(HD_E_CAPACITY, "pre-rotation scratch") : HD_OK;
  for (int j = 1; !s && j * n1 < N; j++) {
    const int32_t step = c->ns - (j * n1) % c->ns;
    const uint64_t *key = evk->find(step);
    if (!key) {
      s = hd_fail(HD_E_MISSING_KEY, "missing rotation key for step " + std::to_string(step));
      break;
    }
    const uint32_t g = (uint32_t)host_powmod(5, (uint64_t)step, 2ull * n);
    if ((e = cudaMemcpyAsync(kp, &key, sizeof(key), cudaMemcpyHostToDevice, c->stream)) ||
        (e = cudaMemcpyAsync(gal, &g, sizeof(g), cudaMemcpyHostToDevice, c->stream))) {
      s = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
      break;
    }
    const uint32_t B = (uint32_t)std::min(n1, N - j * n1);
    for (uint32_t a = 0; a < db->A_loc && !s; a++) {
      uint64_t *base = db->D + ((size_t)a * N + (size_t)j * n1) * ct;  // diagonals j n1 .. j n1 + B - 1
      if ((s = ks_modup(c, base + (size_t)L * n, ct, B, L, dig, tmp))) break;
      if ((s = ks_kip(c, dig, base + (size_t)L * n, ct, B, 1, L, kp, gal, u))) break;
      if ((s = ks_moddown(c, u, B, 1, L, gal, base, ct, out, ct, false, tmp))) break;
      if ((e = cudaMemcpyAsync(base, out, (size_t)B * ct * 8, cudaMemcpyDeviceToDevice, c->stream)))
        s = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
    }
    // the host-side key / Galois values must stay valid until their copies ran
    if (!s && (e = cudaStreamSynchronize(c->stream))) s = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
  }
  if (!s && (e = cudaStreamSynchronize(c->stream))) s = hd_fail(HD_E_CUDA, cudaGetErrorString(e));
  dev_free(c, dig);
  dev_free(c, tmp);
  dev_free(c, u);
  dev_free(c, out);
  dev_free(c, kp);
  dev_free(c, gal);
  if (!s) db->needs_prerotation = false;
  return s;
}

