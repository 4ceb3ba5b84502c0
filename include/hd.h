/*
 * include/hd.h -- C ABI of the B200-native encrypted BSGS similarity scan
 * (arXiv 2604.00546, "Lightweight, Practical Encrypted Face Recognition with GPU
 * Support").  Implemented by libhd.so (paper_2604_00546_b200/csrc, CUDA sm_100a).
 *
 * The calls follow the paper's problem statement (P = /root/reference/PAPER.md):
 *   - the client holds the secret key, generates rotation keys and encrypts the
 *     query                -> hd_keygen, hd_encrypt_query
 *   - the enroller normalises, diagonalises, packs and encodes the database
 *     (Alg. enroller_bsgs)                -> hd_enroll
 *     optionally encrypting the diagonals under the client's public key (the
 *     paper's threat model; NEXT-1)          -> hd_public_keygen,
 *                                                        hd_relin_keygen, hd_enroll_encrypted
 *     and/or in the flat pre-rotated layout (BSGS-RTX-TBE; NEXT-2)
 *                                                     -> hd_enroll_ex, hd_rotation_steps_ex
 *   - the server evaluates the BSGS scan (Alg. sender-bsgs)
 *                                                     -> hd_query
 *   - the client decrypts and reads the scores (reading R4 of DESIGN.md)
 *                                                     -> hd_decrypt_scores
 *   - or the server thresholds them first (encrypted comparison, identification and
 *     membership tails; NEXT-3)
 *                                                     -> hd_chebyshev_coefficients,
 *                                                        hd_compare(_ex), hd_membership
 *   - serving variants (NEXT-4): several queries per call, the online-aggregated
 *     database (Alg. online-aggr) -> hd_query_batch, hd_database_aggregate
 *   - sharded scans over P GPUs: baby-step slices + all-gather
 *                                                     -> hd_baby_steps, hd_query_baby
 *     and the stream-ordered, level-reduced result export of the gather
 *                                                     -> hd_ciphertext_export_level
 *   - device memory from the caller's allocator (the Python binding
 *     passes PyTorch's caching allocator), the pre-upload footprint check
 *                                         -> hd_context_create, hd_enroll_footprint
 *   - the paper-depth key-switching profile (alpha limbs per digit, K special primes,
 *     R31)                                            -> hd_params.digit_limbs / num_special
 *
 * Conventions
 *   - Every function returns hd_status (HD_OK = 0).  No C++ exception crosses the
 *     ABI.  A human-readable detail of the last failure of the calling thread is
 *     in hd_last_error() (e.g. "missing rotation key for step 489").
 *   - Ownership: every handle returned through an `out` pointer belongs to the
 *     caller and is released by the matching *_destroy (NULL-safe).  Host input
 *     arrays are read-only and never retained.  Output arrays are caller-owned
 *     with an explicit capacity; too small -> HD_E_INVALID_ARG.  On error, out
 *     handles are left NULL (no partial results).
 *   - Device: one hd_context is bound to one CUDA device and one CUDA stream (the
 *     caller's, e.g. torch.cuda.current_stream().cuda_stream; NULL = the legacy
 *     default stream).  Calls on one context must be serialised by the caller.
 *     Internally the scan pipelines two queries on two context-owned streams ordered
 *     by events against the caller's stream; nothing synchronises the device.
 *     All device memory of a context, its keys, databases and ciphertexts is
 *     allocated at creation time of those objects (never inside hd_query).
 *   - Residues: u64 in [0, q), NTT form (bit-reversed evaluation order, DESIGN.md
 *     R13).  Ciphertext layout [poly 0..1][limb][coef]; plaintext [limb][coef];
 *     rotation key [digit d < ceil(L/alpha)][poly (0 = b, 1 = a)][modulus l < L+K][coef]
 *     where modulus indices L..L+K-1 are the special primes p_k.
 *   - No CPU fallback: if no CUDA device is usable every call that computes
 *     returns HD_E_CUDA.
 */
#ifndef HD_H
#define HD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HD_OK = 0,
  HD_E_INVALID_ARG = -1, /* NULL pointer, bad size or capacity              */
  HD_E_PARAMS = -2,      /* unsupported ring / limb profile                 */
  HD_E_LAYOUT = -3,      /* vector_dim not a power of two or numSlots % 2N  */
  HD_E_ZERO_VECTOR = -4, /* an all-zero database or query vector (R17)      */
  HD_E_MISSING_KEY = -5, /* rotation key absent; hd_last_error names it     */
  HD_E_LEVEL = -6,       /* ciphertext at the wrong number of limbs         */
  HD_E_CAPACITY = -7,    /* database / workspace exceeds device memory      */
  HD_E_CUDA = -8,        /* CUDA error or no device                         */
  HD_E_STATE = -9,       /* object from another context / not initialised   */
  HD_E_FORMAT = -10      /* bad serialised header                           */
} hd_status;

const char *hd_status_string(hd_status s);
const char *hd_last_error(void);

typedef struct hd_context hd_context;       /* params + tables, one device      */
typedef struct hd_secret_key hd_secret_key; /* client only                      */
typedef struct hd_eval_keys hd_eval_keys;   /* rotation keys, device-resident   */
typedef struct hd_database hd_database;     /* diagonals of aggregates [agg_begin, agg_end) */
typedef struct hd_ciphertext hd_ciphertext; /* device-resident ciphertext       */
typedef struct hd_public_key hd_public_key; /* encrypted-database mode (R26)     */

/* CKKS parameters (R5, R11, R31).  Defaults (when a field is 0): num_limbs 3,
 * q0_bits 60, scale_bits 45, special_bits 60, num_special 1, digit_limbs 1.
 * Hybrid key switching: digit_limbs (alpha) limbs per digit, num_special (K) special
 * primes p_0 > ... > p_{K-1} (the next NTT primes below q0), P = prod p_k; keys hold
 * ceil(num_limbs / alpha) digits over the num_limbs + K moduli.  alpha = K = 1 is the
 * north-star profile (centred single-limb lifts, R12); any other profile uses fast basis
 * conversion with centred digits (R31) -- e.g. the paper's depth: num_limbs
 * 12, digit_limbs 4, num_special 4.  The scan (hd_query and its parts),
 * rotations and keygen support every profile; relinearisation (encrypted database, the
 * comparison) needs alpha = K = 1 (HD_E_PARAMS else).  num_limbs + num_special <= 20,
 * digit_limbs <= num_limbs, log_n in [4, 16].  seed keys the Philox stream of the secret /
 * rotation keys. */
typedef struct {
  uint32_t log_n, num_limbs, q0_bits, scale_bits, special_bits, num_special, digit_limbs;
  uint32_t reserved;
  uint64_t seed;
} hd_params;

/* Enrollment layout (Alg. enroller_bsgs Steps 2-3). */
typedef struct {
  uint32_t vector_dim, n1, num_slots, block_n, blocks_m, groups_per_ct;
  uint64_t num_vectors, num_groups, num_aggregates;
  int32_t giant_min, giant_max;  /* giantSteps J (R6; flat: 0 .. ceil(N/n1) - 1) */
  uint32_t agg_begin, agg_end;   /* aggregates held by this database handle */
  uint32_t packing;              /* HD_PACKING_* */
  uint32_t reserved;
} hd_layout;

/* Database packings.  REPLICATED: Alg. enroller_bsgs, M/2 groups per
 * ciphertext at stride 2N, giant steps preshifted within blocks and one rotate-by-N
 * fold (the north-star scan).  FLAT (NEXT-2, R27; BSGS-RTX-TBE, P:L846-865,
 * P:L883-905): HyDia packing with M groups per ciphertext and no gaps, diagonals
 * pre-rotated by the enroller (diag'_k = Rot_{-floor(k/n1) n1}(diag_k)), giant steps
 * k = j n1 + i with j >= 0 rotated by j n1 online, no fold: half the diagonal bytes. */
enum { HD_PACKING_REPLICATED = 0, HD_PACKING_FLAT = 1, HD_PACKING_FLAT_TBS = 2 };
/* FLAT_TBS (BSGS-RTX-TBS): encrypted flat diagonals enrolled WITHOUT the
 * enroller's pre-rotation; the server pre-rotates them homomorphically once with
 * hd_database_prerotate (negative giant-step keys numSlots - j n1, hd_prerotation_steps)
 * before the first hd_query (HD_E_STATE otherwise).  Requires a public key. */

/* Options of hd_enroll_ex: packing, and for the encrypted-database mode (NEXT-1)
 * the public key and the enroller's encryption seed (pk = NULL: plaintext diagonals). */
typedef struct {
  uint32_t packing;
  uint32_t reserved;
  const struct hd_public_key *pk;
  uint64_t enc_seed;
} hd_enroll_options;

/* ---- device memory ------------------------------------------------------ */
/* Device allocator of a context ("PyTorch is used only for device memory";
 * the Python binding passes the torch caching allocator).  alloc returns a device pointer
 * of at least `bytes` on the context's device, usable on `stream` (a cudaStream_t) and on
 * streams ordered after it, or NULL (the call then fails with HD_E_CAPACITY).  free
 * releases a pointer alloc returned; the library calls it only once no work on any of the
 * context's streams can still touch the memory, or for per-call temporaries on `stream`
 * in stream order.  Both must be callable from the thread that calls libhd.  `user` is
 * passed through.  Every device allocation of libhd goes through it (tables, keys,
 * databases, ciphertexts, workspaces); with a NULL allocator libhd uses the device's
 * stream-ordered pool (cudaMallocAsync / cudaFreeAsync).  Objects made by a context keep it
 * alive: hd_context_destroy releases the caller's reference and the context's tables go
 * with its last object, so handles may be destroyed in any order (e.g. by a garbage
 * collector); the allocator must stay callable until then. */
typedef struct {
  void *(*alloc)(size_t bytes, void *stream, void *user);
  void (*free)(void *ptr, void *stream, void *user);
  void *user;
} hd_allocator;

/* ---- context ------------------------------------------------------------ */
/* Creates the context: moduli (R5), primitive roots (R13), NTT/FFT tables.
 * cuda_stream: cudaStream_t of the caller (NULL = default stream); one context = one
 * device = one caller stream, and calls on a context are serialised by the caller.
 * allocator: copied; NULL = the device's stream-ordered pool (see hd_allocator).       */
hd_status hd_context_create(const hd_params *params, int cuda_device, void *cuda_stream,
                            const hd_allocator *allocator, hd_context **out);
void hd_context_destroy(hd_context *ctx);
hd_status hd_context_set_stream(hd_context *ctx, void *cuda_stream);
/* moduli[0..L-1] = q_i, moduli[L..L+K-1] = p_k; psi likewise (host arrays, L+K each). */
hd_status hd_context_moduli(const hd_context *ctx, uint64_t *moduli, uint64_t *psi, size_t cap);

/* ---- client -------------------------------------------------------------- */
/* Rotation-key set of the fold schedule (R2): baby {1..n1-1}, giant
 * {preRot(j) != 0}, fold {numSlots - N}; sorted ascending, unique.
 * Writes min(count, cap) steps; *count = total.  cap too small -> HD_E_INVALID_ARG. */
/* Rotation keys of a packing: REPLICATED as hd_rotation_steps; FLAT baby {1..n1-1} and
 * giant {j n1 : 1 <= j < ceil(N/n1)} (the paper's S_baby u S_giant). */
hd_status hd_rotation_steps_ex(const hd_context *ctx, uint32_t vector_dim, uint32_t n1, uint32_t packing,
                               int32_t *steps, size_t cap, size_t *count);
hd_status hd_rotation_steps(const hd_context *ctx, uint32_t vector_dim, uint32_t n1,
                            int32_t *steps, size_t cap, size_t *count);
/* Secret key (ternary, R14) and hybrid key-switching keys for every step
 * (R11), generated on the device. */
hd_status hd_keygen(hd_context *ctx, const int32_t *steps, size_t count, hd_secret_key **sk,
                    hd_eval_keys **evk);
/* L2-normalise q (R16), replicate with period N over all slots (R8), encode at
 * Delta = 2^scale_bits over all L limbs (R15), encrypt symmetrically with the
 * Philox stream keyed by enc_seed (R14).  q: host float32[vector_dim]. */
hd_status hd_encrypt_query(hd_context *ctx, const hd_secret_key *sk, const float *q,
                           uint32_t vector_dim, uint64_t enc_seed, hd_ciphertext **out);
/* As hd_encrypt_query with the normalised query multiplied by msg_scale in (0, 1] before
 * encoding: the online-aggregated membership encrypts q / f_G, f_G = 1 + (G-1) 2/sqrt(l),
 * so the aggregated score stays in the comparison's [-1, 1] (R30).
 * msg_scale = 1 is hd_encrypt_query bit for bit. */
hd_status hd_encrypt_query_ex(hd_context *ctx, const hd_secret_key *sk, const float *q,
                              uint32_t vector_dim, uint64_t enc_seed, double msg_scale, hd_ciphertext **out);
/* Decrypt + decode the n_ct output ciphertexts of aggregates
 * [layout->agg_begin, layout->agg_begin + n_ct) and write the score of every
 * database vector they hold, in vector order (R4): scores[v - v_first] for
 * v in [agg_begin*(M/2)*N, min(num_vectors, agg_end*(M/2)*N)).
 * *written (optional) = number of scores.  Decode is floating point: scores match
 * the cosine within the CKKS error, not bit-exactly. */
hd_status hd_decrypt_scores(hd_context *ctx, const hd_secret_key *sk, const hd_layout *layout,
                            const hd_ciphertext *const *cts, size_t n_ct, double *scores,
                            size_t capacity, size_t *written);
/* Decrypt one ciphertext to its plaintext residues (host u64 [limbs][n]); test use. */
hd_status hd_decrypt(hd_context *ctx, const hd_secret_key *sk, const hd_ciphertext *ct,
                     uint64_t *pt_host, size_t cap);

/* ---- enroller / server ----------------------------------------------------- */
/* Enroll aggregates [agg_begin, agg_end) of a database of num_vectors vectors
 * (host float32, row-major num_vectors x vector_dim): Steps 1-5 of Alg.
 * enroller_bsgs with plaintext diagonals encoded at Delta = q_{L-1}
 * (R1, R15), stored device-resident.  Only rows of the requested aggregates are
 * read, so `vectors` may point at row 0 of the whole database.
 * agg_end = 0 means "all aggregates".  Device memory exhausted -> HD_E_CAPACITY. */
hd_status hd_enroll(hd_context *ctx, const float *vectors, uint64_t num_vectors,
                    uint32_t vector_dim, uint32_t n1, uint32_t agg_begin, uint32_t agg_end,
                    hd_database **out);
/* Encrypted-database mode (NEXT-1; the paper's threat model):
 * as hd_enroll, then every diagonal plaintext is encrypted under the public key
 * (R26: c = (v b + e0 + pt, v a + e1), v ternary, e0/e1 CBD(21), Philox key enc_seed,
 * object id agg * vector_dim + k), so the server never sees the database.  hd_query
 * on such a database computes S_j = Relinearize(sum_i r[i] (x) Dct_k)
 * and needs the relinearisation key in evk (hd_relin_keygen; else HD_E_MISSING_KEY).
 * Diagonal bytes double (2 polynomials). */
hd_status hd_enroll_encrypted(hd_context *ctx, const hd_public_key *pk, const float *vectors,
                              uint64_t num_vectors, uint32_t vector_dim, uint32_t n1,
                              uint32_t agg_begin, uint32_t agg_end, uint64_t enc_seed,
                              hd_database **out);
/* General enrollment: hd_enroll = { REPLICATED, pk = NULL }, hd_enroll_encrypted =
 * { REPLICATED, pk, seed }.  opt = NULL: hd_enroll. */
hd_status hd_enroll_ex(hd_context *ctx, const hd_enroll_options *opt, const float *vectors,
                       uint64_t num_vectors, uint32_t vector_dim, uint32_t n1, uint32_t agg_begin,
                       uint32_t agg_end, hd_database **out);
/* Device bytes the database handle of this enrollment would take (diagonals plus the
 * query workspaces), without allocating: the paper's footprint check before the upload
 * (P:L662-664).  With the default allocator hd_enroll* performs the check itself against
 * free device memory (HD_E_CAPACITY); with a caller allocator the caller checks this
 * figure against what it can hand out. */
hd_status hd_enroll_footprint(hd_context *ctx, uint64_t num_vectors, uint32_t vector_dim, uint32_t n1,
                              uint32_t agg_begin, uint32_t agg_end, const hd_enroll_options *opt,
                              size_t *bytes);
hd_status hd_database_layout(const hd_database *db, hd_layout *out);
/* Device bytes of one stored diagonal (R34).  Plaintext diagonals served by the TMA
 * MAC are stored packed: a limb whose modulus is below 2^47 keeps its residues in 6 bytes (a
 * 31-bit low and a 16-bit high plane), other limbs in 8; at L = 3 (one 60-bit and two 45-bit
 * limbs) a diagonal takes 20 n bytes instead of 24 n.  *packed = 1 when that applies, else the
 * diagonal is L n u64 words (2 L n for encrypted diagonals).  Residue values are unchanged:
 * hd_test_stage returns them as u64 either way. */
hd_status hd_database_diagonal_bytes(const hd_database *db, size_t *bytes, int *packed);
/* Online database aggregation (NEXT-4; Alg. online-aggr, membership only): a new
 * handle with ONE aggregate whose diagonals are the sums (mod q) of the diagonals of all
 * aggregates of db (plaintext or encrypted, any packing; a FLAT_TBS database must be
 * pre-rotated first).  hd_query on it returns one ciphertext whose slots hold the per-slot
 * sums of every aggregate's scores (the scan is linear); the paper then compares that
 * aggregated score and EvalSums it (hd_compare, hd_membership). */
hd_status hd_database_aggregate(hd_context *ctx, const hd_database *db, hd_database **out);
/* Keys of the TBS pre-rotation: {numSlots - j n1 : 1 <= j < ceil(N/n1)} (ascending). */
hd_status hd_prerotation_steps(const hd_context *ctx, uint32_t vector_dim, uint32_t n1, int32_t *steps,
                               size_t cap, size_t *count);
/* Server-side pre-rotation of a FLAT_TBS database, in place: Dct_k <- Rot_{-j n1}(Dct_k)
 * for every diagonal k with j = floor(k / n1) >= 1 (full key switch per diagonal, batched
 * per (aggregate, j)).  evk must hold the pre-rotation keys (HD_E_MISSING_KEY). */
hd_status hd_database_prerotate(hd_context *ctx, const hd_eval_keys *evk, hd_database *db);
/* The online scan (Alg. sender-bsgs; fold schedule R2): baby steps
 * (hoisted), MAC over all local aggregates, rescale, giant rotations accumulated in
 * the extended basis with one ModDown per aggregate (R23), fold.  Encrypted databases
 * relinearise each giant-step sum before its rescale (R26); flat databases have no
 * fold (R27).  out[i] receives the score ciphertext (L-1 limbs) of aggregate
 * agg_begin + i; n_out must equal agg_end - agg_begin.  A non-NULL out[i] from a
 * previous call on the same context is overwritten in place (no allocation), after
 * any pending hd_ciphertext_export_async of it.  The call is asynchronous with
 * respect to the host; outputs carry events that later readers wait on. */
hd_status hd_query(hd_context *ctx, const hd_eval_keys *evk, const hd_database *db,
                   const hd_ciphertext *query, hd_ciphertext **out, size_t n_out);
/* Query batching (NEXT-4): the scan of n_queries (1..64) independent query
 * ciphertexts over the same database in one call.  The baby steps, rescale, giant steps and
 * fold run per query as in hd_query, issued back to back on the pipeline streams.  The
 * diagonal MAC runs per query by default (the fastest kernel measured on B200); with the
 * environment variable HD_MAC_BATCH=2|4 one HBM pass over the diagonals serves groups of 2 or
 * 4 queries (mac_cs_batch_kernel: D bytes per query drop 2-4-fold, but its baby-step words
 * come from L2 and it measured slower).  out[q * n_local + i] receives the score ciphertext of aggregate agg_begin + i
 * for query q, bit-identical to hd_query(queries[q]); n_out = n_queries * n_local.  Plaintext
 * diagonals only (HD_E_INVALID_ARG for an encrypted database).  The batch workspace (baby
 * steps and giant-step sums of n_queries queries, double-buffered) is allocated on the first
 * call with a larger n_queries and kept; outputs as in hd_query. */
hd_status hd_query_batch(hd_context *ctx, const hd_eval_keys *evk, const hd_database *db,
                         const hd_ciphertext *const *queries, size_t n_queries, hd_ciphertext **out, size_t n_out);
/* Split baby steps (with the database sharded over P GPUs every rank would
 * otherwise recompute all n1 - 1 baby rotations).  hd_baby_steps writes r[i] = Rot_i(query)
 * for i in [i_begin, i_end) (r[0] = the query itself) into r_dev, a device buffer laid out
 * [n1][2][L][n] u64 (the caller's, e.g. one slice per rank followed by an NCCL all-gather);
 * hd_query_baby then runs the scan (MAC, rescale, giant steps, fold) from a complete r_dev,
 * bit-identical to hd_query of that query.  Both run in order on the context stream; the
 * baby-step keys of [i_begin, i_end) and the scan keys must be in evk. */
hd_status hd_baby_steps(hd_context *ctx, const hd_eval_keys *evk, const hd_database *db,
                        const hd_ciphertext *query, uint32_t i_begin, uint32_t i_end, void *r_dev);
hd_status hd_query_baby(hd_context *ctx, const hd_eval_keys *evk, const hd_database *db, const void *r_dev,
                        hd_ciphertext **out, size_t n_out);
/* Cumulative number of CUDA kernels this context has launched (all entry points). */
hd_status hd_launch_count(const hd_context *ctx, uint64_t *count);
/* Per-phase device times (ms), averaged over the hd_query calls issued since the
 * previous hd_query_stats call (up to 64; synchronises), CUDA events on the streams
 * that run them: [0] baby steps, [1] MAC, [2] rescale, [3] giant rotations, [4] fold,
 * [5] the baby-step key inner product alone (part of [0]; the key-switch HBM stream).
 * n_phases <= 6 values are written. */
hd_status hd_query_stats(const hd_context *ctx, double *phase_ms, size_t n_phases);

/* ---- serialisation (canonical: 64-byte header + u64 residues) --------------- */
/* dst/src on the host (on_device = 0) or on the context's device (on_device = 1);
 * dst = NULL queries the size in *written. */
hd_status hd_ciphertext_export(const hd_ciphertext *ct, void *dst, size_t cap, int dst_on_device,
                               size_t *written);
/* Imports validate untrusted input before it reaches a kernel: HD_E_FORMAT unless the
 * magic, ring and modulus-chain fingerprint match this context, the header's payload size
 * equals the size its shape implies and fits in `bytes`, and every residue is below its
 * modulus (one device pass); key sets also reject rotation steps outside [0, numSlots)
 * and duplicates.  Synchronises the context stream. */
hd_status hd_ciphertext_import(hd_context *ctx, const void *src, size_t bytes, int src_on_device,
                               hd_ciphertext **out);
/* hd_ciphertext_export at a reduced level: the first nlimbs limbs of c0 and c1 (0 = all;
 * dropping limbs is exact modular reduction, R24).  Stream-ordered on the context stream
 * after the ciphertext's last writer: a device destination never synchronises the host
 * (the multi-GPU result gather); a host destination is complete on return.
 * HD_E_LEVEL if nlimbs > limbs. */
hd_status hd_ciphertext_export_level(const hd_ciphertext *ct, uint32_t nlimbs, void *dst, size_t cap,
                                     int dst_on_device, size_t *written);
/* In-place import into an existing ciphertext of the same shape (no allocation).
 * Host sources are uploaded asynchronously on the context's upload stream, after the
 * ciphertext's last reader (the baby steps of an hd_query on it) and last writer; pinned
 * host memory keeps the copy asynchronous and must stay valid until the ciphertext is
 * next read or hd_context_synchronize().  Device sources are copied on the context stream.
 * Unlike hd_ciphertext_import (which checks the header's payload size and that every
 * residue is below its modulus, HD_E_FORMAT otherwise), this hot-path call checks only the
 * header of host sources (shape and payload size) and nothing of device sources: it never
 * synchronises.  Feed it buffers produced by hd_ciphertext_export(_async). */
hd_status hd_ciphertext_import_into(hd_ciphertext *ct, const void *src, size_t bytes,
                                    int src_on_device);
hd_status hd_ciphertext_limbs(const hd_ciphertext *ct, uint32_t *limbs);
/* Asynchronous, level-reduced export (result download).  Writes the header and the
 * limbs 0..nlimbs-1 of c0 and c1 (nlimbs = 0: all limbs) on an internal copy stream
 * ordered after the ciphertext's last writer, and returns without waiting.  Dropping
 * the top limbs is exact modular reduction to the smaller modulus Q' = q_0..q_{k-1}:
 * decryption is unchanged while the plaintext stays below Q'/2 (R24: scores
 * are < 2^46 against q_0 ~ 2^60), and the bytes halve at nlimbs = 1.  dst: pinned
 * host memory (pageable also works but copies synchronously) or device memory.
 * The data is in dst after hd_context_synchronize(); a later writer of ct (hd_query
 * output, import_into) waits for the copy.  Errors: HD_E_LEVEL if nlimbs > limbs,
 * HD_E_INVALID_ARG if cap is too small (dst = NULL queries the size in *written). */
hd_status hd_ciphertext_export_async(hd_ciphertext *ct, uint32_t nlimbs, void *dst, size_t cap,
                                     int dst_on_device, size_t *written);
/* Waits for all work of the context: its stream, the query pipeline and the copies. */
hd_status hd_context_synchronize(hd_context *ctx);
hd_status hd_eval_keys_export(const hd_eval_keys *evk, void *dst, size_t cap, int dst_on_device,
                              size_t *written);
hd_status hd_eval_keys_import(hd_context *ctx, const void *src, size_t bytes, int src_on_device,
                              hd_eval_keys **out);
/* Secret key in NTT form, host u64 [(L+K)][n]; test use. */
hd_status hd_secret_key_export(const hd_secret_key *sk, uint64_t *dst, size_t cap);

/* Public key pk = (b, a) = (-a s + e, a) over the L ciphertext moduli (R26; Philox
 * tags 6/7 under the context seed), for the enroller's encryption. */
hd_status hd_public_keygen(hd_context *ctx, const hd_secret_key *sk, hd_public_key **out);
/* Host u64 [2][L][n] (b then a), NTT form. */
hd_status hd_public_key_export(const hd_public_key *pk, uint64_t *dst, size_t cap);
hd_status hd_public_key_import(hd_context *ctx, const uint64_t *src, size_t count, hd_public_key **out);
/* Adds the relinearisation key (key switching s^2 -> s, layout of a rotation key,
 * Philox tags 10/11, object 0) to an evaluation-key set; exported/imported with it
 * under the reserved step 0.  No-op if present. */
hd_status hd_relin_keygen(hd_context *ctx, const hd_secret_key *sk, hd_eval_keys *evk);
void hd_public_key_destroy(hd_public_key *pk);

/* ---- encrypted comparison and scenario tail (NEXT-3, R29) ------------ */
/* Degree n of the Chebyshev sign approximation for the comparison depth budget kappa,
 * the paper's lookup table: 7 -> 5, 8 -> 13, 9 -> 27, 10 -> 59; other kappa ->
 * HD_E_INVALID_ARG. */
hd_status hd_chebyshev_degree(uint32_t kappa, uint32_t *degree);
/* Client side (host, no device): the coefficients c_0..c_degree of the degree-n Chebyshev
 * interpolant of f(x) = 1/2 (sign(x - delta) + 1) (Eq. eq:cheb-sign) at the
 * first-kind Chebyshev nodes (DCT-II; R29), so sum_i c_i T_i(x) ~ 1 for x >= delta and ~ 0
 * below, on [-1, 1].  coeffs: host double[cap], cap >= degree + 1. */
hd_status hd_chebyshev_coefficients(double delta, uint32_t degree, double *coeffs, size_t cap);
/* ChebyshevCompare (Alg. gpu-chebyshev; R29): out[i] = sum_k coeffs[k] T_k(in[i])
 * slot-wise, by Paterson-Stockmeyer in the Chebyshev basis ((d1, d2) of P:L725-727) at depth
 * ceil(log2(degree + 1)); every product is relinearised (evk must hold the relinearisation
 * key, hd_relin_keygen; else HD_E_MISSING_KEY) and rescaled at once.  All inputs must share
 * one level and scale (e.g. hd_query outputs); slots are expected in [-1, 1].  The count
 * inputs are evaluated together in batches (one launch per step for the whole batch).
 * out[i]: NULL -> allocated; else overwritten in place (same context and level).  The
 * result level is the input's minus the depth (HD_E_LEVEL if the limbs run out: the scan
 * plus degree 13 needs num_limbs >= 6); its scale is in hd_ciphertext_scale.  Identification
 * (Alg. index) = hd_compare over the hd_query outputs. */
hd_status hd_compare(hd_context *ctx, const hd_eval_keys *evk, const hd_ciphertext *const *in, size_t count,
                     const double *coeffs, uint32_t degree, hd_ciphertext **out);
/* As hd_compare with the result at out_limbs limbs (hd_compare: 1).  A membership sum over S
 * slots of values near 1 at scale 2^45 must stay below q_0 / 2 ~ 2^59 (R29): either the client
 * scales the coefficients by 2^-k with 2^(45-k) S < 2^58 (k = 8 for 2^20 slots; the count
 * decodes / 2^k; bench.py's default) or the comparison keeps out_limbs = 2 (num_limbs = 7).
 * HD_E_LEVEL if the input has too few limbs for the degree at that output level. */
hd_status hd_compare_ex(hd_context *ctx, const hd_eval_keys *evk, const hd_ciphertext *const *in, size_t count,
                        const double *coeffs, uint32_t degree, uint32_t out_limbs, hd_ciphertext **out);
/* Rotation steps of the membership RotateAndSum: 1, 2, 4, ..., numSlots / 2. */
hd_status hd_membership_steps(const hd_context *ctx, int32_t *steps, size_t cap, size_t *count);
/* Membership (Alg. membership, Alg. gpu-bsgs-membership): the sum
 * of the count comparison ciphertexts (EvalAddMany), then RotateAndSum over numSlots with the
 * power-of-two keys (HD_E_MISSING_KEY if one is absent): every slot of *out holds the sum of
 * all slots of all inputs (the approximate match count).  Meaningful on the FLAT packing
 * (every slot a vector or zero padding, R29).  The total must stay below q_0 / 2 at the
 * inputs' level: scale the comparison coefficients by 2^-k or keep 2 limbs (hd_compare_ex).
 * *out: NULL -> allocated. */
hd_status hd_membership(hd_context *ctx, const hd_eval_keys *evk, const hd_ciphertext *const *in, size_t count,
                        hd_ciphertext **out);
/* EvalAddMany (Alg. membership): *out = sum of the count ciphertexts (same level and
 * scale).  With the database sharded over GPUs each rank sums its own comparison ciphertexts,
 * rank 0 gathers the partial sums and runs hd_membership on them (the RotateAndSum is linear).
 * *out: NULL -> allocated. */
hd_status hd_eval_add_many(hd_context *ctx, const hd_ciphertext *const *in, size_t count, hd_ciphertext **out);
/* Scale of a ciphertext's message (2^scale_bits for queries and scan outputs). */
hd_status hd_ciphertext_scale(const hd_ciphertext *ct, double *scale);
/* Decrypt + decode one ciphertext at its own scale: slots[0..numSlots) = real parts
 * (host double[cap], cap >= numSlots).  Floating point (CKKS error), not bit-exact. */
hd_status hd_decrypt_slots(hd_context *ctx, const hd_secret_key *sk, const hd_ciphertext *ct, double *slots,
                           size_t cap);

void hd_ciphertext_destroy(hd_ciphertext *ct);
void hd_eval_keys_destroy(hd_eval_keys *evk);
void hd_secret_key_destroy(hd_secret_key *sk);
void hd_database_destroy(hd_database *db);

/* ---- test-only stage entry points (host buffers, canonical layouts) --------- */
/* Batched NTT (inverse != 0: INTT) of n_rows rows of n u64, row r over modulus
 * index modulus_idx[r] (0..L).  data: host, in place. */
hd_status hd_test_ntt(hd_context *ctx, uint64_t *data, uint32_t n_rows,
                      const uint32_t *modulus_idx, int inverse);
/* Stage buffers left by the last hd_query on `db` (host copy):
 *   which 0: baby step r[index]            (ct, L limbs)
 *         1: giant sum S_{agg,j}           (ct, L limbs),   index = j; encrypted
 *            database: the 3 polynomials (d0, d1, d2) as accumulated (relinearised and
 *            rescaled in one step into stage 2)
 *         2: rescaled S'_{agg,j}           (ct, L-1 limbs), index = j
 *         3: y_agg = sum_j Rot(S'_j)       (ct, L-1 limbs)
 *         4: diagonal D[agg][k]            (pt, L limbs; encrypted: ct, L limbs), index = k
 * agg is the global aggregate index.  cap in u64 elements. */
hd_status hd_test_stage(const hd_database *db, int which, uint32_t agg, int32_t index,
                        uint64_t *host_dst, size_t cap);
/* Rotation of one ciphertext by `step` with the key in evk (test use): ModUp,
 * key inner product, ModDown (R11).  out is allocated. */
hd_status hd_test_rotate(hd_context *ctx, const hd_eval_keys *evk, const hd_ciphertext *ct,
                         int32_t step, hd_ciphertext **out);
hd_status hd_test_rescale(hd_context *ctx, const hd_ciphertext *ct, hd_ciphertext **out);
/* Fault injection (test use): XOR one u64 word of a database's diagonal D[agg][k] in device
 * memory with `mask` (word < L n, or 2 L n for encrypted diagonals).  XOR-ing again restores
 * it.  Lets the parity tests prove they detect a single flipped residue bit. */
hd_status hd_test_inject(hd_database *db, uint32_t agg, int32_t k, uint64_t word, uint64_t mask);

#ifdef __cplusplus
}
#endif
#endif /* HD_H */
