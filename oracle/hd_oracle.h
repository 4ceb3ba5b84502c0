/*
 * oracle/hd_oracle.h -- CPU ORACLE for the encrypted BSGS similarity scan of
 * arXiv 2604.00546 ("Lightweight, Practical Encrypted Face Recognition with GPU
 * Support").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load, call or link anything under
 * oracle/.  The product path (paper_2604_00546_b200/, include/hd.h) shares no
 * code, header, table or constant generator with this file and never calls it.
 *
 * Plain, slow, obviously-correct C: every modular product is
 * (unsigned __int128)a*b % m, every step follows the paper's algorithm (or the
 * plain definition of the operation) in the paper's order.  Citations:
 * "P:Lxxx" = /root/reference/PAPER.md line, "S:Lxxx" = SPEC.md line; readings
 * where the paper is silent are listed in DESIGN.md section 3 ("R#").
 *
 * Layouts (all arrays row-major, little-endian u64 residues in [0, m)):
 *   polynomial limb ..... n coefficients; NTT form = bit-reversed evaluation
 *                          order  a^[i] = sum_j a_j psi^{(2 br(i)+1) j}   (R13)
 *   plaintext (ell limbs) [limb][n]
 *   ciphertext (ell) .... [poly 0..1][limb][n]
 *   rotation key ........ [digit d < beta(L)][poly (0=b,1=a)][modulus l < L+K][n]
 *                          modulus indices L..L+K-1 are the special primes p_k.
 *   modup digits (ell) .. [digit d < beta(ell)][ext modulus e < ell+K][n]
 *                          ext index e < ell is q_e, e >= ell is p_{e-ell}.
 *   (alpha = K = 1, the north-star profile: beta(ell) = ell digits, one special prime P.)
 *
 * Every function returns 0 on success or a negative error code:
 */
#ifndef HD_ORACLE_H
#define HD_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define OR_OK 0
#define OR_E_ARG (-1)
#define OR_E_PARAMS (-2)
#define OR_E_LAYOUT (-3)
#define OR_E_ZERO_VECTOR (-4)
#define OR_E_MISSING_KEY (-5)
#define OR_E_RANGE (-6)

#define OR_MAXMOD 20

typedef struct {
  int32_t log_n;      /* ring degree n = 2^log_n                         */
  int32_t n;
  int32_t num_slots;  /* n/2  ("packs N/2 complex values")    */
  int32_t L;          /* ciphertext limbs q_0..q_{L-1} at the MAC (R5)   */
  int32_t q0_bits;    /* 60                                              */
  int32_t scale_bits; /* 45  ("scaling factor is set to 45")     */
  int32_t special_bits; /* 60 */
  int32_t K_sp;       /* special primes p_0..p_{K-1} (P = their product)  */
  int32_t alpha;      /* limbs per key-switching digit (R11, R31)        */
  int32_t pad_;
  uint64_t mod[OR_MAXMOD]; /* mod[0..L-1] = q_i, mod[L..L+K-1] = p_k     */
  uint64_t psi[OR_MAXMOD]; /* smallest primitive 2n-th root of unity      */
  uint64_t seed;           /* Philox key for the secret / rotation keys   */
} or_params;

int or_params_init(or_params *p, int32_t log_n, int32_t L, uint64_t seed);
/* General hybrid key-switching profile (R31; SURVEY 8(d) "paper-depth": L = 12, alpha = 4,
 * K_sp = 4): K_sp special primes (the next NTT primes below q0, descending) and alpha
 * limbs per digit.  or_params_init = or_params_init_ex(.., K_sp = 1, alpha = 1, ..). */
int or_params_init_ex(or_params *p, int32_t log_n, int32_t L, int32_t K_sp, int32_t alpha, uint64_t seed);
/* beta(ell) = ceil(ell / alpha) digits of a ciphertext at ell limbs; digit d holds limbs
 * [d alpha, min((d+1) alpha, ell)). */
int32_t or_num_digits(const or_params *p, int32_t ell);
int or_is_prime(uint64_t x);

/* NTT over modulus index l (0..L); fast (textbook CT / GS) and definitional. */
int or_ntt_forward(const or_params *p, int32_t l, uint64_t *a);
int or_ntt_inverse(const or_params *p, int32_t l, uint64_t *a);
int or_ntt_definition(const or_params *p, int32_t l, const uint64_t *a, uint64_t *out);
int or_negacyclic_schoolbook(const uint64_t *a, const uint64_t *b, int32_t n, uint64_t m,
                             uint64_t *out);

/* Philox4x32-10 (Random123) and the pinned draws (R14). */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* Galois machinery (R7): g = 5^r mod 2n; NTT-domain index permutation. */
uint64_t or_galois_elt(const or_params *p, int64_t step);
int or_automorph_coeff(const or_params *p, uint64_t g, const int64_t *a, int64_t *out);
int or_automorph_ntt(const or_params *p, uint64_t g, const uint64_t *a, uint64_t *out);

/* CKKS encode / decode (R15) over `nlimbs` leading q moduli. */
int or_encode(const or_params *p, const double *z, double delta, int32_t nlimbs, uint64_t *pt);
int or_encode_coeffs(const or_params *p, const double *z, double delta, int64_t *coef);
int or_decode(const or_params *p, const uint64_t *pt, int32_t nlimbs, double delta, double *z);

/* Keys and encryption (R11, R14). */
int or_secret_key(const or_params *p, int64_t *s_coeff, uint64_t *s_ntt /* (L+K) x n */);
int or_rotation_key(const or_params *p, const uint64_t *s_ntt, int64_t step, uint64_t *key);
int or_encrypt(const or_params *p, const uint64_t *s_ntt, const uint64_t *pt, int32_t nlimbs,
               uint64_t enc_seed, uint64_t *ct);
int or_decrypt(const or_params *p, const uint64_t *s_ntt, const uint64_t *ct, int32_t nlimbs,
               uint64_t *pt);

/* Encrypted-database mode (NEXT-1, R26): public key [2][L][n] (b, a); public-key
 * encryption with object id obj; relinearisation key (layout of a rotation key). */
int or_public_key(const or_params *p, const uint64_t *s_ntt, uint64_t *pk);
int or_encrypt_pk(const or_params *p, const uint64_t *pk, const uint64_t *pt, int32_t nlimbs,
                  uint64_t enc_seed, uint32_t obj, uint64_t *ct);
int or_relin_key(const or_params *p, const uint64_t *s_ntt, uint64_t *key);

/* Key switching pieces (R11, R12, R31) at ciphertext level `ell` (limbs q_0..q_{ell-1}). */
int or_modup(const or_params *p, const uint64_t *c1, int32_t ell, uint64_t *dig);
/* Fast basis conversion with centred digits (R31): x [cnt][n] coefficient-form residues of
 * one integer per coefficient modulo mod[bidx[i]] -> out[n] modulo mod[mi]. */
int or_basis_convert(const or_params *p, const uint64_t *x, const int32_t *bidx, int32_t cnt, int32_t mi,
                     uint64_t *out);
/* ModDown of one polynomial u [(ell+K)][n] (NTT form over Q_ell u P) -> out [ell][n]. */
int or_moddown(const or_params *p, const uint64_t *u, int32_t ell, uint64_t *out);
int or_rotate_hoisted(const or_params *p, const uint64_t *ct, const uint64_t *dig, int32_t ell,
                      const uint64_t *key, int64_t step, uint64_t *out);
int or_rotate(const or_params *p, const uint64_t *ct, int32_t ell, const uint64_t *key,
              int64_t step, uint64_t *out);
int or_rescale(const or_params *p, const uint64_t *ct, int32_t ell, uint64_t *out);
/* (d0, d1, d2) [3][ell][n] -> (d0, d1) + KeySwitch_{s^2->s}(d2) [2][ell][n]. */
int or_relinearize(const or_params *p, const uint64_t *S3, int32_t ell, const uint64_t *rlk, uint64_t *out);

/* Enrollment (Alg. enroller_bsgs) and query slot layout (R8). */
int or_normalize(const float *v, int32_t dim, double *u);
int or_query_slots(const or_params *p, const float *q, int32_t dim, double *z);
int or_normalize_rows(const float *vecs, int64_t rows, int32_t dim, double *U);
int or_enroll_slots(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                    int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg, int32_t k,
                    double *z);
int or_enroll_aggregate(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                        int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg,
                        uint64_t *Dagg /* N x pt(L) */);

int or_enroll_aggregate_encrypted(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                                  int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg,
                                  const uint64_t *pk, uint64_t enc_seed, uint64_t *Dct /* N x ct(L) */);

/* Scan layout helpers (R6) */
int or_giant_range(int32_t N, int32_t n1, int32_t *j_min, int32_t *j_max);
int32_t or_pre_rot(int32_t N, int32_t n1, int32_t j);
int or_rotation_steps(const or_params *p, int32_t N, int32_t n1, int32_t *steps, int32_t cap,
                      int32_t *count);

/* Scan (Alg. sender-bsgs; fold reading R2). */
int or_baby_steps(const or_params *p, const uint64_t *q_ct, int32_t n1, const int32_t *steps,
                  int32_t nkeys, const uint64_t *keys, uint64_t *r /* n1 x ct(L) */);
int or_giant_sum(const or_params *p, const uint64_t *r, int32_t n1, int32_t N,
                 const uint64_t *Dagg /* N x pt(L) */, int32_t j, uint64_t *S /* ct(L) */);
int or_scan_aggregate(const or_params *p, const uint64_t *r, int32_t n1, int32_t N,
                      const uint64_t *Dagg, const int32_t *steps, int32_t nkeys,
                      const uint64_t *keys, uint64_t *out /* ct(L-1) */,
                      uint64_t *y_out /* optional ct(L-1): sum before the fold */);
/* Same result with the giant-step sum accumulated in Q u {P} and one ModDown (R23,
 * P:L498-506); bits differ from or_scan_aggregate only by that ModDown's rounding.
 * This is the schedule the CUDA path implements. */
int or_scan_aggregate_hoisted(const or_params *p, const uint64_t *r, int32_t n1, int32_t N,
                              const uint64_t *Dagg, const int32_t *steps, int32_t nkeys,
                              const uint64_t *keys, uint64_t *out, uint64_t *y_out);

/* Encrypted diagonals (NEXT-1): degree-2 giant-step sum [3][L][n], and the scan with
 * Relinearize before the rescale, then the R23 schedule. */
int or_giant_sum_ct(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dct,
                    int32_t j, uint64_t *S /* [3][L][n] */);
int or_scan_aggregate_ct(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dct,
                         const uint64_t *rlk, const int32_t *steps, int32_t nkeys, const uint64_t *keys,
                         uint64_t *out, uint64_t *y_out);

/* Flat pre-rotated layout (NEXT-2, R27; BSGS-RTX-TBE). */
int or_enroll_slots_flat(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                         int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg, int32_t k, double *z);
int or_enroll_aggregate_flat(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                             int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg, uint64_t *Dagg);
int or_rotation_steps_flat(const or_params *p, int32_t N, int32_t n1, int32_t *steps, int32_t cap,
                           int32_t *count);
int or_giant_sum_flat(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dagg,
                      int32_t j, uint64_t *S);
int or_scan_aggregate_flat(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dagg,
                           const int32_t *steps, int32_t nkeys, const uint64_t *keys, uint64_t *out);
int or_enroll_aggregate_flat_encrypted(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                                       int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg,
                                       const uint64_t *pk, uint64_t enc_seed, uint64_t *Dct);
/* BSGS-RTX-TBS: plain flat diagonals encrypted by the enroller, pre-rotated by
 * the server with the negative giant-step keys numSlots - j n1 (in place, eager ModDown). */
int or_enroll_aggregate_flat_tbs(const or_params *p, const double *U, int64_t u_first, int64_t u_count,
                                 int64_t num_vectors, int32_t dim, int32_t n1, int64_t agg, const uint64_t *pk,
                                 uint64_t enc_seed, uint64_t *Dct);
int or_prerotate_tbs(const or_params *p, uint64_t *Dct, int32_t dim, int32_t n1, const int32_t *steps,
                     int32_t nkeys, const uint64_t *keys);
int or_giant_sum_ct_flat(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dct,
                         int32_t j, uint64_t *S);
int or_scan_aggregate_flat_ct(const or_params *p, const uint64_t *r, int32_t n1, int32_t N, const uint64_t *Dct,
                              const uint64_t *rlk, const int32_t *steps, int32_t nkeys, const uint64_t *keys,
                              uint64_t *out);
int or_decrypt_scores_flat(const or_params *p, const uint64_t *s_ntt, const uint64_t *out_ct, int32_t N,
                           int64_t agg, int64_t num_vectors, double *scores);

/* Decrypt + decode one output ciphertext and read the scores of its vectors (R4). */
int or_decrypt_scores(const or_params *p, const uint64_t *s_ntt, const uint64_t *out_ct,
                      int32_t N, int64_t agg, int64_t num_vectors, double *scores /* M/2*N */);

/* Encrypted comparison and scenario tail (NEXT-3, R29; Alg. gpu-chebyshev P:L734-789,
 * Alg. membership). */
int32_t or_cheb_degree(int32_t kappa);
int or_ps_split(int32_t n, int32_t *d1, int32_t *d2);
int or_cheb_coeffs(double delta, int32_t n, double *c /* n + 1 */);
int or_cheb_compare(const or_params *p, const uint64_t *in, int32_t ell, double scale, const double *c,
                    int32_t degree, const uint64_t *rlk, uint64_t *out, int32_t *ell_out, double *scale_out);
int or_cheb_compare_at(const or_params *p, const uint64_t *in, int32_t ell, double scale, const double *c,
                       int32_t degree, const uint64_t *rlk, int32_t need, uint64_t *out, int32_t *ell_out,
                       double *scale_out);
/* Relinearize + Rescale with one rounding by P q_{ell-1}: S3 [3][ell][n] -> out [2][ell-1][n]. */
int or_relin_rescale(const or_params *p, const uint64_t *S3, int32_t ell, const uint64_t *rlk, uint64_t *out);
int or_aggregate_diagonals(const or_params *p, const uint64_t *D, int32_t A, int32_t N, int32_t dpoly, uint64_t *out);
int or_membership(const or_params *p, const uint64_t *cts, int32_t count, int32_t ell, const int32_t *steps,
                  int32_t nkeys, const uint64_t *keys, uint64_t *out);

#ifdef __cplusplus
}
#endif
#endif
