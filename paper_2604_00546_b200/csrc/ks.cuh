// ks.cuh -- host drivers of the key-switching / rescale / MAC / encode kernels.
#pragma once
#include "common.cuh"

// ModUp (R11) of B c1 polynomials at ell limbs (c1 of ciphertext b at c1 + b*c1_stride).
// dig: [B][ell][ell][n] (lifted digits; slot layout: see ks.cu).  tmp: B*ell*n scratch.
hd_status ks_modup(hd_context *c, const uint64_t *c1, size_t c1_stride, uint32_t B, int ell, uint64_t *dig,
                   uint64_t *tmp);
// Key inner product for X = B*K (b, k) pairs -> u [X][2][ell+1][n].
// (the own-modulus digit of c1 is read from c1 itself: c1 of ciphertext b at c1 + b*c1_stride)
hd_status ks_kip(hd_context *c, const uint64_t *dig, const uint64_t *c1, size_t c1_stride, uint32_t B, uint32_t K,
                 int ell, const uint64_t *const *kptr_dev, const uint32_t *gal_dev, uint64_t *u);
// Extended-basis giant-step accumulation (R23), B ciphertexts ct_b = ct + b*ct_stride
// ([2][ell][n]), one key, u [B][2][ell+1][n] accumulated:
//   u_b += KIP(pi_g(dig_b)) + (P pi_g(ct_b.c0), 0)   (a rotation before its ModDown)
hd_status ks_kip_accumulate(hd_context *c, const uint64_t *dig, const uint64_t *ct, size_t ct_stride, uint32_t B,
                            int ell, const uint64_t *const *kptr_dev, const uint32_t *gal_dev, uint64_t *u);
// The hoisted giant-step sum of R23 in one pass (alpha = K = 1): u_b = sum_j (KIP_j + (P pi_j(c0_j), 0))
// + P T0_b over J rotated steps (digits dig[j], sums ct[j] + b ct_stride, key slot[j]) and the
// unrotated sum T0 (may be null); u [B][2][ell+1][n] is written, not accumulated.
hd_status ks_giant_sum(hd_context *c, uint32_t B, int ell, int J, const uint64_t *const *dig, const uint64_t *const *ct,
                       const int *slot, const uint64_t *t0, size_t ct_stride, const uint64_t *const *kptr_dev,
                       const uint32_t *gal_dev, uint64_t *u);
//   u_b += (P ct_b, with P limb 0)                    (a giant step without rotation)
hd_status ks_add_pscaled(hd_context *c, uint64_t *u, const uint64_t *ct, size_t ct_stride, uint32_t B, int ell);
// ModDown of u [X][2][ell+1][n] (P limb INTT'd in place) -> dst_x (+ pi_{g_k}(c0_b)).
hd_status ks_moddown(hd_context *c, uint64_t *u, uint32_t X, uint32_t K, int ell, const uint32_t *gal_dev,
                     const uint64_t *c0, size_t c0_stride, uint64_t *dst, size_t dst_stride, bool accumulate,
                     uint64_t *tmp);
// Rescale B ciphertexts at ell limbs (S_b at S + b*s_stride) -> out_b (ell-1 limbs).
hd_status ks_rescale(hd_context *c, const uint64_t *S, size_t s_stride, uint32_t B, int ell, uint64_t *out,
                     size_t out_stride, uint64_t *tmp1, uint64_t *tmp2);

// Relinearise + rescale with one rounding by P q_{ell-1} (bit-identical to ks_moddown-accumulate
// then ks_rescale: mixed-radix identity, R29): S3 [B][3][ell][n] -> out [B][2][ell-1][n].
// Scratch: dig B ell ell n, u B 2 (ell+1) n, tmp B ell n, V B 2 (ell-1) n.
hd_status ks_relin_rescale(hd_context *c, uint64_t *S3, uint32_t B, int ell, const uint64_t *const *rlk_dev,
                           const uint32_t *gal_dev, uint64_t *out, uint64_t *dig, uint64_t *u, uint64_t *tmp,
                           uint64_t *V);

// MAC (mac.cu)
struct MacPlan {
  int n1, N, L, logn;
  int jmin, nj;        // valid giant steps j = js[0..nj)
  const int32_t *js;   // host
};
// Encrypted diagonals (NEXT-1): degree-2 sums S3 [a][j][3][L][n] of Dct [a][k][2][L][n].
hd_status mac_ct_run(hd_context *c, const uint64_t *Dct, const uint64_t *r, uint64_t *S3, uint32_t A_loc, int n1,
                     int N, const std::vector<int32_t> &js, bool flat, const DPack &dp);
// flat: the giant-step ranges of the flat packing (R27)
// dp: packed diagonals (R34; only the TMA MAC reads them)
hd_status mac_run(hd_context *c, const uint64_t *D, const uint64_t *r, uint64_t *S, uint32_t A_loc, int n1, int N,
                  const std::vector<int32_t> &js, bool flat, const DPack &dp);

// Warp-specialised TMA pipeline for full giant-step ranges (mac_tma.cu); Q <= 4 queries per
// diagonal pass; r [Q][n1][2][L][n], S [Q][A][nj][2][L][n].  HD_MAC_VARIANT=c selects mac.cu.
bool mac_tma_supported(const hd_context *c, int n1, int N, bool flat, uint32_t Q);
// the degree-2 MAC of encrypted diagonals (NEXT-1) on the same pipeline: S3 [A][nj][3][L][n]
hd_status mac_tma_ct_run(hd_context *c, const uint64_t *D, const uint64_t *r, uint64_t *S3, uint32_t A, int n1, int N,
                         const std::vector<int32_t> &js, bool flat, const DPack &dp);
bool mac_tma_ct_supported(const hd_context *c, int n1, int N, bool flat);
hd_status mac_tma_run(hd_context *c, const uint64_t *D, const uint64_t *r, uint64_t *S, uint32_t A, int n1, int N,
                      const std::vector<int32_t> &js, uint32_t Q, bool flat, const DPack &dp);

// Query batching (NEXT-4): Q queries per D pass; r [Q][n1][2][L][n], S [Q][A][nj][2][L][n].
hd_status mac_batch_run(hd_context *c, const uint64_t *D, const uint64_t *r, uint64_t *S, uint32_t A_loc, int n1,
                        int N, const std::vector<int32_t> &js, bool flat, uint32_t Q, const DPack &dp);

// Public-key encryption of count ciphertexts in place (c0 of ct_x = ct + x*ct_stride holds
// the plaintext on entry); object ids obj0 + x; V, E0: count*L*n scratch each (client.cu).
hd_status pk_encrypt_rows(hd_context *c, const hd_public_key *pk, uint64_t *ct, size_t ct_stride, uint32_t count,
                          uint64_t enc_seed, uint32_t obj0, uint64_t *V, uint64_t *E0);

// encode (enroll.cu)
hd_status encode_batch(hd_context *c, double *re, double *im, uint32_t B, double delta, int nlimbs,
                       uint64_t *out, size_t out_stride);
hd_status alloc_ct(hd_context *c, uint32_t limbs, hd_ciphertext **out);
