// mac_tma.cu -- the fused diagonal x ciphertext MAC (a5, Alg. sender-bsgs Step 2b)
// as a warp-specialised TMA pipeline.
//
//   S[b][a][j][p][m][t] = sum_{i < n1} r[b][i][p][m][t] * D[a][k(j,i)][m][t]  mod q_m,
//   k(j,i) = (j n1 + i) mod N   (replicated: preshifted giant steps; flat: j n1 + i < N)
//
// for full giant-step ranges (n1 | N/2 replicated, n1 | N flat), q_m < 2^60, b < QB queries.
//
// Design.  Giant step j reads the diagonal block G(j) = k(j,0) / n1 of
// n1 consecutive diagonals, so D of one aggregate is a 5-D tensor (coefficient, limb, diagonal
// within a block, block, aggregate).  A producer warp streams, per pipeline stage, ONE TMA box
// of 128 coefficients x 1 limb x SPS baby steps x JT blocks x AG aggregates (evict-first; for
// a packed 45-bit limb, R34, a u32 box and a u16 box with the same coordinates) plus one box
// of the baby-step rows r (L2-resident, evict-last) into a ring of shared-memory stages.
// Consumer threads own one coefficient of one aggregate and all JT giant steps of their unit,
// so each r word read from shared memory serves JT diagonal words and each diagonal word
// costs one or two LDS and two Karatsuba 64x64 products (R35; no address arithmetic, no
// register staging of loads in flight).
//
// Work unit = (AG aggregates, JT consecutive blocks, 128-coefficient tile, limb); one
// persistent CTA per SM walks units u = blockIdx.x, + gridDim.x, ... with the aggregate
// group fastest (concurrently resident CTAs share few r tiles: L2 reuse) and the limb next
// (they mix the u64 and packed limbs' streams).
#include "common.cuh"
#include "ks.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <type_traits>

namespace {
constexpr int TC = 128;  // coefficients per aggregate per unit (one per consumer thread)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3, int c4,
                                            uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar)),
      "l"(policy)
      : "memory");
}

struct Unit {
  uint32_t a0;       // first aggregate of the group
  int gg0, tile, m;  // first diagonal block, coefficient tile, limb
};
__device__ __forceinline__ Unit decode(uint32_t u, uint32_t nag, int ngrp, int tiles, int AG, int JT, int L = 0) {
  Unit x;
  x.a0 = (u % nag) * AG;
  u /= nag;
  if (L) {  // limb second-fastest (A/B order: concurrent CTAs mix wide and packed limbs)
    x.m = (int)(u % (uint32_t)L);
    u /= (uint32_t)L;
    x.gg0 = (int)(u % ngrp) * JT;
    x.tile = (int)(u / ngrp);
    return x;
  }
  x.gg0 = (int)(u % ngrp) * JT;
  u /= ngrp;
  x.tile = (int)(u % tiles);
  x.m = (int)(u / tiles);
  return x;
}

// AG aggregates x TC coefficients consumer threads + one producer warp.
// Stage layout (u64): D[AG][JT][SPS][TC] (the 5-D box), then r[QB][SPS][2][TC].
// flags (measurement only): 1 = stream without arithmetic, 2 = arithmetic without the stream.
// Limb classes of packed diagonals (R34): cls 1 = narrow (u32 low + u16 high planes, maps tmLo /
// tmHi), 0 = wide (u64, map tmD); idx = the limb's coordinate in its map.
struct PackCls {
  uint8_t cls[HD_MAXMOD], idx[HD_MAXMOD];
};

template <int AG, int JT, int QB, int SPS, bool FLUSH>
__global__ void __launch_bounds__(AG *TC + 32, 1)
    mac_tma_kernel(const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmLo,
                   const __grid_constant__ CUtensorMap tmHi, const __grid_constant__ CUtensorMap tmR,
                   uint64_t *__restrict__ S, int n1, int N, int L, int logn, int nj, uint32_t A, int flat, int stages,
                   int qrows, size_t s_query_stride, ModTab mt, int flags, PackCls pk) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int D_WORDS = AG * JT * SPS * TC, R_WORDS = QB * SPS * 2 * TC;
  constexpr uint32_t STAGE_BYTES = (D_WORDS + R_WORDS) * 8;
  constexpr uint32_t NARROW_STAGE_BYTES = D_WORDS * 6 + R_WORDS * 8;  // packed limb (R34)
  constexpr int CONSUMERS = AG * TC;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)stages * STAGE_BYTES);
  uint64_t *empty = full + stages;
  const int n = 1 << logn, tiles = n / TC, G = N / n1, ngrp = G / JT, nsb = n1 / SPS;
  const uint32_t nag = A / AG, units = nag * (uint32_t)ngrp * (uint32_t)tiles * (uint32_t)L;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMERS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (threadIdx.x >= CONSUMERS) {  // ---------------- producer warp ----------------
    if (threadIdx.x != CONSUMERS || (flags & 2)) return;
    uint64_t pol_stream, pol_keep;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    int stage = 0;
    uint32_t phase = 0;
    for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
      const Unit x = decode(u, nag, ngrp, tiles, AG, JT, (flags & 4) ? L : 0);
      const bool narrow = pk.cls[x.m];
      const int mi = pk.idx[x.m];
      for (int sb = 0; sb < nsb; sb++) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint64_t *base = reinterpret_cast<uint64_t *>(smem + (size_t)stage * STAGE_BYTES);
        if (!narrow) {
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_5d(base, &tmD, x.tile * TC, mi, sb * SPS, x.gg0, (int)x.a0, &full[stage], pol_stream);
        } else {  // low plane (4 B per word) then high plane (2 B) in the stage's diagonal area
          mbar_arrive_expect_tx(&full[stage], NARROW_STAGE_BYTES);
          tma_load_5d(base, &tmLo, x.tile * TC, mi, sb * SPS, x.gg0, (int)x.a0, &full[stage], pol_stream);
          tma_load_5d(reinterpret_cast<unsigned char *>(base) + 4 * D_WORDS, &tmHi, x.tile * TC, mi, sb * SPS, x.gg0,
                      (int)x.a0, &full[stage], pol_stream);
        }
#pragma unroll
        for (int b = 0; b < QB; b++)
          tma_load_3d(base + D_WORDS + b * SPS * 2 * TC, &tmR, x.tile * TC, x.m, b * qrows + sb * SPS * 2,
                      &full[stage], pol_keep);
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }

  // ---------------- consumers: thread = (aggregate g of the group, coefficient t) ----------------
  const int g = threadIdx.x / TC, t = threadIdx.x % TC;
  int stage = 0;
  uint32_t phase = 0;
  for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
    const Unit x = decode(u, nag, ngrp, tiles, AG, JT, (flags & 4) ? L : 0);
    const bool narrow = pk.cls[x.m];
    const uint64_t q = mt.q[x.m], bar = mt.bar[x.m], r64 = mt.r64[x.m], r64s = mt.r64s[x.m];
    KAcc acc[QB][JT][2];
    uint64_t part[QB][JT][2];
#pragma unroll
    for (int b = 0; b < QB; b++)
#pragma unroll
      for (int jj = 0; jj < JT; jj++) {
        acc[b][jj][0] = acc[b][jj][1] = KAcc{0, 0, 0, 0, 0, 0};
        part[b][jj][0] = part[b][jj][1] = 0;
      }
    for (int sb = 0; sb < nsb; sb++) {
      if (!(flags & 2)) mbar_wait(&full[stage], phase);
      if (!(flags & 1)) {
        const unsigned char *sbase = smem + (size_t)stage * STAGE_BYTES;
        const uint64_t *Rs = reinterpret_cast<const uint64_t *>(sbase) + D_WORDS + t;
        // one stage: the 31-bit halves of every diagonal word and of its baby step's two r
        // words, three Karatsuba products per (word, r word)
        auto consume = [&](auto narrow_tag) {
          constexpr bool NARROW = decltype(narrow_tag)::value;
          const uint64_t *Ds = reinterpret_cast<const uint64_t *>(sbase) + g * JT * SPS * TC + t;
          const uint32_t *Dl = reinterpret_cast<const uint32_t *>(sbase) + g * JT * SPS * TC + t;
          const uint16_t *Dh = reinterpret_cast<const uint16_t *>(sbase + 4 * D_WORDS) + g * JT * SPS * TC + t;
#pragma unroll
          for (int s = 0; s < SPS; s++) {
            uint32_t dl[JT], dh[JT], ds[JT];
#pragma unroll
            for (int jj = 0; jj < JT; jj++) {
              if (NARROW) {  // stored split at bit 31 (R34)
                dl[jj] = Dl[(jj * SPS + s) * TC];
                dh[jj] = Dh[(jj * SPS + s) * TC];
              } else {
                const uint64_t d = Ds[(jj * SPS + s) * TC];
                dl[jj] = (uint32_t)d & 0x7fffffffu;
                dh[jj] = (uint32_t)(d >> 31);
              }
              ds[jj] = dl[jj] + dh[jj];
            }
#pragma unroll
            for (int b = 0; b < QB; b++) {
#pragma unroll
              for (int p = 0; p < 2; p++) {
                const uint64_t r = Rs[(b * SPS * 2 + 2 * s + p) * TC];
                const uint32_t rl = (uint32_t)r & 0x7fffffffu, rh = (uint32_t)(r >> 31), rs = rl + rh;
#pragma unroll
                for (int jj = 0; jj < JT; jj++) kmac<NARROW>(acc[b][jj][p], rl, rh, rs, dl[jj], dh[jj], ds[jj]);
              }
            }
          }
        };
        if (narrow)
          consume(std::true_type{});
        else
          consume(std::false_type{});
      }
      // one arrival per warp once every lane's shared-memory reads of the stage are done
      __syncwarp();
      if (!(flags & 2) && (threadIdx.x & 31) == 0) mbar_arrive(&empty[stage]);
      if (++stage == stages) {
        stage = 0;
        phase ^= 1;
      }
      if (FLUSH && (sb % (128 / SPS)) == (128 / SPS) - 1) {  // n1 > 128: bank every 128 terms
#pragma unroll
        for (int b = 0; b < QB; b++)
#pragma unroll
          for (int jj = 0; jj < JT; jj++)
#pragma unroll
            for (int p = 0; p < 2; p++) {
              part[b][jj][p] = addmod(part[b][jj][p], kacc_reduce(acc[b][jj][p], q, bar, r64, r64s), q);
              acc[b][jj][p] = KAcc{0, 0, 0, 0, 0, 0};
            }
      }
    }
    const size_t ls = (size_t)L * n;
    const uint32_t a = x.a0 + g;
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      // diagonal block gg holds giant step j with (j n1) mod N = gg n1: flat j = gg;
      // replicated j = gg for gg n1 < N/2, else gg - N/n1; S slot j - jmin
      const int gg = x.gg0 + jj;
      const int jslot = flat ? gg : (gg < G / 2 ? gg + G / 2 : gg - G / 2);
#pragma unroll
      for (int b = 0; b < QB; b++) {
        uint64_t *Sa = S + b * s_query_stride + ((size_t)a * nj + jslot) * 2 * ls + (size_t)x.m * n +
                       (size_t)x.tile * TC + t;
#pragma unroll
        for (int p = 0; p < 2; p++)
          Sa[(size_t)p * ls] = addmod(part[b][jj][p], kacc_reduce(acc[b][jj][p], q, bar, r64, r64s), q);
      }
    }
  }
}

// ---- encrypted diagonals (NEXT-1, R26): the degree-2 MAC over the same pipeline ----------
// D [a][k][poly][L][n]: per limb m a 5-D map (coefficient, poly, diagonal within a block, block,
// aggregate) based at limb m; one box per stage = TC x 2 polys x SPS x JT x AG.  Per stage word
// pair (D0, D1) and baby step: d0 += r0 D0, d1 += r0 D1 + r1 D0, d2 += r1 D1,
// Karatsuba sums (R35), all banked every 64 steps (d1 takes 2 products
// per step: 128 products < 2^127).  S3 [a][j][3][L][n].
constexpr int CT_MAXL = 8;
struct CtMaps {  // per limb: the u64 map (wide) or the u32 low-plane map (narrow, R34) + its u16 map
  CUtensorMap m[CT_MAXL], hi[CT_MAXL];
  uint8_t narrow[CT_MAXL];
};
template <int AG, int JT, int SPS>
__global__ void __launch_bounds__(AG *TC + 32, 1)
    mac_tma_ct_kernel(const __grid_constant__ CtMaps tmD, const __grid_constant__ CUtensorMap tmR,
                      uint64_t *__restrict__ S, int n1, int N, int L, int logn, int nj, uint32_t A, int flat,
                      int stages, ModTab mt, uint32_t small_mask, int flags) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int D_WORDS = AG * JT * SPS * 2 * TC, R_WORDS = SPS * 2 * TC;
  constexpr uint32_t STAGE_BYTES = (D_WORDS + R_WORDS) * 8;
  constexpr int CONSUMERS = AG * TC;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)stages * STAGE_BYTES);
  uint64_t *empty = full + stages;
  const int n = 1 << logn, tiles = n / TC, G = N / n1, ngrp = G / JT, nsb = n1 / SPS;
  const uint32_t nag = A / AG, units = nag * (uint32_t)ngrp * (uint32_t)tiles * (uint32_t)L;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMERS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= CONSUMERS) {  // ---------------- producer warp ----------------
    if (threadIdx.x != CONSUMERS || (flags & 2)) return;
    uint64_t pol_stream, pol_keep;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_stream));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
    int stage = 0;
    uint32_t phase = 0;
    for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
      const Unit x = decode(u, nag, ngrp, tiles, AG, JT, (flags & 4) ? L : 0);
      for (int sb = 0; sb < nsb; sb++) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint64_t *base = reinterpret_cast<uint64_t *>(smem + (size_t)stage * STAGE_BYTES);
        if (!tmD.narrow[x.m]) {
          mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_5d(base, &tmD.m[x.m], x.tile * TC, 0, sb * SPS, x.gg0, (int)x.a0, &full[stage], pol_stream);
        } else {  // packed limb: low plane (4 B per word) then high plane (2 B)
          mbar_arrive_expect_tx(&full[stage], D_WORDS * 6 + R_WORDS * 8);
          tma_load_5d(base, &tmD.m[x.m], x.tile * TC, 0, sb * SPS, x.gg0, (int)x.a0, &full[stage], pol_stream);
          tma_load_5d(reinterpret_cast<unsigned char *>(base) + 4 * D_WORDS, &tmD.hi[x.m], x.tile * TC, 0, sb * SPS,
                      x.gg0, (int)x.a0, &full[stage], pol_stream);
        }
        tma_load_3d(base + D_WORDS, &tmR, x.tile * TC, x.m, sb * SPS * 2, &full[stage], pol_keep);
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  const int g = threadIdx.x / TC, t = threadIdx.x % TC;
  int stage = 0;
  uint32_t phase = 0;
  for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
    const Unit x = decode(u, nag, ngrp, tiles, AG, JT, (flags & 4) ? L : 0);
    const uint64_t q = mt.q[x.m], bar = mt.bar[x.m], r64 = mt.r64[x.m], r64s = mt.r64s[x.m];
    // Karatsuba sums (R35); limbs below 2^47 take the narrow form (r_h d_h < 2^32)
    const bool small = (small_mask >> x.m) & 1u;
    KAcc acc[JT][3];
    uint64_t part[JT][3];
#pragma unroll
    for (int jj = 0; jj < JT; jj++)
#pragma unroll
      for (int e = 0; e < 3; e++) {
        acc[jj][e] = KAcc{0, 0, 0, 0, 0, 0};
        part[jj][e] = 0;
      }
    for (int sb = 0; sb < nsb; sb++) {
      if (!(flags & 2)) mbar_wait(&full[stage], phase);
      // box order [AG][JT][SPS][2][TC]
      const unsigned char *sbase = smem + (size_t)stage * STAGE_BYTES;
      const uint64_t *Ds = reinterpret_cast<const uint64_t *>(sbase) + g * JT * SPS * 2 * TC + t;
      const uint32_t *Dl = reinterpret_cast<const uint32_t *>(sbase) + g * JT * SPS * 2 * TC + t;
      const uint16_t *Dh = reinterpret_cast<const uint16_t *>(sbase + 4 * D_WORDS) + g * JT * SPS * 2 * TC + t;
      const uint64_t *Rs = reinterpret_cast<const uint64_t *>(sbase) + D_WORDS + t;
      auto consume = [&](auto small_tag, auto packed_tag) {
        constexpr bool SMALL = decltype(small_tag)::value, PACKED = decltype(packed_tag)::value;
#pragma unroll
        for (int s = 0; s < SPS; s++) {
          const uint64_t r0 = Rs[(2 * s) * TC], r1 = Rs[(2 * s + 1) * TC];
          const uint32_t r0l = (uint32_t)r0 & 0x7fffffffu, r0h = (uint32_t)(r0 >> 31), r0s = r0l + r0h;
          const uint32_t r1l = (uint32_t)r1 & 0x7fffffffu, r1h = (uint32_t)(r1 >> 31), r1s = r1l + r1h;
#pragma unroll
          for (int jj = 0; jj < JT; jj++) {
            uint32_t a0l, a0h, a1l, a1h;
            const int w0 = ((jj * SPS + s) * 2 + 0) * TC, w1 = w0 + TC;
            if (PACKED) {  // stored split at bit 31 (R34)
              a0l = Dl[w0];
              a0h = Dh[w0];
              a1l = Dl[w1];
              a1h = Dh[w1];
            } else {
              const uint64_t d0 = Ds[w0], d1 = Ds[w1];
              a0l = (uint32_t)d0 & 0x7fffffffu;
              a0h = (uint32_t)(d0 >> 31);
              a1l = (uint32_t)d1 & 0x7fffffffu;
              a1h = (uint32_t)(d1 >> 31);
            }
            const uint32_t a0s = a0l + a0h, a1s = a1l + a1h;
            kmac<SMALL>(acc[jj][0], r0l, r0h, r0s, a0l, a0h, a0s);  // d0 += r0 D0
            kmac<SMALL>(acc[jj][1], r0l, r0h, r0s, a1l, a1h, a1s);  // d1 += r0 D1 + r1 D0
            kmac<SMALL>(acc[jj][1], r1l, r1h, r1s, a0l, a0h, a0s);
            kmac<SMALL>(acc[jj][2], r1l, r1h, r1s, a1l, a1h, a1s);  // d2 += r1 D1
          }
        }
      };
      if (flags & 1) {
      } else if (tmD.narrow[x.m]) {
        consume(std::true_type{}, std::true_type{});
      } else if (small) {
        consume(std::true_type{}, std::false_type{});
      } else {
        consume(std::false_type{}, std::false_type{});
      }
      __syncwarp();
      if (!(flags & 2) && (threadIdx.x & 31) == 0) mbar_arrive(&empty[stage]);
      if (++stage == stages) {
        stage = 0;
        phase ^= 1;
      }
      if ((((sb + 1) * SPS) & 63) == 0) {  // bank every 64 baby steps (d1: 128 products)
#pragma unroll
        for (int jj = 0; jj < JT; jj++)
#pragma unroll
          for (int e = 0; e < 3; e++) {
            part[jj][e] = addmod(part[jj][e], kacc_reduce(acc[jj][e], q, bar, r64, r64s), q);
            acc[jj][e] = KAcc{0, 0, 0, 0, 0, 0};
          }
      }
    }
    const size_t ls = (size_t)L * n;
    const uint32_t a = x.a0 + g;
#pragma unroll
    for (int jj = 0; jj < JT; jj++) {
      const int gg = x.gg0 + jj;
      const int jslot = flat ? gg : (gg < G / 2 ? gg + G / 2 : gg - G / 2);
      uint64_t *Sa = S + ((size_t)a * nj + jslot) * 3 * ls + (size_t)x.m * n + (size_t)x.tile * TC + t;
#pragma unroll
      for (int e = 0; e < 3; e++) Sa[(size_t)e * ls] = addmod(part[jj][e], kacc_reduce(acc[jj][e], q, bar, r64, r64s), q);
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

hd_status encode_t(CUtensorMap *map, const void *base, CUtensorMapDataType dt, int rank, const cuuint64_t *dims,
                   const cuuint64_t *strides, const cuuint32_t *box) {
  auto fn = encode_fn();
  if (!fn) return hd_fail(HD_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, dt, (cuuint32_t)rank, const_cast<void *>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return hd_fail(HD_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return HD_OK;
}
hd_status encode(CUtensorMap *map, const uint64_t *base, int rank, const cuuint64_t *dims, const cuuint64_t *strides,
                 const cuuint32_t *box) {
  return encode_t(map, base, CU_TENSOR_MAP_DATA_TYPE_UINT64, rank, dims, strides, box);
}

int g_num_sms = 0;

struct DMaps {  // the diagonal maps of one launch (R34)
  CUtensorMap w, lo, hi;
  PackCls pk;
};

template <int AG, int JT, int QB, int SPS, bool FLUSH>
hd_status launch(hd_context *c, const DMaps &mD, const CUtensorMap &mR, uint64_t *S, int n1, int N, int nj,
                 uint32_t A, bool flat, int qrows, size_t sq) {
  constexpr size_t STAGE_BYTES = (size_t)(AG * JT * SPS * TC + QB * SPS * 2 * TC) * 8;
  const size_t budget = 227 * 1024 - 256;
  int stages = (int)std::min<size_t>(16, budget / STAGE_BYTES);
  if (const char *e = getenv("HD_MAC_STAGES")) stages = std::max(2, std::min(stages, atoi(e)));  // A/B knob
  if (stages < 2) return hd_fail(HD_E_PARAMS, "MAC stage does not fit shared memory");
  const size_t smem = stages * STAGE_BYTES + 2 * stages * sizeof(uint64_t);
  auto kern = mac_tma_kernel<AG, JT, QB, SPS, FLUSH>;
  HD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (!g_num_sms) HD_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, c->device));
  const uint32_t units = (A / AG) * (uint32_t)(nj / JT) * (uint32_t)(c->n / TC) * (uint32_t)c->L;
  const uint32_t grid = std::min<uint32_t>(units, (uint32_t)g_num_sms);
  const char *dry = getenv("HD_MAC_TMA_DRY"), *co = getenv("HD_MAC_COMPUTE_ONLY");  // measurement only
  // unit order (HD_MAC_ORDER, A/B): limb second-fastest by default, so concurrent CTAs mix the
  // wide (u64) and packed limbs' streams (MAC 7.92 -> 7.59 ms, stream alone 7.51 -> 7.09 at C4);
  // HD_MAC_ORDER=0: limb slowest
  const char *ord = getenv("HD_MAC_ORDER");
  const int flags = (dry && dry[0] == '1' ? 1 : 0) | (co && co[0] == '1' ? 2 : 0) | (ord && ord[0] == '0' ? 0 : 4);
  kern<<<grid, AG * TC + 32, smem, c->stream>>>(mD.w, mD.lo, mD.hi, mR, S, n1, N, c->L, c->logn, nj, A, flat ? 1 : 0,
                                                stages, qrows, sq, c->mt, flags, mD.pk);
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

template <int JT, int QB>
hd_status launch_f(hd_context *c, const DMaps &mD, const CUtensorMap &mR, uint64_t *S, int n1, int N, int nj,
                   uint32_t A, bool flat, int qrows, size_t sq, int ag, int sps) {
#define HD_MAC_L(AG_, SPS_)                                                                        \
  return n1 > 128 ? launch<AG_, JT, QB, SPS_, true>(c, mD, mR, S, n1, N, nj, A, flat, qrows, sq) \
                  : launch<AG_, JT, QB, SPS_, false>(c, mD, mR, S, n1, N, nj, A, flat, qrows, sq)
  if (ag == 4 && sps == 2) { HD_MAC_L(4, 2); }
  if (ag == 4) { HD_MAC_L(4, 4); }
  if (ag == 2 && sps == 2) { HD_MAC_L(2, 2); }
  if (ag == 2 && sps == 8) { HD_MAC_L(2, 8); }
  if (ag == 2) { HD_MAC_L(2, 4); }
  if (sps == 2) { HD_MAC_L(1, 2); }
  if (sps == 8) { HD_MAC_L(1, 8); }
  HD_MAC_L(1, 4);
#undef HD_MAC_L
}

template <int AG, int JT, int SPS>
hd_status launch_ct(hd_context *c, const CtMaps &mD, const CUtensorMap &mR, uint64_t *S, int n1, int N, int nj,
                    uint32_t A, bool flat) {
  constexpr size_t STAGE_BYTES = (size_t)(AG * JT * SPS * 2 * TC + SPS * 2 * TC) * 8;
  const size_t budget = 227 * 1024 - 256;
  int stages = (int)std::min<size_t>(16, budget / STAGE_BYTES);
  if (const char *e = getenv("HD_MAC_STAGES")) stages = std::max(2, std::min(stages, atoi(e)));
  if (stages < 2) return hd_fail(HD_E_PARAMS, "MAC stage does not fit shared memory");
  const size_t smem = stages * STAGE_BYTES + 2 * stages * sizeof(uint64_t);
  auto kern = mac_tma_ct_kernel<AG, JT, SPS>;
  HD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (!g_num_sms) HD_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, c->device));
  const uint32_t units = (A / AG) * (uint32_t)(nj / JT) * (uint32_t)(c->n / TC) * (uint32_t)c->L;
  const uint32_t grid = std::min<uint32_t>(units, (uint32_t)g_num_sms);
  uint32_t small_mask = 0;  // limbs whose residues stay below 2^47 (Karatsuba narrow form, R35)
  for (int l = 0; l < c->L && l < 32; l++)
    if (c->mod[l] < kNarrowBound) small_mask |= 1u << l;
  const char *dry = getenv("HD_MAC_TMA_DRY"), *co = getenv("HD_MAC_COMPUTE_ONLY");  // measurement only
  const char *ord = getenv("HD_MAC_ORDER");  // as the plaintext MAC: limb second-fastest unless "0"
  const int flags = (dry && dry[0] == '1' ? 1 : 0) | (co && co[0] == '1' ? 2 : 0) | (ord && ord[0] == '0' ? 0 : 4);
  kern<<<grid, AG * TC + 32, smem, c->stream>>>(mD, mR, S, n1, N, c->L, c->logn, nj, A, flat ? 1 : 0, stages, c->mt,
                                                small_mask, flags);
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}
}  // namespace

// S3 [A][nj][3][L][n] of encrypted diagonals Dct [A][N][2][L][n] (full giant-step ranges).
hd_status mac_tma_ct_run(hd_context *c, const uint64_t *D, const uint64_t *r, uint64_t *S3, uint32_t A, int n1, int N,
                         const std::vector<int32_t> &js, bool flat, const DPack &dp) {
  if (js.empty() || A == 0) return HD_OK;
  const int nj = (int)js.size(), G = N / n1, L = c->L, n = c->n;
  if (nj != G || L > CT_MAXL) return hd_fail(HD_E_STATE, "TMA MAC expects one giant step per diagonal block");
  const char *ag_env = getenv("HD_MAC_AG"), *sps_env = getenv("HD_MAC_SPS"), *jt_env = getenv("HD_MAC_CT_JT");
  int ag = ag_env ? atoi(ag_env) : 2;
  if (ag != 1 && ag != 2) ag = 2;
  while (ag > 1 && A % ag) ag /= 2;
  int sps = sps_env ? atoi(sps_env) : 8;
  if (sps != 4 && sps != 8) sps = 8;
  while (sps > 4 && n1 % sps) sps /= 2;
  if (n1 % sps) sps = 2;  // n1 even (mac_tma_supported)
  int jt = jt_env ? atoi(jt_env) : 2;
  if (jt != 1 && jt != 2 && jt != 4) jt = 2;
  while (jt > 1 && nj % jt) jt /= 2;
  // resolve to an instantiated (AG, JT, SPS) before the maps are encoded: the boxes must have
  // the kernel's SPS (the (2, 4) kernel is built for SPS 4 only; SPS 4 exists for AG 2 only)
  if (ag == 2 && jt == 4) sps = 4;
  else if (!(ag == 2 && jt == 2)) sps = 8;  // (2, 2) keeps the requested 4 or 8
  if (sps != 2 && n1 % sps) sps = 2;        // n1 even (mac_tma_supported)
  if (sps == 2) ag = jt = 1;                // the SPS-2 kernel is (1, 1, 2)
  CtMaps mD;
  hd_status s;
  // D of limb m: (coefficient, poly, diagonal, block, aggregate); packed (R34): per polynomial
  // block the wide limbs as u64 rows, the narrow limbs as u32 low / u16 high planes
  const size_t pp = dp.on ? dp.pp_bytes : (size_t)L * n * 8, db = 2 * pp;
  const int W = dp.on ? dp.W : L, R = dp.on ? dp.R : 0;
  const uint8_t *Db = reinterpret_cast<const uint8_t *>(D);
  const cuuint32_t box[5] = {(cuuint32_t)TC, 2, (cuuint32_t)sps, (cuuint32_t)jt, (cuuint32_t)ag};
  const cuuint64_t dims[5] = {(cuuint64_t)n, 2, (cuuint64_t)n1, (cuuint64_t)G, (cuuint64_t)A};
  const cuuint64_t strides[4] = {(cuuint64_t)pp, (cuuint64_t)db, (cuuint64_t)n1 * db, (cuuint64_t)N * db};
  for (int m = 0; m < L; m++) {
    const bool nw = dp.on && dp.cls[m];
    const int ix = dp.on ? dp.idx[m] : m;
    mD.narrow[m] = nw ? 1 : 0;
    if (!nw) {
      if ((s = encode_t(&mD.m[m], Db + (size_t)ix * n * 8, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, dims, strides, box)))
        return s;
      mD.hi[m] = mD.m[m];
    } else {
      if ((s = encode_t(&mD.m[m], Db + (8 * (size_t)W + 4 * (size_t)ix) * n, CU_TENSOR_MAP_DATA_TYPE_UINT32, 5, dims,
                        strides, box)) ||
          (s = encode_t(&mD.hi[m], Db + (8 * (size_t)W + 4 * (size_t)R + 2 * (size_t)ix) * n,
                        CU_TENSOR_MAP_DATA_TYPE_UINT16, 5, dims, strides, box)))
        return s;
    }
  }
  CUtensorMap mR;
  {
    const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)L, (cuuint64_t)2 * n1};
    const cuuint64_t strides[2] = {(cuuint64_t)n * 8, (cuuint64_t)L * n * 8};
    const cuuint32_t box[3] = {(cuuint32_t)TC, 1, (cuuint32_t)(2 * sps)};
    if ((s = encode(&mR, r, 3, dims, strides, box))) return s;
  }
#define HD_CT_L(AG_, JT_, SPS_) return launch_ct<AG_, JT_, SPS_>(c, mD, mR, S3, n1, N, nj, A, flat)
  if (sps == 2) { HD_CT_L(1, 1, 2); }
  if (ag == 2 && jt == 2 && sps == 8) { HD_CT_L(2, 2, 8); }
  if (ag == 2 && jt == 2 && sps == 4) { HD_CT_L(2, 2, 4); }
  if (ag == 2 && jt == 4) { HD_CT_L(2, 4, 4); }
  if (ag == 2 && jt == 1) { HD_CT_L(2, 1, 8); }
  if (ag == 1 && jt == 4) { HD_CT_L(1, 4, 8); }
  if (ag == 1 && jt == 2) { HD_CT_L(1, 2, 8); }
  HD_CT_L(1, 1, 8);
#undef HD_CT_L
}

bool mac_tma_ct_supported(const hd_context *c, int n1, int N, bool flat) {
  return mac_tma_supported(c, n1, N, flat, 1) && c->L <= CT_MAXL;
}

bool mac_tma_supported(const hd_context *c, int n1, int N, bool flat, uint32_t Q) {
  const char *v = getenv("HD_MAC_VARIANT");  // 'c': the LDG kernels of mac.cu ('g': generic)
  if (v && (v[0] == 'c' || v[0] == 'g')) return false;
  if (c->n % TC || n1 % 2 || n1 > 256 || Q < 1 || Q > 4) return false;
  if ((flat ? N % n1 : (N / 2) % n1) != 0) return false;  // full giant-step ranges only
  for (int l = 0; l < c->L; l++)
    if (c->mod[l] >= (1ull << 60)) return false;  // Karatsuba split: r_l + r_h < 2^32
  return encode_fn() != nullptr;
}

// S [Q][A][nj][2][L][n]; r [Q][n1][2][L][n] (query stride n1 2 L n); D [A][N][L][n].
hd_status mac_tma_run(hd_context *c, const uint64_t *D, const uint64_t *r, uint64_t *S, uint32_t A, int n1, int N,
                      const std::vector<int32_t> &js, uint32_t Q, bool flat, const DPack &dp) {
  if (js.empty() || A == 0) return HD_OK;
  const int nj = (int)js.size(), G = N / n1;
  if (nj != G) return hd_fail(HD_E_STATE, "TMA MAC expects one giant step per diagonal block");
  // aggregates per CTA (HD_MAC_AG, A/B knob), baby steps per stage (HD_MAC_SPS)
  const char *ag_env = getenv("HD_MAC_AG"), *sps_env = getenv("HD_MAC_SPS");
  int ag = ag_env ? atoi(ag_env) : 2;
  if (ag != 1 && ag != 2 && ag != 4) ag = 2;
  while (ag > 1 && A % ag) ag /= 2;
  // measured at 2^20 x 512 (n1 = 128), round 2 (u64 diagonals, carry-save): AG 2 / SPS 8 (2 stages
  // of 80 KB) 8.97 ms; SPS 4 9.35; SPS 2 10.4; AG 1 / SPS 8 10.7; AG 4 / SPS 2 10.3.  Round 3
  // (packed diagonals, Karatsuba, limb-second order): SPS 4 (5 stages of 40 KB) 7.30-7.34 ms vs
  // SPS 8 7.53 (the deeper ring absorbs the compute's jitter); AG 4 / SPS 4 9.8; AG 1 9.0
  // batches (Q > 1) keep SPS 8: 13.19 vs 14.48 ms per pair of queries
  int sps = sps_env ? atoi(sps_env) : (Q == 1 ? 4 : 8);
  if (sps != 2 && sps != 4 && sps != 8) sps = Q == 1 ? 4 : 8;
  if (ag == 4 && sps == 8) sps = 4;  // AG 4 is built for SPS 2 and 4 (launch_f): the boxes must match
  while (sps > 2 && n1 % sps) sps /= 2;
  // giant steps (diagonal blocks) per thread: up to 4 (each r word then serves JT diagonal words)
  const int jt = nj % 4 == 0 ? 4 : (nj % 2 == 0 ? 2 : 1);
  const int jtq = Q == 1 ? jt : (Q == 2 ? std::min(jt, 2) : 1);  // QB x JT <= 4 accumulator pairs
  const int L = c->L, n = c->n;
  DMaps mD;
  CUtensorMap mR;
  hd_status s;
  {  // D: (coefficient, limb, diagonal within block, block, aggregate); packed (R34): the wide
     // limbs as u64 words, the narrow limbs' low / high planes as u32 / u16 (same box, 6 B per word)
    const size_t db = dp.on ? dp.diag_bytes : (size_t)L * n * 8;  // bytes of one diagonal
    const int W = dp.on ? dp.W : L, R = dp.on ? dp.R : 0;
    const cuuint32_t box[5] = {(cuuint32_t)TC, 1, (cuuint32_t)sps, (cuuint32_t)jtq, (cuuint32_t)ag};
    auto enc_plane = [&](CUtensorMap *m, const uint8_t *base, int count, int esize, CUtensorMapDataType dt) {
      const cuuint64_t dims[5] = {(cuuint64_t)n, (cuuint64_t)std::max(1, count), (cuuint64_t)n1, (cuuint64_t)G,
                                  (cuuint64_t)A};
      const cuuint64_t strides[4] = {(cuuint64_t)n * esize, (cuuint64_t)db, (cuuint64_t)n1 * db, (cuuint64_t)N * db};
      return encode_t(m, base, dt, 5, dims, strides, box);
    };
    const uint8_t *Db = reinterpret_cast<const uint8_t *>(D);
    if ((s = enc_plane(&mD.w, Db, W, 8, CU_TENSOR_MAP_DATA_TYPE_UINT64))) return s;
    if ((s = enc_plane(&mD.lo, Db + 8 * (size_t)W * n, R, 4, CU_TENSOR_MAP_DATA_TYPE_UINT32))) return s;
    if ((s = enc_plane(&mD.hi, Db + (8 * (size_t)W + 4 * (size_t)R) * n, R, 2, CU_TENSOR_MAP_DATA_TYPE_UINT16)))
      return s;
    for (int l = 0; l < HD_MAXMOD; l++) {
      mD.pk.cls[l] = l < L && dp.on ? dp.cls[l] : 0;
      mD.pk.idx[l] = l < L ? (dp.on ? dp.idx[l] : (uint8_t)l) : 0;
    }
  }
  {  // r: (coefficient, limb, row = (query, baby step, poly))
    const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)L, (cuuint64_t)Q * 2 * n1};
    const cuuint64_t strides[2] = {(cuuint64_t)n * 8, (cuuint64_t)L * n * 8};
    const cuuint32_t box[3] = {(cuuint32_t)TC, 1, (cuuint32_t)(2 * sps)};
    if ((s = encode(&mR, r, 3, dims, strides, box))) return s;
  }
  const size_t sq = (size_t)A * nj * 2 * L * n;
  const int qrows = 2 * n1;
  if (Q == 1) {
    if (jtq == 4) return launch_f<4, 1>(c, mD, mR, S, n1, N, nj, A, flat, qrows, sq, ag, sps);
    if (jtq == 2) return launch_f<2, 1>(c, mD, mR, S, n1, N, nj, A, flat, qrows, sq, ag, sps);
    return launch_f<1, 1>(c, mD, mR, S, n1, N, nj, A, flat, qrows, sq, ag, sps);
  }
  // query batches (NEXT-4): every diagonal word staged once serves QB queries
  if (Q == 2) {
    if (jtq == 2) return launch_f<2, 2>(c, mD, mR, S, n1, N, nj, A, flat, qrows, sq, ag, sps);
    return launch_f<1, 2>(c, mD, mR, S, n1, N, nj, A, flat, qrows, sq, ag, sps);
  }
  if (Q == 3) return launch_f<1, 3>(c, mD, mR, S, n1, N, nj, A, flat, qrows, sq, ag, sps);
  return launch_f<1, 4>(c, mD, mR, S, n1, N, nj, A, flat, qrows, sq, ag, sps);
}
