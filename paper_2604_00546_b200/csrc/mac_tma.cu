// mac_tma.cu -- the fused diagonal x ciphertext MAC (a5, Alg. sender-bsgs Step 2b)
// as a warp-specialised TMA pipeline.
//
//   S[b][a][j][p][m][t] = sum_{i < n1} r[b][i][p][m][t] * D[a][k(j,i)][m][t]  mod q_m,
//   k(j,i) = (j n1 + i) mod N   (replicated: preshifted giant steps; flat: j n1 + i < N)
//
// for full giant-step ranges (every j uses all n1 baby steps), q_m < 2^60, b < QB queries.
//
// Why this shape: the LDG kernel (mac.cu, mac_cs_kernel) spends ~40
// SASS per diagonal word -- address formation, predicated prefetch, register staging -- and
// sits at ~63 % issue, i.e. it is issue-bound below the HBM roofline.  Here a producer warp
// streams the diagonals with 3-D TMA boxes (128 coefficients x 1 limb x SPS consecutive
// diagonals, evict-first) and the baby-step rows (r, L2-resident) into a ring of shared-memory
// stages; consumer threads own one coefficient of one aggregate and ALL JT giant steps of
// their unit, so each r word read from shared memory serves JT diagonal words and each
// diagonal word costs two carry-save products plus one LDS.  The ring keeps ~200 KB of loads
// in flight per SM without a register per byte.
//
// Work unit = (AG consecutive aggregates, giant-step group of JT, 128-coefficient tile, limb);
// one persistent CTA per SM walks units u = blockIdx.x, + gridDim.x, ... with the aggregate
// group fastest so concurrently resident CTAs share few r tiles (L2 reuse).
#include "common.cuh"
#include "ks.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

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

// carry-save 64x64 multiply-accumulate, as mac.cu (a1, b1 < 2^28): value = lo + mid 2^32 +
// (hi + cnt) 2^64; mid folded every 8 products
struct Acc {
  uint64_t lo, mid, hi;
  uint32_t cnt;
};
__device__ __forceinline__ void acc_mac(Acc &A, uint32_t a0, uint32_t a1, uint32_t b0, uint32_t b1) {
  asm("{\n\t.reg .u64 t;\n\t"
      "mul.wide.u32 t, %4, %6;\n\t"
      "add.cc.u64 %0, %0, t;\n\t"
      "addc.u32 %3, %3, 0;\n\t"
      "mad.wide.u32 %1, %4, %7, %1;\n\t"
      "mad.wide.u32 %1, %5, %6, %1;\n\t"
      "mad.wide.u32 %2, %5, %7, %2;\n\t"
      "}"
      : "+l"(A.lo), "+l"(A.mid), "+l"(A.hi), "+r"(A.cnt)
      : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void acc_fold(Acc &A) {
  const uint64_t ml = A.mid << 32, mh = A.mid >> 32;
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+l"(A.lo), "+r"(A.cnt) : "l"(ml));
  A.hi += mh;
  A.mid = 0;
}

struct Unit {
  uint32_t a0;  // first aggregate of the group
  int jg, tile, m;
};
__device__ __forceinline__ Unit decode(uint32_t u, uint32_t nag, int ngrp, int tiles, int AG) {
  Unit x;
  x.a0 = (u % nag) * AG;
  u /= nag;
  x.jg = (int)(u % ngrp);
  u /= ngrp;
  x.tile = (int)(u % tiles);
  x.m = (int)(u / tiles);
  return x;
}

// Producer state: the next (unit, baby-step block) to load and the ring slot it goes to.
template <int AG, int JT, int QB, int SPS>
struct Producer {
  uint32_t u, units, nag, step;
  int sb, nsb, ngrp, tiles, stage, stages, jmin, n1, N, qrows;
  uint32_t phase;
  uint64_t pol_stream, pol_keep;
  __device__ __forceinline__ bool more() const { return u < units; }
  // wait until the slot is free, then issue its TMA loads (D boxes evict-first, r evict-last)
  __device__ __forceinline__ void issue(unsigned char *smem, uint64_t *full, uint64_t *empty, const CUtensorMap *tmD,
                                        const CUtensorMap *tmR) {
    constexpr int D_WORDS = AG * JT * SPS * TC, R_WORDS = QB * SPS * 2 * TC;
    constexpr uint32_t STAGE_BYTES = (D_WORDS + R_WORDS) * 8;
    const Unit x = decode(u, nag, ngrp, tiles, AG);
    mbar_wait(&empty[stage], phase ^ 1);
    mbar_arrive_expect_tx(&full[stage], STAGE_BYTES);
    uint64_t *base = reinterpret_cast<uint64_t *>(smem + (size_t)stage * STAGE_BYTES);
#pragma unroll
    for (int g = 0; g < AG; g++)
#pragma unroll
      for (int jj = 0; jj < JT; jj++) {
        const int j = jmin + x.jg * JT + jj;
        const int k0 = ((j * n1 + sb * SPS) % N + N) % N;  // SPS consecutive diagonals (no wrap)
        tma_load_3d(base + (g * JT + jj) * SPS * TC, tmD, x.tile * TC, x.m, (int)((x.a0 + g) * N + k0), &full[stage],
                    pol_stream);
      }
#pragma unroll
    for (int b = 0; b < QB; b++)
      tma_load_3d(base + D_WORDS + b * SPS * 2 * TC, tmR, x.tile * TC, x.m, b * qrows + sb * SPS * 2, &full[stage],
                  pol_keep);
    if (++stage == stages) {
      stage = 0;
      phase ^= 1;
    }
    if (++sb == nsb) {
      sb = 0;
      u += step;
    }
  }
};

// AG aggregates x TC coefficients consumer threads (+ one producer warp unless INLINE: then
// thread 0 also issues the loads, one slot per iteration, and all 4 AG warps compute).
// Stage layout (u64): D[AG][JT][SPS][TC], then r[QB][SPS][2][TC].
template <int AG, int JT, int QB, int SPS, bool FLUSH, bool INLINE>
__global__ void __launch_bounds__(AG *TC + (INLINE ? 0 : 32), 1)
    mac_tma_kernel(const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmR,
                   uint64_t *__restrict__ S, int n1, int N, int L, int logn, int jmin, int nj, uint32_t A,
                   int stages, int qrows, size_t s_query_stride, ModTab mt, int dry) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int D_WORDS = AG * JT * SPS * TC, R_WORDS = QB * SPS * 2 * TC;
  constexpr uint32_t STAGE_BYTES = (D_WORDS + R_WORDS) * 8;
  constexpr int CONSUMERS = AG * TC;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)stages * STAGE_BYTES);
  uint64_t *empty = full + stages;
  const int n = 1 << logn, tiles = n / TC, ngrp = nj / JT, nsb = n1 / SPS;
  const uint32_t nag = A / AG, units = nag * (uint32_t)ngrp * (uint32_t)tiles * (uint32_t)L;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMERS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  Producer<AG, JT, QB, SPS> pr;
  const bool is_producer = INLINE ? threadIdx.x == 0 : threadIdx.x == CONSUMERS;
  if (is_producer) {
    pr.u = blockIdx.x;
    pr.units = units;
    pr.nag = nag;
    pr.step = gridDim.x;
    pr.sb = 0;
    pr.nsb = nsb;
    pr.ngrp = ngrp;
    pr.tiles = tiles;
    pr.stage = 0;
    pr.stages = stages;
    pr.jmin = jmin;
    pr.n1 = n1;
    pr.N = N;
    pr.qrows = qrows;
    pr.phase = 0;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pr.pol_stream));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pr.pol_keep));
  }
  if (!INLINE && threadIdx.x >= CONSUMERS) {  // ---------------- producer warp ----------------
    if (is_producer)
      while (pr.more()) pr.issue(smem, full, empty, &tmD, &tmR);
    return;
  }
  if (INLINE && is_producer)  // prefill every slot (fresh slots are free)
    for (int k = 0; k < stages && pr.more(); k++) pr.issue(smem, full, empty, &tmD, &tmR);
  bool first = true;

  // ---------------- consumers: thread = (aggregate g of the group, coefficient t) ----------------
  const int g = threadIdx.x / TC, t = threadIdx.x % TC;
  int stage = 0;
  uint32_t phase = 0;
  for (uint32_t u = blockIdx.x; u < units; u += gridDim.x) {
    const Unit x = decode(u, nag, ngrp, tiles, AG);
    const uint64_t q = mt.q[x.m], bar = mt.bar[x.m], r64 = mt.r64[x.m], r64s = mt.r64s[x.m];
    Acc acc[QB][JT][2];
    uint64_t part[QB][JT][2];
#pragma unroll
    for (int b = 0; b < QB; b++)
#pragma unroll
      for (int jj = 0; jj < JT; jj++) {
        acc[b][jj][0] = acc[b][jj][1] = Acc{0, 0, 0, 0};
        part[b][jj][0] = part[b][jj][1] = 0;
      }
    for (int sb = 0; sb < nsb; sb++) {
      // inline producer: refill the slot the CTA released last iteration (waits for the
      // slowest warp to finish it), `stages - 1` blocks ahead of this one
      if (INLINE && is_producer && !first && pr.more()) pr.issue(smem, full, empty, &tmD, &tmR);
      first = false;
      mbar_wait(&full[stage], phase);
      if (dry) {  // measurement only (HD_MAC_TMA_DRY=1): the TMA stream without the arithmetic
        mbar_arrive(&empty[stage]);
        if (++stage == stages) {
          stage = 0;
          phase ^= 1;
        }
        continue;
      }
      const uint64_t *Ds = reinterpret_cast<const uint64_t *>(smem + (size_t)stage * STAGE_BYTES) + g * JT * SPS * TC + t;
      const uint64_t *Rs = reinterpret_cast<const uint64_t *>(smem + (size_t)stage * STAGE_BYTES) + D_WORDS + t;
#pragma unroll
      for (int s = 0; s < SPS; s++) {
        uint64_t d[JT];
#pragma unroll
        for (int jj = 0; jj < JT; jj++) d[jj] = Ds[(jj * SPS + s) * TC];
#pragma unroll
        for (int b = 0; b < QB; b++) {
          const uint64_t r0 = Rs[(b * SPS * 2 + 2 * s) * TC], r1 = Rs[(b * SPS * 2 + 2 * s + 1) * TC];
          const uint32_t r00 = (uint32_t)r0, r01 = (uint32_t)(r0 >> 32), r10 = (uint32_t)r1, r11 = (uint32_t)(r1 >> 32);
#pragma unroll
          for (int jj = 0; jj < JT; jj++) {
            const uint32_t b0 = (uint32_t)d[jj], b1 = (uint32_t)(d[jj] >> 32);
            acc_mac(acc[b][jj][0], r00, r01, b0, b1);
            acc_mac(acc[b][jj][1], r10, r11, b0, b1);
          }
        }
      }
      mbar_arrive(&empty[stage]);  // this thread's reads of the stage are done
      if (++stage == stages) {
        stage = 0;
        phase ^= 1;
      }
      if ((((sb + 1) * SPS) & 7) == 0) {  // every 8 baby steps: 16 mid terms < 2^64
#pragma unroll
        for (int b = 0; b < QB; b++)
#pragma unroll
          for (int jj = 0; jj < JT; jj++) {
            acc_fold(acc[b][jj][0]);
            acc_fold(acc[b][jj][1]);
          }
      }
      if (FLUSH && (sb % (128 / SPS)) == (128 / SPS) - 1) {  // n1 > 128: bank every 128 terms
#pragma unroll
        for (int b = 0; b < QB; b++)
#pragma unroll
          for (int jj = 0; jj < JT; jj++)
#pragma unroll
            for (int p = 0; p < 2; p++) {
              Acc &X = acc[b][jj][p];
              acc_fold(X);
              part[b][jj][p] = addmod(part[b][jj][p], reduce128(X.hi + X.cnt, X.lo, q, bar, r64, r64s), q);
              X = Acc{0, 0, 0, 0};
            }
      }
    }
    const size_t ls = (size_t)L * n;
    const uint32_t a = x.a0 + g;
#pragma unroll
    for (int b = 0; b < QB; b++)
#pragma unroll
      for (int jj = 0; jj < JT; jj++) {
        uint64_t *Sa = S + b * s_query_stride + ((size_t)a * nj + x.jg * JT + jj) * 2 * ls + (size_t)x.m * n +
                       (size_t)x.tile * TC + t;
#pragma unroll
        for (int p = 0; p < 2; p++) {
          Acc &X = acc[b][jj][p];
          acc_fold(X);
          Sa[(size_t)p * ls] = addmod(part[b][jj][p], reduce128(X.hi + X.cnt, X.lo, q, bar, r64, r64s), q);
        }
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

// rows of n u64 coefficients grouped as [rows][L][n]: a 3-D map (coef, limb, row), box
// (TC, 1, box_rows)
hd_status make_map(CUtensorMap *map, const uint64_t *base, int n, int L, uint64_t rows, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return hd_fail(HD_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)L, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)n * 8, (cuuint64_t)L * n * 8};
  cuuint32_t box[3] = {(cuuint32_t)TC, 1, box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<uint64_t *>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return hd_fail(HD_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return HD_OK;
}

int g_num_sms = 0;

template <int AG, int JT, int QB, int SPS, bool FLUSH, bool INLINE>
hd_status launch(hd_context *c, const CUtensorMap &mD, const CUtensorMap &mR, uint64_t *S, int n1, int N, int jmin,
                 int nj, uint32_t A, int qrows, size_t sq) {
  constexpr size_t STAGE_BYTES = (size_t)(AG * JT * SPS * TC + QB * SPS * 2 * TC) * 8;
  const size_t budget = 227 * 1024 - 256;
  int stages = (int)std::min<size_t>(8, budget / STAGE_BYTES);
  if (const char *e = getenv("HD_MAC_STAGES")) stages = std::max(2, std::min(stages, atoi(e)));  // A/B knob
  if (stages < 2) return hd_fail(HD_E_PARAMS, "MAC stage does not fit shared memory");
  const size_t smem = stages * STAGE_BYTES + 2 * stages * sizeof(uint64_t);
  auto kern = mac_tma_kernel<AG, JT, QB, SPS, FLUSH, INLINE>;
  HD_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (!g_num_sms) HD_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, c->device));
  const uint32_t units = (A / AG) * (uint32_t)(nj / JT) * (uint32_t)(c->n / TC) * (uint32_t)c->L;
  const uint32_t grid = std::min<uint32_t>(units, (uint32_t)g_num_sms);
  const char *dry = getenv("HD_MAC_TMA_DRY");
  kern<<<grid, AG * TC + (INLINE ? 0 : 32), smem, c->stream>>>(mD, mR, S, n1, N, c->L, c->logn, jmin, nj, A, stages, qrows, sq,
                                                c->mt, dry && dry[0] == '1');
  ++c->launches;
  HD_CUDA(cudaGetLastError());
  return HD_OK;
}

// Per-launch choice: AG aggregates per CTA (consumer warps = 4 AG), SPS baby steps per stage.
template <int JT, int QB>
hd_status launch_f(hd_context *c, const CUtensorMap &mD, const CUtensorMap &mR, uint64_t *S, int n1, int N, int jmin,
                   int nj, uint32_t A, int qrows, size_t sq, int ag, int sps) {
#define HD_MAC_L(AG_, SPS_, IN_)                                                                               \
  return n1 > 128 ? launch<AG_, JT, QB, SPS_, true, IN_>(c, mD, mR, S, n1, N, jmin, nj, A, qrows, sq)            \
                  : launch<AG_, JT, QB, SPS_, false, IN_>(c, mD, mR, S, n1, N, jmin, nj, A, qrows, sq)
  const char *in_env = getenv("HD_MAC_INLINE");
  const bool inl = !(in_env && in_env[0] == '0');
  if (ag == 4 && inl) { HD_MAC_L(4, 2, true); }
  if (ag == 4) { HD_MAC_L(4, 2, false); }
  if (ag == 2 && sps == 2) { HD_MAC_L(2, 2, false); }
  if (ag == 2) { HD_MAC_L(2, 4, false); }
  if (sps == 2) { HD_MAC_L(1, 2, false); }
  HD_MAC_L(1, 4, false);
#undef HD_MAC_L
}
}  // namespace

bool mac_tma_supported(const hd_context *c, int n1, int N, bool flat, uint32_t Q) {
  const char *v = getenv("HD_MAC_VARIANT");  // 'c': the LDG kernels of mac.cu ('g': generic)
  if (v && (v[0] == 'c' || v[0] == 'g')) return false;
  if (c->n % TC || n1 % 2 || n1 > 256 || Q < 1 || Q > 4) return false;
  if ((flat ? N % n1 : (N / 2) % n1) != 0) return false;  // full giant-step ranges only
  for (int l = 0; l < c->L; l++)
    if (c->mod[l] >= (1ull << 60)) return false;  // carry-save operand split
  return encode_fn() != nullptr;
}

// S [Q][A][nj][2][L][n]; r [Q][n1][2][L][n] (query stride n1 2 L n).
hd_status mac_tma_run(hd_context *c, const uint64_t *D, const uint64_t *r, uint64_t *S, uint32_t A, int n1, int N,
                      const std::vector<int32_t> &js, uint32_t Q) {
  if (js.empty() || A == 0) return HD_OK;
  const int jmin = js.front(), nj = (int)js.size();
  // aggregates per CTA (HD_MAC_AG, A/B knob): 4 -> 16 consumer warps per SM with the producer
  // inline (128 registers each); 2 / 1 with a separate producer warp
  const char *ag_env = getenv("HD_MAC_AG");
  int ag = ag_env ? atoi(ag_env) : 4;
  if (ag != 1 && ag != 2 && ag != 4) ag = 4;
  while (ag > 1 && A % ag) ag /= 2;
  const char *sps_env = getenv("HD_MAC_SPS");
  const int sps = (sps_env && atoi(sps_env) == 2) || n1 % 4 || ag == 4 ? 2 : 4;  // baby steps per stage
  CUtensorMap mD, mR;
  hd_status s;
  if ((s = make_map(&mD, D, c->n, c->L, (uint64_t)A * N, sps))) return s;
  if ((s = make_map(&mR, r, c->n, c->L, (uint64_t)Q * 2 * n1, 2 * sps))) return s;
  const size_t sq = (size_t)A * nj * 2 * c->L * c->n;
  const int qrows = 2 * n1;
  // giant steps per thread: all of them up to 4 (each r word then serves JT diagonal words)
  const int jt = nj % 4 == 0 ? 4 : (nj % 2 == 0 ? 2 : 1);
  if (Q == 1) {
    if (jt == 4) return launch_f<4, 1>(c, mD, mR, S, n1, N, jmin, nj, A, qrows, sq, ag, sps);
    if (jt == 2) return launch_f<2, 1>(c, mD, mR, S, n1, N, jmin, nj, A, qrows, sq, ag, sps);
    return launch_f<1, 1>(c, mD, mR, S, n1, N, jmin, nj, A, qrows, sq, ag, sps);
  }
  // query batches (NEXT-4): every diagonal word staged once serves QB queries; QB x JT <= 4
  if (Q == 2) {
    if (jt >= 2) return launch_f<2, 2>(c, mD, mR, S, n1, N, jmin, nj, A, qrows, sq, ag, sps);
    return launch_f<1, 2>(c, mD, mR, S, n1, N, jmin, nj, A, qrows, sq, ag, sps);
  }
  if (Q == 3) return launch_f<1, 3>(c, mD, mR, S, n1, N, jmin, nj, A, qrows, sq, ag, sps);
  return launch_f<1, 4>(c, mD, mR, S, n1, N, jmin, nj, A, qrows, sq, ag, sps);
}
