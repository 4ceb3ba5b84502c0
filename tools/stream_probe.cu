// stream_probe.cu -- HBM read-pattern probe (profiling aid, not part of libhd).
//
// Measures the read bandwidth of the MAC kernel's access pattern against plain
// streaming, with trivial arithmetic, to separate "layout / DRAM locality" from
// "latency / issue" limits.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -o stream_probe tools/stream_probe.cu ; run: ./stream_probe [GB]
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); exit(1); } } while (0)

// 1. flat grid-stride 16-byte loads
__global__ void flat16(const ulonglong2 *__restrict__ p, size_t n16, uint64_t *out) {
  uint64_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    ulonglong2 v = __ldcs(p + i);
    acc ^= v.x + v.y;
  }
  if (acc == 0x123456789ull) out[0] = acc;
}

// 2. MAC pattern: grid (A, n/128, Z); CTA reads rows of 128 words (1 KB), JT rows per
// step, rows of consecutive steps `stride` words apart; `run` consecutive words per
// thread-step (run = 1: exactly the MAC kernel; run > 1: longer contiguous runs).
template <int JT, int RUN>
__global__ void __launch_bounds__(128) macpat(const uint64_t *__restrict__ D, size_t a_stride, size_t stride,
                                              int steps, int L, int n, uint64_t *out) {
  const int l = blockIdx.z % L, jg = blockIdx.z / L;
  const uint64_t *b = D + blockIdx.x * a_stride + (size_t)l * n + (size_t)jg * JT * steps * stride +
                      (size_t)blockIdx.y * 128 * RUN + threadIdx.x;
  uint64_t acc = 0;
  for (int i = 0; i < steps; i++) {
#pragma unroll
    for (int j = 0; j < JT; j++)
#pragma unroll
      for (int k = 0; k < RUN; k++) acc ^= __ldcs(b + (size_t)(j * steps + i) * stride + k * 128);
  }
  if (acc == 0x123456789ull) out[0] = acc;
}

// 3. MAC pattern plus the baby-step table reads of the MAC kernel: per step, JT D rows
// and 2 r rows (r[i][p][l][t], L2-resident per (l, tile)); RSH > 0 reads r only every
// 2^RSH steps (emulates r reuse across threads).
template <int JT, int RSH>
__global__ void __launch_bounds__(128) macpat_r(const uint64_t *__restrict__ D, const uint64_t *__restrict__ r,
                                                size_t a_stride, size_t stride, int steps, int L, int n,
                                                uint64_t *out) {
  const int l = blockIdx.z % L, jg = blockIdx.z / L;
  const uint64_t *b = D + blockIdx.x * a_stride + (size_t)l * n + (size_t)jg * JT * steps * stride +
                      (size_t)blockIdx.y * 128 + threadIdx.x;
  const uint64_t *rq = r + (size_t)l * n + (size_t)blockIdx.y * 128 + threadIdx.x;
  uint64_t acc = 0;
  for (int i = 0; i < steps; i++) {
#pragma unroll
    for (int j = 0; j < JT; j++) acc ^= __ldcs(b + (size_t)(j * steps + i) * stride);
    if ((i & ((1 << RSH) - 1)) == 0) acc += __ldg(rq + (size_t)(2 * i) * stride) ^ __ldg(rq + (size_t)(2 * i + 1) * stride);
  }
  if (acc == 0x123456789ull) out[0] = acc;
}

int main(int argc, char **argv) {
  const double gb = argc > 1 ? atof(argv[1]) : 48.0;
  const size_t words = (size_t)(gb * 1e9 / 8) & ~((size_t)(1 << 20) - 1);
  uint64_t *D, *out;
  CK(cudaMalloc(&D, words * 8));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemset(D, 1, words * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char *name, size_t bytes, auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 3; r++) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%-44s %8.3f ms  %7.0f GB/s\n", name, best, bytes / (best * 1e-3) / 1e9);
  };
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mult : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, sizeof nm, "flat16 grid=%dx SMs x 512", mult);
    timeit(nm, words * 8, [&] { flat16<<<sms * mult, 512>>>((const ulonglong2 *)D, words / 2, out); });
  }
  // MAC geometry at C4: A = 64 aggregates, ring 2^16, L = 3, n1 = 128, nj = 4 (JT = 2 -> 2 groups)
  const int n = 1 << 16, L = 3, n1 = 128, A = 64;
  const size_t ls = (size_t)L * n, a_stride = (size_t)512 * ls;
  const size_t need = (size_t)A * a_stride;
  if (need <= words) {
    const size_t bytes = need * 8;
    timeit("macpat JT=2 run=1 (MAC kernel addressing)", bytes, [&] {
      macpat<2, 1><<<dim3(A, n / 128, L * 2), 128>>>(D, a_stride, ls, n1, L, n, out);
    });
    timeit("macpat JT=4 run=1", bytes, [&] {
      macpat<4, 1><<<dim3(A, n / 128, L), 128>>>(D, a_stride, ls, n1, L, n, out);
    });
    timeit("macpat JT=2 run=2 (2 KB rows)", bytes, [&] {
      macpat<2, 2><<<dim3(A, n / 256, L * 2), 128>>>(D, a_stride, ls, n1, L, n, out);
    });
    timeit("macpat JT=2 run=4 (4 KB rows)", bytes, [&] {
      macpat<2, 4><<<dim3(A, n / 512, L * 2), 128>>>(D, a_stride, ls, n1, L, n, out);
    });
    uint64_t *R;
    CK(cudaMalloc(&R, (size_t)2 * n1 * ls * 8));
    CK(cudaMemset(R, 2, (size_t)2 * n1 * ls * 8));
    timeit("macpat_r JT=2 + r every step (MAC traffic)", bytes, [&] {
      macpat_r<2, 0><<<dim3(A, n / 128, L * 2), 128>>>(D, R, a_stride, ls, n1, L, n, out);
    });
    timeit("macpat_r JT=2 + r every 2nd step", bytes, [&] {
      macpat_r<2, 1><<<dim3(A, n / 128, L * 2), 128>>>(D, R, a_stride, ls, n1, L, n, out);
    });
    timeit("macpat_r JT=2 + r every 4th step", bytes, [&] {
      macpat_r<2, 2><<<dim3(A, n / 128, L * 2), 128>>>(D, R, a_stride, ls, n1, L, n, out);
    });
    cudaFree(R);
  } else {
    printf("macpat skipped: need %.1f GB\n", need * 8 / 1e9);
  }
  return 0;
}
