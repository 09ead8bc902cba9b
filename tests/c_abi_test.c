/* Plain C11 client of include/gemm_f16.h (no C++, no Python): proves the
 * boundary is a C ABI.  `c_abi_test` checks argument handling without a GPU;
 * `c_abi_test gpu` also runs C += A.B on device buffers from cudaMalloc
 * (all-ones inputs: every element must equal C_in + K exactly). */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gemm_f16.h"

#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      return 1;                                                       \
    }                                                                 \
  } while (0)

/* cudart entry points, declared here so this file stays plain C without CUDA headers */
int cudaMalloc(void** p, size_t n);
int cudaFree(void* p);
int cudaMemcpy(void* dst, const void* src, size_t n, int kind);
int cudaDeviceSynchronize(void);

static int cpu_checks(void) {
  const void* p = (const void*)(uintptr_t)256;
  CHECK(gemm_f16(-1, 8, 8, p, 8, p, 8, (void*)p, 8, GEMM_ACC_F32, NULL) == GEMM_ERR_INVALID_VALUE);
  CHECK(gemm_f16(8, 8, 8, p, 4, p, 8, (void*)p, 8, GEMM_ACC_F32, NULL) == GEMM_ERR_INVALID_VALUE);
  CHECK(gemm_f16(8, 8, 8, p, 8, p, 8, (void*)p, 8, 7, NULL) == GEMM_ERR_INVALID_VALUE);
  CHECK(gemm_f16(8, 8, 12, p, 12, p, 8, (void*)p, 8, GEMM_ACC_F32, NULL) == GEMM_ERR_MISALIGNED);
  CHECK(gemm_f16(0, 8, 8, p, 8, p, 8, (void*)p, 8, GEMM_ACC_F16, NULL) == GEMM_OK);
  CHECK(gemm_f16_last_launches() == 0);
  CHECK(strcmp(gemm_status_string(GEMM_ERR_MISALIGNED), "GEMM_ERR_MISALIGNED") == 0);
  int tm = 0, tn = 0, cg = 0, st = 0, sm = 0;
  CHECK(gemm_f16_config_info(GEMM_CFG_PAIR_256x256_K128, GEMM_ACC_F32, &tm, &tn, &cg, &st, &sm) == GEMM_OK);
  CHECK(tm == 256 && tn == 256 && cg == 2 && sm <= 232448);
  CHECK(gemm_f16_config_info(GEMM_CFG_COUNT, GEMM_ACC_F32, &tm, &tn, &cg, &st, &sm) == GEMM_ERR_INVALID_VALUE);
  gemm_options_t opt;
  memset(&opt, 0, sizeof opt);
  opt.config = 99;
  CHECK(gemm_f16_ex(8, 8, 8, p, 8, p, 8, (void*)p, 8, GEMM_ACC_F32, NULL, &opt) == GEMM_ERR_INVALID_VALUE ||
        gemm_f16_ex(8, 8, 8, p, 8, p, 8, (void*)p, 8, GEMM_ACC_F32, NULL, &opt) == GEMM_ERR_CUDA ||
        gemm_f16_ex(8, 8, 8, p, 8, p, 8, (void*)p, 8, GEMM_ACC_F32, NULL, &opt) == GEMM_ERR_UNSUPPORTED_DEVICE);
  return 0;
}

static int gpu_checks(void) {
  const int64_t M = 300, N = 264, K = 520;
  uint16_t* hA = (uint16_t*)malloc(M * K * 2);
  uint16_t* hB = (uint16_t*)malloc(K * N * 2);
  float* hC = (float*)malloc(M * N * 4);
  for (int64_t i = 0; i < M * K; ++i) hA[i] = 0x3C00; /* 1.0 in binary16 */
  for (int64_t i = 0; i < K * N; ++i) hB[i] = 0x3C00;
  for (int64_t i = 0; i < M * N; ++i) hC[i] = (float)(i % 7);
  void *dA, *dB, *dC;
  CHECK(cudaMalloc(&dA, M * K * 2) == 0 && cudaMalloc(&dB, K * N * 2) == 0 && cudaMalloc(&dC, M * N * 4) == 0);
  CHECK(cudaMemcpy(dA, hA, M * K * 2, 1) == 0 && cudaMemcpy(dB, hB, K * N * 2, 1) == 0 &&
        cudaMemcpy(dC, hC, M * N * 4, 1) == 0);
  CHECK(gemm_f16(M, N, K, dA, K, dB, N, dC, N, GEMM_ACC_F32, NULL) == GEMM_OK);
  CHECK(gemm_f16_last_launches() == 1);
  CHECK(cudaDeviceSynchronize() == 0);
  float* out = (float*)malloc(M * N * 4);
  CHECK(cudaMemcpy(out, dC, M * N * 4, 2) == 0);
  for (int64_t i = 0; i < M * N; ++i) CHECK(out[i] == (float)(i % 7) + (float)K);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  free(hA);
  free(hB);
  free(hC);
  free(out);
  return 0;
}

int main(int argc, char** argv) {
  if (cpu_checks()) return 1;
  if (argc > 1 && strcmp(argv[1], "gpu") == 0 && gpu_checks()) return 1;
  printf("c_abi_test OK%s\n", argc > 1 ? " (gpu)" : "");
  return 0;
}
