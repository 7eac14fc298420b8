/*
 * c_abi_demo.c -- the C ABI from plain C (no Python, no torch): synthesise a small
 * bf16 batch on the device, prove it, verify it against a jittered copy and print the
 * proof bytes' FNV-1a hash and the verdicts.  tests/test_c_abi.py builds and runs it
 * and checks the output against the Python path.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_demo.c \
 *       -L paper_2505_07291_b200/_lib -ltoploc_b200 -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2505_07291_b200/_lib -o c_abi_demo
 */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "toploc_b200.h"

#define CK(x) do { int rc_ = (int)(x); if (rc_) { fprintf(stderr, "%s -> %d (%s)\n", #x, rc_, \
                     rc_ < 0 ? tl_strerror(rc_) : cudaGetErrorString((cudaError_t)rc_)); return 1; } } while (0)

int main(int argc, char** argv) {
  const int32_t H = argc > 1 ? atoi(argv[1]) : 1024;
  const int64_t row_off_host[4] = {0, 70, 128, 300};   /* three rollouts, the last ragged */
  const int32_t n_roll = 3, C = 32, K = 128;
  const int64_t n_rows = row_off_host[n_roll];
  const int64_t n_chunks = tl_count_chunks(row_off_host, n_roll, C);
  const int PB = TL_PROOF_BYTES(K);
  uint16_t *prv, *val, *table;
  int64_t* row_off;
  uint8_t *proofs, *accept;
  void* ws;
  const size_t ws_bytes = tl_workspace_bytes(n_roll, n_chunks, K);
  CK(cudaMalloc((void**)&prv, n_rows * H * 2));
  CK(cudaMalloc((void**)&val, n_rows * H * 2));
  CK(cudaMalloc((void**)&row_off, sizeof(row_off_host)));
  CK(cudaMalloc((void**)&proofs, n_chunks * PB));
  CK(cudaMalloc((void**)&accept, n_roll));
  CK(cudaMalloc(&ws, ws_bytes));
  CK(cudaMemcpy(row_off, row_off_host, sizeof(row_off_host), cudaMemcpyHostToDevice));
  /* inverse-normal table for the synthetic generator: any monotone table works for a
   * demo; use the identity bit pattern ramp of small bf16 magnitudes */
  uint16_t* tab_host = (uint16_t*)malloc(65536 * 2);
  for (int i = 0; i < 65536; ++i) tab_host[i] = (uint16_t)(0x3000 + (i >> 4));
  CK(cudaMalloc((void**)&table, 65536 * 2));
  CK(cudaMemcpy(table, tab_host, 65536 * 2, cudaMemcpyHostToDevice));
  CK(tl_synth_bf16(prv, 0, n_rows, H, 0x1234567ull, 0, table, NULL, 0, 0, NULL));
  CK(tl_synth_bf16(val, 0, n_rows, H, 0x1234567ull, 0, table, NULL, 3277, 0x99ull, NULL));

  CK(tl_prove(prv, row_off, n_roll, n_rows, H, C, K, n_chunks, proofs, NULL, NULL, ws, ws_bytes, NULL));
  const tl_thresholds th = {38, 0, 10.0, 8.0};
  CK(tl_verify(val, row_off, n_roll, n_rows, H, C, K, n_chunks, proofs, &th, NULL, NULL, accept, ws, ws_bytes,
               NULL));
  CK(cudaDeviceSynchronize());

  uint8_t* host = (uint8_t*)malloc(n_chunks * PB);
  uint8_t acc_host[3];
  CK(cudaMemcpy(host, proofs, n_chunks * PB, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(acc_host, accept, n_roll, cudaMemcpyDeviceToHost));
  uint64_t h = 1469598103934665603ull;
  for (int64_t i = 0; i < n_chunks * PB; ++i) h = (h ^ host[i]) * 1099511628211ull;
  printf("chunks %lld proof_fnv1a %016llx verdicts %d %d %d\n", (long long)n_chunks, (unsigned long long)h,
         acc_host[0], acc_host[1], acc_host[2]);
  return 0;
}
