/* A plain-C caller of the drop-in boundary (include/tpf.h): reads a model and
 * loads from binary files, runs tpf_dense_solve_host_c128 on host buffers and
 * writes V, the per-case counts and the summary.  Used by
 * tests/test_c_abi_gpu.py (built there with gcc against libtpf.so). */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "tpf.h"

static void* slurp(const char* path, size_t* n) {
  FILE* f = fopen(path, "rb");
  if (!f) return NULL;
  fseek(f, 0, SEEK_END);
  *n = (size_t)ftell(f);
  fseek(f, 0, SEEK_SET);
  void* p = malloc(*n ? *n : 1);
  if (fread(p, 1, *n, f) != *n) {
    fclose(f);
    free(p);
    return NULL;
  }
  fclose(f);
  return p;
}

int main(int argc, char** argv) {
  if (argc != 3) {
    fprintf(stderr, "usage: %s <in_dir> <out_dir>\n", argv[0]);
    return 2;
  }
  char path[4096];
  size_t n;
  int64_t dims[2];  /* b, tau */
  snprintf(path, sizeof path, "%s/dims.bin", argv[1]);
  int64_t* d = (int64_t*)slurp(path, &n);
  if (!d) return 3;
  dims[0] = d[0];
  dims[1] = d[1];
  const int32_t b = (int32_t)dims[0];
  const int64_t tau = dims[1];
  const char* names[] = {"K", "W", "rp", "ci", "yv", "src", "S", "vflat"};
  void* buf[8];
  for (int i = 0; i < 8; ++i) {
    snprintf(path, sizeof path, "%s/%s.bin", argv[1], names[i]);
    buf[i] = slurp(path, &n);
    if (!buf[i]) return 4;
  }
  const double* vflat = (const double*)buf[7];
  double* V = (double*)malloc((size_t)b * (size_t)tau * 16);
  int32_t* iters = (int32_t*)malloc((size_t)tau * 4);
  double* resid = (double*)malloc((size_t)tau * 8);
  uint8_t* mask = (uint8_t*)malloc((size_t)tau);
  int32_t summary[2];
  int rc = tpf_dense_solve_host_c128(tau, b, (const double*)buf[6], tau, 1, (const double*)buf[0],
                                     (const double*)buf[1], (const int32_t*)buf[2], (const int32_t*)buf[3],
                                     (const double*)buf[4], (const double*)buf[5], vflat[0], vflat[1], 1e-10, 100,
                                     1e-8, V, tau, 1, iters, resid, mask, summary, 0, 0, NULL, 0);
  if (rc != TPF_OK) {
    fprintf(stderr, "tpf_dense_solve_host_c128: %s\n", tpf_last_error());
    return 5;
  }
  snprintf(path, sizeof path, "%s/V.bin", argv[2]);
  FILE* f = fopen(path, "wb");
  fwrite(V, 16, (size_t)b * (size_t)tau, f);
  fclose(f);
  snprintf(path, sizeof path, "%s/iters.bin", argv[2]);
  f = fopen(path, "wb");
  fwrite(iters, 4, (size_t)tau, f);
  fclose(f);
  printf("%d %d\n", summary[0], summary[1]);
  return 0;
}
