/* cpa_c_smoke.c -- the C ABI (include/cpa.h) driven from plain C, no Python or torch: device buffers
 * from cudaMalloc, one cpa_chunk_step (estimator -> tables -> paged attention) on
 * inputs written by tests/test_c_abi.py (seeded synth workload) next to the fp64 oracle's tables and
 * outputs; checks the tables bit for bit and the outputs within 1e-2 x RMS (north_star tolerance).
 *   cpa_c_smoke <dir>     files: meta.txt q.bin k.bin v.bin pt.bin ip.bin ix.bin o.bin
 * Exit 0 on success; prints one line. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "cpa.h"

static void* load(const char* dir, const char* name, size_t* bytes) {
  char path[4096];
  snprintf(path, sizeof path, "%s/%s", dir, name);
  FILE* f = fopen(path, "rb");
  if (!f) { fprintf(stderr, "cannot open %s\n", path); exit(2); }
  fseek(f, 0, SEEK_END);
  long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  void* buf = malloc(n > 0 ? (size_t)n : 1);
  if (n > 0 && fread(buf, 1, (size_t)n, f) != (size_t)n) { fprintf(stderr, "short read %s\n", path); exit(2); }
  fclose(f);
  *bytes = (size_t)n;
  return buf;
}

static void* to_dev(const void* h, size_t bytes) {
  void* d = NULL;
  if (cudaMalloc(&d, bytes ? bytes : 4) != cudaSuccess) { fprintf(stderr, "cudaMalloc failed\n"); exit(3); }
  if (bytes && cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice) != cudaSuccess) { fprintf(stderr, "H2D failed\n"); exit(3); }
  return d;
}

int main(int argc, char** argv) {
  if (argc < 2) { fprintf(stderr, "usage: %s <dir>\n", argv[0]); return 2; }
  const char* dir = argv[1];
  char mpath[4096];
  snprintf(mpath, sizeof mpath, "%s/meta.txt", dir);
  FILE* mf = fopen(mpath, "r");
  if (!mf) { fprintf(stderr, "no meta.txt\n"); return 2; }
  int B, Hq, Hkv, d, bs, C, P, num_pages, max_blocks;
  float alpha;
  if (fscanf(mf, "%d %d %d %d %d %d %d %d %d %f", &B, &Hq, &Hkv, &d, &bs, &C, &P, &num_pages, &max_blocks, &alpha) != 10) {
    fprintf(stderr, "bad meta.txt\n");
    return 2;
  }
  fclose(mf);
  size_t nq, nk, nv, npt, nip, nix, no;
  void* q = load(dir, "q.bin", &nq);
  void* k = load(dir, "k.bin", &nk);
  void* v = load(dir, "v.bin", &nv);
  int32_t* pt = (int32_t*)load(dir, "pt.bin", &npt);
  int32_t* ip_ref = (int32_t*)load(dir, "ip.bin", &nip);
  int32_t* ix_ref = (int32_t*)load(dir, "ix.bin", &nix);
  double* o_ref = (double*)load(dir, "o.bin", &no);

  cpa_params p;
  memset(&p, 0, sizeof p);
  p.batch = B; p.num_q_heads = Hq; p.num_kv_heads = Hkv; p.head_dim = d; p.block_size = bs;
  p.chunk_len = C; p.prefix_len = P; p.alpha = alpha;
  p.flags = CPA_F_SINK | CPA_F_OUT_F32;
  const int L = P + C, nkvb = (L + bs - 1) / bs, Gn = Hq / (Hq / Hkv);

  cpa_kv_cache cache;
  memset(&cache, 0, sizeof cache);
  cache.k_pages = to_dev(k, nk);
  cache.v_pages = to_dev(v, nv);
  cache.page_table = (const int32_t*)to_dev(pt, npt);
  cache.max_blocks_per_seq = max_blocks;
  cache.num_pages = num_pages;

  cpa_tables t;
  memset(&t, 0, sizeof t);
  t.capacity = (int64_t)B * Gn * nkvb;
  cudaMalloc((void**)&t.kv_indptr, sizeof(int32_t) * (size_t)(B * Gn + 1));
  cudaMalloc((void**)&t.kv_indices, sizeof(int32_t) * (size_t)t.capacity);

  const size_t n_out = (size_t)B * C * Hq * d;
  void* dq = to_dev(q, nq);
  float* dout = NULL;
  cudaMalloc((void**)&dout, n_out * sizeof(float));
  const size_t wsb = cpa_workspace_bytes(&p);
  void* ws = NULL;
  cudaMalloc(&ws, wsb ? wsb : 256);

  int rc = cpa_chunk_step(&p, dq, NULL, NULL, &cache, &t, dout, ws, wsb, NULL);
  if (rc != CPA_OK) { fprintf(stderr, "cpa_chunk_step: %s (%s)\n", cpa_status_string(rc), cpa_last_error()); return 4; }
  if (cudaDeviceSynchronize() != cudaSuccess) { fprintf(stderr, "device fault\n"); return 4; }

  /* a 16-byte workspace is rejected synchronously (CPA_ERR_WORKSPACE) */
  rc = cpa_chunk_step(&p, dq, NULL, NULL, &cache, &t, dout, ws, 16, NULL);
  if (rc != CPA_ERR_WORKSPACE) { fprintf(stderr, "undersized workspace not rejected: %d\n", rc); return 5; }

  const int rows = B * Gn;
  int32_t* ip = (int32_t*)malloc(sizeof(int32_t) * (size_t)(rows + 1));
  cudaMemcpy(ip, t.kv_indptr, sizeof(int32_t) * (size_t)(rows + 1), cudaMemcpyDeviceToHost);
  if (nip != sizeof(int32_t) * (size_t)(rows + 1) || memcmp(ip, ip_ref, nip) != 0) { fprintf(stderr, "kv_indptr differs\n"); return 6; }
  int32_t* ix = (int32_t*)malloc(nix ? nix : 4);
  cudaMemcpy(ix, t.kv_indices, nix, cudaMemcpyDeviceToHost);
  if ((size_t)ip[rows] * sizeof(int32_t) != nix || memcmp(ix, ix_ref, nix) != 0) { fprintf(stderr, "kv_indices differ\n"); return 6; }

  float* out = (float*)malloc(n_out * sizeof(float));
  cudaMemcpy(out, dout, n_out * sizeof(float), cudaMemcpyDeviceToHost);
  if (no != n_out * sizeof(double)) { fprintf(stderr, "o.bin size\n"); return 2; }
  double ss = 0.0, maxd = 0.0;
  for (size_t i = 0; i < n_out; ++i) ss += o_ref[i] * o_ref[i];
  const double rms = sqrt(ss / (double)n_out);
  for (size_t i = 0; i < n_out; ++i) {
    const double e = fabs((double)out[i] - o_ref[i]);
    if (!(e <= maxd)) maxd = e;  /* NaN-propagating */
  }
  const double rel = maxd / rms;
  printf("c abi ok=%d: tables bit-exact (%d blocks), max|d|/rms = %.3e, workspace %zu bytes\n", rel <= 1e-2, ip[rows],
         rel, wsb);
  return rel <= 1e-2 ? 0 : 7;
}
