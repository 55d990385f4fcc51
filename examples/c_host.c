/*
 * A non-Python host of the PbP-QLP boundary: plain C against include/pbq.h
 * and the CUDA runtime, no Python anywhere.  This is the call sequence a
 * cgo/JNI/N-API binding would wrap.
 *
 *   usage: c_host A.bin n1 n2 d q seed out.bin
 *
 * A.bin holds n1·n2 float64 (row-major).  out.bin receives, in order:
 * the status word, the 2q+1 rank flags (int32), then Q (n1×d), L (d×d),
 * P (n2×d), R (d×d) as dense row-major float64, then Φ (n1×d).
 * Exit code: 0 ok, otherwise the pbq_status / 100 + CUDA error.
 */
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pbq.h"

#define CK(call)                                                                  \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess) {                                                      \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
      return 100 + (int)e_;                                                       \
    }                                                                             \
  } while (0)

static int64_t even(int64_t n) { return n + (n & 1); }

/* device matrix with an even row stride; host copies go through cudaMemcpy2D */
static int dmalloc(double** p, int64_t rows, int64_t cols, int64_t* ld) {
  *ld = even(cols);
  return cudaMalloc((void**)p, (size_t)rows * (size_t)(*ld) * sizeof(double)) == cudaSuccess ? 0 : 1;
}

static int pull(FILE* f, const double* d, int64_t rows, int64_t cols, int64_t ld) {
  double* h = (double*)malloc((size_t)rows * (size_t)cols * sizeof(double));
  if (!h) return 1;
  CK(cudaMemcpy2D(h, (size_t)cols * 8, d, (size_t)ld * 8, (size_t)cols * 8, (size_t)rows, cudaMemcpyDeviceToHost));
  fwrite(h, sizeof(double), (size_t)rows * (size_t)cols, f);
  free(h);
  return 0;
}

int main(int argc, char** argv) {
  if (argc != 8) {
    fprintf(stderr, "usage: %s A.bin n1 n2 d q seed out.bin\n", argv[0]);
    return 2;
  }
  const int64_t n1 = atoll(argv[2]), n2 = atoll(argv[3]), d = atoll(argv[4]), q = atoll(argv[5]);
  const uint64_t seed = strtoull(argv[6], NULL, 10);
  double* ha = (double*)malloc((size_t)(n1 * n2) * sizeof(double));
  FILE* fa = fopen(argv[1], "rb");
  if (!ha || !fa || fread(ha, sizeof(double), (size_t)(n1 * n2), fa) != (size_t)(n1 * n2)) {
    fprintf(stderr, "cannot read %s\n", argv[1]);
    return 2;
  }
  fclose(fa);

  pbq_ctx* ctx = NULL;
  int st = pbq_ctx_create(0, &ctx);
  if (st != PBQ_OK) {
    fprintf(stderr, "pbq_ctx_create: %d\n", st);
    return st;
  }
  cudaStream_t stream;
  CK(cudaStreamCreate(&stream));

  double *A, *Q, *L, *P, *R, *Phi;
  int64_t lda, ldq, ldl, ldp, ldr, ldphi;
  if (dmalloc(&A, n1, n2, &lda) || dmalloc(&Q, n1, d, &ldq) || dmalloc(&L, d, d, &ldl) || dmalloc(&P, n2, d, &ldp) ||
      dmalloc(&R, d, d, &ldr) || dmalloc(&Phi, n1, d, &ldphi))
    return 106;
  CK(cudaMemcpy2D(A, (size_t)lda * 8, ha, (size_t)n2 * 8, (size_t)n2 * 8, (size_t)n1, cudaMemcpyHostToDevice));
  int32_t *flags, *status;
  CK(cudaMalloc((void**)&flags, sizeof(int32_t) * (size_t)(2 * q + 1)));
  CK(cudaMalloc((void**)&status, sizeof(int32_t)));

  pbq_problem prob;
  memset(&prob, 0, sizeof(prob));
  prob.n1 = n1; prob.n2 = n2; prob.d = d; prob.q = q;
  prob.a = A; prob.lda = lda;
  prob.phi = NULL;  /* seeded mode: the library draws Φ = numpy Philox(key=seed).standard_normal((n1, d)) */
  prob.seed_lo = seed; prob.seed_hi = 0;
  prob.reorthonormalize = 1;
  prob.check_finite = 1;
  pbq_outputs out;
  memset(&out, 0, sizeof(out));
  out.q = Q; out.ldq = ldq; out.l = L; out.ldl = ldl; out.p = P; out.ldp = ldp; out.r = R; out.ldr = ldr;
  out.phi = Phi; out.ldphi = ldphi;
  out.rank_flags = flags; out.nonfinite = status;

  size_t ws_bytes = 0;
  st = pbq_pbp_qlp_workspace_bytes(ctx, &prob, &ws_bytes);
  if (st != PBQ_OK) {
    fprintf(stderr, "workspace: %d %s\n", st, pbq_last_error(ctx));
    return st;
  }
  void* ws;
  CK(cudaMalloc(&ws, ws_bytes));
  st = pbq_pbp_qlp(ctx, &prob, &out, ws, ws_bytes, (void*)stream);
  if (st != PBQ_OK) {
    fprintf(stderr, "pbq_pbp_qlp: %d %s\n", st, pbq_last_error(ctx));
    return st;
  }
  CK(cudaStreamSynchronize(stream));

  int32_t hstatus, hflags[64];
  CK(cudaMemcpy(&hstatus, status, sizeof(int32_t), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(hflags, flags, sizeof(int32_t) * (size_t)(2 * q + 1), cudaMemcpyDeviceToHost));
  FILE* fo = fopen(argv[7], "wb");
  if (!fo) return 2;
  fwrite(&hstatus, sizeof(int32_t), 1, fo);
  fwrite(hflags, sizeof(int32_t), (size_t)(2 * q + 1), fo);
  if (pull(fo, Q, n1, d, ldq) || pull(fo, L, d, d, ldl) || pull(fo, P, n2, d, ldp) || pull(fo, R, d, d, ldr) ||
      pull(fo, Phi, n1, d, ldphi))
    return 107;
  fclose(fo);
  printf("pbq_pbp_qlp ok: %lld launches, status %d\n", (long long)pbq_ctx_launch_count(ctx), hstatus);
  cudaFree(ws);
  pbq_ctx_destroy(ctx);
  free(ha);
  return 0;
}
