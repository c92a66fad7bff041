"""The boundary from C: a C99 program compiled with -Wall -Werror against include/fmm.h and linked
with libfmm.so calls the host-only entry points (no GPU needed) and checks their results -- the
header is valid C, the symbols resolve at link time, and the calls behave as documented."""
import os
import subprocess

import pytest

from conftest import ROOT

PROG = r'''
#include <stdio.h>
#include <string.h>
#include "fmm.h"
#define CHECK(c) do { if (!(c)) { printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); return 1; } } while (0)
int main(void) {
  fmm_alg* a = NULL;
  fmm_alg* t = NULL;
  int dims[4], nnz[3];
  double ms = 0.0;
  int used = -1;
  int64_t first = -1, last = -1, bfs = -1, dfs = -1;
  fmm_plan_options o;
  CHECK(fmm_version() != NULL && strlen(fmm_version()) > 0);
  CHECK(fmm_alg_load(ALGS "/winograd_class_222_7.txt", &a) == FMM_OK);
  CHECK(fmm_alg_info(a, dims, nnz) == FMM_OK);
  CHECK(dims[0] == 2 && dims[1] == 2 && dims[2] == 2 && dims[3] == 7);
  CHECK(fmm_alg_permute(a, 2, &t) == FMM_OK && fmm_alg_info(t, dims, nnz) == FMM_OK && dims[3] == 7);
  fmm_alg_destroy(t);
  CHECK(fmm_alg_load(ALGS "/no_such_file.txt", &t) != FMM_OK && strlen(fmm_last_error()) > 0);
  CHECK(fmm_plan_predict(a, 8192, 8192, 8192, 2, FMM_COL_MAJOR, &ms, &used) == FMM_OK && ms > 1.0 && used == 2);
  CHECK(fmm_plan_predict(a, -1, 8, 8, 1, FMM_ROW_MAJOR, &ms, &used) == FMM_E_SHAPE);
  fmm_plan_options_default(&o);
  CHECK(o.strategy == FMM_ADD_STREAMING && o.cse == 1 && o.collapse_levels == 1 && o.cuda_graphs == 1);
  CHECK(fmm_dist_slab(10, 4, FMM_ROW_MAJOR, 3, 2, &first, &last) == FMM_OK && first == 6 && last == 10);
  CHECK(fmm_hybrid_split(7, 2, 8, &bfs, &dfs) == FMM_OK && bfs == 48 && dfs == 1);
  fmm_alg_destroy(a);
  printf("OK\n");
  return 0;
}
'''


def test_c_program_against_the_header(tmp_path):
    import __graft_entry__
    __graft_entry__.build()
    src = tmp_path / "abi.c"
    src.write_text(PROG)
    exe = tmp_path / "abi"
    lib = os.path.join(ROOT, "paper_1409_2908_b200")
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", f"-I{os.path.join(ROOT, 'include')}",
           f'-DALGS="{os.path.join(ROOT, "algs")}"', str(src), "-o", str(exe), f"-L{lib}", "-lfmm",
           f"-Wl,-rpath,{lib}"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == "OK", r.stdout + r.stderr


GPU_PROG = r'''
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <cuda_runtime.h>
#include "fmm.h"
#define CHECK(c) do { if (!(c)) { printf("FAIL %s:%d %s [%s]\n", __FILE__, __LINE__, #c, fmm_last_error()); return 1; } } while (0)

static double* load(const char* path, size_t n) {
  double* x = (double*)malloc(n * sizeof(double));
  FILE* f = fopen(path, "rb");
  if (!f || !x || fread(x, sizeof(double), n, f) != n) { printf("cannot read %s\n", path); exit(2); }
  fclose(f);
  return x;
}

/* max |C - ref| over the logical P x N matrix; C stored row- (col = 0) or column-major with ldc */
static double maxdiff(const double* C, int64_t ldc, int col, const double* ref, int64_t P, int64_t N) {
  double m = 0.0;
  for (int64_t i = 0; i < P; ++i)
    for (int64_t j = 0; j < N; ++j) {
      const double v = col ? C[j * ldc + i] : C[i * ldc + j];
      const double d = fabs(v - ref[i * N + j]);
      if (!(d <= m)) m = d;  /* NaN propagates */
    }
  return m;
}

/* case: alg file, L, P, Q, N, layout (0 row / 1 col), inputs and the oracle's C in dir/<tag>.{A,B,C} */
static int run_case(const char* dir, const char* tag, const char* algfile, int L, int64_t P, int64_t Q, int64_t N, int col,
                    double tol) {
  char path[1024];
  snprintf(path, sizeof path, "%s/%s.A", dir, tag);
  double* A = load(path, (size_t)(P * Q));
  snprintf(path, sizeof path, "%s/%s.B", dir, tag);
  double* B = load(path, (size_t)(Q * N));
  snprintf(path, sizeof path, "%s/%s.C", dir, tag);
  double* ref = load(path, (size_t)(P * N));
  /* storage with padded leading dimensions: row-major lda = Q + 3 ..., column-major lda = P + 5 ... */
  const int64_t lda = col ? P + 5 : Q + 3, ldb = col ? Q + 1 : N + 7, ldc = col ? P + 2 : N + 1;
  const size_t na = (size_t)(lda * (col ? Q : P)), nb = (size_t)(ldb * (col ? N : Q)), nc = (size_t)(ldc * (col ? N : P));
  double* hA = (double*)calloc(na, sizeof(double));
  double* hB = (double*)calloc(nb, sizeof(double));
  double* hC = (double*)calloc(nc, sizeof(double));
  for (int64_t i = 0; i < P; ++i)
    for (int64_t j = 0; j < Q; ++j) hA[col ? j * lda + i : i * lda + j] = A[i * Q + j];
  for (int64_t i = 0; i < Q; ++i)
    for (int64_t j = 0; j < N; ++j) hB[col ? j * ldb + i : i * ldb + j] = B[i * N + j];
  fmm_alg* alg = NULL;
  CHECK(fmm_alg_load(algfile, &alg) == FMM_OK);
  fmm_plan_options o;
  fmm_plan_options_default(&o);
  o.layout = col ? FMM_COL_MAJOR : FMM_ROW_MAJOR;
  fmm_plan_t* plan = NULL;
  CHECK(fmm_plan_create(alg, P, Q, N, L, &o, 0, &plan) == FMM_OK);
  /* device path: cudaMalloc'd A, B, C, fmm_execute on a stream, twice (the second replays the graph) */
  double *dA = NULL, *dB = NULL, *dC = NULL;
  CHECK(cudaMalloc((void**)&dA, na * 8) == cudaSuccess && cudaMalloc((void**)&dB, nb * 8) == cudaSuccess &&
        cudaMalloc((void**)&dC, nc * 8) == cudaSuccess);
  CHECK(cudaMemcpy(dA, hA, na * 8, cudaMemcpyHostToDevice) == cudaSuccess);
  CHECK(cudaMemcpy(dB, hB, nb * 8, cudaMemcpyHostToDevice) == cudaSuccess);
  cudaStream_t s;
  CHECK(cudaStreamCreate(&s) == cudaSuccess);
  for (int it = 0; it < 3; ++it) {
    CHECK(cudaMemset(dC, 0xff, nc * 8) == cudaSuccess);  /* NaN pattern: every entry must be written */
    CHECK(fmm_execute(plan, dA, lda, dB, ldb, dC, ldc, (void*)s) == FMM_OK);
    CHECK(fmm_sync(plan) == FMM_OK && cudaStreamSynchronize(s) == cudaSuccess);
    CHECK(cudaMemcpy(hC, dC, nc * 8, cudaMemcpyDeviceToHost) == cudaSuccess);
    const double d = maxdiff(hC, ldc, col, ref, P, N);
    printf("%s fmm_execute[%d]: max|C - C_oracle| = %.3e (tol %.3e)\n", tag, it, d, tol);
    CHECK(d <= tol);
  }
  /* host path: fmm_execute_host (copies inside the library) into a fresh host C */
  memset(hC, 0xff, nc * 8);
  CHECK(fmm_execute_host(plan, hA, lda, hB, ldb, hC, ldc, (void*)s) == FMM_OK);
  const double dh = maxdiff(hC, ldc, col, ref, P, N);
  printf("%s fmm_execute_host: max|C - C_oracle| = %.3e\n", tag, dh);
  CHECK(dh <= tol);
  /* errors are reported before any device work: a too-small leading dimension */
  CHECK(fmm_execute(plan, dA, 1, dB, ldb, dC, ldc, (void*)s) == FMM_E_SHAPE && strlen(fmm_last_error()) > 0);
  fmm_plan_destroy(plan);
  fmm_alg_destroy(alg);
  cudaFree(dA); cudaFree(dB); cudaFree(dC);
  cudaStreamDestroy(s);
  free(A); free(B); free(ref); free(hA); free(hB); free(hC);
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  const char* dir = argv[1];
  const char* algs = argv[2];
  char f[1024];
  int rc = 0;
  snprintf(f, sizeof f, "%s/strassen_222_7.txt", algs);
  rc |= run_case(dir, "c1", f, 1, 256, 256, 256, 0, atof(argv[3]));
  snprintf(f, sizeof f, "%s/hk_class_323_15.txt", algs);
  rc |= run_case(dir, "peel", f, 2, 301, 199, 257, 1, atof(argv[4]));
  if (rc) return rc;
  /* the north-star spellings: fmm_plan(alg, M, K, N, levels) and fmm_exec(plan, A, B, C) */
  {
    fmm_alg* a = NULL;
    fmm_plan_t* p = NULL;
    snprintf(f, sizeof f, "%s/strassen_222_7.txt", algs);
    CHECK(fmm_alg_load(f, &a) == FMM_OK && fmm_plan(a, 64, 64, 64, 1, &p) == FMM_OK);
    double *dA, *dB, *dC;
    double h[64 * 64], c[64 * 64];
    for (int i = 0; i < 64 * 64; ++i) h[i] = (double)((i * 7) % 5 - 2);
    CHECK(cudaMalloc((void**)&dA, sizeof h) == cudaSuccess && cudaMalloc((void**)&dB, sizeof h) == cudaSuccess &&
          cudaMalloc((void**)&dC, sizeof h) == cudaSuccess);
    cudaMemcpy(dA, h, sizeof h, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, h, sizeof h, cudaMemcpyHostToDevice);
    CHECK(fmm_exec(p, dA, dB, dC) == FMM_OK && cudaDeviceSynchronize() == cudaSuccess);
    cudaMemcpy(c, dC, sizeof c, cudaMemcpyDeviceToHost);
    for (int i = 0; i < 64; ++i)
      for (int j = 0; j < 64; ++j) {
        double acc = 0.0;  /* small integers: exact in any order */
        for (int q = 0; q < 64; ++q) acc += h[i * 64 + q] * h[q * 64 + j];
        CHECK(c[i * 64 + j] == acc);
      }
    fmm_plan_destroy(p);
    fmm_alg_destroy(a);
    cudaFree(dA); cudaFree(dB); cudaFree(dC);
  }
  printf("OK\n");
  return 0;
}
'''


@pytest.mark.gpu
def test_c_program_executes_on_the_gpu(tmp_path):
    # the boundary from C on the device: cudaMalloc'd buffers through fmm_plan_create / fmm_execute /
    # fmm_execute_host (c1: Strassen L = 1, 256^3 row-major; a peeled <3,2,3;15> L = 2 column-major
    # problem with padded leading dimensions), each checked against the oracle's C written here
    import numpy as np
    import __graft_entry__
    import fmm_inputs as I
    from oracle import oracle as O
    __graft_entry__.build()
    tols = []
    for tag, alg, L, (P, Q, N) in (("c1", "strassen_222_7", 1, (256, 256, 256)),
                                   ("peel", "hk_class_323_15", 2, (301, 199, 257))):
        A, B = I.problem(P, Q, N, seed=41)
        ref = O.fast(A, B, O.load_alg(os.path.join(ROOT, "algs", alg + ".txt")), L)
        for ext, x in (("A", A), ("B", B), ("C", ref)):
            np.ascontiguousarray(x, dtype=np.float64).tofile(str(tmp_path / f"{tag}.{ext}"))
        tols.append(1e-12 * np.linalg.norm(A) * np.linalg.norm(B))  # the north-star parity bound
    src = tmp_path / "gpu_abi.c"
    src.write_text(GPU_PROG)
    exe = tmp_path / "gpu_abi"
    lib = os.path.join(ROOT, "paper_1409_2908_b200")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    cmd = ["gcc", "-std=c99", "-Wall", "-Wextra", "-Werror", f"-I{os.path.join(ROOT, 'include')}",
           f"-I{cuda}/include", str(src), "-o", str(exe), f"-L{lib}", "-lfmm", f"-Wl,-rpath,{lib}",
           f"-L{cuda}/lib64", "-lcudart", f"-Wl,-rpath,{cuda}/lib64", "-lm"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe), str(tmp_path), os.path.join(ROOT, "algs"), "%.17g" % tols[0], "%.17g" % tols[1]],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr
