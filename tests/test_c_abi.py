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
