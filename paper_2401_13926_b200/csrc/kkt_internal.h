// Internal (C++) view of the host analysis shared by analyze.cpp and device.cu.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/kktb200.h"

#define KKT_ABI_VERSION 4

namespace kkt {

// Mirror of LuFactors (direct_lu.py:51-81), int64 on the host like numpy.
struct Symbolic {
  int64_t n = 0;
  int64_t nnz_a = 0;
  std::vector<int64_t> A_row_ptr, A_col_idx;  // the general pattern analysed
  std::vector<int64_t> row_perm, col_perm;
  std::vector<int64_t> Lp, Li, Up, Ui;
  std::vector<double> Lx, Ux, Udiag;
  std::vector<int64_t> so_ptr, so_data;
  std::vector<int64_t> ap_ptr, a_src, a_tgt;
  double diag[4] = {0, 0, 0, 0};
  int64_t stats[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
};

extern thread_local std::string g_last_error;
int set_error(int code, const std::string &msg);
void min_degree(int64_t n, const int64_t *rp, const int64_t *ci, std::vector<int64_t> &order);
int analyze(int64_t n, const int64_t *rp, const int64_t *ci, const double *av, double pivot_tol,
            Symbolic &S);
void compute_schedule_stats(Symbolic &S);

}  // namespace kkt
