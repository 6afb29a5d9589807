// K1 matrix-free space-time operator (see pd_stencil.cu).
#pragma once

#include <vector>

#include "pd_internal.h"

namespace pd {

constexpr int kStMaxM = 9;
constexpr int kGridMaxTabHost = kStMaxM * kStMaxM * 7 + kStMaxM;
constexpr int kGridMaxBlocks = 65536;

struct StOp {
    Ctx& c;
    int64_t Nt, M, S;
    double dt;
    double Kq[kStMaxM * kStMaxM], Mq[kStMaxM * kStMaxM], l0[kStMaxM];
    std::unique_ptr<Csr> Kh;
    DevBuf<double> mh;
    DevBuf<double> coef;  // one time block of Aqh values, [m][m'][p of Kh] (L2-resident)
    int64_t nnzK = 0;
    // structured-grid mode (Dirichlet constant-coefficient stencil on n^dim)
    int grid_dim = 0, grid_n = 0;
    DevBuf<double> grid_tab;  // [m][m'][position] + step coupling per m
    std::vector<double> grid_tab_host;  // the same table on the host (kernel parameters)
    DevBuf<double> grid_partials;  // fused-norm per-block partials (grid_blocks_max)
    int64_t grid_blocks_max = 0;
    bool grid_periodic = false;  // 2D periodic 5-point stencil (wrapped neighbours)
    DevBuf<unsigned int> grid_counter;
    StOp(Ctx& c, int64_t Nt, int M, int64_t S, const double* Kq, const double* Mq,
         const double* l0, double dt, const Csr& Kh, const double* mh_host);
    int64_t size() const { return Nt * M * S; }
    // same contract as csr_spmv (modes 0/1/2, guard, fused |y|^2, non-finite flag on x)
    void apply(const double* x, double* y, int mode, const double* b, const int* guard = nullptr,
               int want = 0, double* norm2_out = nullptr, int* nonfinite = nullptr,
               const double* halo = nullptr) const;
    void residual(const double* u, const double* rhs, double* out, double gamma, int kind) const;
    void detect_grid(const std::vector<int64_t>& rp, const double* mh_host);
};

// Kh a Dirichlet constant-coefficient (2d+1)-point stencil on n^d (d = 2, 3)?
// tv = the value per stencil position in CSR column order; jc = a full row.
bool detect_dirichlet_stencil(const Csr& K, int& dim, int& n, double tv[7], int64_t& jc);

// y = A x through the structured operator when present, else the CSR
inline void apply_A(Ctx& c, const Csr& A, const StOp* op, const double* x, double* y, int mode,
                    const double* b, const int* guard = nullptr, int want = 0,
                    double* norm2 = nullptr, int* nonfinite = nullptr) {
    if (op) op->apply(x, y, mode, b, guard, want, norm2, nonfinite);
    else csr_spmv(c, A, x, y, mode, b, guard, want, norm2, nonfinite);
}

}  // namespace pd
