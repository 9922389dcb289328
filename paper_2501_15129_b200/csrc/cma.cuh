// cma.cuh -- CMA-ES device kernels: the ask GEMM,
// the rank-mu covariance GEMM with the C blend fused into its epilogue, the
// CSA-path GEMVs, and a blocked Jacobi symmetric eigensolver.
#pragma once

#include "common.cuh"

namespace evorl_b200 {

// C[m][n] epilogues of the NT GEMM  acc[m][n] = sum_k A[m*lda+k] * B[n*ldb+k]
enum : int { GEMM_STORE = 0, GEMM_ASK = 1, GEMM_RANKMU = 2 };
struct GemmEpi {
  int mode;
  double* out;
  long long ldo;
  // GEMM_ASK: out = acc * sigma + mean[n]   (proj/src/ec.cpp:230-232)
  double sigma;
  const double* mean;
  // GEMM_RANKMU: out = ((a*C) + (c1*((pc[m]*pc[n]) + (dh*C)))) + (cmu*acc)
  //              (proj/src/ec.cpp:264-271)
  const double* Cold;
  const double* pc;
  double a, c1, dh, cmu;
};
cudaError_t run_gemm_nt(int M, int N, int K, const double* A, long long lda, const double* B,
                        long long ldb, const GemmEpi& epi, cudaStream_t s);

struct CmaDev {
  int d, dp;            // dimension and padded dimension (multiple of 64)
  double* C;            // dp x dp, symmetric
  double* B;            // dp x dp, row-major: B[p*dp + j] = component p of eigenvector j
  double* D;            // d
  double* ps;           // d
  double* pc;           // d
  double* W;            // dp x dp Jacobi work (A)
  double* V;            // dp x dp Jacobi rotations
  double* Bt;           // dp x dp scratch (warm start)
  double* Tt;           // dp x dp scratch (warm start)
  double* U;            // (dp/64) * 64 * 64: per-pair 64x64 rotations
  int* skipf;           // dp/64: pair skipped this round (identity rotation)
  double* evals;        // dp
  int* order;           // dp
  double* zD;           // n x d
  double* ytT;          // d x mu   (y_top transposed)
  double* wyT;          // d x mu   (w_i * y_top)
  double* yw;           // d
  double* t1;           // d
  double* cih;          // d
  double* red;          // reduction scratch (>= 4)
};

cudaError_t run_cma_zD(DKey key, int n, int d, const double* D, double* zD, cudaStream_t s);
cudaError_t run_cma_ytop(const double* cand, const int* order, int mu, int d, const double* mean, double sigma,
                         const double* w, double* ytT, double* wyT, cudaStream_t s);
cudaError_t run_cma_yw_mean(const double* ytT, const double* w, int mu, int d, double sigma, double* yw,
                            double* mean, cudaStream_t s);
// t1[j] = (sum_p B[p][j] * yw[p]) / max(D[j], 1e-300)
cudaError_t run_cma_gemv_t(const double* B, int dp, int d, const double* yw, const double* D, double* t1,
                           cudaStream_t s);
// out[p] = sum_j B[p][j] * v[j]
cudaError_t run_cma_gemv(const double* B, int dp, int d, const double* v, double* out, cudaStream_t s);
// ps = (1-cs) ps + cps * cih ; red[0] = ||ps||^2 (fixed order)
cudaError_t run_cma_ps(double* ps, const double* cih, int d, double cs, double cps, double* red,
                       cudaStream_t s);
// pc = (1-cc) pc + cpc * yw
cudaError_t run_cma_pc(double* pc, const double* yw, int d, double cc, double cpc, cudaStream_t s);
// C = 0.5 (T + T^T) over the d x d block (padding untouched)
cudaError_t run_cma_symmetrize(const double* T, double* C, int d, int dp, cudaStream_t s);
// D = sqrt(max(ev, 0)) (proj/src/ec.cpp:287)
cudaError_t run_cma_sqrt_pos(const double* ev, double* D, int d, cudaStream_t s);
// C[i][i] += v for i < d
cudaError_t run_cma_add_diag(double* C, int d, int dp, double v, cudaStream_t s);

// Symmetric eigendecomposition of the leading d x d block of A (dp x dp):
// evals ascending (d of them), vecs[p*dp + j] = component p of eigenvector j,
// each normalised so its largest-|.| component is positive (the oracle's
// convention; Eigen's signs are arbitrary).  Work buffers from CmaDev.
// Returns the number of sweeps used, or < 0 on error.
// warm_B (optional, dp x dp): previous eigenvectors; Jacobi then runs on
// B^T A B (nearly diagonal when A changed little) and returns B V.
int sym_eig_jacobi(CmaDev& w, const double* A, int d, double* evals_host_min, double* vecs, double* evals,
                   cudaStream_t s, const double* warm_B = nullptr);

}  // namespace evorl_b200
