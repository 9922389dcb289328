// cma.cu -- CMA-ES on the device, restating
// proj/src/ec.cpp:191-288.
//
//  * K5 ask: Y = ((z .* D^T) B^T) sigma + mean -- z regenerated from the ask
//    key, one FP64 tensor-core (DMMA) NT GEMM with the sigma/mean epilogue.
//  * K6 tell: y_top, yw, mean, the CSA path (two GEMVs with B), pc, and the
//    rank-mu update  sum_i w_i y_i y_i^T  as a K = mu DMMA GEMM whose epilogue
//    blends  (1-c1-cmu) C + c1 (pc pc^T + dh C) + cmu rank_mu  in one pass;
//    then symmetrise.
//  * K7 eig: blocked cyclic Jacobi.  Blocks of 32 indices are paired
//    round-robin; each 64x64 block-pair subproblem is diagonalised in shared
//    memory by a parallel scalar Jacobi (32 disjoint rotations per round), and
//    its 64x64 rotation U is applied to the columns and rows of A and to the
//    columns of V by DMMA kernels (all pairs of a round at once: they are
//    disjoint).  Sweeps repeat until the off-diagonal mass is < 1e-28 of the
//    total (fp64 round-off level).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "cma.cuh"

namespace evorl_b200 {

void count_launch(int n);
cudaError_t run_rank(const double* keys, int n, int desc, int* rank, cudaStream_t s);

EVB_DEV void dmma_acc(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

static unsigned nblk(long long n, int t) { return (unsigned)std::max(1LL, (n + t - 1) / t); }

// ------------------------------------------------------------------ GEMM
constexpr int GBM = 64, GBN = 64, GBK = 16, GPAD = 4;

__global__ void __launch_bounds__(256) k_gemm_nt(int M, int N, int K, const double* __restrict__ A,
                                                 long long lda, const double* __restrict__ B, long long ldb,
                                                 const GemmEpi epi) {
  __shared__ double As[GBK][GBM + GPAD];
  __shared__ double Bs[GBK][GBN + GPAD];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int lr = tid >> 2, kq = (tid & 3) * 4;
  for (int k0 = 0; k0 < K; k0 += GBK) {
    const int gm = m0 + lr, gn = n0 + lr;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int gk = k0 + kq + q;
      As[kq + q][lr] = (gm < M && gk < K) ? A[(long long)gm * lda + gk] : 0.0;
      Bs[kq + q][lr] = (gn < N && gk < K) ? B[(long long)gn * ldb + gk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < GBK; kk += 4) {
      double a[4], b[2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) a[mt] = As[kk + t][wm + mt * 8 + g];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) b[nt] = Bs[kk + t][wn + nt * 8 + g];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) dmma_acc(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int m = m0 + wm + mt * 8 + g, n = n0 + wn + nt * 8 + 2 * t + i;
        if (m >= M || n >= N) continue;
        const double v = acc[mt][nt][i];
        const long long o = (long long)m * epi.ldo + n;
        if (epi.mode == GEMM_ASK) {
          epi.out[o] = dadd(dmul(v, epi.sigma), epi.mean[n]);
        } else if (epi.mode == GEMM_RANKMU) {
          const double c = epi.Cold[o];
          epi.out[o] = dadd(dadd(dmul(epi.a, c), dmul(epi.c1, dadd(dmul(epi.pc[m], epi.pc[n]), dmul(epi.dh, c)))),
                            dmul(epi.cmu, v));
        } else {
          epi.out[o] = v;
        }
      }
}

cudaError_t run_gemm_nt(int M, int N, int K, const double* A, long long lda, const double* B, long long ldb,
                        const GemmEpi& epi, cudaStream_t s) {
  dim3 grid((N + GBN - 1) / GBN, (M + GBM - 1) / GBM);
  k_gemm_nt<<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, epi);
  count_launch(1);
  return cudaGetLastError();
}

// ------------------------------------------------------------- ask / tell
// zD[i][j] = z[i][j] * D[j], z = gaussian_matrix(key, n, d) (proj/src/ec.cpp:228-229)
__global__ void k_cma_zD(DKey key, int n, int d, const double* D, double* zD) {
  const long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x;  // Box-Muller block
  const long long total = (long long)n * d;
  if (2 * b >= total) return;
  double c, sn;
  normal_pair(key, (uint64_t)b, c, sn);
  const long long i0 = 2 * b;
  zD[i0] = dmul(c, D[i0 % d]);
  if (i0 + 1 < total) zD[i0 + 1] = dmul(sn, D[(i0 + 1) % d]);
}
cudaError_t run_cma_zD(DKey key, int n, int d, const double* D, double* zD, cudaStream_t s) {
  const long long total = (long long)n * d;
  k_cma_zD<<<nblk((total + 1) / 2, 256), 256, 0, s>>>(key, n, d, D, zD);
  count_launch(1);
  return cudaGetLastError();
}

// y_top[i] = (cand[order[i]] - mean) / sigma, stored transposed; wyT = w_i * y
// (proj/src/ec.cpp:243-245, :264-266)
__global__ void k_cma_ytop(const double* cand, const int* order, int mu, int d, const double* mean,
                           double sigma, const double* w, double* ytT, double* wyT) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)mu * d) return;
  const int i = (int)(idx / d), p = (int)(idx % d);
  const double y = ddiv(dsub(cand[(long long)order[i] * d + p], mean[p]), sigma);
  ytT[(long long)p * mu + i] = y;
  wyT[(long long)p * mu + i] = dmul(w[i], y);
}
cudaError_t run_cma_ytop(const double* cand, const int* order, int mu, int d, const double* mean, double sigma,
                         const double* w, double* ytT, double* wyT, cudaStream_t s) {
  k_cma_ytop<<<nblk((long long)mu * d, 256), 256, 0, s>>>(cand, order, mu, d, mean, sigma, w, ytT, wyT);
  count_launch(1);
  return cudaGetLastError();
}

// yw = y_top^T w (sequential i), mean += sigma * yw (proj/src/ec.cpp:246-248)
__global__ void k_cma_yw_mean(const double* ytT, const double* w, int mu, int d, double sigma, double* yw,
                              double* mean) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= d) return;
  double acc = 0.0;
  for (int i = 0; i < mu; ++i) acc = dadd(acc, dmul(ytT[(long long)p * mu + i], w[i]));
  yw[p] = acc;
  mean[p] = dadd(mean[p], dmul(sigma, acc));
}
cudaError_t run_cma_yw_mean(const double* ytT, const double* w, int mu, int d, double sigma, double* yw,
                            double* mean, cudaStream_t s) {
  k_cma_yw_mean<<<nblk(d, 256), 256, 0, s>>>(ytT, w, mu, d, sigma, yw, mean);
  count_launch(1);
  return cudaGetLastError();
}

// t1[j] = (B^T yw)[j] / max(D[j], 1e-300) (proj/src/ec.cpp:251-252): column
// sums, coalesced across j.
__global__ void k_cma_gemv_t(const double* B, int dp, int d, const double* yw, const double* D, double* t1) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  double acc = 0.0;
  for (int p = 0; p < d; ++p) acc = fma(B[(long long)p * dp + j], yw[p], acc);
  t1[j] = ddiv(acc, D[j] > 1e-300 ? D[j] : 1e-300);
}
cudaError_t run_cma_gemv_t(const double* B, int dp, int d, const double* yw, const double* D, double* t1,
                           cudaStream_t s) {
  k_cma_gemv_t<<<nblk(d, 128), 128, 0, s>>>(B, dp, d, yw, D, t1);
  count_launch(1);
  return cudaGetLastError();
}

// out[p] = (B v)[p]: one warp per row, fixed-order butterfly
__global__ void k_cma_gemv(const double* B, int dp, int d, const double* v, double* out) {
  const int p = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (p >= d) return;
  double acc = 0.0;
  for (int j = lane; j < d; j += 32) acc = fma(B[(long long)p * dp + j], v[j], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) out[p] = acc;
}
cudaError_t run_cma_gemv(const double* B, int dp, int d, const double* v, double* out, cudaStream_t s) {
  k_cma_gemv<<<nblk(d, 8), 256, 0, s>>>(B, dp, d, v, out);
  count_launch(1);
  return cudaGetLastError();
}

// ps update and ||ps||^2 (proj/src/ec.cpp:253-255)
__global__ void k_cma_ps(double* ps, const double* cih, int d, double cs, double cps, double* red) {
  __shared__ double sh[256];
  const int t = threadIdx.x;
  const int chunk = (d + 255) / 256;
  double s = 0.0;
  for (int p = t * chunk; p < min(d, (t + 1) * chunk); ++p) {
    const double v = dadd(dmul(1.0 - cs, ps[p]), dmul(cps, cih[p]));
    ps[p] = v;
    s = dadd(s, dmul(v, v));
  }
  sh[t] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (t < w) sh[t] = dadd(sh[t], sh[t + w]);
    __syncthreads();
  }
  if (t == 0) red[0] = sh[0];
}
cudaError_t run_cma_ps(double* ps, const double* cih, int d, double cs, double cps, double* red, cudaStream_t s) {
  k_cma_ps<<<1, 256, 0, s>>>(ps, cih, d, cs, cps, red);
  count_launch(1);
  return cudaGetLastError();
}

__global__ void k_cma_pc(double* pc, const double* yw, int d, double cc, double cpc) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < d) pc[p] = dadd(dmul(1.0 - cc, pc[p]), dmul(cpc, yw[p]));
}
cudaError_t run_cma_pc(double* pc, const double* yw, int d, double cc, double cpc, cudaStream_t s) {
  k_cma_pc<<<nblk(d, 256), 256, 0, s>>>(pc, yw, d, cc, cpc);
  count_launch(1);
  return cudaGetLastError();
}

// C = 0.5 (T + T^T) (proj/src/ec.cpp:277)
__global__ void k_cma_symmetrize(const double* T, double* C, int d, int dp) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)d * d) return;
  const int r = (int)(idx / d), c = (int)(idx % d);
  C[(long long)r * dp + c] = dmul(0.5, dadd(T[(long long)r * dp + c], T[(long long)c * dp + r]));
}
cudaError_t run_cma_symmetrize(const double* T, double* C, int d, int dp, cudaStream_t s) {
  k_cma_symmetrize<<<nblk((long long)d * d, 256), 256, 0, s>>>(T, C, d, dp);
  count_launch(1);
  return cudaGetLastError();
}

__global__ void k_cma_sqrt_pos(const double* ev, double* D, int d) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d) D[i] = sqrt(ev[i] > 0.0 ? ev[i] : 0.0);
}
cudaError_t run_cma_sqrt_pos(const double* ev, double* D, int d, cudaStream_t s) {
  k_cma_sqrt_pos<<<nblk(d, 256), 256, 0, s>>>(ev, D, d);
  count_launch(1);
  return cudaGetLastError();
}

__global__ void k_cma_add_diag(double* C, int d, int dp, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d) C[(long long)i * dp + i] = dadd(C[(long long)i * dp + i], v);
}
cudaError_t run_cma_add_diag(double* C, int d, int dp, double v, cudaStream_t s) {
  k_cma_add_diag<<<nblk(d, 256), 256, 0, s>>>(C, d, dp, v);
  count_launch(1);
  return cudaGetLastError();
}

// ============================================================ Jacobi eig
constexpr int JB = 32;      // block size; block pairs are 64 x 64
constexpr int JP = 2 * JB;  // pair dimension

// Rotation zeroing S[p][q] (same formulas as the oracle's cyclic Jacobi).
EVB_DEV void jrot(double app, double aqq, double apq, double& c, double& s) {
  if (apq == 0.0) {
    c = 1.0;
    s = 0.0;
    return;
  }
  const double theta = (aqq - app) / (2.0 * apq);
  const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
  c = 1.0 / sqrt(t * t + 1.0);
  s = t * c;
}

// circle-method pair k of round r over n (even) indices
EVB_HD void rr_pair(int n, int r, int k, int& a, int& b) {
  if (k == 0) {
    a = r;
    b = n - 1;
  } else {
    a = (r + k) % (n - 1);
    b = (r - k + (n - 1)) % (n - 1);
  }
  if (a > b) {
    const int tmp = a;
    a = b;
    b = tmp;
  }
}

// One CTA per block pair: diagonalise the 64x64 subproblem in shared memory.
// Threshold Jacobi: a pair whose off-diagonal mass is already below `thr`
// (the global stop tolerance split over all block pairs) is skipped -- its
// rotation is the identity, flagged in skipf so the apply kernels leave its
// rows / columns alone; convergence is still judged on the whole matrix.
__global__ void __launch_bounds__(256) k_jacobi_pairs(const double* __restrict__ A, int dp, int nb, int round,
                                                      double* __restrict__ Uout, int max_sweeps, double thr,
                                                      int* __restrict__ skipf) {
  extern __shared__ __align__(16) double jsm[];
  double(*S)[JP + 1] = reinterpret_cast<double(*)[JP + 1]>(jsm);
  double(*Us)[JP + 1] = reinterpret_cast<double(*)[JP + 1]>(jsm + JP * (JP + 1));
  __shared__ double rc[JB], rs[JB];
  __shared__ double red[2][256];
  const int pair = blockIdx.x, tid = threadIdx.x;
  int P, Q;
  rr_pair(nb, round, pair, P, Q);
  for (int i = tid; i < JP * JP; i += 256) {
    const int r = i / JP, c = i % JP;
    const int gr = r < JB ? P * JB + r : Q * JB + r - JB;
    const int gc = c < JB ? P * JB + c : Q * JB + c - JB;
    S[r][c] = A[(long long)gr * dp + gc];
    Us[r][c] = r == c ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = tid; i < JP * JP; i += 256) {
      const double v = S[i / JP][i % JP];
      tot += v * v;
      if (i / JP != i % JP) off += v * v;
    }
    red[0][tid] = off;
    red[1][tid] = tot;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (tid < w) {
        red[0][tid] += red[0][tid + w];
        red[1][tid] += red[1][tid + w];
      }
      __syncthreads();
    }
    const bool done = red[0][0] <= 1e-30 * red[1][0] || red[0][0] == 0.0;
    const bool skip = sweep == 0 && (done || red[0][0] <= thr);
    __syncthreads();
    if (sweep == 0 && tid == 0) skipf[pair] = skip ? 1 : 0;
    if (skip) return;
    if (done) break;
    for (int r = 0; r < JP - 1; ++r) {
      const int k = tid >> 3, sub = tid & 7;  // 32 pairs x 8 threads
      int p, q;
      rr_pair(JP, r, k, p, q);
      if (sub == 0) jrot(S[p][p], S[q][q], S[p][q], rc[k], rs[k]);
      __syncthreads();
      const double c = rc[k], s = rs[k];
      // columns p, q of S and of U (rows strided over the 8 threads)
      for (int i = sub; i < JP; i += 8) {
        const double xp = S[i][p], xq = S[i][q];
        S[i][p] = c * xp - s * xq;
        S[i][q] = s * xp + c * xq;
        const double up = Us[i][p], uq = Us[i][q];
        Us[i][p] = c * up - s * uq;
        Us[i][q] = s * up + c * uq;
      }
      __syncthreads();
      // rows p, q of S
      for (int j = sub; j < JP; j += 8) {
        const double xp = S[p][j], xq = S[q][j];
        S[p][j] = c * xp - s * xq;
        S[q][j] = s * xp + c * xq;
      }
      __syncthreads();
    }
  }
  double* Ug = Uout + (long long)pair * JP * JP;
  for (int i = tid; i < JP * JP; i += 256) Ug[i] = Us[i / JP][i % JP];
}

// M[:, PQ] <- M[:, PQ] * U  (cols=1)   or   M[PQ, :] <- U^T * M[PQ, :]  (cols=0)
// for every pair of the round; one CTA per (64-row/col tile, pair); DMMA.
__global__ void __launch_bounds__(256) k_jacobi_apply(double* __restrict__ M, int dp, int nb, int round,
                                                      const double* __restrict__ U, int cols) {
  extern __shared__ __align__(16) double jsm[];
  double(*Ts)[JP + 2] = reinterpret_cast<double(*)[JP + 2]>(jsm);  // cols: [row][k], rows: [k][col]
  double(*Us)[JP + 2] = reinterpret_cast<double(*)[JP + 2]>(jsm + JP * (JP + 2));
  const int pair = blockIdx.y, tile0 = blockIdx.x * JP, tid = threadIdx.x;
  int P, Q;
  rr_pair(nb, round, pair, P, Q);
  const double* Ug = U + (long long)pair * JP * JP;
  for (int i = tid; i < JP * JP; i += 256) {
    const int a = i / JP, b = i % JP;
    Us[a][b] = Ug[i];
    if (cols) {  // Ts[row a][k b] = M[tile0 + a][idx(b)]
      const int gc = b < JB ? P * JB + b : Q * JB + b - JB;
      Ts[a][b] = M[(long long)(tile0 + a) * dp + gc];
    } else {  // Ts[k a][col b] = M[idx(a)][tile0 + b]
      const int gr = a < JB ? P * JB + a : Q * JB + a - JB;
      Ts[a][b] = M[(long long)gr * dp + tile0 + b];
    }
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
  for (int k0 = 0; k0 < JP; k0 += 4) {
    double a[4], b[2];
    if (cols) {  // out[r][n] = sum_k Ts[r][k] U[k][n]
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) a[mt] = Ts[wm + mt * 8 + g][k0 + t];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) b[nt] = Us[k0 + t][wn + nt * 8 + g];
    } else {  // out[i][c] = sum_k U[k][i] Ts[k][c]
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) a[mt] = Us[k0 + t][wm + mt * 8 + g];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) b[nt] = Ts[k0 + t][wn + nt * 8 + g];
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) dmma_acc(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
  }
  __syncthreads();
#pragma unroll
  for (int mt = 0; mt < 4; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r = wm + mt * 8 + g, n = wn + nt * 8 + 2 * t + i;
        if (cols) {
          const int gc = n < JB ? P * JB + n : Q * JB + n - JB;
          M[(long long)(tile0 + r) * dp + gc] = acc[mt][nt][i];
        } else {
          const int gr = r < JB ? P * JB + r : Q * JB + r - JB;
          M[(long long)gr * dp + tile0 + n] = acc[mt][nt][i];
        }
      }
}

// 64x64x64 DMMA tile product on shared-memory operands (row stride JP + 2):
// acc = A * B, or A^T * B when transA (A read as A[k][m]).  8 warps, each a
// 32 x 16 output tile (4 x 2 m8n8 fragments).
EVB_DEV void jtile_gemm(const double (*As)[JP + 2], bool transA, const double (*Bs)[JP + 2],
                        double (&acc)[4][2][2], int wm, int wn, int g, int t) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll 4
  for (int k0 = 0; k0 < JP; k0 += 4) {
    double a[4], b[2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) a[mt] = transA ? As[k0 + t][wm + mt * 8 + g] : As[wm + mt * 8 + g][k0 + t];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) b[nt] = Bs[k0 + t][wn + nt * 8 + g];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) dmma_acc(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
  }
}

// W <- J^T W J for the round's block-diagonal rotation J (the pairs' U), one
// CTA per upper-triangle tile (pair a <= pair b):
//   Y = U_a^T (W[PQ_a, PQ_b] U_b)  ->  W[PQ_a, PQ_b] and, transposed, W[PQ_b, PQ_a].
// Replaces the column pass + row pass: W stays exactly symmetric, each entry is
// read and written once per round and the flops halve.
__global__ void __launch_bounds__(256) k_jacobi_apply_sym(double* __restrict__ W, int dp, int nb, int round,
                                                          const double* __restrict__ U,
                                                          const int* __restrict__ skipf) {
  extern __shared__ __align__(16) double jsm[];
  double(*Ts)[JP + 2] = reinterpret_cast<double(*)[JP + 2]>(jsm);
  double(*Ua)[JP + 2] = reinterpret_cast<double(*)[JP + 2]>(jsm + JP * (JP + 2));
  double(*Ub)[JP + 2] = reinterpret_cast<double(*)[JP + 2]>(jsm + 2 * JP * (JP + 2));
  const int np = nb / 2, tid = threadIdx.x;
  int rem = blockIdx.x, a = 0;  // tile -> (a, b), a <= b, row a holds np - a tiles
  while (rem >= np - a) {
    rem -= np - a;
    ++a;
  }
  const int b = a + rem;
  const bool ska = skipf[a] != 0, skb = skipf[b] != 0;  // identity rotations (U not written)
  if (ska && skb) return;                                 // I^T W I
  int Pa, Qa, Pb, Qb;
  rr_pair(nb, round, a, Pa, Qa);
  rr_pair(nb, round, b, Pb, Qb);
  const double* Uga = U + (long long)a * JP * JP;
  const double* Ugb = U + (long long)b * JP * JP;
  for (int i = tid; i < JP * JP; i += 256) {
    const int r = i / JP, c = i % JP;
    if (!ska) Ua[r][c] = Uga[i];
    if (!skb) Ub[r][c] = Ugb[i];
    const int gr = r < JB ? Pa * JB + r : Qa * JB + r - JB;
    const int gc = c < JB ? Pb * JB + c : Qb * JB + c - JB;
    Ts[r][c] = W[(long long)gr * dp + gc];
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;
  double acc[4][2][2];
  if (!skb) {
    jtile_gemm(Ts, false, Ub, acc, wm, wn, g, t);  // X = T U_b
    __syncthreads();
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) Ts[wm + mt * 8 + g][wn + nt * 8 + 2 * t + i] = acc[mt][nt][i];
    __syncthreads();
  }
  if (!ska) {
    jtile_gemm(Ua, true, Ts, acc, wm, wn, g, t);  // Y = U_a^T X
    __syncthreads();
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int i = 0; i < 2; ++i) Ts[wm + mt * 8 + g][wn + nt * 8 + 2 * t + i] = acc[mt][nt][i];
    __syncthreads();
  }
  for (int i = tid; i < JP * JP; i += 256) {  // coalesced: column index fastest
    const int r = i / JP, c = i % JP;
    const int gr = r < JB ? Pa * JB + r : Qa * JB + r - JB;
    const int gc = c < JB ? Pb * JB + c : Qb * JB + c - JB;
    W[(long long)gr * dp + gc] = Ts[r][c];
  }
  if (a != b) {
    for (int i = tid; i < JP * JP; i += 256) {  // transposed tile, row index of Y fastest
      const int c = i / JP, r = i % JP;
      const int gr = r < JB ? Pa * JB + r : Qa * JB + r - JB;
      const int gc = c < JB ? Pb * JB + c : Qb * JB + c - JB;
      W[(long long)gc * dp + gr] = Ts[r][c];
    }
  }
}

EVB_DEV void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
EVB_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
EVB_DEV void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// V <- V J (the accumulated rotations, columns of every pair): persistent
// CTAs walk (64-row tile, pair) work items with a 2-stage cp.async pipeline --
// the next item's V panel and U block stream into shared memory while the
// current one is multiplied on the FP64 tensor cores.
constexpr int JV_STAGE = 2 * JP * (JP + 2);  // doubles per stage: panel + U
__global__ void __launch_bounds__(256, 1) k_jacobi_apply_v(double* __restrict__ M, int dp, int nb, int round,
                                                           const double* __restrict__ U,
                                                           const int* __restrict__ skipf) {
  extern __shared__ __align__(16) double jsm[];
  const int np = nb / 2, ntr = dp / JP;
  const long long items = (long long)np * ntr;
  const int tid = threadIdx.x;
  auto issue = [&](long long item, int stage) {
    double(*Ts)[JP + 2] = reinterpret_cast<double(*)[JP + 2]>(jsm + stage * JV_STAGE);
    double(*Us)[JP + 2] = reinterpret_cast<double(*)[JP + 2]>(jsm + stage * JV_STAGE + JP * (JP + 2));
    const int pair = (int)(item / ntr), tile0 = (int)(item % ntr) * JP;
    int P, Q;
    rr_pair(nb, round, pair, P, Q);
    const double* Ug = U + (long long)pair * JP * JP;
    for (int c = tid; c < JP * JP / 2; c += 256) {  // 16-byte chunks
      const int r = c / (JP / 2), q = (c % (JP / 2)) * 2;
      cp_async16(&Us[r][q], Ug + r * JP + q);
      const int gc = q < JB ? P * JB + q : Q * JB + q - JB;
      cp_async16(&Ts[r][q], M + (long long)(tile0 + r) * dp + gc);
    }
    cp_async_commit();
  };
  const int warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;
  auto live = [&](long long i) {  // next work item at or after i whose pair rotated
    while (i < items && skipf[i / ntr]) i += gridDim.x;
    return i;
  };
  long long item = live(blockIdx.x);
  if (item < items) issue(item, 0);
  for (int it = 0; item < items; ++it) {
    const int st = it & 1;
    const long long next = live(item + gridDim.x);
    if (next < items) {
      issue(next, st ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double(*Ts)[JP + 2] = reinterpret_cast<const double(*)[JP + 2]>(jsm + st * JV_STAGE);
    const double(*Us)[JP + 2] = reinterpret_cast<const double(*)[JP + 2]>(jsm + st * JV_STAGE + JP * (JP + 2));
    double acc[4][2][2];
    jtile_gemm(Ts, false, Us, acc, wm, wn, g, t);
    const int pair = (int)(item / ntr), tile0 = (int)(item % ntr) * JP;
    int P, Q;
    rr_pair(nb, round, pair, P, Q);
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int r = wm + mt * 8 + g, n = wn + nt * 8 + 2 * t;
        const int gc = n < JB ? P * JB + n : Q * JB + n - JB;
        *reinterpret_cast<double2*>(M + (long long)(tile0 + r) * dp + gc) =
            make_double2(acc[mt][nt][0], acc[mt][nt][1]);
      }
    __syncthreads();  // this stage is refilled two items later
    item = next;
  }
}

// off-diagonal / total squared mass of the leading d x d block
__global__ void k_offdiag(const double* A, int d, int dp, double* red) {
  __shared__ double s0[256], s1[256];
  const int t = threadIdx.x;
  double off = 0.0, tot = 0.0;
  for (long long i = blockIdx.x * 256LL + t; i < (long long)d * d; i += (long long)gridDim.x * 256) {
    const int r = (int)(i / d), c = (int)(i % d);
    const double v = A[(long long)r * dp + c];
    tot += v * v;
    if (r != c) off += v * v;
  }
  s0[t] = off;
  s1[t] = tot;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (t < w) {
      s0[t] += s0[t + w];
      s1[t] += s1[t + w];
    }
    __syncthreads();
  }
  if (t == 0) {
    atomicAdd(&red[0], s0[0]);
    atomicAdd(&red[1], s1[0]);
  }
}

__global__ void k_eig_init(const double* A, double* W, double* V, int d, int dp) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)dp * dp) return;
  const int r = (int)(i / dp), c = (int)(i % dp);
  W[i] = (r < d && c < d) ? A[i] : (r == c ? 1.0 : 0.0);  // padding decoupled
  V[i] = r == c ? 1.0 : 0.0;
}
__global__ void k_eig_diag(const double* W, int dp, int d, double* ev) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < d) ev[i] = W[(long long)i * dp + i];
}
// vecs[:, j] = sign_j * V[:, order[j]] with the largest-|.| component positive
// (first maximum), evals_sorted[j] = ev[order[j]]; one warp per column.
__global__ void k_eig_finish(const double* V, int dp, int d, const int* rank, const double* ev, double* vecs,
                             double* evs) {
  const int j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= d) return;
  // column src with rank j
  __shared__ int src_s[8];
  if (lane == 0) src_s[threadIdx.x >> 5] = -1;
  __syncwarp();
  for (int i = lane; i < d; i += 32)
    if (rank[i] == j) src_s[threadIdx.x >> 5] = i;
  __syncwarp();
  const int src = src_s[threadIdx.x >> 5];
  double best = -1.0;
  int bi = 1 << 30;
  for (int p = lane; p < d; p += 32) {
    const double a = fabs(V[(long long)p * dp + src]);
    if (a > best) {
      best = a;
      bi = p;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) {
      best = ob;
      bi = oi;
    }
  }
  const double sg = V[(long long)bi * dp + src] < 0 ? -1.0 : 1.0;
  for (int p = lane; p < d; p += 32) vecs[(long long)p * dp + j] = sg * V[(long long)p * dp + src];
  if (lane == 0) evs[j] = ev[src];
}

// out = in^T over the dp x dp square (32x32 tiles through shared memory)
__global__ void k_transpose(const double* __restrict__ in, double* __restrict__ out, int dp) {
  __shared__ double tile[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) tile[j][threadIdx.x] = in[(long long)(by + j) * dp + bx + threadIdx.x];
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) out[(long long)(bx + j) * dp + by + threadIdx.x] = tile[threadIdx.x][j];
}

// W = 0.5 (T + T^T) on the d x d block, decoupled identity padding; V = I
__global__ void k_warm_init(double* T_then_V, double* W, int d, int dp) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)dp * dp) return;
  const int r = (int)(i / dp), c = (int)(i % dp);
  if (r < d && c < d) {
    W[i] = 0.5 * (T_then_V[i] + T_then_V[(long long)c * dp + r]);
  } else {
    W[i] = r == c ? 1.0 : 0.0;
  }
}
__global__ void k_eye(double* V, int dp) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < (long long)dp * dp) V[i] = (i / dp == i % dp) ? 1.0 : 0.0;
}

int sym_eig_jacobi(CmaDev& w, const double* A, int d, double* evals_min, double* vecs, double* evals,
                   cudaStream_t s, const double* warm_B) {
  const int dp = w.dp;
  const int nb = dp / JB;  // even: dp is a multiple of 64
  const long long n2 = (long long)dp * dp;
  const size_t sm_pairs = sizeof(double) * 2 * JP * (JP + 1), sm_apply = sizeof(double) * 2 * JP * (JP + 2);
  const size_t sm_sym = sizeof(double) * 3 * JP * (JP + 2);
  const size_t sm_v = sizeof(double) * 2 * JV_STAGE;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const unsigned v_grid = (unsigned)std::min<long long>((long long)nsm, (long long)(nb / 2) * (dp / JP));
  const long long np = nb / 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_jacobi_pairs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_pairs);
    cudaFuncSetAttribute(k_jacobi_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_apply);
    cudaFuncSetAttribute(k_jacobi_apply_v, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_v);
    cudaFuncSetAttribute(k_jacobi_apply_sym, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_sym);
    attr = true;
  }
  const double* Vsrc = w.V;
  static const bool trace = getenv("EVORL_EIG_TRACE") != nullptr;
  cudaEvent_t t0 = nullptr, t1 = nullptr, t2 = nullptr;
  if (trace) {
    cudaEventCreate(&t0);
    cudaEventCreate(&t1);
    cudaEventCreate(&t2);
    cudaEventRecord(t0, s);
  }
  if (warm_B != nullptr) {
    // warm start: W = B^T A B with B the previous eigenvectors (nearly
    // diagonal when A changed little), rotations accumulate into V, and the
    // final eigenvectors are B V.  Bt and Tt are scratch (dp x dp).
    k_transpose<<<dim3(dp / 32, dp / 32), dim3(32, 8), 0, s>>>(warm_B, w.Bt, dp);
    GemmEpi e{};
    e.mode = GEMM_STORE;
    e.ldo = dp;
    e.out = w.Tt;  // Tt[n][k] = sum_p B[p][n] A[k][p] = (B^T A)[n][k]
    run_gemm_nt(d, d, d, w.Bt, dp, A, dp, e, s);
    e.out = w.V;  // (B^T A B)[m][n] = sum_k Bt[m][k] Tt[n][k]
    run_gemm_nt(d, d, d, w.Bt, dp, w.Tt, dp, e, s);
    k_warm_init<<<nblk(n2, 256), 256, 0, s>>>(w.V, w.W, d, dp);  // symmetrise + pad
    k_eye<<<nblk(n2, 256), 256, 0, s>>>(w.V, dp);                // V = I
    count_launch(3);
  } else {
    k_eig_init<<<nblk(n2, 256), 256, 0, s>>>(A, w.W, w.V, d, dp);
    count_launch(1);
  }
  if (trace) cudaEventRecord(t1, s);
  int sweep = 0;
  std::vector<double> h(2);
  // Stop when the off-diagonal mass reaches fp64 round-off for this size
  // (each of the d^2 entries carries ~eps |lambda| of noise, so the floor of
  // off/tot is ~d eps^2), or when a sweep stops making progress.
  const double eps = 1.1102230246251565e-16;
  // ... or at off/tot = 1e-24: off-diagonal entries ~1e-12 of ||A||, far below
  // the fp32 tolerance the CMA path is held to (the extra sweeps to the fp64
  // noise floor only crawl, measured: EVORL_EIG_TRACE)
  const double tol = std::max(1e-24, 16.0 * d * eps * eps);
  double prev_off = INFINITY;
  // inner sweeps per block-pair visit: the outer sweeps revisit every pair, so
  // the subproblem need not be diagonalised exactly each time
  static const int inner_sweeps = getenv("EVORL_EIG_INNER") ? atoi(getenv("EVORL_EIG_INNER")) : 1;
  static const bool skip_pairs = !(getenv("EVORL_EIG_NOSKIP") && getenv("EVORL_EIG_NOSKIP")[0] == '1');
  // threshold Jacobi: also skip pairs holding less than skip_frac of the mean
  // per-pair share of the current off-diagonal mass (revisited next sweep)
  static const double skip_frac = getenv("EVORL_EIG_SKIPFRAC") ? atof(getenv("EVORL_EIG_SKIPFRAC")) : 0.0;
  for (; sweep < 30; ++sweep) {
    cudaMemsetAsync(w.red, 0, 2 * sizeof(double), s);
    k_offdiag<<<296, 256, 0, s>>>(w.W, d, dp, w.red);
    count_launch(1);
    cudaMemcpyAsync(h.data(), w.red, 2 * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
    if (trace) fprintf(stderr, "[eig]   sweep %d off/tot %.3e\n", sweep, h[1] > 0 ? h[0] / h[1] : 0.0);
    if (h[0] <= tol * h[1] || h[0] == 0.0) break;
    if (h[0] >= 0.9 * prev_off && h[0] <= 1e-20 * h[1]) break;  // stagnated at the noise floor
    prev_off = h[0];
    // per-pair skip threshold: if every block pair sat below it, the whole
    // off-diagonal mass would be under the stop tolerance
    const double npairs = 0.5 * nb * (nb - 1);
    const double thr = skip_pairs ? std::max(tol * h[1], skip_frac * h[0]) / npairs : -1.0;
    for (int r = 0; r < nb - 1; ++r) {
      k_jacobi_pairs<<<nb / 2, 256, sm_pairs, s>>>(w.W, dp, nb, r, w.U, inner_sweeps, thr, w.skipf);
      k_jacobi_apply_sym<<<(unsigned)(np * (np + 1) / 2), 256, sm_sym, s>>>(w.W, dp, nb, r, w.U, w.skipf);
      k_jacobi_apply_v<<<v_grid, 256, sm_v, s>>>(w.V, dp, nb, r, w.U, w.skipf);
      count_launch(3);
    }
  }
  if (trace) cudaEventRecord(t2, s);
  if (warm_B != nullptr) {  // eigenvectors = B_prev V: Tt = V^T, Bt = B_prev Tt^T
    k_transpose<<<dim3(dp / 32, dp / 32), dim3(32, 8), 0, s>>>(w.V, w.Tt, dp);
    GemmEpi e{};
    e.mode = GEMM_STORE;
    e.ldo = dp;
    e.out = w.Bt;
    run_gemm_nt(d, d, d, warm_B, dp, w.Tt, dp, e, s);
    count_launch(1);
    Vsrc = w.Bt;
  }
  k_eig_diag<<<nblk(d, 256), 256, 0, s>>>(w.W, dp, d, w.t1);
  count_launch(1);
  run_rank(w.t1, d, 0, w.order, s);  // ascending, ties by index
  k_eig_finish<<<nblk(d, 8), 256, 0, s>>>(Vsrc, dp, d, w.order, w.t1, vecs, evals);
  count_launch(1);
  cudaMemcpyAsync(evals_min, evals, sizeof(double), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return -1;
  if (cudaGetLastError() != cudaSuccess) return -1;
  if (trace) {
    float pre = 0, sw = 0;
    cudaEventElapsedTime(&pre, t0, t1);
    cudaEventElapsedTime(&sw, t1, t2);
    fprintf(stderr, "[eig] d=%d warm=%d sweeps=%d prologue=%.1f ms sweeps=%.1f ms (%.1f ms/sweep)\n", d,
            warm_B != nullptr, sweep, pre, sw, sweep ? sw / sweep : 0.f);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    cudaEventDestroy(t2);
  }
  return sweep;
}

}  // namespace evorl_b200
