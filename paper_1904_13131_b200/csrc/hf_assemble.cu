// Element-matrix assembly for the matrix-based baseline (operators.py:436-491,
// AssembledTangent 494-516): the paper's matrix-free vs
// matrix-based comparison on B200.
//
// One thread block per cell builds the (nloc*dim)^2 element matrix
//   a[(n,c),(m,d)] = sum_q JxW_q ( B_k(n,c) M_kl B_l(m,d) + delta_cd gs_n . tau . gs_m )
// from the tensor4 q-point cache (tau, packed Voigt M, s_inv, JxW), with
// gs_n = (unit gradient of N_n) . s_inv the spatial gradient and B the
// engineering-strain Voigt operator (material.py:161-192).  Rows/columns are
// local DoFs n*dim + c (nodes lexicographic, x fastest), as the reference's
// vdofs (operators.py:474).  The global CSR (constrained rows/columns cleared,
// unit diagonal) is formed on the host side of the boundary and multiplied
// with cuSPARSE.
#include "hf_cell.cuh"
#include "hf_dispatch.h"

namespace hf {

template <int DIM, int N>
__global__ void __launch_bounds__(256) k_assemble_local(const CellArgs a, double* __restrict__ vals) {
  constexpr int NQ = Cfg<DIM, N>::NQ;  // nloc == nq
  constexpr int NV = DIM * (DIM + 1) / 2;
  constexpr int NM = NV * (NV + 1) / 2;
  constexpr int NF = CacheFields<DIM, TENSOR4>::NF;  // tensor4 cache fields (JxW folded in)
  constexpr int NLD = NQ * DIM;
  __shared__ double gs[NQ][NQ][DIM];  // [q][n][j]
  __shared__ double Mq[NQ][NV][NV];
  __shared__ double tq[NQ][DIM][DIM];
  __shared__ double wq[NQ];
  __shared__ double sq[NQ][DIM][DIM];
  const long long e = blockIdx.x;
  using TL = TileLayout<DIM, N>;
  for (int q = threadIdx.x; q < NQ; q += blockDim.x) {
    double f[NF];
    for (int k = 0; k < NF; ++k) f[k] = a.cache[TL::index(e, q, k, NF)];
    for (int i = 0; i < DIM; ++i)
      for (int j = 0; j < DIM; ++j) {
        tq[q][i][j] = f[hf_slot<DIM>(i, j)];
        sq[q][i][j] = f[NV + NM + i * DIM + j];
      }
    for (int r = 0; r < NV; ++r)
      for (int c = 0; c < NV; ++c) Mq[q][r][c] = f[NV + (r <= c ? hf_triu<NV>(r, c) : hf_triu<NV>(c, r))];
    wq[q] = 1.0;  // JxW is folded into the cached tau and M (CacheFields)
  }
  __syncthreads();
  // spatial gradients of every node basis at every q-point
  for (int id = threadIdx.x; id < NQ * NQ; id += blockDim.x) {
    const int q = id / NQ, n = id - q * NQ;
    int qi[3] = {q % N, (q / N) % N, DIM == 3 ? q / (N * N) : 0};
    int ni[3] = {n % N, (n / N) % N, DIM == 3 ? n / (N * N) : 0};
    double g[DIM];
    for (int ax = 0; ax < DIM; ++ax) {
      double p = 1.0;
      for (int k = 0; k < DIM; ++k) p *= (k == ax) ? a.tab.D[ni[k] * N + qi[k]] : a.tab.V[ni[k] * N + qi[k]];
      g[ax] = p;
    }
    for (int j = 0; j < DIM; ++j) {
      double s = 0.0;
      for (int ax = 0; ax < DIM; ++ax) s = fma(g[ax], sq[q][ax][j], s);
      gs[q][n][j] = s;
    }
  }
  __syncthreads();
  for (int id = threadIdx.x; id < NLD * NLD; id += blockDim.x) {
    const int r = id / NLD, s = id - r * NLD;
    const int n = r / DIM, c = r - n * DIM;
    const int m = s / DIM, d = s - m * DIM;
    double acc = 0.0;
    for (int q = 0; q < NQ; ++q) {
      double bn[NV], bm[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const int ka = HfSym<DIM>::a(k), kb = HfSym<DIM>::b(k);
        if (ka == kb) {
          bn[k] = (c == ka) ? gs[q][n][ka] : 0.0;
          bm[k] = (d == ka) ? gs[q][m][ka] : 0.0;
        } else {
          bn[k] = (c == ka ? gs[q][n][kb] : 0.0) + (c == kb ? gs[q][n][ka] : 0.0);
          bm[k] = (d == ka ? gs[q][m][kb] : 0.0) + (d == kb ? gs[q][m][ka] : 0.0);
        }
      }
      double v = 0.0;
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        double t = 0.0;
#pragma unroll
        for (int l = 0; l < NV; ++l) t = fma(Mq[q][k][l], bm[l], t);
        v = fma(bn[k], t, v);
      }
      if (c == d) {
#pragma unroll
        for (int j = 0; j < DIM; ++j) {
          double t = 0.0;
#pragma unroll
          for (int k = 0; k < DIM; ++k) t = fma(tq[q][j][k], gs[q][m][k], t);
          v = fma(gs[q][n][j], t, v);
        }
      }
      acc = fma(v, wq[q], acc);
    }
    vals[e * (long long)(NLD * NLD) + id] = acc;
  }
}

// global DoF of every local DoF of every cell (operators.py:474 vdofs)
__global__ void k_cell_dofs(const HfLattice lat, int dim, int degree, long long* __restrict__ dofs) {
  const int n1 = degree + 1;
  const int nloc = dim == 3 ? n1 * n1 * n1 : n1 * n1;
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= lat.n_el * nloc * dim) return;
  const long long e = id / (nloc * dim);
  const int r = (int)(id - e * nloc * dim);
  const int n = r / dim, c = r - n * dim;
  long long rr = e;
  const int ex = (int)(rr % lat.cells[0]);
  rr /= lat.cells[0];
  const int ey = (int)(rr % lat.cells[1]);
  const int ez = dim == 3 ? (int)(rr / lat.cells[1]) : 0;
  const int i = n % n1, j = (n / n1) % n1, k = dim == 3 ? n / (n1 * n1) : 0;
  const long long node = (long long)(ex * degree + i) +
                         (long long)lat.nodes[0] * ((long long)(ey * degree + j) +
                                                    (long long)lat.nodes[1] * (long long)(ez * degree + k));
  dofs[id] = node * dim + c;
}

template <int DIM, int N>
static cudaError_t assemble_n(const CellArgs& a, double* vals, cudaStream_t s) {
  if (a.lat.n_el == 0) return cudaSuccess;
  k_assemble_local<DIM, N><<<(unsigned)a.lat.n_el, 256, 0, s>>>(a, vals);
  return cudaGetLastError();
}

cudaError_t launch_assemble(int dim, int n1, const CellArgs& a, double* vals, cudaStream_t s) {
  if (dim == 2) {
    switch (n1) {
      case 2: return assemble_n<2, 2>(a, vals, s);
      case 3: return assemble_n<2, 3>(a, vals, s);
      case 4: return assemble_n<2, 4>(a, vals, s);
      case 5: return assemble_n<2, 5>(a, vals, s);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (n1) {
    case 2: return assemble_n<3, 2>(a, vals, s);
    case 3: return assemble_n<3, 3>(a, vals, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_cell_dofs(const HfLattice& lat, int dim, int degree, long long* dofs, cudaStream_t s) {
  const int n1 = degree + 1;
  const long long n = lat.n_el * (dim == 3 ? n1 * n1 * n1 : n1 * n1) * dim;
  if (n == 0) return cudaSuccess;
  k_cell_dofs<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(lat, dim, degree, dofs);
  return cudaGetLastError();
}

}  // namespace hf
